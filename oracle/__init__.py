"""CPU oracle for the fdns hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the reference algorithm of arXiv
1610.09146's `fdns` package (the 4th-order compressible Navier-Stokes
residual for the Taylor-Green vortex plus the save-state RK3 update).  It is
the checker the GPU product is compared against, and the CPU baseline that
`bench.py --impl reference` times.  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s cpu-baseline leg may import it; the product package
(`paper_1610_09146_b200`) never does.

Two independent restatements live here:

* `numpy_oracle` -- vectorised numpy, brute-force "store every derivative"
  route (the reference's BL fill path plus the generated residual body).
* `c_oracle` -- a C99 + OpenMP point-kernel restatement ("compute every
  distinct derivative once per point", the reference's SN route), loaded
  with ctypes from `oracle/lib/libfdns_oracle.so`.

Both are pinned against golden vectors produced by the real reference
(`tests/golden/make_golden.py`, run in the build container where
`/root/reference` is importable); see `tests/test_oracle_golden.py`.
"""
