"""Repeat a small run on several kernel paths and count bitwise mismatches
against the first path's first result (a race shows up as intermittent
differences).

    python tools/race_probe.py --variant SS --paths 2,5 --npts 12,16,20 --reps 20
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd
from paper_1610_09146_b200 import _lib
from paper_1610_09146_b200.diagnostics import state_from_conservative
from oracle import numpy_oracle as npo


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="SS")
    ap.add_argument("--paths", default="2,5")
    ap.add_argument("--npts", default="12,16,20")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--mode", default="run", choices=["run", "residual"])
    ap.add_argument("--pdl", type=int, default=1)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    lib = _lib.load()
    lib.fdns_set_pdl(a.pdl)
    npts = tuple(int(x) for x in a.npts.split(","))
    F = npo.manufactured(npts, npo.Consts())
    g = fd.make_grid(npts, (2 * np.pi,) * 3)
    C = fd.PhysicalConstants()
    cons = npo.interior(F[:5], 2)
    ref = None
    for p in map(int, a.paths.split(",")):
        lib.fdns_set_kernel_path(p)
        lib.fdns_set_tiled_grid(a.ctas)
        bad = 0
        for _ in range(a.reps):
            st = state_from_conservative(g, C, cons)
            if a.mode == "run":
                fd.run(st, fd.RKScheme(dt=1e-3), fd.ResidualEvaluator(g, C, a.variant), a.steps)
                out = g.interior(st.bundle[:5]).cpu().numpy()
            else:
                out = fd.assemble_residual(st, C, a.variant).interior_numpy()
            torch.cuda.synchronize()
            if ref is None:
                ref = out
            elif not np.array_equal(out, ref):
                bad += 1
                if bad <= 2:
                    d = np.argwhere(out != ref)
                    print(f"  {len(d)} differing values; fields {sorted(set(d[:, 0].tolist()))}; "
                          f"axis0 {sorted(set(d[:, 1].tolist()))}; axis1 {sorted(set(d[:, 2].tolist()))}; "
                          f"axis2 {sorted(set(d[:, 3].tolist()))}; max rel "
                          f"{np.max(np.abs(out - ref) / (np.abs(ref) + 1e-300)):.3e}", flush=True)
        print(f"path {p}: {bad}/{a.reps} differ", flush=True)
    lib.fdns_set_kernel_path(0)
    lib.fdns_set_tiled_grid(0)


if __name__ == "__main__":
    main()
