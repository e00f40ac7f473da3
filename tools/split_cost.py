"""Single-GPU cost of the multi-GPU stage split (SURVEY 8e overlap):
one fused stage over all planes vs the boundary-planes-first split that
`ResidualEvaluator.stage_exchanged` launches (the exchange itself omitted),
CUDA events, L2 flushed before each.

    python tools/split_cost.py --sizes 64,128 --variants SN,SS
    python tools/split_cost.py --grids 512x512x512,64x512x512 --variants SN,RA,SS,BL
      (a strong-scaling rank's slab of 512^3 on 8 GPUs as a one-GPU grid)
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd
from paper_1610_09146_b200 import _lib


def timed(fn, lib, flush, reps=20):
    ts = []
    for _ in range(reps):
        lib.fdns_l2_flush(_lib.ptr(flush), flush.numel(), _lib.stream_handle())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,128")
    ap.add_argument("--variants", default="SN,SS")
    ap.add_argument("--grids", default="", help="n0xn1xn2,... (overrides --sizes)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    lib = _lib.load()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    c = fd.PhysicalConstants()
    shapes = ([tuple(map(int, x.split("x"))) for x in a.grids.split(",")] if a.grids
              else [(n,) * 3 for n in map(int, a.sizes.split(","))])
    for npts in shapes:
        n = "x".join(map(str, npts))
        g = fd.make_grid(npts, (2 * np.pi,) * 3)
        for v in a.variants.split(","):
            s = fd.taylor_green_init(g, c)
            ev = fd.ResidualEvaluator(g, c, v)
            Y, Z = ev.workspace()
            X = s.bundle
            h = g.halo

            def full():
                ev.stage(X, X, Y, 1e-3)

            def split():   # stage_exchanged without the exchange
                ev.stage_boundary(X, X, Y, 1e-3)
                ev.stage_interior(X, X, Y, 1e-3)

            for f in (full, split):
                f()
            torch.cuda.synchronize()
            tf, ts = timed(full, lib, flush), timed(split, lib, flush)
            print(f"{v}@{n}: one launch {tf * 1e3:8.1f} us   split {ts * 1e3:8.1f} us "
                  f"(+{(ts / tf - 1) * 100:.0f}%)", flush=True)


if __name__ == "__main__":
    main()
