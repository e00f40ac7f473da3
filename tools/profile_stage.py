"""Run a few fused RK stages of chosen variants (for ncu captures).

    python tools/profile_stage.py --n 128 --variants SN,SS --stages 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1610_09146_b200 as fd


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--variants", default="SN")
    ap.add_argument("--stages", type=int, default=2)
    ap.add_argument("--path", type=int, default=0, help="fdns_set_kernel_path (A/B)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    from paper_1610_09146_b200 import _lib
    _lib.load().fdns_set_kernel_path(a.path)
    g = fd.make_grid((a.n,) * 3, (2 * np.pi,) * 3)
    c = fd.PhysicalConstants()
    for v in a.variants.split(","):
        s = fd.taylor_green_init(g, c)
        ev = fd.ResidualEvaluator(g, c, v)
        Y, Z = ev.workspace()
        Y.copy_(s.bundle)
        for _ in range(a.stages):
            ev.stage(Y, s.bundle, Z, 1e-3)   # a stage-1/2 workload (saved != input)
        torch.cuda.synchronize()
        print(v, "ok")
        del s, ev, Y, Z
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
