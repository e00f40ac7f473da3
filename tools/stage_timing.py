"""Per-variant fused-stage kernel time at several grid sizes (CUDA events,
L2 flushed between launches).

    python tools/stage_timing.py --sizes 64,128,256 --variants SN,SS,RA,BL
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1610_09146_b200 as fd
from paper_1610_09146_b200 import _lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,128,256")
    ap.add_argument("--variants", default="SN,SS,RA,BL")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--nopdl", action="store_true")
    ap.add_argument("--b2b", action="store_true",
                    help="also time 3 back-to-back stages (one RK step)")
    ap.add_argument("--path", type=int, default=0,
                    help="kernel family: 0 default, 1 point kernels, 2 single-group SN")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    lib = _lib.load()
    lib.fdns_set_kernel_path(a.path)
    lib.fdns_set_pdl(0 if a.nopdl else 1)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    c = fd.PhysicalConstants()
    out = {}
    for n in map(int, a.sizes.split(",")):
        g = fd.make_grid((n,) * 3, (2 * np.pi,) * 3)
        s = fd.taylor_green_init(g, c)
        for v in a.variants.split(","):
            ev = fd.ResidualEvaluator(g, c, v)
            Y, Z = ev.workspace()
            ts = []
            for r in range(a.reps + 2):
                lib.fdns_l2_flush(_lib.ptr(flush), flush.numel(), _lib.stream_handle())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ev.stage(s.bundle, s.bundle, Y, 1e-3)
                e1.record()
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            out[f"{v}@{n}"] = {"ms": ms, "pt_per_s": n ** 3 / (ms / 1e3)}
            extra = ""
            if a.b2b:
                bb = []
                for r in range(a.reps):
                    lib.fdns_l2_flush(_lib.ptr(flush), flush.numel(), _lib.stream_handle())
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    ev.stage(s.bundle, s.bundle, Y, 1e-3)
                    ev.stage(Y, s.bundle, Z, 1e-3)
                    ev.stage(Z, s.bundle, Y, 1e-3)
                    e1.record()
                    torch.cuda.synchronize()
                    bb.append(e0.elapsed_time(e1) / 3)
                extra = f"  3-stage b2b {np.median(bb) * 1e3:8.1f} us/stage"
            print(f"{v}@{n}: {ms*1e3:9.1f} us  {n**3/(ms/1e3):.3e} pt-stage/s{extra}", flush=True)
            del ev, Y, Z
        del s
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
