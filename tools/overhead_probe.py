"""Fixed vs per-plane cost of the SN stage: time one fused stage on
(n0, 64, 64) grids for several n0 (CUDA events, L2 flushed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd
from paper_1610_09146_b200 import _lib


def main():
    torch.cuda.set_device(0)
    lib = _lib.load()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    c = fd.PhysicalConstants()
    variant = sys.argv[1] if len(sys.argv) > 1 else "SN"
    for n0 in (16, 32, 64, 128, 256):
        g = fd.make_grid((n0, 64, 64), (2 * np.pi,) * 3)
        s = fd.taylor_green_init(g, c)
        ev = fd.ResidualEvaluator(g, c, variant)
        Y, Z = ev.workspace()
        ts = []
        for r in range(8):
            lib.fdns_l2_flush(_lib.ptr(flush), flush.numel(), _lib.stream_handle())
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ev.stage(s.bundle, s.bundle, Y, 1e-3)
            b.record()
            torch.cuda.synchronize()
            if r >= 3:
                ts.append(a.elapsed_time(b) * 1e3)
        print(f"{variant} n0={n0:4d}: {np.median(ts):8.1f} us")


if __name__ == "__main__":
    main()
