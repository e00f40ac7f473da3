"""SN stage on (32, 64, 64): event time with / without an L2 flush before
the launch (cold vs warm ramp)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd
from paper_1610_09146_b200 import _lib

torch.cuda.set_device(0)
lib = _lib.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
c = fd.PhysicalConstants()
for n0 in (32, 64):
    g = fd.make_grid((n0, 64, 64), (2 * np.pi,) * 3)
    s = fd.taylor_green_init(g, c)
    ev = fd.ResidualEvaluator(g, c, "SN")
    Y, Z = ev.workspace()
    for flushing in (True, False):
        ts = []
        for r in range(10):
            if flushing:
                lib.fdns_l2_flush(_lib.ptr(flush), flush.numel(), _lib.stream_handle())
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ev.stage(s.bundle, s.bundle, Y, 1e-3)
            b.record()
            torch.cuda.synchronize()
            if r >= 3:
                ts.append(a.elapsed_time(b) * 1e3)
        print(f"n0={n0} flush={flushing}: {np.median(ts):7.1f} us", flush=True)
    # back-to-back stages (graph-like): 10 stages between one event pair
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for r in range(10):
        ev.stage(s.bundle, s.bundle, Y, 1e-3)
    b.record()
    torch.cuda.synchronize()
    print(f"n0={n0} back-to-back: {a.elapsed_time(b) * 1e3 / 10:7.1f} us/stage", flush=True)
