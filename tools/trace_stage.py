"""Per-CTA timeline of one SN stage (debug stamps): prologue, first-window
ramp, steady part, spread of exit times.

    python tools/trace_stage.py [n0 n1 n2]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd
from paper_1610_09146_b200 import _lib

torch.cuda.set_device(0)
lib = _lib.load()
npts = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (64, 64, 64)
variant = sys.argv[4] if len(sys.argv) > 4 else "SN"
wrap = int(sys.argv[5]) if len(sys.argv) > 5 else 7
g = fd.make_grid(npts, (2 * np.pi,) * 3)
c = fd.PhysicalConstants()
s = fd.taylor_green_init(g, c)
ev = fd.ResidualEvaluator(g, c, variant)
Y, Z = ev.workspace()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cold in (True, False):
    for _ in range(3):
        ev.stage(s.bundle, s.bundle, Y, 1e-3)
    torch.cuda.synchronize()
    _lib.check(lib.fdns_debug_trace(1, None, 0))
    if cold:
        lib.fdns_l2_flush(_lib.ptr(flush), flush.numel(), _lib.stream_handle())
    _lib.check(lib.fdns_stage(ev.plan.variant_id, _lib.ptr(s.bundle), _lib.ptr(s.bundle),
                              _lib.ptr(Y), ev.work_ptr, 1e-3, wrap, ev.problem,
                              _lib.stream_handle()))
    torch.cuda.synchronize()
    buf = (ctypes.c_uint64 * (1024 * 4))()
    _lib.check(lib.fdns_debug_trace(0, buf, 1024 * 4))
    raw = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 4).copy()
    ncta = int((raw[:, 0] > 0).sum())
    raw = raw[:ncta]
    smid = (raw[:, 0] >> np.uint64(48)).astype(int)
    raw[:, 0] &= np.uint64(0x0000FFFFFFFFFFFF)
    mask48 = np.uint64(0x0000FFFFFFFFFFFF)
    t = (raw & mask48).astype(np.float64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    print(f"{variant} {npts} {'cold' if cold else 'warm'} L2: {len(t)} CTAs")
    for k, name in enumerate(("entry", "prologue", "window ready", "exit")):
        print(f"  {name:13s} min {rel[:, k].min():7.2f}  median {np.median(rel[:, k]):7.2f}"
              f"  max {rel[:, k].max():7.2f} us")
    dur = rel[:, 3] - rel[:, 2]
    order = np.argsort(-dur)
    print("  slowest CTAs (cta, smid, steady us):",
          [(int(i), int(smid[i]), round(float(dur[i]), 1)) for i in order[:8]])
    print("  fastest CTAs:", [(int(i), int(smid[i]), round(float(dur[i]), 1)) for i in order[-5:]])
    # SM parity / die split
    for name, sel in (("even smid", smid % 2 == 0), ("odd smid", smid % 2 == 1),
                      ("smid<74", smid < 74), ("smid>=74", smid >= 74)):
        if sel.any():
            print(f"  {name:9s}: mean steady {dur[sel].mean():8.1f} us  max {dur[sel].max():8.1f}")
