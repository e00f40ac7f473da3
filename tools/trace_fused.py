"""Per-CTA timeline of one fused RK3 iteration (fdns_iteration): for each
stage the start (after the neighbourhood wait), first window ready and end,
relative to the earliest stamp.

    python tools/trace_fused.py [n] [variant]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd
from paper_1610_09146_b200 import _lib
from paper_1610_09146_b200.timeloop import IterationState, _fused_iteration

torch.cuda.set_device(0)
lib = _lib.load()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
variant = sys.argv[2] if len(sys.argv) > 2 else "SN"
g = fd.make_grid((n,) * 3, (2 * np.pi,) * 3)
c = fd.PhysicalConstants()
s = fd.taylor_green_init(g, c)
ev = fd.ResidualEvaluator(g, c, variant)
assert ev.fused_iteration
it = IterationState(s, saved=False)
scheme = fd.RKScheme(dt=3.385e-3)
for _ in range(3):
    _fused_iteration(it, scheme, ev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(3):
    lib.fdns_l2_flush(_lib.ptr(flush), flush.numel(), _lib.stream_handle())
    torch.cuda.synchronize()
    _lib.check(lib.fdns_debug_trace(1, None, 0))
    _fused_iteration(it, scheme, ev)
    torch.cuda.synchronize()
    N = 1024 * 9
    buf = (ctypes.c_uint64 * N)()
    _lib.check(lib.fdns_debug_trace(4, buf, N))
    t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 9).astype(np.float64)
    t = t[t[:, 0] > 0]
    t = (t - t[:, 0].min()) / 1e3
    print(f"{variant} {n}^3 rep {rep}: {len(t)} CTAs, end {t[:, 8].max():.1f} us")
    for st in range(3):
        a, b, e = t[:, 3 * st], t[:, 3 * st + 1], t[:, 3 * st + 2]
        print(f"  stage {st}: start med {np.median(a):6.1f} [{a.min():6.1f},{a.max():6.1f}]"
              f"  ready med {np.median(b):6.1f}  end med {np.median(e):6.1f}"
              f" [{e.min():6.1f},{e.max():6.1f}]  work med {np.median(e - b):5.1f}"
              f"  ramp med {np.median(b - a):5.1f}")
