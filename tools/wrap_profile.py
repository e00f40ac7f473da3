"""One SN stage at 256^3 with wrap_mask 7 and 0 (for an ncu A/B of the
ghost-image stores).

    python tools/wrap_profile.py [n]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd
from paper_1610_09146_b200 import _lib

torch.cuda.set_device(0)
lib = _lib.load()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = fd.make_grid((n,) * 3, (2 * np.pi,) * 3)
c = fd.PhysicalConstants()
s = fd.taylor_green_init(g, c)
ev = fd.ResidualEvaluator(g, c, "SN")
Y, Z = ev.workspace()
for wrap in (7, 0):
    _lib.check(lib.fdns_stage(ev.plan.variant_id, _lib.ptr(Y if False else s.bundle),
                              _lib.ptr(s.bundle), _lib.ptr(Y), ev.work_ptr, 1e-3, wrap,
                              ev.problem, _lib.stream_handle()))
    torch.cuda.synchronize()
print("ok")
