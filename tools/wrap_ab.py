"""A/B: ghost images written by the stage epilogue vs a separate ghost-only
wrap kernel after the stage (3 back-to-back stages, CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd
from paper_1610_09146_b200 import _lib

torch.cuda.set_device(0)
lib = _lib.load()
c = fd.PhysicalConstants()
for n in (64, 128, 256):
    g = fd.make_grid((n,) * 3, (2 * np.pi,) * 3)
    s = fd.taylor_green_init(g, c)
    for v in ("SN", "SS"):
        ev = fd.ResidualEvaluator(g, c, v)
        Y, Z = ev.workspace()
        pb = ev.problem
        res = {}
        for mode in ("epilogue", "kernel"):
            def stage(a, b):
                if mode == "epilogue":
                    _lib.check(lib.fdns_stage(ev.plan.variant_id, _lib.ptr(a), _lib.ptr(s.bundle),
                                              _lib.ptr(b), ev.work_ptr, 1e-3, 7, pb, _lib.stream_handle()))
                else:
                    _lib.check(lib.fdns_stage(ev.plan.variant_id, _lib.ptr(a), _lib.ptr(s.bundle),
                                              _lib.ptr(b), ev.work_ptr, 1e-3, 0, pb, _lib.stream_handle()))
                    _lib.check(lib.fdns_halo_wrap(_lib.ptr(b), 8, 7, pb, _lib.stream_handle()))
            for _ in range(2):
                stage(s.bundle, Y)
            torch.cuda.synchronize()
            ts = []
            for r in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                stage(s.bundle, Y); stage(Y, Z); stage(Z, Y)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3 / 3)
            res[mode] = float(np.median(ts))
        print(f"{v}@{n}: epilogue images {res['epilogue']:8.1f} us/stage, "
              f"separate wrap kernel {res['kernel']:8.1f} us/stage", flush=True)
        del ev, Y, Z
