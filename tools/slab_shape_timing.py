"""One rank's share of config C5 on 8 GPUs (1024^3 / 8 = 128 x 1024 x 1024)
as a single-GPU problem: fused-stage time per variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd

torch.cuda.set_device(0)
c = fd.PhysicalConstants()
npts = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "128,1024,1024").split(","))
g = fd.make_grid(npts, (2 * np.pi,) * 3)
s = fd.taylor_green_init(g, c)
for v in (sys.argv[2] if len(sys.argv) > 2 else "SN,SS").split(","):
    ev = fd.ResidualEvaluator(g, c, v)
    Y, Z = ev.workspace()
    ts = []
    for r in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ev.stage(s.bundle, s.bundle, Y, 1e-3)
        b.record()
        torch.cuda.synchronize()
        if r:
            ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    print(f"{v}@{npts}: {ms:.2f} ms  {np.prod(npts) / (ms / 1e3):.3e} pt-stage/s", flush=True)
    del ev, Y, Z
    torch.cuda.empty_cache()
