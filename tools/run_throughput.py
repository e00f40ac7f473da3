"""Throughput of the public `run()` loop (host-launched per stage) vs the
stage kernels, per variant."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd

torch.cuda.set_device(0)
c = fd.PhysicalConstants()
for n in (64, 128):
    g = fd.make_grid((n,) * 3, (2 * np.pi,) * 3)
    for v in ("SN", "SS", "BL"):
        s = fd.taylor_green_init(g, c)
        ev = fd.ResidualEvaluator(g, c, v)
        fd.run(s, fd.RKScheme(dt=1e-3), ev, 3)
        rep = fd.run(s, fd.RKScheme(dt=1e-3), ev, 50)
        print(f"run() {v}@{n}: {n**3 * 3 * 50 / rep.loop_seconds:.3e} pt-stage/s "
              f"({rep.loop_seconds / 50 * 1e3:.3f} ms/step)", flush=True)
