"""Small run of every variant and kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): the GPU analogue of the reference's
static race validator (plan.py:204-217).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
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
    c = fd.PhysicalConstants()
    for path, npts in ((0, (12, 16, 20)), (1, (9, 12, 7))):
        lib.fdns_set_kernel_path(path)
        lib.fdns_set_tiled_grid(5 if path == 0 else 0)
        g = fd.make_grid(npts, (2 * np.pi,) * 3)
        for v in fd.PLAN_NAMES:
            s = fd.taylor_green_init(g, c) if npts[0] == npts[1] == npts[2] else None
            if s is None:
                from paper_1610_09146_b200.diagnostics import state_from_conservative
                x = np.linspace(0, 1, int(np.prod(npts))).reshape(npts)
                cons = np.stack([1 + 0.1 * x, 0.1 * x, -0.05 * x, 0.02 * x, 250 + x])
                s = state_from_conservative(g, c, cons)
            ev = fd.ResidualEvaluator(g, c, v)
            fd.run(s, fd.RKScheme(dt=1e-3), ev, 1, cadence=1,
                   collect=fd.make_collector(g, 1.0))
            fd.assemble_residual(s, c, v)
            torch.cuda.synchronize()
            print(path, v, "ok", flush=True)
    lib.fdns_set_kernel_path(0)
    lib.fdns_set_tiled_grid(0)


if __name__ == "__main__":
    main()
