"""A/B of the host-buffer stepping configurations (upload engine x chunks),
interleaved in one process so box-to-box PCIe variation cancels.

    python tools/e2e_ab.py [n] [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd
from paper_1610_09146_b200.hostio import HostStepper

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
g = fd.make_grid((n,) * 3, (2 * np.pi,) * 3)
c = fd.PhysicalConstants()
ks = tuple(int(x) for x in os.environ.get("E2E_CHUNKS", "1,2,5").split(","))
ups = tuple(os.environ.get("E2E_UPLOAD", "ce,sm").split(","))
configs = [(u, k) for u in ups for k in ks]
res = {cfg: [] for cfg in configs}
for rnd in range(3):
    for up, k in configs:
        st = fd.taylor_green_init(g, c)
        host = HostStepper.pinned_buffers(g)
        host.copy_(st.bundle[:5].cpu())
        hs = HostStepper(st, fd.ResidualEvaluator(g, c, "SN"), fd.RKScheme(dt=3.385e-3), host,
                         chunks=k, upload=up)
        for _ in range(2):
            hs.step()
        hs.wait()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            hs.step()
        hs.wait()
        b.record()
        torch.cuda.synchronize()
        res[(up, k)].append(n ** 3 * 3 * steps / (a.elapsed_time(b) / 1e3))
        del hs, st, host
for cfg in configs:
    v = res[cfg]
    print(f"upload={cfg[0]} chunks={cfg[1]}: median {np.median(v):.3e}  all " +
          " ".join(f"{x:.3e}" for x in v))
