"""e2e A/B: HostStepper wavefront mode vs the whole-step copy pipeline.

    python tools/e2e_wave_ab.py --n 512 --variant SN --steps 10 --chunks 8,16,32
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd
from paper_1610_09146_b200.hostio import HostStepper


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--variant", default="SN")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--chunks", default="8,16,32")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    c = fd.PhysicalConstants()
    g = fd.make_grid((a.n,) * 3, (2 * np.pi,) * 3)
    st = fd.taylor_green_init(g, c)
    ev = fd.ResidualEvaluator(g, c, a.variant)
    scheme = fd.RKScheme(dt=4.2e-4 * 512 / a.n)
    host = HostStepper.pinned_buffers(g)
    host.copy_(st.bundle[:5].cpu())
    configs = [("whole-step", dict(wavefront=False))] + [
        (f"wavefront K={k}", dict(wavefront=True, wave_chunks=k))
        for k in map(int, a.chunks.split(","))]
    for name, kw in configs:
        stepper = HostStepper(st, ev, scheme, host, chunks=5, **kw)
        for _ in range(2):
            stepper.step()
        stepper.wait()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            stepper.step()
        stepper.wait()
        e1.record()
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 1e3
        print(f"{name:18s} {sec / a.steps * 1e3:8.1f} ms/step  "
              f"{3 * a.n ** 3 * a.steps / sec:.3e} pt-stage/s", flush=True)
        del stepper


if __name__ == "__main__":
    main()
