"""Cost of bitwise parity: the same build with FMA contraction (-fmad=true,
alt/fma.so) against the default (-fmad=false).  Run once per library (the
caller swaps the .so); prints whole-step timings and writes the final
conservative fields of a short 256^3 TGV run for the comparison.

    python tools/fma_ab.py /tmp/base.npy            # default library
    python tools/fma_ab.py /tmp/fma.npy /tmp/base.npy   # swapped library: compare
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd


def main():
    out = sys.argv[1]
    torch.cuda.set_device(0)
    c = fd.PhysicalConstants()
    g = fd.make_grid((256,) * 3, (2 * np.pi,) * 3)
    st = fd.taylor_green_init(g, c)
    fd.run(st, fd.RKScheme(dt=8.5e-4), fd.ResidualEvaluator(g, c, "SN"), 10)
    torch.cuda.synchronize()
    cur = g.interior(st.bundle[:5]).cpu().numpy()
    np.save(out, cur)
    if len(sys.argv) > 2:
        ref = np.load(sys.argv[2])
        for f, name in enumerate(("rho", "rhou0", "rhou1", "rhou2", "rhoE")):
            d = np.abs(cur[f] - ref[f])
            print(f"{name:6s} max |diff| {d.max():.3e}  relative to max |field| "
                  f"{d.max() / np.abs(ref[f]).max():.3e}  bitwise equal: "
                  f"{np.array_equal(cur[f], ref[f])}")


if __name__ == "__main__":
    main()
