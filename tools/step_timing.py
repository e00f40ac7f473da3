"""Whole-RK3-step throughput per variant and size (the bench's measurement
at any size): one fused iteration captured as a CUDA graph, K replays timed
with CUDA events, L2 flushed before each.  Unlike stage_timing.py (one stage
with input == saved state), stages 2 and 3 read a saved state that differs
from their input, as in a real run.

    python tools/step_timing.py --sizes 64,128,256 --variants SN,RA,SS,RS,BL
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1610_09146_b200 as fd
from paper_1610_09146_b200 import _lib
from paper_1610_09146_b200.timeloop import IterationState, _fused_iteration


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,128,256")
    ap.add_argument("--variants", default="SN,RA,SS")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--path", type=int, default=0, help="fdns_set_kernel_path (A/B)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    lib = _lib.load()
    lib.fdns_set_kernel_path(a.path)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    c = fd.PhysicalConstants()
    out = {}
    for n in map(int, a.sizes.split(",")):
        g = fd.make_grid((n,) * 3, (2 * np.pi,) * 3)
        for v in a.variants.split(","):
            s = fd.taylor_green_init(g, c)
            ev = fd.ResidualEvaluator(g, c, v)
            it = IterationState(s, saved=False)
            scheme = fd.RKScheme(dt=3.385e-3 * 64 / n)
            for _ in range(2):
                _fused_iteration(it, scheme, ev)
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                _fused_iteration(it, scheme, ev)
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                _fused_iteration(it, scheme, ev)
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.steps):
                lib.fdns_l2_flush(_lib.ptr(flush), flush.numel(), _lib.stream_handle())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                graph.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            pts = 3 * n ** 3 / (ms / 1e3)
            out[f"{v}@{n}"] = {"ms_per_step": ms, "pt_stage_per_s": pts}
            print(f"{v}@{n}: {ms * 1e3:9.1f} us/step  {pts:.3e} pt-stage/s", flush=True)
            del graph, ev, s, it
            torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
