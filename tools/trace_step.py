"""Timeline of whole RK steps (three stage launches each) from the launch log
of the tiled stage kernels: per launch the entry / window-ready / exit
spread, and the gaps between consecutive launches.

    python tools/trace_step.py [n] [variant] [steps]
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
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = fd.make_grid((n,) * 3, (2 * np.pi,) * 3)
c = fd.PhysicalConstants()
s = fd.taylor_green_init(g, c)
ev = fd.ResidualEvaluator(g, c, variant)
it = IterationState(s, saved=False)
scheme = fd.RKScheme(dt=3.385e-3)
for _ in range(3):
    _fused_iteration(it, scheme, ev)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    _fused_iteration(it, scheme, ev)
torch.cuda.current_stream().wait_stream(st)
torch.cuda.synchronize()
with torch.cuda.graph(graph):
    _fused_iteration(it, scheme, ev)
torch.cuda.synchronize()
for _ in range(3):
    graph.replay()
torch.cuda.synchronize()
_lib.check(lib.fdns_debug_trace(2, None, 0))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    graph.replay()
e1.record()
torch.cuda.synchronize()
N = 8192 * 5 + 1
buf = (ctypes.c_uint64 * N)()
_lib.check(lib.fdns_debug_trace(3, buf, N))
raw = np.frombuffer(buf, dtype=np.uint64)
cnt = int(raw[0])
rec = raw[1:1 + cnt * 5].reshape(cnt, 5)
t = rec[:, :4].astype(np.float64)
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
print(f"{variant} {n}^3, {steps} graph steps, event time {e0.elapsed_time(e1) * 1e3 / steps:.1f} us/step, "
      f"{cnt} CTA records")
# split into launches: every CTA of launch L passes griddepcontrol.wait
# (stamp 1) after all CTAs of launch L-1 have exited, so in stamp-1 order a
# new launch begins where stamp 1 passes the running max exit
order = np.argsort(rel[:, 1])
rel = rel[order]
meta = rec[order, 4]
smid_all = ((meta >> np.uint64(16)) & np.uint64(0xFFFF)).astype(int)
cta_all = (meta & np.uint64(0xFFFF)).astype(int)
launch = np.zeros(cnt, dtype=int)
li, mx = 0, -1.0
for i in range(cnt):
    if mx >= 0 and rel[i, 1] >= mx:
        li += 1
        mx = -1.0
    launch[i] = li
    mx = max(mx, rel[i, 3])
prev_exit = None
for L in range(launch.max() + 1):
    r = rel[launch == L]
    print(f"launch {L}: {len(r)} CTAs  entry {r[:, 0].min():7.2f}..{r[:, 0].max():7.2f}  "
          f"wait-done {r[:, 1].min():7.2f}..{r[:, 1].max():7.2f}  ready {np.median(r[:, 2]):7.2f}/{r[:, 2].max():7.2f}  "
          f"exit {r[:, 3].min():7.2f}/{np.median(r[:, 3]):7.2f}/{r[:, 3].max():7.2f}"
          + (f"  prev-exit->wait-done {r[:, 1].min() - prev_exit:5.2f}" if prev_exit is not None else ""))
    prev_exit = r[:, 3].max()
    steady = r[:, 3] - r[:, 2]
    ramp = r[:, 2] - r[:, 1]
    print(f"          ramp (wait-done->ready) med {np.median(ramp):5.2f} max {ramp.max():5.2f}; "
          f"steady med {np.median(steady):6.2f} max {steady.max():6.2f} us")
    sm = smid_all[launch == L]
    ct = cta_all[launch == L]
    for name, sel in (("smid<74", sm < 74), ("smid>=74", sm >= 74), ("even", sm % 2 == 0),
                      ("odd", sm % 2 == 1)):
        if sel.any():
            print(f"          {name:9s} steady mean {steady[sel].mean():7.2f}", end="")
    print()
    o = np.argsort(-steady)[:6]
    print("          slowest (cta, smid, steady):",
          [(int(ct[i]), int(sm[i]), round(float(steady[i]), 1)) for i in o])
