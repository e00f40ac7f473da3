"""Host<->device bandwidth: copy engines (cudaMemcpyAsync) vs an SM copy
kernel reading / writing pinned host memory directly (fdns_copy_sm).

    python tools/pcie_sm_copy.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1610_09146_b200 import _lib

torch.cuda.set_device(0)
lib = _lib.load()
MB = 1 << 20


def bw(fn, size, reps=10):
    best = 0.0
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = max(best, size * reps / e0.elapsed_time(e1) / 1e6)
    return best


for size in (int(2.5 * MB), int(12.6 * MB), 64 * MB):
    h = torch.ones(size // 8, dtype=torch.float64).pin_memory()
    d = torch.empty(size // 8, dtype=torch.float64, device="cuda")
    st = _lib.stream_handle()
    res = {}
    res["ce h2d"] = bw(lambda: d.copy_(h, non_blocking=True), size)
    res["ce d2h"] = bw(lambda: h.copy_(d, non_blocking=True), size)
    for ctas in (148, 592, 1184):
        res[f"sm h2d/{ctas}"] = bw(lambda: lib.fdns_copy_sm(d.data_ptr(), h.data_ptr(), size, ctas, st), size)
        res[f"sm d2h/{ctas}"] = bw(lambda: lib.fdns_copy_sm(h.data_ptr(), d.data_ptr(), size, ctas, st), size)
    torch.cuda.synchronize()
    print(f"{size / MB:6.2f} MB: " + "  ".join(f"{k} {v:5.1f}" for k, v in res.items()), flush=True)
# correctness
h = torch.arange(1 << 20, dtype=torch.float64).pin_memory()
d = torch.zeros(1 << 20, dtype=torch.float64, device="cuda")
_lib.check(lib.fdns_copy_sm(d.data_ptr(), h.data_ptr(), h.numel() * 8, 0, _lib.stream_handle()))
torch.cuda.synchronize()
print("sm copy exact:", bool(torch.equal(d.cpu(), h)))
