"""Host<->device copy bandwidth from pinned memory (one direction and both
at once), for the chunk sizes the host-buffer stepping uses.

    python tools/pcie_probe.py
"""
import torch

torch.cuda.set_device(0)
MB = 1 << 20
for size in (int(0.6 * MB), int(2.5 * MB), int(12.6 * MB), 64 * MB):
    h = torch.empty(size // 8, dtype=torch.float64).pin_memory()
    h2 = torch.empty(size // 8, dtype=torch.float64).pin_memory()
    d = torch.empty(size // 8, dtype=torch.float64, device="cuda")
    d2 = torch.empty(size // 8, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    reps = max(3, int(256 * MB / size))
    res = {}
    for mode in ("h2d", "d2h", "both"):
        for _ in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                if mode in ("h2d", "both"):
                    with torch.cuda.stream(s1):
                        d.copy_(h, non_blocking=True)
                if mode in ("d2h", "both"):
                    with torch.cuda.stream(s2):
                        h2.copy_(d2, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        nbytes = size * reps * (2 if mode == "both" else 1)
        res[mode] = nbytes / ms / 1e6
    print(f"{size / MB:6.2f} MB: h2d {res['h2d']:6.1f} GB/s  d2h {res['d2h']:6.1f} GB/s  "
          f"both {res['both']:6.1f} GB/s total", flush=True)
