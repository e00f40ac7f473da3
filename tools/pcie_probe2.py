import torch, time
torch.cuda.set_device(0)
MB = 1 << 20
for size in (int(2.5 * MB), int(12.6 * MB), 32*MB, 64 * MB):
    h = torch.ones(size // 8, dtype=torch.float64).pin_memory()
    d = torch.empty(size // 8, dtype=torch.float64, device="cuda")
    s1 = torch.cuda.Stream()
    for rep in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s1):
            e0.record(s1)
            for _ in range(10):
                d.copy_(h, non_blocking=True)
            e1.record(s1)
        torch.cuda.synchronize()
        print(f"{size/MB:6.2f} MB rep{rep}: h2d {size*10/e0.elapsed_time(e1)/1e6:6.1f} GB/s", flush=True)
