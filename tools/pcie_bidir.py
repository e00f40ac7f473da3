"""PCIe copy bandwidth: H2D alone, D2H alone, and both at once (pinned host
buffers, copy engines, two streams) -- the ceiling of the e2e path.

    python tools/pcie_bidir.py [GB]
"""
import sys

import torch


def main():
    gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
    n = int(gb * 2 ** 30 / 8)
    torch.cuda.set_device(0)
    h1 = torch.empty(n, dtype=torch.float64).pin_memory()
    h2 = torch.empty(n, dtype=torch.float64).pin_memory()
    d1 = torch.empty(n, dtype=torch.float64, device="cuda")
    d2 = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(h2d, d2h):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        if h2d:
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / 1e3

    for _ in range(2):
        run(True, True)
    t = run(True, False)
    print(f"H2D alone   {n * 8 / t / 1e9:6.1f} GB/s")
    t = run(False, True)
    print(f"D2H alone   {n * 8 / t / 1e9:6.1f} GB/s")
    t = run(True, True)
    print(f"both at once {2 * n * 8 / t / 1e9:6.1f} GB/s aggregate ({n * 8 / t / 1e9:.1f} per direction)")


if __name__ == "__main__":
    main()
