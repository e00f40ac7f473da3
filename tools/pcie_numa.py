"""H2D bandwidth from pinned buffers allocated while the process runs on
the GPU's local NUMA node vs elsewhere (sysfs local_cpulist of the GPU).

    python tools/pcie_numa.py
"""
import os

import torch


def gpu_local_cpus(dev=0):
    p = torch.cuda.get_device_properties(dev)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    base = f"/sys/bus/pci/devices/{bus}"
    node = open(base + "/numa_node").read().strip()
    cpus = open(base + "/local_cpulist").read().strip()
    return bus, node, cpus


def parse(lst):
    out = set()
    for part in lst.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.update(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


def h2d(size, reps=20):
    h = torch.ones(size // 8, dtype=torch.float64).pin_memory()
    d = torch.empty(size // 8, dtype=torch.float64, device="cuda")
    best = 0
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, size * reps / e0.elapsed_time(e1) / 1e6)
    return best


torch.cuda.set_device(0)
bus, node, cpus = gpu_local_cpus()
allc = os.sched_getaffinity(0)
local = parse(cpus) & allc
print(f"GPU {bus} numa_node {node} local_cpulist {cpus}; process cpus {len(allc)}, local {len(local)}")
MB = 1 << 20
for label, cset in (("all", allc), ("local", local), ("remote", allc - local)):
    if not cset:
        print(label, "none")
        continue
    os.sched_setaffinity(0, cset)
    print(label, " ".join(f"{s / MB:.1f}MB:{h2d(s):.1f}" for s in (int(2.5 * MB), int(12.6 * MB))), flush=True)
os.sched_setaffinity(0, allc)
