"""Summarise an ncu launch list (gpu__time_duration per launch) into per-kernel
counts, mean times and shares of the total.

    python tools/launch_shares.py gpurun_out/launches.csv
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in data:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    print(f"{'launches':>8} {'mean_us':>10} {'share':>7}  kernel")
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v) / len(v) / 1e3:10.2f} {sum(v) / total * 100:6.1f}%  {name}")


if __name__ == "__main__":
    main(sys.argv[1])
