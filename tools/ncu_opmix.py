"""Dynamic SASS opcode mix and stall samples of one kernel in an ncu report
(needs a capture with --set full / source counters).

    python tools/ncu_opmix.py gpurun_out/x.ncu-rep [kernel-regex] [launch-skip] [--full]
"""
import collections
import csv
import io
import subprocess
import sys


def load(rep, kern="k_stage_tiled", skip=0):
    out = subprocess.run(
        ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
         "-k", "regex:" + kern, "--launch-skip", str(skip), "--launch-count", "1"],
        capture_output=True, text=True, check=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    return lines[0], rows


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    full = "--full" in sys.argv
    rep = args[0]
    kern = args[1] if len(args) > 1 else "k_stage_tiled"
    skip = int(args[2]) if len(args) > 2 else 0
    name, rows = load(rep, kern, skip)
    ops = collections.Counter()
    stalls = collections.Counter()
    total = 0
    for r in rows:
        src = r["Source"].strip()
        toks = src.split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        if not full:
            op = op.split(".")[0]
        if not (r["Instructions Executed"] or "0").isdigit():
            continue   # repeated header / section rows
        n = int(r["Instructions Executed"] or 0)
        ops[op] += n
        stalls[op] += int(r["Warp Stall Sampling (All Samples)"] or 0)
        total += n
    print(name[:150])
    st = sum(stalls.values())
    print(f"{'opcode':28s} {'warp-insts':>14s} {'share':>7s} {'stall-share':>11s}")
    for op, n in ops.most_common(40):
        print(f"{op:28s} {n:14d} {n / total:7.1%} {stalls[op] / max(st, 1):11.1%}")
    print(f"{'total':28s} {total:14d}")


if __name__ == "__main__":
    main()
