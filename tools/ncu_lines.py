"""Per-source-line instruction counts and stall samples of one kernel in an
ncu report captured with --import-source on and -lineinfo builds.

    python tools/ncu_lines.py gpurun_out/x.ncu-rep [kernel-regex] [launch-skip] [top]
"""
import csv
import io
import os
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kern = sys.argv[2] if len(sys.argv) > 2 else "k_stage_tiled"
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    out = subprocess.run(
        ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
         "-k", "regex:" + kern, "--launch-skip", skip, "--launch-count", "1"],
        capture_output=True, text=True, check=True).stdout
    fname, rows, header = "?", [], None
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = os.path.basename(rec[1])
            continue
        if rec[0] == "Line No":
            header = rec
            continue
        if header is None or not rec[0].isdigit():
            continue
        d = dict(zip(header[2:], rec[2:]))
        try:
            n = int(d.get("Instructions Executed", "0") or 0)
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        rows.append((fname, int(rec[0]), rec[1].strip(), n, s))
    tn = sum(r[3] for r in rows) or 1
    ts = sum(r[4] for r in rows) or 1
    print(f"{'file:line':24s} {'insts':>7s} {'stalls':>7s}  source")
    for f, ln, src, n, s in sorted(rows, key=lambda r: -r[4])[:top]:
        print(f"{f + ':' + str(ln):24s} {n / tn:7.1%} {s / ts:7.1%}  {src[:90]}")


if __name__ == "__main__":
    main()
