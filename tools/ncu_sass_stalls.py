"""Stall samples and executed instructions per SASS opcode (and the top
individual instructions) of one kernel launch in an ncu report.

    python tools/ncu_sass_stalls.py REPORT KERNEL_REGEX [launch-skip] [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "sass", "-k", "regex:" + kern, "--launch-skip", skip,
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_")]
    by_op = defaultdict(lambda: [0, 0])
    by_reason = defaultdict(int)
    insts = []
    for r in rows[2:]:
        if len(r) < len(hdr) or r[ix["Address"]] == "Address":
            continue
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        samp = int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
        ex = int(float(r[ix["Instructions Executed"]] or 0))
        by_op[op][0] += samp
        by_op[op][1] += ex
        for c in stall_cols:
            v = r[ix[c]]
            if v and v != "-":
                by_reason[c] += int(float(v))
        insts.append((samp, r[ix["Address"]], src, {c: r[ix[c]] for c in stall_cols
                                                      if r[ix[c]] not in ("0", "", "-")}))
    tot_s = sum(v[0] for v in by_op.values())
    tot_e = sum(v[1] for v in by_op.values())
    print(f"total samples {tot_s}, warp insts {tot_e}")
    print("-- by opcode (samples%, insts%)")
    for op, (s, e) in sorted(by_op.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{op:12s} {100 * s / tot_s:6.2f}% {100 * e / max(tot_e, 1):6.2f}%")
    print("-- by stall reason")
    for c, v in sorted(by_reason.items(), key=lambda x: -x[1])[:15]:
        print(f"{c:32s} {100 * v / max(tot_s, 1):6.2f}%")
    print("-- top instructions")
    for s, a, src, st in sorted(insts, key=lambda x: -x[0])[:top]:
        print(f"{s:7d} {a[-5:]} {src[:60]:60s} {st}")


if __name__ == "__main__":
    main()
