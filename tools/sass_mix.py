"""Static SASS instruction mix per kernel of the built library.

    python tools/sass_mix.py [substring-of-mangled-name ...]
"""
import collections
import re
import subprocess
import sys

LIB = "paper_1610_09146_b200/libfdns_b200.so"


def mixes(lib=LIB):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True,
                         text=True, check=True).stdout
    cur, res = None, {}
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            res[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9]*)", line)
        if m and cur:
            res[cur][m.group(1)] += 1
    return res


if __name__ == "__main__":
    pats = sys.argv[1:] or ["k_stage_tiled"]
    for name, c in mixes().items():
        if any(p in name for p in pats):
            top = " ".join(f"{k}:{v}" for k, v in c.most_common(14))
            print(f"{name[:70]}\n  total {sum(c.values())}  {top}")
