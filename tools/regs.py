"""Register / spill table of an experimental build (no GPU needed).

    python tools/regs.py OUT.so [filter] -DFOO=1 ...
"""
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1610_09146_b200 import build as b  # noqa: E402

out, filt = sys.argv[1], sys.argv[2]
extra = sys.argv[3:]
cmd = [b.nvcc(), *b.NVCC_FLAGS, *extra, "-o", out, *map(str, b.SOURCES)]
res = subprocess.run(cmd, capture_output=True, text=True)
if res.returncode:
    sys.exit(res.stderr[-3000:])
cur = None
for line in (res.stdout + res.stderr).splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True,
                             text=True).stdout.strip()
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = int(m.group(1)) + int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and re.search(filt, cur):
        print(f"{int(m.group(1)):4d} regs {spill:6d} B spill  {cur[:100]}")
