"""Build an experimental copy of the library with extra nvcc flags (A/B runs).

    python tools/build_alt.py OUT.so -DFDNS_FILL_CS=0 ...
Swap it in on the GPU box with `cp OUT.so paper_1610_09146_b200/libfdns_b200.so`.
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1610_09146_b200 import build as b  # noqa: E402

out, extra = sys.argv[1], sys.argv[2:]
flags = list(b.NVCC_FLAGS)
i = flags.index("-v")
del flags[i - 1:i + 1]   # drop "-Xptxas -v"
cmd = [b.nvcc(), *flags, *extra, "-o", out,
       *map(str, b.SOURCES)]
subprocess.run(cmd, check=True, capture_output=True)
print(out)
