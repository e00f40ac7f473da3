"""In-tree build of the sm_100a CUDA library (libfdns_b200.so).

`python -m paper_1610_09146_b200.build` or `__graft_entry__.build()`.
Flags: -fmad=false keeps every kernel free of FMA contraction (bitwise
parity with the reference, see csrc/fdns_math.cuh); division stays IEEE
(nvcc's default -prec-div=true).
"""

from __future__ import annotations

import os
import pathlib
import shutil
import subprocess
import sys

HERE = pathlib.Path(__file__).parent
ROOT = HERE.parent
SOURCES = [HERE / "csrc" / "fdns_b200.cu"]
DEPS = list((HERE / "csrc").glob("*.cuh")) + [ROOT / "include" / "fdns_b200.h"]
OUT = HERE / "libfdns_b200.so"

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-fmad=false", "-prec-div=true", "-prec-sqrt=true",
              "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
              "-Xptxas", "-v", "-I", str(ROOT / "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"),
                 "/usr/local/cuda/bin/nvcc"):
        if cand and pathlib.Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in SOURCES + DEPS)


def build(force: bool = False, verbose: bool = False) -> pathlib.Path:
    if not force and up_to_date():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(OUT), *map(str, SOURCES)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = res.stdout + res.stderr
    (HERE / "build.log").write_text(log)
    if res.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError("nvcc failed building libfdns_b200.so")
    if verbose:
        print(log)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
