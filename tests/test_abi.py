"""The C-ABI library loads and exports every symbol include/fdns_b200.h
declares (no compute calls: this runs on the CPU)."""

import ctypes
import pathlib
import re

from conftest import ROOT


def declared_symbols():
    text = (ROOT / "include" / "fdns_b200.h").read_text()
    return sorted(set(re.findall(r"\b(fdns_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("fdns_residual", "fdns_stage", "fdns_rk_update",
                 "fdns_primitives", "fdns_halo_wrap", "fdns_reduce_diag",
                 "fdns_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol(built):
    from paper_1610_09146_b200 import _lib
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert missing == []
    # every declared symbol is also bound by the host loader
    assert set(declared_symbols()) == set(_lib.EXPORTS)


def test_host_only_queries(built):
    from paper_1610_09146_b200 import _lib
    lib = _lib.load(require_gpu=False)
    assert lib.fdns_abi_version() == _lib.ABI_VERSION
    counts = {n: lib.fdns_workarray_count(i) for n, i in _lib.VARIANT_IDS.items()}
    assert counts == {"BL": 60, "RA": 0, "RS": 9, "SN": 0, "SS": 9}
    assert lib.fdns_workarray_count(99) == -1


def test_sm100a_code_in_library(built):
    """The shared object carries sm_100a SASS (cuobjdump lists it)."""
    import shutil
    import subprocess
    from paper_1610_09146_b200 import _lib
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not pathlib.Path(exe).exists():
        return
    out = subprocess.run([exe, "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
