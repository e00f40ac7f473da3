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


def test_round_robin_partition_covers_every_step_once(built):
    """Host-side walk of the stage kernels' round-robin split
    (fdns_tiled.cuh:Segments, SPLIT_ROUNDS with the partial last round cut
    into per-CTA plane ranges): every (tile, plane) step is visited exactly
    once and no CTA gets more than about its share -- no GPU needed."""
    import ctypes

    import numpy as np

    from paper_1610_09146_b200 import _lib
    lib = _lib.load(require_gpu=False)
    I32 = ctypes.POINTER(ctypes.c_int32)
    # (tiles, planes, unit, ctas): the 512^3 launches (688 tiles of 32 x 12),
    # 256^3 on the 8-warp kernel (8 x 32 tiles), tiny forced grids
    cases = [(688, 512, 128, 148), (688, 512, 64, 148), (688, 512, 256, 148),
             (256, 256, 128, 148), (176, 256, 64, 148), (2, 12, 4, 5),
             (2, 16, 4, 3), (6, 24, 4, 4), (3, 8, 8, 148), (1, 4, 4, 148)]
    for tiles, planes, unit, ctas in cases:
        cover = np.zeros(tiles * planes, dtype=np.int32)
        steps = np.zeros(ctas, dtype=np.int32)
        segs = np.zeros(ctas, dtype=np.int32)
        g = lib.fdns_debug_rounds_walk(tiles, planes, unit, ctas,
                                       cover.ctypes.data_as(I32),
                                       steps.ctypes.data_as(I32),
                                       segs.ctypes.data_as(I32))
        units = tiles * planes // unit
        assert g == min(ctas, units), (tiles, planes, unit, ctas)
        assert np.all(cover == 1), (tiles, planes, unit, ctas)
        assert steps[:g].sum() == tiles * planes
        # balance: whole rounds are equal, the tail differs by at most a step
        assert steps[:g].max() - steps[:g].min() <= 1, (tiles, planes, unit, ctas)
        # segments: the whole rounds plus at most two tail pieces
        assert segs[:g].max() <= units // g + 2
    bad = np.zeros(4, dtype=np.int32)
    assert lib.fdns_debug_rounds_walk(1, 6, 4, 2, bad.ctypes.data_as(I32), None, None) == -1
