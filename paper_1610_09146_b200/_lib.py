"""ctypes binding of the C ABI in include/fdns_b200.h.

The CUDA library `libfdns_b200.so` is built in-tree by
`__graft_entry__.build()` (or `python -m paper_1610_09146_b200.build`).
There is no CPU fallback: if the library or a GPU is missing every entry
point raises.
"""

from __future__ import annotations

import ctypes
import pathlib

import torch

_HERE = pathlib.Path(__file__).parent
LIB_PATH = _HERE / "libfdns_b200.so"
ABI_VERSION = 1

# variant ids (include/fdns_b200.h, the reference's PLAN_NAMES plan.py:33)
VARIANT_IDS = {"BL": 0, "RA": 1, "RS": 2, "SN": 3, "SS": 4}

_D = ctypes.POINTER(ctypes.c_double)
_VP = ctypes.c_void_p
_I = ctypes.c_int32


class FdnsError(RuntimeError):
    """A CUDA-side failure reported through the C ABI."""


class Problem(ctypes.Structure):
    """Mirror of `fdns_problem` (include/fdns_b200.h)."""

    _fields_ = [("n", ctypes.c_int32 * 3), ("h", ctypes.c_int32),
                ("w", ctypes.c_double * 15), ("kc", ctypes.c_double * 5),
                ("gm1", ctypes.c_double), ("gM2", ctypes.c_double)]


_lib = None

EXPORTS = {
    "fdns_last_error": (ctypes.c_char_p, []),
    "fdns_abi_version": (_I, []),
    "fdns_launch_count": (ctypes.c_int64, []),
    "fdns_workarray_count": (_I, [_I]),
    "fdns_primitives": (_I, [_VP, ctypes.POINTER(Problem), _VP]),
    "fdns_primitives_planes": (_I, [_VP, _I, _I, ctypes.POINTER(Problem), _VP]),
    "fdns_halo_wrap": (_I, [_VP, _I, _I, ctypes.POINTER(Problem), _VP]),
    "fdns_residual": (_I, [_I, _VP, _VP, _VP, ctypes.POINTER(Problem), _VP]),
    "fdns_rk_update": (_I, [_VP, _VP, _VP, ctypes.c_double,
                            ctypes.POINTER(Problem), _VP]),
    "fdns_stage": (_I, [_I, _VP, _VP, _VP, _VP, ctypes.c_double, _I,
                        ctypes.POINTER(Problem), _VP]),
    "fdns_stage_planes": (_I, [_I, _VP, _VP, _VP, _VP, ctypes.c_double, _I, _I,
                               _I, _I, ctypes.POINTER(Problem), _VP]),
    "fdns_set_kernel_path": (None, [_I]),
    "fdns_set_tiled_grid": (None, [_I]),
    "fdns_set_pdl": (None, [_I]),
    "fdns_set_prefetch": (None, [_I]),
    "fdns_set_rounds": (None, [_I]),
    "fdns_set_lockstep": (None, [_I]),
    "fdns_debug_trace": (_I, [_I, ctypes.POINTER(ctypes.c_uint64), _I]),
    "fdns_debug_rounds_walk": (_I, [ctypes.c_int64, _I, _I, _I, ctypes.POINTER(_I),
                                    ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "fdns_diag_partials_size": (_I, [ctypes.POINTER(Problem)]),
    "fdns_reduce_diag": (_I, [_VP, _VP, _VP, _VP, ctypes.POINTER(Problem),
                              _VP]),
    "fdns_fp64_probe": (_I, [_VP, _I, _D, _VP]),
    "fdns_l2_flush": (_I, [_VP, ctypes.c_int64, _VP]),
    "fdns_copy_sm": (_I, [_VP, _VP, ctypes.c_int64, _I, _VP]),
    "fdns_copy_rows": (_I, [_VP, ctypes.c_int64, _VP, ctypes.c_int64, ctypes.c_int64,
                            ctypes.c_int64, _VP]),
    "fdns_derivative": (_I, [_VP, _VP, _I, ctypes.POINTER(Problem), _VP]),
}


def load(require_gpu: bool = True):
    """Load the CUDA library; raise loudly if it (or the GPU) is missing."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FdnsError(
                f"{LIB_PATH} is missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.fdns_abi_version() != ABI_VERSION:
            raise FdnsError("libfdns_b200.so ABI version mismatch")
        _lib = lib
    if require_gpu and not torch.cuda.is_available():
        raise FdnsError("fdns_b200 needs a CUDA device; there is no CPU "
                        "fallback")
    return _lib


def check(status: int, what: str = "fdns call") -> None:
    if status != 0:
        msg = _lib.fdns_last_error().decode() if _lib is not None else ""
        raise FdnsError(f"{what} failed ({status}): {msg}")


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor) -> int:
    return t.data_ptr()
