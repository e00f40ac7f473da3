"""ctypes binding of the C + OpenMP oracle -- TEST INFRASTRUCTURE ONLY.

Thin wrappers over oracle/csrc/fdns_oracle.c (built by `make -C oracle`, or
by `__graft_entry__.build()`), taking the same (10, n0+2h, n1+2h, n2+2h)
float64 bundles as `numpy_oracle`.
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

from . import numpy_oracle as npo

_HERE = pathlib.Path(__file__).parent
_LIB_PATH = _HERE / "lib" / "libfdns_oracle.so"
_lib = None

_D = ctypes.POINTER(ctypes.c_double)


def build():
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(_LIB_PATH))
        i = ctypes.c_int
        _lib.oracle_residual.argtypes = [_D, _D, i, i, i, i, _D, _D, i]
        _lib.oracle_primitives.argtypes = [_D, i, i, i, i, ctypes.c_double,
                                           ctypes.c_double, i]
        _lib.oracle_halo.argtypes = [_D, i, i, i, i, i]
        _lib.oracle_run.argtypes = [_D, _D, _D, i, i, i, i, _D, _D,
                                    ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, i, i]
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def _dims(F, h):
    return [s - 2 * h for s in F.shape[1:]]


def _wk(npts, c):
    w = np.array([x for a in npo.grid_weights(npts) for x in a])
    kc = np.array([c.inv_Re, c.c13, c.c43, c.c23, c.heat_coeff])
    return w, kc


def default_threads() -> int:
    return len(os.sched_getaffinity(0))


def primitives(F, c, h=2, nthreads=0):
    n = _dims(F, h)
    lib().oracle_primitives(_p(F), *n, h, c.gm1, c.gM2, nthreads)
    return F


def residual(F, c, h=2, nthreads=0):
    """Residual (5, n0, n1, n2) interior arrays; primitives must be current."""
    n = _dims(F, h)
    out = np.zeros((5,) + F.shape[1:])
    w, kc = _wk(n, c)
    lib().oracle_residual(_p(F), _p(out), *n, h, _p(w), _p(kc), nthreads)
    return npo.interior(out, h).copy()


def halo(F, nf, h=2):
    n = _dims(F, h)
    lib().oracle_halo(_p(F), nf, *n, h)
    return F


def run(F, c, dt, niter, h=2, nthreads=0):
    """niter RK3 iterations in place on the bundle F (timeloop.py:88-94)."""
    n = _dims(F, h)
    saved = np.zeros((5,) + F.shape[1:])
    res = np.zeros((5,) + F.shape[1:])
    w, kc = _wk(n, c)
    lib().oracle_run(_p(F), _p(saved), _p(res), *n, h, _p(w), _p(kc),
                     c.gm1, c.gM2, dt, niter, nthreads)
    return F
