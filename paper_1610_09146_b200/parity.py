"""Parity mode: the reference's own numpy state objects at the boundary.

A caller of the reference holds `fdns.physics.ConservativeState` /
`Residual` objects whose fields are padded float64 numpy arrays
(`Field.data`, mesh.py:88-115; argument order physics.py:115-119).
`ResidualEvaluator.evaluate`, `assemble_residual` and `run` accept such
objects directly (duck-typed: anything exposing `field_arrays()` /
`arrays()` of numpy arrays in the reference layout): the fields are copied
to a device twin as they are (same layout, no transpose), the device path
runs, and the results are copied back with the reference's side effects --

* `evaluate(state, out)` (plan.py:394-416): the state's primitive arrays
  u, p, T are recomputed over the full padded arrays, the interior of the
  five residual arrays of `out` is written (their halos keep their values);
* `run(state, ...)` (timeloop.py:97-134): the conservative arrays hold the
  final state, and u, p, T the primitives of the last RK stage's input (the
  reference refreshes them only inside `evaluate`); a `collect` callback is
  handed the host state, synchronised before every sample.

The device path itself is unchanged: these are copies around it.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def _arrays(obj, method: str):
    fn = getattr(obj, method, None)
    if fn is None:
        return None
    arrs = fn()
    if not arrs or not all(isinstance(a, np.ndarray) for a in arrs):
        return None
    return arrs


def is_host_state(obj) -> bool:
    """A reference-style state: ten numpy arrays from `field_arrays()`."""
    from .physics import ConservativeState
    if isinstance(obj, ConservativeState):
        return False
    arrs = _arrays(obj, "field_arrays")
    return arrs is not None and len(arrs) == 10


def is_host_residual(obj) -> bool:
    """A reference-style residual: five numpy arrays from `arrays()`."""
    from .physics import Residual
    if isinstance(obj, Residual):
        return False
    arrs = _arrays(obj, "arrays")
    return arrs is not None and len(arrs) == 5


def _check_arrays(arrs, shape):
    for a in arrs:
        if a.shape != tuple(shape) or a.dtype != np.float64:
            raise ValueError(f"parity mode: host arrays must be float64 of the "
                             f"grid's padded shape {tuple(shape)}, got "
                             f"{a.dtype} {a.shape}")


class HostField:
    """A numpy-backed field with the reference `Field`'s attributes
    (mesh.py:88-115), for results returned to host callers."""

    __slots__ = ("grid", "data")

    def __init__(self, grid, data: np.ndarray):
        self.grid = grid
        self.data = data

    @property
    def interior(self) -> np.ndarray:
        h = self.grid.halo
        return self.data[h:-h, h:-h, h:-h]


class HostResidual:
    """Numpy residual with the reference `Residual`'s attributes
    (physics.py:132-156): what `assemble_residual` returns for a host
    state."""

    def __init__(self, grid):
        self.grid = grid
        f = [HostField(grid, np.zeros(grid.shape)) for _ in range(5)]
        self.d_rho, self.d_rhou, self.d_rhoE = f[0], f[1:4], f[4]

    @property
    def fields(self):
        return [self.d_rho, self.d_rhou[0], self.d_rhou[1], self.d_rhou[2],
                self.d_rhoE]

    def arrays(self):
        return tuple(f.data for f in self.fields)


def upload_conservative(host_state, dev_state) -> None:
    """The five padded conservative arrays, as they are, into the device
    twin (halos included: the reference requires them current)."""
    arrs = host_state.field_arrays()[:5]
    _check_arrays(arrs, dev_state.grid.shape)
    host = torch.from_numpy(np.stack([np.ascontiguousarray(a) for a in arrs]))
    dev_state.bundle[:5].copy_(host)


def download_primitives(bundle: torch.Tensor, host_state) -> None:
    """u, p, T (fields 5-9 of a device bundle, full padded arrays) into the
    host state's primitive arrays, in place."""
    arrs = host_state.field_arrays()
    got = bundle[5:10].cpu().numpy()
    for q in range(5):
        np.copyto(arrs[5 + q], got[q])


def download_conservative(bundle: torch.Tensor, host_state) -> None:
    arrs = host_state.field_arrays()
    got = bundle[:5].cpu().numpy()
    for q in range(5):
        np.copyto(arrs[q], got[q])


def write_residual(dev_out, out) -> None:
    """Interior of the device residual into `out` (a host residual: its
    halos are left as they are, like the reference kernel's; or a device
    Residual)."""
    from .physics import Residual
    if isinstance(out, Residual):
        out.grid.interior(out.bundle).copy_(dev_out.grid.interior(dev_out.bundle))
        return
    arrs = out.arrays()
    _check_arrays(arrs, dev_out.grid.shape)
    got = dev_out.grid.interior(dev_out.bundle).cpu().numpy()
    h = dev_out.grid.halo
    for q in range(5):
        arrs[q][h:-h, h:-h, h:-h] = got[q]


def sync_host_state(dev_state, host_state, constants) -> None:
    """Conservative fields of the device state, and the primitives the
    reference's state would hold (those of `prim_source`: the last RK
    stage's input, recomputed in place there -- the stage kernels do not
    store p, T), into the host state."""
    download_conservative(dev_state.bundle, host_state)
    prim = dev_state.prim_source
    if prim is None:
        prim = dev_state.bundle
    else:
        lib = _lib.load()
        _lib.check(lib.fdns_primitives(_lib.ptr(prim),
                                       dev_state.grid.problem(constants),
                                       _lib.stream_handle()), "primitives")
    download_primitives(prim, host_state)
