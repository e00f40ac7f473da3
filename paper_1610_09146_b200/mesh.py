"""Structured periodic grid, device-resident halo-padded fields, halo exchange.

Mirrors the reference's `fdns.mesh` (pkg/src/fdns/mesh.py) with the storage
moved to HBM: every field is a float64 CUDA tensor C-ordered
(n0+2h, n1+2h, n2+2h) with axis 2 contiguous, byte-identical to the
reference's padded numpy array (mesh.py:3-6).  A `Grid` may carry a z-slab
decomposition (`slab`, see decomp.py): axis 0 is then split over ranks and
each rank allocates only its `local_npoints`.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field as dfield

import numpy as np
import torch

from . import _lib

MIN_POINTS = 5   # mesh.py:16
MIN_HALO = 2     # mesh.py:17


class ConfigurationError(ValueError):
    """Invalid grid or solver configuration (mesh.py:20-21)."""


_live_fields = 0


def live_field_count() -> int:
    """Number of live grid-sized device allocations (mesh.py:30-32)."""
    return _live_fields


def _release(n: int) -> None:
    global _live_fields
    _live_fields -= n


@dataclass(frozen=True)
class Grid:
    """Periodic box (mesh.py:40-67) plus an optional z-slab decomposition."""

    npoints: tuple[int, int, int]
    delta: tuple[float, float, float]
    halo: int
    slab: object = dfield(default=None, compare=False)

    ndim = 3

    @property
    def local_npoints(self) -> tuple[int, int, int]:
        if self.slab is None:
            return self.npoints
        return (self.slab.local_n0, self.npoints[1], self.npoints[2])

    @property
    def offset0(self) -> int:
        return 0 if self.slab is None else self.slab.offset0

    @property
    def shape(self) -> tuple[int, int, int]:
        """Padded (local) array shape including halos."""
        h = self.halo
        return tuple(n + 2 * h for n in self.local_npoints)

    @property
    def cell_volume(self) -> float:
        return self.delta[0] * self.delta[1] * self.delta[2]

    def interior(self, data):
        h = self.halo
        return data[..., h:-h, h:-h, h:-h]

    def coordinates(self, axis: int) -> np.ndarray:
        """Interior coordinates x_i = i*delta (mesh.py:65-67); for axis 0 of
        a slab, the rank's global indices."""
        if axis == 0:
            n = self.local_npoints[0]
            return (np.arange(n) + self.offset0) * self.delta[0]
        return np.arange(self.npoints[axis]) * self.delta[axis]

    def problem(self, constants=None) -> _lib.Problem:
        """The C-ABI problem descriptor for this (local) grid."""
        from .stencil import grid_weights
        pb = _lib.Problem()
        for a, n in enumerate(self.local_npoints):
            pb.n[a] = n
        pb.h = self.halo
        flat = []
        for w in grid_weights(self):
            flat.extend((w.first[0], w.first[1], *w.second))
        for i, v in enumerate(flat):
            pb.w[i] = v
        if constants is not None:
            for i, v in enumerate(constants.kernel_constants()):
                pb.kc[i] = v
            pb.gm1 = constants.gm1
            pb.gM2 = constants.gM2
        return pb


def make_grid(npoints, lengths, halo: int = MIN_HALO, slab=None) -> Grid:
    """Periodic grid with delta[a] = lengths[a]/npoints[a] (mesh.py:70-85)."""
    npoints = tuple(int(n) for n in npoints)
    lengths = tuple(float(l) for l in lengths)
    if len(npoints) != 3 or len(lengths) != 3:
        raise ConfigurationError("grid requires 3 point counts and 3 lengths")
    if any(n < MIN_POINTS for n in npoints):
        raise ConfigurationError(
            f"need at least {MIN_POINTS} points per axis for the 5-point "
            f"stencil, got {npoints}")
    if any(l <= 0.0 for l in lengths):
        raise ConfigurationError(f"box lengths must be positive, got {lengths}")
    if halo < MIN_HALO:
        raise ConfigurationError(f"halo width must be >= {MIN_HALO}, got {halo}")
    delta = tuple(l / n for l, n in zip(lengths, npoints))
    if slab is not None:
        slab.validate(npoints[0], halo)
    return Grid(npoints=npoints, delta=delta, halo=halo, slab=slab)


def as_grid(grid) -> Grid:
    """This package's Grid for `grid`, which may be the reference's own
    `fdns.mesh.Grid` (same npoints/delta/halo attributes; parity mode)."""
    if isinstance(grid, Grid):
        return grid
    npoints = tuple(int(n) for n in grid.npoints)
    lengths = tuple(n * d for n, d in zip(npoints, grid.delta))
    g = make_grid(npoints, lengths, halo=int(grid.halo))
    # keep the caller's spacing bits (n * delta / n may round differently)
    return Grid(npoints=g.npoints, delta=tuple(float(d) for d in grid.delta),
                halo=g.halo)


def device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def alloc_bundle(grid: Grid, nf: int) -> torch.Tensor:
    """nf padded fields back to back in one HBM allocation, zeroed; counted
    nf times in the live-field counter (mesh.py:88-115)."""
    global _live_fields
    _lib.load()
    t = torch.zeros((nf,) + grid.shape, dtype=torch.float64, device=device())
    _live_fields += nf
    weakref.finalize(t, _release, nf)
    return t


class Field:
    """One grid-sized float64 device field with halo padding (mesh.py:88-115).

    `data` is a CUDA tensor (usually a view into a bundle).  `numpy()`
    copies the padded array to the host.
    """

    __slots__ = ("grid", "data", "__weakref__")

    def __init__(self, grid: Grid, data: torch.Tensor | None = None):
        self.grid = grid
        if data is None:
            data = alloc_bundle(grid, 1)[0]
        elif tuple(data.shape) != grid.shape or data.dtype != torch.float64:
            raise ConfigurationError(
                f"field data must be float64 with shape {grid.shape}")
        self.data = data

    @property
    def interior(self) -> torch.Tensor:
        return self.grid.interior(self.data)

    def fill_interior(self, values) -> "Field":
        if isinstance(values, np.ndarray):
            values = torch.from_numpy(np.ascontiguousarray(values))
        self.interior.copy_(torch.as_tensor(values, dtype=torch.float64)
                            .to(self.data.device).expand_as(self.interior))
        return self

    def numpy(self) -> np.ndarray:
        return self.data.cpu().numpy()

    def copy(self) -> "Field":
        f = Field(self.grid)
        f.data.copy_(self.data)
        return f


def halo_exchange_bundle(grid: Grid, bundle: torch.Tensor, nf: int | None = None):
    """Periodic ghost fill of the first nf fields of a bundle: local wrap of
    axes 1-2 (and 0 on one rank), slab exchange of axis 0 across ranks."""
    lib = _lib.load()
    nf = bundle.shape[0] if nf is None else nf
    pb = grid.problem()
    multi = grid.slab is not None and grid.slab.distributed
    mask = 0b110 if multi else 0b111
    _lib.check(lib.fdns_halo_wrap(_lib.ptr(bundle), nf, mask, pb,
                                  _lib.stream_handle()), "halo wrap")
    if multi:
        grid.slab.exchange(bundle[:nf], grid.halo)
    return bundle


def halo_exchange(field: Field) -> Field:
    """Fill ghost layers with periodic images, in place (mesh.py:118-139)."""
    halo_exchange_bundle(field.grid, field.data.unsqueeze(0), 1)
    return field


def reduce_sum(field: Field) -> float:
    """Sum over interior points (mesh.py:142-148), across slab ranks."""
    s = field.interior.sum()
    if field.grid.slab is not None and field.grid.slab.distributed:
        s = field.grid.slab.allreduce_sum(s.reshape(1))[0]
    return float(s)
