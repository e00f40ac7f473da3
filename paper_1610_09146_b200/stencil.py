"""Fourth-order central-difference weights (host side).

Mirrors `fdns.stencil` (pkg/src/fdns/stencil.py:21-55): the weights are
evaluated once per grid on the host, pre-divided by the spacing, and handed
to every kernel, so all variants apply identical weights in identical
expression shapes.  The stencil *application* lives in the CUDA kernels
(csrc/fdns_math.cuh); `first_derivative`, `second_derivative` and
`cross_derivative` apply one stencil to one device field through
`fdns_derivative` (stencil.py:71-121), bitwise the reference's values.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class StencilWeights:
    """first = (w1, w2); second = (s0, s1, s2) (stencil.py:21-42)."""

    first: tuple[float, float]
    second: tuple[float, float, float]

    @property
    def first_full(self) -> tuple[float, ...]:
        w1, w2 = self.first
        return (-w2, -w1, 0.0, w1, w2)

    @property
    def second_full(self) -> tuple[float, ...]:
        s0, s1, s2 = self.second
        return (s2, s1, s0, s1, s2)


def make_weights(delta: float) -> StencilWeights:
    """stencil.py:45-51, same operation order."""
    return StencilWeights(
        first=(8.0 / (12.0 * delta), -1.0 / (12.0 * delta)),
        second=(-30.0 / (12.0 * delta * delta),
                16.0 / (12.0 * delta * delta),
                -1.0 / (12.0 * delta * delta)),
    )


def grid_weights(grid):
    """Per-axis weights of a grid (stencil.py:54-55)."""
    return tuple(make_weights(d) for d in grid.delta)


def _check_axis(axis: int) -> None:
    if axis not in (0, 1, 2):
        raise ValueError(f"axis must be 0, 1 or 2, got {axis}")


def _apply(f, op: int, out=None):
    from . import _lib
    from .mesh import Field
    grid = f.grid
    if out is None:
        out = Field(grid)
    lib = _lib.load()
    _lib.check(lib.fdns_derivative(_lib.ptr(f.data), _lib.ptr(out.data), op,
                                   grid.problem(), _lib.stream_handle()),
               "derivative")
    return out


def first_derivative(f, axis: int, out=None):
    """4th-order first derivative along an axis (stencil.py:71-86); the
    halo of `f` must be current; only the interior of the output is
    written."""
    _check_axis(axis)
    return _apply(f, axis, out)


def second_derivative(f, axis: int, out=None):
    """4th-order second derivative along an axis (stencil.py:89-102)."""
    _check_axis(axis)
    return _apply(f, 3 + axis, out)


def cross_derivative(f, axis_a: int, axis_b: int, out=None, scratch=None):
    """d^2 f / (dx_a dx_b) by composition (stencil.py:105-121): inner first
    derivative along b, its halo refreshed, outer first derivative along a."""
    from .mesh import halo_exchange
    _check_axis(axis_a)
    _check_axis(axis_b)
    if axis_a == axis_b:
        raise ValueError("cross_derivative requires distinct axes; "
                         "use second_derivative for repeated axes")
    inner = first_derivative(f, axis_b, out=scratch)
    halo_exchange(inner)
    return first_derivative(inner, axis_a, out=out)
