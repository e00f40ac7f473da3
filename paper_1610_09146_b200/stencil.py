"""Fourth-order central-difference weights (host side).

Mirrors `fdns.stencil` (pkg/src/fdns/stencil.py:21-55): the weights are
evaluated once per grid on the host, pre-divided by the spacing, and handed
to every kernel, so all variants apply identical weights in identical
expression shapes.  The stencil *application* lives in the CUDA kernels
(csrc/fdns_math.cuh).
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
