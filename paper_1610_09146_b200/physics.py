"""Physical constants, device-resident state containers, primitive recovery.

Mirrors `fdns.physics` (pkg/src/fdns/physics.py).  A `ConservativeState`
owns ONE HBM bundle of 10 padded fields in the reference's kernel argument
order rho, rhou0..2, rhoE, u0..2, p, T (physics.py:115-119); the `Field`
attributes are views into it.  `Residual` likewise owns a 5-field bundle.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .mesh import Field, Grid, alloc_bundle


class SolverDivergenceError(RuntimeError):
    """Non-finite solution or non-positive density (physics.py:23-29)."""

    def __init__(self, message, iteration=None, substep=None):
        super().__init__(message)
        self.iteration = iteration
        self.substep = substep


@dataclass(frozen=True)
class PhysicalConstants:
    """Non-dimensional constants plus derived factors (physics.py:32-81)."""

    gamma: float = 1.4
    M: float = 0.1
    Pr: float = 0.71
    Re: float = 1600.0

    def __post_init__(self):
        if not (self.gamma > 1.0 and self.M > 0.0 and self.Pr > 0.0
                and self.Re > 0.0):
            raise ValueError(
                "require gamma > 1 and positive M, Pr, Re; got "
                f"gamma={self.gamma}, M={self.M}, Pr={self.Pr}, Re={self.Re}")

    @property
    def gm1(self) -> float:
        return self.gamma - 1.0

    @property
    def gM2(self) -> float:
        return self.gamma * self.M * self.M

    @property
    def inv_Re(self) -> float:
        return 1.0 / self.Re

    @property
    def heat_coeff(self) -> float:
        return 1.0 / (self.gm1 * self.M * self.M * self.Pr * self.Re)

    @property
    def c13_inv_Re(self) -> float:
        return 1.0 / (3.0 * self.Re)

    @property
    def c43_inv_Re(self) -> float:
        return 4.0 / (3.0 * self.Re)

    @property
    def c23_inv_Re(self) -> float:
        return 2.0 / (3.0 * self.Re)

    def kernel_constants(self) -> tuple[float, ...]:
        return (self.inv_Re, self.c13_inv_Re, self.c43_inv_Re,
                self.c23_inv_Re, self.heat_coeff)


STATE_NAMES = ("rho", "rhou0", "rhou1", "rhou2", "rhoE")
PRIMITIVE_NAMES = ("u0", "u1", "u2", "p", "T")


class ConservativeState:
    """The five prognostic fields plus the derived primitive fields
    (physics.py:84-129), resident in one HBM bundle."""

    def __init__(self, grid: Grid, bundle: torch.Tensor | None = None):
        self.grid = grid
        if bundle is None:
            bundle = alloc_bundle(grid, 10)
        self.bundle = bundle
        # bundle whose fields 5-9 hold the primitives the reference's state
        # would expose (None: this bundle's own); see diagnostics.reduce_state
        self.prim_source = None
        f = [Field(grid, bundle[q]) for q in range(10)]
        self.rho, self.rhou, self.rhoE = f[0], f[1:4], f[4]
        self.u, self.p, self.T = f[5:8], f[8], f[9]

    @property
    def conservative(self) -> list[Field]:
        return [self.rho, self.rhou[0], self.rhou[1], self.rhou[2], self.rhoE]

    @property
    def primitive(self) -> list[Field]:
        return [self.u[0], self.u[1], self.u[2], self.p, self.T]

    def field_arrays(self):
        """Padded device arrays in the kernel argument order."""
        return tuple(self.bundle[q] for q in range(10))

    # -- host interop (parity mode) -------------------------------------
    def load_conservative(self, arrays) -> "ConservativeState":
        """Copy 5 host arrays (interior or padded shape) to the device."""
        h = self.grid.halo
        for f, a in zip(self.conservative, arrays):
            a = np.asarray(a, dtype=np.float64)
            if a.shape == self.grid.shape:
                f.data.copy_(torch.from_numpy(np.ascontiguousarray(a)))
            else:
                f.fill_interior(a)
        return self

    def to_numpy(self) -> np.ndarray:
        """(10, padded...) host copy of the bundle."""
        return self.bundle.cpu().numpy()

    def check_physical(self, iteration=None, substep=None):
        """Finite values and positive density on the interior
        (physics.py:121-129), evaluated by the device reduction."""
        from .diagnostics import reduce_state
        r = reduce_state(self)
        if r[7] > 0:
            raise SolverDivergenceError(
                "non-finite values in the conservative fields", iteration,
                substep)
        if r[8] > 0:
            raise SolverDivergenceError("non-positive density", iteration,
                                        substep)


class Residual:
    """RHS fields of the mass, momentum and energy equations
    (physics.py:132-156), resident in one 5-field HBM bundle."""

    def __init__(self, grid: Grid, bundle: torch.Tensor | None = None):
        self.grid = grid
        if bundle is None:
            bundle = alloc_bundle(grid, 5)
        self.bundle = bundle
        f = [Field(grid, bundle[q]) for q in range(5)]
        self.d_rho, self.d_rhou, self.d_rhoE = f[0], f[1:4], f[4]

    @property
    def fields(self) -> list[Field]:
        return [self.d_rho, self.d_rhou[0], self.d_rhou[1], self.d_rhou[2],
                self.d_rhoE]

    def arrays(self):
        return tuple(self.bundle[q] for q in range(5))

    def interior_numpy(self) -> np.ndarray:
        return self.grid.interior(self.bundle).cpu().numpy()


def eval_primitives_fused(state: ConservativeState,
                          c: PhysicalConstants) -> ConservativeState:
    """u, p, T from the conservative fields over the full padded arrays
    (physics.py:185-202), one fused device pass."""
    lib = _lib.load()
    state.prim_source = None
    _lib.check(lib.fdns_primitives(_lib.ptr(state.bundle),
                                   state.grid.problem(c),
                                   _lib.stream_handle()), "primitives")
    return state


def eval_primitives_grouped(state: ConservativeState,
                            c: PhysicalConstants) -> ConservativeState:
    """The reference's race-free grouped form (physics.py:169-182) is bitwise
    equal to the fused form (test_physics.py:83-100); on the device both run
    as the one fused pass."""
    return eval_primitives_fused(state, c)


# -- building blocks of the unexpanded residual (physics.py:205-253) --------
def stress_tensor(grad_u, c: PhysicalConstants):
    """Symmetric viscous stress tau[i][j] = (1/Re)(du_i/dx_j + du_j/dx_i)
    minus (2/(3Re)) div u on the diagonal, from the nine gradients
    grad_u[i][j] (scalars, arrays or device tensors); same operation order
    as physics.py:205-221, so the same bits."""
    div = grad_u[0][0] + grad_u[1][1] + grad_u[2][2]

    def entry(i, j):
        sym = c.inv_Re * (grad_u[i][j] + grad_u[j][i])
        return sym - c.c23_inv_Re * div if i == j else sym

    upper = {(i, j): entry(i, j) for i in range(3) for j in range(i, 3)}
    return [[upper[min(i, j), max(i, j)] for j in range(3)] for i in range(3)]


def heat_flux(grad_T, c: PhysicalConstants):
    """Fourier heat flux heat_coeff * dT/dx_j per axis (physics.py:224-226)."""
    return [c.heat_coeff * g for g in grad_T]


def skew_convective(phi, uj, rho, axis: int):
    """Skew-symmetric convective split along one axis (physics.py:229-253):
    half the sum of d(rho phi u_j), u_j d(rho phi) and rho phi d(u_j) along
    x_j; phi a Field or the scalar 1.  Products are formed over the padded
    arrays (device tensors), the derivatives by the device stencil."""
    from .mesh import Field
    from .stencil import first_derivative
    grid = uj.grid
    m = Field(grid)                       # rho * phi
    m.data.copy_(rho.data * (phi.data if isinstance(phi, Field) else float(phi)))
    flux = Field(grid)                    # rho * phi * u_j
    flux.data.copy_(m.data * uj.data)
    d_flux, d_m, d_u = (first_derivative(f, axis) for f in (flux, m, uj))
    out = Field(grid)
    out.interior[...] = 0.5 * (d_flux.interior + uj.interior * d_m.interior
                               + m.interior * d_u.interior)
    return out
