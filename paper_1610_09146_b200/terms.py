"""The residual's derivative registry, host side (mirrors `fdns.terms`).

The reference writes the five residual right-hand sides as expression
strings over point fields and ``{D(...)}`` placeholders and generates a
kernel from them (terms.py:135-200, codegen.py).  Here the same term list
is compiled into the device kernels (csrc/fdns_math.cuh, one function per
residual with the reference's association); this module keeps the
introspection side of it: the field and constant names, `Deriv` records of
the 60 distinct derivatives (kind, differentiated expression, axes),
their occurrence counts in the residuals and the nine velocity-gradient
ids the RS/SS plans store.  `build_residual_spec` accepts the reference's
default ``energy_phi="internal"`` form, the one the kernels implement.
"""

from __future__ import annotations

from dataclasses import dataclass, field

STATE_FIELDS = ("rho", "rhou0", "rhou1", "rhou2", "rhoE")          # terms.py:27
PRIMITIVE_FIELDS = ("u0", "u1", "u2", "p", "T")
POINT_FIELDS = STATE_FIELDS + PRIMITIVE_FIELDS
KERNEL_CONSTANTS = ("inv_Re", "c13_inv_Re", "c43_inv_Re", "c23_inv_Re",
                    "heat_coeff")
RESIDUAL_FIELDS = ("d_rho", "d_rhou0", "d_rhou1", "d_rhou2", "d_rhoE")

# internal energy density over stored fields (terms.py:39); the staged
# kernels hold it per point (rho*e) instead of re-forming it per tap
RHOE_INTERNAL = "(rhoE - 0.5*(rhou0*u0 + rhou1*u1 + rhou2*u2))"


@dataclass(frozen=True)
class Deriv:
    """One distinct derivative (terms.py:42-77): kind "d1", "d2" or "cross";
    `expr` the differentiated point expression; `axes` (axis,) or
    (outer, inner)."""

    id: str
    kind: str
    expr: str
    axes: tuple

    @property
    def name(self) -> str:
        """Identifier-safe short name (the reference's spelling rules)."""
        out = self.id
        for a, b in (("(", "_"), (")", ""), (",", "_"), ("*", ""),
                     ("D2", "dd"), ("DD", "dx"), ("D", "d")):
            out = out.replace(a, b)
        return out.lower()

    @property
    def is_product(self) -> bool:
        return self.expr not in POINT_FIELDS

    @property
    def inner_id(self) -> str:
        assert self.kind == "cross"
        return f"D({self.expr},x{self.axes[1]})"


@dataclass
class ResidualSpec:
    """Derivative registry of the compiled term list (terms.py:80-110).
    `residuals` names the device function computing each residual."""

    derivatives: dict = field(default_factory=dict)
    residuals: dict = field(default_factory=dict)
    occurrences: dict = field(default_factory=dict)
    velocity_gradient_ids: tuple = ()


def _deriv(did: str) -> Deriv:
    head, args = did.split("(", 1)
    parts = args.rstrip(")").split(",")
    target = parts[0]
    expr = target.replace("rhoe", RHOE_INTERNAL)
    if head == "D":
        return Deriv(did, "d1", expr, (int(parts[1][1:]),))
    if head == "D2":
        return Deriv(did, "d2", expr, (int(parts[1][1:]),))
    return Deriv(did, "cross", expr, (int(parts[1][1:]), int(parts[2][1:])))


def build_residual_spec(energy_phi: str = "internal") -> ResidualSpec:
    """The term list's registry (terms.py:135-200) for the internal-energy
    skew split, the form the device kernels are compiled for."""
    if energy_phi == "total":
        raise ValueError("the device kernels implement the energy_phi="
                         "'internal' term list only")
    if energy_phi != "internal":
        raise ValueError(f"unknown energy_phi: {energy_phi}")
    from .plan import OCCURRENCES, VELOCITY_GRADIENT_IDS, derivative_ids
    spec = ResidualSpec()
    for did in derivative_ids():
        spec.derivatives[did] = _deriv(did)
    spec.occurrences = dict(OCCURRENCES)
    spec.velocity_gradient_ids = tuple(VELOCITY_GRADIENT_IDS)
    spec.residuals = {
        "d_rho": "csrc/fdns_math.cuh:mass_residual",
        "d_rhou0": "csrc/fdns_math.cuh:momentum_prefix/suffix<0>",
        "d_rhou1": "csrc/fdns_math.cuh:momentum_prefix/suffix<1>",
        "d_rhou2": "csrc/fdns_math.cuh:momentum_prefix/suffix<2>",
        "d_rhoE": "csrc/fdns_math.cuh:energy_prefix/suffix",
    }
    return spec


DEFAULT_SPEC = build_residual_spec()
