"""Variant selector and the residual evaluator (the drop-in boundary).

Mirrors `fdns.plan` (pkg/src/fdns/plan.py): `PLAN_NAMES`, `build_plan`,
`KernelPlan`, `plan_storage`, `workarray_budget`, `ResidualEvaluator`
(`__init__` plan.py:316-337, `evaluate` :394-416) and `assemble_residual`
(:419-426).  The storage class of every derivative -- FETCH (work array in
HBM), LOCAL (register, computed once) or INLINE (re-expanded at each use) --
is the same as the reference's (plan.py:61-73, :162-188); it selects which
hand-written sm_100a kernel path runs (csrc/fdns_math.cuh providers).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .mesh import Grid, alloc_bundle
from .physics import (ConservativeState, PhysicalConstants, Residual,
                      eval_primitives_fused)

PLAN_NAMES = ("BL", "RA", "RS", "SN", "SS")          # plan.py:33
NORTH_STAR_PLANS = ("BL", "RA", "SN", "SS")

FETCH = "FETCH"
LOCAL = "LOCAL"
INLINE = "INLINE"


def derivative_ids() -> tuple[str, ...]:
    """The 60 distinct derivatives of the term list (terms.py:135-200), in
    the device slot order of csrc/fdns_math.cuh (18 per axis, 6 mixed)."""
    ids = []
    for a in range(3):
        x = f"x{a}"
        ids += [f"D(rho,{x})", f"D(p,{x})", f"D(rhoe,{x})",
                f"D(rhoe*u{a},{x})", f"D(u{a}*p,{x})", f"D2(T,{x})"]
        ids += [f"D(rhou{q},{x})" for q in range(3)]
        ids += [f"D(u{q},{x})" for q in range(3)]
        ids += [f"D(rhou{q}*u{a},{x})" for q in range(3)]
        ids += [f"D2(u{q},{x})" for q in range(3)]
    for j in range(3):
        for o in range(3):
            if o != j:
                ids.append(f"DD(u{j},x{o},x{j})")
    return tuple(ids)


VELOCITY_GRADIENT_IDS = tuple(f"D(u{i},x{j})" for i in range(3)
                              for j in range(3))


@dataclass(frozen=True)
class KernelPlan:
    """plan.py:51-58 (loop groups are replaced by the device kernel list)."""

    name: str
    store_derivatives: bool
    derivatives_to_store: frozenset
    local_variables: bool
    primitives: str  # "grouped" or "fused"

    @property
    def variant_id(self) -> int:
        return _lib.VARIANT_IDS[self.name]


def build_plan(name: str, spec=None) -> KernelPlan:
    """The named plan (plan.py:162-188); case-insensitive, ValueError on an
    unknown name."""
    key = str(name).upper()
    if key not in PLAN_NAMES:
        raise ValueError(f"unknown plan {name!r}; expected one of {PLAN_NAMES}")
    velocity = frozenset(VELOCITY_GRADIENT_IDS)
    table = {
        "BL": (True, frozenset(derivative_ids()), False, "grouped"),
        "RA": (False, frozenset(), False, "fused"),
        "SN": (False, frozenset(), True, "fused"),
        "RS": (False, velocity, False, "fused"),
        "SS": (False, velocity, True, "fused"),
    }
    store, to_store, locals_, prims = table[key]
    return KernelPlan(key, store, to_store, locals_, prims)


def plan_storage(plan: KernelPlan, spec=None) -> dict:
    """Storage class per derivative id (plan.py:61-73)."""
    out = {}
    for did in derivative_ids():
        if plan.store_derivatives or did in plan.derivatives_to_store:
            out[did] = FETCH
        elif plan.local_variables:
            out[did] = LOCAL
        else:
            out[did] = INLINE
    return out


def stencil_applications_per_point(plan: KernelPlan) -> int:
    """Stencil applications per grid point per residual evaluation, counted
    as the reference does (plan.py:248-264): FETCH costs 1 (the fill), LOCAL
    costs 1 (5 for a mixed term whose inner derivative is not stored),
    INLINE costs that times the derivative's occurrences in the residuals."""
    storage = plan_storage(plan)
    total = 0
    for did, cls in storage.items():
        cross = did.startswith("DD(")
        inner_stored = False
        if cross:
            j = did[4]
            inner_stored = storage[f"D(u{j},x{j})"] == FETCH
        cost = 5 if cross and not inner_stored else 1
        if cls == FETCH:
            total += 1
        elif cls == LOCAL:
            total += cost
        else:
            total += OCCURRENCES[did] * cost
    return total


# Occurrences of each derivative in the five residual expressions
# (terms.py:190-193), as the reference's term list spells them.
def _occurrences() -> dict:
    occ = {d: 0 for d in derivative_ids()}
    for j in range(3):          # mass
        occ[f"D(rhou{j},x{j})"] += 1
        occ[f"D(rho,x{j})"] += 1
        occ[f"D(u{j},x{j})"] += 1
    for i in range(3):          # momentum i
        for j in range(3):
            occ[f"D(rhou{i}*u{j},x{j})"] += 1
            occ[f"D(rhou{i},x{j})"] += 1
            occ[f"D(u{j},x{j})"] += 1
        occ[f"D(p,x{i})"] += 1
        occ[f"D2(u{i},x{i})"] += 1
        for j in range(3):
            if j != i:
                occ[f"D2(u{i},x{j})"] += 1
                occ[f"DD(u{j},x{i},x{j})"] += 1
    for j in range(3):          # energy: convection, pressure work, heat
        occ[f"D(rhoe*u{j},x{j})"] += 1
        occ[f"D(rhoe,x{j})"] += 1
        occ[f"D(u{j},x{j})"] += 1
        occ[f"D(u{j}*p,x{j})"] += 1
        occ[f"D2(T,x{j})"] += 1
    for i in range(3):          # stress work: tau_ij * D(u_i, x_j)
        for j in range(3):
            if i == j:
                occ[f"D(u{i},x{i})"] += 2
                for q in range(3):
                    occ[f"D(u{q},x{q})"] += 1
            else:
                occ[f"D(u{i},x{j})"] += 2
                occ[f"D(u{j},x{i})"] += 1
    for i in range(3):          # u_i * viscous_i
        occ[f"D2(u{i},x{i})"] += 1
        for j in range(3):
            if j != i:
                occ[f"D2(u{i},x{j})"] += 1
                occ[f"DD(u{j},x{i},x{j})"] += 1
    return occ


OCCURRENCES = _occurrences()


def workarray_budget(plan: KernelPlan, spec=None) -> int:
    """Grid-sized derivative arrays the plan allocates in HBM.

    The reference counts one array per FETCH derivative plus a product
    scratch (plan.py:220-227: BL 61).  Here products are formed in
    registers inside the fill kernel, so BL needs no scratch: BL 60,
    RS/SS 9, RA/SN 0."""
    return int(_lib.load(require_gpu=False).fdns_workarray_count(
        plan.variant_id))


class ResidualEvaluator:
    """Owns the work arrays of one (grid, plan) pair and evaluates the full
    residual on the device (plan.py:312-416).  `workers` is accepted for
    signature compatibility and ignored (one GPU per rank)."""

    def __init__(self, grid: Grid, constants: PhysicalConstants,
                 plan: KernelPlan | str, spec=None, workers: int = 1):
        if isinstance(plan, str):
            plan = build_plan(plan)
        self.grid = grid
        self.constants = constants
        self.plan = plan
        self.workers = workers
        self.lib = _lib.load()
        self.problem = grid.problem(constants)
        nw = workarray_budget(plan)
        self.work = alloc_bundle(grid, nw) if nw > 0 else None
        self._workspace = None

    @property
    def work_ptr(self) -> int:
        return 0 if self.work is None else _lib.ptr(self.work)

    def evaluate(self, state: ConservativeState, out: Residual) -> Residual:
        """Primitives, work-array fills and the residual kernel
        (plan.py:394-416).  Requires current conservative halos; writes the
        interior of `out`."""
        eval_primitives_fused(state, self.constants)
        _lib.check(self.lib.fdns_residual(
            self.plan.variant_id, _lib.ptr(state.bundle), self.work_ptr,
            _lib.ptr(out.bundle), self.problem, _lib.stream_handle()),
            f"residual ({self.plan.name})")
        return out

    def workspace(self):
        """Two extra state bundles for the fused, copy-free RK3 step."""
        if self._workspace is None:
            self._workspace = (alloc_bundle(self.grid, 10),
                               alloc_bundle(self.grid, 10))
        return self._workspace

    @property
    def wrap_mask(self) -> int:
        """Axes whose ghosts the stage kernel fills in place (all three on
        one GPU; axis 0 comes from the slab exchange on several)."""
        slab = self.grid.slab
        return 0b110 if slab is not None and slab.nranks > 1 else 0b111

    def stage(self, inp: torch.Tensor, saved: torch.Tensor, out: torch.Tensor,
              coef: float) -> None:
        """One fused RK stage (residual + update + primitives + periodic
        ghost images) into `out`."""
        _lib.check(self.lib.fdns_stage(
            self.plan.variant_id, _lib.ptr(inp), _lib.ptr(saved),
            _lib.ptr(out), self.work_ptr, coef, self.wrap_mask, self.problem,
            _lib.stream_handle()), f"stage ({self.plan.name})")


    def stage_planes(self, inp: torch.Tensor, saved: torch.Tensor,
                     out: torch.Tensor, coef: float, i_lo: int, i_hi: int,
                     with_fills: bool) -> None:
        """The fused stage on local axis-0 planes [i_lo, i_hi) only."""
        _lib.check(self.lib.fdns_stage_planes(
            self.plan.variant_id, _lib.ptr(inp), _lib.ptr(saved),
            _lib.ptr(out), self.work_ptr, coef, self.wrap_mask, i_lo, i_hi,
            int(with_fills), self.problem, _lib.stream_handle()),
            f"stage ({self.plan.name})")

    def stage_exchanged(self, inp: torch.Tensor, saved: torch.Tensor,
                        out: torch.Tensor, coef: float) -> None:
        """One stage of a z-slab rank with the halo exchange overlapped:
        the 2h boundary planes are updated first, their exchange runs on a
        communication stream while the interior planes are updated, and the
        launching stream then waits for the exchange."""
        slab, h = self.grid.slab, self.grid.halo
        n = self.grid.local_npoints[0]
        if n < 2 * h:
            self.stage(inp, saved, out, coef)
            slab.exchange(out, h)
            return
        main = torch.cuda.current_stream()
        if getattr(self, "_comm", None) is None:
            self._comm = torch.cuda.Stream()
        self.stage_planes(inp, saved, out, coef, 0, h, True)
        self.stage_planes(inp, saved, out, coef, n - h, n, False)
        self._comm.wait_stream(main)
        with torch.cuda.stream(self._comm):
            slab.exchange(out, h)
        self.stage_planes(inp, saved, out, coef, h, n - h, False)
        main.wait_stream(self._comm)


def assemble_residual(state: ConservativeState, constants: PhysicalConstants,
                      plan: KernelPlan | str, spec=None,
                      workers: int = 1) -> Residual:
    """One-shot residual assembly (plan.py:419-426)."""
    ev = ResidualEvaluator(state.grid, constants, plan, spec, workers)
    out = Residual(state.grid)
    return ev.evaluate(state, out)
