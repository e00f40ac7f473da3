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

from . import _lib, parity
from .mesh import Grid, alloc_bundle, as_grid
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


STATE_FIELDS = ("rho", "rhou0", "rhou1", "rhou2", "rhoE")
POINT_FIELDS = STATE_FIELDS + ("u0", "u1", "u2", "p", "T")
RESIDUAL_FIELDS = ("d_rho", "d_rhou0", "d_rhou1", "d_rhou2", "d_rhoE")


@dataclass(frozen=True)
class LoopGroup:
    """One device pass (or a halo barrier) with its grid-field footprint
    (plan.py:40-47).  Here a group is one kernel of the evaluation."""

    name: str
    kind: str  # "loop" or "halo"
    writes: frozenset
    reads: frozenset


@dataclass(frozen=True)
class KernelPlan:
    """plan.py:51-58; `loop_groups` lists the device passes of one residual
    evaluation (see `_device_groups`)."""

    name: str
    store_derivatives: bool
    derivatives_to_store: frozenset
    local_variables: bool
    primitives: str  # "grouped" or "fused" (the reference's form; the
    #                  device runs the fused pass, bitwise equal)
    loop_groups: tuple = ()

    @property
    def variant_id(self) -> int:
        return _lib.VARIANT_IDS[self.name]


def _wa(did: str) -> str:
    return "wa_" + did


def _device_groups(name: str, storage: dict) -> tuple:
    """The kernels one evaluation runs, with their field footprints:
    primitives (one fused pass over the conservative fields, physics.py:
    185-202); BL: the 54 plain/product fills in one kernel (products formed
    in registers, no scratch array), the ghost frames of the three inner
    arrays (the reference's inner halo exchange, plan.py:378-379) and the
    six mixed fills; RS/SS: the nine velocity gradients (+ their ghost
    frames) in one kernel; then the residual kernel."""
    fetched = [d for d in derivative_ids() if storage[d] == FETCH]
    groups = [LoopGroup("primitives:fused", "loop",
                        frozenset({"u0", "u1", "u2", "p", "T"}),
                        frozenset(STATE_FIELDS))]
    if name == "BL":
        plain = frozenset(_wa(d) for d in fetched if not d.startswith("DD("))
        inner = frozenset(_wa(f"D(u{q},x{q})") for q in range(3))
        cross = frozenset(_wa(d) for d in fetched if d.startswith("DD("))
        groups += [LoopGroup("fill:plain+products", "loop", plain, frozenset(POINT_FIELDS)),
                   LoopGroup("halo:velocity-divergence-arrays", "halo", inner, inner),
                   LoopGroup("fill:cross", "loop", cross, inner)]
    elif fetched:
        grads = frozenset(_wa(d) for d in fetched)
        groups += [LoopGroup("fill:velocity-gradients", "loop", grads,
                             frozenset({"u0", "u1", "u2"}))]
    groups.append(LoopGroup("residual", "loop", frozenset(RESIDUAL_FIELDS),
                            frozenset(POINT_FIELDS) | frozenset(_wa(d) for d in fetched)))
    return tuple(groups)


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
    plan = KernelPlan(key, store, to_store, locals_, prims)
    return KernelPlan(key, store, to_store, locals_, prims,
                      _device_groups(key, plan_storage(plan)))


@dataclass(frozen=True)
class RaceViolation:
    group: str
    field: str


def validate_race_freedom(plan: KernelPlan) -> list:
    """plan.py:196-213: the (group, field) pairs where a grid pass writes a
    field it also reads (halo barriers skipped); [] means race-free."""
    out = []
    for g in plan.loop_groups:
        if g.kind != "loop":
            continue
        for f in sorted(g.writes & g.reads):
            out.append(RaceViolation(g.name, f))
    return out


@dataclass
class KernelSchedule:
    """plan.py:229-283: a lowered plan."""

    plan: KernelPlan
    storage: dict
    loop_groups: tuple

    @property
    def fetch_ids(self) -> list:
        return [d for d in derivative_ids() if self.storage[d] == FETCH]

    @property
    def inner_halo_ids(self) -> list:
        """Inner derivatives of the mixed terms read from work arrays."""
        ids = []
        for d in derivative_ids():
            if d.startswith("DD("):
                inner = f"D(u{d[4]},x{d[4]})"
                if self.storage[inner] == FETCH and inner not in ids:
                    ids.append(inner)
        return ids

    def stencil_applications_per_point(self) -> int:
        return stencil_applications_per_point(self.plan)

    def listing(self) -> str:
        """Human-readable schedule (plan.py:266-283 layout)."""
        lines = [f"plan {self.plan.name}",
                 f"primitives {self.plan.primitives}",
                 f"work-array budget {workarray_budget(self.plan)}",
                 f"stencil applications/point {self.stencil_applications_per_point()}",
                 "", "loop groups:"]
        for g in self.loop_groups:
            lines.append(f"  [{g.kind}] {g.name}")
            lines.append(f"      writes: {', '.join(sorted(g.writes))}")
            lines.append(f"      reads:  {', '.join(sorted(g.reads))}")
        lines += ["", "derivative storage:"]
        for did in sorted(derivative_ids()):
            lines.append(f"  {did:24s} {self.storage[did]}")
        lines.append("")
        return "\n".join(lines)


def lower_plan(plan: KernelPlan, spec=None) -> KernelSchedule:
    """plan.py:290-310: lower a plan, rejecting racy groups and groups that
    read a field before any earlier group (or the state) produced it."""
    violations = validate_race_freedom(plan)
    if violations:
        raise ValueError(f"plan {plan.name} is not race-free: {violations}")
    available = set(STATE_FIELDS)
    for g in plan.loop_groups:
        missing = g.reads - available
        if missing:
            raise ValueError(f"group {g.name} reads {sorted(missing)} before "
                             "they are produced")
        available |= g.writes
    return KernelSchedule(plan, plan_storage(plan), plan.loop_groups)


def storage_classes(name: str, store_derivatives: bool,
                    derivatives_to_store: frozenset, local_variables: bool,
                    spec=None) -> dict:
    """Storage class per derivative id (plan.py:61-73)."""
    out = {}
    for did in derivative_ids():
        if store_derivatives or did in derivatives_to_store:
            out[did] = FETCH
        elif local_variables:
            out[did] = LOCAL
        else:
            out[did] = INLINE
    return out


def plan_storage(plan: KernelPlan, spec=None) -> dict:
    """Storage class per derivative id of a plan (plan.py:188-193)."""
    return storage_classes(plan.name, plan.store_derivatives,
                           plan.derivatives_to_store, plan.local_variables, spec)


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
        check_spec(spec)
        grid = as_grid(grid)
        self.grid = grid
        self.constants = constants
        self.plan = plan
        self.workers = workers
        self.lib = _lib.load()
        self.problem = grid.problem(constants)
        nw = workarray_budget(plan)
        self.work = alloc_bundle(grid, nw) if nw > 0 else None
        self._workspace = None
        self._twin = None        # parity mode: device twin of a host state

    @property
    def work_ptr(self) -> int:
        return 0 if self.work is None else _lib.ptr(self.work)

    def evaluate(self, state: ConservativeState, out: Residual) -> Residual:
        """Primitives, work-array fills and the residual kernel
        (plan.py:394-416).  Requires current conservative halos; writes the
        interior of `out`.  `state`/`out` may also be the reference's numpy
        objects (parity mode, `parity.py`): copied in and out around the
        device path, with the reference's side effects."""
        if parity.is_host_state(state) or parity.is_host_residual(out):
            return self._evaluate_host(state, out)
        eval_primitives_fused(state, self.constants)
        _lib.check(self.lib.fdns_residual(
            self.plan.variant_id, _lib.ptr(state.bundle), self.work_ptr,
            _lib.ptr(out.bundle), self.problem, _lib.stream_handle()),
            f"residual ({self.plan.name})")
        return out

    def twin(self):
        """Device state + residual that stand in for host objects."""
        if self._twin is None:
            self._twin = (ConservativeState(self.grid), Residual(self.grid))
        return self._twin

    def _evaluate_host(self, state, out):
        dev_state, dev_out = self.twin()
        if parity.is_host_state(state):
            parity.upload_conservative(state, dev_state)
        elif isinstance(state, ConservativeState):
            dev_state.bundle[:5].copy_(state.bundle[:5])
        else:
            raise TypeError("evaluate: state must be a ConservativeState or "
                            "expose field_arrays() of ten numpy arrays")
        self.evaluate(dev_state, dev_out)
        if parity.is_host_state(state):
            parity.download_primitives(dev_state.bundle, state)
        else:
            state.bundle[5:].copy_(dev_state.bundle[5:])
        parity.write_residual(dev_out, out)
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
        return 0b110 if slab is not None and slab.distributed else 0b111

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

    def stage_boundary(self, inp: torch.Tensor, saved: torch.Tensor,
                       out: torch.Tensor, coef: float) -> None:
        """The first half of an overlapped slab stage: the work-array fills
        and the h planes at each end of the slab, back to back on the
        launching stream (two small launches; running the second on a side
        stream measured slower at 64^3 -- the cross-stream join costs more
        than the launch it overlaps, tools/split_cost.py)."""
        h = self.grid.halo
        n = self.grid.local_npoints[0]
        self.stage_planes(inp, saved, out, coef, 0, h, True)
        self.stage_planes(inp, saved, out, coef, n - h, n, False)

    def stage_interior(self, inp: torch.Tensor, saved: torch.Tensor,
                       out: torch.Tensor, coef: float) -> None:
        """The second half: the planes between the boundary planes."""
        h = self.grid.halo
        n = self.grid.local_npoints[0]
        self.stage_planes(inp, saved, out, coef, h, n - h, False)

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
            slab.exchange_state(out, h, self.problem)
            return
        main = torch.cuda.current_stream()
        if getattr(self, "_comm", None) is None:
            self._comm = torch.cuda.Stream()
        self.stage_boundary(inp, saved, out, coef)
        self._comm.wait_stream(main)
        with torch.cuda.stream(self._comm):
            slab.exchange_state(out, h, self.problem)
        self.stage_interior(inp, saved, out, coef)
        main.wait_stream(self._comm)


def assemble_residual(state: ConservativeState, constants: PhysicalConstants,
                      plan: KernelPlan | str, spec=None,
                      workers: int = 1) -> Residual:
    """One-shot residual assembly (plan.py:419-426); a reference-style host
    state gets a numpy residual back (parity mode)."""
    ev = ResidualEvaluator(state.grid, constants, plan, spec, workers)
    out = (parity.HostResidual(ev.grid) if parity.is_host_state(state)
           else Residual(state.grid))
    return ev.evaluate(state, out)


def check_spec(spec) -> None:
    """The kernels are compiled for the reference's default term list
    (terms.build_residual_spec(), energy_phi="internal", terms.py:135-200).
    Accept None, that spec, or any registry with the same 60 derivatives
    whose `rhoe` is the internal energy; anything else (e.g. the
    energy_phi="total" list) raises instead of being silently ignored."""
    if spec is None:
        return
    from .terms import DEFAULT_SPEC, RHOE_INTERNAL
    if spec is DEFAULT_SPEC:
        return
    derivs = getattr(spec, "derivatives", None)
    if not isinstance(derivs, dict) or set(derivs) != set(derivative_ids()):
        raise NotImplementedError(
            "spec: the device kernels implement the reference's default "
            "term list only (60 derivatives, terms.py:135-200)")
    rhoe = getattr(derivs.get("D(rhoe,x0)"), "expr", None)
    if rhoe != RHOE_INTERNAL:
        raise NotImplementedError(
            "spec: the device kernels implement energy_phi='internal' only "
            f"(rhoe = {RHOE_INTERNAL}); got rhoe = {rhoe!r}")


# The reference's product scratch array name (plan.py:37).  The device fill
# forms products in registers, so no plan allocates it (workarray_budget).
SCRATCH = "scratch0"

from .terms import DEFAULT_SPEC  # noqa: E402  (terms reads this module's tables)
