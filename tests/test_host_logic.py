"""Host-side logic mirrored from the reference (CPU only): plan selector,
storage classes, grid validation, RK scheme, stencil weights, slab
partitioning, time-series I/O."""

import math

import numpy as np
import pytest

import paper_1610_09146_b200 as fd
from paper_1610_09146_b200 import plan as fplan
from oracle import numpy_oracle as npo


def test_plan_names_and_selector():
    assert fd.PLAN_NAMES == ("BL", "RA", "RS", "SN", "SS")   # plan.py:33
    assert fd.build_plan("ss").name == "SS"                   # case-insensitive
    with pytest.raises(ValueError):
        fd.build_plan("XX")
    assert fd.build_plan("BL").primitives == "grouped"
    for n in ("RA", "RS", "SN", "SS"):
        assert fd.build_plan(n).primitives == "fused"


def test_term_list_counts():
    ids = fplan.derivative_ids()
    assert len(ids) == len(set(ids)) == 60                   # test_plan.py:23
    kinds = {"d1": 0, "d2": 0, "cross": 0}
    for d in ids:
        kinds["cross" if d.startswith("DD") else
              "d2" if d.startswith("D2") else "d1"] += 1
    assert kinds == {"d1": 42, "d2": 12, "cross": 6}
    assert set(fplan.VELOCITY_GRADIENT_IDS) <= set(ids)


def test_storage_invariants():
    velocity = set(fplan.VELOCITY_GRADIENT_IDS)
    expect = {"BL": lambda d: fplan.FETCH, "RA": lambda d: fplan.INLINE,
              "SN": lambda d: fplan.LOCAL,
              "RS": lambda d: fplan.FETCH if d in velocity else fplan.INLINE,
              "SS": lambda d: fplan.FETCH if d in velocity else fplan.LOCAL}
    for name, f in expect.items():
        for did, cls in fd.plan_storage(fd.build_plan(name)).items():
            assert cls == f(did), (name, did)


def test_workarray_budgets(built):
    b = {n: fd.workarray_budget(fd.build_plan(n)) for n in fd.PLAN_NAMES}
    # reference: BL 61 = 60 arrays + product scratch (plan.py:220-227);
    # products are formed in registers here, so the scratch is gone
    assert b == {"BL": 60, "RA": 0, "RS": 9, "SN": 0, "SS": 9}


def test_grid_validation():
    with pytest.raises(fd.ConfigurationError):
        fd.make_grid((4, 8, 8), (1, 1, 1))
    with pytest.raises(fd.ConfigurationError):
        fd.make_grid((8, 8, 8), (1, -1, 1))
    with pytest.raises(fd.ConfigurationError):
        fd.make_grid((8, 8, 8), (1, 1, 1), halo=1)
    with pytest.raises(fd.ConfigurationError):
        fd.make_grid((8, 8), (1, 1))
    g = fd.make_grid((8, 10, 12), (2 * math.pi,) * 3, halo=3)
    assert g.shape == (14, 16, 18)
    assert g.delta[1] == (2 * math.pi) / 10


def test_stencil_weights_match_oracle():
    from paper_1610_09146_b200.stencil import make_weights
    for n in (5, 16, 64, 512):
        d = (2 * math.pi) / n
        w = make_weights(d)
        assert (*w.first, *w.second) == npo.weights(d)


def test_problem_descriptor():
    g = fd.make_grid((16, 12, 8), (2 * math.pi,) * 3)
    c = fd.PhysicalConstants()
    pb = g.problem(c)
    assert list(pb.n) == [16, 12, 8] and pb.h == 2
    flat = [x for a in npo.grid_weights((16, 12, 8)) for x in a]
    assert list(pb.w) == flat
    assert list(pb.kc) == list(c.kernel_constants())
    assert (pb.gm1, pb.gM2) == (c.gm1, c.gM2)


def test_rk_scheme_validation():
    s = fd.RKScheme(dt=0.1)
    assert s.stages == 3 and s.alpha == (1.0 / 3.0, 0.5, 1.0)
    with pytest.raises(ValueError):
        fd.RKScheme(dt=0.0)
    with pytest.raises(ValueError):
        fd.RKScheme(dt=0.1, alpha=(0.5, 0.5, 0.5))


def test_rk_stability_polynomial():
    # save-state composition == 1 + z + z^2/2 + z^3/6 (test_timeloop.py:47-53)
    for z in (0.05, -0.3, 0.5 + 0.2j, -1.0 + 1.0j):
        u = 1.0
        for a in fd.RK3_ALPHA:
            u = 1.0 + a * z * u
        exact = 1.0 + z + z ** 2 / 2.0 + z ** 3 / 6.0
        assert abs(u - exact) <= 1e-13 * max(1.0, abs(exact))


@pytest.mark.parametrize("n0,nranks", [(64, 1), (64, 2), (64, 8), (67, 3),
                                       (1024, 8)])
def test_slab_partition_covers_axis(n0, nranks):
    slabs = [fd.Slab.partition(n0, r, nranks) for r in range(nranks)]
    assert sum(s.local_n0 for s in slabs) == n0
    assert slabs[0].offset0 == 0
    for a, b in zip(slabs, slabs[1:]):
        assert b.offset0 == a.offset0 + a.local_n0
    assert max(s.local_n0 for s in slabs) - min(s.local_n0 for s in slabs) <= 1
    assert slabs[0].down == nranks - 1 and slabs[-1].up == 0


def test_slab_needs_halo_planes():
    s = fd.Slab.partition(8, 0, 8)
    with pytest.raises(fd.ConfigurationError):
        fd.make_grid((8, 8, 8), (1, 1, 1), slab=s)


def test_slab_grid_coordinates():
    s = fd.Slab.partition(16, 1, 2)
    g = fd.make_grid((16, 16, 16), (2 * math.pi,) * 3, slab=s)
    assert g.local_npoints == (8, 16, 16)
    assert g.shape == (12, 20, 20)
    np.testing.assert_array_equal(g.coordinates(0),
                                  np.arange(8, 16) * g.delta[0])


def test_timeseries_roundtrip(tmp_path):
    recs = [fd.DiagnosticsRecord(0.1 * i, 0.125 + i * 1e-17, 0.375, 1.0,
                                 (0.0, 1e-300, -2.5), 178.6) for i in range(3)]
    p = tmp_path / "ts.csv"
    fd.write_timeseries(recs, p)
    assert p.read_text().splitlines()[0] == \
        "time,ke,enstrophy,mass,mom0,mom1,mom2,energy"
    assert fd.read_timeseries(p) == recs
    p.write_text("bad,header\n")
    with pytest.raises(ValueError):
        fd.read_timeseries(p)


def test_no_cpu_fallback_without_gpu(built):
    """The product path fails loudly when no CUDA device is present."""
    import torch
    from paper_1610_09146_b200 import _lib
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    g = fd.make_grid((8, 8, 8), (2 * math.pi,) * 3)
    with pytest.raises(_lib.FdnsError):
        fd.taylor_green_init(g, fd.PhysicalConstants())


def test_plan_introspection_matches_reference(built, golden_meta):
    """Occurrence counts, stencil applications per point and work-array
    budgets against the values the reference itself reports
    (terms.py:190-193, plan.py:220-264; tests/golden/make_golden.py)."""
    from paper_1610_09146_b200.plan import (OCCURRENCES,
                                            stencil_applications_per_point)
    assert OCCURRENCES == golden_meta["occurrences"]
    for name, want in golden_meta["stencil_applications_per_point"].items():
        assert stencil_applications_per_point(fd.build_plan(name)) == want
    ref = golden_meta["workarray_budget"]
    assert ref == {"BL": 61, "RA": 0, "RS": 9, "SN": 0, "SS": 9}
    # identical except BL's product scratch array, which this design drops
    for name in fd.PLAN_NAMES:
        assert fd.workarray_budget(fd.build_plan(name)) == \
            ref[name] - (1 if name == "BL" else 0)


def test_bench_tables_formats(tmp_path):
    """bench.csv / speedup.csv / scaling.csv in the reference's formats
    (bench.py:108-126, 199-205)."""
    from paper_1610_09146_b200 import benchtables as bt
    assert bt.auto_dt((64, 64, 64)) == 3.385e-3
    assert abs(bt.auto_dt((128,) * 3) - 3.385e-3 / 2) < 1e-18
    recs = [bt.TimingRecord((64,) * 3, p, 1, 100, t)
            for p, t in (("BL", 2.0), ("SN", 0.5), ("SS", 1.0))]
    bt.write_bench_csv(recs, tmp_path / "bench.csv")
    lines = (tmp_path / "bench.csv").read_text().splitlines()
    assert lines[0] == "Nx,Ny,Nz,plan,workers,iterations,loop_seconds"
    assert lines[2] == "64,64,64,SN,1,100,0.500000"
    bt.write_speedup_csv(recs, tmp_path / "speedup.csv")
    sp = (tmp_path / "speedup.csv").read_text().splitlines()
    assert sp == ["Nx,Ny,Nz,BL,SN,SS", "64,64,64,1.0000,4.0000,2.0000"]
    bench_lines = [{"n_gpus": n, "ms_per_step": 1.0 / n * 1.1 ** (n > 1),
                    "steps": 10, "config": {"grid": [256, 256, 256]}}
                   for n in (1, 2, 4, 8)]
    sc = bt.scaling_records(bench_lines)
    assert [r.ideal for r in sc] == [1.0, 0.5, 0.25, 0.125]
    bt.write_scaling_csv(sc, tmp_path / "scaling.csv")
    assert (tmp_path / "scaling.csv").read_text().splitlines()[0] == \
        "workers,Nx,Ny,Nz,runtime,normalized,ideal"


def test_plan_lowering_and_race_validator():
    """plan.py:196-310 restated for the device schedule: every shipped plan
    lowers (race-free, dependencies satisfied); the reference's criterion-10
    counterexample (a fused primitives pass that reads the velocities it
    writes, test_acceptance.py:238-260) is rejected naming exactly u0-u2;
    a pass reading a field nobody produced is rejected."""
    import dataclasses
    import pytest
    import paper_1610_09146_b200 as fd
    for n in fd.PLAN_NAMES:
        plan = fd.build_plan(n)
        assert fd.validate_race_freedom(plan) == []
        sched = fd.lower_plan(plan)
        assert sched.fetch_ids == [d for d, c in fd.plan_storage(plan).items() if c == "FETCH"]
        want_inner = [] if n in ("RA", "SN") else ["D(u0,x0)", "D(u1,x1)", "D(u2,x2)"]
        assert sched.inner_halo_ids == want_inner
        text = sched.listing()
        assert f"plan {n}" in text and "loop groups:" in text
        assert f"stencil applications/point {sched.stencil_applications_per_point()}" in text
    bad_group = fd.LoopGroup(
        "primitives:bad-fusion", "loop", frozenset({"u0", "u1", "u2", "p"}),
        frozenset({"rho", "rhou0", "rhou1", "rhou2", "rhoE", "u0", "u1", "u2"}))
    template = fd.build_plan("BL")
    bad = dataclasses.replace(template, loop_groups=(bad_group,) + template.loop_groups[1:])
    assert {(v.group, v.field) for v in fd.validate_race_freedom(bad)} == {
        ("primitives:bad-fusion", "u0"), ("primitives:bad-fusion", "u1"),
        ("primitives:bad-fusion", "u2")}
    with pytest.raises(ValueError, match="not race-free"):
        fd.lower_plan(bad)
    early = fd.LoopGroup("fill:early", "loop", frozenset({"wa_x"}), frozenset({"T"}))
    unsat = dataclasses.replace(template, loop_groups=(early,) + template.loop_groups)
    with pytest.raises(ValueError, match="before they are produced"):
        fd.lower_plan(unsat)


def test_terms_registry_matches_reference_goldens(golden_meta):
    """terms.build_residual_spec (terms.py:135-200): the 60 derivatives (42
    d1 incl. 18 product targets, 12 d2, 6 cross), their occurrence counts
    pinned to the reference's own spec, the nine velocity-gradient ids and
    the reference's identifier spelling; only the internal-energy form."""
    import pytest
    import paper_1610_09146_b200 as fd
    spec = fd.terms.build_residual_spec()
    kinds = [d.kind for d in spec.derivatives.values()]
    assert (kinds.count("d1"), kinds.count("d2"), kinds.count("cross")) == (42, 12, 6)
    assert sum(d.is_product for d in spec.derivatives.values()) == 18
    assert spec.occurrences == golden_meta["occurrences"]
    assert len(spec.velocity_gradient_ids) == 9
    assert spec.derivatives["DD(u1,x0,x1)"].inner_id == "D(u1,x1)"
    assert spec.derivatives["D(rhou0*u1,x1)"].name == "d_rhou0u1_x1"
    assert fd.plan.DEFAULT_SPEC.occurrences == spec.occurrences
    with pytest.raises(ValueError):
        fd.terms.build_residual_spec("total")


def test_spec_check_rejects_other_term_lists():
    """ResidualEvaluator(spec=...) no longer ignores spec: the default term
    list passes, anything else raises (plan.check_spec)."""
    from dataclasses import dataclass, field
    fplan.check_spec(None)
    fplan.check_spec(fd.terms.DEFAULT_SPEC)
    fplan.check_spec(fd.terms.build_residual_spec())

    @dataclass
    class D:
        expr: str

    @dataclass
    class Spec:
        derivatives: dict = field(default_factory=dict)

    ok = Spec({d: D("x") for d in fplan.derivative_ids()})
    ok.derivatives["D(rhoe,x0)"] = D(fd.terms.RHOE_INTERNAL)
    fplan.check_spec(ok)                          # a reference-built default spec
    total = Spec({d: D("x") for d in fplan.derivative_ids()})
    total.derivatives["D(rhoe,x0)"] = D("rhoE")   # energy_phi="total"
    with pytest.raises(NotImplementedError):
        fplan.check_spec(total)
    with pytest.raises(NotImplementedError):
        fplan.check_spec(Spec({"D(rho,x0)": D("rho")}))
    with pytest.raises(ValueError):
        fd.terms.build_residual_spec("total")


def test_decompose_workers_and_scaling_drivers():
    """decompose_workers (bench.py:160-173 semantics) and the strong/weak
    drivers' normalisation, with a stand-in timer (no GPU)."""
    from paper_1610_09146_b200 import benchtables as bt
    assert bt.decompose_workers(1) == (1, 1, 1)
    assert bt.decompose_workers(2) == (2, 1, 1)
    assert bt.decompose_workers(4) == (2, 2, 1)
    assert bt.decompose_workers(8) == (2, 2, 2)
    assert bt.decompose_workers(12) == (3, 2, 2)
    assert bt.decompose_workers(6) == (3, 2, 1)
    calls = []

    def timer(npoints, plan, gpus, iterations, constants=None, repeats=1):
        calls.append((npoints, gpus))
        sec = float(np.prod(npoints)) / gpus * 1e-6   # perfect scaling
        return bt.TimingRecord(tuple(npoints), plan, gpus, iterations, sec)

    st = bt.strong_scaling((64, 64, 64), "SS", [1, 2, 4, 8], 10, timer=timer)
    assert [r.ideal for r in st] == [1.0, 0.5, 0.25, 0.125]
    assert [r.normalized for r in st] == pytest.approx([1, 0.5, 0.25, 0.125])
    wk = bt.weak_scaling((32, 32, 32), "SN", [1, 2, 4, 8], 10, timer=timer)
    assert [r.grid for r in wk] == [(32, 32, 32), (64, 32, 32),
                                    (64, 64, 32), (64, 64, 64)]
    assert all(r.ideal == 1.0 for r in wk)
    assert [r.normalized for r in wk] == pytest.approx([1, 1, 1, 1])


@pytest.mark.parametrize("n0,K", [(512, 32), (128, 8), (44, 5), (40, 4), (257, 16)])
def test_wave_schedule_is_a_valid_order(n0, K):
    """hostio.wave_schedule (the e2e wavefront): every chunk's primitives
    and three stages appear once, each after what it reads (stage 1: the
    primitives of c-1..c+1 without wrap, whose planes include the ghosts;
    stages 2-3: the previous stage on c-1..c+1 around the ring); chunk
    ranges tile the interior and the padded planes exactly."""
    from paper_1610_09146_b200.hostio import wave_schedule
    h = 2
    s = wave_schedule(n0, h, K)
    assert sorted(s["order"]) == list(range(K))
    it = s["interior"]
    assert it[0][0] == 0 and it[-1][1] == n0
    assert all(it[c][1] == it[c + 1][0] and it[c][1] - it[c][0] >= n0 // K for c in range(K - 1))
    pd = s["padded"]
    assert pd[0][0] == 0 and pd[-1][1] == n0 + 2 * h
    assert all(pd[c][1] == pd[c + 1][0] for c in range(K - 1))
    assert all(pd[c] == (it[c][0] + h, it[c][1] + h) for c in range(1, K - 1))
    seen = set()
    for item in s["seq"]:
        assert item not in seen
        if item[0] == "S":
            _, sg, c = item
            if sg == 1:
                need = {("P", x) for x in (c - 1, c, c + 1) if 0 <= x < K}
            else:
                need = {("S", sg - 1, x % K) for x in (c - 1, c, c + 1)}
            assert need <= seen, (item, need - seen)
        seen.add(item)
    assert seen == {("P", c) for c in range(K)} | {
        ("S", sg, c) for sg in (1, 2, 3) for c in range(K)}
    assert s["download_needs"][0] == {K - 1, 0, 1 % K}
    # the first chunk's third stage comes before the last upload: the
    # downloads start while uploads are still running
    first_s3 = next(i for i, x in enumerate(s["seq"]) if x[:2] == ("S", 3))
    last_p = max(i for i, x in enumerate(s["seq"]) if x[0] == "P")
    if K >= 8:
        assert first_s3 < last_p
