"""GPU parity: every variant's CUDA path against the reference's golden
vectors and the (reference-pinned) CPU oracle, through the C ABI.

Tolerance: the north star allows rel-Linf <= 1e-12 per residual evaluation
and 1e-10 on fields / KE / enstrophy histories over 100 steps; the kernels
are built bitwise-faithful (-fmad=false, reference association), so the
gates below demand EXACT equality wherever the reference is deterministic
and apply the stated tolerances only to the device-reduced diagnostics
(summation order differs from numpy's pairwise sum).
"""

import numpy as np
import pytest
import torch

from conftest import rel_linf, sha
from oracle import c_oracle, numpy_oracle as npo

pytestmark = pytest.mark.gpu

fd = pytest.importorskip("paper_1610_09146_b200")
TWO_PI = 2.0 * np.pi
C = fd.PhysicalConstants()
CO = npo.Consts()
VARIANTS = fd.PLAN_NAMES
NS_VARIANTS = ("BL", "RA", "SN", "SS")


@pytest.fixture(scope="module", autouse=True)
def _gpu(built):
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    torch.cuda.set_device(0)


def grid_of(npts):
    return fd.make_grid(npts, (TWO_PI,) * 3)


U0_F = 5   # bundle index of u0 (physics.py:115-119)


def state_from_cons(grid, cons):
    from paper_1610_09146_b200.diagnostics import state_from_conservative
    return state_from_conservative(grid, C, cons)


def host_cons(state):
    return state.grid.interior(state.bundle[:5]).cpu().numpy()


def residual_of(state, variant):
    res = fd.assemble_residual(state, C, variant)
    torch.cuda.synchronize()
    return res.interior_numpy()


# ---------------------------------------------------------------- residuals
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("tag,npts", [("m16", (16, 16, 16)),
                                      ("m_ragged", (9, 12, 7))])
def test_residual_matches_reference_golden(golden, variant, tag, npts):
    state = state_from_cons(grid_of(npts), golden[f"{tag}_cons"])
    R = residual_of(state, variant)
    ref = golden[f"{tag}_res"]
    worst = max(rel_linf(R[q], ref[q]) for q in range(5))
    assert worst <= 1e-12                      # north-star per-eval gate
    assert np.array_equal(R, ref), f"{variant}/{tag}: not bitwise (rel {worst})"


@pytest.mark.parametrize("variant", VARIANTS)
def test_perturbed_residual_matches_reference_golden(golden, golden_meta,
                                                     variant):
    F = npo.perturbed_taylor_green(16, CO, golden_meta["perturb_seed"])
    state = state_from_cons(grid_of((16,) * 3), npo.interior(F[:5], 2))
    assert np.array_equal(residual_of(state, variant), golden["p16_res"])


@pytest.mark.parametrize("variant", VARIANTS)
def test_residual_256_matches_c_oracle(variant):
    """Full-size single evaluation at 256^3 (C4's grid) against the C
    oracle, bitwise."""
    n = 256
    F = npo.perturbed_taylor_green(n, CO, 7)
    want = c_oracle.residual(F, CO)
    state = state_from_cons(grid_of((n,) * 3), npo.interior(F[:5], 2))
    got = residual_of(state, variant)
    assert np.array_equal(got, want)


def test_quiescent_state_zero_residual():
    n = 8
    shape = (n,) * 3
    cons = np.stack([np.ones(shape), np.zeros(shape), np.zeros(shape),
                     np.zeros(shape), np.full(shape, (1.0 / C.gM2) / C.gm1)])
    state = state_from_cons(grid_of(shape), cons)
    for v in VARIANTS:
        assert np.max(np.abs(residual_of(state, v))) <= 1e-12


# ------------------------------------------------------- primitives / halos
def test_primitives_known_answer(golden_meta):
    """test_physics.py:65-81 of the reference: rho=2, rhou=(2,0,0),
    rhoE=3 gives u=1, p=0.8, T=0.0056 (allclose), and the device bits equal
    the oracle's for the same input."""
    shape = (5, 5, 5)
    cons = np.stack([np.full(shape, 2.0), np.full(shape, 2.0),
                     np.zeros(shape), np.zeros(shape), np.full(shape, 3.0)])
    state = state_from_cons(grid_of(shape), cons)
    b = state.bundle.cpu().numpy()
    assert b[5, 3, 3, 3] == 1.0
    assert b[8, 3, 3, 3] == pytest.approx(0.8, rel=1e-14)
    assert b[9, 3, 3, 3] == pytest.approx(0.0056, rel=1e-13)
    F = npo.new_fields(shape)
    F[:5] = b[:5]
    c_oracle.primitives(F, CO)
    assert np.array_equal(F, b)


def test_primitives_bitwise_vs_oracle_over_padded():
    F = npo.perturbed_taylor_green(12, CO, 3)
    state = state_from_cons(grid_of((12,) * 3), npo.interior(F[:5], 2))
    assert np.array_equal(state.to_numpy(), F)


@pytest.mark.parametrize("npts,h", [((6, 7, 5), 2), ((8, 8, 8), 3)])
def test_halo_wrap_matches_reference_semantics(npts, h):
    rng = np.random.default_rng(1)
    g = fd.make_grid(npts, (1.0, 1.0, 1.0), halo=h)
    b = fd.mesh.alloc_bundle(g, 3)
    host = rng.standard_normal(b.shape)
    b.copy_(torch.from_numpy(host))
    fd.mesh.halo_exchange_bundle(g, b, 3)
    assert np.array_equal(b.cpu().numpy(), npo.halo_exchange(host.copy(), h))


# ------------------------------------------------------------- time loop
@pytest.mark.parametrize("variant", VARIANTS)
def test_fused_iteration_equals_unfused_substeps(variant):
    n = 12
    F = npo.perturbed_taylor_green(n, CO, 5)
    g = grid_of((n,) * 3)
    scheme = fd.RKScheme(dt=3e-3)
    ev = fd.ResidualEvaluator(g, C, variant)
    a = state_from_cons(g, npo.interior(F[:5], 2))
    it = fd.IterationState(a)
    it.save_state()
    res = fd.Residual(g)
    for k in range(3):
        fd.rk_substep(it, k, scheme, ev, res)
    b = state_from_cons(g, npo.interior(F[:5], 2))
    fd.advance_iteration(fd.IterationState(b), scheme, ev)
    assert np.array_equal(host_cons(a), host_cons(b))


@pytest.mark.parametrize("variant", VARIANTS)
def test_c1_tgv32_10_steps_matches_reference(golden_meta, variant):
    """Config C1 (TGV 32^3, 10 RK3 steps, dt=2e-3): final fields hash-equal
    to the reference's."""
    ref = golden_meta["c1_tgv32_bl"]
    g = grid_of((32,) * 3)
    state = fd.taylor_green_init(g, C)
    assert [sha(f) for f in host_cons(state)] == \
        golden_meta["tgv32_cons_sha256"]
    ev = fd.ResidualEvaluator(g, C, variant)
    fd.run(state, fd.RKScheme(dt=2e-3), ev, 10)
    assert [sha(f) for f in host_cons(state)] == ref["sha256"]


@pytest.mark.parametrize("variant", NS_VARIANTS)
def test_c2_tgv64_100_steps(golden_meta, variant):
    """Config C2: TGV 64^3, dt=3.385e-3, 100 RK3 steps on 1 GPU -- fields
    bitwise equal to the reference, KE/enstrophy/conservation histories
    within 1e-10."""
    ref = golden_meta["c2_tgv64"]
    g = grid_of((64,) * 3)
    state = fd.taylor_green_init(g, C)
    rho0 = fd.mean_density(state)
    assert abs(rho0 - ref["rho0"]) <= 1e-13 * ref["rho0"]
    ev = fd.ResidualEvaluator(g, C, variant)
    rep = fd.run(state, fd.RKScheme(dt=3.385e-3), ev, 100, cadence=10,
                 collect=fd.make_collector(g, ref["rho0"]))
    assert [sha(f) for f in host_cons(state)] == ref["sha256"]
    assert len(rep.records) == len(ref["history"])
    for rec, row in zip(rep.records, ref["history"]):
        assert rec.time == pytest.approx(row[0], rel=1e-15, abs=1e-15)
        assert abs(rec.kinetic_energy - row[1]) <= 1e-10 * abs(row[1])
        assert abs(rec.enstrophy - row[2]) <= 1e-10 * abs(row[2])
        assert abs(rec.total_mass - row[3]) <= 1e-10 * abs(row[3])
        assert abs(rec.total_energy - row[7]) <= 1e-10 * abs(row[7])


@pytest.mark.parametrize("variant", NS_VARIANTS)
def test_c3_perturbed_128_200_steps(golden_meta, variant):
    """Config C3: seeded perturbed TGV 128^3, dt=1.69e-3, 200 steps."""
    ref = golden_meta["c3_ptgv128"]
    F = npo.perturbed_taylor_green(128, CO, golden_meta["perturb_seed"])
    assert [sha(npo.interior(F[q], 2)) for q in range(5)] == \
        golden_meta["c3_ptgv128_cons0_sha256"]
    g = grid_of((128,) * 3)
    state = state_from_cons(g, npo.interior(F[:5], 2))
    ev = fd.ResidualEvaluator(g, C, variant)
    rep = fd.run(state, fd.RKScheme(dt=1.69e-3), ev, 200, cadence=20,
                 collect=fd.make_collector(g, ref["rho0"]))
    assert [sha(f) for f in host_cons(state)] == ref["sha256"]
    for rec, row in zip(rep.records, ref["history"]):
        assert abs(rec.kinetic_energy - row[1]) <= 1e-10 * abs(row[1])
        assert abs(rec.enstrophy - row[2]) <= 1e-10 * abs(row[2])


def _check_history(rep, ref, tol=1e-10):
    assert len(rep.records) == len(ref["history"])
    for rec, row in zip(rep.records, ref["history"]):
        assert rec.time == pytest.approx(row[0], rel=1e-15, abs=1e-15)
        assert abs(rec.kinetic_energy - row[1]) <= tol * abs(row[1])
        assert abs(rec.enstrophy - row[2]) <= tol * abs(row[2])
        assert abs(rec.total_mass - row[3]) <= tol * abs(row[3])
        assert abs(rec.total_energy - row[7]) <= tol * abs(row[7])


def _free_device():
    import gc
    gc.collect()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("variant", ["RA", "SS"])
def test_c4_tgv256_100_steps(golden_meta, variant):
    """Config C4 (BASELINE.json configs[3]): TGV 256^3, dt=8.5e-4, 100 RK3
    steps, the RA and SS variants on one GPU -- final fields bitwise equal
    to the reference's (hashes generated by the reference itself,
    tests/golden/make_golden.py --large), KE/enstrophy/mass/energy sampled
    every 10 steps within 1e-10."""
    ref = golden_meta["c4_tgv256"]
    g = grid_of((256,) * 3)
    state = fd.taylor_green_init(g, C)
    assert abs(fd.mean_density(state) - ref["rho0"]) <= 1e-13 * ref["rho0"]
    ev = fd.ResidualEvaluator(g, C, variant)
    rep = fd.run(state, fd.RKScheme(dt=8.5e-4), ev, 100, cadence=10,
                 collect=fd.make_collector(g, ref["rho0"]))
    assert [sha(f) for f in host_cons(state)] == ref["sha256"]
    _check_history(rep, ref)
    del state, ev
    _free_device()


@pytest.mark.parametrize("variant", NS_VARIANTS)
def test_c5_tgv512_matches_reference(golden_meta, variant):
    """Config C5 (BASELINE.json configs[4]): TGV 512^3 on one GPU (BL's 90
    padded fields ~99 GB of HBM), dt=4.2e-4, 2 RK3 steps -- the most the
    reference itself can run in the build container (62 GB host RAM) --
    every variant's final fields bitwise equal to the reference's, the
    diagnostics of every step within 1e-10.  A common-mode addressing bug at
    the bench's own size would show up here, not only in cross-variant
    agreement."""
    ref = golden_meta["c5_tgv512"]
    g = grid_of((512,) * 3)
    state = fd.taylor_green_init(g, C)
    ev = fd.ResidualEvaluator(g, C, variant)
    rep = fd.run(state, fd.RKScheme(dt=4.2e-4), ev, 2, cadence=1,
                 collect=fd.make_collector(g, ref["rho0"]))
    got = host_cons(state)
    assert [sha(f) for f in got] == ref["sha256"]
    assert [float(np.max(np.abs(f))) for f in got] == ref["absmax"]
    _check_history(rep, ref)
    del state, ev, got
    _free_device()


@pytest.mark.parametrize("variant", ["BL", "RA", "RS", "SN", "SS"])
def test_analytic_rhs_convergence(variant):
    """Known answer (test_plan.py:207-238): rho = 1, u = (sin x, 0, 0),
    p = p0 has closed-form residuals; the device residual is within 0.05 of
    them at 32^3 and converges at fourth order (error ratio 10-25 from 32^3
    to 64^3)."""
    c = C
    errs = []
    for n in (32, 64):
        g = grid_of((n,) * 3)
        shape = (n,) * 3
        x = (np.arange(n) * (2.0 * np.pi / n))[:, None, None]
        rho = np.ones(shape)
        u = [np.sin(x) + np.zeros(shape), np.zeros(shape), np.zeros(shape)]
        p0 = 1.0 / c.gM2
        F = npo.state_from_primitives(shape, CO, rho, u, np.full(shape, p0))
        st = state_from_cons(g, npo.interior(F[:5], 2))
        r = npo.interior(fd.assemble_residual(st, c, variant).bundle.cpu().numpy(), 2)
        d_rho = -np.cos(x) + np.zeros(shape)
        d_rhou0 = -np.sin(2 * x) - c.c43_inv_Re * np.sin(x) + np.zeros(shape)
        d_rhoE = (-(c.gamma / c.gm1) * p0 * np.cos(x) + c.c43_inv_Re * np.cos(2 * x)
                  + np.zeros(shape))
        errs.append(max(np.max(np.abs(r[0] - d_rho)), np.max(np.abs(r[1] - d_rhou0)),
                        np.max(np.abs(r[2])), np.max(np.abs(r[3])),
                        np.max(np.abs(r[4] - d_rhoE))))
    assert errs[0] <= 0.05
    assert 10.0 <= errs[0] / errs[1] <= 25.0


def test_cross_plan_equivalence_50_iterations():
    """The reference's criterion 1 (test_acceptance.py:35-55): all five
    plans after 50 iterations of the 32^3 TGV agree to 1e-10 (here
    bitwise)."""
    g = grid_of((32,) * 3)
    finals = {}
    for v in VARIANTS:
        st = fd.taylor_green_init(g, C)
        fd.run(st, fd.RKScheme(dt=6.77e-3), fd.ResidualEvaluator(g, C, v), 50)
        finals[v] = host_cons(st)
    for v in VARIANTS:
        assert np.array_equal(finals[v], finals["BL"]), v


def test_rk3_temporal_order_on_device():
    """The scheme's temporal accuracy (criterion 9, test_acceptance.py:
    207-235) observed through the device time loop: the TGV at 16^3 to
    t = 0.08 with dt halved twice; the error against a dt/8 run shrinks by
    >= 4x per halving."""
    g = grid_of((16,) * 3)
    T = 0.08
    finals = {}
    for k in (1, 2, 4, 8):
        st = fd.taylor_green_init(g, C)
        dt = 0.02 / k
        fd.run(st, fd.RKScheme(dt=dt), fd.ResidualEvaluator(g, C, "SN"),
               int(round(T / dt)))
        finals[k] = host_cons(st)
    errs = [np.max(np.abs(finals[k] - finals[8])) for k in (1, 2)]
    assert errs[0] > 0 and errs[0] / errs[1] >= 4.0


def test_field_stencil_operators_match_oracle():
    """stencil.first/second/cross_derivative on device Fields (the reference's
    field-level operators, stencil.py:71-121) bitwise equal to the oracle's
    stencils; the interior only is written (halo stays zero)."""
    npts = (20, 36, 28)
    F = npo.manufactured(npts, CO)
    g = grid_of(npts)
    w = npo.grid_weights(npts)
    f = fd.Field(g)
    f.data.copy_(torch.from_numpy(np.ascontiguousarray(F[U0_F])))
    for axis in range(3):
        d = fd.first_derivative(f, axis).numpy()
        assert np.array_equal(npo.interior(d, 2), npo.d1(F[U0_F], 2, axis, w))
        assert np.all(d[:2] == 0) and np.all(d[:, :, -2:] == 0)
        d2 = fd.second_derivative(f, axis).numpy()
        assert np.array_equal(npo.interior(d2, 2), npo.d2(F[U0_F], 2, axis, w))
    inner = np.zeros_like(F[U0_F])
    npo.interior(inner, 2)[...] = npo.d1(F[U0_F], 2, 2, w)
    npo.halo_exchange(inner[None], 2)
    want = npo.d1(inner, 2, 0, w)
    assert np.array_equal(npo.interior(fd.cross_derivative(f, 0, 2).numpy(), 2), want)
    with pytest.raises(ValueError):
        fd.cross_derivative(f, 1, 1)


def test_vorticity_and_physics_helpers():
    """diagnostics.vorticity, physics.stress_tensor / heat_flux /
    skew_convective (physics.py:205-253) on the device, bitwise equal to the
    same formulas over the oracle's stencils."""
    npts = (16, 20, 24)
    F = npo.manufactured(npts, CO)
    g = grid_of(npts)
    w = npo.grid_weights(npts)
    st = state_from_cons(g, npo.interior(F[:5], 2))
    P = st.bundle.cpu().numpy()
    d = {(q, a): npo.d1(P[U0_F + q], 2, a, w) for q in range(3) for a in range(3)}
    om = fd.vorticity(st)
    want = [d[(2, 1)] - d[(1, 2)], d[(0, 2)] - d[(2, 0)], d[(1, 0)] - d[(0, 1)]]
    for got, ref in zip(om, want):
        assert np.array_equal(npo.interior(got.numpy(), 2), ref)
    grad = [[torch.from_numpy(np.ascontiguousarray(d[(q, a)])).cuda() for a in range(3)]
            for q in range(3)]
    tau = fd.stress_tensor(grad, C)
    div = d[(0, 0)] + d[(1, 1)] + d[(2, 2)]
    for i in range(3):
        for j in range(3):
            ref = C.inv_Re * (d[(i, j)] + d[(j, i)])
            if i == j:
                ref = ref - C.c23_inv_Re * div
            assert np.array_equal(tau[i][j].cpu().numpy(), ref)
    q = fd.heat_flux([grad[0][0]], C)[0]
    assert np.array_equal(q.cpu().numpy(), C.heat_coeff * d[(0, 0)])
    sk = fd.skew_convective(st.u[1], st.u[0], st.rho, 0).numpy()
    m = P[0] * P[U0_F + 1]
    fl = m * P[U0_F]
    ref = 0.5 * (npo.d1(fl, 2, 0, w) + npo.interior(P[U0_F], 2) * npo.d1(m, 2, 0, w)
                 + npo.interior(m, 2) * npo.d1(P[U0_F], 2, 0, w))
    assert np.array_equal(npo.interior(sk, 2), ref)


def test_cross_variant_bitwise_after_steps():
    n = 48
    F = npo.perturbed_taylor_green(n, CO, 11)
    g = grid_of((n,) * 3)
    finals = {}
    for v in VARIANTS:
        s = state_from_cons(g, npo.interior(F[:5], 2))
        fd.run(s, fd.RKScheme(dt=4e-3), fd.ResidualEvaluator(g, C, v), 5)
        finals[v] = host_cons(s)
    for v in VARIANTS:
        assert np.array_equal(finals[v], finals["BL"]), v


def test_bitwise_reproducible():
    g = grid_of((16,) * 3)
    runs = []
    for _ in range(2):
        s = fd.taylor_green_init(g, C)
        fd.run(s, fd.RKScheme(dt=6.77e-3), fd.ResidualEvaluator(g, C, "SS"), 3)
        runs.append(host_cons(s))
    assert np.array_equal(*runs)


def test_divergence_reported_with_location():
    g = grid_of((8,) * 3)
    s = fd.taylor_green_init(g, C)
    with pytest.raises(fd.SolverDivergenceError) as err:
        fd.run(s, fd.RKScheme(dt=50.0), fd.ResidualEvaluator(g, C, "SS"), 50,
               cadence=1)
    assert err.value.iteration is not None


# ------------------------------------------------------------ diagnostics
def test_tgv_initial_integrals(golden_meta):
    g = grid_of((32,) * 3)
    s = fd.taylor_green_init(g, C)
    rho0 = fd.mean_density(s)
    assert abs(rho0 - golden_meta["tgv32_rho0"]) <= 1e-14
    ke = fd.kinetic_energy_integral(s, g, rho0)
    en = fd.enstrophy_integral(s, g, rho0)
    assert ke == pytest.approx(0.125, abs=1e-3)
    assert en == pytest.approx(0.375, abs=1e-2)
    assert abs(ke - golden_meta["tgv32_ke0"]) <= 1e-12 * golden_meta["tgv32_ke0"]
    assert abs(en - golden_meta["tgv32_enstrophy0"]) <= \
        1e-12 * golden_meta["tgv32_enstrophy0"]


@pytest.mark.parametrize("variant", VARIANTS)
def test_workarray_allocations_match_budget(variant):
    import gc
    g = grid_of((8,) * 3)
    gc.collect()
    base = fd.live_field_count()
    ev = fd.ResidualEvaluator(g, C, variant)
    assert fd.live_field_count() - base == fd.workarray_budget(ev.plan)
    del ev
    gc.collect()
    assert fd.live_field_count() == base


# ------------------------------------------------- kernel-path coverage
@pytest.fixture
def kernel_path():
    from paper_1610_09146_b200 import _lib
    lib = _lib.load()
    yield lib
    lib.fdns_set_kernel_path(0)
    lib.fdns_set_tiled_grid(0)


@pytest.mark.parametrize("variant,path", [(v, 0) for v in VARIANTS] + [("SN", 5), ("RA", 5),
                                                                        ("SS", 5), ("RS", 5)])
@pytest.mark.parametrize("ctas", [3, 7, 13])
def test_tiled_segment_transitions(kernel_path, variant, ctas, path):
    """Force the persistent tiled kernel onto few CTAs so each walks several
    (tile, plane-range) segments; results stay bitwise equal to the
    one-thread-per-point path.  Path 5 runs SN, RA, SS and RS on the 12-warp kernel (at
    this size the default picks the 8-warp one)."""
    npts = (21, 20, 34)
    F = npo.state_from_primitives(npts, CO, np.ones(npts) + 0.01 * np.arange(
        np.prod(npts)).reshape(npts) / np.prod(npts),
        [0.1 * np.sin(np.arange(np.prod(npts)).reshape(npts))] * 3,
        np.full(npts, 70.0))
    g = grid_of(npts)
    cons = npo.interior(F[:5], 2)
    kernel_path.fdns_set_kernel_path(1)
    a = state_from_cons(g, cons)
    fd.run(a, fd.RKScheme(dt=1e-3), fd.ResidualEvaluator(g, C, variant), 2)
    want = host_cons(a)
    kernel_path.fdns_set_kernel_path(path)
    kernel_path.fdns_set_tiled_grid(ctas)
    b = state_from_cons(g, cons)
    fd.run(b, fd.RKScheme(dt=1e-3), fd.ResidualEvaluator(g, C, variant), 2)
    assert np.array_equal(host_cons(b), want)


@pytest.mark.parametrize("ctas", [0, 5])
def test_sn_kernel_families_agree(kernel_path, ctas):
    """SN with lazily evaluated derivatives (default), with the eager local
    array (path 4), on the 8-warp (path 2) and 12-warp (path 5) tiled
    kernels and on the point kernels (path 1): bitwise equal after two RK3
    steps."""
    npts = (19, 24, 40)
    F = npo.manufactured(npts, CO)
    g = grid_of(npts)
    cons = npo.interior(F[:5], 2)
    finals = []
    for path in (1, 2, 4, 5, 0):
        kernel_path.fdns_set_kernel_path(path)
        kernel_path.fdns_set_tiled_grid(ctas)
        st = state_from_cons(g, cons)
        fd.run(st, fd.RKScheme(dt=1e-3), fd.ResidualEvaluator(g, C, "SN"), 2)
        finals.append(host_cons(st))
    for f in finals[1:]:
        assert np.array_equal(finals[0], f)


# ------------------------------------------------ decomposition invariance
@pytest.mark.parametrize("variant,path", [("SN", 0), ("SS", 0), ("BL", 0), ("RA", 0),
                                          ("SN", 5), ("RA", 5), ("SS", 5),
                                          ("RS", 5)])
@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("split", [False, True])
def test_slab_decomposition_bitwise_invariant(kernel_path, variant, nranks, split, path):
    """z-slab decomposition emulated on one GPU: each 'rank' owns
    a slab grid (wrap_mask 0b110, so its stage kernels write axis-1/2 ghosts
    only) and the axis-0 ghost planes are copied between the ranks' bundles
    after every stage, as Slab.exchange does over NCCL.  The ranks' kernels
    never wait on each other (the host sequences stage -> exchange), so this
    is a faithful single-GPU emulation.  Fields must equal the one-GPU run
    bitwise.  Path 5 runs SN, RA, SS and RS on the 12-warp kernel (plane-range launches of
    the boundary/interior split included)."""
    n0, n1, n2, h = 24, 16, 20, 2
    npts = (n0, n1, n2)
    F = npo.manufactured(npts, CO)
    g1 = grid_of(npts)
    ref = state_from_cons(g1, npo.interior(F[:5], 2))
    scheme = fd.RKScheme(dt=2e-3)
    fd.run(ref, scheme, fd.ResidualEvaluator(g1, C, variant), 2)
    want = host_cons(ref)   # one GPU, default kernels

    kernel_path.fdns_set_kernel_path(path)
    slabs = [fd.Slab.partition(n0, r, nranks) for r in range(nranks)]
    grids, states, evs = [], [], []
    for sl in slabs:
        g = fd.make_grid(npts, (TWO_PI,) * 3, slab=sl)
        st = fd.ConservativeState(g)
        lo = sl.offset0
        st.bundle[:5].copy_(torch.from_numpy(np.ascontiguousarray(
            F[:5, lo:lo + sl.local_n0 + 2 * h])))
        fd.eval_primitives_fused(st, C)        # over the padded slab
        grids.append(g); states.append(st)
        evs.append(fd.ResidualEvaluator(g, C, variant))

    def exchange(bundles):
        for r, sl in enumerate(slabs):
            dn, up = slabs[r - 1], slabs[(r + 1) % nranks]
            b, bd, bu = bundles[r], bundles[r - 1], bundles[(r + 1) % nranks]
            n = sl.local_n0
            b[:5, 0:h].copy_(bd[:5, dn.local_n0:dn.local_n0 + h])
            b[:5, n + h:n + 2 * h].copy_(bu[:5, h:2 * h])
            # what Slab.exchange_state does after receiving the 5 fields
            fd.decomp.ghost_primitives(b, n, h, evs[r].problem)

    for _ in range(2):
        X = [st.bundle for st in states]
        YZ = [ev.workspace() for ev in evs]
        src = [X, [y for y, _ in YZ], [z for _, z in YZ]]
        dst = [src[1], src[2], X]
        for k in range(3):
            coef = scheme.alpha[k] * scheme.dt
            if split:   # the overlapped order of ResidualEvaluator.stage_exchanged
                for r in range(nranks):
                    evs[r].stage_boundary(src[k][r], X[r], dst[k][r], coef)
                exchange(dst[k])
                for r in range(nranks):
                    evs[r].stage_interior(src[k][r], X[r], dst[k][r], coef)
            else:
                for r in range(nranks):
                    evs[r].stage(src[k][r], X[r], dst[k][r], coef)
                exchange(dst[k])
    got = np.concatenate([host_cons(st) for st in states], axis=1)
    assert np.array_equal(got, want)


def _emulated_slab_run(variant, X0, npts, nranks, steps, dt, split=True):
    """Run `steps` RK3 iterations of the device state bundle X0 (10 padded
    fields, consistent ghosts) as `nranks` emulated z-slab ranks on one GPU
    (host-sequenced: every rank's stage launches, then the plane copies of
    Slab.exchange; no kernel waits on another).  Returns the interior
    conservative fields gathered along axis 0, on the device."""
    h = 2
    slabs = [fd.Slab.partition(npts[0], r, nranks) for r in range(nranks)]
    states, evs = [], []
    for sl in slabs:
        g = fd.make_grid(npts, (TWO_PI,) * 3, slab=sl)
        st = fd.ConservativeState(g)
        lo = sl.offset0
        st.bundle[:5].copy_(X0[:5, lo:lo + sl.local_n0 + 2 * h])
        fd.eval_primitives_fused(st, C)
        states.append(st)
        evs.append(fd.ResidualEvaluator(g, C, variant))

    def exchange(bundles):
        for r, sl in enumerate(slabs):
            dn = slabs[r - 1]
            b, bd, bu = bundles[r], bundles[r - 1], bundles[(r + 1) % nranks]
            n = sl.local_n0
            b[:5, 0:h].copy_(bd[:5, dn.local_n0:dn.local_n0 + h])
            b[:5, n + h:n + 2 * h].copy_(bu[:5, h:2 * h])
            # what Slab.exchange_state does after receiving the 5 fields
            fd.decomp.ghost_primitives(b, n, h, evs[r].problem)

    scheme = fd.RKScheme(dt=dt)
    for _ in range(steps):
        X = [st.bundle for st in states]
        YZ = [ev.workspace() for ev in evs]
        src = [X, [y for y, _ in YZ], [z for _, z in YZ]]
        dst = [src[1], src[2], X]
        for k in range(3):
            coef = scheme.alpha[k] * scheme.dt
            if split:
                for r in range(nranks):
                    evs[r].stage_boundary(src[k][r], X[r], dst[k][r], coef)
                exchange(dst[k])
                for r in range(nranks):
                    evs[r].stage_interior(src[k][r], X[r], dst[k][r], coef)
            else:
                for r in range(nranks):
                    evs[r].stage(src[k][r], X[r], dst[k][r], coef)
                exchange(dst[k])
    out = torch.cat([st.bundle[:5, h:h + sl.local_n0, h:-h, h:-h]
                     for st, sl in zip(states, slabs)], dim=1)
    del states, evs
    return out


@pytest.mark.parametrize("variant", ["RA", "SS"])
@pytest.mark.parametrize("nranks,split", [(2, False), (4, True), (8, True)])
def test_c4_256_slab_decomposition_bitwise(variant, nranks, split):
    """Config C4 (TGV 256^3, dt=8.5e-4, RA and SS, z-slabs over 1/2/4/8
    GPUs: 256/128/64/32 planes per rank): two RK3 steps on 2, 4 and 8
    emulated ranks, with the overlapped boundary/interior order, equal the
    one-GPU fields bitwise (SURVEY 8e invariance gate)."""
    n, dt = 256, 8.5e-4
    g = grid_of((n,) * 3)
    st = fd.taylor_green_init(g, C)
    X0 = st.bundle.clone()
    fd.run(st, fd.RKScheme(dt=dt), fd.ResidualEvaluator(g, C, variant), 2)
    want = st.bundle[:5, 2:-2, 2:-2, 2:-2].clone()
    del st
    got = _emulated_slab_run(variant, X0, (n,) * 3, nranks, 2, dt, split)
    assert torch.equal(got, want)


def test_c5_512_slab_decomposition_bitwise():
    """Config C5's multi-GPU layout on one GPU: TGV 512^3 (dt=4.2e-4) as 8
    emulated z-slab ranks of 64 planes (SN on the 12-warp kernel, the
    overlapped order), one RK3 step, bitwise equal to the one-GPU step --
    with the 512^3 cross-variant test, the gate SURVEY 8d sets for sizes
    without a CPU oracle."""
    n, dt = 512, 4.2e-4
    g = grid_of((n,) * 3)
    st = fd.taylor_green_init(g, C)
    X0 = st.bundle.clone()
    fd.run(st, fd.RKScheme(dt=dt), fd.ResidualEvaluator(g, C, "SN"), 1)
    want = st.bundle[:5, 2:-2, 2:-2, 2:-2].clone()
    del st
    torch.cuda.empty_cache()
    got = _emulated_slab_run("SN", X0, (n,) * 3, 8, 1, dt, True)
    assert torch.equal(got, want)
    del X0, got, want
    torch.cuda.empty_cache()


# ------------------------------------------- bounds (compute-sanitizer is closed)
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("npts", [(12, 16, 20), (9, 12, 7)])
def test_no_writes_outside_bundles(variant, npts):
    """Run the fused stage and the residual through the raw C ABI on
    bundles embedded in larger buffers pre-filled with a NaN-payload canary:
    every byte outside the output bundle, and the residual's halo (the
    reference leaves it zero, plan.py:413-415), must be untouched."""
    from paper_1610_09146_b200 import _lib
    lib = _lib.load()
    F = npo.manufactured(npts, CO)
    g = grid_of(npts)
    pb = g.problem(C)
    fs = int(np.prod(g.shape))
    pad = 4096
    canary = np.frombuffer(np.uint64(0x7FF8DEADBEEF0001).tobytes(), dtype=np.float64)[0]

    def framed(nf):
        buf = torch.full((nf * fs + 2 * pad,), canary, dtype=torch.float64, device="cuda")
        return buf, buf[pad:pad + nf * fs].view((nf,) + g.shape)

    nw = lib.fdns_workarray_count(_lib.VARIANT_IDS[variant])
    src_buf, src = framed(10)
    src.copy_(torch.from_numpy(F))
    out_buf, out = framed(10)
    out.zero_()
    work_buf, work = framed(max(nw, 1))
    res_buf, res = framed(5)
    res.zero_()
    _lib.check(lib.fdns_stage(_lib.VARIANT_IDS[variant], _lib.ptr(src), _lib.ptr(src),
                              _lib.ptr(out), _lib.ptr(work), 1e-3, 7, pb,
                              _lib.stream_handle()))
    _lib.check(lib.fdns_residual(_lib.VARIANT_IDS[variant], _lib.ptr(src), _lib.ptr(work),
                                 _lib.ptr(res), pb, _lib.stream_handle()))
    torch.cuda.synchronize()
    for buf in (src_buf, out_buf, work_buf, res_buf):
        h = buf.cpu().numpy().view(np.uint64)
        assert (h[:pad] == 0x7FF8DEADBEEF0001).all()
        assert (h[-pad:] == 0x7FF8DEADBEEF0001).all()
    assert np.array_equal(src.cpu().numpy(), F)          # input untouched
    r = res.cpu().numpy()
    assert np.all(r[:, :2] == 0) and np.all(r[:, -2:] == 0)
    assert np.all(r[:, :, :2] == 0) and np.all(r[:, :, :, -2:] == 0)
    want = c_oracle.residual(F, CO)
    assert np.array_equal(npo.interior(r, 2), want)


# --------------------------------------------------- C4 / C5 / edge cases
@pytest.mark.parametrize("variant", ["RA", "SS"])
def test_c4_256_steps_match_c_oracle(variant):
    """Config C4's grid and variants (TGV 256^3, dt=8.5e-4, RA and SS): five
    RK3 steps on the GPU bitwise equal to the C oracle (the 100-step and
    multi-GPU parts are covered by C2/C3 hashes and the decomposition
    invariance tests)."""
    n, steps, dt = 256, 5, 8.5e-4
    F = npo.taylor_green(n, CO)
    G = F.copy()
    c_oracle.run(G, CO, dt, steps)
    g = grid_of((n,) * 3)
    st = state_from_cons(g, npo.interior(F[:5], 2))
    fd.run(st, fd.RKScheme(dt=dt), fd.ResidualEvaluator(g, C, variant), steps)
    assert np.array_equal(host_cons(st), npo.interior(G[:5], 2))


@pytest.mark.parametrize("variant", ["BL", "RA", "RS", "SN", "SS"])
@pytest.mark.parametrize("npts", [(37, 45, 70), (130, 20, 132), (16, 130, 40),
                                  (256, 20, 44)])
def test_ragged_grids_match_c_oracle(variant, npts):
    """Non-cubic grids whose extents are not multiples of the 32x8 tile
    (partial edge tiles, odd plane counts, n2 >= 128 with the sector-aligned
    point-kernel map, a 1-tile-wide row; 256 planes: SS/RS on the
    round-robin unit split over ragged tiles): three RK3 steps of a
    perturbed TGV state bitwise equal to the C oracle."""
    F = npo.manufactured(npts, CO)
    G = F.copy()
    c_oracle.run(G, CO, 1e-3, 3)
    g = grid_of(npts)
    st = state_from_cons(g, npo.interior(F[:5], 2))
    fd.run(st, fd.RKScheme(dt=1e-3), fd.ResidualEvaluator(g, C, variant), 3)
    assert np.array_equal(host_cons(st), npo.interior(G[:5], 2))


def test_c5_512_cross_variant_bitwise():
    """Config C5 on one GPU (TGV 512^3, dt=4.2e-4, all four variants; BL's
    60 work arrays put it at ~99 GB of HBM): one RK3 step, all variants
    bitwise equal (512^3+ parity rests on cross-variant and
    decomposition invariance)."""
    n, dt = 512, 4.2e-4
    g = grid_of((n,) * 3)
    ref = None
    for v in NS_VARIANTS:
        st = fd.taylor_green_init(g, C)
        ev = fd.ResidualEvaluator(g, C, v)
        fd.run(st, fd.RKScheme(dt=dt), ev, 1)
        got = st.bundle[:5].clone()
        del st, ev
        torch.cuda.empty_cache()
        if ref is None:
            ref = got
        else:
            assert torch.equal(got, ref), v
    assert torch.isfinite(ref).all()


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("h", [3, 4])
def test_halo_width_and_box_lengths(variant, h):
    """Halo widths 3 (point kernels: an odd halo misaligns the TMA box) and
    4 (TMA-staged) -- mesh.py:82 allows any h >= 2 -- on a non-cubic,
    non-2*pi box: primitives and residual bitwise equal to the oracle."""
    npts = (12, 10, 14)
    lengths = (1.0, 2.5, 0.75)
    g = fd.make_grid(npts, lengths, halo=h)
    rng = np.random.default_rng(4)
    shape = npts
    rho = 1.0 + 0.1 * rng.random(shape)
    u = [0.2 * rng.standard_normal(shape) for _ in range(3)]
    p = 70.0 + rng.random(shape)
    F = npo.state_from_primitives(npts, CO, rho, u, p, h=h)
    st = fd.ConservativeState(g)
    st.bundle[:5].copy_(torch.from_numpy(F[:5]))
    fd.eval_primitives_fused(st, C)
    assert np.array_equal(st.to_numpy(), F)
    w = [npo.weights(l / n) for l, n in zip(lengths, npts)]
    want = np.stack(npo.residual(F, h, w, CO))
    got = fd.assemble_residual(st, C, variant).interior_numpy()
    assert np.array_equal(got, want)


def test_bench_variants_tables(tmp_path):
    """The reference's bench harness semantics on the GPU (bench.py:51-88):
    one record per (grid, plan), BL-normalised speedups, CSV files."""
    from paper_1610_09146_b200 import benchtables as bt
    recs = bt.bench_variants([(16, 16, 16)], ("BL", "SN", "SS"), iterations=2)
    assert [r.plan for r in recs] == ["BL", "SN", "SS"]
    assert all(r.loop_seconds > 0 and np.isfinite(r.final_ke) for r in recs)
    kes = {r.final_ke for r in recs}
    assert len(kes) == 1            # identical trajectories across variants
    bt.write_bench_csv(recs, tmp_path / "bench.csv")
    bt.write_speedup_csv(recs, tmp_path / "speedup.csv")
    assert (tmp_path / "speedup.csv").read_text().startswith("Nx,Ny,Nz,BL,SN,SS")


# ------------------------------------------- time-loop contract (test_timeloop.py)
def _quiescent(n=8):
    shape = (n,) * 3
    cons = np.stack([np.ones(shape), np.zeros(shape), np.zeros(shape),
                     np.zeros(shape), np.full(shape, (1.0 / C.gM2) / C.gm1)])
    return state_from_cons(grid_of(shape), cons)


def test_quiescent_state_unchanged():
    """test_timeloop.py:79-86."""
    st = _quiescent()
    before = host_cons(st)
    fd.run(st, fd.RKScheme(dt=1e-2), fd.ResidualEvaluator(st.grid, C, "SS"), 2)
    assert np.array_equal(host_cons(st), before)


def test_zero_iterations():
    """test_timeloop.py:88-97."""
    st = _quiescent()
    before = host_cons(st)
    rep = fd.run(st, fd.RKScheme(dt=1e-2), fd.ResidualEvaluator(st.grid, C, "RA"), 0)
    assert rep.iterations == 0 and rep.records == []
    assert np.array_equal(host_cons(st), before)


def test_save_state_snapshot():
    """test_timeloop.py:99-105."""
    g = grid_of((8,) * 3)
    st = fd.taylor_green_init(g, C)
    it = fd.IterationState(st)
    it.save_state()
    assert torch.equal(it.saved, st.bundle[:5])


def test_timing_and_cadence():
    """test_timeloop.py:138-149, 160-166: samples at iterations 0, 2, 4, 6;
    loop time positive; run completes."""
    g = grid_of((16,) * 3)
    st = fd.taylor_green_init(g, C)
    rho0 = fd.mean_density(st)
    rep = fd.run(st, fd.RKScheme(dt=6.77e-3), fd.ResidualEvaluator(g, C, "SS"), 6,
                 cadence=2, collect=fd.make_collector(g, rho0))
    assert len(rep.records) == 4
    assert rep.records[0].time == 0.0
    assert rep.records[-1].time == pytest.approx(6 * 6.77e-3, rel=1e-12)
    assert rep.loop_seconds > 0.0 and rep.completed


def test_mass_conservation_short_run():
    """test_timeloop.py:130-136: |mass drift| <= 1e-10 relative."""
    g = grid_of((16,) * 3)
    st = fd.taylor_green_init(g, C)
    m0 = fd.reduce_sum(st.rho)
    fd.run(st, fd.RKScheme(dt=6.77e-3), fd.ResidualEvaluator(g, C, "SS"), 20)
    assert abs(fd.reduce_sum(st.rho) - m0) <= 1e-10 * abs(m0)


@pytest.mark.parametrize("variant", ["SS", "SN"])
def test_tgv_physics_to_t12(variant):
    """The reference's TGV acceptance criterion 4 (test_acceptance.py:
    111-137) on the device: 64^3, dt=3.385e-3, to t=12 with diagnostics every
    25 iterations -- initial KE 0.125 +- 1e-3 and enstrophy 0.375 +- 1e-2,
    KE non-increasing for t > 4, and a single enstrophy maximum, in
    [8, 10]."""
    g = grid_of((64,) * 3)
    dt = 3.385e-3
    niter = int(np.ceil(12.0 / dt))
    st = fd.taylor_green_init(g, C)
    rho0 = fd.mean_density(st)
    rep = fd.run(st, fd.RKScheme(dt=dt), fd.ResidualEvaluator(g, C, variant), niter,
                 cadence=25, collect=fd.make_collector(g, rho0))
    rec = rep.records
    assert abs(rec[0].kinetic_energy - 0.125) <= 1e-3
    assert abs(rec[0].enstrophy - 0.375) <= 1e-2
    assert all(b.kinetic_energy <= a.kinetic_energy + 1e-12
               for a, b in zip(rec, rec[1:]) if b.time > 4.0)
    en = [(r.time, r.enstrophy) for r in rec]
    peaks = [en[i][0] for i in range(1, len(en) - 1)
             if en[i][1] > en[i - 1][1] and en[i][1] > en[i + 1][1]]
    t_max = max(en, key=lambda q: q[1])[0]
    assert len(peaks) == 1 and 8.0 <= t_max <= 10.0


@pytest.mark.parametrize("variant", ["BL", "RA", "RS", "SN", "SS"])
def test_residual_sums_conservative(variant):
    """The reference's criterion 3 (test_acceptance.py:88-108) as the
    reference itself behaves: the mass and momentum residuals of the 64^3 TGV
    sum to ~0 relative to their absolute sums (<= 1e-11), the energy
    residual's relative sum is 1.5e-08 -- the reference records that same
    value and FAILS its own 1e-11 bound (pkg/test_output.txt:212, the skew
    split of the energy flux does not telescope exactly) -- and 100 steps
    keep the total mass to 1e-10."""
    g = grid_of((64,) * 3)
    st = fd.taylor_green_init(g, C)
    res = fd.assemble_residual(st, C, variant)
    rel = []
    for f in res.fields:
        scale = float(f.interior.abs().sum()) + 1e-300
        rel.append(abs(fd.reduce_sum(f)) / scale)
    assert max(rel[:4]) <= 1e-11
    assert rel[4] == pytest.approx(1.5e-8, rel=0.05)
    m0 = fd.reduce_sum(st.rho)
    fd.run(st, fd.RKScheme(dt=3.385e-3), fd.ResidualEvaluator(g, C, variant), 100)
    assert abs(fd.reduce_sum(st.rho) - m0) / abs(m0) <= 1e-10


def test_timeseries_csv_from_device_run(tmp_path):
    """diagnostics.py:166-190 round trip of device-sampled records."""
    g = grid_of((16,) * 3)
    st = fd.taylor_green_init(g, C)
    rep = fd.run(st, fd.RKScheme(dt=6.77e-3), fd.ResidualEvaluator(g, C, "SN"), 4,
                 cadence=2, collect=fd.make_collector(g, fd.mean_density(st)))
    fd.write_timeseries(rep.records, tmp_path / "ts.csv")
    assert fd.read_timeseries(tmp_path / "ts.csv") == rep.records


@pytest.mark.parametrize("variant,graphs,chunks", [
    ("SN", True, 4), ("SS", True, 3), ("BL", True, 1), ("SN", False, 4), ("RA", False, 2)])
def test_host_stepper_matches_run(variant, graphs, chunks):
    """hostio.HostStepper (pinned host buffers, chunked copies pipelined
    across steps, graph-captured or eager) advances the host arrays exactly
    as run() advances the device state, including across a wait() in the
    middle of a run."""
    from paper_1610_09146_b200.hostio import HostStepper
    g = grid_of((24, 20, 16))
    F = npo.manufactured((24, 20, 16), CO)
    ref = state_from_cons(g, npo.interior(F[:5], 2))
    fd.run(ref, fd.RKScheme(dt=2e-3), fd.ResidualEvaluator(g, C, variant), 2)
    mid = ref.bundle[:5].cpu().numpy().copy()
    fd.run(ref, fd.RKScheme(dt=2e-3), fd.ResidualEvaluator(g, C, variant), 3)
    st = state_from_cons(g, npo.interior(F[:5], 2))
    host = HostStepper.pinned_buffers(g)
    host.copy_(st.bundle[:5].cpu())
    stepper = HostStepper(st, fd.ResidualEvaluator(g, C, variant), fd.RKScheme(dt=2e-3),
                          host, chunks=chunks, graphs=graphs)
    for _ in range(2):
        stepper.step()
    stepper.wait()
    torch.cuda.synchronize()
    assert np.array_equal(host.numpy(), mid)
    for _ in range(3):
        stepper.step()
    stepper.wait()
    torch.cuda.synchronize()
    assert np.array_equal(host.numpy(), ref.bundle[:5].cpu().numpy())
    assert stepper.it.iteration == 5


@pytest.mark.parametrize("variant", ["SN", "RA"])
@pytest.mark.parametrize("npts,k", [((40, 20, 24), 4), ((44, 16, 36), 5)])
def test_host_stepper_wavefront_matches_run(variant, npts, k):
    """Wavefront HostStepper (per-chunk uploads, primitives, stage launches
    and downloads overlapped across the link directions and the compute
    stream): the host arrays end up holding run()'s result bitwise, across a
    wait() in the middle of the run and a host edit before the next step."""
    from paper_1610_09146_b200.hostio import HostStepper
    g = grid_of(npts)
    F = npo.manufactured(npts, CO)
    ref = state_from_cons(g, npo.interior(F[:5], 2))
    fd.run(ref, fd.RKScheme(dt=2e-3), fd.ResidualEvaluator(g, C, variant), 2)
    mid = ref.bundle[:5].cpu().numpy().copy()
    fd.run(ref, fd.RKScheme(dt=2e-3), fd.ResidualEvaluator(g, C, variant), 3)
    st = state_from_cons(g, npo.interior(F[:5], 2))
    host = HostStepper.pinned_buffers(g)
    host.copy_(st.bundle[:5].cpu())
    stepper = HostStepper(st, fd.ResidualEvaluator(g, C, variant), fd.RKScheme(dt=2e-3),
                          host, wavefront=True, wave_chunks=k)
    assert stepper.wavefront
    for _ in range(2):
        stepper.step()
    stepper.wait()
    torch.cuda.synchronize()
    assert np.array_equal(host.numpy(), mid)
    for _ in range(3):
        stepper.step()
    stepper.wait()
    torch.cuda.synchronize()
    assert np.array_equal(host.numpy(), ref.bundle[:5].cpu().numpy())
    # a host edit between wait() and step() is what the next step advances
    edited = host.clone()
    edited[0, 5:9] *= 1.001
    host.copy_(edited)
    st2 = state_from_cons(g, npo.interior(F[:5], 2))
    st2.bundle[:5].copy_(edited.cuda())
    fd.run(st2, fd.RKScheme(dt=2e-3), fd.ResidualEvaluator(g, C, variant), 1)
    stepper.step()
    stepper.wait()
    torch.cuda.synchronize()
    assert np.array_equal(host.numpy(), st2.bundle[:5].cpu().numpy())


def test_host_stepper_wavefront_is_the_default_from_128_planes():
    """The bench's e2e path: the stepper picks the wavefront by itself for SN
    on one GPU from 128 planes (8 chunks here) and stays bitwise equal to
    run()."""
    from paper_1610_09146_b200.hostio import HostStepper
    npts = (128, 12, 16)
    g = grid_of(npts)
    F = npo.manufactured(npts, CO)
    ref = state_from_cons(g, npo.interior(F[:5], 2))
    fd.run(ref, fd.RKScheme(dt=2e-3), fd.ResidualEvaluator(g, C, "SN"), 3)
    st = state_from_cons(g, npo.interior(F[:5], 2))
    host = HostStepper.pinned_buffers(g)
    host.copy_(st.bundle[:5].cpu())
    stepper = HostStepper(st, fd.ResidualEvaluator(g, C, "SN"), fd.RKScheme(dt=2e-3), host)
    assert stepper.wavefront and stepper._wK == 8
    for _ in range(3):
        stepper.step()
    stepper.wait()
    torch.cuda.synchronize()
    assert np.array_equal(host.numpy(), ref.bundle[:5].cpu().numpy())
    # variants with work arrays keep the whole-step pipeline
    other = HostStepper(state_from_cons(g, npo.interior(F[:5], 2)),
                        fd.ResidualEvaluator(g, C, "SS"), fd.RKScheme(dt=2e-3), host)
    assert not other.wavefront


def test_host_stepper_wavefront_on_reference_numpy_arrays():
    """Wavefront stepping over the reference's own five padded numpy arrays
    (page-locked in place; chunk copies per field): bitwise run()."""
    from paper_1610_09146_b200.hostio import HostStepper
    npts = (40, 20, 24)
    g = grid_of(npts)
    F = npo.manufactured(npts, CO)
    ref = state_from_cons(g, npo.interior(F[:5], 2))
    fd.run(ref, fd.RKScheme(dt=2e-3), fd.ResidualEvaluator(g, C, "SN"), 3)
    st = state_from_cons(g, npo.interior(F[:5], 2))
    arrays = [np.ascontiguousarray(a) for a in st.bundle[:5].cpu().numpy()]
    stepper = HostStepper(st, fd.ResidualEvaluator(g, C, "SN"), fd.RKScheme(dt=2e-3),
                          arrays, wavefront=True, wave_chunks=4)
    for _ in range(3):
        stepper.step()
    stepper.wait()
    torch.cuda.synchronize()
    stepper.close()
    assert np.array_equal(np.stack(arrays), ref.bundle[:5].cpu().numpy())


def test_host_stepper_on_reference_numpy_arrays():
    """HostStepper over five plain padded numpy arrays (the reference's own
    Field.data layout), page-locked in place: the arrays end up holding the
    run() result bitwise."""
    from paper_1610_09146_b200.hostio import HostStepper
    g = grid_of((24, 20, 16))
    F = npo.manufactured((24, 20, 16), CO)
    ref = state_from_cons(g, npo.interior(F[:5], 2))
    fd.run(ref, fd.RKScheme(dt=2e-3), fd.ResidualEvaluator(g, C, "SN"), 3)
    st = state_from_cons(g, npo.interior(F[:5], 2))
    arrays = [np.ascontiguousarray(a) for a in st.bundle[:5].cpu().numpy()]
    stepper = HostStepper(st, fd.ResidualEvaluator(g, C, "SN"), fd.RKScheme(dt=2e-3),
                          arrays, chunks=10)
    for _ in range(3):
        stepper.step()
    stepper.wait()
    torch.cuda.synchronize()
    stepper.close()
    assert np.array_equal(np.stack(arrays), ref.bundle[:5].cpu().numpy())


def test_host_stepper_sees_host_edits():
    """A modification of the host buffer between wait() and the next step()
    is what the next step advances (the upload is real)."""
    from paper_1610_09146_b200.hostio import HostStepper
    g = grid_of((16, 16, 16))
    F = npo.manufactured((16, 16, 16), CO)
    st = state_from_cons(g, npo.interior(F[:5], 2))
    host = HostStepper.pinned_buffers(g)
    host.copy_(st.bundle[:5].cpu())
    stepper = HostStepper(st, fd.ResidualEvaluator(g, C, "SN"), fd.RKScheme(dt=2e-3), host)
    stepper.step()
    stepper.wait()
    torch.cuda.synchronize()
    ref = state_from_cons(g, 1.0001 * npo.interior(F[:5], 2))
    host.copy_(ref.bundle[:5].cpu())
    fd.run(ref, fd.RKScheme(dt=2e-3), fd.ResidualEvaluator(g, C, "SN"), 1)
    stepper.step()
    stepper.wait()
    torch.cuda.synchronize()
    assert np.array_equal(host.numpy(), ref.bundle[:5].cpu().numpy())
