"""Pin the CPU oracle to the reference: every golden vector produced by the
real reference (tests/golden/make_golden.py) must be reproduced bitwise by
both restatements (numpy and C).  CPU only."""

import numpy as np
import pytest

from conftest import rel_linf, sha
from oracle import c_oracle, numpy_oracle as npo

C = npo.Consts()
CASES = (("m16", (16, 16, 16)), ("m_ragged", (9, 12, 7)))


def test_constants_match_reference(golden_meta):
    k = golden_meta["constants"]
    assert (C.gm1, C.gM2, C.inv_Re, C.heat_coeff, C.c13, C.c43, C.c23) == (
        k["gm1"], k["gM2"], k["inv_Re"], k["heat_coeff"], k["c13"],
        k["c43"], k["c23"])
    # reference known answer (test_physics.py:158-161)
    assert C.heat_coeff == pytest.approx(0.22007042253521127, rel=1e-14)


@pytest.mark.parametrize("tag,npts", CASES)
def test_manufactured_state_bits(golden, tag, npts):
    F = npo.manufactured(npts, C)
    assert np.array_equal(npo.interior(F[:5], 2), golden[f"{tag}_cons"])


@pytest.mark.parametrize("tag,npts", CASES)
def test_numpy_residual_bitwise(golden, tag, npts):
    F = npo.manufactured(npts, C)
    R = np.stack(npo.residual(F, 2, npo.grid_weights(npts), C))
    assert np.array_equal(R, golden[f"{tag}_res"])


@pytest.mark.parametrize("tag,npts", CASES)
def test_c_residual_bitwise(built, golden, tag, npts):
    F = npo.manufactured(npts, C)
    R = c_oracle.residual(F, C)
    assert np.array_equal(R, golden[f"{tag}_res"])


def test_perturbed_state_and_residual(built, golden, golden_meta):
    F = npo.perturbed_taylor_green(16, C, golden_meta["perturb_seed"])
    assert [sha(npo.interior(F[q], 2)) for q in range(5)] == \
        golden_meta["p16_cons_sha256"]
    assert np.array_equal(c_oracle.residual(F, C), golden["p16_res"])
    assert np.array_equal(np.stack(npo.residual(F, 2, npo.grid_weights(
        (16,) * 3), C)), golden["p16_res"])


def test_tgv_init_and_integrals(golden_meta):
    F = npo.taylor_green(32, C)
    assert [sha(npo.interior(F[q], 2)) for q in range(5)] == \
        golden_meta["tgv32_cons_sha256"]
    assert [sha(npo.interior(F[q], 2)) for q in range(5, 10)] == \
        golden_meta["tgv32_prim_sha256"]
    d = npo.cube_delta(32)
    rho0 = npo.mean_density(F, 2)
    assert rho0 == golden_meta["tgv32_rho0"]
    assert npo.kinetic_energy(F, 2, (d,) * 3, rho0) == golden_meta["tgv32_ke0"]
    assert npo.enstrophy(F, 2, (d,) * 3, npo.grid_weights((32,) * 3),
                         rho0) == golden_meta["tgv32_enstrophy0"]


def test_primitive_known_answer(built, golden_meta):
    ka = golden_meta["known_answer_prim"]
    F = npo.state_from_primitives((5, 5, 5), C, np.full((5,) * 3, 2.0),
                                  [np.full((5,) * 3, 1.0), np.zeros((5,) * 3),
                                   np.zeros((5,) * 3)], np.full((5,) * 3, 0.8))
    c_oracle.primitives(F, C)
    assert F[5, 2, 2, 2] == ka["u0"] == 1.0
    assert F[8, 2, 2, 2] == ka["p"]
    assert F[9, 2, 2, 2] == ka["T"]
    assert abs(ka["p"] - 0.8) < 1e-14 and abs(ka["T"] - 0.0056) < 1e-15


def test_c1_run_bitwise_numpy_and_c(built, golden, golden_meta):
    """Config C1: TGV 32^3, 10 RK3 steps, dt=2e-3."""
    ref = golden_meta["c1_tgv32_bl"]
    F = npo.taylor_green(32, C)
    G = F.copy()
    w = npo.grid_weights((32,) * 3)
    for _ in range(10):
        npo.rk_step(F, 2, w, C, 2e-3)
    c_oracle.run(G, C, 2e-3, 10)
    for B in (F, G):
        assert [sha(npo.interior(B[q], 2)) for q in range(5)] == ref["sha256"]
    assert np.array_equal(npo.interior(G[0], 2), golden["c1_final_rho"])
    # diagnostics history within the north-star tolerance
    d = npo.cube_delta(32)
    rho0 = ref["rho0"]
    ke = npo.kinetic_energy(G, 2, (d,) * 3, rho0)
    assert abs(ke - ref["history"][-1][1]) <= 1e-12 * abs(ref["history"][-1][1])


def test_c2_64cube_100_steps_c_oracle(built, golden_meta):
    """Config C2: TGV 64^3, 100 steps, dt=3.385e-3 -- the C oracle matches
    the reference's final-state hashes and KE/enstrophy history."""
    ref = golden_meta["c2_tgv64"]
    F = npo.taylor_green(64, C)
    d = npo.cube_delta(64)
    w = npo.grid_weights((64,) * 3)
    hist = []
    for s in range(0, 100, 10):
        c_oracle.run(F, C, 3.385e-3, 10)
        hist.append((npo.kinetic_energy(F, 2, (d,) * 3, ref["rho0"]),
                     npo.enstrophy(F, 2, (d,) * 3, w, ref["rho0"])))
    assert [sha(npo.interior(F[q], 2)) for q in range(5)] == ref["sha256"]
    for (ke, en), row in zip(hist, ref["history"][1:]):
        assert abs(ke - row[1]) <= 1e-10 * abs(row[1])
        assert abs(en - row[2]) <= 1e-10 * abs(row[2])


def test_rel_linf_helper():
    a = np.array([1.0, 2.0])
    assert rel_linf(a, a) == 0.0
    assert rel_linf(np.zeros(2), np.zeros(2)) == 0.0
