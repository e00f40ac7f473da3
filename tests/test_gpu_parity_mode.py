"""Parity mode: the reference's own numpy state objects passed straight to
`ResidualEvaluator.evaluate`, `assemble_residual` and `run`.

The reference package is not importable on the GPU box, so the objects are
stand-ins with exactly its attribute layout (`fdns.mesh.Grid` /
`Field.data`, `fdns.physics.ConservativeState` / `Residual`,
physics.py:84-156): padded float64 numpy arrays, `field_arrays()` in the
kernel argument order, `arrays()` for the residual."""

import math

import numpy as np
import pytest
import torch

from conftest import sha
from oracle import numpy_oracle as npo

pytestmark = pytest.mark.gpu

fd = pytest.importorskip("paper_1610_09146_b200")
C = fd.PhysicalConstants()
CO = npo.Consts()


class RefGrid:
    def __init__(self, npts, h=2):
        self.npoints = tuple(npts)
        self.delta = tuple(2.0 * math.pi / n for n in npts)
        self.halo = h

    @property
    def shape(self):
        return tuple(n + 2 * self.halo for n in self.npoints)


class RefField:
    def __init__(self, grid, data=None):
        self.grid = grid
        self.data = np.zeros(grid.shape) if data is None else data

    @property
    def interior(self):
        h = self.grid.halo
        return self.data[h:-h, h:-h, h:-h]


class RefState:
    def __init__(self, grid, padded10=None):
        f = [RefField(grid, None if padded10 is None else padded10[q].copy())
             for q in range(10)]
        self.grid = grid
        self.rho, self.rhou, self.rhoE = f[0], f[1:4], f[4]
        self.u, self.p, self.T = f[5:8], f[8], f[9]

    @property
    def conservative(self):
        return [self.rho, *self.rhou, self.rhoE]

    def field_arrays(self):
        return (self.rho.data, *(f.data for f in self.rhou), self.rhoE.data,
                *(f.data for f in self.u), self.p.data, self.T.data)


class RefResidual:
    def __init__(self, grid):
        f = [RefField(grid) for _ in range(5)]
        self.d_rho, self.d_rhou, self.d_rhoE = f[0], f[1:4], f[4]

    @property
    def fields(self):
        return [self.d_rho, *self.d_rhou, self.d_rhoE]

    def arrays(self):
        return tuple(f.data for f in self.fields)


@pytest.fixture(scope="module", autouse=True)
def _gpu(built):
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("variant", fd.PLAN_NAMES)
def test_evaluate_on_reference_state_objects(golden, variant):
    """evaluate(ref_state, ref_out): the reference's m16 golden residual
    bitwise in out's interior, out's halos untouched, and the state's
    primitive arrays recomputed over the padded arrays (the reference's
    side effect, physics.py:185-202) -- bitwise the oracle's."""
    npts = (16, 16, 16)
    F = npo.new_fields(npts, 2)
    npo.interior(F[:5], 2)[...] = golden["m16_cons"]
    npo.halo_exchange(F[:5], 2)
    want_prim = npo.primitives(F.copy(), CO)[5:]
    grid = RefGrid(npts)
    state = RefState(grid, F)
    for a in state.field_arrays()[5:]:
        a[...] = -7.0                      # stale primitives on entry
    out = RefResidual(grid)
    for a in out.arrays():
        a[...] = 3.25                      # halos must keep this
    ev = fd.ResidualEvaluator(grid, C, variant)
    got = ev.evaluate(state, out)
    assert got is out
    inner = np.stack([f.interior for f in out.fields])
    assert np.array_equal(inner, golden["m16_res"])
    for a in out.arrays():
        halo = a.copy()
        halo[2:-2, 2:-2, 2:-2] = 3.25
        assert np.all(halo == 3.25)
    assert np.array_equal(np.stack(state.field_arrays()[5:]), want_prim)


def test_assemble_residual_returns_host_residual(golden):
    npts = (9, 12, 7)
    F = npo.new_fields(npts, 2)
    npo.interior(F[:5], 2)[...] = golden["m_ragged_cons"]
    npo.halo_exchange(F[:5], 2)
    res = fd.assemble_residual(RefState(RefGrid(npts), F), C, "SN")
    assert all(isinstance(a, np.ndarray) for a in res.arrays())
    assert np.array_equal(np.stack([f.interior for f in res.fields]),
                          golden["m_ragged_res"])


@pytest.mark.parametrize("variant", ["BL", "SS", "SN"])
def test_run_on_reference_state_c1(golden_meta, variant):
    """run(ref_state, ...) on config C1 (TGV 32^3, 10 steps, dt=2e-3): the
    host conservative arrays end bitwise equal to the reference's, and a
    host-side collector (numpy over the host arrays, the reference's
    kinetic_energy_integral formula) sees the reference's KE history --
    i.e. the host primitives are synchronised with the reference's
    one-stage-stale semantics before every sample."""
    ref = golden_meta["c1_tgv32_bl"]
    n = 32
    grid = RefGrid((n,) * 3)
    state = RefState(grid, npo.taylor_green(n, CO))
    dv = grid.delta[0] * grid.delta[1] * grid.delta[2]
    vol = n ** 3 * dv
    rho0 = ref["rho0"]

    def collect(t, st):
        rho = st.rho.interior
        u = [f.interior for f in st.u]
        ke = np.sum(0.5 * rho * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]))
        return (t, float(ke) * dv / (rho0 * vol))

    ev = fd.ResidualEvaluator(grid, C, variant)
    rep = fd.run(state, fd.RKScheme(dt=2e-3), ev, 10, cadence=1,
                 collect=collect)
    assert [sha(f.interior) for f in state.conservative] == ref["sha256"]
    assert len(rep.records) == len(ref["history"])
    for (t, ke), row in zip(rep.records, ref["history"]):
        assert t == pytest.approx(row[0], rel=1e-15, abs=1e-15)
        assert abs(ke - row[1]) <= 1e-12 * abs(row[1])


def test_run_on_reference_state_with_device_collector(golden_meta):
    """This package's make_collector works in parity mode too (it is handed
    the device twin)."""
    ref = golden_meta["c1_tgv32_bl"]
    grid = RefGrid((32,) * 3)
    state = RefState(grid, npo.taylor_green(32, CO))
    ev = fd.ResidualEvaluator(grid, C, "RA")
    rep = fd.run(state, fd.RKScheme(dt=2e-3), ev, 10, cadence=5,
                 collect=fd.make_collector(ev.grid, ref["rho0"]))
    assert [sha(f.interior) for f in state.conservative] == ref["sha256"]
    for rec, row in zip(rep.records, ref["history"][::5]):
        assert abs(rec.kinetic_energy - row[1]) <= 1e-10 * abs(row[1])
