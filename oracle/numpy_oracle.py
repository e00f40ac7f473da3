"""numpy restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.

Every function cites the reference file:line it restates (paths relative to
the reference package `pkg/src/fdns/`).  Arithmetic follows the reference's
exact left-to-right association so results are bitwise identical to it
(pinned by `tests/test_oracle_golden.py` against vectors the real reference
produced).  Field bundles are float64 arrays of shape (10, n0+2h, n1+2h,
n2+2h) in the reference's kernel argument order rho, rhou0, rhou1, rhou2,
rhoE, u0, u1, u2, p, T (physics.py:115-119), C-ordered with axis 2
contiguous (mesh.py:3-6).
"""

from __future__ import annotations

import math

import numpy as np

RHO, RHOU0, RHOU1, RHOU2, RHOE, U0, U1, U2, P, T = range(10)
GAMMA, MACH, PR, RE = 1.4, 0.1, 0.71, 1600.0
RK3_ALPHA = (1.0 / 3.0, 1.0 / 2.0, 1.0)          # timeloop.py:26


class Consts:
    """Derived constants, each formed exactly as physics.py:53-81 does."""

    def __init__(self, gamma=GAMMA, M=MACH, Pr=PR, Re=RE):
        self.gamma, self.M, self.Pr, self.Re = gamma, M, Pr, Re
        self.gm1 = gamma - 1.0
        self.gM2 = gamma * M * M
        self.inv_Re = 1.0 / Re
        self.heat_coeff = 1.0 / (self.gm1 * M * M * Pr * Re)
        self.c13 = 1.0 / (3.0 * Re)
        self.c43 = 4.0 / (3.0 * Re)
        self.c23 = 2.0 / (3.0 * Re)


def weights(delta: float):
    """(fw1, fw2, s0, s1, s2) pre-divided by the spacing -- stencil.py:45-51."""
    return (8.0 / (12.0 * delta), -1.0 / (12.0 * delta),
            -30.0 / (12.0 * delta * delta), 16.0 / (12.0 * delta * delta),
            -1.0 / (12.0 * delta * delta))


def cube_delta(n: int) -> float:
    """delta = 2*pi / n for the periodic TGV cube -- mesh.py:84."""
    return (2.0 * np.pi) / n


def interior(a: np.ndarray, h: int) -> np.ndarray:
    return a[..., h:-h, h:-h, h:-h]


def halo_exchange(a: np.ndarray, h: int) -> np.ndarray:
    """Periodic ghost fill, axis by axis over full slabs -- mesh.py:118-139.

    Works on a single padded field or on a leading-axis bundle of them.
    """
    nd = a.ndim
    for ax in range(3):
        axis = nd - 3 + ax
        n = a.shape[axis] - 2 * h
        def sl(s):
            idx = [slice(None)] * nd
            idx[axis] = s
            return tuple(idx)
        a[sl(slice(0, h))] = a[sl(slice(n, n + h))]
        a[sl(slice(n + h, n + 2 * h))] = a[sl(slice(h, 2 * h))]
    return a


def primitives(F: np.ndarray, c: Consts) -> np.ndarray:
    """Fused primitive recovery over the full padded arrays --
    physics.py:185-202 (bitwise equal to the grouped form :169-182)."""
    rho = F[RHO]
    u0 = F[RHOU0] / rho
    u1 = F[RHOU1] / rho
    u2 = F[RHOU2] / rho
    F[U0], F[U1], F[U2] = u0, u1, u2
    p = c.gm1 * (F[RHOE] - 0.5 * (F[RHOU0] * u0 + F[RHOU1] * u1
                                  + F[RHOU2] * u2))
    F[P] = p
    F[T] = c.gM2 * p / rho
    return F


def _shift(a, h, axis, off):
    """Interior-shaped view shifted along one axis -- stencil.py:63-68."""
    n = [s - 2 * h for s in a.shape]
    sl = [slice(h, h + m) for m in n]
    sl[axis] = slice(h + off, h + n[axis] + off)
    return a[tuple(sl)]


def d1(a, h, axis, w):
    """First derivative over the interior -- stencil.py:71-86."""
    w1, w2 = w[axis][0], w[axis][1]
    return (w1 * (_shift(a, h, axis, 1) - _shift(a, h, axis, -1))
            + w2 * (_shift(a, h, axis, 2) - _shift(a, h, axis, -2)))


def d2(a, h, axis, w):
    """Second derivative over the interior -- stencil.py:89-102."""
    s0, s1, s2 = w[axis][2], w[axis][3], w[axis][4]
    return (s0 * _shift(a, h, axis, 0)
            + s1 * (_shift(a, h, axis, 1) + _shift(a, h, axis, -1))
            + s2 * (_shift(a, h, axis, 2) + _shift(a, h, axis, -2)))


def _padded_like(a, h, vals):
    out = np.zeros(a.shape)
    out[h:-h, h:-h, h:-h] = vals
    return out


def derivatives(F: np.ndarray, h: int, w) -> dict:
    """All 60 distinct derivatives of the term list, stored (the BL route).

    Term list: terms.py:135-200.  Products are formed over the padded arrays
    and then differentiated (plan.py:383-392); mixed terms differentiate the
    halo-exchanged inner first derivative (plan.py:378-382).
    """
    rho, ru, rE = F[RHO], (F[RHOU0], F[RHOU1], F[RHOU2]), F[RHOE]
    u, p, Tf = (F[U0], F[U1], F[U2]), F[P], F[T]
    rhoe = rE - 0.5 * (ru[0] * u[0] + ru[1] * u[1] + ru[2] * u[2])
    D = {}
    for a in range(3):
        D["rho", a] = d1(rho, h, a, w)
        D["p", a] = d1(p, h, a, w)
        D["rhoe", a] = d1(rhoe, h, a, w)
        D["rhoeu", a] = d1(rhoe * u[a], h, a, w)
        D["up", a] = d1(u[a] * p, h, a, w)
        D["T2", a] = d2(Tf, h, a, w)
        for i in range(3):
            D[f"rhou{i}", a] = d1(ru[i], h, a, w)
            D[f"u{i}", a] = d1(u[i], h, a, w)
            D[f"rhou{i}u", a] = d1(ru[i] * u[a], h, a, w)
            D[f"u{i}2", a] = d2(u[i], h, a, w)
    # mixed: DD(u_j, x_outer, x_j) = D_outer(halo-exchanged D(u_j, x_j))
    for j in range(3):
        inner = halo_exchange(_padded_like(rho, h, D[f"u{j}", j]), h)
        for o in range(3):
            if o != j:
                D[f"uu{j}", o] = d1(inner, h, o, w)
    return D


def _viscous(D, pt, c: Consts, i: int):
    """Expanded viscous term of momentum i -- terms.py:113-123."""
    acc = c.c43 * D[f"u{i}2", i]
    for j in range(3):
        if j == i:
            continue
        acc = acc + c.inv_Re * D[f"u{i}2", j]
        acc = acc + c.c13 * D[f"uu{j}", i]
    return acc


def _tau(D, c: Consts, i: int, j: int):
    """Stress component over velocity-gradient values -- terms.py:126-132."""
    if i == j:
        divu = D["u0", 0] + D["u1", 1] + D["u2", 2]
        return 2.0 * c.inv_Re * D[f"u{i}", i] - c.c23 * divu
    return c.inv_Re * (D[f"u{i}", j] + D[f"u{j}", i])


def residual_from_derivatives(F, h, D, c: Consts):
    """The five residual expressions, evaluated with the reference's
    association (terms.py:151-183).  Returns interior arrays."""
    pt = [interior(F[q], h) for q in range(10)]
    rho, ru, rE = pt[RHO], pt[RHOU0:RHOU2 + 1], pt[RHOE]
    u = pt[U0:U2 + 1]

    # mass -- terms.py:151-156
    acc = None
    for j in range(3):
        for term in (D[f"rhou{j}", j], u[j] * D["rho", j],
                     rho * D[f"u{j}", j]):
            acc = term if acc is None else acc + term
    d_rho = -(0.5 * acc)

    # momentum -- terms.py:158-165
    d_rhou = []
    for i in range(3):
        acc = None
        for j in range(3):
            for term in (D[f"rhou{i}u", j], u[j] * D[f"rhou{i}", j],
                         ru[i] * D[f"u{j}", j]):
                acc = term if acc is None else acc + term
        r = -(0.5 * acc) - D["p", i]
        r = r + c.c43 * D[f"u{i}2", i]
        for j in range(3):
            if j != i:
                r = r + c.inv_Re * D[f"u{i}2", j]
                r = r + c.c13 * D[f"uu{j}", i]
        d_rhou.append(r)

    # energy -- terms.py:167-183
    rhoe_pt = rE - 0.5 * (ru[0] * u[0] + ru[1] * u[1] + ru[2] * u[2])
    acc = None
    for j in range(3):
        for term in (D["rhoeu", j], u[j] * D["rhoe", j],
                     rhoe_pt * D[f"u{j}", j]):
            acc = term if acc is None else acc + term
    pwork = D["up", 0] + D["up", 1] + D["up", 2]
    heat = c.heat_coeff * (D["T2", 0] + D["T2", 1] + D["T2", 2])
    r = -(0.5 * acc) - pwork + heat
    for i in range(3):
        for j in range(3):
            r = r + _tau(D, c, i, j) * D[f"u{i}", j]
    for i in range(3):
        r = r + u[i] * _viscous(D, pt, c, i)
    return [d_rho, d_rhou[0], d_rhou[1], d_rhou[2], r]


def residual(F, h, w, c: Consts):
    """Full residual: primitives must already be current (plan.py:394-416)."""
    return residual_from_derivatives(F, h, derivatives(F, h, w), c)


def rk_step(F, h, w, c: Consts, dt: float):
    """One save-state RK3 iteration -- timeloop.py:75-94.  In place on F."""
    saved = F[:5].copy()
    for a in RK3_ALPHA:
        primitives(F, c)
        R = residual(F, h, w, c)
        coef = a * dt
        for q in range(5):
            interior(F[q], h)[...] = interior(saved[q], h) + coef * R[q]
        halo_exchange(F[:5], h)
    return F


def new_fields(npoints, h=2):
    return np.zeros((10,) + tuple(n + 2 * h for n in npoints))


def state_from_primitives(npoints, c: Consts, rho, u, p, h=2):
    """Conservative bundle from interior primitive arrays --
    tests/helpers.py:50-64 (then halos + primitives)."""
    F = new_fields(npoints, h)
    interior(F[RHO], h)[...] = rho
    for i in range(3):
        interior(F[RHOU0 + i], h)[...] = rho * u[i]
    interior(F[RHOE], h)[...] = (p / c.gm1 + 0.5 * rho * (
        u[0] ** 2 + u[1] ** 2 + u[2] ** 2))
    halo_exchange(F[:5], h)
    primitives(F, c)
    return F


def coords(n: int, delta: float):
    return np.arange(n) * delta                  # mesh.py:65-67


def taylor_green(n: int, c: Consts, h: int = 2):
    """TGV initial state on the 2*pi cube -- diagnostics.py:55-86."""
    d = cube_delta(n)
    x = coords(n, d)[:, None, None]
    y = coords(n, d)[None, :, None]
    z = coords(n, d)[None, None, :]
    u0 = np.sin(x) * np.cos(y) * np.cos(z)
    u1 = -np.cos(x) * np.sin(y) * np.cos(z)
    p0 = 1.0 / (c.gamma * c.M ** 2)
    p = p0 + (np.cos(2 * x) + np.cos(2 * y)) * (np.cos(2 * z) + 2.0) / 16.0
    rho = c.gM2 * p
    F = new_fields((n, n, n), h)
    interior(F[RHO], h)[...] = rho
    interior(F[RHOU0], h)[...] = rho * u0
    interior(F[RHOU1], h)[...] = rho * u1
    interior(F[RHOU2], h)[...] = 0.0
    interior(F[RHOE], h)[...] = p / c.gm1 + 0.5 * rho * (u0 * u0 + u1 * u1)
    halo_exchange(F[:5], h)
    primitives(F, c)
    return F


def perturbed_taylor_green(n: int, c: Consts, seed: int, amp: float = 1e-3,
                           h: int = 2):
    """Config C3's seeded TGV: +U(-amp, amp) on u, v, w, with p and rho kept
    (SURVEY.md section 8d), assembled like tests/helpers.py:50-64."""
    d = cube_delta(n)
    x = coords(n, d)[:, None, None]
    y = coords(n, d)[None, :, None]
    z = coords(n, d)[None, None, :]
    shape = (n, n, n)
    u0 = np.sin(x) * np.cos(y) * np.cos(z) + np.zeros(shape)
    u1 = -np.cos(x) * np.sin(y) * np.cos(z) + np.zeros(shape)
    u2 = np.zeros(shape)
    p0 = 1.0 / (c.gamma * c.M ** 2)
    p = p0 + (np.cos(2 * x) + np.cos(2 * y)) * (np.cos(2 * z) + 2.0) / 16.0
    rho = c.gM2 * p
    rng = np.random.default_rng(seed)
    u0 = u0 + rng.uniform(-amp, amp, shape)
    u1 = u1 + rng.uniform(-amp, amp, shape)
    u2 = u2 + rng.uniform(-amp, amp, shape)
    return state_from_primitives(shape, c, rho + np.zeros(shape),
                                 [u0, u1, u2], p + np.zeros(shape), h)


def manufactured(npoints, c: Consts, h: int = 2):
    """Smooth trig state exercising every term -- tests/helpers.py:67-84."""
    d = [(2.0 * np.pi) / n for n in npoints]
    x = coords(npoints[0], d[0])[:, None, None]
    y = coords(npoints[1], d[1])[None, :, None]
    z = coords(npoints[2], d[2])[None, None, :]
    shape = tuple(npoints)
    rho = 1.0 + 0.1 * np.sin(x) * np.cos(y) * np.cos(z)
    u = [np.sin(x) * np.cos(y) * np.cos(z),
         -0.5 * np.cos(x) * np.sin(y) * np.cos(z),
         0.3 * np.cos(x) * np.cos(y) * np.sin(z)]
    p0 = 1.0 / (c.gamma * c.M ** 2)
    p = p0 * (1.0 + 0.05 * np.cos(2 * x) * np.cos(y)
              + 0.03 * np.sin(z) * np.cos(x))
    return state_from_primitives(shape, c, rho + np.zeros(shape),
                                 [ui + np.zeros(shape) for ui in u],
                                 p + np.zeros(shape), h)


def mean_density(F, h):
    """diagnostics.py:89-91."""
    n = np.prod([s - 2 * h for s in F.shape[1:]])
    return float(np.sum(interior(F[RHO], h))) / float(n)


def kinetic_energy(F, h, delta3, rho0):
    """diagnostics.py:94-102 (delta3 = per-axis spacings)."""
    npts = [s - 2 * h for s in F.shape[1:]]
    dv = delta3[0] * delta3[1] * delta3[2]
    volume = float(np.prod(npts)) * dv
    ke = 0.5 * interior(F[RHO], h) * (interior(F[U0], h) ** 2
                                      + interior(F[U1], h) ** 2
                                      + interior(F[U2], h) ** 2)
    return float(np.sum(ke)) * dv / (rho0 * volume)


def enstrophy(F, h, delta3, w, rho0):
    """diagnostics.py:105-132."""
    npts = [s - 2 * h for s in F.shape[1:]]
    dv = delta3[0] * delta3[1] * delta3[2]
    volume = float(np.prod(npts)) * dv
    u = F[U0:U2 + 1]
    w0 = d1(u[2], h, 1, w) - d1(u[1], h, 2, w)
    w1 = d1(u[0], h, 2, w) - d1(u[2], h, 0, w)
    w2 = d1(u[1], h, 0, w) - d1(u[0], h, 1, w)
    ens = 0.5 * interior(F[RHO], h) * (w0 ** 2 + w1 ** 2 + w2 ** 2)
    return float(np.sum(ens)) * dv / (rho0 * volume)


def rel_linf(a, b) -> float:
    """tests/helpers.py:96-100."""
    scale = np.max(np.abs(b))
    if scale == 0.0:
        return float(np.max(np.abs(a - b)))
    return float(np.max(np.abs(a - b)) / scale)


def grid_weights(npoints):
    return [weights((2.0 * math.pi) / n) for n in npoints]
