"""Generate the golden vectors that pin the oracle (and the GPU path).

Run in the build container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
    FDNS_CACHE_DIR=/tmp/fdns_cache NUMBA_NUM_THREADS=8 \
        python tests/golden/make_golden.py [--big]

Everything written here comes out of the reference package itself
(`fdns.plan.assemble_residual`, `fdns.timeloop.run`,
`fdns.diagnostics.make_collector`, the reference test helpers); nothing is
computed by this repository's code.  Small cases store full arrays; larger
runs store a SHA-256 per final conservative field (bitwise golden) plus the
reference's diagnostics history.  `/root/reference` does not exist on the
GPU box, so tests only ever read the committed `.npz`/`.json` outputs.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import pathlib
import time

import numpy as np

from fdns.diagnostics import make_collector, mean_density, \
    taylor_green_init, kinetic_energy_integral, enstrophy_integral
from fdns.mesh import make_grid
from fdns.physics import PhysicalConstants, eval_primitives_fused
from fdns.plan import PLAN_NAMES, ResidualEvaluator, assemble_residual
from fdns.timeloop import RKScheme, run
from helpers import TWO_PI, cube, manufactured_state, state_from_primitives

OUT = pathlib.Path(__file__).parent
C = PhysicalConstants()
PERTURB_SEED = 20161029   # config C3 seed (arXiv id date); see DESIGN.md


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cons_interior(state):
    return np.stack([f.interior.copy() for f in state.conservative])


def perturbed_tgv(n: int, seed: int = PERTURB_SEED, amp: float = 1e-3):
    """Config C3: TGV plus seeded U(-amp, amp) on u, v, w,
    p and rho kept, assembled through the reference helper."""
    g = cube(n)
    x = g.coordinates(0)[:, None, None]
    y = g.coordinates(1)[None, :, None]
    z = g.coordinates(2)[None, None, :]
    shape = (n, n, n)
    u0 = np.sin(x) * np.cos(y) * np.cos(z) + np.zeros(shape)
    u1 = -np.cos(x) * np.sin(y) * np.cos(z) + np.zeros(shape)
    u2 = np.zeros(shape)
    p0 = 1.0 / (C.gamma * C.M ** 2)
    p = p0 + (np.cos(2 * x) + np.cos(2 * y)) * (np.cos(2 * z) + 2.0) / 16.0
    rho = C.gM2 * p
    rng = np.random.default_rng(seed)
    u0 = u0 + rng.uniform(-amp, amp, shape)
    u1 = u1 + rng.uniform(-amp, amp, shape)
    u2 = u2 + rng.uniform(-amp, amp, shape)
    return g, state_from_primitives(g, C, rho + np.zeros(shape),
                                    [u0, u1, u2], p + np.zeros(shape))


def residual_case(state, tag):
    results = {}
    for name in PLAN_NAMES:
        res = assemble_residual(state, C, name)
        results[name] = np.stack([f.interior.copy() for f in res.fields])
    for name in PLAN_NAMES:   # the reference's own cross-plan contract
        assert np.array_equal(results[name], results["BL"]), (tag, name)
    return results["BL"]


def run_case(grid, state, plan, dt, steps, cadence):
    rho0 = mean_density(state)
    ev = ResidualEvaluator(grid, C, plan, workers=8)
    t0 = time.time()
    rep = run(state, RKScheme(dt=dt), ev, steps, cadence=cadence,
              collect=make_collector(grid, rho0))
    hist = [[r.time, r.kinetic_energy, r.enstrophy, r.total_mass,
             *r.total_momentum, r.total_energy] for r in rep.records]
    final = cons_interior(state)
    return {
        "plan": plan, "n": list(grid.npoints), "dt": dt, "steps": steps,
        "cadence": cadence, "rho0": rho0,
        "sha256": [sha(f) for f in final],
        "absmax": [float(np.max(np.abs(f))) for f in final],
        "history_columns": ["time", "ke", "enstrophy", "mass", "mom0",
                            "mom1", "mom2", "energy"],
        "history": hist,
        "ref_seconds": time.time() - t0,
    }, final


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true",
                    help="also run the 64^3/100-step and 128^3/200-step cases")
    ap.add_argument("--large", action="store_true",
                    help="only the C4 (256^3, 100 steps) and C5 (512^3, 2 "
                         "steps) runs, merged into golden_meta.json")
    args = ap.parse_args()
    if args.large:
        return main_large()
    meta = {"generator": "tests/golden/make_golden.py",
            "reference": "/root/reference/pkg (fdns 0.1.0)",
            "perturb_seed": PERTURB_SEED}

    # A/B: single residual evaluations (plan.py:419-426), cube and ragged
    arrays = {}
    for tag, npts in (("m16", (16, 16, 16)), ("m_ragged", (9, 12, 7))):
        g = make_grid(npts, (TWO_PI,) * 3)
        st = manufactured_state(g, C)
        arrays[f"{tag}_cons"] = cons_interior(st)
        arrays[f"{tag}_res"] = residual_case(st, tag)
    # C: perturbed TGV residual (state pinned by hash, rebuilt from seed)
    g, st = perturbed_tgv(16)
    arrays["p16_res"] = residual_case(st, "p16")
    meta["p16_cons_sha256"] = [sha(f) for f in cons_interior(st)]
    # TGV 32^3 initial state + primitives (diagnostics.py:55-86)
    g32 = cube(32)
    st32 = taylor_green_init(g32, C)
    meta["tgv32_cons_sha256"] = [sha(f) for f in cons_interior(st32)]
    meta["tgv32_prim_sha256"] = [sha(f.interior) for f in
                                 (*st32.u, st32.p, st32.T)]
    rho0 = mean_density(st32)
    meta["tgv32_rho0"] = rho0
    meta["tgv32_ke0"] = kinetic_energy_integral(st32, g32, rho0)
    meta["tgv32_enstrophy0"] = enstrophy_integral(st32, g32, rho0)
    # known answers: primitives and constants (test_physics.py:65-81,158-161)
    g5 = cube(5)
    shape = (5, 5, 5)
    ka = state_from_primitives(g5, C, np.full(shape, 2.0),
                               [np.full(shape, 1.0), np.zeros(shape),
                                np.zeros(shape)], np.full(shape, 0.8))
    eval_primitives_fused(ka, C)
    meta["known_answer_prim"] = {
        "u0": float(ka.u[0].interior[0, 0, 0]),
        "p": float(ka.p.interior[0, 0, 0]),
        "T": float(ka.T.interior[0, 0, 0])}
    # plan introspection (terms.py:190-193, plan.py:220-264)
    from fdns import terms
    from fdns.plan import build_plan, lower_plan, workarray_budget
    spec = terms.build_residual_spec()
    meta["occurrences"] = dict(spec.occurrences)
    meta["stencil_applications_per_point"] = {
        n: lower_plan(build_plan(n)).stencil_applications_per_point()
        for n in PLAN_NAMES}
    meta["workarray_budget"] = {n: workarray_budget(build_plan(n))
                                for n in PLAN_NAMES}
    meta["constants"] = {"gm1": C.gm1, "gM2": C.gM2, "inv_Re": C.inv_Re,
                         "heat_coeff": C.heat_coeff, "c13": C.c13_inv_Re,
                         "c43": C.c43_inv_Re, "c23": C.c23_inv_Re}

    # D: config C1 -- TGV 32^3, BL, 10 steps, dt=2e-3
    st = taylor_green_init(g32, C)
    meta["c1_tgv32_bl"], final = run_case(g32, st, "BL", 2e-3, 10, 1)
    arrays["c1_final_rho"] = final[0]

    if args.big:
        # E: config C2 -- TGV 64^3, 100 steps, dt=3.385e-3 (SS; all plans
        # are bitwise equal in the reference)
        g64 = cube(64)
        st = taylor_green_init(g64, C)
        meta["c2_tgv64"], _ = run_case(g64, st, "SS", 3.385e-3, 100, 10)
        # F: config C3 -- perturbed TGV 128^3, 200 steps, dt=1.69e-3
        g128, st = perturbed_tgv(128)
        meta["c3_ptgv128_cons0_sha256"] = [sha(f) for f in cons_interior(st)]
        meta["c3_ptgv128"], _ = run_case(g128, st, "SN", 1.69e-3, 200, 20)

    np.savez_compressed(OUT / "golden_small.npz", **arrays)
    prev = {}
    path = OUT / "golden_meta.json"
    if path.exists():
        prev = json.loads(path.read_text())
    prev.update(meta)
    path.write_text(json.dumps(prev, indent=1) + "\n")
    print("wrote", sorted(arrays), sorted(meta))


def main_large():
    """Configs C4 and C5 (BASELINE.json configs[3], configs[4]) through the
    reference's SN route (all plans are bitwise equal in the reference,
    `test_output.txt:247`): final-field SHA-256 plus the diagnostics
    history.  C4: TGV 256^3, dt=8.5e-4, 100 steps (sampled every 10);
    C5: TGV 512^3, dt=4.2e-4, 2 steps (sampled every step) -- the most this
    container's 62 GB and the reference's single-threaded numpy stages
    allow in reasonable time."""
    meta = {}
    g256 = cube(256)
    st = taylor_green_init(g256, C)
    meta["c4_tgv256"], _ = run_case(g256, st, "SN", 8.5e-4, 100, 10)
    print("c4", meta["c4_tgv256"]["ref_seconds"], flush=True)
    _merge(meta)
    del st
    g512 = cube(512)
    st = taylor_green_init(g512, C)
    meta = {}
    meta["c5_tgv512"], _ = run_case(g512, st, "SN", 4.2e-4, 2, 1)
    print("c5", meta["c5_tgv512"]["ref_seconds"], flush=True)
    _merge(meta)


def _merge(meta):
    path = OUT / "golden_meta.json"
    prev = json.loads(path.read_text()) if path.exists() else {}
    prev.update(meta)
    path.write_text(json.dumps(prev, indent=1) + "\n")


if __name__ == "__main__":
    main()
