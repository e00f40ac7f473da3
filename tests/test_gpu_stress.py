"""Race stress tests (driver-visible): many repeated short runs of every
TMA-ring stage kernel, each required to be bitwise equal to the
one-thread-per-point kernels (which share no shared memory, no ring and no
prefetch with them).

Round 1 saw intermittent corruption (~50% of repeated 2-step runs) in a
since-removed 12-warp SS/RS layout when the L2 prefetch of the stored
gradients was on.  A race of that kind shows up here as
run-to-run differences: the runs cover the 8-warp SS/RS/RA/SN kernel, the
12-warp SN, RA, SS and RS kernels,
the SS/RS/SN round-robin split (with its lockstep and its partial last
round), forced small CTA counts
(many segment transitions per CTA), ragged grids (partial tiles), and the
gradient / saved-state prefetches both on and off.  compute-sanitizer is not
available on the GPU pool; this is its stand-in.
"""

import itertools

import numpy as np
import pytest
import torch

from oracle import numpy_oracle as npo

pytestmark = pytest.mark.gpu

fd = pytest.importorskip("paper_1610_09146_b200")
TWO_PI = 2.0 * np.pi
C = fd.PhysicalConstants()
CO = npo.Consts()

GRIDS = [(12, 16, 20), (16, 13, 34), (24, 24, 40)]


@pytest.fixture
def lib(built):
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    torch.cuda.set_device(0)
    from paper_1610_09146_b200 import _lib
    lib = _lib.load()
    yield lib
    lib.fdns_set_kernel_path(0)
    lib.fdns_set_tiled_grid(0)
    lib.fdns_set_rounds(-1)
    lib.fdns_set_lockstep(-1)
    lib.fdns_set_prefetch(3)


def _cons(npts):
    F = npo.manufactured(npts, CO)
    return npo.interior(F[:5], 2)


def _run(npts, cons, variant, steps):
    from paper_1610_09146_b200.diagnostics import state_from_conservative
    g = fd.make_grid(npts, (TWO_PI,) * 3)
    st = state_from_conservative(g, C, cons)
    fd.run(st, fd.RKScheme(dt=1e-3), fd.ResidualEvaluator(g, C, variant), steps)
    torch.cuda.synchronize()
    return g.interior(st.bundle[:5]).cpu().numpy()


# (variant, kernel path, forced CTA counts, round-robin unit)
CASES = [("SN", 2, (0, 5, 13), -1), ("SN", 5, (0, 5, 13), -1),
         ("RA", 2, (0, 7), -1), ("RA", 5, (0, 5, 13), -1),
         ("SS", 5, (0, 5, 13), -1), ("SS", 5, (0,), 4),
         ("RS", 5, (0, 5, 13), -1), ("RS", 5, (0,), 4),
         ("SS", 0, (0, 5, 13), -1), ("SS", 0, (0,), 4),
         ("RS", 0, (0, 5, 13), -1), ("RS", 0, (0,), 4),
         # round-robin units on a forced CTA count: whole rounds in lockstep,
         # then the partial last round cut into per-CTA plane ranges
         ("SS", 5, (5, 3), 4), ("SN", 5, (0, 5, 3), 4), ("RS", 5, (4,), 4),
         ("SS", 0, (5, 3), 4), ("RS", 0, (4,), 4)]


@pytest.mark.parametrize("variant,path,ctas_list,rounds", CASES)
def test_repeated_runs_bitwise_stable(lib, variant, path, ctas_list, rounds):
    """>= 100 repeated 2-3 step runs per case, all equal to the point
    kernels' result."""
    runs = 0
    for npts in GRIDS:
        cons = _cons(npts)
        lib.fdns_set_kernel_path(1)
        steps = 3 if npts[0] <= 16 else 2
        want = _run(npts, cons, variant, steps)
        lib.fdns_set_kernel_path(path)
        lib.fdns_set_rounds(rounds)
        reps = max(1, 36 // (len(ctas_list) * 2))
        for ctas, pf in itertools.product(ctas_list, (3, 0)):
            lib.fdns_set_tiled_grid(ctas)
            lib.fdns_set_prefetch(pf)
            for rep in range(reps):
                got = _run(npts, cons, variant, steps)
                runs += 1
                if not np.array_equal(got, want):
                    d = np.argwhere(got != want)
                    pytest.fail(f"{variant} path {path} grid {npts} ctas {ctas} "
                                f"prefetch {pf} rounds {rounds} rep {rep}: "
                                f"{len(d)} values differ, first at {d[0].tolist()}")
        lib.fdns_set_tiled_grid(0)
        lib.fdns_set_prefetch(3)
        lib.fdns_set_rounds(-1)
    assert runs >= 100


@pytest.mark.parametrize("variant,path", [("SS", 5), ("SN", 5), ("RS", 0)])
def test_lockstep_slack_does_not_change_results(lib, variant, path):
    """The round-robin CTAs' lockstep (fdns_set_lockstep) only changes when
    a CTA runs, never what it computes: free running (0), the tightest
    slack (1), the default and a loose one are all bitwise the point
    kernels' result, on a forced 5-CTA grid whose last round is partial."""
    npts = (24, 24, 40)
    cons = _cons(npts)
    lib.fdns_set_kernel_path(1)
    want = _run(npts, cons, variant, 2)
    lib.fdns_set_kernel_path(path)
    lib.fdns_set_rounds(4)
    lib.fdns_set_tiled_grid(5)
    try:
        for slack in (0, 1, -1, 4):
            lib.fdns_set_lockstep(slack)
            for rep in range(3):
                got = _run(npts, cons, variant, 2)
                assert np.array_equal(got, want), (variant, slack, rep)
    finally:
        lib.fdns_set_lockstep(-1)
