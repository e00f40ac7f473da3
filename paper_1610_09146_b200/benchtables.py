"""Per-variant runtime tables and scaling tables in the reference's formats.

Mirrors `fdns.bench` (pkg/src/fdns/bench.py) with GPUs in place of worker
threads: `TimingRecord`, `auto_dt`, `bench_variants` (the `_time_cell`
method of bench.py:51-71: fresh Taylor-Green state per cell, two untimed
warm-up iterations, the timed `run`'s `loop_seconds`, minimum over
repeats), `speedup_rows`, `write_bench_csv`, `write_speedup_csv`
(bench.py:91-126), `ScalingRecord` and `write_scaling_csv`
(bench.py:129-205), and the scaling drivers `strong_scaling`,
`weak_scaling` and `decompose_workers` (bench.py:138-196) with GPUs in
place of threads: one process drives one GPU, so a cell on N > 1 GPUs runs
N ranks under torch.distributed.run (z-slab decomposition, NCCL halo
exchange), each timing its loop, the MAX over ranks reported.  Tables can
also be assembled from `bench.py --gpus N` lines with `scaling_records`.

    python -m paper_1610_09146_b200.benchtables --grids 64,128 \
        --iterations 100 --out results/
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
from dataclasses import dataclass

import numpy as np

TWO_PI = 2.0 * math.pi
DT_64 = 3.385e-3                     # bench.py:28


def auto_dt(npoints) -> float:
    """dt from the 64^3 value, halved per 8x point increase (bench.py:31-34)."""
    factor = float(np.prod(npoints)) / 64 ** 3
    return DT_64 / factor ** (1.0 / 3.0)


@dataclass(frozen=True)
class TimingRecord:
    """bench.py:37-48; `workers` counts GPUs here."""

    grid: tuple
    plan: str
    workers: int
    iterations: int
    loop_seconds: float
    final_ke: float = float("nan")

    @property
    def seconds_per_iteration(self) -> float:
        return self.loop_seconds / max(self.iterations, 1)

    @property
    def pt_stage_per_s(self) -> float:
        return float(np.prod(self.grid)) * 3 * self.iterations / self.loop_seconds


def _time_cell(npoints, plan_name, iterations, constants, warmup=2,
               repeats=1, dt=None, slab=None) -> TimingRecord:
    """bench.py:51-71 on this process's GPU; with `slab`, this rank's share
    of a z-slab decomposed grid (the caller reduces over ranks)."""
    import paper_1610_09146_b200 as fd
    grid = fd.make_grid(npoints, (TWO_PI,) * 3, slab=slab)
    dt = auto_dt(npoints) if dt is None else dt
    scheme = fd.RKScheme(dt=dt)
    best, final_ke = None, float("nan")
    for _ in range(max(repeats, 1)):
        state = fd.taylor_green_init(grid, constants)
        rho0 = fd.mean_density(state)
        ev = fd.ResidualEvaluator(grid, constants, plan_name)
        fd.run(state, scheme, ev, warmup)
        report = fd.run(state, scheme, ev, iterations)
        if best is None or report.loop_seconds < best:
            best = report.loop_seconds
        final_ke = fd.kinetic_energy_integral(state, grid, rho0)
    gpus = 1 if slab is None else slab.nranks
    return TimingRecord(tuple(npoints), plan_name, gpus, iterations, best,
                        final_ke)


def _free_port() -> int:
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    return port


def time_cell_gpus(npoints, plan_name, gpus, iterations, constants=None,
                   repeats=1, dt=None) -> TimingRecord:
    """One timing cell on `gpus` GPUs of this node: in process for one GPU,
    else `gpus` ranks under torch.distributed.run (127.0.0.1 rendezvous)
    running `_cell_worker`; loop_seconds is the MAX over ranks."""
    if gpus == 1:
        import paper_1610_09146_b200 as fd
        return _time_cell(npoints, plan_name, iterations,
                          constants or fd.PhysicalConstants(),
                          repeats=repeats, dt=dt)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", "-m", __name__, "--cell",
           "--cell-grid", ",".join(map(str, npoints)), "--cell-plan",
           plan_name, "--iterations", str(iterations), "--repeats",
           str(repeats)] + (["--cell-dt", repr(dt)] if dt is not None else [])
    out = subprocess.run(cmd, capture_output=True, text=True,
                         cwd=os.path.dirname(os.path.dirname(
                             os.path.abspath(__file__))))
    if out.returncode != 0:
        raise RuntimeError(f"scaling cell on {gpus} GPUs failed:\n"
                           + out.stderr[-2000:])
    rec = json.loads([l for l in out.stdout.splitlines()
                      if l.startswith("{")][-1])
    return TimingRecord(tuple(rec["grid"]), rec["plan"], rec["workers"],
                        rec["iterations"], rec["loop_seconds"],
                        rec["final_ke"])


def _cell_worker(a) -> None:
    """One rank of a multi-GPU cell (launched by time_cell_gpus)."""
    import torch
    import torch.distributed as dist
    import paper_1610_09146_b200 as fd
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    npoints = tuple(int(x) for x in a.cell_grid.split(","))
    slab = fd.Slab.from_process_group(npoints[0])
    rec = _time_cell(npoints, a.cell_plan, a.iterations,
                     fd.PhysicalConstants(), repeats=a.repeats,
                     dt=a.cell_dt, slab=slab)
    t = torch.tensor([rec.loop_seconds], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if dist.get_rank() == 0:
        print(json.dumps({"grid": list(rec.grid), "plan": rec.plan,
                          "workers": rec.workers,
                          "iterations": rec.iterations,
                          "loop_seconds": float(t[0]),
                          "final_ke": rec.final_ke}), flush=True)
    dist.destroy_process_group()


def bench_variants(grids, plans=("BL", "RA", "RS", "SN", "SS"),
                   iterations=100, constants=None, repeats=1,
                   verbose=False):
    """One timing record per (grid, plan) on this process's GPU
    (bench.py:74-88)."""
    import paper_1610_09146_b200 as fd
    constants = constants or fd.PhysicalConstants()
    records = []
    for npoints in grids:
        for plan in plans:
            rec = _time_cell(npoints, plan, iterations, constants,
                             repeats=repeats)
            records.append(rec)
            if verbose:
                print(f"{npoints} {plan}: {rec.loop_seconds:.4f} s "
                      f"({rec.pt_stage_per_s:.3e} pt-stage/s)", flush=True)
    return records


def speedup_rows(records):
    """BL-normalised speedups per grid (bench.py:91-105)."""
    grids, plans = [], []
    for rec in records:
        if rec.grid not in grids:
            grids.append(rec.grid)
        if rec.plan not in plans:
            plans.append(rec.plan)
    by_cell = {(rec.grid, rec.plan): rec for rec in records}
    rows = []
    for grid in grids:
        base = by_cell[(grid, "BL")].loop_seconds
        rows.append((grid, {p: base / by_cell[(grid, p)].loop_seconds
                            for p in plans}))
    return rows


def write_bench_csv(records, path):
    """bench.py:108-113 columns (workers = GPUs)."""
    with open(path, "w", newline="") as fh:
        fh.write("Nx,Ny,Nz,plan,workers,iterations,loop_seconds\n")
        for r in records:
            fh.write(f"{r.grid[0]},{r.grid[1]},{r.grid[2]},{r.plan},"
                     f"{r.workers},{r.iterations},{r.loop_seconds:.6f}\n")


def write_speedup_csv(records, path):
    """bench.py:116-126."""
    plans = []
    for r in records:
        if r.plan not in plans:
            plans.append(r.plan)
    with open(path, "w", newline="") as fh:
        fh.write("Nx,Ny,Nz," + ",".join(plans) + "\n")
        for grid, speedups in speedup_rows(records):
            row = [str(grid[0]), str(grid[1]), str(grid[2])]
            row += [f"{speedups[p]:.4f}" for p in plans]
            fh.write(",".join(row) + "\n")


@dataclass(frozen=True)
class ScalingRecord:
    """bench.py:129-135; `workers` counts GPUs."""

    workers: int
    grid: tuple
    loop_seconds: float
    normalized: float
    ideal: float


def scaling_records(lines, strong=True):
    """Scaling table from `bench.py --gpus N` JSON lines (one per N): the
    per-step time of the headline variant, normalised by the smallest N,
    with the ideal of bench.py:160-163 (strong) or 1.0 (weak)."""
    rows = sorted((json.loads(l) if isinstance(l, str) else l for l in lines),
                  key=lambda d: d["n_gpus"])
    base_n = rows[0]["n_gpus"]
    base_t = rows[0]["ms_per_step"]
    out = []
    for d in rows:
        t = d["ms_per_step"]
        out.append(ScalingRecord(
            workers=d["n_gpus"], grid=tuple(d["config"]["grid"]),
            loop_seconds=t * d["steps"] / 1e3, normalized=t / base_t,
            ideal=(base_n / d["n_gpus"]) if strong else 1.0))
    return out


def decompose_workers(workers: int) -> tuple:
    """Split a GPU count into three near-equal grid scale factors
    (bench.py:160-173): its prime factors, largest first, each multiplied
    into the currently smallest factor; returned in descending order."""
    factors = [1, 1, 1]
    w, d, primes = workers, 2, []
    while w > 1:
        while w % d == 0:
            primes.append(d)
            w //= d
        d += 1
    for p in sorted(primes, reverse=True):
        factors[int(np.argmin(factors))] *= p
    return tuple(sorted(factors, reverse=True))


def strong_scaling(npoints, plan_name, worker_list, iterations,
                   constants=None, repeats=1, verbose=False,
                   timer=time_cell_gpus):
    """Fixed global grid, varying GPU counts (bench.py:138-157): loop times
    normalised by the first count's, with the ideal base/N."""
    raw = []
    for gpus in worker_list:
        rec = timer(tuple(npoints), plan_name, gpus, iterations,
                    constants=constants, repeats=repeats)
        raw.append(rec)
        if verbose:
            print(f"strong {tuple(npoints)} gpus={gpus} "
                  f"{rec.loop_seconds:.3f}s", flush=True)
    base_w, base_t = worker_list[0], raw[0].loop_seconds
    return [ScalingRecord(workers=w, grid=r.grid, loop_seconds=r.loop_seconds,
                          normalized=r.loop_seconds / base_t,
                          ideal=base_w / w)
            for w, r in zip(worker_list, raw)]


def weak_scaling(points_per_worker, plan_name, worker_list, iterations,
                 constants=None, repeats=1, verbose=False,
                 timer=time_cell_gpus):
    """Fixed share per GPU (bench.py:176-196): the global grid is the
    per-GPU grid times decompose_workers(N) axis by axis (the z-slab split
    then hands each rank the same number of points); ideal 1."""
    raw = []
    for gpus in worker_list:
        f = decompose_workers(gpus)
        npoints = tuple(points_per_worker[a] * f[a] for a in range(3))
        rec = timer(npoints, plan_name, gpus, iterations,
                    constants=constants, repeats=repeats)
        raw.append(rec)
        if verbose:
            print(f"weak {npoints} gpus={gpus} {rec.loop_seconds:.3f}s",
                  flush=True)
    base_t = raw[0].loop_seconds
    return [ScalingRecord(workers=w, grid=r.grid, loop_seconds=r.loop_seconds,
                          normalized=r.loop_seconds / base_t, ideal=1.0)
            for w, r in zip(worker_list, raw)]


def write_scaling_csv(records, path):
    """bench.py:199-205."""
    with open(path, "w", newline="") as fh:
        fh.write("workers,Nx,Ny,Nz,runtime,normalized,ideal\n")
        for r in records:
            fh.write(f"{r.workers},{r.grid[0]},{r.grid[1]},{r.grid[2]},"
                     f"{r.loop_seconds:.6f},{r.normalized:.6f},"
                     f"{r.ideal:.6f}\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grids", default="64,128")
    ap.add_argument("--plans", default="BL,RA,RS,SN,SS")
    ap.add_argument("--iterations", type=int, default=100)
    ap.add_argument("--repeats", type=int, default=1)
    ap.add_argument("--out", default=".")
    ap.add_argument("--scaling", choices=["strong", "weak"], default=None,
                    help="write scaling.csv over --gpus-list instead")
    ap.add_argument("--gpus-list", default="1,2,4,8")
    ap.add_argument("--cell", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--cell-grid", help=argparse.SUPPRESS)
    ap.add_argument("--cell-plan", help=argparse.SUPPRESS)
    ap.add_argument("--cell-dt", type=float, default=None,
                    help=argparse.SUPPRESS)
    a = ap.parse_args()
    if a.cell:
        return _cell_worker(a)
    if a.scaling:
        n = int(a.grids.split(",")[0])
        gl = [int(x) for x in a.gpus_list.split(",")]
        plan = a.plans.split(",")[0]
        fn = strong_scaling if a.scaling == "strong" else weak_scaling
        recs = fn((n,) * 3, plan, gl, a.iterations, repeats=a.repeats,
                  verbose=True)
        os.makedirs(a.out, exist_ok=True)
        write_scaling_csv(recs, os.path.join(a.out, "scaling.csv"))
        return None
    grids = [(int(n),) * 3 for n in a.grids.split(",")]
    recs = bench_variants(grids, a.plans.split(","), a.iterations,
                          repeats=a.repeats, verbose=True)
    os.makedirs(a.out, exist_ok=True)
    write_bench_csv(recs, os.path.join(a.out, "bench.csv"))
    if "BL" in a.plans.split(","):
        write_speedup_csv(recs, os.path.join(a.out, "speedup.csv"))


if __name__ == "__main__":
    main()
