"""Benchmark: grid-point x RK-stage updates/s per variant (BL/RA/SN/SS), fp64.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--grid 512]
                    [--variants BL,RA,SN,SS] [--impl ours|reference]
                    [--scaling strong|weak]

Workload (BASELINE.json configs[4], "C5"): Taylor-Green vortex 512^3, fp64,
dt=4.2e-4, RK3 steps of each of BL/RA/SN/SS -- the largest configuration
that fits one GPU (BL's 90 padded fields are ~99 GB of the 180 GB HBM).  A
"step" is one full RK3 iteration (3 stages); the unit of work is one
interior grid point advanced through one RK stage, so value = N^3 * 3 * K /
seconds.  Inputs are larger than L2 (one field is 1.1 GB) and L2 is flushed
between timed steps anyway.

Timing: W untimed warm-up steps, then K steps, each timed with CUDA events
on the launching stream (on one GPU the step is one captured CUDA graph).
Multi-GPU: `--gpus N` without a launcher re-executes this script under
`torch.distributed.run` with N ranks (127.0.0.1); each rank owns a z-slab
(axis 0) of the grid, the periodic 2-plane halo exchange runs over NCCL,
overlapped with the interior planes, and the per-rank time is reduced with
MAX.  --scaling strong (default: the n^3 grid split over N ranks, the
north-star's 8-GPU 512^3 target) or weak (each rank owns n planes).

--impl reference times the reference algorithm's CPU restatement (the C +
OpenMP oracle, pinned bitwise to the reference) on the host cores, on the
same workload and config; the reference package itself is pure
Python/numba and does not exist on the GPU box.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("grid-pt·RK-stage updates/s per variant (BL/RA/SN/SS), fp64; "
          "% of roofline")
UNIT = "grid-pt*RK-stage/s"
DT = {64: 3.385e-3, 128: 1.69e-3, 256: 8.5e-4, 512: 4.2e-4, 32: 2e-3,
      1024: 2.1e-4}
CONFIG_NAMES = {32: "C1", 64: "C2", 128: "C3", 256: "C4", 512: "C5",
                1024: "C5 (weak counterpart)"}

# Algorithmic per-point costs of one RK stage ("Whole RK stage
# per point"):
#   flops F_v = residual source flops + fills + 10 (update) + 13 (primitives)
#   (BL 223 + 360 fill + 18 mixed fill + 23 ... as tabulated there)
#   bytes: model M for the fused stage = read 10 state fields + 5 saved
#   (stage 0: saved == input) + write 10, plus each FETCH array written and
#   read once by the fills/residual.
RESIDUAL_FLOPS = {"BL": 223, "RA": 1318, "RS": 838, "SN": 895, "SS": 730}
STAGE_FLOPS = {"BL": 627, "RA": 1341, "RS": 906, "SN": 918, "SS": 798}
N_WORK = {"BL": 60, "RA": 0, "RS": 9, "SN": 0, "SS": 9}


# Algorithmic HBM bytes per point of one RK stage: SURVEY.md 8d's model M
# (primitives materialised once, each FETCH array written and read once,
# the residual kernel reading its point fields and the RK update its 15
# accesses, save-state 10/3), minus the 80 B of the residual store and
# re-read for a path whose residual and update are fused ("If
# residual and update are fused ... subtract 10 accesses (80 B)") -- the
# contract's per-unit figure.
SURVEY_MODEL_M = {"BL": 1370.7, "RA": 346.7, "RS": 514.7, "SN": 346.7, "SS": 514.7}


def stage_bytes(v: str) -> float:
    """SURVEY 8d model-M bytes per point of one fused RK stage."""
    return SURVEY_MODEL_M[v] - 80.0


def stage_bytes_design(v: str) -> float:
    """The stricter compulsory bytes of this design's fused stage (round
    1's model; primitives are never materialised here -- p, T are derived
    on arrival -- and the save-state copy is gone): read 10 state fields +
    5 saved (stage 0 reads its saved fields as the input) + write 10, plus
    each FETCH array written and read once."""
    state = (10 + 5 * 2.0 / 3.0 + 10) * 8.0
    return state + 2 * 8.0 * N_WORK[v]


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int, period_ms: int = 100):
        self.index = index
        self.period_ms = period_ms
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:6])
                          if v.lower() == "active"})
        pw = [float(r[6]) for r in self.rows
              if len(r) > 6 and r[6].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows),
                "power_w": float(np.median(pw)) if pw else None}


# ------------------------------------------------------------------ setup
def init_dist(args):
    """Rank/world from the launcher's environment; NCCL for N > 1.  A world
    size that disagrees with --gpus is an error, not a silent 1-GPU run."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if (world > 1 or args.loopback) and args.impl == "ours":
        import torch
        import torch.distributed as dist
        if world == 1:   # --loopback: a one-rank NCCL group of our own
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def free_port() -> int:
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    return port


def launcher_cmd(argv, gpus: int, port: int) -> list:
    """The torchrun command that runs this script on `gpus` ranks of one
    node (127.0.0.1 rendezvous), forwarding the original arguments."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1",
            f"--master-port={port}", os.path.abspath(__file__), *argv]


def self_launch(args, argv) -> int | None:
    """`--gpus N` (N > 1) with no launcher around us: re-execute under
    torch.distributed.run with N ranks and return its exit code."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    return subprocess.call(launcher_cmd(argv, args.gpus, free_port()))


def cpu_cores() -> int:
    return len(os.sched_getaffinity(0))


def weak_factors(world: int) -> tuple:
    """Grid scale factors of a weak-scaling run on `world` GPUs: the
    reference's decompose_workers (pkg/src/fdns/bench.py:160-173; the same
    rule as benchtables.decompose_workers, kept here so the reference arm
    needs no package import): 8 GPUs scale n^3 to (2n)^3, so C5's 512^3 on
    one GPU meets its 1024^3 8-GPU counterpart (BASELINE.json configs[4])."""
    factors, w, d, primes = [1, 1, 1], world, 2, []
    while w > 1:
        while w % d == 0:
            primes.append(d)
            w //= d
        d += 1
    for p in sorted(primes, reverse=True):
        factors[factors.index(min(factors))] *= p
    return tuple(sorted(factors, reverse=True))


def global_grid(args, world: int) -> tuple:
    """Global grid points: n^3, or n x weak_factors(world) for weak scaling
    (slabs are still cut along axis 0)."""
    n = args.n
    if world > 1 and args.scaling == "weak":
        return tuple(n * f for f in weak_factors(world))
    return (n, n, n)


def dt_of(npts) -> float:
    """RK3 step of a grid: the configs' dt of its finest axis."""
    return DT.get(max(npts), 3.385e-3)


def config_dict(args, world: int) -> dict:
    """The workload description both arms print (identical by construction)."""
    npts = global_grid(args, world)
    n = args.n
    weak = tuple(npts) != (n, n, n)
    name = CONFIG_NAMES.get(max(npts) if weak and len(set(npts)) == 1 else n, "custom")
    if weak and len(set(npts)) != 1:
        name += f" weak x{world}"
    return {"workload": f"{name}: TGV {'x'.join(map(str, npts))} fp64, "
                        f"dt={dt_of(npts)}, RK3 steps, variants "
                        + "/".join(args.variants)
                        + (f", z-slab over {world} GPUs ({args.scaling} "
                           "scaling)" if world > 1 else ""),
            "grid": list(npts), "dt": dt_of(npts),
            "variants": list(args.variants),
            "parallelism": f"z-slab x{world}" + (" (weak)" if weak else ""),
            "l2": "inputs larger than L2 (1.1 GB per 512^3 field); L2 also "
                  "flushed between timed steps (256 MiB write)"}


def run_cpu_oracle(npts, steps: int, warmup: int = 1, min_seconds: float = 0.0):
    """The C + OpenMP restatement of the reference path (oracle/), timed on
    the host cores: pt-stage/s.  `npts` is n (a cube: the TGV) or a grid
    tuple (a weak-scaled slab grid: the manufactured smooth state of the
    same shape).  Runs `steps` iterations, repeated until at least
    `min_seconds` of CPU work has been timed."""
    from oracle import c_oracle, numpy_oracle as npo
    c = npo.Consts()
    npts = (npts,) * 3 if isinstance(npts, int) else tuple(npts)
    n = npts[1]
    F = npo.taylor_green(n, c) if len(set(npts)) == 1 else npo.manufactured(npts, c)
    # every host thread, explicitly: torchrun exports OMP_NUM_THREADS=1
    threads = cpu_cores()
    if warmup:
        c_oracle.run(F, c, DT.get(n, 3.385e-3), warmup, nthreads=threads)
    done, dt = 0, 0.0
    while done == 0 or dt < min_seconds:
        t0 = time.perf_counter()
        c_oracle.run(F, c, DT.get(n, 3.385e-3), steps, nthreads=threads)
        dt += time.perf_counter() - t0
        done += steps
    return float(np.prod(npts)) * 3 * done / dt, dt, done


# ------------------------------------------------------------------ ours
def fresh_state(fd, grid, cons_host):
    """A device state from the cached host TGV arrays (same bits as
    taylor_green_init; the 512^3 host evaluation runs once per process)."""
    from paper_1610_09146_b200.diagnostics import state_from_conservative
    return state_from_conservative(grid, fd.PhysicalConstants(), cons_host)


def bench_variant(fd, variant, grid, cons_host, steps, warmup, flush_buf, lib,
                  clocks=None, clock_window=0.0):
    import torch
    from paper_1610_09146_b200 import _lib
    from paper_1610_09146_b200.timeloop import IterationState, _fused_iteration
    c = fd.PhysicalConstants()
    state = fresh_state(fd, grid, cons_host)
    ev = fd.ResidualEvaluator(grid, c, variant)
    scheme = fd.RKScheme(dt=dt_of(grid.npoints))
    it = IterationState(state, saved=False)
    multi = grid.slab is not None and grid.slab.distributed
    for _ in range(warmup):
        _fused_iteration(it, scheme, ev)
    torch.cuda.synchronize()

    graph = None
    if not multi:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            _fused_iteration(it, scheme, ev)      # warm the capture stream
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            _fused_iteration(it, scheme, ev)
        torch.cuda.synchronize()

    def step():
        if graph is not None:
            graph.replay()
        else:
            _fused_iteration(it, scheme, ev)

    stream = torch.cuda.current_stream()
    if clock_window > 0:
        # untimed replay of the same step, long enough for nvidia-smi to
        # sample the clocks under exactly this load
        with clocks:
            t_end = time.perf_counter() + clock_window
            while time.perf_counter() < t_end:
                for _ in range(4):
                    step()
                torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    launches_per_step = None
    if graph is not None:
        # graph replays do not pass through the ABI counter: count one
        # eager step's launches instead
        c0 = lib.fdns_launch_count()
        _fused_iteration(it, scheme, ev)
        launches_per_step = lib.fdns_launch_count() - c0
    if multi:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    n_launch0 = lib.fdns_launch_count()
    for k in range(steps):
        _lib.check(lib.fdns_l2_flush(_lib.ptr(flush_buf), flush_buf.numel(),
                                     _lib.stream_handle()), "flush")
        evs[k][0].record(stream)
        step()
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    launches = (launches_per_step * steps if launches_per_step is not None
                else lib.fdns_launch_count() - n_launch0)

    # informational: one stage (all its launches) timed alone after an L2
    # flush, eager launch, with a saved state distinct from the input
    X = state.bundle
    Y, Z = ev.workspace()
    kev = [(torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True)) for _ in range(5)]
    for a, b in kev:
        _lib.check(lib.fdns_l2_flush(_lib.ptr(flush_buf), flush_buf.numel(),
                                     _lib.stream_handle()), "flush")
        a.record(stream)
        if multi:
            ev.stage_exchanged(Y, X, Z, 1e-30)
        else:
            ev.stage(Y, X, Z, 1e-30)   # a stage-1/2 workload
        b.record(stream)
    torch.cuda.synchronize()
    stage_ms = float(np.median([a.elapsed_time(b) for a, b in kev]))
    del graph, state, ev, it, X, Y, Z
    torch.cuda.empty_cache()
    return total_ms, launches, stage_ms


def measured_traffic(variant: str, n: int):
    """DRAM bytes (read + write) of one RK stage -- all its launches: the
    fills and the stage kernel -- from the committed ncu --set full capture
    (profiles/traffic.json, tools/traffic_json.py), if one matches."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    rec = json.load(open(path)).get(f"{variant}@{n}")
    if not rec:
        return None
    return {"bytes_per_launch": rec["dram_bytes"], "unit": "B",
            "bytes_per_point": rec["dram_bytes"] / n ** 3,
            "fp64_insts_per_point": rec.get("fp64_insts_per_point"),
            "kernels": rec.get("kernels"),
            "source": rec["source"]}


def stage_sweep(fd, lib, sizes, variants, flush, fp64_tf, hbm_peak):
    """Steady-state view: one fused stage per variant at larger grids
    (CUDA events, L2 flushed before each launch).  Informational; the
    headline is the C5 workload above."""
    import torch
    from paper_1610_09146_b200 import _lib
    c = fd.PhysicalConstants()
    out = {}
    for n in sizes:
        g = fd.make_grid((n,) * 3, (2 * np.pi,) * 3)
        s = fd.taylor_green_init(g, c)
        for v in variants:
            ev = fd.ResidualEvaluator(g, c, v)
            Y, Z = ev.workspace()
            Y.copy_(s.bundle)
            ts = []
            for r in range(5):
                _lib.check(lib.fdns_l2_flush(_lib.ptr(flush), flush.numel(),
                                             _lib.stream_handle()))
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                ev.stage(Y, s.bundle, Z, 1e-30)   # saved != input
                b.record()
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(a.elapsed_time(b) / 1e3)
            sec = float(np.median(ts))
            pts = n ** 3 / sec
            t_f = STAGE_FLOPS[v] / (fp64_tf * 1e12)
            t_b = stage_bytes(v) / (hbm_peak * 1e9)
            out[f"{v}@{n}"] = {"pt_stage_per_s": pts, "stage_ms": sec * 1e3,
                               "frac_of_roofline": pts * max(t_f, t_b),
                               "bound": "fp64" if t_f >= t_b else "hbm"}
            del ev, Y, Z
        del s
        torch.cuda.empty_cache()
    return out


def fp64_peak(lib):
    """In-run FP64 issue-rate probe (DADD only, 1 flop per instruction)."""
    import torch
    from paper_1610_09146_b200 import _lib
    import ctypes
    scratch = torch.zeros(1, dtype=torch.float64, device="cuda")
    cnt = ctypes.c_double(0)
    iters = 20000
    for _ in range(2):
        _lib.check(lib.fdns_fp64_probe(_lib.ptr(scratch), iters,
                                       ctypes.byref(cnt), _lib.stream_handle()))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    reps = 5
    for _ in range(reps):
        _lib.check(lib.fdns_fp64_probe(_lib.ptr(scratch), iters,
                                       ctypes.byref(cnt), _lib.stream_handle()))
    b.record()
    torch.cuda.synchronize()
    sec = a.elapsed_time(b) / 1e3
    return cnt.value * reps / sec / 1e12   # T FP64 instr/s == TFLOP/s (DADD)


def fp64_peak_sustained(lib, index, seconds=3.0):
    """The same DADD probe looped back to back for `seconds` (under the
    1000 W power cap, like MEASURED_PEAKS.json's bf16_tflops_sustained), the
    rate over the last half, and the SM clock nvidia-smi saw meanwhile: the
    FP64 denominator for a kernel timed inside a long step."""
    import torch
    from paper_1610_09146_b200 import _lib
    import ctypes
    scratch = torch.zeros(1, dtype=torch.float64, device="cuda")
    cnt = ctypes.c_double(0)
    iters = 20000
    probe = lambda: _lib.check(lib.fdns_fp64_probe(   # noqa: E731
        _lib.ptr(scratch), iters, ctypes.byref(cnt), _lib.stream_handle()))
    probe()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cs = ClockSampler(index, period_ms=20)
    with cs:
        t_half = time.perf_counter() + seconds / 2
        while time.perf_counter() < t_half:
            for _ in range(8):
                probe()
            torch.cuda.synchronize()
        n0 = len(cs.rows)
        a.record()
        reps = 0
        t_end = time.perf_counter() + seconds / 2
        while time.perf_counter() < t_end:
            for _ in range(8):
                probe()
            reps += 8
            torch.cuda.synchronize()
        b.record()
        torch.cuda.synchronize()
    sec = a.elapsed_time(b) / 1e3
    rows = cs.rows[n0:]
    sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
    return {"tflops": cnt.value * reps / sec / 1e12,
            "sm_mhz": float(np.median(sm)) if sm else None,
            "seconds": seconds}


def median_mhz(rows):
    sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
    return float(np.median(sm)) if sm else None


def median_watts(rows):
    pw = [float(r[6]) for r in rows if len(r) > 6 and r[6].replace(".", "").isdigit()]
    return float(np.median(pw)) if pw else None


# FP64 lanes per SM per clock: the burst probe's 18.5 T instr/s at 1965 MHz
# over 148 SMs is 63.7
FP64_PER_SM_CLK = 64


E2E_CHUNKS = 5


def bench_e2e(fd, variant, grid, cons_host, steps):
    """Same metric through the public API with host buffers: per step the
    five conservative fields (padded, as the reference holds them) are
    uploaded from pinned memory, one fused RK3 iteration runs, and the new
    fields are downloaded into the same buffers (hostio.HostStepper, which
    pipelines chunked field copies over both PCIe directions).  The timed
    region ends after the last step's download."""
    import torch
    from paper_1610_09146_b200.hostio import HostStepper
    c = fd.PhysicalConstants()
    state = fresh_state(fd, grid, cons_host)
    ev = fd.ResidualEvaluator(grid, c, variant)
    scheme = fd.RKScheme(dt=dt_of(grid.npoints))
    host = HostStepper.pinned_buffers(grid)
    host.copy_(state.bundle[:5].cpu())
    stepper = HostStepper(state, ev, scheme, host, chunks=E2E_CHUNKS)
    for _ in range(2):
        stepper.step()
    stepper.wait()
    torch.cuda.synchronize()
    multi = grid.slab is not None and grid.slab.distributed
    if multi:
        import torch.distributed as dist
        dist.barrier()
    stream = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        stepper.step()
    stepper.wait()
    b.record(stream)
    torch.cuda.synchronize()
    sec = a.elapsed_time(b) / 1e3
    if multi:
        t = torch.tensor([sec], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t[0])
    npts = float(np.prod(grid.npoints))
    nbytes = host.numel() * 8
    wave = getattr(stepper, "wavefront", False)
    graphs = getattr(stepper, "use_graphs", False)
    kw = getattr(stepper, "_wK", None)
    stepper.close() if hasattr(stepper, "close") else None
    del stepper, state, ev, host
    torch.cuda.empty_cache()
    return {"value": npts * 3 * steps / sec, "unit": UNIT,
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
            "steps": steps, "variant": variant,
            "path": ("hostio.HostStepper: pinned host fields -> advance one "
                     "RK3 iteration -> host" + (
                         f"; wavefront mode: {kw} axis-0 plane chunks, each "
                         "uploaded in ring order, its primitives and every "
                         "stage launched as soon as the chunks it reads are "
                         "current, downloaded as its stage 3 completes; the "
                         "next step's upload of a chunk waits only for its "
                         "download (both PCIe directions and the compute "
                         "overlap)" if wave else
                         "; field copies in chunks, each upload chunk right "
                         "behind the previous result's download of it "
                         f"({E2E_CHUNKS} chunks/field)"
                         + (", CUDA graphs" if graphs else ""))
                     + ("; per rank: its slab" if multi else ""))}


def variant_roofline(v, rec, fp64_tf, hbm_peak, hbm_src, n, fp64_sus=None, sms=148):
    """The roofline object of one variant's stage: algorithmic
    flops or bytes per point x points / average stage duration, against the
    in-run FP64 issue probe or the measured HBM copy bandwidth; plus the
    executed-FP64 view where ncu counted the stage kernel's FP64
    instructions.  FP64: the stages are timed inside long steps under the
    power cap, so the denominator is the sustained probe (the rule
    MEASURED_PEAKS.json applies to bf16); the burst probe and the FP64 rate
    at the clock this variant actually ran at are reported beside it."""
    if rec["bound"] == "fp64":
        sus = (fp64_sus or {}).get("tflops")
        roof = {"bound": "fp64", "achieved": rec["achieved_tflops"],
                "peak": sus or fp64_tf, "unit": "TFLOP/s",
                "peak_source": (
                    f"measured in-run, sustained: DADD issue probe (no FMA) "
                    f"looped {fp64_sus['seconds']:.0f} s under the power cap, "
                    f"SM clock {fp64_sus['sm_mhz']} MHz" if sus else
                    "measured in-run (DADD issue probe, no-FMA, burst)")}
        roof["burst_view"] = {"peak": fp64_tf,
                              "frac": rec["achieved_tflops"] / fp64_tf,
                              "peak_source": "DADD probe, 5 launches (~13 ms), burst clock"}
        mhz = rec.get("sm_mhz")
        if mhz:
            at = sms * FP64_PER_SM_CLK * mhz * 1e6 / 1e12
            roof["clock_view"] = {
                "sm_mhz": mhz, "peak": at,
                "frac": rec["achieved_tflops"] / at,
                "peak_source": f"{sms} SMs x {FP64_PER_SM_CLK} FP64/clk x the "
                               "median SM clock under this variant's step"}
    else:
        roof = {"bound": "hbm", "achieved": rec["achieved_gbs"],
                "peak": hbm_peak, "unit": "GB/s",
                "peak_source": f"{hbm_src} (MEASURED_PEAKS.json hbm_gbs)"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["bytes_model"] = ("SURVEY 8d model M, fused residual+update "
                           f"(-80 B): {stage_bytes(v):.1f} B/pt; flops F_v "
                           f"{STAGE_FLOPS[v]}/pt")
    # the stricter design-compulsory byte model (round 1's): same time, the
    # roofline min(FP64, HBM) recomputed with it
    fpk = (fp64_sus or {}).get("tflops") or fp64_tf   # the FP64 denominator
    tb = stage_bytes_design(v) / (hbm_peak * 1e9)
    tf = STAGE_FLOPS[v] / (fpk * 1e12)
    pts_s = rec["local_pts"] / (rec["stage_kernel_ms"] / 1e3)
    roof["design_compulsory_view"] = {
        "bytes_per_pt": stage_bytes_design(v),
        "bound": "fp64" if tf >= tb else "hbm",
        "frac": pts_s * max(tf, tb)}
    tr = measured_traffic(v, n)
    roof["traffic"] = tr["bytes_per_launch"] if tr else None
    roof["traffic_detail"] = tr
    ex = (tr or {}).get("fp64_insts_per_point")
    if ex:
        pts_per_s = rec["local_pts"] / (rec["stage_kernel_ms"] / 1e3)
        roof["executed_fp64_view"] = {
            "fp64_insts_per_point": ex,
            "frac_of_fp64_issue_peak": pts_per_s * ex / (fpk * 1e12),
            "source": tr["source"]}
    roof["kernel"] = (f"RK stage ({v}): " + {
        "SN": "fused stage kernel (residual + RK update + primitives)",
        "RA": "fused stage kernel (residual + RK update + primitives)",
        "SS": "9-gradient fill + fused stage kernel",
        "RS": "9-gradient fill + fused stage kernel",
        "BL": "60-array fills + residual/update kernel"}[v])
    roof["duration"] = ("average stage duration over the timed region = "
                        "timed steps / (3 x steps); L2 flushed before every "
                        "step")
    return roof


def main_ours(args):
    import torch
    rank, world, local = init_dist(args)
    torch.cuda.set_device(local)
    import paper_1610_09146_b200 as fd
    from paper_1610_09146_b200 import _lib
    from paper_1610_09146_b200.diagnostics import taylor_green_conservative
    lib = _lib.load()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "measured" if "hbm_gbs" in peaks else "fallback"

    n = args.n
    npts = global_grid(args, world)
    dist_on = world > 1 or args.loopback
    slab = fd.Slab.from_process_group(npts[0], loopback=args.loopback) \
        if dist_on else None
    grid = fd.make_grid(npts, (2 * np.pi,) * 3, slab=slab)
    npts_total = float(np.prod(grid.npoints))
    comm = None
    if dist_on:
        import torch.distributed as dist
        comm = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                "local_planes": grid.local_npoints[0],
                "loopback": bool(args.loopback)}
    t0 = time.perf_counter()
    cons_host = taylor_green_conservative(grid, fd.PhysicalConstants())
    init_s = time.perf_counter() - t0
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    fp64_tf = fp64_peak(lib)
    fp64_sus = fp64_peak_sustained(lib, local) if args.clock_window > 0 else None
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    results = {}
    clocks = ClockSampler(local, period_ms=20)
    for v in args.variants:
        n_rows = len(clocks.rows)
        total_ms, launches, cold_ms = bench_variant(
            fd, v, grid, cons_host, args.steps, args.warmup, flush, lib,
            clocks, args.clock_window)
        v_mhz = median_mhz(clocks.rows[n_rows:])
        v_watts = median_watts(clocks.rows[n_rows:])
        if dist_on:
            import torch.distributed as dist
            t = torch.tensor([total_ms, cold_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total_ms, cold_ms = t.tolist()
        # average duration of one RK stage over the timed region: the step
        # is exactly three stages' launches back to back
        stage_ms = total_ms / (3 * args.steps)
        local_pts = float(np.prod(grid.local_npoints))
        val = npts_total * 3 * args.steps / (total_ms / 1e3)
        flops = STAGE_FLOPS[v] * local_pts / (stage_ms / 1e3) / 1e12
        gbs = stage_bytes(v) * local_pts / (stage_ms / 1e3) / 1e9
        t_fp64 = STAGE_FLOPS[v] / (((fp64_sus or {}).get("tflops") or fp64_tf) * 1e12)
        t_hbm = stage_bytes(v) / (hbm_peak * 1e9)
        bound = "fp64" if t_fp64 >= t_hbm else "hbm"
        rec = {
            "value": val, "ms_per_step": total_ms / args.steps,
            "gpu_launches": launches,
            "stage_kernel_ms": stage_ms,
            "stage_ms_isolated_cold": cold_ms,
            "stage_flops_per_pt": STAGE_FLOPS[v],
            "stage_bytes_per_pt": stage_bytes(v),
            "achieved_tflops": flops, "achieved_gbs": gbs,
            "bound": bound, "local_pts": local_pts,
            "roofline_pt_stage_per_s": 1.0 / max(t_fp64, t_hbm),
            "sm_mhz": v_mhz, "power_w": v_watts,
        }
        rec["roofline"] = variant_roofline(v, rec, fp64_tf, hbm_peak,
                                           hbm_src, n, fp64_sus, sms)
        results[v] = rec
    head = max(results, key=lambda v: results[v]["value"])   # same on all ranks
    r = results[head]
    # end-to-end through the public API with host buffers (all ranks)
    e2e = bench_e2e(fd, head, grid, cons_host, max(3, min(args.steps,
                                                          args.e2e_steps)))
    if rank != 0:
        if dist_on:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return
    roof = dict(r["roofline"])

    cpu = None
    if world == 1 and not args.no_cpu:
        v, sec, done = run_cpu_oracle(n, 1, warmup=args.cpu_warmup,
                                      min_seconds=args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": cpu_cores(), "kind": "port",
               "sample": f"C+OpenMP oracle (SN route, pinned bitwise to the "
                         f"reference), TGV {n}^3, {done} RK3 steps after "
                         f"{args.cpu_warmup} warm-up, {sec:.1f} s"}
    sizes = {}
    if world == 1 and args.sizes:
        sizes = stage_sweep(fd, lib, [int(x) for x in args.sizes.split(",")],
                            args.variants, flush, fp64_tf, hbm_peak)

    line = {
        "metric": METRIC, "value": r["value"], "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": r["ms_per_step"], "higher_is_better": True,
        "scaling": args.scaling if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: analytic Taylor-Green vortex initial state "
                "(BASELINE.json configs[4]; host numpy, the reference's "
                "expressions)",
        "config": config_dict(args, world),
        "headline_variant": head,
        "variants": results,
        "roofline": roof,
        "fp64_peak_tflops_measured": fp64_tf,
        "fp64_peak_sustained": fp64_sus,
        "cpu_baseline": cpu,
        "stage_sweep": sizes,
        "e2e": e2e,
        "gpu_launches": r["gpu_launches"],
        "comm": comm,
        "host_init_seconds": init_s,
        "clocks": {**clocks.summary(),
                   "window": f"{args.clock_window:.1f} s replay of each "
                             "variant's step right before its timed region"},
    }
    print(json.dumps(line), flush=True)
    if dist_on:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def main_reference(args):
    rank, world, _ = init_dist(args)
    if rank != 0:
        return
    npts = global_grid(args, world)
    # each "step" is one RK3 iteration of the configured grid; the timed
    # sample is at least --cpu-seconds of them (a 512^3 iteration is
    # ~8-10 s on 16 cores, so the sample is a bounded number of iterations).
    # A weak-scaled grid beyond 512^3 points (1024^3 on 8 GPUs: 86 GB of
    # host fields) is sampled on one rank's slab of it (the CPU rate per
    # point does not depend on the grid at these sizes).
    sample = npts
    if float(np.prod(npts)) > 512.0 ** 3:
        sample = (max(4, npts[0] // world), npts[1], npts[2])
    val, sec, iters = run_cpu_oracle(sample, 1, warmup=args.cpu_warmup,
                                     min_seconds=args.cpu_seconds)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "rk3_iterations_timed": iters,
        "ms_per_step": sec / iters * 1e3, "higher_is_better": True,
        "scaling": args.scaling if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: analytic Taylor-Green vortex initial state"
                if len(set(sample)) == 1 else
                "synthetic: smooth manufactured state of the slab grid's shape",
        "config": config_dict(args, world),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cpu_cores(),
                         "kind": "port",
                         "sample": f"C+OpenMP restatement of the reference "
                                   f"(SN route), grid {list(sample)}, {iters} "
                                   f"RK3 iterations after {args.cpu_warmup} "
                                   f"warm-up, {sec:.1f} s, rank 0 only"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def parse_args(argv):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--grid", dest="n", type=int, default=512,
                    help="cube edge n (the workload is TGV n^3)")
    ap.add_argument("--variants", default="BL,RA,SN,SS")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="minimum timed CPU work for the baseline sample")
    ap.add_argument("--cpu-warmup", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--clock-window", type=float, default=0.5,
                    help="seconds of untimed step replay sampled for clocks")
    ap.add_argument("--sizes", default="",
                    help="extra grid sizes for a single-stage sweep")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--loopback", action="store_true",
                    help="one GPU as a one-rank z-slab over NCCL: the "
                         "boundary/interior split and the axis-0 exchange "
                         "(rank 0 -> rank 0) run as on N GPUs")
    args = ap.parse_args(argv)
    args.variants = [v.strip().upper() for v in args.variants.split(",")]
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    return args


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse_args(argv)
    rc = self_launch(args, argv)
    if rc is not None:
        sys.exit(rc)
    if args.impl == "reference":
        main_reference(args)
    else:
        main_ours(args)


if __name__ == "__main__":
    main()
