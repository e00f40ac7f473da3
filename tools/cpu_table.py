"""CPU baseline table on the host this runs on (the GPU box's cores, for
profiles/): the C + OpenMP restatement of the reference path (SN route,
bitwise equal to the reference) at 64^3 / 128^3 / 256^3 on 1 thread and on
all host threads, and the numpy restatement (the reference's BL route:
every derivative array materialised, single-threaded numpy) at 64^3.
Units: grid-point x RK-stage updates/s, TGV initial state.  Test/measurement
infrastructure only (it executes oracle/).

    python tools/cpu_table.py [--seconds 3]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from oracle import c_oracle, numpy_oracle as npo

DT = {64: 3.385e-3, 128: 1.69e-3, 256: 8.5e-4}


def time_c(n, threads, seconds):
    c = npo.Consts()
    F = npo.taylor_green(n, c)
    c_oracle.run(F, c, DT[n], 1, nthreads=threads)
    done, el = 0, 0.0
    while done == 0 or el < seconds:
        t0 = time.perf_counter()
        c_oracle.run(F, c, DT[n], 1, nthreads=threads)
        el += time.perf_counter() - t0
        done += 1
    return n ** 3 * 3 * done / el, done, el


def time_numpy_bl(n, seconds):
    c = npo.Consts()
    F = npo.taylor_green(n, c)
    w = npo.grid_weights((n,) * 3)
    npo.rk_step(F, 2, w, c, DT[n])
    done, el = 0, 0.0
    while done == 0 or el < seconds:
        t0 = time.perf_counter()
        npo.rk_step(F, 2, w, c, DT[n])
        el += time.perf_counter() - t0
        done += 1
    return n ** 3 * 3 * done / el, done, el


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    a = ap.parse_args()
    allc = c_oracle.default_threads()
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo")
                 if l.startswith("model name")][0]
    except Exception:
        model = "?"
    print(f"host: {model}; {allc} threads available (sched_getaffinity)")
    print(f"{'path':<34} {'n':>4} {'threads':>7} {'pt-stage/s':>11} {'RK3 steps':>9} {'s':>6}")
    for n in (64, 128, 256):
        for th in (1, allc):
            v, d, el = time_c(n, th, a.seconds)
            print(f"{'C+OpenMP oracle (SN route)':<34} {n:4d} {th:7d} {v:11.3e} {d:9d} {el:6.1f}")
    v, d, el = time_numpy_bl(64, a.seconds)
    print(f"{'numpy oracle (BL route)':<34} {64:4d} {1:7d} {v:11.3e} {d:9d} {el:6.1f}")


if __name__ == "__main__":
    main()
