"""The z-slab NCCL path on one GPU: a one-rank NCCL group whose slab
exchanges its axis-0 ghost planes with itself (rank 0 -> rank 0, decomp.py
`Slab(loopback=True)`), so the boundary/interior split, the exchange on the
communication stream, the ghost-plane primitives and the all-reduce of the
diagnostics all execute as on N GPUs.  Every result must equal the plain
one-GPU run bitwise (KE/enstrophy: the same device reduction, then an
all-reduce over one rank).

Run as a subprocess by tests/test_gpu_nccl.py (a hung communicator cannot
then stall the GPU suite); prints one JSON line per case and exits 0 only if
all pass.
"""

import json
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1610_09146_b200 as fd  # noqa: E402
from paper_1610_09146_b200.diagnostics import make_collector  # noqa: E402
from paper_1610_09146_b200.hostio import HostStepper  # noqa: E402

TWO_PI = 2.0 * np.pi
C = fd.PhysicalConstants()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def host_cons(state):
    return state.grid.interior(state.bundle[:5]).cpu().numpy()


def case(variant, npts, steps, dt):
    g1 = fd.make_grid(npts, (TWO_PI,) * 3)
    ref = fd.taylor_green_init(g1, C)
    col1 = make_collector(g1, 1.0)
    rep1 = fd.run(ref, fd.RKScheme(dt=dt), fd.ResidualEvaluator(g1, C, variant),
                  steps, cadence=1, collect=col1)
    want = host_cons(ref)

    slab = fd.Slab.from_process_group(npts[0], loopback=True)
    g = fd.make_grid(npts, (TWO_PI,) * 3, slab=slab)
    st = fd.taylor_green_init(g, C)
    col = make_collector(g, 1.0)
    ev = fd.ResidualEvaluator(g, C, variant)
    assert ev.wrap_mask == 0b110   # axis 0 comes from the exchange
    rep = fd.run(st, fd.RKScheme(dt=dt), ev, steps, cadence=1, collect=col)
    got = host_cons(st)
    diag_eq = all(a == b for a, b in zip(rep1.records, rep.records))

    # host-buffer stepping on the slab (no CUDA graphs, no wavefront: the
    # exchange runs between the stages)
    st2 = fd.taylor_green_init(g, C)
    host = HostStepper.pinned_buffers(g)
    host.copy_(st2.bundle[:5].cpu())
    stepper = HostStepper(st2, fd.ResidualEvaluator(g, C, variant),
                          fd.RKScheme(dt=dt), host)
    for _ in range(steps):
        stepper.step()
    stepper.wait()
    torch.cuda.synchronize()
    hs = g.interior(host).numpy()
    return {"variant": variant, "npts": list(npts), "steps": steps,
            "fields_bitwise": bool(np.array_equal(got, want)),
            "diagnostics_equal": bool(diag_eq),
            "hoststepper_bitwise": bool(np.array_equal(hs, want)),
            "graphs": bool(stepper.use_graphs), "wavefront": bool(stepper.wavefront)}


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    ok = True
    cases = [(v, (24, 16, 20), 2, 2e-3) for v in fd.PLAN_NAMES]
    cases += [(v, (64, 64, 64), 3, 4e-3) for v in ("SN", "RA", "SS")]
    for v, npts, steps, dt in cases:
        r = case(v, npts, steps, dt)
        good = (r["fields_bitwise"] and r["diagnostics_equal"]
                and r["hoststepper_bitwise"] and not r["graphs"]
                and not r["wavefront"])
        ok &= good
        print(json.dumps({**r, "ok": good}), flush=True)
    print(json.dumps({"nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                      "backend": dist.get_backend(), "all_ok": ok}), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
