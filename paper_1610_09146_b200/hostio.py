"""Host-buffer stepping for reference-style callers (parity mode).

A caller of the reference keeps its state in host numpy arrays
(`Field.data`, mesh.py:88-115) and advances it in place
(timeloop.py:88-94).  `HostStepper` offers that contract on the device path:
each `step()` uploads the five conservative fields from a pinned host
buffer, runs one fused RK3 iteration on the GPU, and the new fields land in
the same host buffer (complete once the stream `wait()` returns on is
synchronised).

Copies are chunked (the contiguous five-field block split into `chunks`
pieces) and pipelined over both PCIe directions (copy engines; an SM
copy kernel reading the pinned host buffer directly, `upload="sm"`,
`fdns_copy_sm`, measured slower inside this schedule: 1.52e9 vs 1.70e9
pt-stage/s at 64^3, tools/e2e_ab.py): the upload of a chunk waits only for
the download of that chunk of the previous step's result, so the previous
result's download and the next input's upload overlap chunk by chunk on the
full-duplex link.  To keep that overlap across the step boundary, the
download of step n is issued at the start of step n+1 (or by `wait()`).  On
one GPU the three copy/compute programs (first step, steady step, final
download) are captured once as CUDA graphs, so a step costs one graph
launch of host time.  Results are bitwise those of `advance_iteration`.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .physics import ConservativeState, eval_primitives_fused
from .plan import ResidualEvaluator
from .timeloop import IterationState, RKScheme, _fused_iteration


UPLOAD_CTAS = 296


class HostStepper:
    """Advance a host-resident conservative state on the GPU, one RK3
    iteration per `step`, with pipelined host<->device copies.

    The host buffer (`pinned_buffers(grid)`, padded fields in the reference
    layout) is owned by the stepper between `step()` and `wait()`; read or
    modify it only after `wait()` and a synchronize."""

    def __init__(self, state: ConservativeState, evaluator: ResidualEvaluator,
                 scheme: RKScheme, host, chunks: int = 5,
                 graphs: bool | None = None, upload: str = "ce"):
        """`host`: a pinned float64 (5, padded...) tensor
        (`pinned_buffers`), or the reference's own five padded numpy arrays
        (rho, rhou0, rhou1, rhou2, rhoE as `Field.data` holds them), which
        are page-locked in place (cudaHostRegister) until `close()`."""
        shape = tuple(state.bundle.shape[1:])
        self._registered = []
        if isinstance(host, torch.Tensor):
            if not host.is_pinned() or host.dtype != torch.float64 or \
                    tuple(host.shape) != (5,) + shape:
                raise ValueError("host must be a pinned float64 (5, padded...) "
                                 "tensor (HostStepper.pinned_buffers)")
            fields = [host[f] for f in range(5)]
        else:
            arrays = list(host)
            if len(arrays) != 5 or any(
                    not isinstance(a, np.ndarray) or a.dtype != np.float64 or
                    a.shape != shape or not a.flags.c_contiguous for a in arrays):
                raise ValueError("host must be five C-contiguous float64 padded "
                                 f"arrays of shape {shape}")
            cudart = torch.cuda.cudart()
            for a in arrays:
                err = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
                if int(err) != 0:
                    self.close()
                    raise _lib.FdnsError(f"cudaHostRegister failed ({int(err)})")
                self._registered.append(a)
            fields = [torch.from_numpy(a) for a in arrays]
        self.state = state
        self.ev = evaluator
        self.scheme = scheme
        self.host = host
        self._host_fields = fields
        self.it = IterationState(state, saved=False)
        self.h2d = torch.cuda.Stream()
        self.d2h = torch.cuda.Stream()
        # copied as `chunks` contiguous pieces: of the five-field block when
        # the host side is one block too, else of each field
        if isinstance(host, torch.Tensor):
            sides = [(state.bundle[:5].reshape(-1), host.reshape(-1), chunks)]
        else:
            per = max(1, chunks // 5)
            sides = [(state.bundle[f].reshape(-1), fields[f].reshape(-1), per)
                     for f in range(5)]
        self._pairs = []
        for d, h, k in sides:
            n = d.numel()
            cuts = [(n * c // k) & ~1 for c in range(k)] + [n]   # 16-byte cuts
            self._pairs += [(d[a:b], h[a:b]) for a, b in zip(cuts, cuts[1:]) if b > a]
        self._lib = _lib.load()
        if upload not in ("sm", "ce"):
            raise ValueError("upload must be 'sm' or 'ce'")
        self.upload = upload
        slab = state.grid.slab
        single = slab is None or slab.nranks == 1
        self.use_graphs = single if graphs is None else graphs
        self._graphs = None
        self._pending = False   # the last step's result is not downloaded yet

    @staticmethod
    def pinned_buffers(grid) -> torch.Tensor:
        """(5, padded...) pinned host buffers for the conservative fields."""
        return torch.empty((5,) + grid.shape, dtype=torch.float64).pin_memory()

    # -- the three programs ------------------------------------------------
    def _roundtrip(self, download: bool, upload: bool) -> None:
        main = torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(main)
        self.h2d.wait_event(start)
        self.d2h.wait_event(start)
        for d, h in self._pairs:
            if download:
                with torch.cuda.stream(self.d2h):
                    h.copy_(d, non_blocking=True)
                if upload:
                    done = torch.cuda.Event()
                    done.record(self.d2h)
                    self.h2d.wait_event(done)
            if upload:
                # "sm": every SM reads the pinned host chunk directly
                with torch.cuda.stream(self.h2d):
                    if self.upload == "sm":
                        _lib.check(self._lib.fdns_copy_sm(
                            d.data_ptr(), h.data_ptr(), d.numel() * 8,
                            UPLOAD_CTAS, _lib.stream_handle()), "host upload")
                    else:
                        d.copy_(h, non_blocking=True)
        main.wait_stream(self.h2d)
        main.wait_stream(self.d2h)

    def _program(self, which: str) -> None:
        if which != "last":
            self._roundtrip(download=(which == "mid"), upload=True)
            # one fused RK3 iteration, primitives refreshed from the uploads
            eval_primitives_fused(self.state, self.ev.constants)
            _fused_iteration(self.it, self.scheme, self.ev)
        else:
            self._roundtrip(download=True, upload=False)

    def _run(self, which: str) -> None:
        if not self.use_graphs:
            self._program(which)
            return
        if self._graphs is None:
            self._capture()
        self._graphs[which].replay()

    def _capture(self) -> None:
        # warm every program once eagerly on a side stream (first-use setup
        # of the library and allocator), on a scratch copy of the state
        saved = self.state.bundle.clone()
        host_saved = [h.clone() for h in self._host_fields]
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for which in ("first", "mid", "last"):
                self._program(which)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graphs = {}
        for which in ("first", "mid", "last"):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._program(which)
            graphs[which] = g
        torch.cuda.synchronize()
        self.state.bundle.copy_(saved)
        for h, hs in zip(self._host_fields, host_saved):
            h.copy_(hs)
        torch.cuda.synchronize()
        self._graphs = graphs

    # -- public ------------------------------------------------------------
    def step(self) -> None:
        """Upload the host fields, advance one RK3 iteration; the previous
        step's result is downloaded first, chunk by chunk, as the uploads
        proceed."""
        self._run("mid" if self._pending else "first")
        self._pending = True
        self.it.time += self.scheme.dt
        self.it.iteration += 1

    def close(self) -> None:
        """Release the page-locking of registered numpy arrays (after the
        last `wait()` and a synchronize)."""
        if self._registered:
            torch.cuda.synchronize()
            cudart = torch.cuda.cudart()
            for a in self._registered:
                cudart.cudaHostUnregister(a.ctypes.data)
            self._registered = []

    def wait(self) -> None:
        """Download the last step's result into the host buffer; the buffer
        is complete once the current stream is synchronised."""
        if self._pending:
            self._run("last")
            self._pending = False
