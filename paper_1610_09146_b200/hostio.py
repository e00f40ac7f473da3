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

Wavefront mode (round 2; one GPU, variants without work arrays -- SN, RA
-- on grids of at least 128 planes; `wave_chunks` defaults to min(32,
n0 / 16)): the step is cut into
`wave_chunks` axis-0 plane chunks and the copies overlap the step's own
compute as well.  Chunks are uploaded in ring order outward from chunk 0
(0, 1, K-1, 2, K-2, ...), each one's primitives formed as it lands, and every
stage of every chunk is launched (`fdns_stage_planes`, one compute stream)
as soon as the chunks it reads are current: stage 1 of chunk c needs the
uploads of c-1..c+1 (the padded ghost planes travel with the end chunks),
stages 2 and 3 the previous stage on c-1..c+1 around the ring (their axis-0
ghosts are the periodic images the other end's stage kernel wrote).  A
chunk is downloaded once its third stage (and its neighbours', for the
images) is done, and the next step's upload of a chunk waits only for that
download.  Both link directions then stay busy across steps and the ~28 ms
of compute of a 512^3 SN step hides under the copies: 162-173 -> 118 ms per
step at 512^3 (K = 32; a chunk is one 2-D copy-engine operation over the
five fields, `fdns_copy_rows`), against 113 ms for 5.5 GB each way at the
measured 97 GB/s two-way PCIe aggregate (`tools/pcie_bidir.py`,
`profiles/r02_e2e_wavefront.txt`).  Steps are
enqueued eagerly (CUDA events between the copy and compute streams; a
graph could not wait on the previous step's downloads).  Same kernels on
plane ranges, so the same bits.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .physics import ConservativeState, eval_primitives_fused
from .plan import ResidualEvaluator
from .timeloop import IterationState, RKScheme, _fused_iteration


UPLOAD_CTAS = 296


def wave_schedule(n0: int, h: int, K: int) -> dict:
    """The wavefront step's plan for n0 interior planes (halo h) in K chunks:
    interior and padded plane ranges per chunk (the end chunks carry the
    padded ghost planes), the upload order (ring distance from chunk 0),
    the compute sequence -- ("P", c) primitives of an uploaded chunk,
    ("S", stage, c) a stage of a chunk, each as soon as what it reads is
    current: stage 1 the uploads of c-1..c+1 (no wrap: the ghosts travel
    with the end chunks), stages 2-3 the previous stage on c-1..c+1 around
    the ring (their axis-0 ghosts are the images the far end wrote) -- and
    the stage-3 chunks each download waits for (itself and its ring
    neighbours, whose images land in its ghost planes)."""
    P0 = n0 + 2 * h
    a = [n0 * c // K for c in range(K + 1)]
    interior = [(a[c], a[c + 1]) for c in range(K)]
    padded = [(0 if c == 0 else a[c] + h, P0 if c == K - 1 else a[c + 1] + h)
              for c in range(K)]
    order = [0]
    for d in range(1, K // 2 + 1):
        for c in (d, K - d):
            if c not in order:
                order.append(c)
    ring = lambda c: {(c - 1) % K, c, (c + 1) % K}            # noqa: E731
    line = lambda c: {x for x in (c - 1, c, c + 1) if 0 <= x < K}  # noqa: E731
    seq, up, done = [], set(), {1: set(), 2: set(), 3: set()}
    for c in order:
        seq.append(("P", c))
        up.add(c)
        progress = True
        while progress:
            progress = False
            for sg in (1, 2, 3):
                for x in order:
                    if x in done[sg]:
                        continue
                    if (line(x) <= up) if sg == 1 else (ring(x) <= done[sg - 1]):
                        seq.append(("S", sg, x))
                        done[sg].add(x)
                        progress = True
    assert all(len(done[sg]) == K for sg in (1, 2, 3))
    return {"interior": interior, "padded": padded, "order": order, "seq": seq,
            "download_needs": {c: ring(c) for c in range(K)}}


class HostStepper:
    """Advance a host-resident conservative state on the GPU, one RK3
    iteration per `step`, with pipelined host<->device copies.

    The host buffer (`pinned_buffers(grid)`, padded fields in the reference
    layout) is owned by the stepper between `step()` and `wait()`; read or
    modify it only after `wait()` and a synchronize."""

    def __init__(self, state: ConservativeState, evaluator: ResidualEvaluator,
                 scheme: RKScheme, host, chunks: int = 5,
                 graphs: bool | None = None, upload: str = "ce",
                 wavefront: bool | None = None, wave_chunks: int | None = None):
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
        single = slab is None or not slab.distributed
        self.use_graphs = single if graphs is None else graphs
        self._graphs = None
        self._pending = False   # the last step's result is not downloaded yet
        n0 = state.grid.local_npoints[0]
        if wave_chunks is None:     # 16-plane chunks, at most 32 (e2e A/B at
            wave_chunks = min(32, n0 // 16)   # 512^3: K=8/16/32 -> 151/136/131 ms)
        can_wave = (single and evaluator.work is None and scheme.stages == 3
                    and upload == "ce" and wave_chunks >= 8 and n0 >= 8 * wave_chunks)
        if wavefront and not (single and evaluator.work is None and scheme.stages == 3
                              and upload == "ce" and wave_chunks >= 2
                              and n0 >= 8 * wave_chunks):
            raise ValueError("wavefront stepping needs one GPU, a variant without "
                             "work arrays and >= 8 planes per chunk")
        self.wavefront = can_wave if wavefront is None else bool(wavefront)
        if self.wavefront:
            self._wave_setup(wave_chunks)

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

    # -- wavefront mode ----------------------------------------------------
    def _wave_setup(self, K: int) -> None:
        g = self.state.grid
        sched = wave_schedule(g.local_npoints[0], g.halo, K)
        self._wK = K
        self._wi, self._wp = sched["interior"], sched["padded"]
        self._worder, self._wseq = sched["order"], sched["seq"]
        self._wdl_needs = sched["download_needs"]
        self._wev_dl = [None] * K       # previous step's download of each chunk
        self._lib_w = _lib.load()

    def _copy_chunk(self, X, host_fields, lo: int, hi: int, upload: bool) -> None:
        """Planes [lo, hi) of the five conservative fields, one copy-engine
        operation when the host side is one pinned block (five rows of a
        2-D copy, a field apart), else one copy per field."""
        if isinstance(self.host, torch.Tensor):
            plane = X.stride(1) * 8
            dev, hst = X[0, lo].data_ptr(), self.host[0, lo].data_ptr()
            dst, src = (dev, hst) if upload else (hst, dev)
            _lib.check(self._lib_w.fdns_copy_rows(
                dst, X.stride(0) * 8, src, self.host.stride(0) * 8,
                (hi - lo) * plane, 5, _lib.stream_handle()), "chunk copy")
            return
        for f in range(5):
            if upload:
                X[f, lo:hi].copy_(host_fields[f][lo:hi], non_blocking=True)
            else:
                host_fields[f][lo:hi].copy_(X[f, lo:hi], non_blocking=True)

    def _wave_step(self) -> None:
        K, X = self._wK, self.state.bundle
        Y, Z = self.ev.workspace()
        src, dst = (X, Y, Z), (Y, Z, X)
        main = torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(main)
        self.h2d.wait_event(start)
        self.d2h.wait_event(start)
        ev_up = {}
        for c in self._worder:                      # uploads, ring order
            if self._wev_dl[c] is not None:
                self.h2d.wait_event(self._wev_dl[c])
            lo, hi = self._wp[c]
            with torch.cuda.stream(self.h2d):
                self._copy_chunk(X, self._host_fields, lo, hi, upload=True)
            ev_up[c] = torch.cuda.Event()
            ev_up[c].record(self.h2d)
        problem, lib = self.ev.problem, self._lib_w
        ev_s3 = {}
        for item in self._wseq:                     # compute, one stream
            if item[0] == "P":
                c = item[1]
                main.wait_event(ev_up[c])
                lo, hi = self._wp[c]
                _lib.check(lib.fdns_primitives_planes(_lib.ptr(X), lo, hi, problem,
                                                      _lib.stream_handle()),
                           "chunk primitives")
                continue
            _, sg, c = item
            coef = self.scheme.alpha[sg - 1] * self.scheme.dt
            i_lo, i_hi = self._wi[c]
            self.ev.stage_planes(src[sg - 1], X, dst[sg - 1], coef, i_lo, i_hi, False)
            if sg == 3:
                ev_s3[c] = torch.cuda.Event()
                ev_s3[c].record(main)
        # downloads, in the order the chunks' neighbourhoods finish stage 3
        done3, queued = set(), set()
        for item in self._wseq:
            if item[0] != "S" or item[1] != 3:
                continue
            done3.add(item[2])
            for c in self._worder:
                if c in queued or not self._wdl_needs[c] <= done3:
                    continue
                queued.add(c)
                for x in self._wdl_needs[c]:
                    self.d2h.wait_event(ev_s3[x])
                lo, hi = self._wp[c]
                with torch.cuda.stream(self.d2h):
                    self._copy_chunk(X, self._host_fields, lo, hi, upload=False)
                e = torch.cuda.Event()
                e.record(self.d2h)
                self._wev_dl[c] = e
        self.it.state.prim_source = Z

    # -- public ------------------------------------------------------------
    def step(self) -> None:
        """Upload the host fields, advance one RK3 iteration; the previous
        step's result is downloaded first, chunk by chunk, as the uploads
        proceed (wavefront mode: this step's result is downloaded chunk by
        chunk as its stages complete)."""
        if self.wavefront:
            self._wave_step()
        else:
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
        if self.wavefront:
            torch.cuda.current_stream().wait_stream(self.d2h)
            return
        if self._pending:
            self._run("last")
            self._pending = False
