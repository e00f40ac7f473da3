"""Host-buffer stepping for reference-style callers (parity mode).

A caller of the reference keeps its state in host numpy arrays
(`Field.data`, mesh.py:88-115) and advances it in place
(timeloop.py:88-94).  `HostStepper` offers that contract on the device path:
each `step(host)` uploads the five conservative fields from (pinned) host
memory, runs one fused RK3 iteration on the GPU, and writes the new fields
back to the same host buffers.

The round trip is pipelined per field over two copy streams: the upload of
field f waits only for the download of field f from the previous step, so
downloads and uploads of different fields overlap on the full-duplex PCIe
link and separate copy engines, and the first kernel waits only for the last
upload.  Results are bitwise those of `advance_iteration`.
"""

from __future__ import annotations

import numpy as np
import torch

from .mesh import halo_exchange_bundle
from .physics import ConservativeState, eval_primitives_fused
from .plan import ResidualEvaluator
from .timeloop import IterationState, RKScheme, _fused_iteration


class HostStepper:
    """Advance a host-resident conservative state on the GPU, one RK3
    iteration per `step`, with pipelined host<->device copies."""

    def __init__(self, state: ConservativeState, evaluator: ResidualEvaluator,
                 scheme: RKScheme):
        self.state = state
        self.ev = evaluator
        self.scheme = scheme
        self.it = IterationState(state, saved=False)
        self.h2d = torch.cuda.Stream()
        self.d2h = torch.cuda.Stream()
        self.down_done = [torch.cuda.Event() for _ in range(5)]
        self.up_done = [torch.cuda.Event() for _ in range(5)]
        self.step_done = torch.cuda.Event()
        self._first = True

    @staticmethod
    def pinned_buffers(grid) -> torch.Tensor:
        """(5, padded...) pinned host buffers for the conservative fields."""
        return torch.empty((5,) + grid.shape, dtype=torch.float64).pin_memory()

    def step(self, host: torch.Tensor) -> None:
        """host: (5, padded...) pinned float64 tensor, updated in place
        (halos included, as the reference leaves them after
        timeloop.py:85)."""
        dev = self.state.bundle
        main = torch.cuda.current_stream()
        # uploads: field f after the previous step's download of field f
        for f in range(5):
            if not self._first:
                self.h2d.wait_event(self.down_done[f])
            else:
                self.h2d.wait_stream(main)
            with torch.cuda.stream(self.h2d):
                dev[f].copy_(host[f], non_blocking=True)
                self.up_done[f].record(self.h2d)
        for f in range(5):
            main.wait_event(self.up_done[f])
        # one fused RK3 iteration (primitives refreshed from the uploads)
        eval_primitives_fused(self.state, self.ev.constants)
        _fused_iteration(self.it, self.scheme, self.ev)
        self.it.time += self.scheme.dt
        self.it.iteration += 1
        self.step_done.record(main)
        # downloads, field by field, as soon as the iteration is done
        self.d2h.wait_event(self.step_done)
        for f in range(5):
            with torch.cuda.stream(self.d2h):
                host[f].copy_(dev[f], non_blocking=True)
                self.down_done[f].record(self.d2h)
        self._first = False

    def wait(self) -> None:
        """Make the current stream wait for the last step's downloads (the
        host buffers are complete once that stream is synchronised)."""
        torch.cuda.current_stream().wait_stream(self.d2h)
