"""z-slab domain decomposition and the periodic 2-plane halo exchange.

The reference runs in one process with an in-place periodic copy
(mesh.py:118-139); the paper decomposed the domain with OPS/MPI
(PAPER.md:247-249).  Here axis 0 (the slowest, so every plane is one
contiguous run of (n1+2h)(n2+2h) doubles per field) is split into contiguous
slabs, one per rank/GPU.  Axes 1 and 2 stay local-periodic (fdns_halo_wrap);
per RK stage each rank sends its top h interior planes to rank+1 (they become
that rank's low ghosts) and its bottom h planes to rank-1, all fields in one
batched send/recv group over NCCL (NVLink/NVSwitch) -- or gloo for the CPU
tests.  With two ranks both neighbours are the same peer; the posting order
below keeps the matching unambiguous.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class Slab:
    """This rank's share of axis 0."""

    rank: int
    nranks: int
    n0: int          # global points along axis 0
    offset0: int     # first global index owned
    local_n0: int
    group: object = None
    loopback: bool = False   # one rank exchanging with itself over the backend

    @property
    def distributed(self) -> bool:
        """Axis 0 goes through the exchange (several ranks, or a one-rank
        loopback slab: the axis-0 ghosts then travel rank 0 -> rank 0 over
        the communication backend, which runs the NCCL path on one GPU)."""
        return self.nranks > 1 or self.loopback

    @staticmethod
    def partition(n0: int, rank: int, nranks: int, group=None,
                  loopback: bool = False) -> "Slab":
        base, rem = divmod(n0, nranks)
        local = base + (1 if rank < rem else 0)
        offset = rank * base + min(rank, rem)
        return Slab(rank, nranks, n0, offset, local, group, loopback)

    @staticmethod
    def from_process_group(n0: int, group=None, loopback: bool = False) -> "Slab":
        return Slab.partition(n0, dist.get_rank(group), dist.get_world_size(group),
                              group, loopback)

    def validate(self, n0: int, halo: int) -> None:
        from .mesh import ConfigurationError
        if n0 != self.n0:
            raise ConfigurationError("slab built for a different axis-0 size")
        if self.local_n0 < halo:
            raise ConfigurationError(
                f"rank {self.rank} owns {self.local_n0} planes; the halo "
                f"exchange needs at least {halo}")

    @property
    def up(self) -> int:
        return (self.rank + 1) % self.nranks

    @property
    def down(self) -> int:
        return (self.rank - 1) % self.nranks

    def _peer(self, r: int) -> int:
        return r if self.group is None else dist.get_global_rank(self.group, r)

    def exchange(self, bundle: torch.Tensor, h: int, nf: int | None = None) -> None:
        """Fill the axis-0 ghost planes of the first `nf` fields (default all)
        of `bundle` (nf, n0+2h, P1, P2) from the neighbouring ranks, in
        place.  Each field's h planes are one contiguous run, so they are
        sent from and received into the bundle itself: no pack or unpack
        copies, 4 * nf point-to-point operations in one group."""
        n = self.local_n0
        nf = bundle.shape[0] if nf is None else nf
        up, dn = self._peer(self.up), self._peer(self.down)
        ops = []
        for f in range(nf):
            fb = bundle[f]
            ops += [dist.P2POp(dist.isend, fb[n:n + h], up, self.group),       # top planes
                    dist.P2POp(dist.isend, fb[h:2 * h], dn, self.group),       # bottom planes
                    dist.P2POp(dist.irecv, fb[0:h], dn, self.group),           # low ghosts
                    dist.P2POp(dist.irecv, fb[n + h:n + 2 * h], up, self.group)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()

    def exchange_state(self, bundle: torch.Tensor, h: int, problem) -> None:
        """The per-stage exchange of a state bundle: only the five
        conservative fields travel (5 x 2h padded planes per neighbour,
        SURVEY 8e); u, p, T of the received ghost planes are then formed on
        this rank by the primitives kernel -- the same expressions the
        sender's stage kernel evaluated, so the same bits."""
        self.exchange(bundle, h, nf=5)
        ghost_primitives(bundle, self.local_n0, h, problem)

    def allreduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t


def ghost_primitives(bundle: torch.Tensor, n: int, h: int, problem) -> None:
    """Primitives (physics.py:185-202) of the 2h axis-0 ghost planes of a
    state bundle whose conservative ghosts were just received."""
    from . import _lib
    lib = _lib.load()
    for lo in (0, n + h):
        _lib.check(lib.fdns_primitives_planes(_lib.ptr(bundle), lo, lo + h,
                                              problem, _lib.stream_handle()),
                   "ghost-plane primitives")
