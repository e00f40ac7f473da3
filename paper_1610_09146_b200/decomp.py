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

    @staticmethod
    def partition(n0: int, rank: int, nranks: int, group=None) -> "Slab":
        base, rem = divmod(n0, nranks)
        local = base + (1 if rank < rem else 0)
        offset = rank * base + min(rank, rem)
        return Slab(rank, nranks, n0, offset, local, group)

    @staticmethod
    def from_process_group(n0: int, group=None) -> "Slab":
        return Slab.partition(n0, dist.get_rank(group), dist.get_world_size(group),
                              group)

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

    def exchange(self, bundle: torch.Tensor, h: int) -> None:
        """Fill the axis-0 ghost planes of every field of `bundle`
        (nf, n0+2h, P1, P2) from the neighbouring ranks, in place."""
        n = self.local_n0
        send_up = bundle[:, n:n + h].contiguous()      # top interior planes
        send_dn = bundle[:, h:2 * h].contiguous()      # bottom interior planes
        recv_lo = torch.empty_like(send_up)
        recv_hi = torch.empty_like(send_dn)
        ops = [dist.P2POp(dist.isend, send_up, self._peer(self.up), self.group),
               dist.P2POp(dist.isend, send_dn, self._peer(self.down), self.group),
               dist.P2POp(dist.irecv, recv_lo, self._peer(self.down), self.group),
               dist.P2POp(dist.irecv, recv_hi, self._peer(self.up), self.group)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        bundle[:, 0:h].copy_(recv_lo)
        bundle[:, n + h:n + 2 * h].copy_(recv_hi)

    def allreduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t
