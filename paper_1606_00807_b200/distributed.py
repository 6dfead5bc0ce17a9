"""Sharding of the sub-domains across ranks (one process per GPU).

Tiles are independent units with read-only inputs and disjoint outputs (driver.py:196-204,
PAPER.md:201), so the only exchange is moving the background in and the analysis out:
rank 0's background is broadcast, every rank analyses a contiguous block of tile block-rows
(tile id = bi*pc + bj, geometry.py:216) and the owned interior rows are all-gathered.  The
collectives go through torch.distributed (NCCL over NVLink on GPUs, gloo in the CPU tests);
no collective is fused into a compute kernel because none follows one.
"""

from __future__ import annotations

import numpy as np

from .plan import INTERIOR, INTERIOR_PTR


def block_row_cuts(pr: int, world: int) -> list[int]:
    """Balanced contiguous split of pr block rows over `world` ranks."""
    return [(pr * r) // world for r in range(world + 1)]


class TileShard:
    def __init__(self, plan, geometry, rank: int, world: int):
        self.plan, self.rank, self.world = plan, rank, world
        pr, pc = plan.size(7), plan.size(8)
        cuts = block_row_cuts(pr, world)
        self.tile_ranges = [(cuts[r] * pc, cuts[r + 1] * pc) for r in range(world)]
        ip, it = plan.get(INTERIOR_PTR), plan.get(INTERIOR)
        n2d, nf = geometry.n2d, geometry.nfields
        self.rows = []
        for t0, t1 in self.tile_ranges:
            own2d = np.sort(it[ip[t0]:ip[t1]])
            self.rows.append((np.arange(nf)[:, None] * n2d + own2d[None, :]).ravel().astype(np.int64))
        self.maxcount = max((r.size for r in self.rows), default=0)
        self._dev = None

    def apply(self) -> None:
        self.plan.set_tile_range(*self.tile_ranges[self.rank])

    def _tensors(self, like):
        import torch

        if self._dev is None or self._dev[0].device != like.device:
            own = torch.from_numpy(self.rows[self.rank]).to(like.device)
            sel = np.concatenate([r * self.maxcount + np.arange(self.rows[r].size) for r in range(self.world)])
            dst = np.concatenate(self.rows)
            self._dev = (own, torch.from_numpy(sel.astype(np.int64)).to(like.device),
                         torch.from_numpy(dst).to(like.device))
        return self._dev

    def broadcast_background(self, X) -> None:
        import torch.distributed as dist

        if self.world > 1:
            dist.broadcast(X, src=0)

    def gather_analysis(self, Xa) -> None:
        """All ranks end with every rank's owned interior rows in Xa."""
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return
        own, sel, dst = self._tensors(Xa)
        send = torch.zeros((self.maxcount, Xa.shape[1]), dtype=Xa.dtype, device=Xa.device)
        send[: own.numel()] = Xa.index_select(0, own)
        recv = torch.empty((self.world * self.maxcount, Xa.shape[1]), dtype=Xa.dtype, device=Xa.device)
        dist.all_gather_into_tensor(recv, send)
        Xa.index_copy_(0, dst, recv.index_select(0, sel))
