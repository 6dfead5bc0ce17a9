"""Sharding of the sub-domains across ranks (one process per GPU).

Tiles are independent units with read-only inputs and disjoint outputs (driver.py:196-204,
PAPER.md:201), so the only exchange is moving the background in and the analysis out
(north_star: "NCCL over NVLink is used only to scatter the background ensemble and gather the
analysis").  Every rank owns a contiguous block of tile block-rows (tile id = bi*pc + bj,
geometry.py:216).  The root scatters to each rank exactly the state rows its tiles read -- its
latitude band plus zeta halo rows, for every field -- and the rows of the perturbed
observations that fall inside them (grouped point-to-point sends); the owned interior rows are
all-gathered afterwards.  The collectives go through torch.distributed (NCCL over NVLink on
GPUs, gloo in the CPU tests); no collective is fused into a compute kernel because none
follows one.  All exchange buffers are allocated once and reused every cycle.
"""

from __future__ import annotations

import numpy as np

from .plan import INTERIOR, INTERIOR_PTR, LOCAL_ORDER, TILE_PTR


def block_row_cuts(pr: int, world: int) -> list[int]:
    """Balanced contiguous split of pr block rows over `world` ranks."""
    return [(pr * r) // world for r in range(world + 1)]


class TileShard:
    def __init__(self, plan, geometry, rank: int, world: int, obs_indices=None):
        self.plan, self.rank, self.world = plan, rank, world
        pr, pc = plan.size(7), plan.size(8)
        cuts = block_row_cuts(pr, world)
        self.tile_ranges = [(cuts[r] * pc, cuts[r + 1] * pc) for r in range(world)]
        ip, it = plan.get(INTERIOR_PTR), plan.get(INTERIOR)
        tp, lo = plan.get(TILE_PTR), plan.get(LOCAL_ORDER)
        n2d, nf = getattr(geometry, "nfield", geometry.n2d), geometry.nfields   # rows of one field's block (all levels)
        fields = np.arange(nf, dtype=np.int64)[:, None] * n2d
        self.rows, self.need = [], []          # owned interior rows / rows read (interiors + halos), all fields
        for t0, t1 in self.tile_ranges:
            own2d = np.sort(it[ip[t0]:ip[t1]])
            self.rows.append((fields + own2d[None, :]).ravel().astype(np.int64))
            need2d = np.unique(lo[tp[t0]:tp[t1]])
            self.need.append((fields + need2d[None, :]).ravel().astype(np.int64))
        self.maxcount = max((r.size for r in self.rows), default=0)
        self.need_obs = None
        if obs_indices is not None:
            self.set_observations(obs_indices)
        self._dev = None
        self._bufs = {}

    def set_observations(self, obs_indices) -> None:
        """Rows of Ys / r_diag each rank needs: the observations inside the rows it reads."""
        obs = np.asarray(obs_indices, dtype=np.int64)
        self.need_obs = []
        for need in self.need:
            pos = np.searchsorted(need, obs)
            hit = (pos < need.size) & (need[np.minimum(pos, max(need.size - 1, 0))] == obs) if need.size else np.zeros(obs.size, bool)
            self.need_obs.append(np.flatnonzero(hit).astype(np.int64))
        self._bufs = {}

    def apply(self) -> None:
        self.plan.set_tile_range(*self.tile_ranges[self.rank])

    def memory_fraction(self) -> float:
        """Share of the local rows (hence of the T / D / band workspace) this rank owns."""
        tp = self.plan.get(TILE_PTR)
        t0, t1 = self.tile_ranges[self.rank]
        return float(tp[t1] - tp[t0]) / float(max(tp[-1], 1))

    # -- device-side index tensors and reusable buffers --------------------------------
    def _tensors(self, like):
        import torch

        if self._dev is None or self._dev[0].device != like.device:
            own = torch.from_numpy(self.rows[self.rank]).to(like.device)
            sel = np.concatenate([r * self.maxcount + np.arange(self.rows[r].size) for r in range(self.world)])
            dst = np.concatenate(self.rows)
            self._dev = (own, torch.from_numpy(sel.astype(np.int64)).to(like.device),
                         torch.from_numpy(dst).to(like.device))
        return self._dev

    def _buffer(self, key, shape, like):
        import torch

        b = self._bufs.get(key)
        if b is None or tuple(b.shape) != tuple(shape) or b.device != like.device or b.dtype != like.dtype:
            b = torch.empty(shape, dtype=like.dtype, device=like.device)
            self._bufs[key] = b
        return b

    def _index(self, key, rows, like):
        import torch

        t = self._bufs.get(key)
        if t is None or t.device != like.device:
            t = torch.from_numpy(np.ascontiguousarray(rows)).to(like.device)
            self._bufs[key] = t
        return t

    # -- exchanges -----------------------------------------------------------------------
    def _scatter_rows(self, A, lists, tag, root):
        """Root sends A[lists[r]] to every other rank r, which stores them at the same rows of its A."""
        import torch.distributed as dist

        if self.world == 1:
            return
        ops, keep = [], []
        if self.rank == root:
            for r in range(self.world):
                if r == root or lists[r].size == 0:
                    continue
                buf = self._buffer((tag, "send", r), (lists[r].size,) + tuple(A.shape[1:]), A)
                buf.copy_(A.index_select(0, self._index((tag, "idx", r), lists[r], A)))
                ops.append(dist.P2POp(dist.isend, buf, r))
                keep.append(buf)
        elif lists[self.rank].size:
            buf = self._buffer((tag, "recv"), (lists[self.rank].size,) + tuple(A.shape[1:]), A)
            ops.append(dist.P2POp(dist.irecv, buf, root))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if self.rank != root and lists[self.rank].size:
            A.index_copy_(0, self._index((tag, "idx", self.rank), lists[self.rank], A), self._bufs[(tag, "recv")])

    def scatter_background(self, X, Ys=None, root: int = 0) -> None:
        """Root's background rows (and perturbed-observation rows) go to the ranks that read them; everything else in
        the other ranks' X / Ys is left untouched (never read by their tiles)."""
        self._scatter_rows(X, self.need, "x", root)
        if Ys is not None and self.need_obs is not None:
            self._scatter_rows(Ys, self.need_obs, "ys", root)

    def broadcast_background(self, X) -> None:
        """Whole-ensemble broadcast (kept for comparison; scatter_background moves only what is read)."""
        import torch.distributed as dist

        if self.world > 1:
            dist.broadcast(X, src=0)

    def gather_analysis(self, Xa) -> None:
        """All ranks end with every rank's owned interior rows in Xa."""
        import torch.distributed as dist

        if self.world == 1:
            return
        own, sel, dst = self._tensors(Xa)
        send = self._buffer(("gather", "send"), (self.maxcount, Xa.shape[1]), Xa)
        recv = self._buffer(("gather", "recv"), (self.world * self.maxcount, Xa.shape[1]), Xa)
        send[: own.numel()] = Xa.index_select(0, own)
        dist.all_gather_into_tensor(recv, send)
        Xa.index_copy_(0, dst, recv.index_select(0, sel))
