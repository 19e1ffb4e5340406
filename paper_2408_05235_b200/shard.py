"""Multi-GPU plumbing: instance sharding and the single decision gather.

Instances are independent (they share only the read-only model, the frequency list and the TBT
SLO), so each rank decides a contiguous shard with no data-path collective.  The only collective
is one all-gather of the per-instance (level, status) rows after K3 -- NCCL over NVLink on GPUs,
gloo in the CPU tests.  bench.py and the tests use the same `DecisionGather`.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, equal-count (+-1) instance range [i0, i1) of ``rank``."""
    return n_total * rank // world, n_total * (rank + 1) // world


def shard_by_engine(tp, rank: int, world: int):
    """Strong scaling, grouped by engine size: the global indices of ``rank``'s instances.

    The instances are ordered by (tp, index) and cut into ``world`` contiguous equal-count (+-1)
    chunks.  The model is evaluated once per distinct cell (rank_tp, rank_B, rank_KV) a rank's
    instances touch, and tp is one coordinate of the cell, so a rank that holds one or two engine
    sizes evaluates a quarter or a half of the cells a mixed shard touches -- the K2 work that
    does not shrink with N under index-contiguous sharding.  The decisions are the
    same; only who decides which instance changes."""
    import numpy as np
    order = np.argsort(np.asarray(tp), kind="stable")
    i0, i1 = shard_range(len(order), rank, world)
    return order[i0:i1]


def shard_counts(n_total: int, world: int) -> list[int]:
    return [b - a for a, b in (shard_range(n_total, r, world) for r in range(world))]


def weak_range(n_per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: every rank decides ``n_per_rank`` new instances of the same generator."""
    return n_per_rank * rank, n_per_rank * (rank + 1)


class DecisionGather:
    """All-gather of every rank's [2, I_r] int32 (level, status) rows into [2, sum I_r].

    Shards may differ in size by one (strong scaling with a world size that does not divide the
    instance count): every rank writes its rows into a preallocated [2, max I_r] send buffer
    (the padding column stays zero), one ``all_gather_into_tensor`` moves [world * 2, max I_r],
    and `result()` drops the padding.  Buffers are allocated once, so the per-step gather is one
    collective (plus one device copy when the caller's rows are not the send buffer itself).

    ``host_staging=True`` (gloo on one GPU, TP_BENCH_DIST_TEST): the collective runs on host
    copies of the buffers."""

    def __init__(self, counts: list[int], device, host_staging: bool = False):
        self.counts = list(counts)
        self.world = len(counts)
        self.mx = max(max(counts), 1)
        self.host = host_staging
        dev = torch.device("cpu") if host_staging else torch.device(device)
        self.send = torch.zeros((2, self.mx), dtype=torch.int32, device=device)
        self.out = torch.empty((self.world * 2, self.mx), dtype=torch.int32, device=device)
        if host_staging:
            self._hs = torch.zeros((2, self.mx), dtype=torch.int32, device=dev)
            self._ho = torch.empty((self.world * 2, self.mx), dtype=torch.int32, device=dev)

    def rows(self) -> torch.Tensor:
        """The send buffer's [2, I_r] view: kernels may write level / status straight into it."""
        return self.send[:, :self.counts[dist.get_rank()]]

    def gather(self, dec: torch.Tensor | None = None) -> torch.Tensor:
        """Gather ``dec`` (default: the send buffer's rows, already written in place)."""
        if dec is not None and dec.data_ptr() != self.send.data_ptr():
            self.send[:, :dec.shape[1]].copy_(dec)
        if self.host:
            self._hs.copy_(self.send)
            dist.all_gather_into_tensor(self._ho, self._hs)
            self.out.copy_(self._ho)
        else:
            dist.all_gather_into_tensor(self.out, self.send)
        return self.out

    def result(self) -> torch.Tensor:
        """[2, sum I_r] in global instance order (padding dropped)."""
        o = self.out.view(self.world, 2, self.mx)
        return torch.cat([o[r, :, :self.counts[r]] for r in range(self.world)], dim=1)


def gather_decisions(dec: torch.Tensor, counts: list[int]) -> torch.Tensor:
    """One-shot form of `DecisionGather` (the same buffers and collective)."""
    g = DecisionGather(counts, dec.device)
    g.gather(dec)
    return g.result()
