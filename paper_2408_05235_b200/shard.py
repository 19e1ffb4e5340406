"""Multi-GPU plumbing: instance sharding and the single decision gather.

Instances are independent (they share only the read-only model, the frequency list and the TBT
SLO), so each rank decides a contiguous shard with no data-path collective.  The only collective
is one all-gather of the per-instance (level, status) rows after K3 -- NCCL over NVLink on GPUs,
gloo in the CPU tests.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, equal-count (+-1) instance range [i0, i1) of ``rank``."""
    return n_total * rank // world, n_total * (rank + 1) // world


def weak_range(n_per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: every rank decides ``n_per_rank`` new instances of the same generator."""
    return n_per_rank * rank, n_per_rank * (rank + 1)


def gather_decisions(dec: torch.Tensor, counts: list[int]) -> torch.Tensor:
    """All-gather the [2, I_r] (level, status) int32 rows of every rank into [2, sum I_r].

    Shards may differ in size by one (strong scaling); each rank pads to the largest count, one
    all_gather_into_tensor moves everything, and the padding is dropped."""
    world = dist.get_world_size()
    mx = max(counts)
    buf = dec
    if dec.shape[1] != mx:
        buf = torch.zeros((2, mx), dtype=dec.dtype, device=dec.device)
        buf[:, :dec.shape[1]] = dec
    out = torch.empty((world * 2, mx), dtype=dec.dtype, device=dec.device)
    dist.all_gather_into_tensor(out, buf.contiguous())
    out = out.view(world, 2, mx)
    return torch.cat([out[r, :, :counts[r]] for r in range(world)], dim=1)
