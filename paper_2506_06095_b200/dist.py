"""Multi-GPU plumbing for the hot path: one process per GPU, torch.distributed.

The attention path has no exchange: units are (b, h, query-row-block) for a masked MHA sweep and
whole sequences for layers, partitioned contiguously over ranks; every rank rebuilds the formats
from the mask descriptor locally (deterministic, microseconds), so nothing is broadcast. The
only collectives are the timing reduction (max over ranks of device time) and the optional
end-to-end gather of layer outputs (NCCL all-gather over NVLink on GPUs, gloo on CPU tests).
"""
from __future__ import annotations

from typing import Tuple

import torch
import torch.distributed as dist


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced [begin, end) share of `total` units for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def mha_units(bs: int, heads: int, seq_len: int, block_m: int = 128) -> int:
    """(b, h, row-block) work units of one masked-MHA call (cfg1 at 128-row blocks: 48)."""
    return bs * heads * ((seq_len + block_m - 1) // block_m)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the timing rule: the slowest rank defines the step)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local: torch.Tensor) -> torch.Tensor:
    """Concatenate every rank's (rows, cols) output along rows (rank order): the end-to-end gather."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    parts = [torch.empty_like(local) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, local.contiguous())
    return torch.cat(parts, 0)
