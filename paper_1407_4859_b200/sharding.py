"""Multi-GPU sharding of the remap.

Record i of the output depends only on record i of the input, so the record array
is split by contiguous index range (adha_shard_range, reading Q10) and every rank
remaps its own shard as its own layout instance: no halo, no data-path
collective.  torch.distributed is used only for a barrier and one all_reduce(MAX)
of the elapsed time (works on NCCL with CUDA tensors and on gloo with CPU tensors).
"""
from __future__ import annotations

from typing import Tuple

from . import shard_range


def shard_for(n_cfg: int, world: int, rank: int, scaling: str) -> Tuple[int, int, int]:
    """(n_total, lo, hi): weak scaling keeps n_cfg records per rank, strong splits n_cfg."""
    if scaling not in ("weak", "strong"):
        raise ValueError(scaling)
    n_total = n_cfg * world if scaling == "weak" else n_cfg
    lo, hi = shard_range(n_total, world, rank)
    return n_total, lo, hi


def max_over_ranks(value: float, device=None) -> float:
    """all_reduce(MAX) of one float across the default process group (identity if none)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    if dist.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_gbs(n_total: int, record_bytes: int, remaps_per_step: int, steps: int, ms_max: float) -> float:
    """Whole-job remap GB/s: (read + write) payload bytes of all ranks / max-over-ranks time."""
    return 2.0 * n_total * record_bytes * remaps_per_step * steps / (ms_max * 1e-3) / 1e9
