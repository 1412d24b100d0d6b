"""Multi-GPU plumbing: views sharded over ranks, Gaussian set replicated, one broadcast
of the frame packet per frame.

The only exchange step of the path is the frame packet (decoders,
integer latents, COO positions), broadcast from rank 0.  Every rank then applies it
with the same deterministic kernels (so the replicated SoAs stay bit-identical without
further communication) and renders its own views v = rank mod N.  Images stay on the
rendering rank.  torch.distributed (NCCL on GPUs, gloo in the CPU tests) is plumbing.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def rank_views(n_views: int, rank: int, world: int) -> list[int]:
    """Round-robin view partition: every view exactly once, counts differ by at most one."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return [v for v in range(n_views) if v % world == rank]


def view_balance(n_views: int, world: int) -> float:
    """Scaling ceiling from view imbalance: ideal views per rank / max views per rank."""
    return (n_views / world) / max(len(rank_views(n_views, r, world)) for r in range(world))


def broadcast_packet(buf: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """In-place broadcast of a contiguous uint8 wire packet (packet.py layout) from `src`.
    On GPUs this is one ncclBroadcast over NVLink/NVSwitch on the current stream."""
    if not buf.is_contiguous() or buf.dtype != torch.uint8:
        raise ValueError("packet buffer must be a contiguous uint8 tensor")
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(buf, src=src, group=group)
    return buf


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Device-timed values are reduced with MAX over ranks (the job finishes with the slowest)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
