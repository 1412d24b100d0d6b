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


def world_info(group=None) -> tuple[int, int]:
    """(rank, world) of the initialised process group, or (0, 1)."""
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


class ShardedStream:
    """One rank of the view-sharded streaming renderer.

    The rank renders views v = rank mod N (rank_views) of every frame from a replicated
    Gaussian set.  Frame packets arrive on rank 0 (wire buffers, packet.py layout) and are
    broadcast into one of two packet slots on every rank (the double buffer lets packet t+1
    land while frame t still reads slot t % 2); every rank then entropy-decodes + applies the
    packet with the same deterministic kernels, so the SoAs stay bit-identical with no other
    exchange.  With one rank the packets are used in place (no collective).

    hdr: the stream-static packet fields (n, n_pad, deg, lat, k_cap, section offsets; plus
    ans_off for entropy-coded packets); nbytes: the fixed wire-buffer size."""

    def __init__(self, planes, n: int, deg: int, cams_all, hdr: dict, nbytes: int, *, entropy: bool = True,
                 device: int = 0, views_per_batch: int | None = None, group=None, resident=None, views=None,
                 **player_kw):
        from .runtime import EntropyPacket, Player, wire_packet
        self.rank, self.world = world_info(group)
        self.group = group
        self.views = list(views) if views is not None else rank_views(len(cams_all), self.rank, self.world)
        cams = [cams_all[v] for v in self.views]
        self.dev = torch.device(f"cuda:{device}")
        self.player = Player(planes, n, deg, cams, device=device, views_per_batch=views_per_batch, **player_kw)
        mk = (lambda b: EntropyPacket(b, hdr)) if entropy else (lambda b: wire_packet(b, hdr))
        if self.world == 1 and resident is not None:
            self.slots = list(resident)  # one rank: the resident packets are used in place
        else:
            self.slots = [torch.zeros(int(nbytes), dtype=torch.uint8, device=self.dev) for _ in range(2)]
        self.packets = [mk(s) for s in self.slots]
        self.resident = resident

    def share_scene(self):
        """One-time broadcast of rank 0's frame-0 Gaussian set A_0 (the SoA planes) to every rank
        (SURVEY.md §8(e)); the other ranks may start from any buffer of the right shape."""
        if self.world > 1:
            dist.broadcast(self.player.planes, 0, group=self.group)

    def receive(self, t: int, src: torch.Tensor | None = None):
        """Packet of frame t on this rank: rank 0 copies `src` (packet t, resident on its GPU) into
        slot t % 2 and broadcasts the slot (N > 1); returns the slot's queen packet.  With one rank
        and resident packets, packet t is resident[t % len(resident)] itself."""
        if self.world == 1 and self.resident is not None:
            return self.packets[t % len(self.packets)]
        slot = t % 2
        if self.rank == 0 and src is not None:
            self.slots[slot].copy_(src)
        broadcast_packet(self.slots[slot], 0, self.group)
        return self.packets[slot]

    def frame(self, t: int, src: torch.Tensor | None = None, out=None):
        """Serial frame step: receive packet t, decode + apply it, render this rank's views."""
        self.player.apply(self.receive(t, src))
        return self.player.render(out=out)

    def step2(self, t: int, src_next: torch.Tensor | None = None, out=None, rendered=None, consumed=None,
              last: bool = False):
        """Two-lane pipelined step (runtime.Player.step2): render frame t (already applied) and
        receive + decode + apply packet t+1 under its blend (none when `last`).  Call
        apply_first(src0) before the first step."""
        nxt = None if last else self.receive(t + 1, src_next)
        return self.player.step2(nxt, out=out, rendered=rendered, consumed=consumed)

    def apply_first(self, src0: torch.Tensor | None = None):
        """Frame 0 of a pipelined run: receive and apply packet 0."""
        self.player.apply(self.receive(0, src0))
