"""Multi-rank host logic on CPU (gloo, world_size 2): view sharding, frame-packet broadcast
(bit-identical on every rank), max-over-ranks timing reduction, and that the replicated
apply stays bit-identical across ranks (oracle stands in for the per-rank apply here:
the GPU kernels are deterministic, tests/test_gpu_parity.py checks them against it)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_04469_b200.dist import broadcast_packet, max_over_ranks, rank_views, view_balance


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_rank_views_partition():
    for V in (1, 13, 20, 46, 64):
        for R in (1, 2, 4, 8):
            parts = [rank_views(V, r, R) for r in range(R)]
            flat = sorted(v for p in parts for v in p)
            assert flat == list(range(V))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
    # SURVEY §8(e) ceilings
    assert view_balance(20, 8) == pytest.approx(20 / 8 / 3)
    assert view_balance(46, 4) == pytest.approx(46 / 4 / 12)
    assert view_balance(13, 2) == pytest.approx(13 / 2 / 7)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from harness import synth
        from paper_2412_04469_b200 import packet as wire
        cfg = synth.get_config("n3dv")
        sc = synth.make_scene(cfg, n=3001)  # every rank builds A_0 from the same seed
        k_cap = 400
        lay = wire.layout(sc.n_pad, cfg.deg, cfg.lat, k_cap)
        planes = sc.planes
        for t in (1, 2, 3):
            buf = torch.zeros(lay["total"], dtype=torch.uint8)
            if rank == 0:
                pkt = synth.make_packet(sc, t)
                buf.copy_(torch.from_numpy(wire.pack(pkt, frame=t, k_cap=k_cap)))
            broadcast_packet(buf)
            b = buf.numpy()
            h = wire.header(b)
            assert h["frame"] == t and h["k_cap"] == k_cap
            # rebuild the packet from the wire bytes and apply it (replicated apply)
            SL = sum(h["lat"])

            class P:
                pass
            p = P()
            p.n, p.n_pad, p.deg, p.lat = h["n"], h["n_pad"], h["deg"], h["lat"]
            p.latents = b[h["lat_off"]:h["lat_off"] + SL * h["n_pad"]].view(np.int8).reshape(SL, h["n_pad"]).copy()
            p.decoders = b[h["dec_off"]:h["dec_off"] + 4 * h["ndec"]].view(np.float32).copy()
            p.coo_idx = b[h["idx_off"]:h["idx_off"] + 4 * h["k"]].view(np.uint32).copy()
            p.coo_val = b[h["val_off"]:h["val_off"] + 12 * k_cap].view(np.float32).reshape(3, k_cap)[:, :h["k"]].copy()
            p.latents_f32 = None
            planes, st, _ = oracle.apply(planes, p)
            assert st == 0
        digest = torch.tensor([int(np.frombuffer(planes.tobytes(), np.uint64).sum() % (1 << 62))], dtype=torch.int64)
        allg = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allg, digest)
        mx = max_over_ranks(float(rank + 1))
        out[rank] = (int(allg[0]), int(allg[1]), mx, rank_views(20, rank, world))
    finally:
        dist.destroy_process_group()


def test_two_rank_packet_broadcast_and_replicated_apply():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert set(out.keys()) == {0, 1}
    d0, d1, mx, v0 = out[0]
    assert d0 == d1  # replicated SoA bit-identical on both ranks
    assert mx == 2.0 and out[1][2] == 2.0
    assert sorted(v0 + out[1][3]) == list(range(20))
