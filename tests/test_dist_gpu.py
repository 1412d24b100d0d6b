"""The multi-rank product path on the GPU (:255-257; §8(e)).

Two processes share cuda:0 and a gloo process group (host-side collectives: no kernel of one
rank waits on the other).  Each rank runs the product's dist.ShardedStream -- the class bench.py
drives under torchrun -- over its views v = rank mod 2: the one-time frame-0 SoA broadcast from
rank 0 (the other rank starts from zeros), then per frame the wire-packet broadcast into a
double-buffered slot, GPU entropy decode + apply, and the render, both as serial frames and as
two-lane pipelined steps.  Every image of every rank must equal the one-rank run's image of the
same view bit for bit, and every rank's final SoA must equal the one-rank SoA (replicated apply
is deterministic; PAPER.md:1384-1390 fixes what the packet carries)."""
import os
import socket
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

F = 4  # frames


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    import paper_2412_04469_b200 as Q
    from harness import synth
    from paper_2412_04469_b200 import packet as wire
    cfg = synth.get_config("n3dv", width=333, height=250, focal=280.0)
    sc = synth.make_scene(cfg, n=20003)
    cams = synth.make_cameras(cfg, 5)
    pkts = [synth.make_packet(sc, t) for t in range(1, F + 1)]  # packet t applies to frame t
    streams = [wire.ans_streams(p, Q.queen_entropy_encode) for p in pkts]
    cap = [max(st[c].size for st in streams) for c in range(5)]
    kc = max(p.k for p in pkts)
    bufs = [wire.pack_entropy(p, st, frame=t + 1, k_cap=kc, ans_cap=cap) for t, (p, st) in enumerate(zip(pkts, streams))]
    hdr = wire.header_entropy(bufs[0])
    return sc, cams, bufs, hdr


def _run(rank, world, out_path):
    from paper_2412_04469_b200.dist import ShardedStream
    sc, cams, bufs, hdr = _case()
    dev = torch.device("cuda:0")
    srcs = [torch.from_numpy(b).to(dev) for b in bufs] if rank == 0 else [None] * F
    planes0 = sc.planes if rank == 0 else np.zeros_like(sc.planes)
    res = {}
    # serial frames: frame t = A_0 + packets 1..t+1 ... (packet index t applied before render t)
    ss = ShardedStream(planes0, sc.n, sc.deg, cams, hdr, bufs[0].size, resident=srcs if world == 1 else None)
    ss.share_scene()
    ss.player.fit_capacity()
    serial = []
    for t in range(F):
        serial.append(ss.frame(t, srcs[t]).clone())
    torch.cuda.synchronize()
    assert ss.player.check_status()[0] == 0
    res["serial"] = np.stack([x.cpu().numpy() for x in serial])
    res["planes"] = ss.player.planes.cpu().numpy()
    # two-lane pipelined steps (the bench headline's step)
    ss2 = ShardedStream(planes0, sc.n, sc.deg, cams, hdr, bufs[0].size, resident=srcs if world == 1 else None,
                        keys_cap=ss.player.keys_cap)
    ss2.share_scene()
    ss2.apply_first(srcs[0])
    outs = [torch.empty_like(ss2.player.rgb) for _ in range(F)]
    for t in range(F):
        last = t + 1 >= F
        ss2.step2(t, None if last else srcs[t + 1], out=outs[t], last=last)
    ss2.player.sync_lanes()
    torch.cuda.synchronize()
    assert ss2.player.check_status()[0] == 0
    res["twolane"] = np.stack([x.cpu().numpy() for x in outs])
    res["planes2"] = ss2.player.planes.cpu().numpy()
    res["views"] = np.array(ss.views)
    np.savez(out_path, **res)


def _worker(rank, world, port, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _run(rank, world, os.path.join(outdir, f"rank{rank}.npz"))
    finally:
        dist.destroy_process_group()


def test_two_ranks_equal_one_rank_bit_for_bit():
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        _run(0, 1, os.path.join(d, "ref.npz"))
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        ref = np.load(os.path.join(d, "ref.npz"))
        seen = set()
        for r in range(2):
            got = np.load(os.path.join(d, f"rank{r}.npz"))
            views = [int(v) for v in got["views"]]
            assert views == [v for v in range(5) if v % 2 == r]
            seen.update(views)
            for key in ("serial", "twolane"):
                for k, v in enumerate(views):
                    a = got[key][:, k].view(np.uint32)
                    b = ref[key][:, v].view(np.uint32)
                    assert np.array_equal(a, b), (key, r, v)
            for key in ("planes", "planes2"):
                assert np.array_equal(got[key].view(np.uint32), ref[key].view(np.uint32)), (key, r)
        assert seen == set(range(5))
        # the pipelined steps equal the serial frames
        assert np.array_equal(ref["serial"].view(np.uint32), ref["twolane"].view(np.uint32))
