"""Where does the end-to-end frame time go?  Streams N3DV-shaped entropy-coded frames through
runtime.Player like bench.py's e2e (pinned H2D of the packet, decode + apply + render, D2H of the
u8 images, copies on their own streams) with parts switched off:
    python tools/e2e_probe.py [config] [frames]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2412_04469_b200 as Q  # noqa: E402
from harness import synth  # noqa: E402
from paper_2412_04469_b200 import packet as wire  # noqa: E402
from paper_2412_04469_b200.runtime import EntropyPacket, Player  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "n3dv"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cfg = synth.get_config(name)
sc, cams = synth.make_scene(cfg), synth.make_cameras(cfg)
P = 4
pkts = [synth.make_packet(sc, t + 1) for t in range(P)]
streams = [wire.ans_streams(p, Q.queen_entropy_encode) for p in pkts]
ans_cap = [max(int(st[c].size) for st in streams) + 4096 for c in range(5)]
k_cap = max(p.k for p in pkts)
bufs = [wire.pack_entropy(p, st, frame=t + 1, k_cap=k_cap, ans_cap=ans_cap) for t, (p, st) in enumerate(zip(pkts, streams))]
used = [wire.header_entropy(b)["used"] for b in bufs]
lay = wire.layout_entropy(sc.n_pad, cfg.deg, cfg.lat, k_cap, ans_cap)
hdr = dict(n=sc.n, n_pad=sc.n_pad, deg=cfg.deg, lat=tuple(cfg.lat), k_cap=k_cap, ans_off=lay["ans_off"],
           **{k: lay[k] for k in ("dec_off", "lat_off", "idx_off", "val_off")})
pl = Player(sc.planes, sc.n, sc.deg, cams)
pl.fit_capacity()
dev = pl.dev
pin = [torch.from_numpy(b).pin_memory() for b in bufs]
recv = [torch.zeros(lay["total"], dtype=torch.uint8, device=dev) for _ in range(2)]
dps = [EntropyPacket(r, hdr) for r in recv]
out_dev = [torch.empty(pl.rgb.shape, dtype=torch.uint8, device=dev) for _ in range(2)]
out_host = [torch.empty(pl.rgb.shape, dtype=torch.uint8).pin_memory() for _ in range(2)]
main = torch.cuda.current_stream(dev)
s_h2d, s_d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)


def run(n, h2d=True, d2h=True, compute=True):
    ev = lambda: torch.cuda.Event()  # noqa: E731
    e_h, e_a, e_r, e_d = [ev() for _ in range(n)], [ev() for _ in range(n)], [ev() for _ in range(n)], [ev() for _ in range(n)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(main)
    s_h2d.wait_stream(main)
    s_d2h.wait_stream(main)
    for q in range(n):
        slot = q % 2
        with torch.cuda.stream(s_h2d):
            if q >= 2:
                s_h2d.wait_event(e_a[q - 2])
            if h2d:
                recv[slot][:used[q % P]].copy_(pin[q % P][:used[q % P]], non_blocking=True)
            e_h[q].record(s_h2d)
        main.wait_event(e_h[q])
        if compute:
            pl.apply(dps[slot])
        e_a[q].record(main)
        if q >= 2:
            main.wait_event(e_d[q - 2])
        if compute:
            pl.render(out=out_dev[slot], rgb8=True)
        e_r[q].record(main)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(e_r[q])
            if d2h:
                out_host[slot].copy_(out_dev[slot], non_blocking=True)
            e_d[q].record(s_d2h)
    main.wait_event(e_d[n - 1])
    t1.record(main)
    torch.cuda.synchronize()
    return n / (t0.elapsed_time(t1) / 1e3)


run(5)
for label, kw in [("full", {}), ("no D2H", {"d2h": False}), ("no H2D", {"h2d": False}), ("compute only", {"h2d": False, "d2h": False}),
                  ("copies only", {"compute": False}), ("D2H only", {"compute": False, "h2d": False}), ("full again", {})]:
    print(f"{name} {label:14s} {run(frames, **kw):8.1f} frames/s")
