"""Frame throughput of the eager frame loops: serial (apply, render), pipelined (Player.step:
decode/apply of t+1 under the blend of t) and two-lane (Player.step2: also frame t+1's binning
under the blend of t), over K frames timed as one interval (no L2 flush: a frame's working set
is several times the L2).  python tools/lanes_probe.py [config] [frames]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2412_04469_b200 as Q  # noqa: E402
from harness import synth  # noqa: E402
from paper_2412_04469_b200 import packet as wire  # noqa: E402
from paper_2412_04469_b200.runtime import EntropyPacket, Player  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "n3dv"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cfg = synth.get_config(name)
sc, cams = synth.make_scene(cfg), synth.make_cameras(cfg)
P = 4
pkts = [synth.make_packet(sc, t + 1) for t in range(P)]
streams = [wire.ans_streams(p, Q.queen_entropy_encode) for p in pkts]
cap = [max(int(st[c].size) for st in streams) + 4096 for c in range(5)]
kc = max(p.k for p in pkts)
bufs = [wire.pack_entropy(p, st, frame=t + 1, k_cap=kc, ans_cap=cap) for t, (p, st) in enumerate(zip(pkts, streams))]
hdr = wire.header_entropy(bufs[0])
eps = [EntropyPacket(torch.from_numpy(b).cuda(), hdr) for b in bufs]
pl = Player(sc.planes, sc.n, sc.deg, cams)
pl.fit_capacity()
A0 = torch.from_numpy(sc.planes).cuda()
outs = [torch.empty_like(pl.rgb) for _ in range(2)]
main = torch.cuda.current_stream()


def timed(fn):
    pl.planes.copy_(A0)
    pl.apply(eps[0])
    for t in range(5):
        fn(t)
    pl.sync_lanes()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(5, 5 + K):
        fn(t)
    pl.sync_lanes()
    e1.record()
    torch.cuda.synchronize()
    return K / (e0.elapsed_time(e1) / 1e3)


def serial(t):
    pl.render(out=outs[t & 1])
    pl.apply(eps[(t + 1) % P])


def piped(t):
    pl.step(eps[(t + 1) % P], out=outs[t & 1])


def lanes2(t):
    pl.step2(eps[(t + 1) % P], out=outs[t & 1])


for label, fn in [("serial", serial), ("pipelined", piped), ("two-lane", lanes2), ("serial again", serial)]:
    print(f"{name} {label:12s} {timed(fn):8.1f} frames/s")
# the two-lane images equal the serial ones
ref, got = [], []
pl.planes.copy_(A0)
pl.apply(eps[0])
for t in range(4):
    serial(t)
    ref.append(outs[t & 1].clone())
pl.planes.copy_(A0)
pl.apply(eps[0])
for t in range(4):
    ev = torch.cuda.Event()
    pl.step2(eps[(t + 1) % P], out=outs[t & 1], rendered=ev)
    main.wait_event(ev)
    got.append(outs[t & 1].clone())
pl.sync_lanes()
torch.cuda.synchronize()
print("two-lane images bit-identical:", all(torch.equal(a, b) for a, b in zip(ref, got)), "status", pl.check_status())
