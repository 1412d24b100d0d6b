"""Host cost of the frame step's pieces (no GPU sync inside the loops): queen_render_views (the C
call: ~25 kernel launches), the entropy decode + apply calls, and the whole Player.step2, for a
rank's view set.  python tools/host_probe.py [config] [views]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_04469_b200 as Q  # noqa: E402
from harness import synth  # noqa: E402
from paper_2412_04469_b200 import packet as wire  # noqa: E402
from paper_2412_04469_b200.runtime import EntropyPacket, Player  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "meetroom"
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = synth.get_config(name)
sc, cams = synth.make_scene(cfg), synth.make_cameras(cfg)[:nv]
pl = Player(sc.planes, sc.n, sc.deg, cams)
pl.fit_capacity()
pkts = [synth.make_packet(sc, t) for t in (1, 2)]
streams = [wire.ans_streams(p, Q.queen_entropy_encode) for p in pkts]
cap = [max(s[c].size for s in streams) for c in range(5)]
kc = max(p.k for p in pkts)
bufs = [wire.pack_entropy(p, s, frame=t + 1, k_cap=kc, ans_cap=cap) for t, (p, s) in enumerate(zip(pkts, streams))]
hdr = wire.header_entropy(bufs[0])
eps = [EntropyPacket(torch.from_numpy(b).cuda(), hdr) for b in bufs]
R = 200


def host(fn, reps=R):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return (t1 - t0) * 1e6 / reps, (t2 - t0) * 1e6 / reps


print(name, nv, "views")
print("render (C call)      host %.1f us, wall %.1f us" % host(lambda: pl.render()))
print("entropy decode       host %.1f us, wall %.1f us" % host(lambda: eps[0].decode(pl.ctx)))
print("apply                host %.1f us, wall %.1f us" % host(lambda: pl.apply(eps[0])))
out = [torch.empty_like(pl.rgb) for _ in range(4)]
pl.frame_lanes = 4
k = [0]


def s2():
    pl.step2(eps[k[0] & 1], out=out[k[0] & 3])
    k[0] += 1


print("step2 (4 lanes)      host %.1f us, wall %.1f us" % host(s2))
pl.sync_lanes()
ev = torch.cuda.Event()
print("torch event record   host %.1f us" % host(lambda: ev.record())[0])
s = torch.cuda.Stream()
print("stream.wait_stream   host %.1f us" % host(lambda: s.wait_stream(torch.cuda.current_stream()))[0])
