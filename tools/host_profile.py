"""cProfile of Player.step2's host side for a rank's view set: python tools/host_profile.py [config] [views]"""
import cProfile
import os
import pstats
import sys

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
pl.frame_lanes = 4
pkts = [synth.make_packet(sc, t) for t in (1, 2)]
streams = [wire.ans_streams(p, Q.queen_entropy_encode) for p in pkts]
cap = [max(s[c].size for s in streams) for c in range(5)]
kc = max(p.k for p in pkts)
bufs = [wire.pack_entropy(p, s, frame=t + 1, k_cap=kc, ans_cap=cap) for t, (p, s) in enumerate(zip(pkts, streams))]
hdr = wire.header_entropy(bufs[0])
eps = [EntropyPacket(torch.from_numpy(b).cuda(), hdr) for b in bufs]
outs = [torch.empty_like(pl.rgb) for _ in range(4)]
for t in range(20):
    pl.step2(eps[t & 1], out=outs[t & 3])
pl.sync_lanes()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for t in range(300):
    pl.step2(eps[t & 1], out=outs[t & 3])
pr.disable()
pl.sync_lanes()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
