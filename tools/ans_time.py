"""Device time of the GPU entropy decode (k_ans_table + k_ans_decode) of one coded frame packet,
for A/B experiments: python tools/ans_time.py [config] [reps]  (L2 flushed between reps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_04469_b200 as Q  # noqa: E402
from harness import synth  # noqa: E402
from paper_2412_04469_b200 import packet as wire  # noqa: E402
from paper_2412_04469_b200.runtime import EntropyPacket, Player  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "n3dv"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = synth.get_config(name)
sc, cams = synth.make_scene(cfg), synth.make_cameras(cfg)
pl = Player(sc.planes, sc.n, sc.deg, cams)
pkt = synth.make_packet(sc, 1)
streams = wire.ans_streams(pkt, Q.queen_entropy_encode)
ans_cap = [int(s.size) for s in streams]
buf = wire.pack_entropy(pkt, streams, frame=1, ans_cap=ans_cap)
hdr = wire.header_entropy(buf)
lay = wire.layout_entropy(sc.n_pad, cfg.deg, cfg.lat, pkt.k, ans_cap)
hdr.update(n=sc.n, n_pad=sc.n_pad, deg=cfg.deg, lat=tuple(cfg.lat), k_cap=pkt.k,
           **{k: lay[k] for k in ("dec_off", "lat_off", "idx_off", "val_off", "ans_off")})
ep = EntropyPacket(torch.from_numpy(buf).to(pl.dev), hdr)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=pl.dev)
ts = []
for r in range(reps + 3):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ep.decode(pl.ctx)
    e1.record()
    torch.cuda.synchronize()
    if r >= 3:
        ts.append(e0.elapsed_time(e1))
ok = np.array_equal(ep.latents[:, :sc.n].cpu().numpy(), pkt.latents[:, :sc.n])
print(f"{name}: entropy decode {1e3 * float(np.median(ts)):.1f} us (median of {reps}), "
      f"{sum(ans_cap)} coded bytes, latents match: {ok}")
