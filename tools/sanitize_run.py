"""Small frames through every product kernel, for compute-sanitizer:
    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_run.py [tiny|small]
tiny: BASELINE configs[0] (1 view 64x64); small: a 3-view 333x250 N3DV-shaped frame.  Runs the
entropy decode, decode + apply, two-lane pipelined steps (project, binning, blend on two
contexts), the masked render, densify and the backward pass; checks the sticky status."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_04469_b200 as Q  # noqa: E402
from harness import synth  # noqa: E402
from paper_2412_04469_b200 import packet as wire  # noqa: E402
from paper_2412_04469_b200.runtime import EntropyPacket, Player, device_packet  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "tiny"
if which == "tiny":
    cfg = synth.get_config("tiny")
    sc = synth.make_scene(cfg)
    cams = synth.make_cameras(cfg)
else:
    cfg = synth.get_config("n3dv", width=333, height=250, focal=280.0)
    sc = synth.make_scene(cfg, n=20003)
    cams = synth.make_cameras(cfg, 3)
F = 3
pkts = [synth.make_packet(sc, t) for t in range(1, F + 1)]
streams = [wire.ans_streams(p, Q.queen_entropy_encode) for p in pkts]
cap = [max(st[c].size for st in streams) for c in range(5)]
kc = max(p.k for p in pkts)
bufs = [wire.pack_entropy(p, st, frame=t + 1, k_cap=kc, ans_cap=cap) for t, (p, st) in enumerate(zip(pkts, streams))]
hdr = wire.header_entropy(bufs[0])
eps = [EntropyPacket(torch.from_numpy(b).cuda(), hdr) for b in bufs]
pl = Player(sc.planes, sc.n, sc.deg, cams, with_T=True)
pl.fit_capacity()
pl.apply(eps[0])
outs = [torch.empty_like(pl.rgb) for _ in range(F)]
for t in range(F):
    pl.step2(eps[t + 1] if t + 1 < F else None, out=outs[t])
pl.sync_lanes()
h = torch.empty(pl.rgb.shape, dtype=torch.float16, device="cuda")
pl.render(out=h)
u8 = torch.empty(pl.rgb.shape, dtype=torch.uint8, device="cuda")
pl.render(out=u8, rgb8=True)
idx = torch.from_numpy(np.ascontiguousarray(pkts[0].coo_idx, np.uint32)).cuda()
pl.render_mask(idx)
# trainer-state packet (gates + f32 latents) through decode_residuals and apply
dp = device_packet(pkts[0], pl.dev, gates=True, f32_latents=True)
pl.apply(dp)
# backward of the first batch
from paper_2412_04469_b200.stages import Stages  # noqa: E402
stg = Stages(pl.planes.cpu().numpy(), sc.n, sc.deg, cams, keys_cap=pl.keys_cap)
stg.project().bin_sort().rasterize()
gimg = torch.randn((len(cams), 3, cfg.height, cfg.width), dtype=torch.float32, device="cuda")
grec = torch.empty((len(cams), stg.n_pad, 9), dtype=torch.float32, device="cuda")
gpl = torch.empty((sc.planes.shape[0], stg.n_pad), dtype=torch.float32, device="cuda")
Q.queen_rasterize_backward(stg.ctx, stg.proj, stg.bins, cams, gimg, grec)
Q.queen_project_backward(stg.ctx, stg.scene, cams, grec, gpl)
torch.cuda.synchronize()
st, info = pl.check_status()
st2, _ = stg.ctx.check_status()
print(f"sanitize_run {which}: status {st} / {st2}")
sys.exit(0 if st >= 0 and st2 >= 0 else 1)
