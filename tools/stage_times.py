"""Per-stage device milliseconds of one N3DV-shaped frame (libqueen's stage profiler), for
quick A/B experiments: python tools/stage_times.py [config] [frames] [--flush].
--flush writes 512 MB between frames (L2 cold at every frame start, as in bench.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from harness import synth
from paper_2412_04469_b200.runtime import Player, device_packet

flags = {a for a in sys.argv[1:] if a.startswith("--")}
args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if len(args) > 0 else "n3dv"
frames = int(args[1]) if len(args) > 1 else 10
cfg = synth.get_config(name)
sc = synth.make_scene(cfg)
cams = synth.make_cameras(cfg)
vpb = {"stress": 8}.get(name)
pl = Player(sc.planes, sc.n, sc.deg, cams, views_per_batch=vpb)
pkt = device_packet(synth.make_packet(sc, 1), pl.dev)
pl.fit_capacity()
for _ in range(3):
    pl.frame(pkt)
torch.cuda.synchronize()
pl.profile(True)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=pl.dev) if "--flush" in flags else None
for _ in range(frames):
    if flush is not None:
        flush.fill_(1)
    pl.frame(pkt)
prof = pl.profile_read()
print(name, {k: round(ms / frames, 4) for k, (ms, n) in prof.items()}, "total", round(sum(ms for ms, _ in prof.values()) / frames, 4))
