"""Blend work counts (queen_blend_counts) of the first view batch: evaluated / composited pairs.
python tools/blend_counts.py [config]   (QUEEN_LIB_PATH=exp/cw.so: counts restricted to warp lists)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_04469_b200 as Q  # noqa: E402
from harness import synth  # noqa: E402
from paper_2412_04469_b200.runtime import Player  # noqa: E402
from paper_2412_04469_b200.stages import Stages  # noqa: E402

cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "n3dv")
sc, cams = synth.make_scene(cfg), synth.make_cameras(cfg)
pl = Player(sc.planes, sc.n, sc.deg, cams)
pl.fit_capacity()
bc = cams[pl.batches[0][0]:pl.batches[0][1]]
stg = Stages(pl.planes.cpu().numpy(), sc.n, sc.deg, bc, keys_cap=pl.keys_cap, device=0)
stg.project().bin_sort()
e = torch.zeros(len(bc), dtype=torch.int64, device=pl.dev)
c = torch.zeros(len(bc), dtype=torch.int64, device=pl.dev)
Q.queen_blend_counts(stg.ctx, stg.proj, stg.bins, bc, e, c)
print("views", len(bc), "K", stg.bins_np()["K"], "evaluated", int(e.sum()), "composited", int(c.sum()))
