"""One N3DV-shaped backward (rasterize_backward over a frame's views) for profiling."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_04469_b200 as Q  # noqa: E402
from harness import synth  # noqa: E402
from paper_2412_04469_b200.stages import Stages  # noqa: E402

cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "n3dv")
sc = synth.make_scene(cfg)
cams = synth.make_cameras(cfg)
st = Stages(sc.planes, sc.n, sc.deg, cams, keys_cap=8 * sc.n * len(cams)).project().bin_sort()
g = torch.randn((len(cams), 3, cfg.height, cfg.width), device="cuda")
grec = torch.empty((len(cams), st.n_pad, 9), device="cuda")
for _ in range(2):
    Q.queen_rasterize_backward(st.ctx, st.proj, st.bins, cams, g, grec)
torch.cuda.synchronize()
print("status", st.ctx.check_status())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    Q.queen_rasterize_backward(st.ctx, st.proj, st.bins, cams, g, grec)
e1.record()
torch.cuda.synchronize()
print("rasterize_backward ms", e0.elapsed_time(e1) / 3)
