"""How many of the K (tile, Gaussian) entries of the rect duplication have an alpha >= 1/255 ellipse
that misses every pixel centre of the tile (same test as the blend's touches())?  Experiment tool."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from harness import synth  # noqa: E402
from paper_2412_04469_b200.runtime import Player  # noqa: E402
from paper_2412_04469_b200.stages import Stages  # noqa: E402

cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "n3dv")
sc, cams = synth.make_scene(cfg), synth.make_cameras(cfg)
pl = Player(sc.planes, sc.n, sc.deg, cams)
pl.fit_capacity()
bc = cams[pl.batches[0][0]:pl.batches[0][1]]
stg = Stages(pl.planes.cpu().numpy(), sc.n, sc.deg, bc, keys_cap=pl.keys_cap, device=0)
stg.project()
torch.cuda.synchronize()
rect = stg.rect.reshape(-1, 4).long()
rec = stg.rec.reshape(-1, 12)
nt = stg.tiles.reshape(-1).long()
vis = nt > 0
rect, rec, nt = rect[vis], rec[vis], nt[vis]
w = rect[:, 2] - rect[:, 0] + 1
K = int(nt.sum())
tot_keep = 0
B = 1 << 20
for s in range(0, rect.shape[0], B):
    r, q, n, ww = rect[s:s + B], rec[s:s + B], nt[s:s + B], w[s:s + B]
    pid = torch.repeat_interleave(torch.arange(r.shape[0], device=r.device), n)
    start = torch.cumsum(n, 0) - n
    j = torch.arange(pid.shape[0], device=r.device) - start[pid]
    tx = r[pid, 0] + j % ww[pid]
    ty = r[pid, 1] + j // ww[pid]
    u, v, hx, hy, A, Bc, C, T2 = [q[pid, i] for i in range(8)]
    x0, x1 = (16 * tx).float(), (16 * tx + 15).float()
    y0, y1 = (16 * ty).float(), (16 * ty + 15).float()
    inside = (u >= x0) & (u <= x1) & (v >= y0) & (v <= y1)
    iA, iC = (-0.5 * Bc) / A, (-0.5 * Bc) / C
    dxl, dxh, dyl, dyh = u - x1, u - x0, v - y1, v - y0
    best = torch.full_like(u, -float("inf"))
    for dy in (dyh, dyl):
        dx = torch.minimum(torch.maximum(iA * dy, dxl), dxh)
        best = torch.maximum(best, A * dx * dx + C * dy * dy + Bc * dx * dy)
    for ex in (dxh, dxl):
        ey = torch.minimum(torch.maximum(iC * ex, dyl), dyh)
        best = torch.maximum(best, A * ex * ex + C * ey * ey + Bc * ex * ey)
    S = A.abs() * hx * hx + Bc.abs() * hx * hy + C.abs() * hy * hy
    keep = inside | (best >= T2 - (1e-5 * S + 1e-6))
    tot_keep += int(keep.sum())
print(f"pairs {int(vis.sum())} K {K} kept {tot_keep} ({100 * tot_keep / K:.1f}%)")
