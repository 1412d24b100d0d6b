"""Blend tail estimate: list-schedule the tiles (cost = entries in the tile's list) on
148 SMs x S slots in grid order vs longest-first, report makespan / ideal.  Experiment tool."""
import heapq
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

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
r = stg.ranges.cpu().numpy().astype(np.int64)
cost = (r[:, 1] - r[:, 0]).astype(np.float64) + 8.0  # + fixed per-CTA overhead
print("tiles", len(cost), "mean", cost.mean(), "max", cost.max(), "p99", np.percentile(cost, 99))


def sim(order, slots):
    h = [0.0] * slots
    for c in order:
        t = heapq.heappop(h)
        heapq.heappush(h, t + c)
    return max(h)


for S in (8, 16, 32):
    slots = 148 * S
    ideal = cost.sum() / slots
    a = sim(cost, slots)
    b = sim(np.sort(cost)[::-1], slots)
    print(f"slots/SM {S}: grid order {a / ideal:.3f} x ideal, longest-first {b / ideal:.3f} x ideal")
