"""Explicit-buffer stage runner over the C-ABI (queen_project -> queen_bin_sort -> queen_rasterize).

Used by the parity tests and by bench.py's evidence pass (key counts, blend work
counters).  Marshalling only: every step runs in libqueen's kernels."""
from __future__ import annotations

import numpy as np
import torch

from . import (Context, bins_struct, gaussians_struct, proj_struct, queen_bin_sort, queen_project,
               queen_rasterize)


def to_np(t):
    return t.detach().cpu().numpy()


class Stages:
    """Explicit project / bin_sort / rasterize buffers for one batch of views."""

    def __init__(self, planes: np.ndarray, n: int, deg: int, cams, keys_cap: int | None = None, device=0):
        self.dev = torch.device(f"cuda:{device}")
        self.ctx = Context(device)
        self.planes_t = torch.from_numpy(np.ascontiguousarray(planes, np.float32)).to(self.dev)
        self.n, self.deg, self.cams = n, deg, list(cams)
        self.n_pad = planes.shape[1]
        V = len(cams)
        self.V = V
        self.W, self.H = cams[0].width, cams[0].height
        self.T = ((self.W + 15) // 16) * ((self.H + 15) // 16)
        if keys_cap is None:
            keys_cap = max(1024, 64 * n * V)
        self.keys_cap = min(int(keys_cap), (1 << 30) - 1)
        self.ctx.set_workspace(self.n_pad, V, self.W, self.H, self.keys_cap)
        d = self.dev
        self.rec = torch.zeros((V, self.n_pad, 12), dtype=torch.float32, device=d)
        self.depth = torch.zeros((V, self.n_pad), dtype=torch.int32, device=d)
        self.tiles = torch.zeros((V, self.n_pad), dtype=torch.int32, device=d)
        self.rect = torch.zeros((V, self.n_pad, 4), dtype=torch.int16, device=d)
        self.keys = torch.zeros(self.keys_cap, dtype=torch.int32, device=d)
        self.keys_alt = torch.zeros_like(self.keys)
        self.vals = torch.zeros(self.keys_cap, dtype=torch.int32, device=d)
        self.vals_alt = torch.zeros_like(self.vals)
        self.ranges = torch.zeros((V * self.T, 2), dtype=torch.int32, device=d)
        self.K = torch.zeros(4, dtype=torch.int32, device=d)
        self.rgb = torch.zeros((V, 3, self.H, self.W), dtype=torch.float32, device=d)
        self.Tout = torch.zeros((V, self.H, self.W), dtype=torch.float32, device=d)
        self.proj = proj_struct(self.rec, self.depth, self.tiles, self.rect)
        self.bins = bins_struct(self.keys, self.keys_alt, self.vals, self.vals_alt, self.ranges, self.K)
        self.scene = gaussians_struct(self.planes_t, n, deg)

    def project(self):
        queen_project(self.ctx, self.scene, self.cams, self.proj)
        return self

    def bin_sort(self):
        queen_bin_sort(self.ctx, self.proj, self.cams, self.bins)
        return self

    def rasterize(self, bg=(0.0, 0.0, 0.0)):
        queen_rasterize(self.ctx, self.proj, self.bins, self.cams, self.rgb, self.Tout, bg)
        return self

    def run(self, bg=(0.0, 0.0, 0.0)):
        return self.project().bin_sort().rasterize(bg)

    def proj_np(self):
        torch.cuda.synchronize()
        return dict(rec=to_np(self.rec), depth=to_np(self.depth).view(np.uint32), tiles=to_np(self.tiles).view(np.uint32),
                    rect=to_np(self.rect))

    def bins_np(self):
        """K, M, P (pieces), the sorted Gaussian indices, the ranges, and each entry's gt (rebuilt
        from the ranges: after queen_bin_sort the key buffers are scratch)."""
        torch.cuda.synchronize()
        K = int(to_np(self.K)[0])
        vs = self.vals_alt if self.bins.sorted_in_alt else self.vals
        ranges = to_np(self.ranges).view(np.uint32)
        lens = (ranges[:, 1].astype(np.int64) - ranges[:, 0].astype(np.int64))
        keys = np.repeat(np.arange(ranges.shape[0], dtype=np.uint32), lens)
        return dict(K=K, M=int(to_np(self.K)[1]), P=int(to_np(self.K)[3]), keys=keys, vals=to_np(vs[:K]).view(np.uint32),
                    ranges=ranges)

    def image_np(self):
        torch.cuda.synchronize()
        return to_np(self.rgb), to_np(self.Tout)
