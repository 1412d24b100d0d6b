"""Run libqueen stages through the C-ABI binding and bring results back as numpy (GPU tests only)."""
from __future__ import annotations

import numpy as np
import torch

import paper_2412_04469_b200 as Q
from paper_2412_04469_b200.runtime import device_packet


def to_np(t):
    return t.detach().cpu().numpy()


from paper_2412_04469_b200.stages import Stages  # noqa: E402,F401


def psnr(a, b):
    a = np.clip(np.asarray(a, np.float64), 0, 1)
    b = np.clip(np.asarray(b, np.float64), 0, 1)
    mse = float(np.mean((a - b) ** 2))
    return 100.0 if mse < 1e-10 else -10.0 * np.log10(mse)


def gpu_apply(planes: np.ndarray, pkt, *, gates=False, f32=False, frames_pkts=None, device=0):
    ctx = Q.Context(device)
    ctx.set_workspace(planes.shape[1], 1, 16, 16, 1024)
    pl = torch.from_numpy(np.ascontiguousarray(planes, np.float32)).cuda(device)
    g = Q.gaussians_struct(pl, pkt.n, pkt.deg)
    for p in (frames_pkts or [pkt]):
        dp = device_packet(p, pl.device, gates=gates, f32_latents=f32)
        Q.queen_apply_frame(ctx, g, dp.struct)
    st, info = ctx.check_status()
    return to_np(pl), st
