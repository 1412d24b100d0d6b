"""Small builders for hand-made test scenes (no method arithmetic)."""
from __future__ import annotations

import math

import numpy as np

from harness import synth


def planes_from(pos, quat, logscale, opl, sh, deg, n_pad=None):
    """SoA float32 [11+3B][n_pad] from per-Gaussian arrays (pos (n,3), quat (n,4) wxyz, ...)."""
    pos = np.atleast_2d(np.asarray(pos, np.float64))
    n = pos.shape[0]
    n_pad = n_pad or max(4, (n + 3) // 4 * 4)
    B = (deg + 1) ** 2
    pl = np.zeros((11 + 3 * B, n_pad), np.float32)
    pl[0:3, :n] = pos.T
    pl[3:7, :n] = np.atleast_2d(np.asarray(quat, np.float64)).T
    pl[7:10, :n] = np.atleast_2d(np.asarray(logscale, np.float64)).T
    pl[10, :n] = np.asarray(opl, np.float64).reshape(-1)
    sh = np.asarray(sh, np.float64).reshape(n, B, 3)
    for b in range(B):
        for ch in range(3):
            pl[11 + 3 * b + ch, :n] = sh[:, b, ch]
    return pl


def identity_camera(W, H, f, cx=None, cy=None, near=0.2):
    cam = synth.make_camera(np.eye(3), np.zeros(3), f, f, W, H, near)
    if cx is not None:
        cam.cx = float(np.float32(cx))
    if cy is not None:
        cam.cy = float(np.float32(cy))
    return cam


def logit(o):
    return math.log(o / (1 - o))


def sh_for_rgb(rgb, deg):
    """SH coefficients whose degree-0 colour is rgb (Y00 c0 + 0.5 = rgb), higher bands zero."""
    B = (deg + 1) ** 2
    sh = np.zeros((B, 3))
    sh[0] = (np.asarray(rgb, np.float64) - 0.5) / 0.28209479177387814
    return sh


def ulp_dist(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Distance in float32 ulps between float32 a and exact (float64) b."""
    a = np.asarray(a, np.float32)
    b64 = np.asarray(b, np.float64)
    ulp = np.spacing(np.abs(b64).astype(np.float32)).astype(np.float64)
    return np.abs(a.astype(np.float64) - b64) / ulp
