"""Independent float64 textbook reference used ONLY to pin the oracle (never the GPU path).

Written from the paper's equations with numpy/scipy primitives, with no shared code
with oracle/queen_oracle.cpp and none of its fp32 operation-order contract:
  * Sigma = R S S^T R^T, R from the unit quaternion
  * Sigma' = J W Sigma W^T J^T (Eq. 1), J the affine Jacobian
  * alpha_i = o_i exp(-1/2 d^T Sigma'^-1 d), front-to-back compositing (Eq. 2)
  * SH colour from scipy.special.sph_harm_y real harmonics (Condon-Shortley phase)
with the 3D-GS cut-offs of DESIGN reading R14 (skip alpha < 1/255, clamp 0.99, stop at T < 1e-4).
"""
from __future__ import annotations

import numpy as np
from scipy import special


def quat_to_rot(q):
    q = q / np.linalg.norm(q, axis=0, keepdims=True)
    w, x, y, z = q
    R = np.empty((q.shape[1], 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - w * z)
    R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y)
    R[:, 2, 1] = 2 * (y * z + w * x)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def real_sh(deg, dirs):
    """[B][n] real SH (Condon-Shortley), order m = -l..l within each degree."""
    x, y, z = dirs
    theta = np.arccos(np.clip(z, -1, 1))
    phi = np.arctan2(y, x)
    out = []
    for l in range(deg + 1):
        for m in range(-l, l + 1):
            Y = special.sph_harm_y(l, abs(m), theta, phi)
            out.append(np.sqrt(2) * Y.real if m > 0 else (np.sqrt(2) * Y.imag if m < 0 else Y.real))
    return np.array(out)


def project64(planes, n, deg, cam):
    pl = planes[:, :n].astype(np.float64)
    R = cam.R.astype(np.float64)
    t = cam.t.astype(np.float64)
    p = pl[0:3]
    pc = R @ p + t[:, None]
    z = pc[2]
    valid = z > cam.near
    Rq = quat_to_rot(pl[3:7])
    s = np.exp(pl[7:10])
    M = Rq * s.T[:, None, :]
    Sigma = M @ np.transpose(M, (0, 2, 1))
    zz = np.where(valid, z, 1.0)
    tx = np.clip(pc[0] / zz, -cam.limx * 1.0, cam.limx) * zz
    ty = np.clip(pc[1] / zz, -cam.limy * 1.0, cam.limy) * zz
    J = np.zeros((n, 2, 3))
    J[:, 0, 0] = cam.fx / zz
    J[:, 0, 2] = -cam.fx * tx / zz ** 2
    J[:, 1, 1] = cam.fy / zz
    J[:, 1, 2] = -cam.fy * ty / zz ** 2
    T = J @ R
    S2 = T @ Sigma @ np.transpose(T, (0, 2, 1))
    S2[:, 0, 0] += 0.3
    S2[:, 1, 1] += 0.3
    det = S2[:, 0, 0] * S2[:, 1, 1] - S2[:, 0, 1] ** 2
    valid &= det > 0
    conic = np.linalg.inv(np.where(valid[:, None, None], S2, np.eye(2)))
    o = 1.0 / (1.0 + np.exp(-pl[10]))
    valid &= 255.0 * o > 1.0
    u = cam.fx * pc[0] / zz + cam.cx
    v = cam.fy * pc[1] / zz + cam.cy
    d = p - cam.C.astype(np.float64)[:, None]
    d /= np.linalg.norm(d, axis=0, keepdims=True)
    Y = real_sh(deg, d)
    B = (deg + 1) ** 2
    rgb = np.zeros((3, n))
    for ch in range(3):
        for b in range(B):
            rgb[ch] += Y[b] * pl[11 + 3 * b + ch]
    rgb = np.maximum(rgb + 0.5, 0.0)
    return dict(valid=valid, u=u, v=v, conic=conic, o=o, rgb=rgb, z=z, S2=S2)


def render64(planes, n, deg, cam, bg=(0.0, 0.0, 0.0)):
    pr = project64(planes, n, deg, cam)
    W, H = cam.width, cam.height
    ys, xs = np.mgrid[0:H, 0:W]
    xs = xs.reshape(-1).astype(np.float64)
    ys = ys.reshape(-1).astype(np.float64)
    C = np.zeros((3, xs.size))
    T = np.ones(xs.size)
    live = np.ones(xs.size, bool)
    idx = np.nonzero(pr["valid"])[0]
    order = idx[np.lexsort((idx, pr["z"][idx]))]
    for i in order:
        dx = xs - pr["u"][i]
        dy = ys - pr["v"][i]
        cn = pr["conic"][i]
        maha = cn[0, 0] * dx * dx + 2 * cn[0, 1] * dx * dy + cn[1, 1] * dy * dy
        alpha = pr["o"][i] * np.exp(-0.5 * maha)
        use = live & (alpha >= 1.0 / 255.0)
        a = np.minimum(alpha, 0.99)
        C[:, use] += pr["rgb"][:, i:i + 1] * (a * T)[use]
        T = np.where(use, T * (1 - a), T)
        live &= ~(use & (T < 1e-4))
    out = C + T * np.asarray(bg, np.float64)[:, None]
    return out.reshape(3, H, W), T.reshape(H, W)
