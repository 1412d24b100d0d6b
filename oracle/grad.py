"""Gradient oracle for NEXT #4 (backward rasterizer + projection), plain PyTorch CPU float64.

TEST INFRASTRUCTURE ONLY (same rule as the rest of oracle/): only tests/ may import this.

The backward pass differentiates the forward equations as written -- Eq. 1 (EWA projection,
P:219-226) and Eq. 2 (front-to-back compositing) -- with torch autograd in float64.
The forward's discrete decisions (which records a pixel composites, in which order, where it
terminates, whether alpha hit the 0.99 clamp, which Gaussians are culled, whether the
Jacobian's x/z, y/z hit the 1.3 tan(FoV/2) clamp, whether an SH channel hit max(0, .)) are
piecewise-constant: they are taken from the fp32 oracle (contributors(), project()), exactly
as the GPU takes them, and held fixed while differentiating, which is the derivative of the
piece the input lies in.

Record gradient layout (per view, per Gaussian): 9 values
    d/du, d/dv, d/dA2, d/dB2, d/dC2, d/do, d/dr, d/dg, d/db
for the blend's record words u, v, A2, B2, C2 (base-2 conic, p2 = A2 dx^2 + B2 dx dy + C2 dy^2
with dx = u - x, dy = v - y), o, rgb.
"""
from __future__ import annotations

import math

import numpy as np
import torch

REC_GRAD = 9  # u, v, A2, B2, C2, o, r, g, b
LOG2E = 1.0 / math.log(2.0)


def blend_forward64(rec_t: dict, offsets, gid, clamp, V: int, n_pad: int, W: int, H: int, bg):
    """Eq. 2 on fixed contributor lists, float64: out [V][3][H][W].  rec_t: dict of float64
    tensors [V*n_pad] (u, v, A2, B2, C2, o) and rgb [V*n_pad][3]."""
    P = V * H * W
    counts = np.diff(offsets)
    pix = np.repeat(np.arange(P), counts)
    view = pix // (H * W)
    y = (pix // W) % H
    x = pix % W
    rid = torch.from_numpy(view * n_pad + gid.astype(np.int64))
    xs = torch.from_numpy(x.astype(np.float64))
    ys = torch.from_numpy(y.astype(np.float64))
    dx = rec_t["u"][rid] - xs
    dy = rec_t["v"][rid] - ys
    p2 = rec_t["A2"][rid] * dx * dx + rec_t["B2"][rid] * dx * dy + rec_t["C2"][rid] * dy * dy
    alpha = rec_t["o"][rid] * torch.pow(2.0, p2)
    cl = torch.from_numpy(clamp.astype(bool))
    alpha = torch.where(cl, torch.full_like(alpha, 0.99), alpha)
    l1m = torch.log1p(-alpha)
    cs = torch.cumsum(l1m, 0)
    ex = cs - l1m                                           # exclusive prefix (global)
    seg0 = torch.from_numpy(offsets[:-1][counts > 0])        # first pair of each non-empty pixel
    base = torch.zeros(P, dtype=torch.float64)
    base[torch.from_numpy(np.nonzero(counts)[0])] = ex[seg0]
    pt = torch.from_numpy(pix)
    Ti = torch.exp(ex - base[pt])
    w = alpha * Ti
    C = torch.zeros((P, 3), dtype=torch.float64)
    C = C.index_add(0, pt, rec_t["rgb"][rid] * w[:, None])
    logT = torch.zeros(P, dtype=torch.float64).index_add(0, pt, l1m)
    Tf = torch.exp(logT)
    out = C + Tf[:, None] * torch.tensor(bg, dtype=torch.float64)[None, :]
    return out.reshape(V, H, W, 3).permute(0, 3, 1, 2), Tf.reshape(V, H, W)


def _rec_tensors(rec: np.ndarray, requires_grad: bool):
    V, n_pad, _ = rec.shape
    r = torch.from_numpy(rec.reshape(V * n_pad, 12).astype(np.float64))
    t = {"u": r[:, 0].clone(), "v": r[:, 1].clone(), "A2": r[:, 4].clone(), "B2": r[:, 5].clone(),
         "C2": r[:, 6].clone(), "o": r[:, 8].clone(), "rgb": r[:, 9:12].clone()}
    if requires_grad:
        for k in t:
            t[k].requires_grad_(True)
    return t


def blend_grad(rec: np.ndarray, contrib, W: int, H: int, bg, dL_dout: np.ndarray) -> np.ndarray:
    """dL/d(record) [V][n_pad][9] for L = sum(out * dL_dout), out = Eq. 2 (float64)."""
    V, n_pad, _ = rec.shape
    offsets, gid, clamp = contrib
    t = _rec_tensors(rec, True)
    out, _ = blend_forward64(t, offsets, gid, clamp, V, n_pad, W, H, bg)
    L = (out * torch.from_numpy(dL_dout.astype(np.float64))).sum()
    L.backward()
    g = torch.zeros((V * n_pad, REC_GRAD), dtype=torch.float64)
    for j, k in enumerate(("u", "v", "A2", "B2", "C2", "o")):
        if t[k].grad is not None:
            g[:, j] = t[k].grad
    if t["rgb"].grad is not None:
        g[:, 6:9] = t["rgb"].grad
    return g.reshape(V, n_pad, REC_GRAD).numpy()


# ----------------------------------------------------------------------------- projection
_SH_C0 = 0.28209479177387814
_SH_C1 = 0.4886025119029199
_SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792, 0.5462742152960396)
_SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154, -0.4570457994644658,
          1.445305721320277, -0.5900435899266435)


def _sh_basis64(deg, x, y, z):
    """Real SH basis (3D-GS constants and signs, DESIGN R10), float64 torch."""
    Y = [torch.full_like(x, _SH_C0)]
    if deg >= 1:
        Y += [-_SH_C1 * y, _SH_C1 * z, -_SH_C1 * x]
    if deg >= 2:
        xx, yy, zz, xy, yz, xz = x * x, y * y, z * z, x * y, y * z, x * z
        Y += [_SH_C2[0] * xy, _SH_C2[1] * yz, _SH_C2[2] * (2 * zz - xx - yy), _SH_C2[3] * xz, _SH_C2[4] * (xx - yy)]
    if deg >= 3:
        Y += [_SH_C3[0] * y * (3 * xx - yy), _SH_C3[1] * xy * z, _SH_C3[2] * y * (4 * zz - xx - yy),
              _SH_C3[3] * z * (2 * zz - 3 * xx - 3 * yy), _SH_C3[4] * x * (4 * zz - xx - yy),
              _SH_C3[5] * z * (xx - yy), _SH_C3[6] * x * (xx - 3 * yy)]
    return torch.stack(Y, 0)


def project_forward64(planes_t, n: int, deg: int, cam, live: np.ndarray, jclamp: np.ndarray, shclamp: np.ndarray):
    """Eq. 1 + SH colour for one camera in float64 on the raw SoA (rows: 0-2 p, 3-6 raw q,
    7-9 log s, 10 opacity logit, 11+ SH), for the Gaussians flagged live.  jclamp [n][2]:
    x/z resp. y/z hit the Jacobian clamp (their clamped value is then a constant);
    shclamp [n][3]: the channel hit max(0, .) (colour 0, constant).  Returns the record
    values u, v, A2, B2, C2, o, r, g, b as float64 tensors [n] (zeros where not live)."""
    Pl = planes_t[:, :n]
    p = Pl[0:3]
    q = Pl[3:7]
    q = q / torch.sqrt((q * q).sum(0, keepdim=True))
    w, x, y, z = q
    R = torch.stack([torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)]),
                     torch.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)]),
                     torch.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)])])  # [3][3][n]
    s = torch.exp(Pl[7:10])
    M = R * s[None, :, :]
    Sig = torch.einsum("ikn,jkn->ijn", M, M)
    Rw = torch.tensor(np.asarray(cam.R, np.float64).reshape(3, 3))
    tw = torch.tensor(np.asarray(cam.t, np.float64).reshape(3))
    xc = torch.einsum("ij,jn->in", Rw, p) + tw[:, None]
    X, Yc, Z = xc
    tx, ty = X / Z, Yc / Z
    jc = torch.from_numpy(jclamp.astype(bool))
    txc = torch.where(jc[:, 0], torch.clamp(tx, -cam.limx, cam.limx).detach(), tx)
    tyc = torch.where(jc[:, 1], torch.clamp(ty, -cam.limy, cam.limy).detach(), ty)
    zero = torch.zeros_like(Z)
    J = torch.stack([torch.stack([cam.fx / Z, zero, -cam.fx * txc / Z]),
                     torch.stack([zero, cam.fy / Z, -cam.fy * tyc / Z])])  # [2][3][n]
    Tm = torch.einsum("ikn,kj->ijn", J, Rw)
    Sp = torch.einsum("ikn,kln,jln->ijn", Tm, Sig, Tm)
    a = Sp[0, 0] + 0.3
    b = Sp[0, 1]
    c = Sp[1, 1] + 0.3
    det = a * c - b * b
    ca, cb, cc = c / det, -b / det, a / det
    A2 = -0.5 * ca * LOG2E
    B2 = -cb * LOG2E
    C2 = -0.5 * cc * LOG2E
    u = cam.fx * tx + cam.cx
    v = cam.fy * ty + cam.cy
    o = torch.sigmoid(Pl[10])
    Cw = torch.tensor(np.asarray(cam.C, np.float64).reshape(3))
    d = p - Cw[:, None]
    d = d / torch.sqrt((d * d).sum(0, keepdim=True))
    Yb = _sh_basis64(deg, d[0], d[1], d[2])
    B = (deg + 1) ** 2
    sh = Pl[11:11 + 3 * B].reshape(B, 3, n)
    col = torch.einsum("bn,bcn->cn", Yb, sh) + 0.5
    shc = torch.from_numpy(shclamp.astype(bool)).T
    col = torch.where(shc, torch.zeros_like(col), col)
    lv = torch.from_numpy(live.astype(bool))
    outs = [u, v, A2, B2, C2, o, col[0], col[1], col[2]]
    return [torch.where(lv, t_, torch.zeros_like(t_)) for t_ in outs]


def project_decisions(proj, planes: np.ndarray, n: int, deg: int, cams):
    """The fp32 forward's decisions per (view, Gaussian): live (a record was written: o > 0),
    Jacobian clamp of x/z and y/z, SH max(0, .) clamp (channel exactly 0)."""
    V = len(cams)
    rec = proj["rec"]
    live = rec[:, :n, 8] > 0
    shc = rec[:, :n, 9:12] == 0.0
    jc = np.zeros((V, n, 2), bool)
    for vi, cam in enumerate(cams):
        R = np.asarray(cam.R, np.float32).reshape(3, 3)
        t = np.asarray(cam.t, np.float32).reshape(3)
        xc = (R.astype(np.float64) @ planes[0:3, :n].astype(np.float64)) + t[:, None]
        tx, ty = xc[0] / xc[2], xc[1] / xc[2]
        jc[vi, :, 0] = np.abs(tx) > cam.limx
        jc[vi, :, 1] = np.abs(ty) > cam.limy
    return live, jc, shc


def project_grad(planes: np.ndarray, n: int, deg: int, cams, proj, G_rec: np.ndarray) -> np.ndarray:
    """dL/d(planes) [P][n] (float64) for L = sum over views and live Gaussians of
    G_rec[v][i] . record(v, i), the record values of project_forward64."""
    live, jc, shc = project_decisions(proj, planes, n, deg, cams)
    pt = torch.from_numpy(planes.astype(np.float64)).requires_grad_(True)
    L = torch.zeros((), dtype=torch.float64)
    for vi, cam in enumerate(cams):
        outs = project_forward64(pt, n, deg, cam, live[vi], jc[vi], shc[vi])
        G = torch.from_numpy(G_rec[vi, :n].astype(np.float64))
        for j in range(REC_GRAD):
            L = L + (outs[j] * G[:, j]).sum()
    L.backward()
    return pt.grad[:, :n].numpy()


# ----------------------------------------------------------------------------- decode / gates
def decode_forward64(pkt, lhat_t, dec_t, la_t, pre_t, planes0: np.ndarray, use_gates: bool = True):
    """A_t = A_{t-1} + R_t in float64 (Eq. 4-5; gates P:319-338): attribute rows get
    D_c round(l_hat_c) with the straight-through estimator (round acts as the identity in the
    backward pass, "straight-through estimator"), positions get g * l_p on the
    gate's mask (log alpha > theta0, decided in fp32 as the forward does); g's clamp to [0, 1]
    is held at the forward's decision.  Returns the float64 planes [P][n]."""
    from oracle import theta0
    n, deg = pkt.n, pkt.deg
    B = (deg + 1) ** 2
    M = (4, 3, 1, 3, 3 * (B - 1))  # rot, scale, opacity, SH-DC, SH-rest rows (R2, R3)
    lat = pkt.lat
    rows = []
    r0 = 0
    d0 = 0
    l_st = lhat_t + (torch.round(lhat_t) - lhat_t).detach()  # STE
    for c in range(5):
        L = lat[c]
        Mc = M[c]
        if L == 0:
            rows.append(torch.zeros((Mc, n), dtype=torch.float64))
            continue
        D = dec_t[d0:d0 + Mc * L].reshape(Mc, L)
        rows.append(D @ l_st[r0:r0 + L, :n])
        r0 += L
        d0 += Mc * L
    R = torch.cat(rows, 0)
    A0 = torch.from_numpy(planes0[:, :n].astype(np.float64))
    pos = A0[0:3]
    if use_gates:
        tau, g0, g1 = pkt.gate
        th0 = float(theta0(*pkt.gate))
        mask = torch.from_numpy(pkt.log_alpha[:n].astype(np.float32) > np.float32(th0))
        gt = torch.sigmoid(la_t[:n] / tau) * (g1 - g0) + g0
        clamp_lo = (gt.detach() <= 0)
        clamp_hi = (gt.detach() >= 1)
        g = torch.where(clamp_hi, torch.ones_like(gt), torch.where(clamp_lo, torch.zeros_like(gt), gt))
        g = torch.where(mask, g, torch.zeros_like(g))
        pos = pos + g[None, :] * pre_t[:, :n]
    return torch.cat([pos, A0[3:] + R], 0)


def decode_grad(pkt, planes0: np.ndarray, gA: np.ndarray, use_gates: bool = True):
    """dL/d(decoders [ndec], l_hat [sum L][n], log_alpha [n], pregate [3][n]) for
    L = sum(gA * A_t), float64 autograd of decode_forward64."""
    n = pkt.n
    lhat = torch.from_numpy(np.ascontiguousarray(pkt.latents_f32[:, :n], np.float64)).requires_grad_(True)
    dec = torch.from_numpy(np.asarray(pkt.decoders, np.float64)).requires_grad_(True)
    la = torch.from_numpy(np.asarray(pkt.log_alpha[:n], np.float64)).requires_grad_(True)
    pre = torch.from_numpy(np.ascontiguousarray(pkt.pos_pregate[:, :n], np.float64)).requires_grad_(True)
    A = decode_forward64(pkt, lhat, dec, la, pre, planes0, use_gates)
    (A * torch.from_numpy(gA[:, :n].astype(np.float64))).sum().backward()
    z = lambda t: t.grad.numpy() if t.grad is not None else np.zeros(t.shape)  # noqa: E731
    return z(dec), z(lhat), z(la), z(pre)
