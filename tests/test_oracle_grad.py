"""NEXT #4 oracle pins: the float64 gradient oracle (oracle/grad.py).

  * blend_forward64 on the fp32 forward's contributor lists reproduces the fp32 oracle image
    (Eq. 2) to 1e-5: the lists, their order, termination and clamps are right;
  * project_forward64 reproduces the fp32 oracle's projection records (Eq. 1) to
    fp32 rounding: the float64 formula is the same function;
  * both gradients equal central finite differences of those float64 functions;
  * a single Gaussian's colour gradient is the closed form alpha (Eq. 2 with one term).
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import grad as G
from harness import synth


def _case(n=300, deg=1, seed=5):
    cfg = synth.get_config("tiny", deg=deg)
    sc = synth.make_scene(cfg, n=n)
    cams = synth.make_cameras(cfg)
    proj, bins, rgb, T = oracle.render(sc.planes, sc.n, sc.deg, cams, bg=(0.1, 0.2, 0.3))
    contrib = oracle.contributors(proj, bins, cams[0].width, cams[0].height)
    return sc, cams, proj, bins, rgb, T, contrib


def test_blend_forward64_reproduces_fp32_image():
    sc, cams, proj, bins, rgb, T, contrib = _case()
    V, n_pad, _ = proj["rec"].shape
    t = G._rec_tensors(proj["rec"], False)
    out, Tf = G.blend_forward64(t, *contrib, V, n_pad, cams[0].width, cams[0].height, (0.1, 0.2, 0.3))
    assert np.abs(out.numpy() - rgb).max() < 2e-5
    assert np.abs(Tf.numpy() - T).max() < 2e-5
    assert contrib[0][-1] > 1000


def test_blend_grad_matches_finite_differences():
    sc, cams, proj, bins, rgb, T, contrib = _case(n=120)
    V, n_pad, _ = proj["rec"].shape
    W, H = cams[0].width, cams[0].height
    rng = np.random.default_rng(0)
    gout = rng.standard_normal((V, 3, H, W))
    g = G.blend_grad(proj["rec"], contrib, W, H, (0.1, 0.2, 0.3), gout)
    base = G._rec_tensors(proj["rec"], False)
    live = np.nonzero(np.abs(g[0]).sum(1) > 1e-3)[0]
    assert live.size > 10
    keys = ("u", "v", "A2", "B2", "C2", "o")
    for i in rng.choice(live, 6, replace=False):
        for j, k in enumerate(keys + ("r", "g", "b")):
            h = 1e-6
            vals = []
            for sgn in (1, -1):
                t = {kk: vv.clone() for kk, vv in base.items()}
                if j < 6:
                    t[k][i] += sgn * h
                else:
                    t["rgb"][i, j - 6] += sgn * h
                out, _ = G.blend_forward64(t, *contrib, V, n_pad, W, H, (0.1, 0.2, 0.3))
                vals.append(float((out.numpy() * gout).sum()))
            fd = (vals[0] - vals[1]) / (2 * h)
            assert abs(fd - g[0, i, j]) <= 1e-5 * max(1.0, abs(fd)), (i, k, fd, g[0, i, j])


def test_single_gaussian_colour_gradient_closed_form():
    """One Gaussian at a pixel: out = c a + (1 - a) bg, so d out / dc = a (Eq. 2, one term)."""
    from tests.util import planes_from
    pl = planes_from([[0.0, 0.0, 3.0]], [[1, 0, 0, 0]], [[np.log(0.05)] * 3], [0.5], [np.zeros((1, 3))], 0)
    cams = [synth.make_camera(np.eye(3), np.zeros(3), 100.0, 100.0, 32, 32)]
    proj, bins, rgb, T = oracle.render(pl, 1, 0, cams)
    contrib = oracle.contributors(proj, bins, 32, 32)
    gout = np.zeros((1, 3, 32, 32))
    gout[0, 0, 16, 16] = 1.0  # the pixel at the Gaussian's centre (u = cx = 16)
    g = G.blend_grad(proj["rec"], contrib, 32, 32, (0, 0, 0), gout)
    a = 1.0 - float(T[0, 16, 16])
    assert abs(g[0, 0, 6] - a) < 1e-6 and abs(g[0, 0, 7]) < 1e-12


def test_project_forward64_reproduces_fp32_records():
    sc, cams, proj, bins, rgb, T, contrib = _case(n=400, deg=3)
    live, jc, shc = G.project_decisions(proj, sc.planes, sc.n, sc.deg, cams)
    outs = G.project_forward64(torch.from_numpy(sc.planes.astype(np.float64)), sc.n, sc.deg, cams[0], live[0], jc[0],
                               shc[0])
    rec = proj["rec"][0, :sc.n]
    conic_scale = np.maximum(np.abs(rec[:, 4]), np.abs(rec[:, 6])).astype(np.float64)
    for j, w in enumerate((0, 1, 4, 5, 6, 8, 9, 10, 11)):
        ref = rec[:, w].astype(np.float64)
        got = outs[j].numpy()
        tol = 2e-5 * (conic_scale if w in (4, 5, 6) else np.maximum(np.abs(ref), 1.0))
        assert np.all(np.abs(got - ref) <= tol), (w, np.abs(got - ref).max())


def test_project_grad_matches_finite_differences():
    sc, cams, proj, bins, rgb, T, contrib = _case(n=60, deg=2)
    V, n_pad, _ = proj["rec"].shape
    rng = np.random.default_rng(1)
    Grec = rng.standard_normal((V, n_pad, G.REC_GRAD))
    g = G.project_grad(sc.planes, sc.n, sc.deg, cams, proj, Grec)
    live, jc, shc = G.project_decisions(proj, sc.planes, sc.n, sc.deg, cams)

    def L(pl64):
        outs = G.project_forward64(torch.from_numpy(pl64), sc.n, sc.deg, cams[0], live[0], jc[0], shc[0])
        return sum(float((outs[j].numpy() * Grec[0, :sc.n, j]).sum()) for j in range(G.REC_GRAD))

    base = sc.planes.astype(np.float64)
    ids = np.nonzero(live[0])[0]
    for i in rng.choice(ids, 4, replace=False):
        for r in (0, 2, 3, 5, 7, 9, 10, 11, 14, 20):
            if r >= base.shape[0]:
                continue
            h = 1e-6
            a, b = base.copy(), base.copy()
            a[r, i] += h
            b[r, i] -= h
            fd = (L(a) - L(b)) / (2 * h)
            assert abs(fd - g[r, i]) <= 2e-5 * max(1.0, abs(fd)), (i, r, fd, g[r, i])


def test_decode_grad_finite_differences_and_ste():
    """Decoder and gate gradients equal central differences of the float64 decode; latent
    gradients are the straight-through ones, D_c^T dL/dr_c."""
    cfg = synth.get_config("tiny", deg=1)
    sc = synth.make_scene(cfg, n=200)
    pkt = synth.make_packet(sc, 1)
    rng = np.random.default_rng(2)
    gA = rng.standard_normal(sc.planes.shape)
    gdec, glat, gla, gpre = G.decode_grad(pkt, sc.planes, gA)

    def L(dec=None, la=None, pre=None):
        t = lambda a: torch.from_numpy(np.asarray(a, np.float64))  # noqa: E731
        A = G.decode_forward64(pkt, t(pkt.latents_f32[:, :sc.n]), t(pkt.decoders if dec is None else dec),
                               t(pkt.log_alpha[:sc.n] if la is None else la),
                               t(pkt.pos_pregate[:, :sc.n] if pre is None else pre), sc.planes)
        return float((A.numpy() * gA[:, :sc.n]).sum())

    h = 1e-6
    for j in rng.choice(pkt.decoders.size, 5, replace=False):
        a, b = pkt.decoders.astype(np.float64), pkt.decoders.astype(np.float64)
        a[j] += h
        b[j] -= h
        assert abs((L(dec=a) - L(dec=b)) / (2 * h) - gdec[j]) < 1e-6 * max(1, abs(gdec[j]))
    on = np.nonzero(np.abs(gla) > 0)[0]
    assert on.size > 3
    for i in on[:5]:
        a, b = pkt.log_alpha[:sc.n].astype(np.float64), pkt.log_alpha[:sc.n].astype(np.float64)
        a[i] += h
        b[i] -= h
        assert abs((L(la=a) - L(la=b)) / (2 * h) - gla[i]) < 1e-5 * max(1, abs(gla[i]))
    # STE: dL/dl_hat for category 0 (rotation, rows 3-6) = D_0^T gA[3:7]
    L0, M0 = pkt.lat[0], 4
    D0 = pkt.decoders[:M0 * L0].reshape(M0, L0).astype(np.float64)
    assert np.allclose(glat[:L0], D0.T @ gA[3:7, :sc.n], rtol=1e-12, atol=1e-12)
