"""NEXT #4 on the GPU: backward rasterizer and projection backward vs the float64 gradient oracle
(oracle/grad.py: torch autograd of Eq. 1-2 on the forward's fixed decisions).

Tolerances: the GPU works in fp32 (ex2.approx alphas, T recovered by division, float-atomic
accumulation), the oracle in float64; per gradient component the max error is compared with
the component's max magnitude (2e-3), and most entries agree far tighter.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import grad as G  # noqa: E402
from harness import synth  # noqa: E402


def _scene(n=6000, views=3, deg=3, max_logit=3.8):
    cfg = synth.get_config("n3dv", width=160, height=120, focal=140.0, deg=deg)
    sc = synth.make_scene(cfg, n=n)
    sc.planes[10, :sc.n] = np.minimum(sc.planes[10, :sc.n], max_logit)  # o <= 0.978: no 0.99 clamps
    cams = synth.make_cameras(cfg, views)
    return sc, cams


def _stages(sc, cams):
    from tests.gpu_helpers import Stages
    st = Stages(sc.planes, sc.n, sc.deg, cams).project().bin_sort()
    return st


def _close(got, ref, tol=2e-3):
    for k in range(ref.shape[-1]):
        r = ref[..., k]
        m = np.abs(r).max()
        if m == 0:
            assert np.abs(got[..., k]).max() < 1e-6, k
            continue
        err = np.abs(got[..., k] - r).max() / m
        assert err <= tol, (k, err, m)


@pytest.mark.parametrize("deg", [0, 3])
def test_rasterize_backward_matches_oracle(deg):
    import paper_2412_04469_b200 as Q
    sc, cams = _scene(deg=deg)
    st = _stages(sc, cams)
    W, H = cams[0].width, cams[0].height
    bg = (0.1, 0.2, 0.3)
    rng = np.random.default_rng(7)
    gout = rng.standard_normal((len(cams), 3, H, W)).astype(np.float32)
    grec = torch.empty((len(cams), st.n_pad, 9), dtype=torch.float32, device="cuda")
    Q.queen_rasterize_backward(st.ctx, st.proj, st.bins, cams, torch.from_numpy(gout).cuda(), grec, bg)
    assert st.ctx.check_status()[0] == 0
    proj, bins, _, _ = oracle.render(sc.planes, sc.n, sc.deg, cams, bg=bg)
    contrib = oracle.contributors(proj, bins, W, H)
    ref = G.blend_grad(proj["rec"], contrib, W, H, bg, gout.astype(np.float64))
    got = grec.cpu().numpy()
    assert np.abs(ref).max() > 0
    _close(got, ref)
    # records that never composite get exactly zero
    dead = np.abs(ref).sum(-1) == 0
    assert np.all(got[dead] == 0)


def test_rasterize_backward_clamped_alpha():
    """A Gaussian whose alpha hits the 0.99 clamp at some pixels: there d/do and d/dp2 vanish."""
    import paper_2412_04469_b200 as Q
    from tests.gpu_helpers import Stages
    from tests.util import planes_from
    pl = planes_from([[0.0, 0.0, 3.0], [0.02, 0.01, 4.0]], [[1, 0, 0, 0]] * 2, [[np.log(0.2)] * 3, [np.log(0.05)] * 3],
                     [6.0, 1.0],
                     [np.ones((1, 3)) * 0.3] * 2, 0)
    cams = [synth.make_camera(np.eye(3), np.zeros(3), 100.0, 100.0, 48, 40)]
    st = Stages(pl, 2, 0, cams).project().bin_sort()
    rng = np.random.default_rng(1)
    gout = rng.standard_normal((1, 3, 40, 48)).astype(np.float32)
    grec = torch.empty((1, st.n_pad, 9), dtype=torch.float32, device="cuda")
    Q.queen_rasterize_backward(st.ctx, st.proj, st.bins, cams, torch.from_numpy(gout).cuda(), grec)
    proj, bins, _, _ = oracle.render(pl, 2, 0, cams)
    contrib = oracle.contributors(proj, bins, 48, 40)
    assert contrib[2].sum() > 0  # some clamped pairs
    ref = G.blend_grad(proj["rec"], contrib, 48, 40, (0, 0, 0), gout.astype(np.float64))
    _close(grec.cpu().numpy(), ref)


@pytest.mark.parametrize("deg", [1, 3])
def test_project_backward_matches_oracle(deg):
    import paper_2412_04469_b200 as Q
    sc, cams = _scene(n=3000, deg=deg)
    st = _stages(sc, cams)
    proj, _, _, _ = oracle.render(sc.planes, sc.n, sc.deg, cams)
    live = proj["rec"][:, :, 8] > 0
    rng = np.random.default_rng(3)
    Grec = (rng.standard_normal((len(cams), st.n_pad, 9)) * live[..., None]).astype(np.float32)
    Grec[..., 2:5] *= 1e3  # conic entries are small numbers: scale their gradients to matter
    gpl = torch.empty((sc.planes.shape[0], st.n_pad), dtype=torch.float32, device="cuda")
    Q.queen_project_backward(st.ctx, st.scene, cams, torch.from_numpy(Grec).cuda(), gpl)
    assert st.ctx.check_status()[0] == 0
    ref = G.project_grad(sc.planes, sc.n, sc.deg, cams, proj, Grec.astype(np.float64))
    got = gpl.cpu().numpy()
    _close(got[:, :sc.n].T, ref.T, tol=3e-3)
    assert np.all(got[:, sc.n:] == 0)


def test_full_backward_chain_matches_oracle():
    """Image-space gradient -> raw attributes: project_backward(rasterize_backward(g))."""
    import paper_2412_04469_b200 as Q
    sc, cams = _scene(n=4000, deg=2)
    st = _stages(sc, cams)
    W, H = cams[0].width, cams[0].height
    rng = np.random.default_rng(11)
    gout = rng.standard_normal((len(cams), 3, H, W)).astype(np.float32)
    grec = torch.empty((len(cams), st.n_pad, 9), dtype=torch.float32, device="cuda")
    Q.queen_rasterize_backward(st.ctx, st.proj, st.bins, cams, torch.from_numpy(gout).cuda(), grec)
    gpl = torch.empty((sc.planes.shape[0], st.n_pad), dtype=torch.float32, device="cuda")
    Q.queen_project_backward(st.ctx, st.scene, cams, grec, gpl)
    proj, bins, _, _ = oracle.render(sc.planes, sc.n, sc.deg, cams)
    contrib = oracle.contributors(proj, bins, W, H)
    ref_rec = G.blend_grad(proj["rec"], contrib, W, H, (0, 0, 0), gout.astype(np.float64))
    ref = G.project_grad(sc.planes, sc.n, sc.deg, cams, proj, ref_rec)
    _close(gpl.cpu().numpy()[:, :sc.n].T, ref.T, tol=3e-3)


@pytest.mark.parametrize("f32", [True, False])
def test_decode_backward_matches_oracle(f32):
    """Decoder / straight-through latent / gate gradients vs the float64 oracle (decode_grad)."""
    import paper_2412_04469_b200 as Q
    from paper_2412_04469_b200.runtime import device_packet
    cfg = synth.get_config("n3dv")
    sc = synth.make_scene(cfg, n=30001)
    pkt = synth.make_packet(sc, 2)
    rng = np.random.default_rng(5)
    gA = rng.standard_normal(sc.planes.shape).astype(np.float32)
    gA[:, sc.n:] = 0
    ctx = Q.Context(0)
    ctx.set_workspace(sc.n_pad, 1, 16, 16, 1024)
    dp = device_packet(pkt, "cuda", gates=True, f32_latents=f32)
    ndec = pkt.decoders.size
    gdec = torch.empty(ndec, dtype=torch.float32, device="cuda")
    glat = torch.empty((sum(pkt.lat), sc.n_pad), dtype=torch.float32, device="cuda")
    gla = torch.empty(sc.n_pad, dtype=torch.float32, device="cuda")
    gpre = torch.empty((3, sc.n_pad), dtype=torch.float32, device="cuda")
    Q.queen_decode_backward(ctx, dp.struct, torch.from_numpy(gA).cuda(), gdec, glat, gla, gpre)
    assert ctx.check_status()[0] == 0
    rdec, rlat, rla, rpre = G.decode_grad(pkt, sc.planes, gA.astype(np.float64))
    n = sc.n
    assert np.abs(gdec.cpu().numpy() - rdec).max() <= 1e-4 * np.abs(rdec).max()
    assert np.abs(glat.cpu().numpy()[:, :n] - rlat).max() <= 1e-5 * np.abs(rlat).max()
    assert np.abs(gla.cpu().numpy()[:n] - rla).max() <= 1e-5 * max(np.abs(rla).max(), 1e-12)
    assert np.abs(gpre.cpu().numpy()[:, :n] - rpre).max() <= 1e-5 * np.abs(rpre).max()
    assert np.count_nonzero(rla) > 100
