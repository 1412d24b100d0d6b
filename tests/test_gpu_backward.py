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
