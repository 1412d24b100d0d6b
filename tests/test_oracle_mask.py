"""NEXT #3 oracle pins: masked / dynamic-subset rendering.

  * dilate() against the definition, pixel by pixel (brute-force window OR), even and odd d,
    d = 1 (identity), d larger than the image, a single mark -> a clipped d x d block;
  * render_mask(): empty subset -> all zero; monotone in the alpha threshold and in the
    subset; the full subset equals the dilated alpha mask of the ordinary render;
  * marks at threshold 1e-3 equal "some subset Gaussian reaches alpha >= 1/255 at the pixel"
    computed by the independent float64 textbook renderer (tests/ref64.py), except pixels whose
    float64 alpha is within 1e-5 of 1/255 (fp32 vs fp64 decision).
"""
import numpy as np
import pytest

import oracle
from harness import synth
from tests import ref64


def _brute_dilate(m, d):
    H, W = m.shape
    a = d // 2
    out = np.zeros_like(m, dtype=bool)
    for y in range(H):
        for x in range(W):
            y0, y1 = max(0, y - a), min(H, y - a + d)
            x0, x1 = max(0, x - a), min(W, x - a + d)
            out[y, x] = m[y0:y1, x0:x1].any()
    return out


@pytest.mark.parametrize("d", [1, 2, 3, 7, 48, 100])
def test_dilate_matches_definition(d):
    rng = np.random.default_rng(d)
    m = rng.random((37, 53)) < 0.01
    assert np.array_equal(oracle.dilate(m, d), _brute_dilate(m, d))


def test_dilate_single_mark_block():
    m = np.zeros((100, 120), bool)
    m[50, 60] = True
    out = oracle.dilate(m, 48)
    ys, xs = np.nonzero(out)
    assert out.sum() == 48 * 48
    assert (ys.min(), ys.max(), xs.min(), xs.max()) == (50 - 23, 50 + 24, 60 - 23, 60 + 24)
    m2 = np.zeros((100, 120), bool)
    m2[0, 119] = True  # corner: clipped block
    out2 = oracle.dilate(m2, 48)
    assert out2.sum() == 25 * 24 and out2[0, 119] and out2[24, 96] and not out2[25, 119]


def _scene(n=600):
    cfg = synth.get_config("tiny")
    sc = synth.make_scene(cfg, n=n)
    cams = synth.make_cameras(cfg)
    return sc, cams


def test_empty_subset_all_zero():
    sc, cams = _scene()
    m = oracle.render_mask(sc.planes, sc.n, sc.deg, cams, np.zeros(0, np.int64))
    assert m.shape == (1, cams[0].height, cams[0].width) and not m.any()


def test_full_subset_equals_dilated_render_alpha():
    sc, cams = _scene()
    full = oracle.render_mask(sc.planes, sc.n, sc.deg, cams, np.arange(sc.n), 1e-3, 9)
    _, _, _, T = oracle.render(sc.planes, sc.n, sc.deg, cams)
    assert np.array_equal(full, oracle.dilate((np.float32(1) - T) > np.float32(1e-3), 9).astype(np.uint8))


def test_monotone_in_threshold_and_subset():
    sc, cams = _scene()
    rng = np.random.default_rng(3)
    sub = np.sort(rng.choice(sc.n, 200, replace=False))
    sub_small = sub[::3]
    m_lo = oracle.render_mask(sc.planes, sc.n, sc.deg, cams, sub, 1e-3, 5)
    m_hi = oracle.render_mask(sc.planes, sc.n, sc.deg, cams, sub, 0.3, 5)
    m_small = oracle.render_mask(sc.planes, sc.n, sc.deg, cams, sub_small, 1e-3, 5)
    assert np.all(m_hi <= m_lo) and np.all(m_small <= m_lo)
    assert m_lo.sum() > m_hi.sum() > 0


def test_marks_are_alpha_reach_of_float64_reference():
    sc, cams = _scene(400)
    rng = np.random.default_rng(4)
    sub = np.sort(rng.choice(sc.n, 150, replace=False))
    marks = oracle.render_mask(sc.planes, sc.n, sc.deg, cams, sub, 1e-3, 1)[0].astype(bool)
    cam = cams[0]
    kp = (sub.size + 3) // 4 * 4
    P = np.zeros((sc.planes.shape[0], kp), np.float32)
    P[:, :sub.size] = sc.planes[:, sub]
    pr = ref64.project64(P, sub.size, sc.deg, cam)
    H, W = cam.height, cam.width
    ys, xs = np.mgrid[0:H, 0:W].astype(np.float64)
    amax = np.zeros((H, W))
    for i in np.nonzero(pr["valid"])[0]:
        dx, dy = xs - pr["u"][i], ys - pr["v"][i]
        cn = pr["conic"][i]
        maha = cn[0, 0] * dx * dx + 2 * cn[0, 1] * dx * dy + cn[1, 1] * dy * dy
        amax = np.maximum(amax, pr["o"][i] * np.exp(-0.5 * maha))
    ref = amax >= 1.0 / 255.0
    near = np.abs(amax - 1.0 / 255.0) < 1e-5
    assert ref.sum() > 50
    assert np.all((marks == ref) | near)
