"""Oracle pins: projection (Eq. 1), binning/sort/ranges, compositing (Eq. 2).

Pins: SPEC worked examples (project_point, Sigma for a 90-degree rotation, single
and two-Gaussian compositing), the isotropic-footprint closed form, quaternion sign
invariance, the z-scaling law, tiled == brute force bit-for-bit, an independent
float64 textbook renderer (tests/ref64.py) within the stated error bound, and
sort / range invariants checked against numpy's lexsort.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from harness import synth
from tests import ref64
from tests.util import identity_camera, logit, planes_from, sh_for_rgb

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_spec_examples.json")))
L2E = 1.4426950408889634


def _conic_to_sigma(rec):
    """Recover Sigma' (float64) from a record's base-2 conic (A2, B2, C2)."""
    ca = rec[4] / (-0.5 * L2E)
    cb = rec[5] / (-L2E)
    cc = rec[6] / (-0.5 * L2E)
    return np.linalg.inv(np.array([[ca, cb], [cb, cc]], np.float64))


def _one(pos, quat=(1, 0, 0, 0), ls=(math.log(0.5),) * 3, o=0.9, rgb=(0.7, 0.5, 0.3), deg=0, cam=None):
    pl = planes_from([pos], [quat], [ls], [logit(o)], [sh_for_rgb(rgb, deg)], deg)
    return oracle.project(pl, 1, deg, [cam])


def test_project_point_spec_examples():
    ex = GOLD["project_point"]
    cam = identity_camera(64, 64, 60.0)  # cx = cy = 31.5
    pr = _one(ex["on_axis"]["p"], cam=cam)
    assert pr["rec"][0, 0, 0] == ex["on_axis"]["uv"][0] and pr["rec"][0, 0, 1] == ex["on_axis"]["uv"][1]
    assert np.uint32(pr["depth"][0, 0]).view(np.float32) == ex["on_axis"]["depth"]
    st = ex["similar_triangles"]
    cam2 = identity_camera(400, 64, st["fx"], cx=st["cx"])
    pr2 = _one(st["p"], cam=cam2)
    assert pr2["rec"][0, 0, 0] == st["u"]


def test_isotropic_footprint_closed_form():
    ex = GOLD["isotropic_footprint"]
    cam = identity_camera(200, 200, ex["f"])  # limx = 1.3 > x/z
    pr = _one(ex["p"], ls=(math.log(ex["sigma"]),) * 3, cam=cam)
    S2 = _conic_to_sigma(pr["rec"][0, 0])
    assert np.allclose(S2, np.array(ex["Sigma2d"]), rtol=2e-6, atol=0)
    # S:59 on-axis (f s / z)^2 + 0.3
    ax = GOLD["on_axis_footprint"]
    pr = _one([0, 0, ax["z"]], ls=(math.log(ax["sigma"]),) * 3, cam=identity_camera(200, 200, ax["f"]))
    S2 = _conic_to_sigma(pr["rec"][0, 0])
    assert np.allclose(np.diag(S2), ax["Sigma2d_diag"], rtol=2e-6) and abs(S2[0, 1]) < 1e-9


def test_covariance_rot90z_spec_example():
    ex = GOLD["covariance_rot90z"]
    f, z = 100.0, 10.0
    pr = _one([0, 0, z], quat=ex["q"], ls=[math.log(s) for s in ex["s"]], cam=identity_camera(200, 200, f))
    S2 = _conic_to_sigma(pr["rec"][0, 0])
    k = (f / z) ** 2
    expect = np.diag([k * ex["Sigma_diag"][0] + 0.3, k * ex["Sigma_diag"][1] + 0.3])
    assert np.allclose(S2, expect, rtol=2e-6, atol=2e-4)  # fp32 quaternion rounding: off-diagonal ~1e-7 relative


def test_quaternion_sign_invariance_and_scale():
    rng = np.random.default_rng(5)
    cam = identity_camera(128, 96, 80.0)
    for _ in range(20):
        q = rng.standard_normal(4)
        p = [rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), rng.uniform(2, 5)]
        ls = rng.normal(math.log(0.05), 0.5, 3)
        a = _one(p, quat=q, ls=ls, cam=cam)
        b = _one(p, quat=-q, ls=ls, cam=cam)
        c = _one(p, quat=3.0 * q, ls=ls, cam=cam)
        for key in ("rec", "depth", "tiles", "rect"):
            assert np.array_equal(a[key], b[key])  # Sigma(q) = Sigma(-q), bit-exact
        # unnormalised storage: normalisation applied; equal within rounding
        assert np.allclose(a["rec"], c["rec"], rtol=1e-5, atol=1e-6)


def test_z_scaling_law():
    """doubling z quarters the pre-floor 2D covariance on the axis."""
    cam = identity_camera(256, 256, 200.0)
    s1 = _conic_to_sigma(_one([0, 0, 3.0], ls=(math.log(0.2),) * 3, cam=cam)["rec"][0, 0])
    s2 = _conic_to_sigma(_one([0, 0, 6.0], ls=(math.log(0.2),) * 3, cam=cam)["rec"][0, 0])
    assert np.allclose((s1 - 0.3 * np.eye(2)) / 4.0, s2 - 0.3 * np.eye(2), rtol=1e-5, atol=1e-6)


def test_culling_rules():
    cam = identity_camera(64, 64, 60.0)
    behind = _one([0, 0, 0.1], cam=cam)            # z <= near (0.2)
    faint = _one([0, 0, 3.0], o=1.0 / 300.0, cam=cam)  # 255 o <= 1: alpha never reaches 1/255
    for pr in (behind, faint):
        assert pr["tiles"][0, 0] == 0 and np.all(pr["rec"] == 0) and not pr["nonfinite"]
    pl = planes_from([[0, 0, 3.0]], [[1, 0, 0, 0]], [[-2, -2, -2]], [2.0], [sh_for_rgb((1, 1, 1), 0)], 0)
    pl[8, 0] = np.nan
    pr = oracle.project(pl, 1, 0, [cam])
    assert pr["nonfinite"] and pr["tiles"][0, 0] == 0


def test_single_and_two_gaussian_compositing():
    ex = GOLD["composite_single"]
    cam = identity_camera(32, 32, 50.0, cx=16.0, cy=16.0)
    pl = planes_from([[0, 0, 3.0]], [[1, 0, 0, 0]], [[math.log(0.01)] * 3], [logit(ex["o"])],
                     [sh_for_rgb(ex["c"], 0)], 0)
    proj, bins, rgb, T = oracle.render(pl, 1, 0, [cam])
    o = proj["rec"][0, 0, 8]
    c = proj["rec"][0, 0, 9:12]
    assert np.allclose(rgb[0, :, 16, 16], c * o, rtol=1e-6) and np.allclose(c, ex["c"], atol=1e-6)
    assert T[0, 16, 16] == pytest.approx(1 - o, abs=1e-7) and abs(o - ex["o"]) < 1e-6
    assert np.allclose(rgb[0, :, 16, 16], ex["C"], atol=2e-6)
    ex2 = GOLD["composite_two"]
    pl = planes_from([[0, 0, 3.0], [0, 0, 4.0]], [[1, 0, 0, 0]] * 2, [[math.log(0.01)] * 3] * 2,
                     [logit(ex2["o"][0]), logit(ex2["o"][1])],
                     [sh_for_rgb([ex2["c"][0]] * 3, 0), sh_for_rgb([ex2["c"][1]] * 3, 0)], 0)
    proj, bins, rgb, T = oracle.render(pl, 2, 0, [cam])
    assert rgb[0, 0, 16, 16] == pytest.approx(ex2["C"], abs=2e-6)
    assert T[0, 16, 16] == pytest.approx(ex2["T"], abs=2e-6)


def test_empty_scene():
    cam = identity_camera(40, 24, 30.0)
    pl = planes_from([[0, 0, -5.0]], [[1, 0, 0, 0]], [[-3] * 3], [2.0], [sh_for_rgb((1, 1, 1), 0)], 0)
    proj, bins, rgb, T = oracle.render(pl, 1, 0, [cam], bg=(0.25, 0.5, 1.0))
    assert bins["K"] == 0
    assert np.all(T == 1.0)
    assert np.all(rgb[0, 0] == 0.25) and np.all(rgb[0, 1] == 0.5) and np.all(rgb[0, 2] == 1.0)


def _check_bins(proj, bins, W, H):
    V, n_pad = proj["tiles"].shape
    gx, gy = (W + 15) // 16, (H + 15) // 16
    T = gx * gy
    K = bins["K"]
    assert K == int(proj["tiles"].astype(np.int64).sum())
    off = np.concatenate([[0], np.cumsum(proj["tiles"].reshape(-1).astype(np.int64))[:-1]])
    assert np.array_equal(bins["offsets"].reshape(-1).astype(np.int64), off)
    keys, vals = bins["keys"].astype(np.uint64), bins["vals"]
    # sorted by (key, val): numpy lexsort of the emitted pairs (independent sort)
    order = np.lexsort((bins["vals_emit"], bins["keys_emit"]))
    assert np.array_equal(keys, bins["keys_emit"][order]) and np.array_equal(vals, bins["vals_emit"][order])
    gt = (keys >> np.uint64(31)).astype(np.int64)
    dep = (keys & np.uint64(0x7FFFFFFF)).astype(np.uint32)
    v = gt // T
    t = gt % T
    tx, ty = t % gx, t // gx
    r = proj["rect"][v, vals]
    assert np.all((tx >= r[:, 0]) & (tx <= r[:, 2]) & (ty >= r[:, 1]) & (ty <= r[:, 3]))
    assert np.array_equal(dep, proj["depth"][v, vals])
    rg = bins["ranges"].astype(np.int64)
    assert int((rg[:, 1] - rg[:, 0]).sum()) == K
    for g in np.nonzero(rg[:, 1] > rg[:, 0])[0][:200]:
        assert np.all(gt[rg[g, 0]:rg[g, 1]] == g)
    # brute-force rect enumeration: every (view, Gaussian, tile) appears exactly once
    cnt = np.zeros((V, n_pad), np.int64)
    np.add.at(cnt, (v, vals), 1)
    assert np.array_equal(cnt, proj["tiles"].astype(np.int64))


@pytest.mark.parametrize("seed_n", [(0, 1000), (1, 337)])
def test_tiny_bins_and_tiled_equals_bruteforce(seed_n):
    seed, n = seed_n
    cfg = synth.get_config("tiny", index=seed)
    sc = synth.make_scene(cfg, n=n)
    cams = synth.make_cameras(cfg)
    W, H = cams[0].width, cams[0].height
    proj, bins, rgb, T = oracle.render(sc.planes, sc.n, sc.deg, cams)
    _check_bins(proj, bins, W, H)
    rgb_b, T_b = oracle.rasterize_bruteforce(proj, sc.n, W, H)
    assert np.array_equal(rgb, rgb_b) and np.array_equal(T, T_b)  # bit-for-bit
    assert np.all((T > 0) & (T <= 1))
    assert T.min() < 0.5  # non-trivial coverage


def test_tiled_equals_bruteforce_large_gaussians_ragged_image():
    """Big / off-screen / near-plane Gaussians on a ragged 70x45 image (partial tiles)."""
    rng = np.random.default_rng(7)
    n = 300
    pos = np.stack([rng.uniform(-3, 3, n), rng.uniform(-2, 2, n), rng.uniform(0.1, 6, n)], 1)
    quat = rng.standard_normal((n, 4))
    ls = rng.normal(math.log(0.15), 0.8, (n, 3))
    opl = rng.normal(0, 2.5, n)
    sh = rng.normal(0, 0.5, (n, 16, 3))
    pl = planes_from(pos, quat, ls, opl, sh, 3)
    cam = synth.make_camera(np.eye(3), np.zeros(3), 40.0, 40.0, 70, 45)
    proj, bins, rgb, T = oracle.render(pl, n, 3, [cam])
    _check_bins(proj, bins, 70, 45)
    rgb_b, T_b = oracle.rasterize_bruteforce(proj, n, 70, 45)
    assert np.array_equal(rgb, rgb_b) and np.array_equal(T, T_b)


def test_transmittance_monotone_and_alpha_bound():
    cfg = synth.get_config("tiny")
    sc = synth.make_scene(cfg)
    cams = synth.make_cameras(cfg)
    proj, bins, rgb, T = oracle.render(sc.planes, sc.n, sc.deg, cams)
    # accumulated alpha 1 - T in [0, 1); colour bounded by max rgb * (1 - T)
    assert np.all(T <= 1) and np.all(T > 0)
    cmax = proj["rec"][0, :, 9:12].max()
    assert np.all(rgb[0] <= cmax * (1 - T[0]) * (1 + 1e-5) + 1e-7)
    # prefix renders: compositing only the first j entries of every tile list can only lower T
    r2 = dict(bins)
    prev = np.ones_like(T)
    for frac in (0.25, 0.5, 0.75, 1.0):
        rg = bins["ranges"].astype(np.int64).copy()
        rg[:, 1] = rg[:, 0] + np.floor((rg[:, 1] - rg[:, 0]) * frac).astype(np.int64)
        r2["ranges"] = rg.astype(np.uint32)
        _, Tj = oracle.rasterize(proj, r2, cams[0].width, cams[0].height)
        assert np.all(Tj <= prev)
        prev = Tj


@pytest.mark.parametrize("deg", [0, 3])
def test_oracle_vs_float64_textbook_renderer(deg):
    """Eq. 1-2 in float64 (independent code) vs the fp32 oracle: PSNR > 60 dB, max-abs small."""
    cfg = synth.get_config("tiny", deg=deg, lat=(8, 8, 8, 8, 8 if deg else 0))
    sc = synth.make_scene(cfg)
    cam = synth.make_cameras(cfg)[0]
    proj, bins, rgb, T = oracle.render(sc.planes, sc.n, deg, [cam])
    ref, Tref = ref64.render64(sc.planes, sc.n, deg, cam)
    a = np.clip(rgb[0], 0, 1).astype(np.float64)
    b = np.clip(ref, 0, 1)
    mse = np.mean((a - b) ** 2)
    psnr = 10 * math.log10(1.0 / max(mse, 1e-20))
    assert psnr > 60.0, psnr
    assert np.abs(T[0] - Tref).max() < 2e-2
    # projected footprint vs float64 Eq. 1 for every non-culled Gaussian
    pr = ref64.project64(sc.planes, sc.n, deg, cam)
    live = proj["rec"][0, : sc.n, 8] > 0
    assert np.array_equal(live, pr["valid"])
    rec = proj["rec"][0, : sc.n][live]
    con = pr["conic"][live]
    assert np.allclose(rec[:, 4], -0.5 * L2E * con[:, 0, 0], rtol=1e-4, atol=1e-7)
    assert np.allclose(rec[:, 5], -L2E * con[:, 0, 1], rtol=1e-4, atol=1e-6)
    assert np.allclose(rec[:, 6], -0.5 * L2E * con[:, 1, 1], rtol=1e-4, atol=1e-7)
    assert np.allclose(rec[:, 0], pr["u"][live], rtol=1e-6, atol=1e-4)
    assert np.allclose(rec[:, 9:12], pr["rgb"][:, live].T, rtol=1e-5, atol=1e-6)
    # extent: hx = sqrt(2 ln(255 o) S'_xx) (tight bounding box of the alpha = 1/255 ellipse), 1e-4 slack
    e2 = 2 * np.log(255 * pr["o"][live])
    assert np.allclose(rec[:, 2], 1.0001 * np.sqrt(e2 * pr["S2"][live, 0, 0]), rtol=1e-4)
    assert np.allclose(rec[:, 3], 1.0001 * np.sqrt(e2 * pr["S2"][live, 1, 1]), rtol=1e-4)


def test_extent_contains_every_contributing_pixel():
    """Every pixel whose (fp32) p2 >= T2 lies within [u +- hx] x [v +- hy] (the blend's cull box)
    and inside the Gaussian's tile rect: brute force over all pixels of a ragged image."""
    rng = np.random.default_rng(9)
    n = 400
    pos = np.stack([rng.uniform(-2, 2, n), rng.uniform(-1.5, 1.5, n), rng.uniform(1.0, 5, n)], 1)
    pl = planes_from(pos, rng.standard_normal((n, 4)), rng.normal(math.log(0.08), 0.9, (n, 3)),
                     rng.normal(1, 2.5, n), rng.normal(0, 0.5, (n, 1, 3)), 0)
    cam = synth.make_camera(np.eye(3), np.zeros(3), 50.0, 50.0, 90, 61)
    pr = oracle.project(pl, n, 0, [cam])
    rec = pr["rec"][0, :n].astype(np.float32)
    ys, xs = np.mgrid[0:61, 0:90]
    xs = xs.reshape(-1).astype(np.float32)
    ys = ys.reshape(-1).astype(np.float32)
    for i in np.nonzero(rec[:, 8] > 0)[0]:
        r = rec[i]
        dx = (r[0] - xs).astype(np.float32)
        dy = (r[1] - ys).astype(np.float32)
        p2 = (r[4] * dx).astype(np.float32) * dx + ((r[6] * dy).astype(np.float32) * dy + (r[5] * dx).astype(np.float32) * dy)
        hit = (p2 >= r[7] - 1e-4) & (p2 <= 1e-6)
        assert np.all(np.abs(dx[hit]) <= r[2]) and np.all(np.abs(dy[hit]) <= r[3])
        tx, ty = (xs[hit] // 16).astype(int), (ys[hit] // 16).astype(int)
        rc = pr["rect"][0, i]
        assert np.all((tx >= rc[0]) & (tx <= rc[2]) & (ty >= rc[1]) & (ty <= rc[3]))


# ---------------------------------------------------------------------------------------------
# Pins for the sampled-pixel rasterizers and the blend work counters (VERDICT r1 "What's
# missing" 3).  rasterize_pixels / rasterize_pixels_direct must equal the full tiled rasterizer
# bit for bit at every pixel they are asked for; blend_counts must be 0 on an empty scene, equal
# hand-counted values on one-tile scenes, and agree with a recount from the contributor lists.
# ---------------------------------------------------------------------------------------------
def _ragged_scene(seed, n=300, W=70, H=45, needle=False):
    rng = np.random.default_rng(seed)
    pos = np.stack([rng.uniform(-3, 3, n), rng.uniform(-2, 2, n), rng.uniform(0.1, 6, n)], 1)
    quat = rng.standard_normal((n, 4))
    if needle:
        # needle ellipses: one long axis, two ~100x shorter ones
        ls = np.stack([rng.normal(math.log(0.4), 0.3, n), rng.normal(math.log(0.003), 0.3, n),
                       rng.normal(math.log(0.003), 0.3, n)], 1)
        ls = ls[np.arange(n)[:, None], np.argsort(rng.random((n, 3)), 1)]  # long axis in any slot
    else:
        ls = rng.normal(math.log(0.15), 0.8, (n, 3))
    opl = rng.normal(1.0, 2.5, n)
    sh = rng.normal(0, 0.5, (n, 16, 3))
    pl = planes_from(pos, quat, ls, opl, sh, 3)
    cam = synth.make_camera(np.eye(3), np.zeros(3), 40.0, 40.0, W, H)
    return pl, n, cam


def _all_pixels(V, W, H):
    v, y, x = np.meshgrid(np.arange(V), np.arange(H), np.arange(W), indexing="ij")
    return np.stack([v.reshape(-1), x.reshape(-1), y.reshape(-1)], 1).astype(np.int32)


@pytest.mark.parametrize("case", ["tiny", "ragged", "needle"])
def test_rasterize_pixels_and_direct_equal_full_rasterizer(case):
    if case == "tiny":
        cfg = synth.get_config("tiny")
        sc = synth.make_scene(cfg, n=337)
        cams = synth.make_cameras(cfg)
        pl, n, deg = sc.planes, sc.n, sc.deg
    else:
        pl, n, cam = _ragged_scene(11, needle=(case == "needle"))
        cams, deg = [cam, synth.make_camera(np.eye(3), np.array([0.3, -0.1, 0.5]), 40.0, 40.0, 70, 45)], 3
    W, H = cams[0].width, cams[0].height
    proj, bins, rgb, T = oracle.render(pl, n, deg, cams, bg=(0.1, 0.2, 0.3))
    pix = _all_pixels(len(cams), W, H)
    r1, T1 = oracle.rasterize_pixels(proj["rec"], bins["ranges"], bins["vals"], W, H, pix, bg=(0.1, 0.2, 0.3))
    r2, T2 = oracle.rasterize_pixels_direct(proj, n, W, H, pix, bg=(0.1, 0.2, 0.3))
    full_rgb = rgb[pix[:, 0], :, pix[:, 2], pix[:, 1]]
    full_T = T[pix[:, 0], pix[:, 2], pix[:, 1]]
    for r, t in ((r1, T1), (r2, T2)):
        assert np.array_equal(r.view(np.uint32), full_rgb.view(np.uint32))
        assert np.array_equal(t.view(np.uint32), full_T.view(np.uint32))
    assert T.min() < 0.5  # the scene covers pixels non-trivially
    # a random subset in a shuffled order gives the same values (no state between pixels)
    sel = np.random.default_rng(3).permutation(pix.shape[0])[:500]
    r3, T3 = oracle.rasterize_pixels_direct(proj, n, W, H, pix[sel], bg=(0.1, 0.2, 0.3))
    assert np.array_equal(r3, full_rgb[sel]) and np.array_equal(T3, full_T[sel])


@pytest.mark.parametrize("seed", range(6))
def test_needle_ellipses_tiled_equals_bruteforce(seed):
    """R13 (opacity-aware bounding box) must hold for needle-shaped footprints too: the tiled
    result equals brute force over all Gaussians bit for bit (VERDICT r1 weak 1 probe)."""
    pl, n, cam = _ragged_scene(100 + seed, n=250, W=83, H=57, needle=True)
    proj, bins, rgb, T = oracle.render(pl, n, 3, [cam])
    _check_bins(proj, bins, 83, 57)
    rgb_b, T_b = oracle.rasterize_bruteforce(proj, n, 83, 57)
    assert np.array_equal(rgb, rgb_b) and np.array_equal(T, T_b)
    assert T.min() < 0.9


def test_blend_counts_empty_scene():
    cam = identity_camera(40, 24, 30.0)
    pl = planes_from([[0, 0, -5.0]], [[1, 0, 0, 0]], [[-3] * 3], [2.0], [sh_for_rgb((1, 1, 1), 0)], 0)
    proj, bins, _, _ = oracle.render(pl, 1, 0, [cam])
    ev, cp = oracle.blend_counts(proj, bins, 40, 24)
    assert ev.tolist() == [0] and cp.tolist() == [0]


def test_blend_counts_one_tile_hand_counted():
    """16x16 image = one tile.  (a) One small isotropic Gaussian: every pixel evaluates its single
    entry (E = 256); the composited pixels are those with alpha >= 1/255, counted in float64 from
    the textbook projection (tests/ref64.py) on a scene whose pixels all sit far from the
    threshold.  (b) Three coincident, near-opaque, very wide Gaussians: alpha clamps to 0.99 at
    every pixel, T = 0.01 after the first and 0.01^2 < 1e-4 after the second, so every pixel
    stops there: E = Cp = 2 x 256."""
    cam = identity_camera(16, 16, 40.0, cx=7.3, cy=8.6)
    pl = planes_from([[0.0, 0.0, 4.0]], [[1, 0, 0, 0]], [[math.log(0.25)] * 3], [logit(0.8)],
                     [sh_for_rgb((0.5, 0.5, 0.5), 0)], 0)
    proj, bins, _, _ = oracle.render(pl, 1, 0, [cam])
    ev, cp = oracle.blend_counts(proj, bins, 16, 16)
    pr = ref64.project64(pl, 1, 0, cam)
    ys, xs = np.mgrid[0:16, 0:16]
    dx, dy = xs - pr["u"][0], ys - pr["v"][0]
    cn = pr["conic"][0]
    alpha = pr["o"][0] * np.exp(-0.5 * (cn[0, 0] * dx * dx + 2 * cn[0, 1] * dx * dy + cn[1, 1] * dy * dy))
    assert np.abs(np.log(alpha * 255.0)).min() > 0.01  # no pixel near the skip threshold
    n_hit = int((alpha >= 1 / 255).sum())
    assert 0 < n_hit < 256
    assert ev.tolist() == [256] and cp.tolist() == [n_hit]
    pl3 = planes_from([[0.0, 0.0, 4.0]] * 3, [[1, 0, 0, 0]] * 3, [[math.log(500.0)] * 3] * 3,
                      [logit(0.9999)] * 3, [sh_for_rgb((0.5, 0.5, 0.5), 0)] * 3, 0)
    proj, bins, _, T = oracle.render(pl3, 3, 0, [cam])
    ev, cp = oracle.blend_counts(proj, bins, 16, 16)
    assert bins["K"] == 3 and np.all(T < 1e-4)
    assert ev.tolist() == [512] and cp.tolist() == [512]


@pytest.mark.parametrize("case", ["tiny", "ragged"])
def test_blend_counts_equal_contributor_recount(case):
    """Cp = number of contributors of every pixel; E = per pixel the tile-list length, or, where
    compositing stopped (T < 1e-4), the list position of the last contributor + 1."""
    if case == "tiny":
        cfg = synth.get_config("tiny")
        sc = synth.make_scene(cfg)
        cams = synth.make_cameras(cfg)
        pl, n, deg = sc.planes, sc.n, sc.deg
    else:
        pl, n, cam = _ragged_scene(21, n=400)
        # a wall of opaque Gaussians makes many pixels terminate early
        wall = planes_from([[0.0, 0.0, 0.5]] * 4, [[1, 0, 0, 0]] * 4, [[math.log(3.0)] * 3] * 4, [logit(0.999)] * 4,
                           [sh_for_rgb((0.2, 0.4, 0.6), 3)] * 4, 3)
        pl = np.concatenate([pl[:, :n], wall[:, :4]], 1)
        n += 4
        cams, deg = [cam, synth.make_camera(np.eye(3), np.array([0.2, 0.1, 0.0]), 40.0, 40.0, 70, 45)], 3
    W, H = cams[0].width, cams[0].height
    proj, bins, rgb, T = oracle.render(pl, n, deg, cams)
    ev, cp = oracle.blend_counts(proj, bins, W, H)
    off, gid, _ = oracle.contributors(proj, bins, W, H)
    cnt = np.diff(off)
    V = len(cams)
    gx = (W + 15) // 16
    Tt = gx * ((H + 15) // 16)
    ev_re = np.zeros(V, np.int64)
    stopped_any = False
    for v in range(V):
        for y in range(H):
            for x in range(W):
                p = (v * H + y) * W + x
                a, b = bins["ranges"][v * Tt + (y >> 4) * gx + (x >> 4)]
                if T[v, y, x] < 1e-4:
                    stopped_any = True
                    last = gid[off[p + 1] - 1]
                    pos = np.nonzero(bins["vals"][a:b] == last)[0]
                    assert pos.size == 1
                    ev_re[v] += int(pos[0]) + 1
                else:
                    ev_re[v] += int(b) - int(a)
    assert cp.tolist() == cnt.reshape(V, -1).sum(1).tolist()
    assert ev.tolist() == ev_re.tolist()
    assert np.all(cp <= ev) and cp.sum() > 0
    if case == "ragged":
        assert stopped_any
