"""GPU (libqueen, sm_100a) vs CPU oracle parity, element by element, on seeded inputs.

Bars (BASELINE north_star):
  bit-exact  : quantised latents, gate mask / COO indices, projection records except
               rgb (u, v, A2, B2, C2, T2, o, depth, tiles, rect), K, sorted keys,
               vals, ranges
  tolerance  : decoded attributes |d| <= 1e-5 max(|ref|, 1e-6) (bit-exact expected);
               per-Gaussian rgb 1e-5 relative; image RGB max-abs <= 2e-3 on [0,1],
               PSNR > 60 dB; T max-abs <= 2e-3
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from harness import synth  # noqa: E402
from tests.util import planes_from  # noqa: E402

RGB_TOL = 2e-3
ATTR_REL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run with -m 'not gpu' on CPU)")
    import paper_2412_04469_b200 as Q
    Q.lib()  # loud failure if the extension was not built


def _attr_close(got, ref):
    got = got.astype(np.float64)
    ref = ref.astype(np.float64)
    return np.all(np.abs(got - ref) <= ATTR_REL * np.maximum(np.abs(ref), 1e-6))


def _scene(name, n=None, **over):
    cfg = synth.get_config(name, **over)
    return cfg, synth.make_scene(cfg, n)


# ------------------------------------------------------------------ decode / apply
@pytest.mark.parametrize("name,n", [("tiny", 1000), ("n3dv", 20011), ("immersive", 5003)])
@pytest.mark.parametrize("f32", [False, True])
def test_decode_residuals_parity(name, n, f32):
    import paper_2412_04469_b200 as Q
    from paper_2412_04469_b200.runtime import device_packet
    cfg, sc = _scene(name, n)
    pkt = synth.make_packet(sc, 1)
    ref = oracle.decode(pkt)
    ctx = Q.Context(0)
    ctx.set_workspace(sc.n_pad, 1, 16, 16, 1024)
    dp = device_packet(pkt, "cuda", gates=True, f32_latents=f32)
    resid = torch.zeros(ref.shape, dtype=torch.float32, device="cuda")
    q = torch.zeros(pkt.latents.shape, dtype=torch.int8, device="cuda")
    idx = torch.zeros(max(sc.n, 1), dtype=torch.int32, device="cuda")
    val = torch.zeros((3, max(sc.n, 1)), dtype=torch.float32, device="cuda")
    k = torch.zeros(1, dtype=torch.int32, device="cuda")
    Q.queen_decode_residuals(ctx, dp.struct, resid, q, idx, val, k)
    st, _ = ctx.check_status()
    assert st == 0
    r = resid.cpu().numpy()
    assert _attr_close(r[:, : sc.n], ref[:, : sc.n])
    assert np.array_equal(r[:, : sc.n].view(np.uint32), ref[:, : sc.n].view(np.uint32))  # expected bit-identical
    qref, bad = oracle.quantize(pkt.latents_f32) if f32 else (pkt.latents, 0)
    assert np.array_equal(q.cpu().numpy()[:, : sc.n], qref[:, : sc.n])
    oi, ov = oracle.gate(pkt)
    kk = int(k.item())
    assert kk == oi.shape[0]
    assert np.array_equal(idx.cpu().numpy()[:kk].view(np.uint32), oi)
    gv = val.cpu().numpy()[:, :kk]
    assert np.array_equal(gv.view(np.uint32), ov.view(np.uint32))


@pytest.mark.parametrize("mode", ["coo_int8", "gates_f32"])
@pytest.mark.parametrize("name,n", [("tiny", 1000), ("n3dv", 30001), ("stress", 4099)])
def test_apply_frame_parity(mode, name, n):
    from tests.gpu_helpers import gpu_apply
    cfg, sc = _scene(name, n)
    pkt = synth.make_packet(sc, 2)
    gates = mode.startswith("gates")
    f32 = mode.endswith("f32")
    ref, st, _ = oracle.apply(sc.planes, pkt, use_gates=gates, use_f32_latents=f32)
    got, gst = gpu_apply(sc.planes, pkt, gates=gates, f32=f32)
    assert st == 0 and gst == 0
    assert _attr_close(got[:, : sc.n], ref[:, : sc.n])
    assert np.array_equal(got[:, : sc.n].view(np.uint32), ref[:, : sc.n].view(np.uint32))
    assert np.array_equal(got[:, sc.n:], sc.planes[:, sc.n:])  # padding untouched


def test_dyadic_stream_exact_on_gpu():
    """Drift-free streaming: 10 frames of dyadic packets, GPU == int64 closed form (exact)."""
    from tests.gpu_helpers import gpu_apply
    cfg = synth.get_config("n3dv")
    sc = synth.make_dyadic_scene(cfg, n=5000)
    pkts = [synth.make_packet(sc, t, dyadic=True) for t in range(1, 11)]
    got, st = gpu_apply(sc.planes, pkts[0], frames_pkts=pkts)
    A = sc.planes.copy()
    for p in pkts:
        A, s, _ = oracle.apply(A, p)
    assert st == 0
    assert np.array_equal(got, A)


def test_zero_residual_keeps_scene():
    from tests.gpu_helpers import gpu_apply
    cfg, sc = _scene("n3dv", 10000)
    pkt = synth.zero_packet(sc)
    got, st = gpu_apply(sc.planes, pkt)
    assert st == 0 and np.array_equal(got, sc.planes)


def test_device_errors_reported():
    from tests.gpu_helpers import gpu_apply
    cfg, sc = _scene("tiny")
    pkt = synth.make_packet(sc, 1)
    pkt.coo_idx = pkt.coo_idx.copy()
    pkt.coo_idx[3] = pkt.coo_idx[2]  # not strictly increasing
    _, st = gpu_apply(sc.planes, pkt)
    assert st == -3
    pkt = synth.make_packet(sc, 1)
    pkt.coo_idx = pkt.coo_idx.copy()
    pkt.coo_idx[-1] = sc.n  # out of range
    _, st = gpu_apply(sc.planes, pkt)
    assert st == -3
    pkt = synth.make_packet(sc, 1)
    pkt.latents_f32[2, 5] = 200.0
    _, st = gpu_apply(sc.planes, pkt, f32=True)
    assert st == -4


# ------------------------------------------------------------------ render stages
def _render_case(name, n=None, views=None, **over):
    cfg, sc = _scene(name, n, **over)
    cams = synth.make_cameras(cfg, views)
    return cfg, sc, cams


def _check_proj(got, ref, n):
    for key in ("depth", "tiles", "rect"):
        assert np.array_equal(got[key][:, :n], ref[key][:, :n]), key
    g, r = got["rec"][:, :n], ref["rec"][:, :n]
    assert np.array_equal(g[..., :9].view(np.uint32), r[..., :9].view(np.uint32))  # u v hx hy A2 B2 C2 T2 o
    assert np.all(np.abs(g[..., 9:] - r[..., 9:]) <= 1e-5 * np.maximum(np.abs(r[..., 9:]), 1e-6) + 1e-7)


def _check_bins(got, ref, depth=None, T=None):
    """Sorted entries bit-exact: gt, Gaussian index, ranges, K; and the full composite key
    (gt << 31 | depth bits) rebuilt from the entry equals the oracle's sorted key."""
    assert got["K"] == ref["K"]
    assert np.array_equal(got["keys"].astype(np.uint64), ref["keys"] >> np.uint64(31))
    assert np.array_equal(got["vals"], ref["vals"])
    assert np.array_equal(got["ranges"], ref["ranges"])
    if depth is not None:
        v = got["keys"].astype(np.int64) // T
        full = (got["keys"].astype(np.uint64) << np.uint64(31)) | depth[v, got["vals"]].astype(np.uint64)
        assert np.array_equal(full, ref["keys"])


def _check_image(rgb, T, rref, Tref):
    a, b = np.clip(rgb, 0, 1), np.clip(rref, 0, 1)
    from tests.gpu_helpers import psnr
    err = np.abs(a - b).max()
    assert err <= RGB_TOL, err
    assert np.abs(T - Tref).max() <= RGB_TOL
    assert psnr(a, b) > 60.0


@pytest.mark.parametrize("case", [("tiny", None, None, {}),
                                  ("tiny", 337, None, {"index": 7}),
                                  ("n3dv", 20003, 3, {"width": 333, "height": 250, "focal": 280.0}),
                                  ("immersive", 12001, 5, {"width": 320, "height": 240, "focal": 160.0}),
                                  ("meetroom", 8000, 13, {"width": 160, "height": 90, "focal": 125.0})])
def test_render_stages_parity(case):
    from tests.gpu_helpers import Stages
    name, n, views, over = case
    cfg, sc, cams = _render_case(name, n, views, **over)
    W, H = cams[0].width, cams[0].height
    proj, bins, rgb, T = oracle.render(sc.planes, sc.n, sc.deg, cams)
    st = Stages(sc.planes, sc.n, sc.deg, cams).run()
    gp = st.proj_np()
    _check_proj(gp, proj, sc.n)
    gb = st.bins_np()
    _check_bins(gb, bins, gp["depth"], st.T)
    assert gb["M"] == int(np.count_nonzero(proj["tiles"]))
    g_rgb, g_T = st.image_np()
    _check_image(g_rgb, g_T, rgb, T)
    s, _ = st.ctx.check_status()
    assert s == 0


def test_render_big_gaussians_ragged():
    """Large, overlapping, off-screen and near-plane Gaussians; ragged 70x45 image; degree 3."""
    from tests.gpu_helpers import Stages
    rng = np.random.default_rng(11)
    n = 2001
    pos = np.stack([rng.uniform(-3, 3, n), rng.uniform(-2, 2, n), rng.uniform(0.1, 6, n)], 1)
    pl = planes_from(pos, rng.standard_normal((n, 4)), rng.normal(math.log(0.15), 0.8, (n, 3)), rng.normal(0, 2.5, n),
                     rng.normal(0, 0.5, (n, 16, 3)), 3)
    cams = [synth.make_camera(np.eye(3), np.zeros(3), 40.0, 40.0, 70, 45)]
    proj, bins, rgb, T = oracle.render(pl, n, 3, cams, bg=(0.1, 0.2, 0.3))
    st = Stages(pl, n, 3, cams).run(bg=(0.1, 0.2, 0.3))
    gp = st.proj_np()
    _check_proj(gp, proj, n)
    _check_bins(st.bins_np(), bins, gp["depth"], st.T)
    _check_image(*st.image_np(), rgb, T)


def test_empty_and_all_culled():
    from tests.gpu_helpers import Stages
    pl = planes_from([[0, 0, -5.0]] * 8, [[1, 0, 0, 0]] * 8, [[-3] * 3] * 8, [2.0] * 8,
                     [np.zeros((1, 3))] * 8, 0)
    cams = [synth.make_camera(np.eye(3), np.zeros(3), 30.0, 30.0, 40, 24)]
    st = Stages(pl, 8, 0, cams).run(bg=(0.25, 0.5, 1.0))
    rgb, T = st.image_np()
    assert st.bins_np()["K"] == 0
    assert np.all(T == 1.0) and np.all(rgb[0, 0] == 0.25) and np.all(rgb[0, 2] == 1.0)


def test_nonfinite_warns_and_culls():
    from tests.gpu_helpers import Stages
    cfg, sc, cams = _render_case("tiny")
    pl = sc.planes.copy()
    pl[8, 10] = np.inf
    pl[20 % pl.shape[0], 11] = np.nan
    proj, bins, rgb, T = oracle.render(pl, sc.n, sc.deg, cams)
    st = Stages(pl, sc.n, sc.deg, cams).run()
    s, _ = st.ctx.check_status()
    assert s == 1  # QUEEN_WARN_NONFINITE
    _check_proj(st.proj_np(), proj, sc.n)
    _check_image(*st.image_np(), rgb, T)


def test_capacity_error_reports_needed_keys():
    from tests.gpu_helpers import Stages
    cfg, sc, cams = _render_case("tiny")
    proj, bins, rgb, T = oracle.render(sc.planes, sc.n, sc.deg, cams)
    st = Stages(sc.planes, sc.n, sc.deg, cams, keys_cap=max(1, bins["K"] // 2)).run()
    s, info = st.ctx.check_status()
    assert s == -5 and info == bins["K"]
    assert st.bins_np()["K"] == 0  # nothing emitted, every range empty
    assert not np.any(st.ranges.cpu().numpy())


def test_long_tile_lists():
    """Very long tile lists (thousands of entries; several onesweep tiles per gt): 12000 small
    Gaussians crowded into a 40x36 image, 30 % of them at one shared depth (ties broken by
    index)."""
    from tests.gpu_helpers import Stages
    rng = np.random.default_rng(23)
    n = 12000
    z = np.where(rng.random(n) < 0.3, 2.0, rng.uniform(1.0, 4.0, n))  # 30 % share one depth
    pos = np.stack([rng.normal(0, 0.08, n) * z, rng.normal(0, 0.08, n) * z, z], 1)
    pl = planes_from(pos, rng.standard_normal((n, 4)), rng.normal(math.log(0.01), 0.3, (n, 3)), rng.normal(-1, 1, n),
                     rng.normal(0, 0.5, (n, 1, 3)), 0)
    cams = [synth.make_camera(np.eye(3), np.zeros(3), 60.0, 60.0, 40, 36)]
    proj, bins, rgb, T = oracle.render(pl, n, 0, cams)
    lens = np.diff(bins["ranges"].astype(np.int64), axis=1)
    assert lens.max() > 4096 and np.any((lens > 256) & (lens <= 4096))
    st = Stages(pl, n, 0, cams).run()
    gp = st.proj_np()
    _check_proj(gp, proj, n)
    _check_bins(st.bins_np(), bins, gp["depth"], st.T)
    _check_image(*st.image_np(), rgb, T)


def test_render_views_equals_stages_and_deterministic():
    import paper_2412_04469_b200 as Q
    from paper_2412_04469_b200.runtime import Player
    from tests.gpu_helpers import Stages
    cfg, sc, cams = _render_case("n3dv", 20003, 4, width=200, height=150, focal=170.0)
    st = Stages(sc.planes, sc.n, sc.deg, cams).run()
    rgb_s, T_s = st.image_np()
    pl = Player(sc.planes, sc.n, sc.deg, cams, with_T=True)
    pl.fit_capacity()
    a = pl.render().cpu().numpy()
    b = pl.render().cpu().numpy()
    assert np.array_equal(a, rgb_s) and np.array_equal(pl.T.cpu().numpy(), T_s)
    assert np.array_equal(a, b)
    # 2 batches of 2 views == 1 batch of 4 views (bit-identical)
    pl2 = Player(sc.planes, sc.n, sc.deg, cams, views_per_batch=2)
    pl2.fit_capacity()
    assert np.array_equal(pl2.render().cpu().numpy(), a)
    assert Q.QUEEN_MAX_VIEWS == 64


def test_wire_packet_roundtrip_apply():
    """Packed wire packet (k read on device) applies exactly like the host-side COO packet."""
    from paper_2412_04469_b200 import packet as wire
    import paper_2412_04469_b200 as Q
    from paper_2412_04469_b200.runtime import wire_packet
    cfg, sc = _scene("n3dv", 9001)
    pkt = synth.make_packet(sc, 3)
    buf = wire.pack(pkt, frame=3, k_cap=pkt.k + 100)
    hdr = wire.header(buf)
    dbuf = torch.from_numpy(buf).cuda()
    dp = wire_packet(dbuf, hdr)
    ctx = Q.Context(0)
    ctx.set_workspace(sc.n_pad, 1, 16, 16, 1024)
    pl = torch.from_numpy(sc.planes.copy()).cuda()
    Q.queen_apply_frame(ctx, Q.gaussians_struct(pl, sc.n, sc.deg), dp.struct)
    s, _ = ctx.check_status()
    ref, _, _ = oracle.apply(sc.planes, pkt)
    assert s == 0 and np.array_equal(pl.cpu().numpy(), ref)


# ------------------------------------------------------------------ full-size configs (sampled)
@pytest.mark.parametrize("name", ["n3dv", "immersive", "meetroom"])
def test_full_size_frame_sampled(name):
    """BASELINE configs at full size, in bench.py's launch configuration (Player with bench's
    views per batch, frame 1 applied): SoA after apply bit-exact; projection records for all
    views bit-exact; bins bit-exact for the first batch; 4096 sampled pixels per view within
    tolerance."""
    import bench
    from paper_2412_04469_b200.runtime import Player, device_packet
    cfg = synth.get_config(name)
    sc = synth.make_scene(cfg)
    cams = synth.make_cameras(cfg)
    pkt = synth.make_packet(sc, 1)
    pl = Player(sc.planes, sc.n, sc.deg, cams, views_per_batch=min(len(cams), bench.default_vpb(cfg)))
    pl.apply(device_packet(pkt, pl.dev))
    A1, st, _ = oracle.apply(sc.planes, pkt)
    assert np.array_equal(pl.planes.cpu().numpy(), A1)
    pl.fit_capacity()
    rgb = pl.render().cpu().numpy()
    s, _ = pl.check_status()
    assert s == 0
    W, H = cams[0].width, cams[0].height
    rng = np.random.default_rng(5)
    for bi, (a, b) in enumerate(pl.batches):
        bc = cams[a:b]
        proj = oracle.project(A1, sc.n, sc.deg, bc)
        bins = oracle.bin_sort(proj, W, H)
        if bi == 0:
            from tests.gpu_helpers import Stages
            stg = Stages(A1, sc.n, sc.deg, bc, keys_cap=pl.keys_cap).project().bin_sort()
            gp = stg.proj_np()
            _check_proj(gp, proj, sc.n)
            _check_bins(stg.bins_np(), bins, gp["depth"], stg.T)
            del stg
        V = len(bc)
        pix = np.stack([np.repeat(np.arange(V), 4096), rng.integers(0, W, V * 4096), rng.integers(0, H, V * 4096)], 1)
        orgb, oT = oracle.rasterize_pixels(proj["rec"], bins["ranges"], bins["vals"], W, H, pix)
        g = rgb[a + pix[:, 0], :, pix[:, 2], pix[:, 1]]
        assert np.abs(np.clip(g, 0, 1) - np.clip(orgb, 0, 1)).max() <= RGB_TOL
        del proj, bins


def test_full_size_stress_sampled():
    """BASELINE configs[4] (3 M Gaussians, 64 views at 3840x2160) at full size in bench.py's
    launch configuration: SoA after apply bit-exact; the first batch's projection records
    bit-exact; its binning checked by properties (K = sum of tiles touched, ranges tile the
    entries, every entry's Gaussian touches its tile, per-tile lists in (depth, index) order);
    256 sampled pixels of each of the batch's views against the oracle composited straight from
    the records (no binning, R13)."""
    import bench
    from paper_2412_04469_b200.runtime import Player, device_packet
    from tests.gpu_helpers import Stages
    cfg = synth.get_config("stress")
    sc = synth.make_scene(cfg)
    cams = synth.make_cameras(cfg)
    pkt = synth.make_packet(sc, 1)
    vpb = min(len(cams), bench.default_vpb(cfg))
    pl = Player(sc.planes, sc.n, sc.deg, cams, views_per_batch=vpb)
    pl.apply(device_packet(pkt, pl.dev))
    A1, st, _ = oracle.apply(sc.planes, pkt)
    assert np.array_equal(pl.planes.cpu().numpy(), A1)
    pl.fit_capacity()
    rgb = pl.render()
    s, _ = pl.check_status()
    assert s == 0
    W, H = cams[0].width, cams[0].height
    a, b = pl.batches[0]
    bc = cams[a:b]
    proj = oracle.project(A1, sc.n, sc.deg, bc)
    stg = Stages(A1, sc.n, sc.deg, bc, keys_cap=pl.keys_cap).project().bin_sort()
    gp = stg.proj_np()
    _check_proj(gp, proj, sc.n)
    gb = stg.bins_np()
    tiles = proj["tiles"].astype(np.int64)
    assert gb["K"] == int(tiles.sum())
    lens = gb["ranges"][:, 1].astype(np.int64) - gb["ranges"][:, 0].astype(np.int64)
    assert lens.sum() == gb["K"] and np.all(gb["ranges"][1:, 0][lens[1:] > 0] >= gb["ranges"][:-1, 1][lens[1:] > 0])
    gt = gb["keys"].astype(np.int64)
    v = gt // stg.T
    t = gt % stg.T
    gx = (W + 15) // 16
    r = proj["rect"][v, gb["vals"]]
    tx, ty = t % gx, t // gx
    assert np.all((tx >= r[:, 0]) & (tx <= r[:, 2]) & (ty >= r[:, 1]) & (ty <= r[:, 3]))
    full = (gt.astype(np.uint64) << np.uint64(32)) | (proj["depth"][v, gb["vals"]].astype(np.uint64) << np.uint64(0))
    same = gt[1:] == gt[:-1]
    k2 = full * np.uint64(1)  # (gt, depth) then index: check non-decreasing (gt, depth, index)
    prev, nxt = k2[:-1], k2[1:]
    ordered = (nxt > prev) | ((nxt == prev) & (gb["vals"][1:] > gb["vals"][:-1]))
    assert np.all(ordered | ~same)
    del stg, gb, full, k2, prev, nxt, ordered, same
    rng = np.random.default_rng(8)
    V = len(bc)
    pix = np.stack([np.repeat(np.arange(V), 256), rng.integers(0, W, V * 256), rng.integers(0, H, V * 256)], 1)
    orgb, oT = oracle.rasterize_pixels_direct(proj, sc.n, W, H, pix)
    g = rgb[a + torch.from_numpy(pix[:, 0]).cuda(), :, torch.from_numpy(pix[:, 2]).cuda(),
            torch.from_numpy(pix[:, 1]).cuda()].cpu().numpy()
    assert np.abs(np.clip(g, 0, 1) - np.clip(orgb, 0, 1)).max() <= RGB_TOL


# ------------------------------------------------------------------ blend work (culling is exact)
def test_blend_warp_mask_is_exact():
    """The blend's per-warp record mask (touches(): conservative ellipse-vs-sub-tile test) only
    skips records no pixel of the warp hits: the image is bit-identical to the unmasked kernel
    (per-thread box cull only), on a scene with thin, rotated and large Gaussians."""
    from tests.gpu_helpers import Stages
    rng = np.random.default_rng(31)
    n = 6001
    pos = np.stack([rng.uniform(-2, 2, n), rng.uniform(-1.5, 1.5, n), rng.uniform(0.5, 6, n)], 1)
    scale = np.stack([rng.normal(-4.5, 1.2, n), rng.normal(-2.5, 1.0, n), rng.normal(-3, 1, n)], 1)
    pl = planes_from(pos, rng.standard_normal((n, 4)), scale, rng.normal(0.5, 2.0, n), rng.normal(0, 0.5, (n, 4, 3)), 1)
    cams = [synth.make_camera(np.eye(3), np.zeros(3), 300.0, 300.0, 333, 250)]
    st = Stages(pl, n, 1, cams).project().bin_sort().rasterize()
    rgb_a, T_a = st.image_np()
    import paper_2412_04469_b200 as Q
    st.ctx.set_options(Q.QUEEN_OPT_BLEND_NOMASK | Q.QUEEN_OPT_BLEND_GRID_ORDER)
    st.rasterize()
    rgb_b, T_b = st.image_np()
    st.ctx.set_options(0)
    assert np.array_equal(rgb_a.view(np.uint32), rgb_b.view(np.uint32))
    assert np.array_equal(T_a.view(np.uint32), T_b.view(np.uint32))
    proj, bins, rgb, T = oracle.render(pl, n, 1, cams)
    _check_image(rgb_a, T_a, rgb, T)


def test_render_tile_schedule_from_binning_is_exact():
    """queen_render_views blends with the tile schedule the binning built (k_slab_compact class
    counts + k_piece_count permutation): into NaN-filled outputs, the image equals the
    grid-order render bit for bit (so the schedule covers every tile exactly once) and the
    oracle's, for one and two view batches."""
    import paper_2412_04469_b200 as Q
    from paper_2412_04469_b200.runtime import Player
    cfg, sc, cams = _render_case("n3dv", 20003, 4, width=333, height=250, focal=280.0)
    ref_rgb, ref_T = None, None
    for vpb in (None, 2):
        pl = Player(sc.planes, sc.n, sc.deg, cams, views_per_batch=vpb, with_T=True)
        pl.fit_capacity()
        outs = []
        for opts in (0, Q.QUEEN_OPT_BLEND_GRID_ORDER):
            for c in pl.ctxs:
                c.set_options(opts)
            pl.rgb.fill_(float("nan"))
            pl.T.fill_(float("nan"))
            pl.render()
            torch.cuda.synchronize()
            outs.append((pl.rgb.clone(), pl.T.clone()))
        for c in pl.ctxs:
            c.set_options(0)
        (a_rgb, a_T), (b_rgb, b_T) = outs
        assert not torch.isnan(a_rgb).any() and not torch.isnan(a_T).any(), vpb
        assert torch.equal(a_rgb.view(torch.int32), b_rgb.view(torch.int32)), vpb
        assert torch.equal(a_T.view(torch.int32), b_T.view(torch.int32)), vpb
        if ref_rgb is None:
            ref_rgb, ref_T = a_rgb, a_T
        else:
            assert torch.equal(a_rgb.view(torch.int32), ref_rgb.view(torch.int32))
        assert pl.check_status()[0] == 0
    proj, bins, rgb, T = oracle.render(sc.planes, sc.n, sc.deg, cams)
    _check_image(ref_rgb.cpu().numpy(), ref_T.cpu().numpy(), rgb, T)


def test_blend_counts_match_oracle():
    """queen_blend_counts (the bench's roofline work counters) == the oracle's counts: evaluated
    (alive pixel x record) and composited pairs; equal up to the rare pixel whose T crosses 1e-4
    one record apart (GPU ex2.approx vs the oracle's exp2)."""
    import paper_2412_04469_b200 as Q
    from tests.gpu_helpers import Stages
    cfg, sc, cams = _render_case("n3dv", 20003, 3, width=333, height=250, focal=280.0)
    W, H = cams[0].width, cams[0].height
    proj = oracle.project(sc.planes, sc.n, sc.deg, cams)
    bins = oracle.bin_sort(proj, W, H)
    ev_o, cp_o = oracle.blend_counts(proj, bins, W, H)
    st = Stages(sc.planes, sc.n, sc.deg, cams).project().bin_sort()
    e = torch.zeros(len(cams), dtype=torch.int64, device="cuda")
    c = torch.zeros_like(e)
    Q.queen_blend_counts(st.ctx, st.proj, st.bins, cams, e, c)
    e, c = e.cpu().numpy(), c.cpu().numpy()
    assert np.all(np.abs(e - ev_o) <= 1e-4 * ev_o + 50), (e, ev_o)
    assert np.all(np.abs(c - cp_o) <= 1e-4 * cp_o + 5), (c, cp_o)


def test_view_larger_than_4k_rejected():
    """Binning keeps a view's tile grid in shared memory: an 8K view is refused with
    QUEEN_ERR_SHAPE (no silent fallback), a 4K view is accepted."""
    import paper_2412_04469_b200 as Q
    from tests.gpu_helpers import Stages
    pl = planes_from([[0, 0, 3.0]] * 4, [[1, 0, 0, 0]] * 4, [[-2] * 3] * 4, [2.0] * 4, [np.zeros((1, 3))] * 4, 0)
    big = [synth.make_camera(np.eye(3), np.zeros(3), 3000.0, 3000.0, 7680, 4320)]
    st = Stages(pl, 4, 0, big, keys_cap=4096).project()
    with pytest.raises(Q.QueenError) as ei:
        st.bin_sort()
    assert ei.value.status == -2  # QUEEN_ERR_SHAPE
    ok = [synth.make_camera(np.eye(3), np.zeros(3), 3000.0, 3000.0, 3840, 2160)]
    st = Stages(pl, 4, 0, ok, keys_cap=1 << 20).run()
    assert st.bins_np()["K"] > 0


def test_render_views_rgb8_display_format():
    """queen_render_views_rgb8 = the fp32 render quantised round-half-even(clamp(c, 0, 1) * 255)
    (GPU vs GPU: identical compositing, so bit-exact), and within 1 LSB of the oracle."""
    from paper_2412_04469_b200.runtime import Player
    cfg, sc, cams = _render_case("n3dv", 20003, 3, width=333, height=250, focal=280.0)
    pl = Player(sc.planes, sc.n, sc.deg, cams, bg=(0.2, 0.4, 0.6))
    pl.fit_capacity()
    f32 = pl.render().clone()
    u8 = torch.empty(f32.shape, dtype=torch.uint8, device="cuda")
    pl.render(out=u8, rgb8=True)
    q = torch.round(torch.clamp(f32, 0, 1) * 255.0).to(torch.uint8)  # torch.round: half to even
    assert torch.equal(u8, q)
    _, _, ref, _ = oracle.render(sc.planes, sc.n, sc.deg, cams, bg=(0.2, 0.4, 0.6))
    ref8 = np.rint(np.clip(ref, 0, 1) * np.float32(255)).astype(np.int16)
    assert np.abs(u8.cpu().numpy().astype(np.int16) - ref8).max() <= 1


def test_render_views_f16_output():
    """queen_render_views_f16 = the fp32 render rounded to nearest binary16 (GPU vs GPU: identical
    compositing, bit-exact), and within the 2e-3 RGB bar of the oracle (binary16 adds <= 2^-11)."""
    from paper_2412_04469_b200.runtime import Player
    cfg, sc, cams = _render_case("n3dv", 20003, 3, width=333, height=250, focal=280.0)
    pl = Player(sc.planes, sc.n, sc.deg, cams, bg=(0.2, 0.4, 0.6))
    pl.fit_capacity()
    f32 = pl.render().clone()
    h = torch.empty(f32.shape, dtype=torch.float16, device="cuda")
    pl.render(out=h)
    assert torch.equal(h, f32.to(torch.float16))  # torch: round to nearest even
    _, _, ref, _ = oracle.render(sc.planes, sc.n, sc.deg, cams, bg=(0.2, 0.4, 0.6))
    err = np.abs(np.clip(h.float().cpu().numpy(), 0, 1) - np.clip(ref, 0, 1)).max()
    assert err <= RGB_TOL, err


def test_render_views_rgb10_output():
    """queen_render_views_rgb10 = the fp32 render packed as R10G10B10A2 (each channel
    round-half-even(clamp(x, 0, 1) * 1023) in fp32: GPU vs GPU bit-exact, also through the
    Player's two-lane step), and within the 2e-3 RGB bar of the oracle (1/2 LSB = 4.9e-4)."""
    from paper_2412_04469_b200.runtime import Player
    cfg, sc, cams = _render_case("n3dv", 20003, 3, width=333, height=250, focal=280.0)
    bg = (0.2, 0.4, 0.6)
    pl = Player(sc.planes, sc.n, sc.deg, cams, bg=bg)
    pl.fit_capacity()
    f32 = pl.render().clone()
    V, _, H, W = f32.shape
    p10 = torch.empty((V, H, W), dtype=torch.int32, device="cuda")
    pl.render(out=p10)
    torch.cuda.synchronize()
    q = torch.round(torch.clamp(f32, 0.0, 1.0) * 1023.0).to(torch.int64)  # torch.round: half to even
    want = q[:, 0] | (q[:, 1] << 10) | (q[:, 2] << 20) | (3 << 30)
    got = p10.to(torch.int64) & 0xffffffff
    assert torch.equal(got, want)
    dec = torch.stack([(got >> (10 * c)) & 1023 for c in range(3)], 1).double() / 1023.0
    _, _, ref, _ = oracle.render(sc.planes, sc.n, sc.deg, cams, bg=bg)
    err = np.abs(dec.cpu().numpy() - np.clip(ref, 0, 1)).max()
    assert err <= RGB_TOL, err
    # the two-lane step into per-frame rgb10 buffers
    out2 = torch.empty_like(p10)
    pl.step2(None, out=out2)
    pl.sync_lanes()
    torch.cuda.synchronize()
    assert torch.equal(out2, p10)


def test_cuda_graph_frame_equals_eager():
    """A captured frame step (entropy decode + apply + render, Player.capture) replays to the
    same SoA and images, bit for bit, as the eager calls."""
    import paper_2412_04469_b200 as Q
    from paper_2412_04469_b200 import packet as wire
    from paper_2412_04469_b200.runtime import EntropyPacket, Player
    cfg, sc, cams = _render_case("n3dv", 20003, 3, width=333, height=250, focal=280.0)
    pkts = [synth.make_packet(sc, t) for t in (1, 2)]
    streams = [wire.ans_streams(p, Q.queen_entropy_encode) for p in pkts]
    cap = [max(s[c].size for s in streams) for c in range(5)]
    kc = max(p.k for p in pkts)
    bufs = [wire.pack_entropy(p, s, frame=t + 1, k_cap=kc, ans_cap=cap) for t, (p, s) in enumerate(zip(pkts, streams))]
    hdr = wire.header_entropy(bufs[0])
    slot = torch.from_numpy(bufs[0]).cuda()
    ep = EntropyPacket(slot, hdr)
    eager = Player(sc.planes, sc.n, sc.deg, cams)
    eager.fit_capacity()
    graphed = Player(sc.planes, sc.n, sc.deg, cams, keys_cap=eager.keys_cap)
    g = graphed.capture(ep)  # runs frame 1 once while warming up + capturing side effects
    graphed.planes.copy_(torch.from_numpy(sc.planes).cuda())
    for b in bufs:  # frames 1, 2: eager vs replay on the same packet slot
        slot.copy_(torch.from_numpy(b).cuda())
        eager.apply(ep)
        ref = eager.render().clone()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(graphed.planes, eager.planes)
        assert torch.equal(graphed.rgb, ref)
    assert graphed.check_status()[0] == 0


def test_pipelined_steps_equal_serial_frames():
    """Pipelined steps (Player.step / capture_step: frame t rendered while packet t+1 is decoded
    and applied on a side stream after the render's binning; Player.step2: in addition frame t+1
    binned on a second context under frame t's blend, packet t+1 applied after frame t's
    projection or binning) give, frame by frame, the same images and
    final SoA, bit for bit, as serial apply-then-render; also with two view batches (the apply
    waits for the LAST batch's binning)."""
    import paper_2412_04469_b200 as Q
    from paper_2412_04469_b200 import packet as wire
    from paper_2412_04469_b200.runtime import EntropyPacket, Player
    cfg, sc, cams = _render_case("n3dv", 20003, 3, width=333, height=250, focal=280.0)
    pkts = [synth.make_packet(sc, t) for t in range(1, 7)]  # 6 frames: 4 lanes reuse a slot
    streams = [wire.ans_streams(p, Q.queen_entropy_encode) for p in pkts]
    cap = [max(s[c].size for s in streams) for c in range(5)]
    kc = max(p.k for p in pkts)
    bufs = [wire.pack_entropy(p, s, frame=t + 1, k_cap=kc, ans_cap=cap) for t, (p, s) in enumerate(zip(pkts, streams))]
    hdr = wire.header_entropy(bufs[0])
    eps = [EntropyPacket(torch.from_numpy(b).cuda(), hdr) for b in bufs]
    for vpb in (None, 2):
        serial = Player(sc.planes, sc.n, sc.deg, cams, views_per_batch=vpb)
        serial.fit_capacity()
        refs = []
        for ep in eps:
            serial.apply(ep)
            refs.append(serial.render().clone())
        # eager pipelined steps
        pipe = Player(sc.planes, sc.n, sc.deg, cams, keys_cap=serial.keys_cap, views_per_batch=vpb)
        pipe.apply(eps[0])
        for t in range(len(eps)):
            out = pipe.step(eps[t + 1] if t + 1 < len(eps) else None, out=torch.empty_like(pipe.rgb))
            torch.cuda.synchronize()
            assert torch.equal(out, refs[t]), (vpb, t)
        assert torch.equal(pipe.planes, serial.planes)
        assert pipe.check_status()[0] == 0
        # graph replays of the pipelined step (graph j applies packet j)
        gp = Player(sc.planes, sc.n, sc.deg, cams, keys_cap=serial.keys_cap, views_per_batch=vpb)
        graphs = [gp.capture_step(ep) for ep in eps]
        gp.planes.copy_(torch.from_numpy(sc.planes).cuda())
        gp.apply(eps[0])
        for t in range(len(eps) - 1):
            graphs[t + 1].replay()
            torch.cuda.synchronize()
            assert torch.equal(gp.rgb, refs[t]), (vpb, t)
        gp.render()
        torch.cuda.synchronize()
        assert torch.equal(gp.rgb, refs[-1])
        assert gp.check_status()[0] == 0
        # two-lane steps (Player.step2): frame t+1's binning under frame t's blend, 2 contexts;
        # the next packet applied after the frame's projection (default) or after its binning
        for after, nl in (("binned", 2), ("projected", 2), ("projected", 3)):
            tl = Player(sc.planes, sc.n, sc.deg, cams, keys_cap=serial.keys_cap, views_per_batch=vpb)
            tl.apply_after, tl.frame_lanes = after, nl
            tl.apply(eps[0])
            outs = [torch.empty_like(tl.rgb) for _ in range(len(eps))]
            evs = [torch.cuda.Event() for _ in range(len(eps))]
            for t in range(len(eps)):
                tl.step2(eps[t + 1] if t + 1 < len(eps) else None, out=outs[t], rendered=evs[t])
            tl.sync_lanes()
            torch.cuda.synchronize()
            for t in range(len(eps)):
                assert torch.equal(outs[t], refs[t]), ("two-lane", after, nl, vpb, t)
            assert torch.equal(tl.planes, serial.planes)
        # out=None: the per-lane image buffers (frame t's is valid once `rendered` fires)
        tl2 = Player(sc.planes, sc.n, sc.deg, cams, keys_cap=serial.keys_cap, views_per_batch=vpb)
        tl2.apply(eps[0])
        for t in range(len(eps)):
            ev = torch.cuda.Event()
            img = tl2.step2(eps[t + 1] if t + 1 < len(eps) else None, rendered=ev)
            torch.cuda.current_stream().wait_event(ev)
            assert torch.equal(img.clone(), refs[t]), ("two-lane, own buffers", vpb, t)
        tl2.sync_lanes()
        # out=None read on a consumer stream without host syncs: `consumed` fences the reuse of
        # each lane's buffer two frames later
        for nl in (2, 4):  # per-frame-slot image buffers, reused nl frames later
            tl3 = Player(sc.planes, sc.n, sc.deg, cams, keys_cap=serial.keys_cap, views_per_batch=vpb)
            tl3.frame_lanes = nl
            tl3.apply(eps[0])
            reader = torch.cuda.Stream()
            copies = []
            for t in range(len(eps)):
                ev, done = torch.cuda.Event(), torch.cuda.Event()
                img = tl3.step2(eps[t + 1] if t + 1 < len(eps) else None, rendered=ev, consumed=done)
                reader.wait_event(ev)
                with torch.cuda.stream(reader):
                    copies.append(img.clone())
                    done.record(reader)
            tl3.sync_lanes()
            torch.cuda.synchronize()
            for t in range(len(eps)):
                assert torch.equal(copies[t], refs[t]), ("two-lane, consumer stream", nl, vpb, t)
        # a plain render after two-lane steps (the lane-0 blend ran on its own stream)
        again = tl.render().clone()
        torch.cuda.synchronize()
        assert torch.equal(again, refs[-1])
        assert tl.check_status()[0] == 0


def test_depth_keys_spanning_more_than_27_bits():
    """Depth keys relative to the smallest depth: when the scene's depths span more than 2^27
    float ulps (z from 0.3 to 1e6) the 4th depth pass (bits 27..31) is a real pass, otherwise a
    copy; the sorted entries are bit-exact either way."""
    from tests.gpu_helpers import Stages
    rng = np.random.default_rng(17)
    n = 3001
    z = np.exp(rng.uniform(np.log(0.3), np.log(1e6), n))
    pos = np.stack([rng.uniform(-0.5, 0.5, n) * z, rng.uniform(-0.4, 0.4, n) * z, z], 1)
    scale = np.log(np.maximum(0.02 * z, 1e-3))[:, None].repeat(3, 1)
    pl = planes_from(pos, rng.standard_normal((n, 4)), scale, rng.normal(1.0, 1.0, n), rng.normal(0, 0.5, (n, 1, 3)), 0)
    cams = [synth.make_camera(np.eye(3), np.zeros(3), 200.0, 200.0, 320, 240)]
    proj, bins, rgb, T = oracle.render(pl, n, 0, cams)
    d = proj["depth"][0][proj["tiles"][0] > 0].astype(np.int64)
    assert d.max() - d.min() >= (1 << 27)
    st = Stages(pl, n, 0, cams).run()
    gp = st.proj_np()
    _check_proj(gp, proj, n)
    _check_bins(st.bins_np(), bins, gp["depth"], st.T)
    _check_image(*st.image_np(), rgb, T)
