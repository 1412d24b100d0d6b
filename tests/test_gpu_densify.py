"""NEXT #2 on the GPU: queen_densify vs the oracle (bit-exact: pure data movement + exact
binary16 -> fp32 conversion), its error reporting, and a densifying stream (N changes every
frame) decoded + densified on the GPU == the oracle's sequence, then rendered."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from harness import synth  # noqa: E402
from tests.gpu_helpers import psnr  # noqa: E402


def test_densify_matches_oracle():
    import paper_2412_04469_b200 as Q
    cfg = synth.get_config("n3dv")
    sc = synth.make_scene(cfg, n=20003)
    cap = 21000
    st = synth.Scene(sc.cfg, sc.n, cap, sc.deg, sc.planes, sc.dynamic)
    d = synth.make_delta(st, 1, rem_frac=0.02, add_frac=0.03)
    ctx = Q.Context(0)
    ctx.set_workspace(cap, 1, 16, 16, 1024)
    src = torch.zeros((sc.planes.shape[0], cap), dtype=torch.float32, device="cuda")
    src[:, :sc.n_pad] = torch.from_numpy(sc.planes).cuda()
    dst = torch.full_like(src, 7.0)
    n_new = sc.n - d.rem.size + d.add.shape[1]
    Q.queen_densify(ctx, Q.gaussians_struct(src, sc.n, sc.deg), torch.from_numpy(d.rem.view(np.int32)).cuda(),
                    d.rem.size, torch.from_numpy(d.add.view(np.int16)).cuda(), d.add.shape[1],
                    Q.gaussians_struct(dst, n_new, sc.deg))
    assert ctx.check_status()[0] == 0
    ref, n_ref, s = oracle.densify(src.cpu().numpy(), sc.n, d.rem, d.add, cap)
    assert s == 0 and n_ref == n_new
    assert np.array_equal(dst.cpu().numpy().view(np.uint32), ref.view(np.uint32))


def test_densify_errors():
    import paper_2412_04469_b200 as Q
    ctx = Q.Context(0)
    ctx.set_workspace(64, 1, 16, 16, 1024)
    a = torch.zeros((14, 64), dtype=torch.float32, device="cuda")
    b = torch.zeros_like(a)
    add = torch.zeros((14, 2), dtype=torch.int16, device="cuda")
    bad = torch.tensor([5, 3], dtype=torch.int32, device="cuda")
    Q.queen_densify(ctx, Q.gaussians_struct(a, 50, 0), bad, 2, add, 2, Q.gaussians_struct(b, 50, 0))
    assert ctx.check_status()[0] == -3
    with pytest.raises(Q.QueenError) as e1:  # in place
        Q.queen_densify(ctx, Q.gaussians_struct(a, 50, 0), bad, 0, add, 2, Q.gaussians_struct(a, 52, 0))
    assert e1.value.status == -1
    with pytest.raises(Q.QueenError) as e2:  # wrong destination count
        Q.queen_densify(ctx, Q.gaussians_struct(a, 50, 0), bad, 0, add, 2, Q.gaussians_struct(b, 50, 0))
    assert e2.value.status == -2


def test_densify_bad_removals_stay_in_bounds():
    """a removal list with duplicates / out-of-range entries is flagged (-3) and must
    not write past the kept columns (into the additions) or past the destination's n_pad."""
    import paper_2412_04469_b200 as Q
    ctx = Q.Context(0)
    ctx.set_workspace(64, 1, 16, 16, 1024)
    a = torch.arange(14 * 64, dtype=torch.float32, device="cuda").reshape(14, 64)
    # destination [14][48] at the start of a larger buffer: the 64 floats after it are a guard
    big = torch.full((14 * 48 + 64,), -7.0, dtype=torch.float32, device="cuda")
    dst = big[:14 * 48].view(14, 48)
    add = torch.zeros((14, 1), dtype=torch.int16, device="cuda")  # binary16 +0.0
    # 4 "removals" of which only one is real (duplicates + out of range): 50 - 4 + 1 = 47 <= 48
    bad = torch.tensor([3, 3, 3, 999], dtype=torch.int32, device="cuda")
    g_dst = Q.gaussians_struct(dst, 47, 0)
    Q.queen_densify(ctx, Q.gaussians_struct(a, 50, 0), bad, 4, add, 1, g_dst)
    assert ctx.check_status()[0] == -3
    b = big.cpu().numpy()
    # the addition (column 46 = n_old - n_rem) is intact and nothing crossed it or n_pad
    assert np.all(b[:14 * 48].reshape(14, 48)[:, 46] == 0.0)
    assert np.all(b[14 * 48:] == -7.0)


def test_densifying_stream_matches_oracle():
    from paper_2412_04469_b200.runtime import Player, device_packet
    cfg = synth.get_config("n3dv", width=333, height=250, focal=280.0)
    sc = synth.make_scene(cfg, n=15001)
    cams = synth.make_cameras(cfg, 2)
    cap = 16000
    A = np.zeros((sc.planes.shape[0], cap), np.float32)
    A[:, :sc.n_pad] = sc.planes
    pl = Player(A, sc.n, sc.deg, cams, n_cap=cap)
    st = synth.Scene(sc.cfg, sc.n, cap, sc.deg, None, sc.dynamic)
    n = sc.n
    for t in range(1, 7):
        pkt = synth.make_packet(st, t)
        pl.apply(device_packet(pkt, pl.dev))
        A, s, _ = oracle.apply(A, pkt)
        assert s == 0
        st_planes = synth.Scene(st.cfg, st.n, cap, st.deg, A, st.dynamic)
        d = synth.make_delta(st_planes, t, rem_frac=0.01, add_frac=0.012)
        pl.densify(torch.from_numpy(d.rem.view(np.int32)).cuda(), d.rem.size,
                   torch.from_numpy(d.add.view(np.int16)).cuda(), d.add.shape[1])
        A, n, s = oracle.densify(A, n, d.rem, d.add, cap)
        assert s == 0
        st = synth.advance_state(st, d, cap)
        assert pl.n == n == st.n
        s, _ = pl.check_status()
        assert s == 0
        assert np.array_equal(pl.planes.cpu().numpy().view(np.uint32), A.view(np.uint32)), t
    pl.fit_capacity()
    rgb = pl.render().cpu().numpy()
    _, _, ref, _ = oracle.render(A, n, sc.deg, cams)
    assert np.abs(np.clip(rgb, 0, 1) - np.clip(ref, 0, 1)).max() <= 2e-3
    assert psnr(np.clip(rgb, 0, 1), np.clip(ref, 0, 1)) > 60.0
