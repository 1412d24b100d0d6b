"""NEXT #3 on the GPU: queen_render_mask vs the oracle.

Bit-exact masks: at alpha_thresh = 1e-3 (< 1/255) a pixel is marked iff a subset Gaussian passes
the 1/255 skip test there, a decision both sides take bit-identically (DESIGN "Arithmetic
contract"), and the dilation is integer work.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from harness import synth  # noqa: E402


def _player(sc, cams, **kw):
    from paper_2412_04469_b200.runtime import Player
    pl = Player(sc.planes, sc.n, sc.deg, cams, **kw)
    pl.fit_capacity()
    return pl


@pytest.mark.parametrize("name,n,views,over,frac,d", [
    ("tiny", 1000, None, {}, 0.02, 9),
    ("tiny", 1000, None, {}, 0.3, 48),
    ("tiny", 337, None, {"index": 7}, 1.0, 1),
    ("n3dv", 20003, 3, {"width": 333, "height": 250, "focal": 280.0}, 0.1, 48),
    ("immersive", 12001, 4, {"width": 320, "height": 240, "focal": 160.0}, 0.3, 17),
])
def test_render_mask_matches_oracle(name, n, views, over, frac, d):
    cfg = synth.get_config(name, **over)
    sc = synth.make_scene(cfg, n=n)
    cams = synth.make_cameras(cfg, views)
    rng = np.random.default_rng(n)
    sub = np.sort(rng.choice(sc.n, max(1, int(frac * sc.n)), replace=False)).astype(np.uint32)
    pl = _player(sc, cams)
    got = pl.render_mask(torch.from_numpy(sub).cuda(), dilation=d).cpu().numpy()
    s, _ = pl.check_status()
    assert s == 0
    ref = oracle.render_mask(sc.planes, sc.n, sc.deg, cams, sub.astype(np.int64), 1e-3, d)
    assert got.shape == ref.shape
    assert np.array_equal(got, ref), int((got != ref).sum())
    assert ref.sum() > 0


def test_render_mask_gated_coo_device_count():
    """The dynamic set of a frame = its packet's gated COO indices, count read on the device."""
    from paper_2412_04469_b200.runtime import device_packet
    cfg = synth.get_config("n3dv", width=333, height=250, focal=280.0)
    sc = synth.make_scene(cfg, n=20003)
    cams = synth.make_cameras(cfg, 2)
    pkt = synth.make_packet(sc, 1)
    pl = _player(sc, cams)
    dp = device_packet(pkt, pl.dev)
    idx = dp._keep["idx"]  # the packet's own device COO indices
    kdev = torch.tensor([pkt.k], dtype=torch.int32, device="cuda")
    got = pl.render_mask(idx, k=idx.numel(), k_dev=kdev, dilation=48).cpu().numpy()
    ref = oracle.render_mask(sc.planes, sc.n, sc.deg, cams, pkt.coo_idx.astype(np.int64), 1e-3, 48)
    assert np.array_equal(got, ref)
    # a device count of 0 selects nothing
    kdev.zero_()
    assert not pl.render_mask(idx, k=idx.numel(), k_dev=kdev).any()


def test_render_mask_errors_and_empty():
    import paper_2412_04469_b200 as Q
    cfg = synth.get_config("tiny")
    sc = synth.make_scene(cfg, n=500)
    cams = synth.make_cameras(cfg)
    pl = _player(sc, cams)
    empty = torch.zeros(0, dtype=torch.int32, device="cuda")
    assert not pl.render_mask(empty).any()
    bad = torch.tensor([5, 3], dtype=torch.int32, device="cuda")  # not increasing
    pl.render_mask(bad)
    assert pl.check_status()[0] == -3
    oob = torch.tensor([sc.n], dtype=torch.int32, device="cuda")
    pl.render_mask(oob)
    assert pl.check_status()[0] == -3
    with pytest.raises(Q.QueenError):
        pl.render_mask(torch.tensor([1], dtype=torch.int32, device="cuda"), dilation=0)
