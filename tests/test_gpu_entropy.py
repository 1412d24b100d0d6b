"""NEXT #1 on the GPU: libqueen's warp-per-chunk rANS decoder vs the original latents.

Bit-exact (integer) parity: decoding the product's stream AND the oracle's independently
encoded stream reproduces the int8 latent matrix exactly; padding columns are untouched;
corrupt streams raise QUEEN_ERR_INDEX; an entropy-coded wire packet applied through the
public runtime gives the same A_t as the oracle's apply of the uncoded packet.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from tests.test_entropy import CASES, _laplace  # noqa: E402


def _ctx():
    import paper_2412_04469_b200 as Q
    ctx = Q.Context(0)
    ctx.set_workspace(4, 1, 16, 16, 1024)
    return ctx


@pytest.mark.parametrize("L,n,n_pad,beta", CASES)
@pytest.mark.parametrize("encoder", ["product", "oracle"])
def test_gpu_ans_decode_bit_exact(L, n, n_pad, beta, encoder):
    import paper_2412_04469_b200 as Q
    lat = _laplace(L, n, n_pad, beta, seed=11 + n)
    s = Q.queen_entropy_encode(lat, n) if encoder == "product" else oracle.ans_encode(lat, n)
    ctx = _ctx()
    dev = torch.from_numpy(s).cuda()
    out = torch.full((L, n_pad), 77, dtype=torch.int8, device="cuda")
    Q.queen_entropy_decode(ctx, dev, L, n, out)
    st, _ = ctx.check_status()
    got = out.cpu().numpy()
    assert st == 0
    assert np.array_equal(got[:, :n], lat[:, :n])
    assert np.all(got[:, n:] == 77)  # padding untouched


def test_gpu_ans_corrupt_stream_flags():
    import paper_2412_04469_b200 as Q
    lat = _laplace(6, 20000, 20000, 0.5, seed=2)
    s = Q.queen_entropy_encode(lat, 20000)
    bad = s.copy()
    nch = (6 * 20000 + 8191) // 8192
    bad[528 + 4 * (nch + 1) + 4 * 13 + 1] ^= 0x5A  # lane 13's initial state (chunk 0)
    ctx = _ctx()
    out = torch.zeros((6, 20000), dtype=torch.int8, device="cuda")
    Q.queen_entropy_decode(ctx, torch.from_numpy(bad).cuda(), 6, 20000, out)
    assert ctx.check_status()[0] == -3
    Q.queen_entropy_decode(ctx, torch.from_numpy(s).cuda(), 6, 19999, out)  # shape mismatch
    assert ctx.check_status()[0] == -3


def test_gpu_ans_hostile_headers_stay_in_bounds():
    """the stream header is wire input.  A header claiming more symbols or chunks than
    (L, n) imply, chunk word offsets past the stream's byte size, or a stream too small for its
    tables must never read or write out of bounds: the mismatched category writes nothing and
    QUEEN_ERR_INDEX is raised (or QUEEN_ERR_SHAPE on the host for a truncated stream)."""
    import paper_2412_04469_b200 as Q
    L, n = 3, 20000
    lat = _laplace(L, n, n, 0.3, seed=5)
    s = Q.queen_entropy_encode(lat, n)
    hdr = np.frombuffer(s[:16].tobytes(), np.uint32)
    n_chunks = int(hdr[2])
    ctx = _ctx()
    # guard bytes after the output: an out-of-bounds write would change them
    out = torch.full((L + 1, n), 55, dtype=torch.int8, device="cuda")
    for word, val in ((1, 10 ** 9), (1, 8191), (2, n_chunks + 5), (2, 0)):
        bad = s.copy()
        bad[4 * word:4 * word + 4] = np.array([val], np.uint32).view(np.uint8)
        Q.queen_entropy_decode(ctx, torch.from_numpy(bad).cuda(), L, n, out[:L])
        assert ctx.check_status()[0] == -3, (word, val)
        assert np.all(out.cpu().numpy() == 55), (word, val)  # mismatched header: nothing written
    # a chunk's end offset far past the stream
    bad = s.copy()
    woff = 528 + 4 * 1
    bad[woff:woff + 4] = np.array([1 << 30], np.uint32).view(np.uint8)
    Q.queen_entropy_decode(ctx, torch.from_numpy(bad).cuda(), L, n, out[:L])
    assert ctx.check_status()[0] == -3
    assert np.all(out[L].cpu().numpy() == 55)
    # truncated stream (the byte size cannot hold the chunk tables): host error, nothing enqueued
    with pytest.raises(Q.QueenError):
        Q.queen_entropy_decode(ctx, torch.from_numpy(s[:600].copy()).cuda(), L, n, out[:L])
    # the intact stream still decodes exactly afterwards
    Q.queen_entropy_decode(ctx, torch.from_numpy(s).cuda(), L, n, out[:L])
    assert ctx.check_status()[0] == 0
    assert np.array_equal(out[:L].cpu().numpy(), lat)


def test_entropy_packet_apply_matches_oracle():
    import paper_2412_04469_b200 as Q
    from harness import synth
    from paper_2412_04469_b200 import packet as wire
    from paper_2412_04469_b200.runtime import EntropyPacket, Player
    cfg = synth.get_config("n3dv")
    sc = synth.make_scene(cfg, n=40003)
    cams = synth.make_cameras(cfg, 2)
    pl = Player(sc.planes, sc.n, sc.deg, cams)
    A = sc.planes.copy()
    for t in (1, 2, 3):
        pkt = synth.make_packet(sc, t)
        streams = wire.ans_streams(pkt, Q.queen_entropy_encode)
        buf = wire.pack_entropy(pkt, streams, frame=t, k_cap=pkt.k + 64)
        hdr = wire.header_entropy(buf)
        assert hdr["used"] <= buf.size
        ep = EntropyPacket(torch.from_numpy(buf).cuda(), hdr)
        pl.apply(ep)
        A, st, _ = oracle.apply(A, pkt)
        assert st == 0
    s, _ = pl.check_status()
    assert s == 0
    assert np.array_equal(pl.planes.cpu().numpy(), A)
