"""NEXT #1: entropy coding of the integer latents, QANS rANS streams.

CPU pins of the reference codec (oracle) and of the product's host encoder:
  * round trip decode(encode(x)) == x on ragged shapes, multi-chunk matrices, n < 32,
    all-zero and full-range symbol sets;
  * the product encoder (libqueen host code) and the oracle encoder, both written from the
    DESIGN.md text, emit byte-identical streams;
  * the coded size stays within the order-0 entropy bound: 8*bytes <= n_sym*H + overhead;
  * corrupt / mismatched streams are rejected (-3).
GPU: libqueen's warp-per-chunk decoder reproduces the latents bit-exactly (test_gpu_entropy).
"""
import math

import numpy as np
import pytest

import oracle


def _laplace(L, n, n_pad, beta, seed):
    rng = np.random.default_rng(seed)
    lat = np.zeros((L, n_pad), np.int8)
    lat[:, :n] = np.clip(np.round(rng.laplace(0.0, beta, (L, n))), -127, 127).astype(np.int8)
    return lat


CASES = [(6, 997, 1000, 0.22), (1, 5, 8, 0.5), (3, 31, 32, 3.0), (12, 33001, 33024, 0.5), (8, 20000, 20000, 0.0),
         (4, 4096, 4096, 80.0)]


@pytest.mark.parametrize("L,n,n_pad,beta", CASES)
def test_oracle_roundtrip_and_entropy_bound(L, n, n_pad, beta):
    lat = _laplace(L, n, n_pad, beta, seed=L * 7 + n)
    s = oracle.ans_encode(lat, n)
    dec, st = oracle.ans_decode(s, L, n, n_pad)
    assert st == 0
    assert np.array_equal(dec[:, :n], lat[:, :n])
    # order-0 entropy bound (closed form): payload bits <= n_sym * H + per-symbol ANS
    # inefficiency (4096-quantised probabilities) + per-chunk states and word padding
    vals, cnt = np.unique(lat[:, :n], return_counts=True)
    p = cnt / cnt.sum()
    H = float(-(p * np.log2(p)).sum()) if cnt.sum() else 0.0
    nsym = L * n
    nch = (nsym + 8191) // 8192
    overhead_bits = 8 * (528 + 4 * (nch + 1) + 4 * 32 * nch + 2 * 32 * nch + 4) + 0.01 * nsym + 16 * 32 * nch
    assert 8 * s.size <= nsym * H * 1.01 + overhead_bits


def test_product_encoder_matches_reference_bytes():
    import paper_2412_04469_b200 as Q
    for L, n, n_pad, beta in CASES:
        lat = _laplace(L, n, n_pad, beta, seed=3 + n)
        a = oracle.ans_encode(lat, n)
        b = Q.queen_entropy_encode(lat, n)
        assert a.size == b.size and np.array_equal(a, b)


def test_packet_latents_bits_per_attribute():
    """The N3DV-shaped packet (P(l=0) ~ 0.9) codes near the paper's 0.68 bits/attribute."""
    from harness import synth
    cfg = synth.get_config("n3dv")
    sc = synth.make_scene(cfg, n=60000)
    pkt = synth.make_packet(sc, 1)
    row = 0
    bits = 0
    for c in range(5):
        L = pkt.lat[c]
        s = oracle.ans_encode(pkt.latents[row:row + L], sc.n)
        bits += 8 * s.size
        dec, st = oracle.ans_decode(s, L, sc.n, sc.n_pad)
        assert st == 0 and np.array_equal(dec[:, :sc.n], pkt.latents[row:row + L, :sc.n])
        row += L
    bpa = bits / (sum(pkt.lat) * sc.n)
    assert 0.4 < bpa < 1.0, bpa


def test_corrupt_and_mismatched_streams_rejected():
    lat = _laplace(6, 5000, 5000, 0.5, seed=1)
    s = oracle.ans_encode(lat, 5000)
    assert oracle.ans_decode(s, 6, 4999, 5000)[1] == -3        # wrong shape
    assert oracle.ans_decode(s[:600], 6, 5000, 5000)[1] == -3  # truncated
    nch = (6 * 5000 + 8191) // 8192
    bad = s.copy()
    bad[528 + 4 * (nch + 1) + 4 * 7 + 1] ^= 0x55               # lane 7's initial state (chunk 0)
    assert oracle.ans_decode(bad, 6, 5000, 5000)[1] == -3
    bad = s.copy()
    lc = 528 + 4 * (nch + 1) + 4 * 32 * nch                    # lane word counts
    bad[lc + 2 * 3] ^= 0x01                                    # lane 3's word count (chunk 0)
    assert oracle.ans_decode(bad, 6, 5000, 5000)[1] == -3
    bad = s.copy()
    bad[0] ^= 1                                                # magic
    assert oracle.ans_decode(bad, 6, 5000, 5000)[1] == -3
