"""Oracle pins: latent decode (Eq. 5), apply (Eq. 4) and the COO position step.

Pins: SPEC worked example D = I; zero residual reproduces the previous frame;
linearity; numpy float64 matmul (a library primitive) within fp32 rounding; and
the dyadic family, whose decode/apply is exact in fp32 in ANY order, compared
with the closed form A_0 + sum_t R_t computed in exact int64 arithmetic.
"""
import json
import os

import numpy as np
import pytest

import oracle
from harness import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_spec_examples.json")))


def _tiny():
    cfg = synth.get_config("tiny")
    sc = synth.make_scene(cfg)
    return cfg, sc


def test_decode_identity_spec_example():
    # P:296 r = D float(l); D = I (2x2), l = (3, -2) -> (3, -2).  Embed in the opacity
    # category? It has M = 1; use the scale category (M = 3, L = 3) with D = I3, l = (3, -2, 0).
    cfg, sc = _tiny()
    pkt = synth.zero_packet(sc, lat=(1, 3, 1, 1, 0))
    M = synth.category_m(0)
    D = [np.zeros((M[c], pkt.lat[c]), np.float32) for c in range(5)]
    D[1] = np.eye(3, dtype=np.float32)
    pkt.decoders = np.concatenate([d.reshape(-1) for d in D])
    pkt.latents[1:4, 0] = [3, -2, 0]
    r = oracle.decode(pkt)
    ex = GOLD["decode_identity"]["r"]
    assert r[4, 0] == ex[0] and r[5, 0] == ex[1] and r[6, 0] == 0.0  # rows 4..6 = scale (planes 7..9)
    assert np.all(r[:, 1:pkt.n] == 0)


def test_zero_residual_reproduces_previous_frame():
    cfg, sc = _tiny()
    pkt = synth.make_packet(sc, 1)
    pkt.latents[:] = 0
    pkt.coo_idx = np.zeros(0, np.uint32)
    pkt.coo_val = np.zeros((3, 0), np.float32)
    out, st, _ = oracle.apply(sc.planes, pkt)
    assert st == 0
    assert np.array_equal(out, sc.planes)  # IEEE == (x + 0.0 keeps the value; -0 -> +0 compares equal)


def test_decode_matches_float64_matmul_and_linearity():
    cfg = synth.get_config("n3dv")
    sc = synth.make_scene(cfg, n=3000)
    pkt = synth.make_packet(sc, 3)
    r = oracle.decode(pkt).astype(np.float64)
    # library matmul per category in float64
    M = synth.category_m(3)
    q = pkt.latents.astype(np.float64)
    lrow = drow = orow = 0
    for c in range(5):
        L = pkt.lat[c]
        D = pkt.decoders[drow:drow + M[c] * L].reshape(M[c], L).astype(np.float64)
        ref = D @ q[lrow:lrow + L, :pkt.n]
        got = r[orow:orow + M[c], :pkt.n]
        bound = L * np.finfo(np.float32).eps * (np.abs(D) @ np.abs(q[lrow:lrow + L, :pkt.n])) + 1e-30
        assert np.all(np.abs(got - ref) <= bound)
        lrow += L; drow += M[c] * L; orow += M[c]
    # linearity in l on integer-valued, exactly representable combinations
    pkt2 = synth.make_packet(sc, 4)
    pkt2.decoders = pkt.decoders
    s = synth.make_packet(sc, 3)
    s.latents = (pkt.latents.astype(np.int16) + pkt2.latents.astype(np.int16)).clip(-127, 127).astype(np.int8)
    ok = np.all(np.abs(pkt.latents.astype(np.int16) + pkt2.latents.astype(np.int16)) <= 127, axis=0)
    rs = oracle.decode(s).astype(np.float64)
    r2 = oracle.decode(pkt2).astype(np.float64)
    diff = np.abs(rs - (r + r2))[:, :pkt.n][:, ok[:pkt.n]]
    assert diff.max() <= 1e-6 * max(np.abs(rs).max(), 1e-12)


@pytest.mark.parametrize("frames", [1, 12])
def test_dyadic_streaming_exact(frames):
    """Drift-free streaming: decode frames 1..T in order == A_0 + sum R_t in exact int64."""
    cfg = synth.get_config("n3dv")
    sc = synth.make_dyadic_scene(cfg, n=2000)
    A = sc.planes.copy()
    acc = np.round(sc.planes.astype(np.float64) * 1024).astype(np.int64)
    M = synth.category_m(3)
    for t in range(1, frames + 1):
        pkt = synth.make_packet(sc, t, dyadic=True)
        A, st, _ = oracle.apply(A, pkt)
        assert st == 0
        q = pkt.latents.astype(np.int64)
        lrow = drow = 0
        orow = 3
        for c in range(5):
            L = pkt.lat[c]
            D = np.round(pkt.decoders[drow:drow + M[c] * L].reshape(M[c], L).astype(np.float64) * 1024).astype(np.int64)
            acc[orow:orow + M[c], :pkt.n] += D @ q[lrow:lrow + L, :pkt.n]
            lrow += L; drow += M[c] * L; orow += M[c]
        vi = np.round(pkt.coo_val.astype(np.float64) * 1024).astype(np.int64)
        acc[0:3, pkt.coo_idx.astype(np.int64)] += vi
    exact = acc.astype(np.float64) / 1024.0
    assert np.array_equal(A[:, :sc.n].astype(np.float64), exact[:, :sc.n])


def test_coo_moves_only_gated_rows_and_validates():
    cfg, sc = _tiny()
    pkt = synth.make_packet(sc, 1)
    pkt.latents[:] = 0
    out, st, _ = oracle.apply(sc.planes, pkt)
    assert st == 0
    moved = np.nonzero(np.any(out[0:3] != sc.planes[0:3], axis=0))[0]
    assert set(moved.tolist()) <= set(pkt.coo_idx.tolist())
    assert np.array_equal(out[3:], sc.planes[3:])
    # empty COO -> nothing moves
    pkt.coo_idx = np.zeros(0, np.uint32)
    pkt.coo_val = np.zeros((3, 0), np.float32)
    out2, st2, _ = oracle.apply(sc.planes, pkt)
    assert st2 == 0 and np.array_equal(out2, sc.planes)
    # out-of-range / non-increasing index -> QUEEN_ERR_INDEX (-3)
    pkt.coo_idx = np.array([5, 5], np.uint32)
    pkt.coo_val = np.zeros((3, 2), np.float32)
    assert oracle.apply(sc.planes, pkt)[1] == -3
    pkt.coo_idx = np.array([sc.n], np.uint32)
    pkt.coo_val = np.zeros((3, 1), np.float32)
    assert oracle.apply(sc.planes, pkt)[1] == -3


def test_gates_path_equals_coo_path():
    """Gate -> COO -> scatter gives the same A_t as feeding the oracle's own COO."""
    cfg, sc = _tiny()
    pkt = synth.make_packet(sc, 1)
    a, st, _ = oracle.apply(sc.planes, pkt, use_gates=True, use_f32_latents=True)
    idx, val = oracle.gate(pkt)
    pkt.coo_idx, pkt.coo_val = idx, val
    b, st2, _ = oracle.apply(sc.planes, pkt)
    assert st == 0 and st2 == 0 and np.array_equal(a, b)


def test_latent_range_error():
    cfg, sc = _tiny()
    pkt = synth.make_packet(sc, 1)
    pkt.latents_f32[0, 3] = 127.6
    _, st, _ = oracle.apply(sc.planes, pkt, use_f32_latents=True)
    assert st == -4


# ------------------------------------------------------------------ first-frame SH "set" decode
def test_set_sh_rest_identity_decoder():
    """P:1380-1381 first-frame quantisation, D = I (L = M = 9 at degree 1): the SH-rest planes
    become float(l) exactly; every other plane and the padding columns are untouched."""
    rng = np.random.default_rng(3)
    n, n_pad, deg = 37, 40, 1
    planes = rng.standard_normal((11 + 3 * 4, n_pad)).astype(np.float32)
    lat = rng.integers(-127, 128, (9, n_pad)).astype(np.int8)
    out = oracle.set_sh_rest(planes, n, deg, lat, np.eye(9, dtype=np.float32))
    assert np.array_equal(out[14:, :n], lat[:, :n].astype(np.float32))
    assert np.array_equal(out[:14].view(np.uint32), planes[:14].view(np.uint32))
    assert np.array_equal(out[:, n:].view(np.uint32), planes[:, n:].view(np.uint32))


def test_set_sh_rest_dyadic_exact():
    """Dyadic family (D on the 2^-10 grid, |l| <= 8, L = 12, degree 3: M = 45): every partial sum
    is exact in fp32, so the result equals the integer-arithmetic value sum_k D_k l_k exactly,
    and it REPLACES the old coefficients (set, not add)."""
    from harness import synth
    cfg = synth.get_config("immersive")
    sc = synth.make_scene(cfg, n=3001)
    ff = synth.make_first_frame_sh(sc, dyadic=True)
    assert ff.latents.shape[0] == 12 and ff.decoder.shape == (45, 12)
    out = oracle.set_sh_rest(sc.planes, sc.n, sc.deg, ff.latents, ff.decoder)
    Di = np.rint(ff.decoder.astype(np.float64) * 1024).astype(np.int64)      # exact integers
    exact = (Di @ ff.latents[:, :sc.n].astype(np.int64)).astype(np.float64) / 1024.0
    assert np.array_equal(out[14:, :sc.n].astype(np.float64), exact)
    assert np.array_equal(out[:14].view(np.uint32), sc.planes[:14].view(np.uint32))


def test_set_sh_rest_zero_latents_give_positive_zero():
    """All-zero latents decode to +0.0 (fmaf chain from +0, R7), whatever the decoder's signs."""
    n, n_pad, deg = 8, 8, 2
    planes = np.full((11 + 3 * 9, n_pad), 7.0, np.float32)
    dec = -np.ones((24, 3), np.float32)
    out = oracle.set_sh_rest(planes, n, deg, np.zeros((3, n_pad), np.int8), dec)
    assert np.all(out[14:].view(np.uint32) == 0)
