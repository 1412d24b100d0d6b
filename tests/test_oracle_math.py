"""Oracle pins: elementwise functions (det_exp/det_log, quantise, gate, SH basis).

Each check pins the oracle to something other than itself: double-precision libm,
SPEC/PAPER worked examples (tests/golden/paper_spec_examples.json), closed forms,
scipy's spherical harmonics, and quadrature orthonormality.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from tests.util import ulp_dist

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_spec_examples.json")))


def test_det_exp_vs_double_libm():
    rng = np.random.default_rng(1)
    xs = np.concatenate([rng.uniform(-87, 88, 20000), rng.uniform(-2, 2, 5000),
                         np.array([0.0, 1.0, -1.0, 88.0, -87.0, 0.5, -0.5, 1e-8, -1e-8])]).astype(np.float32)
    got = np.array([oracle.det_exp(x) for x in xs], np.float32)
    ref = np.exp(xs.astype(np.float64))
    assert ulp_dist(got, ref).max() <= 2.0
    assert oracle.det_exp(0.0) == 1.0  # exp(0) = 1 exactly


def test_det_log_vs_double_libm():
    rng = np.random.default_rng(2)
    ys = np.concatenate([rng.uniform(1.0, 255.0, 20000), np.exp(rng.uniform(-60, 60, 5000)),
                         np.array([1.0, 2.0, 255.0, 1.41421356, 1.4142137, 0.70710677, 1.0000001])]).astype(np.float32)
    got = np.array([oracle.det_log(y) for y in ys], np.float32)
    ref = np.log(ys.astype(np.float64))
    big = np.abs(ref) > 1e-3
    assert ulp_dist(got[big], ref[big]).max() <= 2.0
    assert np.abs(got[~big] - ref[~big]).max() <= 2 ** -30
    assert oracle.det_log(1.0) == 0.0


def test_quantize_spec_examples():
    cases = GOLD["quantize_round"]["cases"]
    lhat = np.array([c[0] for c in cases], np.float32)
    q, bad = oracle.quantize(lhat)
    assert bad == 0
    assert q.tolist() == [c[1] for c in cases]


def test_quantize_idempotent_and_range():
    rng = np.random.default_rng(3)
    lhat = rng.uniform(-130, 130, 10000).astype(np.float32)
    q, bad = oracle.quantize(lhat)
    l64 = lhat.astype(np.float64)
    assert bad == int(np.sum(np.floor(np.abs(l64) + 0.5) > 127))
    inr = np.abs(lhat) < 126.5
    q2, bad2 = oracle.quantize(q[inr].astype(np.float32))
    assert bad2 == 0 and np.array_equal(q2, q[inr])
    # half away from zero vs a plain definition: sign(x) * floor(|x| + 0.5) in double
    ref = np.sign(lhat[inr].astype(np.float64)) * np.floor(np.abs(lhat[inr].astype(np.float64)) + 0.5)
    assert np.array_equal(q[inr].astype(np.float64), ref)


@pytest.mark.parametrize("preset", ["n3dv", "immersive"])
def test_gate_closed_forms(preset):
    hp = GOLD["gate_hyperparams"][preset]
    tau, g0, g1 = hp["tau"], hp["gamma0"], hp["gamma1"]
    th0 = float(oracle.theta0(tau, g0, g1))
    assert th0 == pytest.approx(GOLD["gate_value"]["theta0_" + preset], abs=1e-6)
    # saturation: large +/- log alpha -> 1 / 0
    assert oracle.gate_value(1e4, tau, g0, g1) == 1.0
    assert oracle.gate_value(-1e4, tau, g0, g1) == 0.0
    # boundary: g_tilde = 0 at theta0
    assert oracle.gate_value(th0, tau, g0, g1) <= 1e-6
    assert oracle.gate_value(th0 - 1e-3, tau, g0, g1) == 0.0
    assert oracle.gate_value(th0 + 1e-3, tau, g0, g1) > 0.0
    # g = 1 for log alpha >= theta1 = tau ln((1-g0)/(g1-1))
    th1 = tau * math.log((1 - g0) / (g1 - 1))
    assert oracle.gate_value(th1 + 1e-3, tau, g0, g1) == 1.0
    assert oracle.gate_value(th1 - 1e-2, tau, g0, g1) < 1.0
    # monotone non-decreasing and equal to the paper's formula evaluated in double
    la = np.linspace(-6, 6, 4001).astype(np.float32)
    g = np.array([oracle.gate_value(x, tau, g0, g1) for x in la])
    assert np.all(np.diff(g) >= 0)
    gt = 1 / (1 + np.exp(-la.astype(np.float64) / tau)) * (g1 - g0) + g0
    assert np.abs(g - np.clip(gt, 0, 1)).max() < 1e-6


def test_gate_value_n3dv_paper_example():
    hp = GOLD["gate_hyperparams"]["n3dv"]
    g = oracle.gate_value(0.0, hp["tau"], hp["gamma0"], hp["gamma1"])
    assert g == pytest.approx(GOLD["gate_value"]["log_alpha_zero_n3dv"], abs=1e-6)


def test_gate_mask_matches_double_formula():
    from harness import synth
    cfg = synth.get_config("tiny")
    sc = synth.make_scene(cfg)
    pkt = synth.make_packet(sc, 1)
    # add log alphas right around the boundary
    th0 = oracle.theta0(*pkt.gate)
    pkt.log_alpha[:8] = np.array([th0, np.nextafter(th0, np.float32(1)), np.nextafter(th0, np.float32(-1)),
                                  th0 + 1e-4, th0 - 1e-4, 0.0, 10.0, -10.0], np.float32)
    idx, val = oracle.gate(pkt)
    la = pkt.log_alpha[: pkt.n].astype(np.float64)
    tau, g0, g1 = pkt.gate
    gt = 1 / (1 + np.exp(-la / tau)) * (g1 - g0) + g0
    far = np.abs(la - float(th0)) > 1e-5
    mask = np.zeros(pkt.n, bool)
    mask[idx] = True
    assert np.array_equal(mask[far], (gt > 0)[far])
    assert np.all(np.diff(idx.astype(np.int64)) > 0)
    g = np.clip(gt[idx], 0, 1)
    ref = g[None, :] * pkt.pos_pregate[:, idx].astype(np.float64)
    assert np.abs(val - ref).max() <= 1e-6 * np.abs(pkt.pos_pregate).max() + 1e-12


def test_sh_basis_matches_scipy_and_deg0():
    from tests.ref64 import real_sh
    rng = np.random.default_rng(4)
    d = rng.standard_normal((3, 200))
    d /= np.linalg.norm(d, axis=0)
    ref = real_sh(3, d)
    for j in range(d.shape[1]):
        Y = oracle.sh_basis(3, d[:, j])
        assert np.abs(Y - ref[:, j]).max() < 2e-6
    assert oracle.sh_basis(0, (0, 0, 1))[0] == pytest.approx(GOLD["eval_sh_deg0"]["Y00"], abs=1e-9)


def test_sh_basis_orthonormal_quadrature():
    # Gauss-Legendre in cos(theta) x uniform phi: exact for polynomials of degree <= 6 on the sphere
    xg, wg = np.polynomial.legendre.leggauss(12)
    nphi = 24
    G = np.zeros((16, 16))
    for ct, w in zip(xg, wg):
        st = math.sqrt(1 - ct * ct)
        for k in range(nphi):
            ph = 2 * math.pi * k / nphi
            Y = oracle.sh_basis(3, (st * math.cos(ph), st * math.sin(ph), ct)).astype(np.float64)
            G += np.outer(Y, Y) * w * (2 * math.pi / nphi)
    assert np.abs(G - np.eye(16)).max() < 1e-5
