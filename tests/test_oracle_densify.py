"""NEXT #2 oracle pins: densification deltas (DESIGN reading R21).

  * empty delta -> identical set; removing everything then adding -> exactly the additions;
  * survivors keep their relative order and their exact values (checked through an ID plane);
  * binary16 additions convert exactly (every binary16 value is a float32);
  * removal lists that are unsorted, repeated or out of range are rejected (-3);
  * the synthetic stream bookkeeping (advance_state) re-indexes the dynamic pool consistently.
"""
import numpy as np
import pytest

import oracle
from harness import synth


def _planes(n, P=14, seed=0):
    rng = np.random.default_rng(seed)
    pl = np.zeros((P, (n + 3) // 4 * 4), np.float32)
    pl[:, :n] = rng.standard_normal((P, n)).astype(np.float32)
    pl[0, :n] = np.arange(n, dtype=np.float32)  # ID plane
    return pl


def test_empty_delta_identity():
    pl = _planes(101)
    out, n, st = oracle.densify(pl, 101, np.zeros(0, np.uint32), np.zeros((14, 0), np.float16), pl.shape[1])
    assert st == 0 and n == 101 and np.array_equal(out, pl)


def test_survivor_order_and_values():
    pl = _planes(500)
    rng = np.random.default_rng(1)
    rem = np.sort(rng.choice(500, 37, replace=False))
    add = rng.standard_normal((14, 11)).astype(np.float16)
    out, n, st = oracle.densify(pl, 500, rem, add)
    assert st == 0 and n == 500 - 37 + 11
    ids = out[0, :463].astype(np.int64)
    assert np.all(np.diff(ids) > 0) and not np.isin(ids, rem).any() and ids.size == 463
    assert np.array_equal(out[:, :463], pl[:, ids])
    assert np.array_equal(out[:, 463:n], add.astype(np.float32))
    assert np.all(out[:, n:] == 0)


def test_remove_all_then_add():
    pl = _planes(40)
    add = np.arange(14 * 3, dtype=np.float16).reshape(14, 3)
    out, n, st = oracle.densify(pl, 40, np.arange(40), add)
    assert st == 0 and n == 3 and np.array_equal(out[:, :3], add.astype(np.float32))


def test_binary16_exact():
    vals = np.array([65504.0, -65504.0, 6.1e-5, 5.96e-8, 0.1, -0.0, 1.0 / 3.0], np.float16)
    out, n, _ = oracle.densify(np.zeros((1, 4), np.float32), 0, [], vals[None, :])
    assert np.array_equal(out[0, :n], vals.astype(np.float64).astype(np.float32))


@pytest.mark.parametrize("rem", [[3, 2], [4, 4], [50], [-1]])
def test_bad_removals_rejected(rem):
    pl = _planes(50)
    assert oracle.densify(pl, 50, np.array(rem), np.zeros((14, 0), np.float16))[2] == -3


def test_stream_bookkeeping():
    cfg = synth.get_config("tiny")
    sc = synth.make_scene(cfg, n=1000)
    st = synth.Scene(sc.cfg, sc.n, 1200, sc.deg, sc.planes, sc.dynamic)
    d = synth.make_delta(st, 1, rem_frac=0.05, add_frac=0.08)
    nxt = synth.advance_state(st, d)
    assert nxt.n == 1000 - d.rem.size + d.add.shape[1]
    keep = np.setdiff1d(np.arange(1000), d.rem)
    old_dyn_kept = np.intersect1d(sc.dynamic, keep)
    assert np.array_equal(keep[nxt.dynamic[:old_dyn_kept.size]], old_dyn_kept)
    assert np.array_equal(nxt.dynamic[old_dyn_kept.size:], np.arange(keep.size, nxt.n))
    assert d.add.dtype == np.float16 and d.add.shape[0] == sc.planes.shape[0]
