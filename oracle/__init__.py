"""CPU oracle for QUEEN's per-frame decode -> apply -> splat path (ctypes over queen_oracle.cpp).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  The product
package ``paper_2412_04469_b200`` never imports it, and it imports nothing from
the product package (the two share no code).

Every function follows the PAPER.md passage cited in queen_oracle.cpp.  The only
Python-side arithmetic is theta0 = tau*ln(-gamma0/gamma1) in double (DESIGN
reading R6), rounded to float32, and array bookkeeping.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "queen_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", *CFLAGS, _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        p, i32, i64, f32 = C.c_void_p, C.c_int, C.c_int64, C.c_float
        sig = {
            "oracle_det_exp": (f32, [f32]),
            "oracle_det_log": (f32, [f32]),
            "oracle_quantize": (i64, [p, p, i64]),
            "oracle_decode": (None, [i32, i32, i32, p, p, p, p]),
            "oracle_apply": (i32, [i32, i32, i32, p, p, p, p, i32, p, p]),
            "oracle_set_sh_rest": (None, [i32, i32, i32, i32, p, p, p]),
            "oracle_gate_value": (f32, [f32, f32, f32, f32]),
            "oracle_gate": (i32, [i32, i32, p, p, f32, f32, f32, f32, p, p, i32]),
            "oracle_sh_basis": (None, [i32, f32, f32, f32, p]),
            "oracle_project": (i32, [i32, i32, i32, p, i32, p, p, p, p, p, i32]),
            "oracle_bin": (i64, [i32, i32, i32, i32, p, p, p, p, p, p, p, p, p, i64]),
            "oracle_rasterize": (None, [i32, i32, i32, i32, p, p, p, p, p, p, i32]),
            "oracle_rasterize_bruteforce": (None, [i32, i32, i32, i32, i32, p, p, p, p, p, i32]),
            "oracle_rasterize_pixels": (None, [i32, i32, i32, p, p, p, p, i64, p, p, p, i32]),
            "oracle_ans_encode": (i64, [p, i32, i32, i32, p, i64]),
            "oracle_ans_decode": (i32, [p, i64, i32, i32, i32, p]),
            "oracle_blend_counts": (None, [i32, i32, i32, i32, p, p, p, p, p, i32]),
            "oracle_contrib": (None, [i32, i32, i32, i32, p, p, p, p, p, p, p, i32]),
            "oracle_rasterize_pixels_direct": (None, [i32, i32, i32, i32, p, p, p, p, p, i64, p, p, p, i32]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


def default_threads() -> int:
    return os.cpu_count() or 1


# ---------------------------------------------------------------- elementwise
def det_exp(x: float) -> float:
    return lib().oracle_det_exp(float(x))


def det_log(y: float) -> float:
    return lib().oracle_det_log(float(y))


def quantize(lhat: np.ndarray):
    lhat = np.ascontiguousarray(lhat, np.float32)
    q = np.zeros(lhat.shape, np.int8)
    bad = lib().oracle_quantize(_p(lhat), _p(q), lhat.size)
    return q, int(bad)


def gate_value(log_alpha: float, tau: float, gamma0: float, gamma1: float) -> float:
    return lib().oracle_gate_value(float(log_alpha), float(tau), float(gamma0), float(gamma1))


def theta0(tau: float, gamma0: float, gamma1: float) -> np.float32:
    """Exact mask threshold on log alpha (DESIGN reading R6): g_tilde > 0 <=> log a > tau ln(-g0/g1)."""
    return np.float32(float(np.float32(tau)) * math.log(-float(np.float32(gamma0)) / float(np.float32(gamma1))))


def sh_basis(deg: int, d) -> np.ndarray:
    Y = np.zeros(16, np.float32)
    lib().oracle_sh_basis(int(deg), float(d[0]), float(d[1]), float(d[2]), _p(Y))
    return Y[: (deg + 1) ** 2]


# ---------------------------------------------------------------- decode / apply
def decode(pkt) -> np.ndarray:
    """r = D_c float(l_c) for every non-position plane: float32 [sum M][n_pad]."""
    from_lat = np.ascontiguousarray(pkt.latents, np.int8)
    lat = np.array(pkt.lat, np.int32)
    B = (pkt.deg + 1) ** 2
    Mtot = 4 + 3 + 1 + 3 + 3 * (B - 1)
    out = np.zeros((Mtot, pkt.n_pad), np.float32)
    lib().oracle_decode(pkt.n, pkt.n_pad, pkt.deg, _p(lat), _p(from_lat), _p(np.ascontiguousarray(pkt.decoders)), _p(out))
    return out


def gate(pkt):
    """Trainer-state gates -> (COO idx uint32 [k], COO val float32 [3][k])."""
    tau, g0, g1 = (np.float32(x) for x in pkt.gate)
    th0 = theta0(*pkt.gate)
    cap = pkt.n
    idx = np.zeros(max(cap, 1), np.uint32)
    val = np.zeros((3, max(cap, 1)), np.float32)
    k = lib().oracle_gate(pkt.n, pkt.n_pad, _p(np.ascontiguousarray(pkt.log_alpha)), _p(np.ascontiguousarray(pkt.pos_pregate)),
                          float(tau), float(g0), float(g1), float(th0), _p(idx), _p(val), max(cap, 1))
    return idx[:k].copy(), np.ascontiguousarray(val[:, :k])


def set_sh_rest(planes: np.ndarray, n: int, deg: int, latents: np.ndarray, decoder: np.ndarray) -> np.ndarray:
    """First-frame SH "set" decode: a copy of planes with the SH-rest rows
    (14 .. 11+3B-1) of the first n Gaussians replaced by D . float(l)."""
    out = np.array(planes, np.float32, copy=True, order="C")
    lat = np.ascontiguousarray(latents, np.int8)
    dec = np.ascontiguousarray(decoder, np.float32)
    L = lat.shape[0]
    assert lat.shape[1] == out.shape[1] and dec.shape == (3 * ((deg + 1) ** 2 - 1), L)
    lib().oracle_set_sh_rest(int(n), out.shape[1], int(deg), int(L), _p(lat), _p(dec), _p(out))
    return out


def apply(planes: np.ndarray, pkt, *, use_gates: bool = False, use_f32_latents: bool = False):
    """A_t = A_{t-1} + R_t on a COPY of planes; returns (planes_t, status, q)."""
    out = np.array(planes, np.float32, copy=True, order="C")
    if use_f32_latents:
        q, bad = quantize(pkt.latents_f32)
    else:
        q, bad = np.ascontiguousarray(pkt.latents), 0
    if use_gates:
        idx, val = gate(pkt)
    else:
        idx, val = np.ascontiguousarray(pkt.coo_idx, np.uint32), np.ascontiguousarray(pkt.coo_val, np.float32)
    lat = np.array(pkt.lat, np.int32)
    st = lib().oracle_apply(pkt.n, pkt.n_pad, pkt.deg, _p(lat), _p(q), _p(np.ascontiguousarray(pkt.decoders)), _p(out),
                            int(idx.shape[0]), _p(idx if idx.size else np.zeros(1, np.uint32)),
                            _p(val if val.size else np.zeros((3, 1), np.float32)))
    if bad:
        st = -4 if st == 0 else st
    return out, st, q


# ---------------------------------------------------------------- entropy coding (NEXT #1)
def ans_encode(latents: np.ndarray, n: int) -> np.ndarray:
    """Reference QANS encoder of one category's int8 latent matrix [L][n_pad]."""
    lat = np.ascontiguousarray(latents, np.int8)
    L, n_pad = lat.shape
    need = lib().oracle_ans_encode(_p(lat), L, n, n_pad, None, 0)
    out = np.zeros(max(int(need), 1), np.uint8)
    got = lib().oracle_ans_encode(_p(lat), L, n, n_pad, _p(out), int(need))
    assert got == need
    return out[:need]


def ans_decode(stream: np.ndarray, L: int, n: int, n_pad: int):
    """Reference QANS decoder -> (int8 [L][n_pad], status 0 / -3)."""
    s = np.ascontiguousarray(stream, np.uint8)
    lat = np.zeros((max(L, 1), n_pad), np.int8)
    st = lib().oracle_ans_decode(_p(s), s.size, L, n, n_pad, _p(lat))
    return lat[:L], int(st)


# ---------------------------------------------------------------- render
def cams_array(cams) -> np.ndarray:
    return np.ascontiguousarray(np.stack([c.as_floats() for c in cams]), np.float32)


def project(planes: np.ndarray, n: int, deg: int, cams, threads: int | None = None):
    planes = np.ascontiguousarray(planes, np.float32)
    n_pad = planes.shape[1]
    V = len(cams)
    rec = np.zeros((V, n_pad, 12), np.float32)
    depth = np.zeros((V, n_pad), np.uint32)
    tiles = np.zeros((V, n_pad), np.uint32)
    rect = np.zeros((V, n_pad, 4), np.int16)
    nf = lib().oracle_project(n, n_pad, deg, _p(planes), V, _p(cams_array(cams)), _p(rec), _p(depth), _p(tiles), _p(rect),
                              threads or default_threads())
    return dict(rec=rec, depth=depth, tiles=tiles, rect=rect, nonfinite=bool(nf))


def bin_sort(proj, W: int, H: int):
    tiles, rect, depth = proj["tiles"], proj["rect"], proj["depth"]
    V, n_pad = tiles.shape
    K = int(tiles.astype(np.int64).sum())
    T = ((W + 15) // 16) * ((H + 15) // 16)
    offsets = np.zeros((V, n_pad), np.uint32)
    ke = np.zeros(max(K, 1), np.uint64)
    ve = np.zeros(max(K, 1), np.uint32)
    ks = np.zeros(max(K, 1), np.uint64)
    vs = np.zeros(max(K, 1), np.uint32)
    ranges = np.zeros((V * T, 2), np.uint32)
    got = lib().oracle_bin(n_pad, V, W, H, _p(tiles), _p(rect), _p(depth), _p(offsets), _p(ke), _p(ve), _p(ks), _p(vs),
                           _p(ranges), K)
    assert got == K
    return dict(offsets=offsets, K=K, keys_emit=ke[:K], vals_emit=ve[:K], keys=ks[:K], vals=vs[:K], ranges=ranges)


def rasterize(proj, bins, W: int, H: int, bg=(0.0, 0.0, 0.0), threads: int | None = None):
    rec = proj["rec"]
    V, n_pad, _ = rec.shape
    rgb = np.zeros((V, 3, H, W), np.float32)
    T = np.zeros((V, H, W), np.float32)
    bgv = np.asarray(bg, np.float32)
    vals = bins["vals"] if bins["K"] else np.zeros(1, np.uint32)
    lib().oracle_rasterize(n_pad, V, W, H, _p(rec), _p(bins["ranges"]), _p(np.ascontiguousarray(vals)), _p(bgv), _p(rgb), _p(T),
                           threads or default_threads())
    return rgb, T


def rasterize_pixels(rec: np.ndarray, ranges: np.ndarray, vals: np.ndarray, W: int, H: int, pix: np.ndarray,
                     bg=(0.0, 0.0, 0.0), threads: int | None = None):
    """Composite only the sampled pixels pix[(v, x, y)] (full-size parity checks)."""
    rec = np.ascontiguousarray(rec, np.float32)
    n_pad = rec.shape[1]
    pix = np.ascontiguousarray(pix, np.int32)
    rgb = np.zeros((pix.shape[0], 3), np.float32)
    T = np.zeros(pix.shape[0], np.float32)
    bgv = np.asarray(bg, np.float32)
    vals = np.ascontiguousarray(vals if vals.size else np.zeros(1, np.uint32), np.uint32)
    lib().oracle_rasterize_pixels(n_pad, W, H, _p(rec), _p(np.ascontiguousarray(ranges, np.uint32)), _p(vals), _p(bgv),
                                  pix.shape[0], _p(pix), _p(rgb), _p(T), threads or default_threads())
    return rgb, T


def rasterize_bruteforce(proj, n: int, W: int, H: int, bg=(0.0, 0.0, 0.0), threads: int | None = None):
    rec = proj["rec"]
    V, n_pad, _ = rec.shape
    rgb = np.zeros((V, 3, H, W), np.float32)
    T = np.zeros((V, H, W), np.float32)
    bgv = np.asarray(bg, np.float32)
    lib().oracle_rasterize_bruteforce(n, n_pad, V, W, H, _p(rec), _p(proj["depth"]), _p(bgv), _p(rgb), _p(T),
                                      threads or default_threads())
    return rgb, T


def blend_counts(proj, bins, W: int, H: int, threads: int | None = None):
    rec = proj["rec"]
    V, n_pad, _ = rec.shape
    ev = np.zeros(V, np.int64)
    cp = np.zeros(V, np.int64)
    vals = bins["vals"] if bins["K"] else np.zeros(1, np.uint32)
    lib().oracle_blend_counts(n_pad, V, W, H, _p(rec), _p(bins["ranges"]), _p(np.ascontiguousarray(vals)), _p(ev), _p(cp),
                              threads or default_threads())
    return ev, cp


def render(planes, n: int, deg: int, cams, bg=(0.0, 0.0, 0.0), threads: int | None = None):
    """project -> bin/sort -> rasterize for a batch of equally-sized views."""
    W, H = cams[0].width, cams[0].height
    proj = project(planes, n, deg, cams, threads)
    bins = bin_sort(proj, W, H)
    rgb, T = rasterize(proj, bins, W, H, bg, threads)
    return proj, bins, rgb, T


# ----------------------------------------------------------------------------- NEXT #3
def dilate(marks: np.ndarray, d: int) -> np.ndarray:
    """Square d x d dilation of boolean marks [..., H, W], clipped at the borders: output (x, y)
    is set iff a mark lies in [x - d//2, x - d//2 + d - 1] x [y - d//2, y - d//2 + d - 1]
    ("dilate the image mask by a 48x48 kernel"; anchor = centre of the kernel, the
    convention of a centred structuring element).  Window sums of a 2D prefix-sum table."""
    m = np.asarray(marks, bool)
    H, W = m.shape[-2:]
    a = d // 2
    S = np.zeros(m.shape[:-2] + (H + 1, W + 1), np.int64)
    S[..., 1:, 1:] = m.astype(np.int64).cumsum(-2).cumsum(-1)
    y = np.arange(H)
    x = np.arange(W)
    y0, y1 = np.clip(y - a, 0, H), np.clip(y - a + d, 0, H)
    x0, x1 = np.clip(x - a, 0, W), np.clip(x - a + d, 0, W)
    tot = (S[..., y1[:, None], x1[None, :]] - S[..., y0[:, None], x1[None, :]]
           - S[..., y1[:, None], x0[None, :]] + S[..., y0[:, None], x0[None, :]])
    return tot > 0


def render_mask(planes: np.ndarray, n: int, deg: int, cams, subset, alpha_thresh: float = 1e-3, dilation: int = 48,
                threads: int | None = None) -> np.ndarray:
    """Masked / dynamic-subset rendering: render only the
    Gaussians in `subset` (ascending indices), mark pixels with accumulated alpha 1 - T >
    alpha_thresh, dilate.  Rendering the subset alone = rendering the scene restricted to those
    columns (same per-Gaussian arithmetic; the index order, hence the depth tie-break, is
    preserved).  Returns uint8 [V][H][W]."""
    subset = np.asarray(subset, np.int64)
    W, H = cams[0].width, cams[0].height
    V = len(cams)
    if subset.size == 0:
        return np.zeros((V, H, W), np.uint8)
    k = subset.size
    kp = max(4, (k + 3) // 4 * 4)
    sub = np.zeros((planes.shape[0], kp), np.float32)
    sub[:, :k] = planes[:, subset]
    _, _, _, T = render(sub, k, deg, cams, threads=threads)
    marks = (np.float32(1.0) - T) > np.float32(alpha_thresh)
    return dilate(marks, dilation).astype(np.uint8)


# ----------------------------------------------------------------------------- NEXT #2
def densify(planes: np.ndarray, n: int, rem, add16, n_pad_out: int | None = None):
    """Densification delta (DESIGN reading R21): the set without the removed columns
    (survivors in order) followed by the additions (binary16 raw parameters -> float32, exact).
    Returns (planes_out [P][n_pad_out], n_out, status) with status -3 for a removal list that is
    not strictly increasing or out of range (planes_out then None)."""
    rem = np.asarray(rem, np.int64)
    add = np.asarray(add16, np.float16)
    if rem.size and (rem.min() < 0 or rem.max() >= n or np.any(np.diff(rem) <= 0)):
        return None, 0, -3
    keep = np.ones(n, bool)
    keep[rem] = False
    cols = [planes[:, :n][:, keep], add.astype(np.float32)]
    body = np.concatenate(cols, axis=1)
    n_out = body.shape[1]
    n_pad_out = max(4, (n_out + 3) // 4 * 4) if n_pad_out is None else n_pad_out
    out = np.zeros((planes.shape[0], n_pad_out), np.float32)
    out[:, :n_out] = body
    return out, n_out, 0


# ----------------------------------------------------------------------------- NEXT #4 support
def contributors(proj, bins, W: int, H: int, threads: int | None = None):
    """Per-pixel contributor lists of the forward compositing (fp32 decisions, exactly a12's):
    CSR (offsets [V*H*W+1] int64, gid int32, clamped uint8), pixel index = (v*H + y)*W + x."""
    rec = proj["rec"]
    V, n_pad, _ = rec.shape
    th = threads or default_threads()
    vals = bins["vals"] if bins["K"] else np.zeros(1, np.uint32)
    vals = np.ascontiguousarray(vals)
    counts = np.zeros(V * H * W, np.int32)
    lib().oracle_contrib(n_pad, V, W, H, _p(rec), _p(bins["ranges"]), _p(vals), _p(counts), None, None, None, th)
    offsets = np.zeros(V * H * W + 1, np.int64)
    offsets[1:] = np.cumsum(counts)
    gid = np.zeros(max(1, int(offsets[-1])), np.int32)
    clamp = np.zeros(max(1, int(offsets[-1])), np.uint8)
    lib().oracle_contrib(n_pad, V, W, H, _p(rec), _p(bins["ranges"]), _p(vals), _p(counts), _p(offsets), _p(gid),
                         _p(clamp), th)
    return offsets, gid[:offsets[-1]], clamp[:offsets[-1]]


def rasterize_pixels_direct(proj, n: int, W: int, H: int, pix: np.ndarray, bg=(0.0, 0.0, 0.0),
                            threads: int | None = None):
    """Sampled pixels from the projection records alone (no binning; R13: tiled == brute
    force).  pix int32 [npix][3] = (view, x, y).  Returns rgb [npix][3], T [npix]."""
    rec = proj["rec"]
    V, n_pad, _ = rec.shape
    pix = np.ascontiguousarray(pix, np.int32)
    rgb = np.zeros((pix.shape[0], 3), np.float32)
    T = np.zeros(pix.shape[0], np.float32)
    lib().oracle_rasterize_pixels_direct(n, n_pad, W, H, _p(rec), _p(proj["depth"]), _p(proj["tiles"]),
                                         _p(proj["rect"]), _p(np.asarray(bg, np.float32)), pix.shape[0], _p(pix),
                                         _p(rgb), _p(T), threads or default_threads())
    return rgb, T
