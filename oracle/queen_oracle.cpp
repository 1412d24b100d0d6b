// QUEEN per-frame decode -> apply -> 3D-GS splat: CPU ORACLE.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  The product path
// (paper_2412_04469_b200/) never links, imports or executes anything under oracle/,
// and this file shares no code, header, table or constant generator with csrc/.
//
// Plain, slow, literal scalar C++17.  Each function cites the passage it follows:
//   P:n  = /root/reference/PAPER.md line n (section / equation named beside it)
//   S:n  = /root/reference/SPEC.md line n (interfaces / test ideas only)
//   R#n  = DESIGN.md reading #n (where the paper is silent)
//
// Arithmetic contract: IEEE fp32, round to
// nearest even, no FMA contraction (compiled with -ffp-contract=off, no fast-math),
// fmaf() only where written.  The operation order below IS the contract that the
// GPU path reproduces bit-for-bit for every value that decides an integer (cull,
// tile rect, skip test, mask, quantised latent).  OpenMP is used only to spread
// independent elements over host cores for timing; it never changes per-element
// arithmetic or any result.
//
// Parity pins: every function here is pinned by tests/test_oracle_*.py against
// closed forms, paper/SPEC worked examples, invariants, brute force and double
// precision.  No function is "parity unpinned".

#pragma STDC FP_CONTRACT OFF
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <tuple>
#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

// ---------------------------------------------------------------------------
// bit helpers
// ---------------------------------------------------------------------------
static inline float f_from_bits(uint32_t b) { float f; std::memcpy(&f, &b, 4); return f; }
static inline uint32_t bits_of(float f) { uint32_t b; std::memcpy(&b, &f, 4); return b; }

// ---------------------------------------------------------------------------
// det_exp / det_log: deterministic exp / log built only from IEEE + - * / fmaf
// rintf fminf fmaxf and bit casts (R#8).  The exp / log are
// the activations of the 3D-GS parameterisation the paper builds on (P:213-215,
// scale s = exp(log s), opacity = sigmoid(logit)) and of the hard-concrete gate
// sigmoid.  Pinned against double libm (<= 2 ulp) in tests.
// ---------------------------------------------------------------------------
float oracle_det_exp(float x) {
    const float L2E = f_from_bits(0x3fb8aa3bu);     // log2(e)
    const float LN2_HI = f_from_bits(0x3f317200u);  // 6.9314575195e-01
    const float LN2_LO = f_from_bits(0x35bfbe8eu);  // 1.4286067653e-06
    x = std::fmin(std::fmax(x, -87.0f), 88.0f);
    float k = std::rint(x * L2E);
    float r = std::fma(-k, LN2_HI, x);
    r = std::fma(-k, LN2_LO, r);
    // Taylor series of e^r, Horner, degree 7
    float p = 1.0f / 5040.0f;
    p = std::fma(p, r, 1.0f / 720.0f);
    p = std::fma(p, r, 1.0f / 120.0f);
    p = std::fma(p, r, 1.0f / 24.0f);
    p = std::fma(p, r, 1.0f / 6.0f);
    p = std::fma(p, r, 0.5f);
    p = std::fma(p, r, 1.0f);
    p = std::fma(p, r, 1.0f);
    int ki = (int)k;
    float scale = f_from_bits((uint32_t)(ki + 127) << 23);  // 2^k, k in [-126, 127]
    return p * scale;
}

float oracle_det_log(float y) {  // y: normal, > 0
    const float LN2_HI = f_from_bits(0x3f317200u);
    const float LN2_LO = f_from_bits(0x35bfbe8eu);
    uint32_t b = bits_of(y);
    int e = (int)((b >> 23) & 255u) - 127;
    float m = f_from_bits((b & 0x7fffffu) | 0x3f800000u);  // m in [1, 2)
    if (m > 1.41421356f) { m = m * 0.5f; e += 1; }
    float f = m - 1.0f;
    float s = f / (2.0f + f);
    float z = s * s;
    // ln(1+f) = 2 atanh(s) = 2s + s*R(z), R = z*(2/3 + 2/5 z + 2/7 z^2 + 2/9 z^3)
    float R = std::fma(z, 2.0f / 9.0f, 2.0f / 7.0f);
    R = std::fma(z, R, 2.0f / 5.0f);
    R = std::fma(z, R, 2.0f / 3.0f);
    R = z * R;
    float hfsq = (0.5f * f) * f;
    float lnm = f - (hfsq - s * (hfsq + R));
    float ef = (float)e;
    return std::fma(ef, LN2_HI, std::fma(ef, LN2_LO, lnm));
}

// ---------------------------------------------------------------------------
// a1. Quantise trainer-state latents: l = round(l_hat) (Eq. 5 "rounded
// to the nearest integer"); tie rule half away from zero (R#5).  Returns the
// number of entries whose |l| > 127 (wire range, R#4); those are stored clamped.
// ---------------------------------------------------------------------------
int64_t oracle_quantize(const float* lhat, int8_t* q, int64_t count) {
    int64_t bad = 0;
    for (int64_t j = 0; j < count; ++j) {
        float r = std::round(lhat[j]);  // C round(): half away from zero
        if (!(r >= -127.0f && r <= 127.0f)) { ++bad; r = r < 0 ? -127.0f : 127.0f; }
        q[j] = (int8_t)(int)r;
    }
    return bad;
}

// residual dimension M_c per category (rot, scale, opacity, sh_dc, sh_rest):
// P:290-292 footnote (categories), P:447 (separate decoders), R#2/R#3.
static void category_m(int deg, int M[5]) {
    int B = (deg + 1) * (deg + 1);
    M[0] = 4; M[1] = 3; M[2] = 1; M[3] = 3; M[4] = 3 * (B - 1);
}

// ---------------------------------------------------------------------------
// a2. Latent decode r_i = D . float(l_i) (Eq. 5), one decoder per
// category per frame.  Accumulation order (R#7): ascending k,
// from +0.0f, one fmaf per term.  resid: float [sum M_c][n_pad], row m of
// category c at row (sum_{c'<c} M_c') + m, which is plane 3 + that row.
// ---------------------------------------------------------------------------
void oracle_decode(int n, int n_pad, int deg, const int* lat, const int8_t* q,
                   const float* dec, float* resid) {
    int M[5];
    category_m(deg, M);
    int lat_row = 0, dec_off = 0, out_row = 0;
    for (int c = 0; c < 5; ++c) {
        int L = lat[c];
        if (L == 0) { out_row += M[c]; continue; }  // category absent: residual 0
        for (int m = 0; m < M[c]; ++m) {
            for (int i = 0; i < n; ++i) {
                float r = +0.0f;
                for (int k = 0; k < L; ++k)
                    r = std::fma(dec[dec_off + m * L + k], (float)q[(int64_t)(lat_row + k) * n_pad + i], r);
                resid[(int64_t)(out_row + m) * n_pad + i] = r;
            }
        }
        lat_row += L;
        dec_off += M[c] * L;
        out_row += M[c];
    }
    // category with L == 0: rows already counted; write zeros for them
    out_row = 0;
    for (int c = 0; c < 5; ++c) {
        if (lat[c] == 0)
            for (int m = 0; m < M[c]; ++m)
                for (int i = 0; i < n; ++i) resid[(int64_t)(out_row + m) * n_pad + i] = 0.0f;
        out_row += M[c];
    }
}

// ---------------------------------------------------------------------------
// First-frame quantisation ("First-frame Quantization"): only frame 0's
// high-frequency SH coefficients (DC excluded) are stored as integer latents + a decoder.
// They are decoded once and written (A_0 is set, not updated): SH-rest coefficient m
// (m = 3 (b - 1) + ch, plane 14 + m) of Gaussian i = D[m] . float(l_i), same accumulation
// order as a2 (R#7).  q: int8 [L][n_pad]; dec: [3(B-1)][L]; planes: [11+3B][n_pad].
// ---------------------------------------------------------------------------
void oracle_set_sh_rest(int n, int n_pad, int deg, int L, const int8_t* q, const float* dec, float* planes) {
    const int B = (deg + 1) * (deg + 1);
    for (int m = 0; m < 3 * (B - 1); ++m)
        for (int i = 0; i < n; ++i) {
            float r = +0.0f;
            for (int k = 0; k < L; ++k) r = std::fma(dec[m * L + k], (float)q[(int64_t)k * n_pad + i], r);
            planes[(int64_t)(14 + m) * n_pad + i] = r;
        }
}

// ---------------------------------------------------------------------------
// a3 + a5. Apply A_t = A_{t-1} + R_t (Eq. 4) on the raw non-position
// planes (R#1), then the COO position residual p[I_k] += E_p[k].
// planes: float [11+3B][n_pad]; non-position plane 3+row receives resid row.
// Returns 0, or -3 if a COO index is >= n or indices are not strictly increasing.
// ---------------------------------------------------------------------------
int oracle_apply(int n, int n_pad, int deg, const int* lat, const int8_t* q, const float* dec,
                 float* planes, int k, const uint32_t* idx, const float* val) {
    int M[5];
    category_m(deg, M);
    int Mtot = M[0] + M[1] + M[2] + M[3] + M[4];
    std::vector<float> resid((size_t)Mtot * n_pad, 0.0f);
    oracle_decode(n, n_pad, deg, lat, q, dec, resid.data());
    for (int m = 0; m < Mtot; ++m)
        for (int i = 0; i < n; ++i)
            planes[(int64_t)(3 + m) * n_pad + i] = planes[(int64_t)(3 + m) * n_pad + i] + resid[(int64_t)m * n_pad + i];
    int err = 0;
    for (int j = 0; j < k; ++j) {
        if (idx[j] >= (uint32_t)n || (j > 0 && idx[j] <= idx[j - 1])) { err = -3; continue; }
        for (int d = 0; d < 3; ++d)
            planes[(int64_t)d * n_pad + idx[j]] = planes[(int64_t)d * n_pad + idx[j]] + val[(int64_t)d * k + j];
    }
    return err;
}

// ---------------------------------------------------------------------------
// a4. Hard-concrete gate: g_hat = sigmoid(log alpha / tau),
// g_tilde = g_hat (gamma1 - gamma0) + gamma0, g = min(1, max(0, g_tilde)).
// Deterministic at inference (R#6).  The sigmoid is 1/(1+det_exp(-x)).
// ---------------------------------------------------------------------------
float oracle_gate_value(float log_alpha, float tau, float gamma0, float gamma1) {
    float ghat = 1.0f / (1.0f + oracle_det_exp((-log_alpha) / tau));
    float gt = std::fma(ghat, gamma1 - gamma0, gamma0);
    return std::fmin(1.0f, std::fmax(0.0f, gt));
}

// Gate -> mask -> COO (P:319-320 dp = g l_p; P:1389 I = {i : g_i != 0}).
// mask_i = (log alpha_i > theta0), theta0 = tau ln(-gamma0/gamma1) computed in
// double by the caller and rounded to float (R#6: the exact threshold where
// g_tilde crosses 0; the same shift as Eq. 8).  Writes ascending indices
// and values dp = g * l_p ([3][n_pad] layout in, [3][cap] out).  Returns k.
// ---------------------------------------------------------------------------
int oracle_gate(int n, int n_pad, const float* log_alpha, const float* lp, float tau, float gamma0,
                float gamma1, float theta0, uint32_t* idx_out, float* val_out, int cap) {
    int k = 0;
    for (int i = 0; i < n; ++i) {
        if (!(log_alpha[i] > theta0)) continue;
        float g = oracle_gate_value(log_alpha[i], tau, gamma0, gamma1);
        if (k < cap) {
            idx_out[k] = (uint32_t)i;
            for (int d = 0; d < 3; ++d) val_out[(int64_t)d * cap + k] = g * lp[(int64_t)d * n_pad + i];
        }
        ++k;
    }
    return k;
}

// ---------------------------------------------------------------------------
// Real SH basis, degree <= 3, 3D-GS constants and signs (R#10; "view-
// dependent RGB value c_i computed from h_i").  Pinned in tests against
// scipy.special spherical harmonics and quadrature orthonormality.
// ---------------------------------------------------------------------------
void oracle_sh_basis(int deg, float x, float y, float z, float* Y) {
    const float C0 = 0.28209479177387814f;
    const float C1 = 0.4886025119029199f;
    const float C2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                         -1.0925484305920792f, 0.5462742152960396f};
    const float C3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f, 0.3731763325901154f,
                         -0.4570457994644658f, 1.445305721320277f, -0.5900435899266435f};
    Y[0] = C0;
    if (deg < 1) return;
    Y[1] = -C1 * y;
    Y[2] = C1 * z;
    Y[3] = -C1 * x;
    if (deg < 2) return;
    float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    Y[4] = C2[0] * xy;
    Y[5] = C2[1] * yz;
    Y[6] = C2[2] * (2.0f * zz - xx - yy);
    Y[7] = C2[3] * xz;
    Y[8] = C2[4] * (xx - yy);
    if (deg < 3) return;
    Y[9] = C3[0] * y * (3.0f * xx - yy);
    Y[10] = C3[1] * xy * z;
    Y[11] = C3[2] * y * (4.0f * zz - xx - yy);
    Y[12] = C3[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    Y[13] = C3[4] * x * (4.0f * zz - xx - yy);
    Y[14] = C3[5] * z * (xx - yy);
    Y[15] = C3[6] * x * (xx - 3.0f * yy);
}

// camera record: 24 words  fx fy cx cy R[9] t[3] C[3] limx limy near | width height (int32)
struct Cam {
    float fx, fy, cx, cy, R[9], t[3], C[3], limx, limy, near_z;
    int W, H;
};
static Cam load_cam(const float* w) {
    Cam c;
    c.fx = w[0]; c.fy = w[1]; c.cx = w[2]; c.cy = w[3];
    for (int j = 0; j < 9; ++j) c.R[j] = w[4 + j];
    for (int j = 0; j < 3; ++j) { c.t[j] = w[13 + j]; c.C[j] = w[16 + j]; }
    c.limx = w[19]; c.limy = w[20]; c.near_z = w[21];
    std::memcpy(&c.W, &w[22], 4);
    std::memcpy(&c.H, &w[23], 4);
    return c;
}

// ---------------------------------------------------------------------------
// a6 + a7. Projection of Gaussian i into view v (Eq. 1; colour P:226).
// Records (R#13, R#14): rec[12] = u, v, hx, hy | A2, B2, C2, T2 | o, r, g, b
//   A2,B2,C2 = base-2 conic: p2 = A2 dx^2 + B2 dx dy + C2 dy^2 = -0.5 log2(e) d^T S'^-1 d
//   T2 = log2(1/(255 o)): alpha < 1/255  <=>  p2 < T2
//   hx, hy = 1.0001 sqrt(e2 S'_xx), 1.0001 sqrt(e2 S'_yy): half-extents of the ellipse
//   d^T S'^-1 d <= e2 = 2 ln(255 o) (where alpha reaches 1/255) -- its tight axis-aligned
//   bounding box, with 1e-4 relative slack
// depth = bits(z_c); rect = 16x16 tiles overlapping [u +- ceil(hx)] x [v +- ceil(hy)]
// (tx0, ty0, tx1, ty1 inclusive); tiles = their number.  A culled Gaussian gets zeros.
// Returns 1 if any Gaussian had a non-finite input (culled + QUEEN_WARN_NONFINITE).
// ---------------------------------------------------------------------------
static int project_one(int i, int n_pad, int deg, const float* pl, const Cam& c, float* rec, uint32_t* depth,
                       uint32_t* tiles, int16_t* rect) {
    const int B = (deg + 1) * (deg + 1);
    const int P = 11 + 3 * B;
    for (int j = 0; j < 12; ++j) rec[j] = 0.0f;
    *depth = 0; *tiles = 0;
    rect[0] = rect[1] = rect[2] = rect[3] = 0;
    // 0. non-finite input -> cull (must precede fminf/fmaxf, which would hide a NaN)
    for (int p = 0; p < P; ++p)
        if (!std::isfinite(pl[(int64_t)p * n_pad + i])) return 1;
    const float px = pl[0 * (int64_t)n_pad + i], py = pl[1 * (int64_t)n_pad + i], pz = pl[2 * (int64_t)n_pad + i];
    // 1. camera transform x_c = W p (P:220 viewing transform W), near cull (R#11)
    const float* Rw = c.R;
    float xc = std::fma(Rw[0], px, std::fma(Rw[1], py, std::fma(Rw[2], pz, c.t[0])));
    float yc = std::fma(Rw[3], px, std::fma(Rw[4], py, std::fma(Rw[5], pz, c.t[1])));
    float zc = std::fma(Rw[6], px, std::fma(Rw[7], py, std::fma(Rw[8], pz, c.t[2])));
    if (!(zc > c.near_z)) return 0;
    // 2. quaternion normalisation ("rotation matrix parameterized by a quaternion")
    float qw = pl[3 * (int64_t)n_pad + i], qx = pl[4 * (int64_t)n_pad + i], qy = pl[5 * (int64_t)n_pad + i],
          qz = pl[6 * (int64_t)n_pad + i];
    float n2 = std::fma(qw, qw, std::fma(qx, qx, std::fma(qy, qy, qz * qz)));
    if (!(n2 > 0.0f)) return 0;
    float inv = 1.0f / std::sqrt(n2);
    qw = qw * inv; qx = qx * inv; qy = qy * inv; qz = qz * inv;
    // 3. Sigma = R S S^T R^T, s = exp(log s) (R#8)
    float s[3];
    for (int j = 0; j < 3; ++j) s[j] = oracle_det_exp(pl[(int64_t)(7 + j) * n_pad + i]);
    float Rq[9];
    Rq[0] = 1.0f - 2.0f * std::fma(qy, qy, qz * qz);
    Rq[1] = 2.0f * (qx * qy - qw * qz);
    Rq[2] = 2.0f * (qx * qz + qw * qy);
    Rq[3] = 2.0f * (qx * qy + qw * qz);
    Rq[4] = 1.0f - 2.0f * std::fma(qx, qx, qz * qz);
    Rq[5] = 2.0f * (qy * qz - qw * qx);
    Rq[6] = 2.0f * (qx * qz - qw * qy);
    Rq[7] = 2.0f * (qy * qz + qw * qx);
    Rq[8] = 1.0f - 2.0f * std::fma(qx, qx, qy * qy);
    float Mm[9];
    for (int j = 0; j < 3; ++j)
        for (int m = 0; m < 3; ++m) Mm[j * 3 + m] = Rq[j * 3 + m] * s[m];
    float S[9];
    for (int j = 0; j < 3; ++j)
        for (int k = j; k < 3; ++k) {
            float v = std::fma(Mm[j * 3 + 0], Mm[k * 3 + 0], std::fma(Mm[j * 3 + 1], Mm[k * 3 + 1], Mm[j * 3 + 2] * Mm[k * 3 + 2]));
            S[j * 3 + k] = v;
            S[k * 3 + j] = v;
        }
    // 4. Jacobian of the affine approximation of the projective transform,
    //    with the 3D-GS 1.3x frustum clamp (R#11)
    //    (one reciprocal of z_c; DESIGN "Arithmetic contract")
    float iz = 1.0f / zc;
    float tx = xc * iz, ty = yc * iz;
    float j00 = c.fx * iz;
    float j02 = -(c.fx * std::fmin(c.limx, std::fmax(-c.limx, tx))) * iz;
    float j11 = c.fy * iz;
    float j12 = -(c.fy * std::fmin(c.limy, std::fmax(-c.limy, ty))) * iz;
    // 5. Sigma' = J W Sigma W^T J^T (Eq. 1) + 0.3 px^2 (R#11)
    float A[6];
    for (int m = 0; m < 3; ++m) {
        A[0 * 3 + m] = std::fma(j00, Rw[0 * 3 + m], j02 * Rw[2 * 3 + m]);
        A[1 * 3 + m] = std::fma(j11, Rw[1 * 3 + m], j12 * Rw[2 * 3 + m]);
    }
    float Bm[6];
    for (int r = 0; r < 2; ++r)
        for (int m = 0; m < 3; ++m)
            Bm[r * 3 + m] = std::fma(A[r * 3 + 0], S[0 * 3 + m], std::fma(A[r * 3 + 1], S[1 * 3 + m], A[r * 3 + 2] * S[2 * 3 + m]));
    float a = std::fma(Bm[0], A[0], std::fma(Bm[1], A[1], Bm[2] * A[2]));
    float b = std::fma(Bm[0], A[3], std::fma(Bm[1], A[4], Bm[2] * A[5]));
    float cc2 = std::fma(Bm[3], A[3], std::fma(Bm[4], A[4], Bm[5] * A[5]));
    a = a + 0.3f;
    cc2 = cc2 + 0.3f;
    // 6. conic = Sigma'^-1 (Eq. 2 exponent)
    float det = std::fma(a, cc2, -(b * b));
    if (!(det > 0.0f)) return 0;
    float idet = 1.0f / det;
    float ca = cc2 * idet, cb = -b * idet, ccn = a * idet;
    // 7. opacity o = sigmoid(logit) in [0,1]; alpha can reach 1/255 only if 255 o > 1 (R#14)
    float o = 1.0f / (1.0f + oracle_det_exp(-pl[10 * (int64_t)n_pad + i]));
    if (!(255.0f * o > 1.0f)) return 0;
    float e2 = 2.0f * oracle_det_log(255.0f * o);
    // 8. opacity-aware extent (R#13): the ellipse d^T S'^-1 d <= e2 has axis-aligned
    //    half-extents sqrt(e2 S'_xx), sqrt(e2 S'_yy); 1e-4 relative slack, integer radii
    float hx = 1.0001f * std::sqrt(e2 * a);
    float hy = 1.0001f * std::sqrt(e2 * cc2);
    float rx = std::ceil(hx), ry = std::ceil(hy);
    float u = std::fma(c.fx, tx, c.cx);
    float v = std::fma(c.fy, ty, c.cy);
    // 9. 16x16 tile rect (inclusive), clamped in float before the int conversion
    int gx = (c.W + 15) / 16, gy = (c.H + 15) / 16;
    float ftx0 = std::fmin(std::fmax(std::ceil(((u - rx) - 15.0f) * 0.0625f), 0.0f), (float)gx);
    float ftx1 = std::fmin(std::fmax(std::floor((u + rx) * 0.0625f), -1.0f), (float)(gx - 1));
    float fty0 = std::fmin(std::fmax(std::ceil(((v - ry) - 15.0f) * 0.0625f), 0.0f), (float)gy);
    float fty1 = std::fmin(std::fmax(std::floor((v + ry) * 0.0625f), -1.0f), (float)(gy - 1));
    int tx0 = (int)ftx0, tx1 = (int)ftx1, ty0 = (int)fty0, ty1 = (int)fty1;
    uint32_t nt = (tx0 <= tx1 && ty0 <= ty1) ? (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1)) : 0u;
    // 10. base-2 blend coefficients
    const float L2E = 1.4426950408889634f;
    float A2 = (-0.5f * ca) * L2E;
    float B2 = (-cb) * L2E;
    float C2 = (-0.5f * ccn) * L2E;
    float T2 = -(0.5f * e2) * L2E;
    // 11. view-dependent colour from SH, +0.5 and clamp at 0 (R#8)
    float dx = px - c.C[0], dy = py - c.C[1], dz = pz - c.C[2];
    float dn = std::sqrt(std::fma(dx, dx, std::fma(dy, dy, dz * dz)));
    float idn = 1.0f / dn;
    dx = dx * idn; dy = dy * idn; dz = dz * idn;
    float Y[16];
    oracle_sh_basis(deg, dx, dy, dz, Y);
    float rgb[3];
    for (int ch = 0; ch < 3; ++ch) {
        float acc = Y[0] * pl[(int64_t)(11 + ch) * n_pad + i];
        for (int bb = 1; bb < B; ++bb) acc = std::fma(Y[bb], pl[(int64_t)(11 + 3 * bb + ch) * n_pad + i], acc);
        rgb[ch] = std::fmax(0.0f, acc + 0.5f);
    }
    rec[0] = u; rec[1] = v; rec[2] = hx; rec[3] = hy;
    rec[4] = A2; rec[5] = B2; rec[6] = C2; rec[7] = T2;
    rec[8] = o; rec[9] = rgb[0]; rec[10] = rgb[1]; rec[11] = rgb[2];
    *depth = bits_of(zc);  // 12. depth key: z_c > 0 so its bits order like the float (R#15)
    *tiles = nt;
    rect[0] = (int16_t)tx0; rect[1] = (int16_t)ty0; rect[2] = (int16_t)tx1; rect[3] = (int16_t)ty1;
    return 0;
}

// batch of views: cams [V][24]; rec [V][n_pad][12]; depth/tiles [V][n_pad]; rect [V][n_pad][4]
int oracle_project(int n, int n_pad, int deg, const float* planes, int V, const float* cams, float* rec,
                   uint32_t* depth, uint32_t* tiles, int16_t* rect, int threads) {
    int nonfinite = 0;
    for (int v = 0; v < V; ++v) {
        Cam c = load_cam(cams + 24 * v);
        int nf = 0;
#pragma omp parallel for num_threads(threads) reduction(| : nf) schedule(static)
        for (int i = 0; i < n_pad; ++i) {
            int64_t o = (int64_t)v * n_pad + i;
            if (i >= n) {
                for (int j = 0; j < 12; ++j) rec[o * 12 + j] = 0.0f;
                depth[o] = 0; tiles[o] = 0;
                rect[o * 4 + 0] = rect[o * 4 + 1] = rect[o * 4 + 2] = rect[o * 4 + 3] = 0;
                continue;
            }
            nf |= project_one(i, n_pad, deg, planes, c, rec + o * 12, depth + o, tiles + o, rect + o * 4);
        }
        nonfinite |= nf;
    }
    return nonfinite;
}

// ---------------------------------------------------------------------------
// a8-a11. Scan / duplicate / sort / ranges over a batch of V views of one size
// (W x H, T = gx*gy tiles each).  Global tile id gt = v*T + ty*gx + tx.
//   offsets = exclusive prefix sum of tiles over the flattened [V][n_pad] array
//   key = (gt << 31) | depth_bits   (depth bits < 2^31: z_c > 0), val = i
//   emitted for (v, i) ascending, then ty ascending, then tx ascending
//   sorted ascending by (key, val)  (R#15: depth, ties by index; "depth-sorted")
//   ranges[gt] = [first, last+1) of gt in the sorted array, [0,0) if empty
// keys/vals arrays must hold K = offsets total; K is returned (or -1 if > cap).
// ---------------------------------------------------------------------------
int64_t oracle_bin(int n_pad, int V, int W, int H, const uint32_t* tiles, const int16_t* rect,
                   const uint32_t* depth, uint32_t* offsets, uint64_t* keys_emit, uint32_t* vals_emit,
                   uint64_t* keys_sorted, uint32_t* vals_sorted, uint32_t* ranges, int64_t cap) {
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int64_t T = (int64_t)gx * gy;
    int64_t total = 0;
    for (int64_t j = 0; j < (int64_t)V * n_pad; ++j) {
        offsets[j] = (uint32_t)total;
        total += tiles[j];
    }
    if (total > cap) return -1;
    for (int v = 0; v < V; ++v)
        for (int i = 0; i < n_pad; ++i) {
            int64_t j = (int64_t)v * n_pad + i;
            if (tiles[j] == 0) continue;
            int64_t w = offsets[j];
            const int16_t* r = rect + j * 4;
            for (int ty = r[1]; ty <= r[3]; ++ty)
                for (int tx = r[0]; tx <= r[2]; ++tx) {
                    uint64_t gt = (uint64_t)v * T + (uint64_t)ty * gx + tx;
                    keys_emit[w] = (gt << 31) | (uint64_t)depth[j];
                    vals_emit[w] = (uint32_t)i;
                    ++w;
                }
        }
    std::vector<std::pair<uint64_t, uint32_t>> kv((size_t)total);
    for (int64_t j = 0; j < total; ++j) kv[j] = {keys_emit[j], vals_emit[j]};
    std::sort(kv.begin(), kv.end());
    for (int64_t j = 0; j < total; ++j) { keys_sorted[j] = kv[j].first; vals_sorted[j] = kv[j].second; }
    for (int64_t t = 0; t < V * T; ++t) { ranges[2 * t] = 0; ranges[2 * t + 1] = 0; }
    for (int64_t j = 0; j < total; ++j) {
        uint64_t gt = keys_sorted[j] >> 31;
        if (j == 0 || (keys_sorted[j - 1] >> 31) != gt) ranges[2 * gt] = (uint32_t)j;
        if (j == total - 1 || (keys_sorted[j + 1] >> 31) != gt) ranges[2 * gt + 1] = (uint32_t)(j + 1);
    }
    return total;
}

// ---------------------------------------------------------------------------
// a12. Front-to-back compositing, Eq. 2: c = sum c_i a_i prod_{j<i}(1-a_j),
// a_i = o_i exp(-1/2 d^T S'^-1 d), over the pixel's tile list in depth order.
// 3D-GS cut-offs as read in R#14: skip when a_i < 1/255 (exact test p2 < T2), a_i
// clamped at 0.99, composite-then-stop when T < 1e-4.  p2 is mathematically <= 0 (the conic
// is positive definite); a positive computed p2 is rounding at the ellipse's centre and is
// composited like the centre (R#14; 3D-GS's "power > 0" skip is not kept).  Pixel (x, y)
// is sampled at ((float)x, (float)y) (R#12).  Output C + T*bg and T (R#16).
// ---------------------------------------------------------------------------
// record words: 0 u, 1 v, 4 A2, 5 B2, 6 C2, 7 T2, 8 o, 9-11 rgb (hx, hy unused here)
static inline float rec_p2(const float* rc, float fx, float fy) {
    // Horner in dy (DESIGN "Arithmetic contract"): p2 = (C2 dy + B2 dx) dy + (A2 dx) dx
    float dx = rc[0] - fx, dy = rc[1] - fy;
    return std::fma(std::fma(rc[6], dy, rc[5] * dx), dy, (rc[4] * dx) * dx);
}

static inline bool blend_step(const float* rc, float fx, float fy, float C[3], float& T) {
    float p2 = rec_p2(rc, fx, fy);
    if (p2 < rc[7]) return false;
    float alpha = std::fmin(0.99f, rc[8] * std::exp2(p2));
    float aT = alpha * T;
    C[0] = std::fma(rc[9], aT, C[0]);
    C[1] = std::fma(rc[10], aT, C[1]);
    C[2] = std::fma(rc[11], aT, C[2]);
    T = T * (1.0f - alpha);
    return T < 1e-4f;
}

void oracle_rasterize(int n_pad, int V, int W, int H, const float* rec, const uint32_t* ranges,
                      const uint32_t* vals_sorted, const float* bg, float* rgb_out, float* T_out, int threads) {
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int64_t T = (int64_t)gx * gy;
    for (int v = 0; v < V; ++v) {
#pragma omp parallel for num_threads(threads) schedule(dynamic, 4)
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                int64_t gt = (int64_t)v * T + (int64_t)(y >> 4) * gx + (x >> 4);
                float C[3] = {0.0f, 0.0f, 0.0f}, Tr = 1.0f;
                for (uint32_t j = ranges[2 * gt]; j < ranges[2 * gt + 1]; ++j) {
                    const float* rc = rec + ((int64_t)v * n_pad + vals_sorted[j]) * 12;
                    if (blend_step(rc, (float)x, (float)y, C, Tr)) break;
                }
                int64_t pix = (int64_t)y * W + x;
                for (int ch = 0; ch < 3; ++ch)
                    rgb_out[((int64_t)v * 3 + ch) * H * W + pix] = C[ch] + Tr * bg[ch];
                T_out[(int64_t)v * H * W + pix] = Tr;
            }
    }
}

// Same compositing for a list of sampled pixels (v, x, y) -- used to check full-size
// configurations pixel by pixel.  out: rgb [npix][3] (C + T*bg), T [npix].
void oracle_rasterize_pixels(int n_pad, int W, int H, const float* rec, const uint32_t* ranges,
                             const uint32_t* vals_sorted, const float* bg, int64_t npix, const int32_t* pix,
                             float* rgb_out, float* T_out, int threads) {
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int64_t T = (int64_t)gx * gy;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 16)
    for (int64_t q = 0; q < npix; ++q) {
        const int v = pix[3 * q], x = pix[3 * q + 1], y = pix[3 * q + 2];
        int64_t gt = (int64_t)v * T + (int64_t)(y >> 4) * gx + (x >> 4);
        float C[3] = {0.0f, 0.0f, 0.0f}, Tr = 1.0f;
        for (uint32_t j = ranges[2 * gt]; j < ranges[2 * gt + 1]; ++j) {
            const float* rc = rec + ((int64_t)v * n_pad + vals_sorted[j]) * 12;
            if (blend_step(rc, (float)x, (float)y, C, Tr)) break;
        }
        for (int ch = 0; ch < 3; ++ch) rgb_out[3 * q + ch] = C[ch] + Tr * bg[ch];
        T_out[q] = Tr;
    }
}

// Brute force: every non-culled Gaussian of the view (record o > 0), globally
// sorted by (depth, index), composited at every pixel with the same per-pixel
// arithmetic.  No tiles, no ranges.  Pins the tiled path bit-for-bit (R#13).
void oracle_rasterize_bruteforce(int n, int n_pad, int V, int W, int H, const float* rec, const uint32_t* depth,
                                 const float* bg, float* rgb_out, float* T_out, int threads) {
    for (int v = 0; v < V; ++v) {
        std::vector<std::pair<uint32_t, uint32_t>> order;
        for (int i = 0; i < n; ++i)
            if (rec[((int64_t)v * n_pad + i) * 12 + 8] > 0.0f) order.push_back({depth[(int64_t)v * n_pad + i], (uint32_t)i});
        std::sort(order.begin(), order.end());
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1)
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                float C[3] = {0.0f, 0.0f, 0.0f}, Tr = 1.0f;
                for (auto& di : order) {
                    const float* rc = rec + ((int64_t)v * n_pad + di.second) * 12;
                    if (blend_step(rc, (float)x, (float)y, C, Tr)) break;
                }
                int64_t pix = (int64_t)y * W + x;
                for (int ch = 0; ch < 3; ++ch)
                    rgb_out[((int64_t)v * 3 + ch) * H * W + pix] = C[ch] + Tr * bg[ch];
                T_out[(int64_t)v * H * W + pix] = Tr;
            }
    }
}

// Work counters for the blend roofline: evaluated (pixel, Gaussian)
// pairs and composited pairs, per view, for the tiled order.
void oracle_blend_counts(int n_pad, int V, int W, int H, const float* rec, const uint32_t* ranges,
                         const uint32_t* vals_sorted, int64_t* evaluated, int64_t* composited, int threads) {
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int64_t T = (int64_t)gx * gy;
    for (int v = 0; v < V; ++v) {
        int64_t ev = 0, cp = 0;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 4) reduction(+ : ev, cp)
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                int64_t gt = (int64_t)v * T + (int64_t)(y >> 4) * gx + (x >> 4);
                float C[3] = {0.0f, 0.0f, 0.0f}, Tr = 1.0f;
                for (uint32_t j = ranges[2 * gt]; j < ranges[2 * gt + 1]; ++j) {
                    const float* rc = rec + ((int64_t)v * n_pad + vals_sorted[j]) * 12;
                    ++ev;
                    float p2 = rec_p2(rc, (float)x, (float)y);
                    if (!(p2 < rc[7])) ++cp;
                    if (blend_step(rc, (float)x, (float)y, C, Tr)) break;
                }
            }
        evaluated[v] = ev;
        composited[v] = cp;
    }
}


// Sampled pixels straight from the projection records, no binning: for pixel (v, x, y) every
// Gaussian of view v whose tile rect contains the pixel's tile, ordered by (depth, index), then
// the same compositing (blend_step).  By R#13 (tiled == brute force) this equals the tiled
// rasterizer; it lets full-size configurations whose key lists are too large for oracle_bin be
// checked pixel by pixel.  out: rgb [npix][3] (C + T bg), T [npix].
void oracle_rasterize_pixels_direct(int n, int n_pad, int W, int H, const float* rec, const uint32_t* depth,
                                    const uint32_t* tiles, const int16_t* rect, const float* bg, int64_t npix,
                                    const int32_t* pix, float* rgb_out, float* T_out, int threads) {
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1)
    for (int64_t q = 0; q < npix; ++q) {
        const int v = pix[3 * q], x = pix[3 * q + 1], y = pix[3 * q + 2];
        const int tx = x >> 4, ty = y >> 4;
        std::vector<std::pair<uint32_t, uint32_t>> list;
        for (int i = 0; i < n; ++i) {
            const int64_t o = (int64_t)v * n_pad + i;
            if (!tiles[o]) continue;
            const int16_t* r = rect + o * 4;
            if (tx < r[0] || tx > r[2] || ty < r[1] || ty > r[3]) continue;
            list.push_back({depth[o], (uint32_t)i});
        }
        std::sort(list.begin(), list.end());
        float C[3] = {0.0f, 0.0f, 0.0f}, Tr = 1.0f;
        for (auto& di : list) {
            const float* rc = rec + ((int64_t)v * n_pad + di.second) * 12;
            if (blend_step(rc, (float)x, (float)y, C, Tr)) break;
        }
        (void)W; (void)H;
        for (int ch = 0; ch < 3; ++ch) rgb_out[3 * q + ch] = C[ch] + Tr * bg[ch];
        T_out[q] = Tr;
    }
}

// ---------------------------------------------------------------------------
// NEXT #4 support: the contributor list of every pixel -- the records a12 composites, in
// order, up to and including the one after which T < 1e-4 -- with the 0.99-clamp decision,
// taken in the forward pass's fp32 arithmetic (blend_step).  The gradient oracle
// (oracle/grad.py) differentiates Eq. 2 in float64 on exactly these lists.
// counts[V*H*W]; then lists at offsets[pix]: gid (Gaussian index), clamped (0/1).
void oracle_contrib(int n_pad, int V, int W, int H, const float* rec, const uint32_t* ranges, const uint32_t* vals_sorted,
                    int32_t* counts, const int64_t* offsets, int32_t* gid_out, uint8_t* clamp_out, int threads) {
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int64_t T = (int64_t)gx * gy;
    for (int v = 0; v < V; ++v) {
#pragma omp parallel for num_threads(threads) schedule(dynamic, 4)
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                const int64_t pix = ((int64_t)v * H + y) * W + x;
                int64_t gt = (int64_t)v * T + (int64_t)(y >> 4) * gx + (x >> 4);
                float C[3] = {0.0f, 0.0f, 0.0f}, Tr = 1.0f;
                int32_t c = 0;
                for (uint32_t j = ranges[2 * gt]; j < ranges[2 * gt + 1]; ++j) {
                    const float* rc = rec + ((int64_t)v * n_pad + vals_sorted[j]) * 12;
                    const float p2 = rec_p2(rc, (float)x, (float)y);
                    if (p2 < rc[7]) continue;
                    if (offsets) {
                        gid_out[offsets[pix] + c] = (int32_t)vals_sorted[j];
                        clamp_out[offsets[pix] + c] = rc[8] * std::exp2(p2) > 0.99f ? 1 : 0;
                    }
                    ++c;
                    if (blend_step(rc, (float)x, (float)y, C, Tr)) break;
                }
                counts[pix] = c;
            }
    }
}

// ---------------------------------------------------------------------------
// NEXT #1: entropy coding of the integer latents ("flattens our integer
// latent matrix for each attribute ... then encoded using standard entropy coding
// approaches such as arithmetic coding").  Plain reference codec for the "QAN2" stream of
// order-0 static model, probabilities normalised to 4096, rANS with a
// 32-bit state in [2^16, 2^32) and 16-bit renormalisation, the flattened matrix
// (row-major, k*n + i) cut into 8192-symbol chunks, each chunk split over 32 lanes
// (symbol p of a chunk belongs to lane p % 32), every lane an independent rANS coder with
// its own word sequence.  Decoding a lane: for t = 0.. : decode symbol 32 t + lane, then
// (if the state fell below 2^16) read the lane's next 16-bit word.  A chunk's words are
// lane 0's sequence, then lane 1's, ... (lane_count[c][l] words each).  Written from that
// text, independently of csrc/.
// ---------------------------------------------------------------------------
static void oracle_ans_freq(const uint64_t cnt[256], uint64_t total, uint16_t f[256]) {
    // deterministic normalisation: floor(count * 4096 / total), at least 1 for present
    // symbols; the remainder goes to (or, if negative, is taken from) the most frequent
    for (int s = 0; s < 256; ++s) f[s] = 0;
    int64_t sum = 0;
    int best = -1;
    for (int s = 0; s < 256; ++s) {
        if (cnt[s] == 0) continue;
        uint64_t v = cnt[s] * 4096u / total;
        if (v < 1) v = 1;
        f[s] = (uint16_t)v;
        sum += (int64_t)v;
        if (best < 0 || cnt[s] > cnt[best]) best = s;
    }
    if (best < 0) return;
    if (sum <= 4096) { f[best] = (uint16_t)(f[best] + (4096 - sum)); return; }
    while (sum > 4096) {
        int m = -1;
        for (int s = 0; s < 256; ++s)
            if (f[s] > 1 && (m < 0 || f[s] > f[m])) m = s;
        f[m] = (uint16_t)(f[m] - 1);
        --sum;
    }
}

// returns the stream size; writes it to out if out != NULL and cap is large enough
int64_t oracle_ans_encode(const int8_t* lat, int L, int n, int n_pad, uint8_t* out, int64_t cap) {
    const int64_t CH = 8192;
    const int64_t nsym = (int64_t)L * n;
    const int64_t nch = (nsym + CH - 1) / CH;
    uint64_t cnt[256] = {0};
    for (int64_t q = 0; q < nsym; ++q) cnt[(uint8_t)(lat[(q / n) * (int64_t)n_pad + q % n] + 128)]++;
    uint16_t f[256];
    oracle_ans_freq(cnt, nsym > 0 ? (uint64_t)nsym : 1u, f);
    uint32_t cum[256];
    uint32_t run = 0;
    for (int s = 0; s < 256; ++s) { cum[s] = run; run += f[s]; }
    std::vector<uint32_t> off(nch + 1, 0), st(nch * 32, 1u << 16);
    std::vector<uint16_t> lcount(nch * 32, 0);
    std::vector<uint16_t> words;
    for (int64_t c = 0; c < nch; ++c) {
        const int64_t len = std::min(CH, nsym - c * CH);
        off[c] = (uint32_t)words.size();
        for (int l = 0; l < 32; ++l) {
            uint32_t x = 1u << 16;
            std::vector<uint16_t> emitted;  // in encoding order (reverse of decoding)
            for (int64_t p = ((len + 31) / 32) * 32 - 32 + l; p >= 0; p -= 32) {  // t descending
                if (p >= len) continue;
                const int64_t q = c * CH + p;
                const uint32_t s = (uint8_t)(lat[(q / n) * (int64_t)n_pad + q % n] + 128);
                if ((uint64_t)x >= ((uint64_t)f[s] << 20)) { emitted.push_back((uint16_t)(x & 0xffff)); x >>= 16; }
                x = (x / f[s]) * 4096u + x % f[s] + cum[s];
            }
            st[c * 32 + l] = x;
            lcount[c * 32 + l] = (uint16_t)emitted.size();
            for (int64_t q = (int64_t)emitted.size() - 1; q >= 0; --q) words.push_back(emitted[q]);
        }
    }
    off[nch] = (uint32_t)words.size();
    const int64_t fixed = 528 + 4 * (nch + 1) + 4 * 32 * nch + 2 * 32 * nch;
    const int64_t bytes = fixed + ((2 * (int64_t)words.size() + 3) / 4) * 4;
    if (!out || cap < bytes) return bytes;
    std::memset(out, 0, bytes);
    const uint32_t hdr[4] = {0x324e4151u, (uint32_t)nsym, (uint32_t)nch, 0u};
    std::memcpy(out, hdr, 16);
    std::memcpy(out + 16, f, 512);
    std::memcpy(out + 528, off.data(), 4 * (nch + 1));
    std::memcpy(out + 528 + 4 * (nch + 1), st.data(), 4 * 32 * nch);
    std::memcpy(out + 528 + 4 * (nch + 1) + 4 * 32 * nch, lcount.data(), 2 * 32 * nch);
    if (!words.empty()) std::memcpy(out + fixed, words.data(), 2 * words.size());
    return bytes;
}

// decode into lat[L][n_pad]; returns 0, or -3 for a corrupt / mismatched stream
int oracle_ans_decode(const uint8_t* in, int64_t bytes, int L, int n, int n_pad, int8_t* lat) {
    if (bytes < 528) return -3;
    uint32_t hdr[4];
    std::memcpy(hdr, in, 16);
    if (hdr[0] != 0x324e4151u || (int64_t)hdr[1] != (int64_t)L * n) return -3;
    const int64_t CH = 8192, nsym = hdr[1], nch = hdr[2];
    if (nch != (nsym + CH - 1) / CH) return -3;
    uint16_t f[256];
    std::memcpy(f, in + 16, 512);
    uint32_t cum[256], run = 0;
    uint8_t sym[4096];
    for (int s = 0; s < 256; ++s) {
        cum[s] = run;
        for (uint32_t k = run; k < run + f[s] && k < 4096; ++k) sym[k] = (uint8_t)s;
        run += f[s];
    }
    if (run != 4096) return -3;
    const int64_t fixed = 528 + 4 * (nch + 1) + 4 * 32 * nch + 2 * 32 * nch;
    if (bytes < fixed) return -3;
    std::vector<uint32_t> off(nch + 1), st(nch * 32);
    std::vector<uint16_t> lcount(nch * 32);
    std::memcpy(off.data(), in + 528, 4 * (nch + 1));
    std::memcpy(st.data(), in + 528 + 4 * (nch + 1), 4 * 32 * nch);
    std::memcpy(lcount.data(), in + 528 + 4 * (nch + 1) + 4 * 32 * nch, 2 * 32 * nch);
    const uint8_t* wbase = in + fixed;
    const int64_t nwords = (bytes - fixed) / 2;
    int err = 0;
    for (int64_t c = 0; c < nch; ++c) {
        const int64_t len = std::min(CH, nsym - c * CH);
        int64_t ptr = off[c];
        for (int l = 0; l < 32; ++l) {
            uint32_t x = st[c * 32 + l];
            const int64_t end = ptr + lcount[c * 32 + l];
            for (int64_t p = l; p < len; p += 32) {
                const uint32_t slot = x & 4095u;
                const uint32_t s = sym[slot];
                x = f[s] * (x >> 12) + slot - cum[s];
                const int64_t q = c * CH + p;
                lat[(q / n) * (int64_t)n_pad + q % n] = (int8_t)((int)s - 128);
                if (x < (1u << 16)) {
                    uint16_t w = 0;
                    if (ptr < end && ptr < nwords) std::memcpy(&w, wbase + 2 * ptr, 2);
                    else err = -3;
                    ++ptr;
                    x = (x << 16) | w;
                }
            }
            if (ptr != end || x != (1u << 16)) err = -3;
            ptr = end;
        }
        if (ptr != (int64_t)off[c + 1]) err = -3;
    }
    return err;
}

}  // extern "C"
