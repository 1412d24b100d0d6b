// NEXT #4: backward rasterizer -- gradients of the rendered images with respect
// to the per-(view, Gaussian) blend records (Eq. 2) and, through the projection
// (Eq. 1) and SH colour, to the raw Gaussian attributes (P:239-251 trains them).
//
// The forward's discrete decisions (skip test, 0.99 clamp, composite-then-stop, culls, Jacobian
// clamp, max(0, .) on colour) are re-taken in the forward's exact fp32 arithmetic and held
// fixed, i.e. this is the derivative of the piece the input lies in (the gradient oracle,
// oracle/grad.py, differentiates the same pieces in float64).
//
// k_blend_bwd   one 64-thread CTA per 16x16 tile, thread = 1 column x 4 rows (the forward's
//               mapping).  Phase A replays the forward per pixel (bit-identical T sequence,
//               hence the same last contributor and final T).  Phase B walks the tile's
//               records backwards from the last contributor, recovering T_i = T_{i+1}/(1-a_i):
//                 dL/dc_i = a_i T_i g,   dL/da_i = sum_ch g (c_i T_i - (S_i + T_N bg)/(1 - a_i))
//               (S_i = colour composited after i), then through a = o 2^p2 (unclamped) and
//               p2 = A2 dx^2 + B2 dx dy + C2 dy^2 to (u, v, A2, B2, C2, o, rgb).  Per record the
//               warp sums its lanes' contributions (shuffles) and one lane adds them to the
//               record's gradient with float atomics (accumulation order is not fixed).
// k_project_bwd one thread per Gaussian, all views in order (deterministic): record gradient
//               -> raw position, quaternion (through normalisation), log-scale, opacity
//               logit, SH coefficients.
#include "queen_internal.cuh"

namespace queen {

__device__ __forceinline__ float ex2b(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

constexpr int BW_RPT = 4;
constexpr int BW_NT = 256 / BW_RPT;  // 64 threads per tile
constexpr int BW_BATCH = 64;

__global__ void __launch_bounds__(BW_NT) k_blend_bwd(const float4* __restrict__ rec, int n_pad,
                                                     const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
                                                     int W, int H, int gx, int T, float bg0, float bg1, float bg2,
                                                     const float* __restrict__ gout, float* __restrict__ grec) {
    __shared__ float4 sA[BW_BATCH], sB[BW_BATCH], sC[BW_BATCH];
    __shared__ uint32_t sI[BW_BATCH];
    __shared__ int s_jmax[BW_NT / 32];
    const int gt = blockIdx.x;
    const int v = gt / T;
    const int t = gt - v * T;
    const int px = (t % gx) * 16 + (threadIdx.x & 15);
    const int py0 = (t / gx) * 16 + (threadIdx.x >> 4) * BW_RPT;
    const float fx = (float)px;
    const uint2 rg = ranges[gt];
    const int rs = (int)rg.x, re = (int)rg.y;
    const float4* vrec = rec + (int64_t)v * n_pad * 3;
    float Tf[BW_RPT];
    int last[BW_RPT];
#pragma unroll
    for (int r = 0; r < BW_RPT; ++r) {
        Tf[r] = (px < W && py0 + r < H) ? 1.0f : 0.0f;  // off-image pixels start terminated
        last[r] = -1;
    }
    // ---- phase A: replay the forward (same fp32 operations as k_blend / the oracle)
    for (int b0 = rs; b0 < re; b0 += BW_BATCH) {
        const int cnt = min(BW_BATCH, re - b0);
        __syncthreads();
        for (int q = threadIdx.x; q < cnt; q += BW_NT) {
            const float4* g = vrec + (int64_t)vals[b0 + q] * 3;
            sA[q] = g[0];
            sB[q] = g[1];
            sC[q] = g[2];
        }
        __syncthreads();
        for (int q = 0; q < cnt; ++q) {
            const float4 a = sA[q], bq = sB[q];
            const float dx = a.x - fx;
            const float tA = bq.x * dx, tB = bq.y * dx;
#pragma unroll
            for (int r = 0; r < BW_RPT; ++r) {
                if (Tf[r] < 1e-4f) continue;
                const float dy = a.y - (float)(py0 + r);
                const float p2 = fmaf(tA, dx, fmaf(bq.z * dy, dy, tB * dy));
                if (p2 > 0.0f || p2 < bq.w) continue;
                const float alpha = fminf(0.99f, sC[q].x * ex2b(p2));
                Tf[r] = Tf[r] * (1.0f - alpha);
                last[r] = b0 + q;
            }
        }
    }
    // ---- phase B: reverse walk
    int jmax = -1;
#pragma unroll
    for (int r = 0; r < BW_RPT; ++r) jmax = max(jmax, last[r]);
    for (int o = 16; o > 0; o >>= 1) jmax = max(jmax, __shfl_xor_sync(0xffffffffu, jmax, o));
    if ((threadIdx.x & 31) == 0) s_jmax[threadIdx.x >> 5] = jmax;
    __syncthreads();
    jmax = max(s_jmax[0], s_jmax[1]);
    const int64_t plane = (int64_t)H * W;
    float g[BW_RPT][3], S[BW_RPT][3], Tc[BW_RPT];
#pragma unroll
    for (int r = 0; r < BW_RPT; ++r) {
        const bool in = px < W && py0 + r < H;
        const int64_t pix = (int64_t)v * 3 * plane + (int64_t)(py0 + r) * W + px;
        g[r][0] = in ? gout[pix] : 0.f;
        g[r][1] = in ? gout[pix + plane] : 0.f;
        g[r][2] = in ? gout[pix + 2 * plane] : 0.f;
        S[r][0] = S[r][1] = S[r][2] = 0.f;
        Tc[r] = Tf[r];
    }
    const float bgc[3] = {bg0, bg1, bg2};
    const float LN2 = 0.69314718055994531f;
    for (int bend = jmax + 1; bend > rs; bend -= BW_BATCH) {
        const int b0 = max(rs, bend - BW_BATCH);
        const int cnt = bend - b0;
        __syncthreads();
        for (int q = threadIdx.x; q < cnt; q += BW_NT) {
            const uint32_t gi = vals[b0 + q];
            const float4* gp = vrec + (int64_t)gi * 3;
            sA[q] = gp[0];
            sB[q] = gp[1];
            sC[q] = gp[2];
            sI[q] = gi;
        }
        __syncthreads();
        for (int q = cnt - 1; q >= 0; --q) {
            const int j = b0 + q;
            const float4 a = sA[q], bq = sB[q], c = sC[q];
            const float dx = a.x - fx;
            const float tA = bq.x * dx, tB = bq.y * dx;
            float acc[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // u v A2 B2 C2 o r g b
            bool any = false;
#pragma unroll
            for (int r = 0; r < BW_RPT; ++r) {
                if (j > last[r]) continue;
                const float dy = a.y - (float)(py0 + r);
                const float p2 = fmaf(tA, dx, fmaf(bq.z * dy, dy, tB * dy));
                if (p2 > 0.0f || p2 < bq.w) continue;
                any = true;
                const float e = ex2b(p2);
                const float raw = c.x * e;
                const float alpha = fminf(0.99f, raw);
                const float om = 1.0f - alpha;
                const float Ti = Tc[r] / om;
                const float w = alpha * Ti;
                const float col[3] = {c.y, c.z, c.w};
                float dal = 0.f;
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    acc[6 + ch] += w * g[r][ch];
                    dal += g[r][ch] * (col[ch] * Ti - (S[r][ch] + Tf[r] * bgc[ch]) / om);
                    S[r][ch] += col[ch] * w;
                }
                Tc[r] = Ti;
                if (raw <= 0.99f) {  // unclamped: a = o 2^p2
                    acc[5] += dal * e;
                    const float dp2 = dal * alpha * LN2;
                    acc[0] += dp2 * (2.0f * bq.x * dx + bq.y * dy);
                    acc[1] += dp2 * (bq.y * dx + 2.0f * bq.z * dy);
                    acc[2] += dp2 * dx * dx;
                    acc[3] += dp2 * dx * dy;
                    acc[4] += dp2 * dy * dy;
                }
            }
            if (__any_sync(0xffffffffu, any)) {
#pragma unroll
                for (int k = 0; k < 9; ++k)
                    for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
                if ((threadIdx.x & 31) == 0) {
                    float* gr = grec + ((int64_t)v * n_pad + sI[q]) * 9;
#pragma unroll
                    for (int k = 0; k < 9; ++k)
                        if (acc[k] != 0.f) atomicAdd(gr + k, acc[k]);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// projection backward
__device__ __forceinline__ void sh_basis_grad(int deg, float x, float y, float z, float* Y, float* dYx, float* dYy,
                                              float* dYz) {
    const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
    const float C2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f, -1.0925484305920792f,
                         0.5462742152960396f};
    const float C3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f, 0.3731763325901154f,
                         -0.4570457994644658f, 1.445305721320277f, -0.5900435899266435f};
    for (int b = 0; b < 16; ++b) Y[b] = dYx[b] = dYy[b] = dYz[b] = 0.f;
    Y[0] = C0;
    if (deg < 1) return;
    Y[1] = -C1 * y; dYy[1] = -C1;
    Y[2] = C1 * z;  dYz[2] = C1;
    Y[3] = -C1 * x; dYx[3] = -C1;
    if (deg < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    Y[4] = C2[0] * xy;               dYx[4] = C2[0] * y; dYy[4] = C2[0] * x;
    Y[5] = C2[1] * yz;               dYy[5] = C2[1] * z; dYz[5] = C2[1] * y;
    Y[6] = C2[2] * (2.f * zz - xx - yy); dYx[6] = -2.f * C2[2] * x; dYy[6] = -2.f * C2[2] * y; dYz[6] = 4.f * C2[2] * z;
    Y[7] = C2[3] * xz;               dYx[7] = C2[3] * z; dYz[7] = C2[3] * x;
    Y[8] = C2[4] * (xx - yy);        dYx[8] = 2.f * C2[4] * x; dYy[8] = -2.f * C2[4] * y;
    if (deg < 3) return;
    Y[9] = C3[0] * y * (3.f * xx - yy);  dYx[9] = 6.f * C3[0] * xy; dYy[9] = C3[0] * (3.f * xx - 3.f * yy);
    Y[10] = C3[1] * xy * z;          dYx[10] = C3[1] * yz; dYy[10] = C3[1] * xz; dYz[10] = C3[1] * xy;
    Y[11] = C3[2] * y * (4.f * zz - xx - yy);
    dYx[11] = -2.f * C3[2] * xy; dYy[11] = C3[2] * (4.f * zz - xx - 3.f * yy); dYz[11] = 8.f * C3[2] * yz;
    Y[12] = C3[3] * z * (2.f * zz - 3.f * xx - 3.f * yy);
    dYx[12] = -6.f * C3[3] * xz; dYy[12] = -6.f * C3[3] * yz; dYz[12] = C3[3] * (6.f * zz - 3.f * xx - 3.f * yy);
    Y[13] = C3[4] * x * (4.f * zz - xx - yy);
    dYx[13] = C3[4] * (4.f * zz - 3.f * xx - yy); dYy[13] = -2.f * C3[4] * xy; dYz[13] = 8.f * C3[4] * xz;
    Y[14] = C3[5] * z * (xx - yy);   dYx[14] = 2.f * C3[5] * xz; dYy[14] = -2.f * C3[5] * yz; dYz[14] = C3[5] * (xx - yy);
    Y[15] = C3[6] * x * (xx - 3.f * yy); dYx[15] = C3[6] * (3.f * xx - 3.f * yy); dYy[15] = -6.f * C3[6] * xy;
}

template <int DEG>
__global__ void __launch_bounds__(128) k_project_bwd(const float* __restrict__ planes, int n, int n_pad, const CamBatch cams,
                                                     int n_views, const float* __restrict__ grec, float* __restrict__ gpl) {
    constexpr int B = (DEG + 1) * (DEG + 1);
    constexpr int P = 11 + 3 * B;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_pad) return;
    const int64_t np = n_pad;
    float gp[P];
#pragma unroll
    for (int q = 0; q < P; ++q) gp[q] = 0.f;
    if (i < n) {
        float a[P];
#pragma unroll
        for (int q = 0; q < P; ++q) a[q] = planes[(int64_t)q * np + i];
        // view-independent forward pieces (same operations as k_project)
        float qw = a[3], qx = a[4], qy = a[5], qz = a[6];
        const float n2 = fmaf(qw, qw, fmaf(qx, qx, fmaf(qy, qy, qz * qz)));
        const float qn = sqrtf(n2), inv = 1.0f / qn;
        qw *= inv; qx *= inv; qy *= inv; qz *= inv;
        const float s[3] = {det_exp(a[7]), det_exp(a[8]), det_exp(a[9])};
        float Rq[9];
        Rq[0] = 1.0f - 2.0f * fmaf(qy, qy, qz * qz);
        Rq[1] = 2.0f * (qx * qy - qw * qz);
        Rq[2] = 2.0f * (qx * qz + qw * qy);
        Rq[3] = 2.0f * (qx * qy + qw * qz);
        Rq[4] = 1.0f - 2.0f * fmaf(qx, qx, qz * qz);
        Rq[5] = 2.0f * (qy * qz - qw * qx);
        Rq[6] = 2.0f * (qx * qz - qw * qy);
        Rq[7] = 2.0f * (qy * qz + qw * qx);
        Rq[8] = 1.0f - 2.0f * fmaf(qx, qx, qy * qy);
        float Mm[9], Sg[9];
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k) Mm[j * 3 + k] = Rq[j * 3 + k] * s[k];
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k)
                Sg[j * 3 + k] = fmaf(Mm[j * 3 + 0], Mm[k * 3 + 0], fmaf(Mm[j * 3 + 1], Mm[k * 3 + 1], Mm[j * 3 + 2] * Mm[k * 3 + 2]));
        const float o = 1.0f / (1.0f + det_exp(-a[10]));
        float dSig[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        float dp[3] = {0.f, 0.f, 0.f};
        float dlogit = 0.f;
        for (int v = 0; v < n_views; ++v) {
            const float* G = grec + ((int64_t)v * np + i) * 9;
            float gr[9];
            bool nz = false;
#pragma unroll
            for (int k = 0; k < 9; ++k) { gr[k] = G[k]; nz |= gr[k] != 0.f; }
            if (!nz) continue;  // culled or never composited in this view
            const queen_camera& c = cams.cam[v];
            const float* Rw = c.R;
            const float X = fmaf(Rw[0], a[0], fmaf(Rw[1], a[1], fmaf(Rw[2], a[2], c.t[0])));
            const float Y = fmaf(Rw[3], a[0], fmaf(Rw[4], a[1], fmaf(Rw[5], a[2], c.t[1])));
            const float Z = fmaf(Rw[6], a[0], fmaf(Rw[7], a[1], fmaf(Rw[8], a[2], c.t[2])));
            const float tx = X / Z, ty = Y / Z;
            const bool clx = fabsf(tx) > c.limx, cly = fabsf(ty) > c.limy;
            const float txc = fminf(c.limx, fmaxf(-c.limx, tx)), tyc = fminf(c.limy, fmaxf(-c.limy, ty));
            const float J00 = c.fx / Z, J02 = -(c.fx * txc) / Z, J11 = c.fy / Z, J12 = -(c.fy * tyc) / Z;
            float Tm[6];
            for (int m = 0; m < 3; ++m) {
                Tm[m] = fmaf(J00, Rw[m], J02 * Rw[6 + m]);
                Tm[3 + m] = fmaf(J11, Rw[3 + m], J12 * Rw[6 + m]);
            }
            float TS[6];  // Tm * Sigma (2x3)
            for (int r = 0; r < 2; ++r)
                for (int m = 0; m < 3; ++m)
                    TS[r * 3 + m] = fmaf(Tm[r * 3 + 0], Sg[m], fmaf(Tm[r * 3 + 1], Sg[3 + m], Tm[r * 3 + 2] * Sg[6 + m]));
            const float sa = fmaf(TS[0], Tm[0], fmaf(TS[1], Tm[1], TS[2] * Tm[2])) + 0.3f;
            const float sb = fmaf(TS[0], Tm[3], fmaf(TS[1], Tm[4], TS[2] * Tm[5]));
            const float sc = fmaf(TS[3], Tm[3], fmaf(TS[4], Tm[4], TS[5] * Tm[5])) + 0.3f;
            const float det = fmaf(sa, sc, -(sb * sb));
            // record (u, v, A2, B2, C2) -> Sigma' entries (a, b, c) and camera-space position
            const float L2E = 1.4426950408889634f;
            const float gca = gr[2] * (-0.5f * L2E), gcb = gr[3] * (-L2E), gcc = gr[4] * (-0.5f * L2E);
            const float id2 = 1.0f / (det * det);
            const float da = (-sc * sc * gca + sb * sc * gcb - sb * sb * gcc) * id2;
            const float db = (2.f * sb * sc * gca - (sa * sc + sb * sb) * gcb + 2.f * sa * sb * gcc) * id2;
            const float dc = (-sb * sb * gca + sa * sb * gcb - sa * sa * gcc) * id2;
            // dL/dSigma' as a symmetric 2x2 G = [[da, db/2], [db/2, dc]]; Sigma' = Tm Sigma Tm^T
            const float G00 = da, G01 = 0.5f * db, G11 = dc;
            float GT[6];  // G * Tm (2x3)
            for (int m = 0; m < 3; ++m) {
                GT[m] = G00 * Tm[m] + G01 * Tm[3 + m];
                GT[3 + m] = G01 * Tm[m] + G11 * Tm[3 + m];
            }
            for (int j = 0; j < 3; ++j)  // dL/dSigma += Tm^T G Tm
                for (int k = 0; k < 3; ++k) dSig[j * 3 + k] += Tm[j] * GT[k] + Tm[3 + j] * GT[3 + k];
            float dTm[6];  // dL/dTm = 2 G Tm Sigma
            for (int r = 0; r < 2; ++r)
                for (int m = 0; m < 3; ++m)
                    dTm[r * 3 + m] = 2.f * (GT[r * 3 + 0] * Sg[m] + GT[r * 3 + 1] * Sg[3 + m] + GT[r * 3 + 2] * Sg[6 + m]);
            // Tm = J W -> dJ = dTm W^T (only J00, J02, J11, J12 are non-zero)
            const float dJ00 = dTm[0] * Rw[0] + dTm[1] * Rw[1] + dTm[2] * Rw[2];
            const float dJ02 = dTm[0] * Rw[6] + dTm[1] * Rw[7] + dTm[2] * Rw[8];
            const float dJ11 = dTm[3] * Rw[3] + dTm[4] * Rw[4] + dTm[5] * Rw[5];
            const float dJ12 = dTm[3] * Rw[6] + dTm[4] * Rw[7] + dTm[5] * Rw[8];
            const float iz = 1.0f / Z, iz2 = iz * iz;
            float dX = gr[0] * c.fx * iz, dY = gr[1] * c.fy * iz;
            float dZ = -(gr[0] * c.fx * X + gr[1] * c.fy * Y) * iz2;
            dZ += -dJ00 * c.fx * iz2 - dJ11 * c.fy * iz2;
            if (clx) {
                dZ += dJ02 * c.fx * txc * iz2;
            } else {  // J02 = -fx X / Z^2
                dX += -dJ02 * c.fx * iz2;
                dZ += 2.f * dJ02 * c.fx * X * iz2 * iz;
            }
            if (cly) {
                dZ += dJ12 * c.fy * tyc * iz2;
            } else {
                dY += -dJ12 * c.fy * iz2;
                dZ += 2.f * dJ12 * c.fy * Y * iz2 * iz;
            }
            // colour: rgb = max(0, sum Y_b h_b + 0.5), dir = (p - C) / |p - C|
            float ddx = a[0] - c.C[0], ddy = a[1] - c.C[1], ddz = a[2] - c.C[2];
            const float dn = sqrtf(fmaf(ddx, ddx, fmaf(ddy, ddy, ddz * ddz)));
            const float ux = ddx / dn, uy = ddy / dn, uz = ddz / dn;
            float Yb[16], Yx[16], Yy[16], Yz[16];
            sh_basis_grad(DEG, ux, uy, uz, Yb, Yx, Yy, Yz);
            float gdx = 0.f, gdy = 0.f, gdz = 0.f;
            for (int ch = 0; ch < 3; ++ch) {
                float col = 0.5f;
                for (int b = 0; b < B; ++b) col = fmaf(Yb[b], a[11 + 3 * b + ch], col);
                if (!(col > 0.0f)) continue;  // max(0, .) clamped
                const float gc = gr[6 + ch];
                for (int b = 0; b < B; ++b) {
                    gp[11 + 3 * b + ch] += gc * Yb[b];
                    gdx += gc * a[11 + 3 * b + ch] * Yx[b];
                    gdy += gc * a[11 + 3 * b + ch] * Yy[b];
                    gdz += gc * a[11 + 3 * b + ch] * Yz[b];
                }
            }
            const float dotd = gdx * ux + gdy * uy + gdz * uz;
            dp[0] += (gdx - dotd * ux) / dn;
            dp[1] += (gdy - dotd * uy) / dn;
            dp[2] += (gdz - dotd * uz) / dn;
            // camera transform: xc = W p + t
            for (int k = 0; k < 3; ++k) dp[k] += Rw[k] * dX + Rw[3 + k] * dY + Rw[6 + k] * dZ;
            dlogit += gr[5] * o * (1.0f - o);
        }
        // Sigma = M M^T -> dM = (dSig + dSig^T) M ; M = R diag(s)
        float dM[9];
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k) {
                float acc = 0.f;
                for (int m = 0; m < 3; ++m) acc += (dSig[j * 3 + m] + dSig[m * 3 + j]) * Mm[m * 3 + k];
                dM[j * 3 + k] = acc;
            }
        float dR[9], ds[3] = {0.f, 0.f, 0.f};
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k) {
                dR[j * 3 + k] = dM[j * 3 + k] * s[k];
                ds[k] += dM[j * 3 + k] * Rq[j * 3 + k];
            }
        for (int k = 0; k < 3; ++k) gp[7 + k] = ds[k] * s[k];
        const float dw = 2.f * (-qz * dR[1] + qy * dR[2] + qz * dR[3] - qx * dR[5] - qy * dR[6] + qx * dR[7]);
        const float dx_ = 2.f * (qy * dR[1] + qz * dR[2] + qy * dR[3] - 2.f * qx * dR[4] - qw * dR[5] + qz * dR[6] +
                                 qw * dR[7] - 2.f * qx * dR[8]);
        const float dy_ = 2.f * (-2.f * qy * dR[0] + qx * dR[1] + qw * dR[2] + qx * dR[3] + qz * dR[5] - qw * dR[6] +
                                 qz * dR[7] - 2.f * qy * dR[8]);
        const float dz_ = 2.f * (-2.f * qz * dR[0] - qw * dR[1] + qx * dR[2] + qw * dR[3] - 2.f * qz * dR[4] +
                                 qy * dR[5] + qx * dR[6] + qy * dR[7]);
        const float dq = dw * qw + dx_ * qx + dy_ * qy + dz_ * qz;  // through the normalisation
        gp[3] = (dw - dq * qw) / qn;
        gp[4] = (dx_ - dq * qx) / qn;
        gp[5] = (dy_ - dq * qy) / qn;
        gp[6] = (dz_ - dq * qz) / qn;
        gp[0] = dp[0];
        gp[1] = dp[1];
        gp[2] = dp[2];
        gp[10] = dlogit;
    }
#pragma unroll
    for (int q = 0; q < P; ++q) gpl[(int64_t)q * np + i] = gp[q];
}

cudaError_t launch_blend_bwd(const float* rec, int n_pad, const uint32_t* ranges, const uint32_t* vals, int n_views,
                             int W, int H, float bg0, float bg1, float bg2, const float* gout, float* grec,
                             cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(grec, 0, sizeof(float) * 9 * (size_t)n_views * n_pad, s);
    if (e) return e;
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int T = gx * gy;
    const int64_t blocks = (int64_t)T * n_views;
    if (blocks == 0) return cudaSuccess;
    k_blend_bwd<<<(unsigned)blocks, BW_NT, 0, s>>>(reinterpret_cast<const float4*>(rec), n_pad,
                                                   reinterpret_cast<const uint2*>(ranges), vals, W, H, gx, T, bg0, bg1,
                                                   bg2, gout, grec);
    return cudaGetLastError();
}

cudaError_t launch_project_bwd(const float* planes, int n, int n_pad, int deg, const CamBatch& cams, int n_views,
                               const float* grec, float* gpl, cudaStream_t s) {
    const int blocks = (n_pad + 127) / 128;
    if (blocks == 0) return cudaSuccess;
    switch (deg) {
        case 0: k_project_bwd<0><<<blocks, 128, 0, s>>>(planes, n, n_pad, cams, n_views, grec, gpl); break;
        case 1: k_project_bwd<1><<<blocks, 128, 0, s>>>(planes, n, n_pad, cams, n_views, grec, gpl); break;
        case 2: k_project_bwd<2><<<blocks, 128, 0, s>>>(planes, n, n_pad, cams, n_views, grec, gpl); break;
        default: k_project_bwd<3><<<blocks, 128, 0, s>>>(planes, n, n_pad, cams, n_views, grec, gpl); break;
    }
    return cudaGetLastError();
}

}  // namespace queen
