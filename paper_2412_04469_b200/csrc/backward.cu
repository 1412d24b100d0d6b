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

__device__ __forceinline__ float rcpa(float x) {  // MUFU.RCP without the denormal fix-up (|x| >= 0.01 here)
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float ex2b(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void bw_cp16(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}

constexpr int BW_RPT = 4;
constexpr int BW_NT = 256 / BW_RPT;  // 64 threads per tile
constexpr int BW_BATCH = 64;

#ifndef QUEEN_BWD_MINB
#define QUEEN_BWD_MINB 12  // 80 registers (a few spilled words): rasterize_backward 7.27 -> 7.00 ms (92 regs uncapped)
#endif
#define BWD_BOUNDS __launch_bounds__(BW_NT, QUEEN_BWD_MINB)
__global__ void BWD_BOUNDS k_blend_bwd(const float4* __restrict__ rec, int n_pad,
                                                     const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
                                                     int W, int H, int gx, int T, float bg0, float bg1, float bg2,
                                                     const float* __restrict__ gout, float* __restrict__ grec,
                                                     const uint32_t* __restrict__ order) {
    __shared__ __align__(16) float4 sA[2][BW_BATCH], sB[2][BW_BATCH], sC[2][BW_BATCH];
    __shared__ uint32_t sI[BW_BATCH];
    __shared__ int s_jmax[BW_NT / 32];
    __shared__ uint8_t s_list[BW_NT / 32][BW_BATCH];
    const int gt = order ? (int)order[blockIdx.x] : (int)blockIdx.x;
    const int v = gt / T;
    const int t = gt - v * T;
    const int px = (t % gx) * 16 + (threadIdx.x & 15);
    const int py0 = (t / gx) * 16 + (threadIdx.x >> 4) * BW_RPT;
    const float fx = (float)px;
    const float wx0 = (float)((t % gx) * 16), wy0 = (float)((t / gx) * 16 + (threadIdx.x >> 5) * 8);
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
    constexpr int NP = BW_RPT / 2;
    const float NEG_INF = __int_as_float(0xff800000);
    float2 TA[NP], nfy[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        TA[k] = make_float2(Tf[2 * k], Tf[2 * k + 1]);
        nfy[k] = make_float2(-(float)(py0 + 2 * k), -(float)(py0 + 2 * k + 1));
    }
    // ---- phase A: replay the forward (same fp32 operations as k_blend / the oracle), with the
    // forward's skips: the CTA stops once every pixel has terminated, and each warp visits only
    // the batch records whose alpha >= 1/255 ellipse reaches its 16 x 8 sub-tile (touches());
    // skipped records hit none of the warp's pixels, so T and the last contributor are unchanged
    const unsigned lane_lt = (1u << (threadIdx.x & 31)) - 1u;
    // records staged by cp.async, double-buffered (batch b+1 in flight while batch b replays),
    // as in k_blend; one record per thread per batch (BW_NT == BW_BATCH)
    static_assert(BW_NT == BW_BATCH, "one staged record per thread");
    const int nbA = (re - rs + BW_BATCH - 1) / BW_BATCH;
    auto stageA = [&](int b, int buf) {
        const int j = rs + b * BW_BATCH + (int)threadIdx.x;
        if (j < re) {
            const float4* g = vrec + (int64_t)vals[j] * 3;
            bw_cp16(&sA[buf][threadIdx.x], g);
            bw_cp16(&sB[buf][threadIdx.x], g + 1);
            bw_cp16(&sC[buf][threadIdx.x], g + 2);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    if (nbA > 0) stageA(0, 0);
    for (int b = 0; b < nbA; ++b) {
        const int buf = b & 1;
        const int b0 = rs + b * BW_BATCH;
        const int cnt = min(BW_BATCH, re - b0);
        bool alive = false;
#pragma unroll
        for (int k = 0; k < NP; ++k) alive |= !(TA[k].x < 1e-4f) | !(TA[k].y < 1e-4f);
        if (__syncthreads_count(alive) == 0) break;  // (also: every warp is done with buffer buf ^ 1)
        if (b + 1 < nbA) stageA(b + 1, buf ^ 1);
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncthreads();
        if (!__any_sync(0xffffffffu, alive)) continue;
        uint8_t* lst = s_list[threadIdx.x >> 5];
        int nq = 0;
#pragma unroll
        for (int e2 = 0; e2 < BW_BATCH / 32; ++e2) {
            const int q = (int)(threadIdx.x & 31) + 32 * e2;
            const bool want = q < cnt && touches(sA[buf][q], sB[buf][q], wx0, wx0 + 15.0f, wy0, wy0 + 7.0f);
            const unsigned bal = __ballot_sync(0xffffffffu, want);
            if (want) lst[nq + __popc(bal & lane_lt)] = (uint8_t)q;
            nq += __popc(bal);
        }
        __syncwarp();
        for (int i = 0; i < nq; ++i) {  // the forward's paired row arithmetic, lane for lane
            const int q = lst[i];
            const float4 a = sA[buf][q], bq = sB[buf][q];
            const float dx = a.x - fx;
            const float tAdx = (bq.x * dx) * dx, tB = bq.y * dx;
            const float2 vv = make_float2(a.y, a.y), cc = make_float2(bq.z, bq.z);
            const float2 ta2 = make_float2(tAdx, tAdx), tb2 = make_float2(tB, tB);
            float2 p2[NP];
            bool h[2 * NP];
            bool anyh = false;
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                const float2 dy = __fadd2_rn(vv, nfy[k]);
                p2[k] = __ffma2_rn(__ffma2_rn(cc, dy, tb2), dy, ta2);
                h[2 * k] = !(TA[k].x < 1e-4f) && !(p2[k].x < bq.w);
                h[2 * k + 1] = !(TA[k].y < 1e-4f) && !(p2[k].y < bq.w);
                anyh |= h[2 * k] | h[2 * k + 1];
            }
            if (!anyh) continue;
            // branch-free over the row pairs (a non-hitting row gets alpha = +0: T unchanged)
            const float o = sC[buf][q].x;
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                const float2 e = make_float2(ex2b(h[2 * k] ? p2[k].x : NEG_INF), ex2b(h[2 * k + 1] ? p2[k].y : NEG_INF));
                float2 al = __fmul2_rn(make_float2(o, o), e);
                al = make_float2(fminf(0.99f, al.x), fminf(0.99f, al.y));
                // the forward's transmittance update (k_blend composite2: T - aT, QUEEN_BLEND_TSUB)
                if (QUEEN_BLEND_TSUB) {
                    const float2 aT = __fmul2_rn(al, TA[k]);
                    TA[k] = __fadd2_rn(TA[k], make_float2(-aT.x, -aT.y));
                } else {
                    TA[k] = __fmul2_rn(TA[k], __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-al.x, -al.y)));
                }
                last[2 * k] = h[2 * k] ? b0 + q : last[2 * k];
                last[2 * k + 1] = h[2 * k + 1] ? b0 + q : last[2 * k + 1];
            }
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        Tf[2 * k] = TA[k].x;
        Tf[2 * k + 1] = TA[k].y;
    }
    // ---- phase B: reverse walk
    int jmax = -1;
#pragma unroll
    for (int r = 0; r < BW_RPT; ++r) jmax = max(jmax, last[r]);
    for (int o = 16; o > 0; o >>= 1) jmax = max(jmax, __shfl_xor_sync(0xffffffffu, jmax, o));
    const int wjmax = jmax;  // this warp's last contributor: later records hit none of its pixels
    if ((threadIdx.x & 31) == 0) s_jmax[threadIdx.x >> 5] = jmax;
    __syncthreads();
    jmax = max(s_jmax[0], s_jmax[1]);
    const int64_t plane = (int64_t)H * W;
    // Per row pair (paired FP32 ops, as in the forward): the image gradient g, the colour behind
    // each record plus the background term Sb = S_i + T_N bg (S_i = colour composited after i),
    // and the running transmittance Tc (T_i = T_{i+1} / (1 - a_i)).
    float2 g2[NP][3], Sb[NP][3], Tc[NP];
    const float bgc[3] = {bg0, bg1, bg2};
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        float gg[2][3];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = 2 * k + h;
            const bool in = px < W && py0 + r < H;
            const int64_t pix = (int64_t)v * 3 * plane + (int64_t)(py0 + r) * W + px;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) gg[h][ch] = in ? gout[pix + ch * plane] : 0.f;
        }
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            g2[k][ch] = make_float2(gg[0][ch], gg[1][ch]);
            Sb[k][ch] = make_float2(Tf[2 * k] * bgc[ch], Tf[2 * k + 1] * bgc[ch]);
        }
        Tc[k] = make_float2(Tf[2 * k], Tf[2 * k + 1]);
    }
    const float LN2 = 0.69314718055994531f;
    for (int bend = jmax + 1; bend > rs; bend -= BW_BATCH) {
        const int b0 = max(rs, bend - BW_BATCH);
        const int cnt = bend - b0;
        __syncthreads();
        for (int q = threadIdx.x; q < cnt; q += BW_NT) {
            const uint32_t gi = vals[b0 + q];
            const float4* gp = vrec + (int64_t)gi * 3;
            sA[0][q] = gp[0];
            sB[0][q] = gp[1];
            sC[0][q] = gp[2];
            sI[q] = gi;
        }
        __syncthreads();
        // this warp's records of the batch: those whose alpha >= 1/255 ellipse can reach its 16 x 8
        // sub-tile (touches(), lane q tests record q; the others have no hit in the warp)
        unsigned long long wmask = 0ull;
#pragma unroll
        for (int e2 = 0; e2 < BW_BATCH / 32; ++e2) {
            const int q = (int)(threadIdx.x & 31) + 32 * e2;
            const bool want = q < cnt && b0 + q <= wjmax && touches(sA[0][q], sB[0][q], wx0, wx0 + 15.0f, wy0, wy0 + 7.0f);
            wmask |= (unsigned long long)__ballot_sync(0xffffffffu, want) << (32 * e2);
        }
        while (wmask) {
            const int q = 63 - __clzll((long long)wmask);  // descending order
            wmask &= ~(1ull << q);
            const int j = b0 + q;
            const float4 a = sA[0][q], bq = sB[0][q], c = sC[0][q];
            const float dx = a.x - fx;
            const float tAdx = (bq.x * dx) * dx, tB = bq.y * dx;
            const float2 vv = make_float2(a.y, a.y), cc = make_float2(bq.z, bq.z);
            const float2 ta2 = make_float2(tAdx, tAdx), tb2 = make_float2(tB, tB);
            const float2 o2 = make_float2(c.x, c.x);
            const float2 col[3] = {make_float2(c.y, c.y), make_float2(c.z, c.z), make_float2(c.w, c.w)};
            // pair accumulators: colour r g b, opacity, and the moments of dp2 (1, dy, dy^2)
            float2 aC[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
            float2 aO = make_float2(0.f, 0.f), m0 = aO, m1 = aO, m2 = aO;
            bool any = false;
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                const bool l0 = j <= last[2 * k], l1 = j <= last[2 * k + 1];
                if (!(l0 | l1)) continue;
                const float2 dy = __fadd2_rn(vv, nfy[k]);
                const float2 p2 = __ffma2_rn(__ffma2_rn(cc, dy, tb2), dy, ta2);
                const bool h0 = l0 && !(p2.x < bq.w);
                const bool h1 = l1 && !(p2.y < bq.w);
                if (!(h0 | h1)) continue;
                any = true;
                // a non-hit lane of the pair runs with a = 0: T, Sb and every sum stay unchanged
                const float2 e = make_float2(ex2b(h0 ? p2.x : NEG_INF), ex2b(h1 ? p2.y : NEG_INF));
                const float2 raw = __fmul2_rn(o2, e);
                const float2 al = make_float2(fminf(0.99f, raw.x), fminf(0.99f, raw.y));
                const float2 om = __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-al.x, -al.y));
                const float2 niom = make_float2(-rcpa(om.x), -rcpa(om.y));  // 1 - a >= 0.01
                const float2 Ti = __fmul2_rn(Tc[k], make_float2(-niom.x, -niom.y));
                const float2 w = __fmul2_rn(al, Ti);
                float2 dal = make_float2(0.f, 0.f);
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    // dL/da = sum_ch g (c T_i - Sb / (1 - a))
                    dal = __ffma2_rn(g2[k][ch], __ffma2_rn(col[ch], Ti, __fmul2_rn(Sb[k][ch], niom)), dal);
                    Sb[k][ch] = __ffma2_rn(col[ch], w, Sb[k][ch]);
                    aC[ch] = __ffma2_rn(w, g2[k][ch], aC[ch]);
                }
                Tc[k] = Ti;
                // unclamped hits only: a = o 2^p2
                const float2 dm = make_float2(h0 && raw.x <= 0.99f ? dal.x : 0.f, h1 && raw.y <= 0.99f ? dal.y : 0.f);
                aO = __ffma2_rn(dm, e, aO);
                const float2 dp2 = __fmul2_rn(__fmul2_rn(dm, al), make_float2(LN2, LN2));
                m0 = __fadd2_rn(m0, dp2);
                const float2 t = __fmul2_rn(dp2, dy);
                m1 = __fadd2_rn(m1, t);
                m2 = __ffma2_rn(t, dy, m2);
            }
            if (!__any_sync(0xffffffffu, any)) continue;
            float acc[9];
            {  // per lane: u, v, A2, B2, C2 from the moments (dx constant over the lane's rows)
                const float s0 = m0.x + m0.y, s1 = m1.x + m1.y, s2 = m2.x + m2.y;
                acc[0] = 2.0f * bq.x * dx * s0 + bq.y * s1;  // d/du = sum dp2 (2 A2 dx + B2 dy)
                acc[1] = bq.y * dx * s0 + 2.0f * bq.z * s1;  // d/dv = sum dp2 (B2 dx + 2 C2 dy)
                acc[2] = dx * dx * s0;                        // d/dA2
                acc[3] = dx * s1;                             // d/dB2
                acc[4] = s2;                                  // d/dC2
                acc[5] = aO.x + aO.y;
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) acc[6 + ch] = aC[ch].x + aC[ch].y;
            }
            // warp reduce-scatter of the 9 (padded to 16) sums: 8 + 4 + 2 + 1 + 1 shuffles; lane l
            // ends with the total of value l >> 1, and lanes 0, 2, .., 16 add them (one atomic each)
            float v8[8];
            const uint32_t lane = threadIdx.x & 31;
            {
                const bool b = (lane >> 4) & 1;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float lo = acc[k], hi = k + 8 < 9 ? acc[k + 8] : 0.f;
                    const float send = b ? lo : hi, keep = b ? hi : lo;
                    v8[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                }
            }
            float v4[4];
            {
                const bool b = (lane >> 3) & 1;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float send = b ? v8[k] : v8[k + 4], keep = b ? v8[k + 4] : v8[k];
                    v4[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                }
            }
            float v2[2];
            {
                const bool b = (lane >> 2) & 1;
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const float send = b ? v4[k] : v4[k + 2], keep = b ? v4[k + 2] : v4[k];
                    v2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
                }
            }
            float v1;
            {
                const bool b = (lane >> 1) & 1;
                const float send = b ? v2[0] : v2[1], keep = b ? v2[1] : v2[0];
                v1 = keep + __shfl_xor_sync(0xffffffffu, send, 2);
            }
            v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
            const int idx = (int)(lane >> 1);  // = 8 b4 + 4 b3 + 2 b2 + b1
            if ((lane & 1) == 0 && idx < 9 && v1 != 0.f)
                atomicAdd(grec + ((int64_t)v * n_pad + sI[q]) * 9 + idx, v1);
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
            const float izf = 1.0f / Z;  // the forward's operations (k_project)
            const float tx = X * izf, ty = Y * izf;
            const bool clx = fabsf(tx) > c.limx, cly = fabsf(ty) > c.limy;
            const float txc = fminf(c.limx, fmaxf(-c.limx, tx)), tyc = fminf(c.limy, fmaxf(-c.limy, ty));
            const float J00 = c.fx * izf, J02 = -(c.fx * txc) * izf, J11 = c.fy * izf, J12 = -(c.fy * tyc) * izf;
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
                             uint32_t* order_ws, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(grec, 0, sizeof(float) * 9 * (size_t)n_views * n_pad, s);
    if (e) return e;
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int T = gx * gy;
    const int64_t blocks = (int64_t)T * n_views;
    if (blocks == 0) return cudaSuccess;
    const uint32_t* order = nullptr;  // longest tile lists first (the forward's schedule)
    if ((e = launch_tile_order(ranges, blocks, order_ws, s, &order))) return e;
    k_blend_bwd<<<(unsigned)blocks, BW_NT, 0, s>>>(reinterpret_cast<const float4*>(rec), n_pad,
                                                   reinterpret_cast<const uint2*>(ranges), vals, W, H, gx, T, bg0, bg1,
                                                   bg2, gout, grec, order);
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

// ---------------------------------------------------------------------------
// decode backward (the encode side of Eq. 4-5 and the gates): given dL/dA_t,
//   dL/dD_c[m][k] = sum_i dL/dA[row(c,m)][i] round(l)_c[k][i]        (k_dec_grad_partial/_sum,
//                                                                     deterministic 2-stage sum)
//   dL/dl_hat_c[k][i] = sum_m D_c[m][k] dL/dA[row(c,m)][i]            (straight-through round)
//   dL/dl_p,i = g_i dL/dp_i ;  dL/dlog alpha_i = (l_p,i . dL/dp_i) dg/dlog alpha (k_gate_grad)
namespace queen {

struct DecBwdParams {
    int n, n_pad;
    int lat[5], M[5], lat_row0[5], dec_off[5], out_row0[5];
    int ndec, chunks, f32;
    const void* latents;
    const float* decoders;
    const float* gA;
};

__device__ __forceinline__ float latent_value(const DecBwdParams& p, int row, int i) {
    if (p.f32) return roundf(static_cast<const float*>(p.latents)[(int64_t)row * p.n_pad + i]);
    return (float)static_cast<const int8_t*>(p.latents)[(int64_t)row * p.n_pad + i];
}

// block (r, chunk): attribute row r = out_row0[c] + m; partial sums over the chunk's Gaussians
__global__ void __launch_bounds__(256) k_dec_grad_partial(DecBwdParams p, float* __restrict__ part) {
    __shared__ float s_w[8][16];
    const int r = blockIdx.x, chunk = blockIdx.y;
    int c = 0;
    while (c < 4 && r >= p.out_row0[c] + p.M[c]) ++c;
    const int m = r - p.out_row0[c];
    const int L = p.lat[c];
    if (L == 0) return;
    const int64_t per = ((int64_t)p.n + p.chunks - 1) / p.chunks;
    const int i0 = (int)(chunk * per), i1 = (int)min((int64_t)p.n, (chunk + 1) * per);
    float acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = 0.f;
    const float* g = p.gA + (int64_t)(3 + r) * p.n_pad;
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const float gi = g[i];
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (k < L) acc[k] = fmaf(gi, latent_value(p, p.lat_row0[c] + k, i), acc[k]);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        if (k >= L) break;
        float x = acc[k];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) s_w[w][k] = x;
    }
    __syncthreads();
    if (threadIdx.x < L) {
        float x = 0.f;
        for (int q = 0; q < 8; ++q) x += s_w[q][threadIdx.x];
        part[(int64_t)chunk * p.ndec + p.dec_off[c] + m * L + threadIdx.x] = x;
    }
}

__global__ void k_dec_grad_sum(const float* __restrict__ part, int ndec, int chunks, float* __restrict__ gdec) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ndec) return;
    float x = 0.f;
    for (int q = 0; q < chunks; ++q) x += part[(int64_t)q * ndec + j];
    gdec[j] = x;
}

__global__ void __launch_bounds__(256) k_lat_grad(DecBwdParams p, float* __restrict__ glat) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n_pad) return;
    for (int c = 0; c < 5; ++c) {
        const int L = p.lat[c];
        if (L == 0) continue;
        float acc[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = 0.f;
        if (i < p.n) {
            for (int m = 0; m < p.M[c]; ++m) {
                const float gi = p.gA[(int64_t)(3 + p.out_row0[c] + m) * p.n_pad + i];
                const float* d = p.decoders + p.dec_off[c] + m * L;
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    if (k < L) acc[k] = fmaf(__ldg(d + k), gi, acc[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (k < L) glat[(int64_t)(p.lat_row0[c] + k) * p.n_pad + i] = acc[k];
    }
}

__global__ void __launch_bounds__(256) k_gate_grad(const float* __restrict__ gA, const float* __restrict__ la,
                                                   const float* __restrict__ pre, int n, int n_pad, float tau, float g0,
                                                   float g1, float theta0, float* __restrict__ gla,
                                                   float* __restrict__ gpre) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_pad) return;
    float dla = 0.f, dpre[3] = {0.f, 0.f, 0.f};
    if (i < n && la[i] > theta0) {  // the forward's mask (R#6)
        const float ghat = 1.0f / (1.0f + det_exp((-la[i]) / tau));
        const float gt = fmaf(ghat, g1 - g0, g0);
        const float g = fminf(1.0f, fmaxf(0.0f, gt));
        float dg = 0.f;
        for (int d = 0; d < 3; ++d) {
            const float gp = gA[(int64_t)d * n_pad + i];
            dpre[d] = g * gp;
            dg = fmaf(pre[(int64_t)d * n_pad + i], gp, dg);
        }
        if (gt > 0.0f && gt < 1.0f) dla = dg * (g1 - g0) * ghat * (1.0f - ghat) / tau;
    }
    if (gla) gla[i] = dla;
    if (gpre)
        for (int d = 0; d < 3; ++d) gpre[(int64_t)d * n_pad + i] = dpre[d];
}

float host_theta0(float tau, float g0, float g1);

cudaError_t launch_decode_bwd(const queen_packet& pk, const float* gA, float* gdec, float* glat, float* gla, float* gpre,
                              float* scratch, size_t scratch_floats, cudaStream_t s) {
    DecBwdParams p{};
    const int B = (pk.sh_degree + 1) * (pk.sh_degree + 1);
    const int Mc[5] = {4, 3, 1, 3, 3 * (B - 1)};
    int lr = 0, dof = 0, orow = 0;
    for (int c = 0; c < 5; ++c) {
        p.lat[c] = pk.lat_dim[c];
        p.M[c] = Mc[c];
        p.lat_row0[c] = lr;
        p.dec_off[c] = dof;
        p.out_row0[c] = orow;
        lr += pk.lat_dim[c];
        dof += Mc[c] * pk.lat_dim[c];
        orow += Mc[c];
    }
    p.ndec = dof;
    p.n = pk.n;
    p.n_pad = pk.n_pad;
    p.f32 = pk.latent_kind == QUEEN_LAT_F32;
    p.latents = pk.latents;
    p.decoders = pk.decoders;
    p.gA = gA;
    cudaError_t e;
    if (gdec && p.ndec > 0) {
        int chunks = (pk.n + 8191) / 8192;
        chunks = chunks < 1 ? 1 : (chunks > 64 ? 64 : chunks);
        while (chunks > 1 && (size_t)chunks * p.ndec > scratch_floats) --chunks;
        if ((size_t)chunks * p.ndec > scratch_floats) return cudaErrorInvalidValue;
        p.chunks = chunks;
        if ((e = cudaMemsetAsync(scratch, 0, sizeof(float) * chunks * p.ndec, s))) return e;
        k_dec_grad_partial<<<dim3((unsigned)orow, (unsigned)chunks), 256, 0, s>>>(p, scratch);
        k_dec_grad_sum<<<(p.ndec + 255) / 256, 256, 0, s>>>(scratch, p.ndec, chunks, gdec);
    }
    if (glat) k_lat_grad<<<(pk.n_pad + 255) / 256, 256, 0, s>>>(p, glat);
    if (gla || gpre) {
        if (pk.pos_kind == QUEEN_POS_GATES) {
            k_gate_grad<<<(pk.n_pad + 255) / 256, 256, 0, s>>>(gA, pk.log_alpha, pk.pos_pregate, pk.n, pk.n_pad, pk.tau,
                                                              pk.gamma0, pk.gamma1, host_theta0(pk.tau, pk.gamma0, pk.gamma1),
                                                              gla, gpre);
        } else {
            if (gla && (e = cudaMemsetAsync(gla, 0, sizeof(float) * pk.n_pad, s))) return e;
            if (gpre && (e = cudaMemsetAsync(gpre, 0, sizeof(float) * 3 * (size_t)pk.n_pad, s))) return e;
        }
    }
    return cudaGetLastError();
}

}  // namespace queen
