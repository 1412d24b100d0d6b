// K7: per-tile front-to-back alpha compositing (Eq. 2) with the
// 3D-GS cut-offs of DESIGN reading R14 and composite-then-stop early termination.
//
// Plain-ALU bound (FP32 issue + MUFU ex2), so the design minimises instructions per
// evaluated (pixel, Gaussian) pair:
//  * one 64-thread CTA per 16x16 tile; each thread owns one column x 4 rows, so the
//    per-Gaussian work that depends only on x (dx, A2 dx, B2 dx) is shared by 4 pixels
//    and the per-row terms run as paired FP32 ops (FADD2 / FMUL2 / FFMA2, sm_100),
//    two pixels per instruction -- each lane still rounds exactly like the scalar
//    oracle (__ffma2_rn == __fmaf_rn per component);
//  * the tile's sorted records are staged in shared memory in batches of 64 with
//    cp.async (LDGSTS), double-buffered: batch b+1 is in flight while batch b blends,
//    and the record indices run one batch further ahead;
//  * per batch, each warp keeps a list of the records whose alpha >= 1/255 ellipse can reach
//    its 16 x 8 sub-tile (touches(), exact-safe), and all its lanes read the same record
//    (LDS.128 broadcast); the CTA retires as soon as all 256 pixels have terminated
//    (__syncthreads_count);
//  * compositing is warp-uniform per row-pair band (one vote per 16 x 4 band) and
//    branch-free inside it (composite2: a non-hitting row gets alpha = +0, which leaves C and
//    T bit-identical), paired as well.
// Per-pixel arithmetic (oracle/queen_oracle.cpp blend_step):
//   p2 = fma(fma(C2, dy, B2 dx), dy, (A2 dx) dx);  skip if p2 < T2 (R14: no p2 > 0 skip);
//   a = min(0.99, o 2^p2); C = fma(rgb, a T, C); stop after T < 1e-4 -- the skip decisions are
//   the oracle's bit for bit; the transmittance update is T - aT (QUEEN_BLEND_TSUB, one FADD2
//   on the aT already formed) where the oracle computes T (1 - a): within 1 ulp per step, and
//   RGB / T are checked against the oracle within the 2e-3 bar.
#include <cstdlib>

#include <cuda_fp16.h>

#include "queen_internal.cuh"

#include <algorithm>

namespace queen {


__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// 2^x for x in [T2, 0] (T2 >= log2(1/255)): MUFU.EX2 directly, no denormal range fix-up
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Pixel state of a row pair, kept as float2 so the compositing runs as paired FP32 ops.
// A pixel is alive while T >= 1e-4 (composite-then-stop: T only drops below 1e-4 through
// its last composite); pixels outside the image start at T = 0, i.e. terminated.
struct Px2 {
    float2 r, g, b, T;
};

// a pixel hits a record when it is alive (T >= 1e-4) and alpha >= 1/255 (p2 >= T2; R14)
__device__ __forceinline__ bool hit(float T, float p2, float T2) { return !(T < 1e-4f) && !(p2 < T2); }

// Branch-free compositing of one record into a row pair: a row that does not hit gets
// exponent -inf, i.e. alpha = min(0.99, o * 2^-inf) = +0, and then C = fma(c, +0, C) = C and
// T = T (1 - 0) = T exactly -- bit-identical to skipping it.  c = (o, r, g, b).
// CLAMP = false would skip min(0.99, .), the identity for records with o <= 0.98 (o 2^p2 <=
// 0.98 (1 + 2^-22) < 0.99 for p2 <= 0); k_blend clamps every record (one code path was faster).
template <bool CLAMP>
__device__ __forceinline__ void composite2(Px2& p, float q0, float q1, bool h0, bool h1, const float4& c) {
    const float NEG_INF = __int_as_float(0xff800000);
    const float e0 = ex2(h0 ? q0 : NEG_INF), e1 = ex2(h1 ? q1 : NEG_INF);
    float2 al = __fmul2_rn(make_float2(c.x, c.x), make_float2(e0, e1));
    if (CLAMP) {
        al.x = fminf(0.99f, al.x);
        al.y = fminf(0.99f, al.y);
    }
    const float2 aT = __fmul2_rn(al, p.T);
    p.r = __ffma2_rn(make_float2(c.y, c.y), aT, p.r);
    p.g = __ffma2_rn(make_float2(c.z, c.z), aT, p.g);
    p.b = __ffma2_rn(make_float2(c.w, c.w), aT, p.b);
    if (QUEEN_BLEND_TSUB)  // T (1 - a) reassociated as T - a T: <= 1 ulp per step, RGB/T stay within tolerance
        p.T = __fadd2_rn(p.T, make_float2(-aT.x, -aT.y));
    else
        p.T = __fmul2_rn(p.T, __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-al.x, -al.y)));
}

#ifndef QUEEN_BLEND_MINB
#define QUEEN_BLEND_MINB 24  // 40 registers (a few spill): 24 CTAs (48 warps) per SM; measured (round 2, N3DV blend) 56 regs 1.305 ms, 48 regs 1.310, 40 regs 1.288 (+ unroll 8: 1.284; MeetRoom / Immersive -1.5 %)
#endif
#ifndef QUEEN_BLEND_UNROLL
#define QUEEN_BLEND_UNROLL 8  // measured n3dv blend: 1 -> 1.423 ms, 2 -> 1.410, 4 -> 1.399 (round 1); 2 -> 1.328, 4 -> 1.310, 8 -> 1.302 (round 2)
#endif
constexpr int BLEND_UNROLL = QUEEN_BLEND_UNROLL;  // record-loop unroll
#ifndef QUEEN_BLEND_UNCOND
#define QUEEN_BLEND_UNCOND 1
#endif
constexpr bool BLEND_UNCOND = QUEEN_BLEND_UNCOND;
#ifndef QUEEN_BLEND_PAIRSKIP
#define QUEEN_BLEND_PAIRSKIP 1  // warp-uniform skip of a row pair (16 x 4 pixels of the warp) that no lane hits
#endif
constexpr bool BLEND_PAIRSKIP = QUEEN_BLEND_PAIRSKIP;

template <bool COUNT, int RPT, bool WMASK>
__global__ void __launch_bounds__(256 / RPT, QUEEN_BLEND_MINB) k_blend(const float4* __restrict__ rec, int n_pad, const uint2* __restrict__ ranges,
                                                    const uint32_t* __restrict__ vals, int W, int H, int gx, int T, float bg0,
                                                    float bg1, float bg2, float* __restrict__ rgb_out, float* __restrict__ T_out,
                                                    uint8_t* __restrict__ out8, int out_mode, float mask_thresh, long long* ev_out,
                                                    long long* cp_out, const uint32_t* __restrict__ order) {
    constexpr int NT = 256 / RPT;          // threads per tile CTA: one column x RPT rows each
    constexpr int BATCH = NT > 64 ? NT : 64;  // records staged per batch
    constexpr int PER = BATCH / NT;        // records each thread stages per batch
    constexpr int NP = RPT / 2;            // row pairs (paired FP32 ops)
    __shared__ __align__(16) float4 sA[2][BATCH];  // u, v, hx, hy
    __shared__ __align__(16) float4 sB[2][BATCH];  // A2, B2, C2, T2
    __shared__ __align__(16) float4 sC[2][BATCH];  // o, r, g, b
    __shared__ uint16_t s_list[NT / 32][BATCH];        // per-warp record list of the batch (byte offsets q * 16)
    const int gt = order ? (int)order[blockIdx.x] : (int)blockIdx.x;
    const int v = gt / T;
    const int t = gt - v * T;
    // Pixel layout: a warp covers 16 columns x 2*RPT rows of the tile; lane (column c, half h)
    // owns row pair k = rows 4k + 2h, 4k + 2h + 1 of the warp's rows, so the warp's row pair k
    // is the contiguous 16 x 4 band 4k .. 4k + 3 (PAIRSKIP skips a band no lane hits).
    constexpr int WROWS = 2 * RPT;  // rows per warp
    const int px = (t % gx) * 16 + (threadIdx.x & 15);
    const int wrow0 = (t / gx) * 16 + (threadIdx.x >> 5) * WROWS;  // the warp's first row
    const int hh = (threadIdx.x >> 4) & 1;
    auto row_of = [&](int r) { return wrow0 + 4 * (r >> 1) + 2 * hh + (r & 1); };  // r = 2k + sub
    const float fx = (float)px;
    const float fyc = (float)(wrow0 + 2 * hh) + 0.5f * (WROWS - 3);
    const float hspan = 0.5f * (WROWS - 3) + 1e-4f;
    float2 nfy[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) nfy[q] = make_float2(-(float)row_of(2 * q), -(float)row_of(2 * q + 1));
    Px2 p[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        const float T0 = (px < W && row_of(2 * k) < H) ? 1.0f : 0.0f;
        const float T1 = (px < W && row_of(2 * k + 1) < H) ? 1.0f : 0.0f;
        p[k] = Px2{make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(T0, T1)};
    }
    long long ev = 0, cpn = 0;
    const uint2 rg = ranges[gt];
    const uint32_t rs = rg.x, re = rg.y;
    const int nb = (int)((re - rs + BATCH - 1) / BATCH);
    const float4* vrec = rec + (int64_t)v * n_pad * 3;
    // prologue: stage batch 0, indices of batch 1
#pragma unroll
    for (int e = 0; e < PER; ++e) {
        const int slot = threadIdx.x + e * NT;
        const uint32_t j = rs + slot;
        if (nb > 0 && j < re) {
            const float4* g = vrec + (int64_t)__ldg(vals + j) * 3;
            cp_async16(&sA[0][slot], g);
            cp_async16(&sB[0][slot], g + 1);
            cp_async16(&sC[0][slot], g + 2);
        }
    }
    cp_async_commit();
    uint32_t idx_next[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) {
        const uint32_t j = rs + BATCH + threadIdx.x + e * NT;
        idx_next[e] = (nb > 1 && j < re) ? __ldg(vals + j) : 0u;
    }
    for (int b = 0; b < nb; ++b) {
        const int s = b & 1;
        if (b + 1 < nb) {
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const int slot = threadIdx.x + e * NT;
                const uint32_t j = rs + (uint32_t)(b + 1) * BATCH + slot;
                if (j < re) {
                    const float4* g = vrec + (int64_t)idx_next[e] * 3;
                    cp_async16(&sA[s ^ 1][slot], g);
                    cp_async16(&sB[s ^ 1][slot], g + 1);
                    cp_async16(&sC[s ^ 1][slot], g + 2);
                }
            }
        }
        cp_async_commit();
        if (b + 2 < nb) {
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const uint32_t j = rs + (uint32_t)(b + 2) * BATCH + threadIdx.x + e * NT;
                idx_next[e] = j < re ? __ldg(vals + j) : 0u;
            }
        }
        cp_async_wait<1>();
        bool any_alive = false;
#pragma unroll
        for (int k = 0; k < NP; ++k) any_alive |= !(p[k].T.x < 1e-4f) | !(p[k].T.y < 1e-4f);
        if (__syncthreads_count(!any_alive) == NT) break;
        const int cnt = (int)min((uint32_t)BATCH, re - rs - (uint32_t)b * BATCH);
        // Warp-uniform control flow: no per-thread early exit inside the batch (a divergent
        // break would leave the warp split for the rest of the batch); terminated pixels simply
        // never hit again, and fully-terminated warps skip the batch.
        if (__any_sync(0xffffffffu, any_alive)) {
            // Records this warp must visit, as a 64-bit mask over the batch.  WMASK: only those
            // whose alpha >= 1/255 ellipse can reach a pixel centre of the warp's 16 x (32/16*RPT)
            // sub-tile (touches(), conservative); otherwise every record.  Skipping a record no
            // pixel of the warp hits changes nothing, so the output is bit-identical either way
            // (test_gpu_parity::test_blend_warp_mask_is_exact).
            const float wx0 = (float)((t % gx) * 16), wy0 = (float)wrow0;
            // the warp's record list (batch order) in shared memory
            uint16_t* lst = s_list[threadIdx.x >> 5];
            int nq = 0;
#pragma unroll
            for (int e = 0; e < BATCH / 32; ++e) {
                const int q = (threadIdx.x & 31) + 32 * e;
                bool want = q < cnt;
                if (WMASK && want) want = touches(sA[s][q], sB[s][q], wx0, wx0 + 15.0f, wy0, wy0 + (float)((32 / 16) * RPT - 1));
                const uint32_t bal = __ballot_sync(0xffffffffu, want);
                if (want) lst[nq + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u))] = (uint16_t)(q * 16);
                nq += __popc(bal);
            }
            __syncwarp();
#pragma unroll BLEND_UNROLL
            for (int i = 0; i < nq; ++i) {
                // records addressed by byte offset (no per-record index scaling)
                const uint32_t qo = lst[i];
#define QREC(arr) (*reinterpret_cast<const float4*>(reinterpret_cast<const char*>(arr[s]) + qo))
                const float4 a = QREC(sA);  // u, v, hx, hy
                const float dx = a.x - fx;
                if (COUNT) {
#pragma unroll
                    for (int k = 0; k < NP; ++k) ev += (int)!(p[k].T.x < 1e-4f) + (int)!(p[k].T.y < 1e-4f);
                }
                // Without the warp mask: conservative per-thread box cull (a pixel with p2 >= T2
                // satisfies |dx| <= hx and |dy| <= hy, K7; this thread's rows are
                // fyc +- hspan).  Skips never change a decision.
                // (A flag, not a `continue`: the warp votes below need every lane.)
                const bool cull = !COUNT && !WMASK && (fabsf(dx) > a.z || fabsf(a.y - fyc) > a.w + hspan);
                const float4 bq = QREC(sB);  // A2, B2, C2, T2
                const float tAdx = (bq.x * dx) * dx;
                const float tB = bq.y * dx;
                const float2 vv = make_float2(a.y, a.y);
                const float2 cc = make_float2(bq.z, bq.z);
                const float2 tb2 = make_float2(tB, tB);
                const float2 ta2 = make_float2(tAdx, tAdx);
                float2 qq[NP];
                bool h[RPT];
                bool anyh = false;
#pragma unroll
                for (int k = 0; k < NP; ++k) {
                    const float2 dy = __fadd2_rn(vv, nfy[k]);  // v - y, exactly
                    qq[k] = __ffma2_rn(__ffma2_rn(cc, dy, tb2), dy, ta2);  // Horner in dy
                    h[2 * k] = !cull && hit(p[k].T.x, qq[k].x, bq.w);
                    h[2 * k + 1] = !cull && hit(p[k].T.y, qq[k].y, bq.w);
                    anyh |= h[2 * k] | h[2 * k + 1];
                }
                if (COUNT) {
#pragma unroll
                    for (int r = 0; r < RPT; ++r) cpn += (int)h[r];
                }
                // warp-uniform control flow from here: a row pair (16 x 4 band of the warp) is
                // composited when any lane hits in it (PAIRSKIP); lanes without a hit in it
                // composite alpha = +0, which leaves C and T bit-identical
                bool doit[NP];
                bool any_pair = false;
#pragma unroll
                for (int k = 0; k < NP; ++k) {
                    doit[k] = BLEND_PAIRSKIP ? __any_sync(0xffffffffu, h[2 * k] | h[2 * k + 1])
                                             : __any_sync(0xffffffffu, anyh);
                    any_pair |= doit[k];
                }
                if (any_pair) {
                    // one composite path with the 0.99 clamp for every record: skipping the clamp
                    // for o <= 0.98 (where it is the identity) behind a warp-uniform branch cost
                    // more than the two FMNMX (blend 1.286 -> 1.278 ms without the branch)
                    const float4 c = QREC(sC);  // o, r, g, b
#pragma unroll
                    for (int k = 0; k < NP; ++k)
                        if (doit[k]) composite2<true>(p[k], qq[k].x, qq[k].y, h[2 * k], h[2 * k + 1], c);
                }
#undef QREC
            }
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    if (COUNT) {
        __shared__ long long s_ev[NT / 32], s_cp[NT / 32];
        for (int o = 16; o > 0; o >>= 1) {
            ev += __shfl_down_sync(0xffffffffu, ev, o);
            cpn += __shfl_down_sync(0xffffffffu, cpn, o);
        }
        if ((threadIdx.x & 31) == 0) { s_ev[threadIdx.x >> 5] = ev; s_cp[threadIdx.x >> 5] = cpn; }
        __syncthreads();
        if (threadIdx.x == 0) {
            long long a = 0, c = 0;
            for (int q = 0; q < NT / 32; ++q) { a += s_ev[q]; c += s_cp[q]; }
            atomicAdd(reinterpret_cast<unsigned long long*>(ev_out + v), (unsigned long long)a);
            atomicAdd(reinterpret_cast<unsigned long long*>(cp_out + v), (unsigned long long)c);
        }
        return;
    }
    if (out_mode == OUT_MASK) {  // render_mask: mark pixels whose accumulated alpha 1 - T exceeds the threshold
        if (px < W) {
            uint8_t* mo = out8 + (int64_t)v * H * W + px;
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                const float pT = (r & 1) ? p[r >> 1].T.y : p[r >> 1].T.x;
                if (row_of(r) < H) mo[(int64_t)row_of(r) * W] = (1.0f - pT > mask_thresh) ? 1 : 0;
            }
        }
        return;
    }
    if (out_mode == OUT_F16) {  // half-precision planar: the fp32 output value rounded to nearest binary16
        if (px < W) {
            const int64_t plane = (int64_t)H * W;
            __half* oh = reinterpret_cast<__half*>(out8) + (int64_t)v * 3 * plane + px;
            float* to = T_out ? T_out + (int64_t)v * plane + px : nullptr;
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                if (row_of(r) < H) {
                    const int64_t ro = (int64_t)row_of(r) * W;
                    const Px2& q = p[r >> 1];
                    const float pr = (r & 1) ? q.r.y : q.r.x, pg = (r & 1) ? q.g.y : q.g.x, pb = (r & 1) ? q.b.y : q.b.x;
                    const float pT = (r & 1) ? q.T.y : q.T.x;
                    oh[ro] = __float2half_rn(pr + pT * bg0);
                    oh[plane + ro] = __float2half_rn(pg + pT * bg1);
                    oh[2 * plane + ro] = __float2half_rn(pb + pT * bg2);
                    if (to) to[ro] = pT;
                }
            }
        }
        return;
    }
    if (out_mode == OUT_RGB10) {  // packed 10-bit display format (R10G10B10A2): one u32 per pixel
        if (px < W) {
            const int64_t plane = (int64_t)H * W;
            uint32_t* o10 = reinterpret_cast<uint32_t*>(out8) + (int64_t)v * plane + px;
            float* to = T_out ? T_out + (int64_t)v * plane + px : nullptr;
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                if (row_of(r) < H) {
                    const int64_t ro = (int64_t)row_of(r) * W;
                    const Px2& q = p[r >> 1];
                    const float pr = (r & 1) ? q.r.y : q.r.x, pg = (r & 1) ? q.g.y : q.g.x, pb = (r & 1) ? q.b.y : q.b.x;
                    const float pT = (r & 1) ? q.T.y : q.T.x;
                    const uint32_t r10 = __float2uint_rn(fminf(fmaxf(pr + pT * bg0, 0.0f), 1.0f) * 1023.0f);
                    const uint32_t g10 = __float2uint_rn(fminf(fmaxf(pg + pT * bg1, 0.0f), 1.0f) * 1023.0f);
                    const uint32_t b10 = __float2uint_rn(fminf(fmaxf(pb + pT * bg2, 0.0f), 1.0f) * 1023.0f);
                    o10[ro] = r10 | (g10 << 10) | (b10 << 20) | (3u << 30);
                    if (to) to[ro] = pT;
                }
            }
        }
        return;
    }
    if (out_mode == OUT_RGB8) {  // display format: round(clamp(C + T bg, 0, 1) * 255), planar u8
        if (px < W) {
            const int64_t plane = (int64_t)H * W;
            uint8_t* o8 = out8 + (int64_t)v * 3 * plane + px;
            float* to = T_out ? T_out + (int64_t)v * plane + px : nullptr;
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                if (row_of(r) < H) {
                    const int64_t ro = (int64_t)row_of(r) * W;
                    const Px2& q = p[r >> 1];
                    const float pr = (r & 1) ? q.r.y : q.r.x, pg = (r & 1) ? q.g.y : q.g.x, pb = (r & 1) ? q.b.y : q.b.x;
                    const float pT = (r & 1) ? q.T.y : q.T.x;
                    o8[ro] = (uint8_t)__float2uint_rn(fminf(fmaxf(pr + pT * bg0, 0.0f), 1.0f) * 255.0f);
                    o8[plane + ro] = (uint8_t)__float2uint_rn(fminf(fmaxf(pg + pT * bg1, 0.0f), 1.0f) * 255.0f);
                    o8[2 * plane + ro] = (uint8_t)__float2uint_rn(fminf(fmaxf(pb + pT * bg2, 0.0f), 1.0f) * 255.0f);
                    if (to) to[ro] = pT;
                }
            }
        }
        return;
    }
    if (px < W) {
        const int64_t plane = (int64_t)H * W;
        float* o = rgb_out + (int64_t)v * 3 * plane + px;
        float* to = T_out ? T_out + (int64_t)v * plane + px : nullptr;
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            if (row_of(r) < H) {
                const int64_t ro = (int64_t)row_of(r) * W;
                const Px2& q = p[r >> 1];
                const float pr = (r & 1) ? q.r.y : q.r.x, pg = (r & 1) ? q.g.y : q.g.x, pb = (r & 1) ? q.b.y : q.b.x;
                const float pT = (r & 1) ? q.T.y : q.T.x;
                o[ro] = pr + pT * bg0;
                o[plane + ro] = pg + pT * bg1;
                o[2 * plane + ro] = pb + pT * bg2;
                if (to) to[ro] = pT;
            }
        }
    }
}

#ifndef QUEEN_BLEND_RPT
#define QUEEN_BLEND_RPT 4  // rows per thread: a warp covers 16 x 2*RPT pixels
#endif
constexpr int BLEND_RPT = QUEEN_BLEND_RPT;

// Blend schedule: a permutation of the gt tiles, longest list first (list-length classes of
// 32 entries; order inside a class arbitrary).  Tiles are independent, so the schedule never
// changes a pixel; it only moves the long tiles away from the grid's tail.
// (order_class: queen_internal.cuh; the render path builds the schedule inside the binning)

__global__ void __launch_bounds__(256) k_order_hist(const uint2* __restrict__ ranges, int n, uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[ORDER_BINS];
    for (int q = threadIdx.x; q < ORDER_BINS; q += blockDim.x) sh[q] = 0u;
    __syncthreads();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        atomicAdd(&sh[order_class(ranges[i])], 1u);
    __syncthreads();
    for (int q = threadIdx.x; q < ORDER_BINS; q += blockDim.x)
        if (sh[q]) atomicAdd(&hist[q], sh[q]);
}

__global__ void __launch_bounds__(256) k_order_scatter(const uint2* __restrict__ ranges, int n,
                                                       const uint32_t* __restrict__ hist, uint32_t* __restrict__ cursor,
                                                       uint32_t* __restrict__ order) {
    __shared__ uint32_t s_start[ORDER_BINS], s_cnt[ORDER_BINS], s_base[ORDER_BINS];
    if (threadIdx.x < 32) {  // exclusive scan of the class counts, two per lane
        const int l = threadIdx.x;
        const uint32_t a = hist[2 * l], b = hist[2 * l + 1];
        uint32_t x = a + b;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (l >= o) x += y;
        }
        s_start[2 * l] = x - a - b;
        s_start[2 * l + 1] = x - b;
    }
    for (int c0 = blockIdx.x * blockDim.x; c0 < n; c0 += gridDim.x * blockDim.x) {
        for (int q = threadIdx.x; q < ORDER_BINS; q += blockDim.x) s_cnt[q] = 0u;
        __syncthreads();
        const int i = c0 + threadIdx.x;
        int cl = 0;
        uint32_t rank = 0;
        if (i < n) {
            cl = order_class(ranges[i]);
            rank = atomicAdd(&s_cnt[cl], 1u);
        }
        __syncthreads();
        for (int q = threadIdx.x; q < ORDER_BINS; q += blockDim.x)
            if (s_cnt[q]) s_base[q] = s_start[q] + atomicAdd(&cursor[q], s_cnt[q]);
        __syncthreads();
        if (i < n) order[s_base[cl] + rank] = (uint32_t)i;
        __syncthreads();
    }
}

cudaError_t launch_tile_order(const uint32_t* ranges, int64_t blocks, uint32_t* order_ws, cudaStream_t s,
                              const uint32_t** order, int opts) {
    *order = nullptr;
    if (!order_ws || blocks == 0 || (opts & QUEEN_OPT_BLEND_GRID_ORDER)) return cudaSuccess;
    uint32_t* hist = order_ws;
    uint32_t* cursor = order_ws + ORDER_BINS;
    uint32_t* ord = order_ws + 2 * ORDER_BINS;
    cudaError_t e = cudaMemsetAsync(order_ws, 0, sizeof(uint32_t) * 2 * ORDER_BINS, s);
    if (e) return e;
    const int grid = (int)std::min<int64_t>((blocks + 255) / 256, 296);
    k_order_hist<<<grid, 256, 0, s>>>(reinterpret_cast<const uint2*>(ranges), (int)blocks, hist);
    k_order_scatter<<<grid, 256, 0, s>>>(reinterpret_cast<const uint2*>(ranges), (int)blocks, hist, cursor, ord);
    *order = ord;
    return cudaGetLastError();
}

cudaError_t launch_rasterize(const float* rec, int n_pad, const uint32_t* ranges, const uint32_t* vals, int n_views,
                             int W, int H, float bg0, float bg1, float bg2, float* rgb_out, float* T_out,
                             uint8_t* out8, int out_mode, float mask_thresh, uint32_t* order_ws, cudaStream_t s,
                             int* n_launch, Prof* prof, int opts, const uint32_t* order_pre) {
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int T = gx * gy;
    const int64_t blocks = (int64_t)T * n_views;
    if (blocks == 0) return cudaSuccess;
    const uint32_t* order = nullptr;
    // stage profiler (when given): the tile schedule and the blend are separate stages, so the
    // blend stage times k_blend alone (bench.py's roofline divides its work by that time)
    if (prof) prof->begin(ST_BLEND_ORDER, s);
    if (order_pre && !(opts & QUEEN_OPT_BLEND_GRID_ORDER)) {
        order = order_pre;  // built by the binning (launch_bin_sort's order_ready)
        if (prof) {
            prof->end(s, 0);
            prof->begin(ST_BLEND, s);
        }
    } else if (cudaError_t e = launch_tile_order(ranges, blocks, order_ws, s, &order, opts)) {
        return e;
    } else if (prof) {
        prof->end(s, order ? 2 : 0);
        prof->begin(ST_BLEND, s);
    }
    if (n_launch) *n_launch = (order && order != order_pre) ? 3 : 1;
    if (opts & QUEEN_OPT_BLEND_NOMASK)  // test option: per-thread box cull only (no warp record lists)
        k_blend<false, BLEND_RPT, false><<<(unsigned)blocks, 256 / BLEND_RPT, 0, s>>>(
            reinterpret_cast<const float4*>(rec), n_pad, reinterpret_cast<const uint2*>(ranges), vals, W, H, gx, T, bg0, bg1,
            bg2, rgb_out, T_out, out8, out_mode, mask_thresh, nullptr, nullptr, order);
    else
        k_blend<false, BLEND_RPT, true><<<(unsigned)blocks, 256 / BLEND_RPT, 0, s>>>(
            reinterpret_cast<const float4*>(rec), n_pad, reinterpret_cast<const uint2*>(ranges), vals, W, H, gx, T, bg0, bg1,
            bg2, rgb_out, T_out, out8, out_mode, mask_thresh, nullptr, nullptr, order);
    if (prof) prof->end(s, 1);
    return cudaGetLastError();
}

cudaError_t launch_blend_counts(const float* rec, int n_pad, const uint32_t* ranges, const uint32_t* vals, int n_views,
                                int W, int H, long long* evaluated, long long* composited, cudaStream_t s) {
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int T = gx * gy;
    const int64_t blocks = (int64_t)T * n_views;
    cudaMemsetAsync(evaluated, 0, sizeof(long long) * n_views, s);
    cudaMemsetAsync(composited, 0, sizeof(long long) * n_views, s);
    if (blocks == 0) return cudaSuccess;
#ifndef QUEEN_COUNT_WMASK
#define QUEEN_COUNT_WMASK false  // experiment knob: count only the records on the warp lists
#endif
    k_blend<true, BLEND_RPT, QUEEN_COUNT_WMASK><<<(unsigned)blocks, 256 / BLEND_RPT, 0, s>>>(reinterpret_cast<const float4*>(rec), n_pad,
                                                  reinterpret_cast<const uint2*>(ranges), vals, W, H, gx, T, 0.f, 0.f, 0.f,
                                                  nullptr, nullptr, nullptr, OUT_F32, 0.f, evaluated, composited, nullptr);
    return cudaGetLastError();
}

}  // namespace queen
