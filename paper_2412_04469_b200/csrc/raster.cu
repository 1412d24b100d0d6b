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
//  * all lanes read the same record (LDS.128 broadcast), and the CTA retires as soon
//    as all 256 pixels have terminated (__syncthreads_count).
// Per-pixel arithmetic is exactly the oracle's (oracle/queen_oracle.cpp blend_step):
//   p2 = fma(A2 dx, dx, fma(C2 dy, dy, (B2 dx) dy));  skip if p2 > 0 or p2 < T2;
//   a = min(0.99, o 2^p2); C = fma(rgb, a T, C); T = T (1 - a); stop after T < 1e-4.
#include "queen_internal.cuh"

namespace queen {

constexpr int BT = 64;      // threads per tile CTA
constexpr int BATCH = 64;   // records staged per batch (one per thread)

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

struct Px {
    float r, g, b, T;
    bool alive;
};

__device__ __forceinline__ bool hit(const Px& p, float p2, float T2) { return p.alive && !(p2 > 0.0f) && !(p2 < T2); }

__device__ __forceinline__ void composite(Px& p, float p2, const float4& c) {  // c = (o, r, g, b)
    const float alpha = fminf(0.99f, c.x * ex2(p2));
    const float aT = alpha * p.T;
    p.r = fmaf(c.y, aT, p.r);
    p.g = fmaf(c.z, aT, p.g);
    p.b = fmaf(c.w, aT, p.b);
    p.T = p.T * (1.0f - alpha);
    if (p.T < 1e-4f) p.alive = false;
}

template <bool COUNT>
__global__ void __launch_bounds__(BT) k_blend(const float4* __restrict__ rec, int n_pad, const uint2* __restrict__ ranges,
                                              const uint32_t* __restrict__ vals, int W, int H, int gx, int T, float bg0,
                                              float bg1, float bg2, float* __restrict__ rgb_out, float* __restrict__ T_out,
                                              long long* ev_out, long long* cp_out) {
    __shared__ __align__(16) float4 sA[2][BATCH];  // u, v, hx, hy
    __shared__ __align__(16) float4 sB[2][BATCH];  // A2, B2, C2, T2
    __shared__ __align__(16) float4 sC[2][BATCH];  // o, r, g, b
    const int gt = blockIdx.x;
    const int v = gt / T;
    const int t = gt - v * T;
    const int px = (t % gx) * 16 + (threadIdx.x & 15);
    const int py0 = (t / gx) * 16 + (threadIdx.x >> 4) * 4;
    const float fx = (float)px;
    const float fyc = (float)py0 + 1.5f;
    const float2 nfy01 = make_float2(-(float)py0, -(float)(py0 + 1));
    const float2 nfy23 = make_float2(-(float)(py0 + 2), -(float)(py0 + 3));
    Px p0{0.f, 0.f, 0.f, 1.f, px < W && py0 < H};
    Px p1{0.f, 0.f, 0.f, 1.f, px < W && py0 + 1 < H};
    Px p2{0.f, 0.f, 0.f, 1.f, px < W && py0 + 2 < H};
    Px p3{0.f, 0.f, 0.f, 1.f, px < W && py0 + 3 < H};
    long long ev = 0, cpn = 0;
    const uint2 rg = ranges[gt];
    const uint32_t rs = rg.x, re = rg.y;
    const int nb = (int)((re - rs + BATCH - 1) / BATCH);
    const float4* vrec = rec + (int64_t)v * n_pad * 3;
    // prologue: stage batch 0, index of batch 1
    if (nb > 0) {
        const uint32_t j = rs + threadIdx.x;
        if (j < re) {
            const float4* g = vrec + (int64_t)__ldg(vals + j) * 3;
            cp_async16(&sA[0][threadIdx.x], g);
            cp_async16(&sB[0][threadIdx.x], g + 1);
            cp_async16(&sC[0][threadIdx.x], g + 2);
        }
    }
    cp_async_commit();
    uint32_t idx_next = 0;
    {
        const uint32_t j = rs + BATCH + threadIdx.x;
        if (nb > 1 && j < re) idx_next = __ldg(vals + j);
    }
    for (int b = 0; b < nb; ++b) {
        const int s = b & 1;
        if (b + 1 < nb) {
            const uint32_t j = rs + (uint32_t)(b + 1) * BATCH + threadIdx.x;
            if (j < re) {
                const float4* g = vrec + (int64_t)idx_next * 3;
                cp_async16(&sA[s ^ 1][threadIdx.x], g);
                cp_async16(&sB[s ^ 1][threadIdx.x], g + 1);
                cp_async16(&sC[s ^ 1][threadIdx.x], g + 2);
            }
        }
        cp_async_commit();
        if (b + 2 < nb) {
            const uint32_t j = rs + (uint32_t)(b + 2) * BATCH + threadIdx.x;
            idx_next = j < re ? __ldg(vals + j) : 0u;
        }
        cp_async_wait<1>();
        const bool done = !(p0.alive || p1.alive || p2.alive || p3.alive);
        if (__syncthreads_count(done) == BT) break;
        const int cnt = (int)min((uint32_t)BATCH, re - rs - (uint32_t)b * BATCH);
        // Warp-uniform control flow: no per-thread early exit inside the batch (a divergent
        // break would leave the warp split for the rest of the batch); terminated pixels simply
        // never hit again, and fully-terminated warps skip the batch.
        if (__any_sync(0xffffffffu, !done)) {
#pragma unroll 2
            for (int q = 0; q < cnt; ++q) {
                const float4 a = sA[s][q];  // u, v, hx, hy
                const float dx = a.x - fx;
                if (COUNT) ev += (int)p0.alive + (int)p1.alive + (int)p2.alive + (int)p3.alive;
                // Conservative box cull: a pixel with p2 >= T2 satisfies |dx| <= hx and |dy| <= hy
                // (bounding box of the alpha = 1/255 ellipse, 1e-4 relative slack, K7);
                // this thread's 4 rows are py0 + 1.5 +- 1.5.  Skips never change a decision.
                if (!COUNT && (fabsf(dx) > a.z || fabsf(a.y - fyc) > a.w + 1.5001f)) continue;
                const float4 bq = sB[s][q];  // A2, B2, C2, T2
                const float tA = bq.x * dx;
                const float tB = bq.y * dx;
                const float2 vv = make_float2(a.y, a.y);
                const float2 cc = make_float2(bq.z, bq.z);
                const float2 tb2 = make_float2(tB, tB);
                const float2 ta2 = make_float2(tA, tA);
                const float2 dx2 = make_float2(dx, dx);
                const float2 dy01 = __fadd2_rn(vv, nfy01);  // v - y, exactly
                const float2 dy23 = __fadd2_rn(vv, nfy23);
                const float2 q01 = __ffma2_rn(ta2, dx2, __ffma2_rn(__fmul2_rn(cc, dy01), dy01, __fmul2_rn(tb2, dy01)));
                const float2 q23 = __ffma2_rn(ta2, dx2, __ffma2_rn(__fmul2_rn(cc, dy23), dy23, __fmul2_rn(tb2, dy23)));
                const bool h0 = hit(p0, q01.x, bq.w), h1 = hit(p1, q01.y, bq.w);
                const bool h2 = hit(p2, q23.x, bq.w), h3 = hit(p3, q23.y, bq.w);
                if (COUNT) cpn += (int)h0 + (int)h1 + (int)h2 + (int)h3;
                if (h0 || h1 || h2 || h3) {
                    const float4 c = sC[s][q];  // o, r, g, b
                    if (h0) composite(p0, q01.x, c);
                    if (h1) composite(p1, q01.y, c);
                    if (h2) composite(p2, q23.x, c);
                    if (h3) composite(p3, q23.y, c);
                }
            }
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    if (COUNT) {
        __shared__ long long s_ev[BT / 32], s_cp[BT / 32];
        for (int o = 16; o > 0; o >>= 1) {
            ev += __shfl_down_sync(0xffffffffu, ev, o);
            cpn += __shfl_down_sync(0xffffffffu, cpn, o);
        }
        if ((threadIdx.x & 31) == 0) { s_ev[threadIdx.x >> 5] = ev; s_cp[threadIdx.x >> 5] = cpn; }
        __syncthreads();
        if (threadIdx.x == 0) {
            long long a = 0, c = 0;
            for (int q = 0; q < BT / 32; ++q) { a += s_ev[q]; c += s_cp[q]; }
            atomicAdd(reinterpret_cast<unsigned long long*>(ev_out + v), (unsigned long long)a);
            atomicAdd(reinterpret_cast<unsigned long long*>(cp_out + v), (unsigned long long)c);
        }
        return;
    }
    if (px < W) {
        const int64_t plane = (int64_t)H * W;
        float* o = rgb_out + (int64_t)v * 3 * plane + (int64_t)py0 * W + px;
        float* to = T_out ? T_out + (int64_t)v * plane + (int64_t)py0 * W + px : nullptr;
        const Px* ps[4] = {&p0, &p1, &p2, &p3};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (py0 + r < H) {
                const Px& q = *ps[r];
                o[(int64_t)r * W] = q.r + q.T * bg0;
                o[plane + (int64_t)r * W] = q.g + q.T * bg1;
                o[2 * plane + (int64_t)r * W] = q.b + q.T * bg2;
                if (to) to[(int64_t)r * W] = q.T;
            }
        }
    }
}

cudaError_t launch_rasterize(const float* rec, int n_pad, const uint32_t* ranges, const uint32_t* vals, int n_views,
                             int W, int H, float bg0, float bg1, float bg2, float* rgb_out, float* T_out,
                             cudaStream_t s) {
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int T = gx * gy;
    const int64_t blocks = (int64_t)T * n_views;
    if (blocks == 0) return cudaSuccess;
    k_blend<false><<<(unsigned)blocks, BT, 0, s>>>(reinterpret_cast<const float4*>(rec), n_pad,
                                                   reinterpret_cast<const uint2*>(ranges), vals, W, H, gx, T, bg0, bg1,
                                                   bg2, rgb_out, T_out, nullptr, nullptr);
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
    k_blend<true><<<(unsigned)blocks, BT, 0, s>>>(reinterpret_cast<const float4*>(rec), n_pad,
                                                  reinterpret_cast<const uint2*>(ranges), vals, W, H, gx, T, 0.f, 0.f, 0.f,
                                                  nullptr, nullptr, evaluated, composited);
    return cudaGetLastError();
}

}  // namespace queen
