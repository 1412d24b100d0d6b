// K7: per-tile front-to-back alpha compositing (Eq. 2) with the
// 3D-GS cut-offs of DESIGN reading R14 and composite-then-stop early termination.
//
// One 256-thread CTA per 16x16 tile (one pixel per thread).  The tile's sorted
// Gaussian list is consumed in batches of 256: each thread gathers one 48-byte
// record (three 16-byte loads via the sorted index) into shared memory, then every
// thread walks the batch for its pixel.  The CTA leaves as soon as every pixel has
// terminated (__syncthreads_count).  Per-pixel arithmetic is exactly the oracle's.
#include "queen_internal.cuh"

namespace queen {

constexpr int BLEND_THREADS = 256;

template <bool COUNT>
__global__ void __launch_bounds__(BLEND_THREADS) k_blend(const float4* __restrict__ rec, int n_pad,
                                                         const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
                                                         int W, int H, int gx, int T, float bg0, float bg1, float bg2,
                                                         float* __restrict__ rgb_out, float* __restrict__ T_out,
                                                         long long* ev_out, long long* cp_out) {
    __shared__ float4 s_a[BLEND_THREADS];  // u, v, A2, B2
    __shared__ float4 s_b[BLEND_THREADS];  // C2, T2, o, -
    __shared__ float4 s_c[BLEND_THREADS];  // r, g, b, -
    const int gt = blockIdx.x;
    const int v = gt / T;
    const int t = gt - v * T;
    const int px = (t % gx) * 16 + (threadIdx.x & 15);
    const int py = (t / gx) * 16 + (threadIdx.x >> 4);
    const bool inside = px < W && py < H;
    const float fx = (float)px, fy = (float)py;
    const uint2 rg = ranges[gt];
    const float4* vrec = rec + (int64_t)v * n_pad * 3;
    float C0 = 0.f, C1 = 0.f, C2c = 0.f, Tr = 1.f;
    bool done = !inside;
    long long ev = 0, cp = 0;
    for (uint32_t b = rg.x; b < rg.y; b += BLEND_THREADS) {
        if (__syncthreads_count(done) == BLEND_THREADS) break;
        const uint32_t j = b + threadIdx.x;
        if (j < rg.y) {
            const int64_t i = vals[j];
            s_a[threadIdx.x] = __ldg(vrec + i * 3 + 0);
            s_b[threadIdx.x] = __ldg(vrec + i * 3 + 1);
            s_c[threadIdx.x] = __ldg(vrec + i * 3 + 2);
        }
        __syncthreads();
        const int cnt = (int)min((uint32_t)BLEND_THREADS, rg.y - b);
        if (!done) {
            for (int q = 0; q < cnt; ++q) {
                const float4 A = s_a[q];
                const float4 Bq = s_b[q];
                const float dx = A.x - fx, dy = A.y - fy;
                const float p2 = fmaf(A.z * dx, dx, fmaf(Bq.x * dy, dy, (A.w * dx) * dy));
                if (COUNT) ++ev;
                if (p2 > 0.0f || p2 < Bq.y) continue;
                if (COUNT) ++cp;
                const float alpha = fminf(0.99f, Bq.z * exp2f(p2));
                const float aT = alpha * Tr;
                const float4 c = s_c[q];
                C0 = fmaf(c.x, aT, C0);
                C1 = fmaf(c.y, aT, C1);
                C2c = fmaf(c.z, aT, C2c);
                Tr = Tr * (1.0f - alpha);
                if (Tr < 1e-4f) { done = true; break; }
            }
        }
    }
    if (COUNT) {
        // per-view totals (debug/evidence only): block reduce then one atomic
        __shared__ long long s_ev[BLEND_THREADS / 32], s_cp[BLEND_THREADS / 32];
        for (int o = 16; o > 0; o >>= 1) {
            ev += __shfl_down_sync(0xffffffffu, ev, o);
            cp += __shfl_down_sync(0xffffffffu, cp, o);
        }
        if ((threadIdx.x & 31) == 0) { s_ev[threadIdx.x >> 5] = ev; s_cp[threadIdx.x >> 5] = cp; }
        __syncthreads();
        if (threadIdx.x == 0) {
            long long a = 0, c = 0;
            for (int q = 0; q < BLEND_THREADS / 32; ++q) { a += s_ev[q]; c += s_cp[q]; }
            atomicAdd(reinterpret_cast<unsigned long long*>(ev_out + v), (unsigned long long)a);
            atomicAdd(reinterpret_cast<unsigned long long*>(cp_out + v), (unsigned long long)c);
        }
        return;
    }
    if (inside) {
        const int64_t pix = (int64_t)py * W + px;
        const int64_t plane = (int64_t)H * W;
        float* o = rgb_out + (int64_t)v * 3 * plane + pix;
        o[0] = C0 + Tr * bg0;
        o[plane] = C1 + Tr * bg1;
        o[2 * plane] = C2c + Tr * bg2;
        if (T_out) T_out[(int64_t)v * plane + pix] = Tr;
    }
}

cudaError_t launch_rasterize(const float* rec, int n_pad, const uint32_t* ranges, const uint32_t* vals, int n_views,
                             int W, int H, float bg0, float bg1, float bg2, float* rgb_out, float* T_out,
                             cudaStream_t s) {
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int T = gx * gy;
    const int64_t blocks = (int64_t)T * n_views;
    if (blocks == 0) return cudaSuccess;
    k_blend<false><<<(unsigned)blocks, BLEND_THREADS, 0, s>>>(reinterpret_cast<const float4*>(rec), n_pad,
                                                              reinterpret_cast<const uint2*>(ranges), vals, W, H, gx, T,
                                                              bg0, bg1, bg2, rgb_out, T_out, nullptr, nullptr);
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
    k_blend<true><<<(unsigned)blocks, BLEND_THREADS, 0, s>>>(reinterpret_cast<const float4*>(rec), n_pad,
                                                             reinterpret_cast<const uint2*>(ranges), vals, W, H, gx, T,
                                                             0.f, 0.f, 0.f, nullptr, nullptr, evaluated, composited);
    return cudaGetLastError();
}

}  // namespace queen
