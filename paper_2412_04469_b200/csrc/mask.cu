// NEXT #3: masked / dynamic-subset rendering -- "we render dynamic Gaussians
// for each training view to identify corresponding dynamic image regions" and
// "we additionally dilate the image mask by a 48x48 kernel"; SPEC S:322-326:
// pixels whose accumulated alpha exceeds 1e-3 are marked, then dilated with a square kernel
// clipped at the image borders.
//
// queen_render_mask = k_select (subset -> per-Gaussian flags) -> k_project with the flags
// (others culled) -> binning -> k_blend writing marks (1 - T > threshold) -> k_dilate_rows
// -> k_dilate_cols.  The dilation window of output pixel x is [x - d/2, x - d/2 + d - 1] on
// each axis (the anchor convention of a centred d x d structuring element), clipped.
#include "queen_internal.cuh"

namespace queen {

// subset indices (strictly increasing, < n) -> select[i] = 1; invalid lists raise
// QUEEN_ERR_INDEX and select nothing for the offending entry
__global__ void __launch_bounds__(256) k_select(const uint32_t* __restrict__ idx, int kcap, const int32_t* k_dev, int n,
                                                uint8_t* __restrict__ select, DevFlags* fl) {
    int k = kcap;
    if (k_dev) k = min(max(*k_dev, 0), kcap);
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    const uint32_t i = idx[j];
    if (i >= (uint32_t)n || (j > 0 && i <= idx[j - 1])) {
        raise_flag(fl, FLAG_INDEX);
        return;
    }
    select[i] = 1;
}

// rows: one block per (row, view); exclusive prefix counts of the row's marks in shared
// memory, then out[x] = any mark in the clipped window
__global__ void __launch_bounds__(256) k_dilate_rows(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int W,
                                                     int H, int d) {
    extern __shared__ uint32_t cnt[];  // [W + 1]
    __shared__ uint32_t s_w[8];
    const int y = blockIdx.x, v = blockIdx.y;
    const uint8_t* row = in + ((int64_t)v * H + y) * W;
    uint8_t* orow = out + ((int64_t)v * H + y) * W;
    const int per = (W + blockDim.x - 1) / blockDim.x;
    const int x0 = threadIdx.x * per, x1 = min(W, x0 + per);
    uint32_t c = 0;
    for (int x = x0; x < x1; ++x) c += row[x] ? 1u : 0u;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = c;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    uint32_t pre = 0;
    for (int q = 0; q < w; ++q) pre += s_w[q];
    uint32_t run = pre + inc - c;
    for (int x = x0; x < x1; ++x) {
        cnt[x] = run;
        run += row[x] ? 1u : 0u;
    }
    if (x1 == W && x0 < W) cnt[W] = run;
    if (W == 0 && threadIdx.x == 0) cnt[0] = 0;
    __syncthreads();
    const int a = d / 2;
    for (int x = threadIdx.x; x < W; x += blockDim.x) {
        const int lo = max(0, x - a), hi = min(W, x - a + d);  // window [lo, hi)
        orow[x] = (lo < hi && cnt[hi] - cnt[lo] > 0) ? 1 : 0;
    }
}

// columns: one thread per column, a sliding window count down the column (coalesced rows)
__global__ void __launch_bounds__(256) k_dilate_cols(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int W,
                                                     int H, int d) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, v = blockIdx.y;
    if (x >= W) return;
    const uint8_t* col = in + (int64_t)v * H * W + x;
    uint8_t* ocol = out + (int64_t)v * H * W + x;
    const int a = d / 2;
    // window of output row y: [y - a, y - a + d - 1] clipped to [0, H)
    int c = 0;
    for (int r = 0; r < min(H, d - a); ++r) c += col[(int64_t)r * W] ? 1 : 0;  // window of y = 0: [-a, d - a - 1]
    for (int y = 0; y < H; ++y) {
        ocol[(int64_t)y * W] = c > 0 ? 1 : 0;
        const int add = y + 1 - a + d - 1, rem = y - a;  // window of y + 1 gains row add, loses row rem
        if (add >= 0 && add < H) c += col[(int64_t)add * W] ? 1 : 0;
        if (rem >= 0 && rem < H) c -= col[(int64_t)rem * W] ? 1 : 0;
    }
}

cudaError_t launch_select(const uint32_t* idx, int k, const int32_t* k_dev, int n, int n_pad, uint8_t* select,
                          DevFlags* fl, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(select, 0, (size_t)n_pad, s);
    if (e) return e;
    if (k > 0) k_select<<<(k + 255) / 256, 256, 0, s>>>(idx, k, k_dev, n, select, fl);
    return cudaGetLastError();
}

// marks (in/out, [V][H][W]) dilated in place through tmp
cudaError_t launch_dilate(uint8_t* marks, uint8_t* tmp, int n_views, int W, int H, int d, cudaStream_t s) {
    if (n_views <= 0 || W <= 0 || H <= 0 || d <= 1) return cudaSuccess;
    k_dilate_rows<<<dim3((unsigned)H, (unsigned)n_views), 256, sizeof(uint32_t) * (W + 1), s>>>(marks, tmp, W, H, d);
    k_dilate_cols<<<dim3((unsigned)((W + 255) / 256), (unsigned)n_views), 256, 0, s>>>(tmp, marks, W, H, d);
    return cudaGetLastError();
}

}  // namespace queen
