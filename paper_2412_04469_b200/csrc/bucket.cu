// Binning, BUCKET mode (queen_set_binning): the same (gt, depth, index) order as
// the onesweep LSD sort of binning.cu, built without any global sort:
//   1. k_diff_rects       each visible (view, Gaussian) adds its tile rect to the view's 2D
//                         difference array of per-tile entry counts (4 corner increments)
//   2. k_tile_counts      per-view 2D prefix sums -> entries per global tile gt (binning.cu)
//   3. k_ranges_finalize  exclusive scan -> ranges[gt] = [first, last+1) (binning.cu); K,
//                         capacity overflow
//   4. k_emit             every entry takes a slot inside its tile's range with an atomic
//                         per-tile cursor and stores (depth bits, Gaussian index) there --
//                         the order inside a tile is arbitrary at this point
//   5. k_tile_sort        one CTA per tile sorts its (depth bits << 32 | index) keys with a
//                         Batcher odd-even merge network (shared memory up to 2048 entries,
//                         in place in global memory beyond), then writes vals = index and
//                         keys = gt
// Inside a tile the keys (depth, index) are unique, so the result is exactly the oracle's
// std::sort order, independent of the atomic slot order (deterministic output).
#include "queen_internal.cuh"

namespace queen {

constexpr int TS_THREADS = 128;
constexpr int TS_CAP = 2048;  // entries sorted in shared memory (16 KB of u64 keys)

__global__ void __launch_bounds__(256) k_diff_rects(const uint32_t* __restrict__ tiles, const short4* __restrict__ rect,
                                                    int64_t count, int n_pad, int gx, int gy, int* __restrict__ diff) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= count || tiles[j] == 0) return;
    const int v = (int)(j / n_pad);
    const short4 r = rect[j];
    const int dw = gx + 1;
    int* d = diff + (int64_t)v * dw * (gy + 1);
    atomicAdd(d + r.y * dw + r.x, 1);
    atomicAdd(d + r.y * dw + r.z + 1, -1);
    atomicAdd(d + (r.w + 1) * dw + r.x, -1);
    atomicAdd(d + (r.w + 1) * dw + r.z + 1, 1);
}

// one (view, Gaussian) element: lanes with small rects emit their own entries; rects with
// more than 32 tiles are emitted cooperatively by the whole warp (lanes stride the tiles)
__global__ void __launch_bounds__(256) k_emit(const uint32_t* __restrict__ tiles, const short4* __restrict__ rect,
                                              const uint32_t* __restrict__ depth, int64_t count, int n_pad, int gx,
                                              uint32_t T, const uint2* __restrict__ ranges, uint32_t* __restrict__ fill,
                                              const uint32_t* Kd, uint32_t* __restrict__ dkey, uint32_t* __restrict__ dval) {
    if (Kd[2] != 0u) return;  // capacity overflow: no entries (flagged)
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t nt = j < count ? tiles[j] : 0u;
    const uint32_t lane = threadIdx.x & 31;
    short4 r = make_short4(0, 0, -1, -1);
    uint32_t d = 0, i = 0, vT = 0;
    if (nt) {
        const uint32_t v = (uint32_t)(j / n_pad);
        r = rect[j];
        d = depth[j];
        i = (uint32_t)(j - (int64_t)v * n_pad);
        vT = v * T;
    }
    if (nt && nt <= 32) {
        const int wx = r.z - r.x + 1;
        for (uint32_t c = 0; c < nt; ++c) {
            const int row = (int)c / wx;
            const uint32_t g = vT + (uint32_t)(r.y + row) * (uint32_t)gx + (uint32_t)(r.x + (int)c - row * wx);
            const uint32_t pos = ranges[g].x + atomicAdd(&fill[g], 1u);
            dkey[pos] = d;
            dval[pos] = i;
        }
    }
    uint32_t big = __ballot_sync(0xffffffffu, nt > 32);
    while (big) {
        const int src = __ffs(big) - 1;
        big &= big - 1;
        const uint32_t bnt = __shfl_sync(0xffffffffu, nt, src);
        const int bx0 = __shfl_sync(0xffffffffu, (int)r.x, src), by0 = __shfl_sync(0xffffffffu, (int)r.y, src);
        const int bwx = __shfl_sync(0xffffffffu, (int)(r.z - r.x + 1), src);
        const uint32_t bd = __shfl_sync(0xffffffffu, d, src), bi = __shfl_sync(0xffffffffu, i, src);
        const uint32_t bvT = __shfl_sync(0xffffffffu, vT, src);
        for (uint32_t c = lane; c < bnt; c += 32) {
            const int row = (int)c / bwx;
            const uint32_t g = bvT + (uint32_t)(by0 + row) * (uint32_t)gx + (uint32_t)(bx0 + (int)c - row * bwx);
            const uint32_t pos = ranges[g].x + atomicAdd(&fill[g], 1u);
            dkey[pos] = bd;
            dval[pos] = bi;
        }
    }
}

// Batcher's odd-even merge sort network on n keys (arbitrary n: comparators reaching past
// n are dropped, valid because every comparator puts the minimum at the lower index).
template <typename Cswap>
__device__ __forceinline__ void oddeven_merge_sort(uint32_t n, Cswap cswap) {
    for (uint32_t p = 1; p < n; p <<= 1) {
        for (uint32_t k = p; k >= 1; k >>= 1) {
            const uint32_t j0 = k % p;
            for (uint32_t a = j0 + threadIdx.x; a + k < n; a += blockDim.x) {
                if (((a - j0) % (2 * k)) < k && (a / (2 * p)) == ((a + k) / (2 * p))) cswap(a, a + k);
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(TS_THREADS) k_tile_sort(const uint2* __restrict__ ranges, uint32_t* __restrict__ dkey,
                                                          uint32_t* __restrict__ dval, uint32_t* __restrict__ keys,
                                                          uint32_t* __restrict__ vals) {
    __shared__ unsigned long long sk[TS_CAP];
    const uint32_t g = blockIdx.x;
    const uint2 rg = ranges[g];
    const uint32_t n = rg.y - rg.x;
    if (n == 0) return;
    if (n <= TS_CAP) {
        for (uint32_t q = threadIdx.x; q < n; q += blockDim.x)
            sk[q] = ((unsigned long long)dkey[rg.x + q] << 32) | dval[rg.x + q];
        __syncthreads();
        oddeven_merge_sort(n, [&](uint32_t a, uint32_t b) {
            const unsigned long long x = sk[a], y = sk[b];
            if (y < x) { sk[a] = y; sk[b] = x; }
        });
        for (uint32_t q = threadIdx.x; q < n; q += blockDim.x) {
            vals[rg.x + q] = (uint32_t)sk[q];
            keys[rg.x + q] = g;
        }
    } else {  // rare long lists: the same network in place on the global (depth, index) arrays
        uint32_t* k0 = dkey + rg.x;
        uint32_t* v0 = dval + rg.x;
        oddeven_merge_sort(n, [&](uint32_t a, uint32_t b) {
            const unsigned long long x = ((unsigned long long)k0[a] << 32) | v0[a];
            const unsigned long long y = ((unsigned long long)k0[b] << 32) | v0[b];
            if (y < x) {
                k0[a] = (uint32_t)(y >> 32); v0[a] = (uint32_t)y;
                k0[b] = (uint32_t)(x >> 32); v0[b] = (uint32_t)x;
            }
        });
        for (uint32_t q = threadIdx.x; q < n; q += blockDim.x) {
            vals[rg.x + q] = v0[q];
            keys[rg.x + q] = g;
        }
    }
}

// defined in binning.cu (k_tile_counts / k_ranges_finalize)
void launch_tile_counts(const int* diff, int gx, int gy, int n_views, uint32_t* counts, uint32_t* lstart,
                        uint32_t* view_tot, cudaStream_t s);
void launch_ranges_finalize(const uint32_t* counts, const uint32_t* lstart, const uint32_t* view_tot, int n_views,
                            uint32_t T, uint32_t cap, const uint32_t* Kd, uint2* ranges, int grid, cudaStream_t s);

// K, overflow flag and capacity error from the per-view totals (one thread)
__global__ void k_bucket_total(const uint32_t* __restrict__ view_tot, int n_views, uint32_t cap, uint32_t* Kd,
                               DevFlags* fl) {
    unsigned long long K = 0;
    for (int v = 0; v < n_views; ++v) K += view_tot[v];
    const bool over = K > cap;
    if (over) {
        raise_flag(fl, FLAG_CAPACITY);
        atomicMax(&fl->info, K);
    }
    Kd[0] = over ? 0u : (uint32_t)K;
    Kd[2] = over ? 1u : 0u;
}

__global__ void __launch_bounds__(256) k_count_visible(const uint32_t* __restrict__ tiles, int64_t count, uint32_t* Md) {
    uint32_t c = 0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x)
        c += tiles[j] ? 1u : 0u;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(Md, c);
}

cudaError_t launch_bin_bucket(const queen_proj& proj, int n_views, int W, int H, queen_bins& bins, void* scratch,
                              const WsLayout& L, DevFlags* fl, cudaStream_t s, Prof* prof, int sms) {
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int64_t T = (int64_t)gx * gy;
    const int64_t G = T * n_views;
    const int64_t count = (int64_t)n_views * proj.n_pad;
    const uint32_t cap = (uint32_t)bins.keys_cap;
    unsigned char* ws = static_cast<unsigned char*>(scratch);
    int* diff = reinterpret_cast<int*>(ws + L.diff);
    uint32_t* tcounts = reinterpret_cast<uint32_t*>(ws + L.counts);  // counts | local starts | fill cursors
    uint32_t* lstart = tcounts + G;
    uint32_t* fill = tcounts + 2 * G;
    uint32_t* view_tot = reinterpret_cast<uint32_t*>(ws + L.view_tot);
    const size_t dplane = (size_t)(gx + 1) * (gy + 1);
    cudaError_t e;
    prof->begin(ST_COMPACT, s);
    if ((e = cudaMemsetAsync(diff, 0, sizeof(int) * dplane * n_views, s))) return e;
    if ((e = cudaMemsetAsync(fill, 0, sizeof(uint32_t) * G, s))) return e;
    if ((e = cudaMemsetAsync(bins.K, 0, sizeof(uint32_t) * 4, s))) return e;
    const unsigned eb = (unsigned)((count + 255) / 256);
    if (count > 0) {
        k_diff_rects<<<eb, 256, 0, s>>>(proj.tiles, reinterpret_cast<const short4*>(proj.rect), count, proj.n_pad, gx, gy,
                                       diff);
        k_count_visible<<<sms * 2, 256, 0, s>>>(proj.tiles, count, bins.K + 1);
    }
    prof->end(s, count > 0 ? 2 : 0);
    prof->begin(ST_RANGES, s);
    launch_tile_counts(diff, gx, gy, n_views, tcounts, lstart, view_tot, s);
    k_bucket_total<<<1, 1, 0, s>>>(view_tot, n_views, cap, bins.K, fl);
    launch_ranges_finalize(tcounts, lstart, view_tot, n_views, (uint32_t)T, cap, bins.K,
                           reinterpret_cast<uint2*>(bins.ranges), sms * 2, s);
    prof->end(s, 3);
    prof->begin(ST_DUPLICATE, s);
    if (count > 0)
        k_emit<<<eb, 256, 0, s>>>(proj.tiles, reinterpret_cast<const short4*>(proj.rect), proj.depth, count, proj.n_pad,
                                 gx, (uint32_t)T, reinterpret_cast<const uint2*>(bins.ranges), fill, bins.K,
                                 bins.keys_alt, bins.vals_alt);
    prof->end(s);
    prof->begin(ST_TILE_SORT, s);
    if (G > 0)
        k_tile_sort<<<(unsigned)G, TS_THREADS, 0, s>>>(reinterpret_cast<const uint2*>(bins.ranges), bins.keys_alt,
                                                       bins.vals_alt, bins.keys, bins.vals);
    prof->end(s);
    bins.sorted_in_alt = 0;
    return cudaGetLastError();
}

}  // namespace queen
