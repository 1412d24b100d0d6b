// K3-K6: binning for a batch of equally-sized views (BASELINE north_star: "warp-level
// scans and a custom onesweep radix sort").
//   K3 k_scan_tiles   single-pass decoupled look-back exclusive scan of tiles touched
//   K4 k_duplicate    one (key, val) per touched 16x16 tile, key = (gt << 31) | depth
//   K5 k_hist + k_onesweep  LSD radix sort, 8-bit digits: one global histogram pass
//                     for all digits, then one pass per digit that ranks a 4096-key tile
//                     with warp match_any multisplit (stable), resolves the tile's
//                     global digit offsets by decoupled look-back, stages the tile in
//                     shared memory in digit order and writes it out coalesced.
//   K6 k_ranges       [first, last+1) per global tile from the sorted keys
// Order = (view, tile, depth, index): the sort is stable and keys are emitted in
// ascending Gaussian index, so results equal the oracle's std::sort on (key, val).
#include "queen_internal.cuh"

namespace queen {

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
    *reinterpret_cast<volatile unsigned long long*>(p) = v;
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }
__device__ __forceinline__ void st_volatile_u32(uint32_t* p, uint32_t v) { *reinterpret_cast<volatile uint32_t*>(p) = v; }

constexpr unsigned long long SCAN_AGG = 1ull << 62, SCAN_INC = 2ull << 62, SCAN_MASK = (1ull << 62) - 1;
constexpr uint32_t LB_AGG = 1u << 30, LB_INC = 2u << 30, LB_MASK = (1u << 30) - 1;
constexpr long long SPIN_LIMIT = 1ll << 24;

// ---------------------------------------------------------------------------
// K3: offsets[j] = sum_{j' < j} tiles[j'] over the flattened [V][n_pad] array; K = total
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_tiles(const uint32_t* __restrict__ tiles,
                                                             uint32_t* __restrict__ offsets, int64_t count,
                                                             unsigned long long* lb, DevFlags* fl, uint32_t* K_out,
                                                             int64_t cap) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_wsum[SCAN_THREADS / 32];
    __shared__ unsigned long long s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(&fl->tickets[8], 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t ntiles = (count + SCAN_TILE - 1) / SCAN_TILE;
    const int64_t base = (int64_t)tile * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    uint32_t v[SCAN_ITEMS];
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS / 4; ++q) {
        uint4 x = make_uint4(0, 0, 0, 0);
        if (base + 4 * q < count) x = __ldg(reinterpret_cast<const uint4*>(tiles + base + 4 * q));
        v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
    }
    uint32_t tsum = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) tsum += v[j];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[w] = x;
    __syncthreads();
    uint32_t wpre = 0, agg = 0;
#pragma unroll
    for (int q = 0; q < SCAN_THREADS / 32; ++q) {
        const uint32_t s = s_wsum[q];
        if (q < w) wpre += s;
        agg += s;
    }
    if (threadIdx.x == 0) {
        unsigned long long prefix = 0;
        if (tile == 0) {
            st_volatile_u64(&lb[0], SCAN_INC | agg);
        } else {
            st_volatile_u64(&lb[tile], SCAN_AGG | agg);
            int64_t look = (int64_t)tile - 1;
            long long spins = 0;
            while (look >= 0) {
                const unsigned long long e = ld_volatile_u64(&lb[look]);
                if ((e >> 62) == 0) {
                    if (++spins > SPIN_LIMIT) { raise_flag(fl, FLAG_TIMEOUT); break; }
                    continue;
                }
                prefix += e & SCAN_MASK;
                if ((e >> 62) == 2) break;
                --look;
            }
            st_volatile_u64(&lb[tile], SCAN_INC | (prefix + agg));
        }
        s_prefix = prefix;
        if ((int64_t)tile == ntiles - 1) {
            const unsigned long long total = prefix + agg;
            if ((long long)total > cap) {
                raise_flag(fl, FLAG_CAPACITY);
                atomicMax(&fl->info, total);
            }
            K_out[0] = (uint32_t)(total > (unsigned long long)cap ? cap : total);
        }
    }
    __syncthreads();
    unsigned long long run = s_prefix + wpre + (x - tsum);
    uint32_t o[SCAN_ITEMS];
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        o[j] = (uint32_t)run;
        run += v[j];
    }
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS / 4; ++q)
        if (base + 4 * q < count)
            *reinterpret_cast<uint4*>(offsets + base + 4 * q) = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
}

// ---------------------------------------------------------------------------
// K4: duplicate.  For (v, i) ascending, ty ascending, tx ascending (R#15).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_duplicate(const uint32_t* __restrict__ tiles, const uint32_t* __restrict__ offsets,
                                                   const short4* __restrict__ rect, const uint32_t* __restrict__ depth,
                                                   int64_t count, int n_pad, int gx, int64_t T,
                                                   uint64_t* __restrict__ keys, uint32_t* __restrict__ vals, int64_t cap) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= count) return;
    const uint32_t nt = tiles[j];
    if (nt == 0) return;
    const int64_t v = j / n_pad;
    const uint32_t i = (uint32_t)(j - v * n_pad);
    const short4 r = rect[j];
    const uint64_t d = depth[j];
    int64_t w = offsets[j];
    const uint64_t gbase = (uint64_t)v * (uint64_t)T;
    for (int ty = r.y; ty <= r.w; ++ty) {
        const uint64_t rowg = gbase + (uint64_t)ty * gx;
        for (int tx = r.x; tx <= r.z; ++tx) {
            if (w < cap) {
                keys[w] = ((rowg + (uint64_t)tx) << 31) | d;
                vals[w] = i;
            }
            ++w;
        }
    }
}

// ---------------------------------------------------------------------------
// K5a: histograms of every 8-bit digit of every key (one read of the keys)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_hist(const uint64_t* __restrict__ keys, const uint32_t* K, int64_t cap,
                                              int passes, uint32_t* hist) {
    __shared__ uint32_t sh[MAX_PASSES * 256];
    for (int q = threadIdx.x; q < MAX_PASSES * 256; q += blockDim.x) sh[q] = 0;
    __syncthreads();
    const int64_t Kn = min((int64_t)*K, cap);
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < Kn; j += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[j];
        for (int p = 0; p < passes; ++p) atomicAdd(&sh[p * 256 + ((k >> (8 * p)) & 255u)], 1u);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < passes * 256; q += blockDim.x)
        if (sh[q]) atomicAdd(&hist[q], sh[q]);
}

// K5b: exclusive scan of each pass's 256 digit counts (one block, one warp per pass)
__global__ void k_hist_scan(const uint32_t* hist, uint32_t* excl, int passes) {
    const int p = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (p >= passes) return;
    uint32_t v[8], s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) { v[q] = hist[p * 256 + lane * 8 + q]; s += v[q]; }
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    uint32_t run = x - s;
#pragma unroll
    for (int q = 0; q < 8; ++q) { excl[p * 256 + lane * 8 + q] = run; run += v[q]; }
}

// ---------------------------------------------------------------------------
// K5c: one onesweep pass (persistent CTAs, dynamic tile tickets => forward progress)
// ---------------------------------------------------------------------------
constexpr int SORT_WARPS = SORT_THREADS / 32;
constexpr size_t ONESWEEP_SMEM = (size_t)SORT_TILE * 8 + (size_t)SORT_TILE * 4 + (size_t)SORT_WARPS * 256 * 4 + 256 * 4 * 2;

__global__ void __launch_bounds__(SORT_THREADS) k_onesweep(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                           uint64_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                           const uint32_t* K, int64_t cap, int shift,
                                                           const uint32_t* __restrict__ hist_excl, uint32_t* lb,
                                                           uint32_t* ticket, DevFlags* fl) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* sk = reinterpret_cast<uint64_t*>(smem);
    uint32_t* sv = reinterpret_cast<uint32_t*>(sk + SORT_TILE);
    uint32_t* whist = sv + SORT_TILE;          // [warps][256]
    uint32_t* dstart = whist + SORT_WARPS * 256;  // [256] tile-local exclusive digit start
    uint32_t* dbase = dstart + 256;            // [256] global base minus local start
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_wtot[SORT_WARPS];
    const uint32_t Kn = (uint32_t)min((int64_t)*K, cap);
    const uint32_t ntiles = (Kn + SORT_TILE - 1) / SORT_TILE;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
#pragma unroll
        for (int q = 0; q < SORT_WARPS; ++q) whist[q * 256 + threadIdx.x] = 0u;
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= ntiles) break;
        const uint32_t base = tile * SORT_TILE;
        uint64_t k[SORT_ITEMS];
        uint32_t val[SORT_ITEMS], rank[SORT_ITEMS], dig[SORT_ITEMS];
#pragma unroll
        for (int j = 0; j < SORT_ITEMS; ++j) {
            const uint32_t idx = base + w * (32 * SORT_ITEMS) + j * 32 + lane;
            const bool ok = idx < Kn;
            k[j] = ok ? kin[idx] : 0ull;
            val[j] = ok ? vin[idx] : 0u;
            dig[j] = ok ? (uint32_t)((k[j] >> shift) & 255u) : 256u;
        }
        // warp multisplit, in key order => stable
#pragma unroll
        for (int j = 0; j < SORT_ITEMS; ++j) {
            const uint32_t d = dig[j];
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            const uint32_t below = peers & lt_mask;
            uint32_t prior = 0;
            if (d < 256u) prior = whist[w * 256 + d];
            __syncwarp();
            if (below == 0 && d < 256u) whist[w * 256 + d] = prior + __popc(peers);
            __syncwarp();
            rank[j] = prior + __popc(below);
        }
        __syncthreads();
        // thread t <-> digit t: exclusive over warps, tile count
        const uint32_t d = threadIdx.x;
        uint32_t cnt = 0;
#pragma unroll
        for (int q = 0; q < SORT_WARPS; ++q) {
            const uint32_t c = whist[q * 256 + d];
            whist[q * 256 + d] = cnt;
            cnt += c;
        }
        uint32_t* lbt = lb + (size_t)tile * 256;
        st_volatile_u32(&lbt[d], (tile == 0 ? LB_INC : LB_AGG) | cnt);
        // tile-local exclusive scan over digits
        uint32_t x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_wtot[w] = x;
        // decoupled look-back for this digit
        uint32_t prefix = 0;
        if (tile > 0) {
            int64_t look = (int64_t)tile - 1;
            long long spins = 0;
            while (look >= 0) {
                const uint32_t e = ld_volatile_u32(&lb[(size_t)look * 256 + d]);
                const uint32_t f = e >> 30;
                if (f == 0) {
                    if (++spins > SPIN_LIMIT) { raise_flag(fl, FLAG_TIMEOUT); break; }
                    continue;
                }
                prefix += e & LB_MASK;
                if (f == 2) break;
                --look;
            }
            st_volatile_u32(&lbt[d], LB_INC | (prefix + cnt));
        }
        __syncthreads();
        uint32_t wpre = 0;
#pragma unroll
        for (int q = 0; q < SORT_WARPS; ++q) wpre += (q < w) ? s_wtot[q] : 0u;
        const uint32_t excl = wpre + x - cnt;
        dstart[d] = excl;
        dbase[d] = hist_excl[d] + prefix - excl;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < SORT_ITEMS; ++j) {
            const uint32_t dj = dig[j];
            if (dj < 256u) {
                const uint32_t pos = dstart[dj] + whist[w * 256 + dj] + rank[j];
                sk[pos] = k[j];
                sv[pos] = val[j];
            }
        }
        __syncthreads();
        const uint32_t nvalid = min((uint32_t)SORT_TILE, Kn - base);
        for (uint32_t p = threadIdx.x; p < nvalid; p += SORT_THREADS) {
            const uint64_t key = sk[p];
            const uint32_t dest = dbase[(uint32_t)((key >> shift) & 255u)] + p;
            kout[dest] = key;
            vout[dest] = sv[p];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// K6: ranges[gt] = [first, last+1)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_ranges(const uint64_t* __restrict__ keys, const uint32_t* K, int64_t cap,
                                                uint2* __restrict__ ranges) {
    const uint32_t Kn = (uint32_t)min((int64_t)*K, cap);
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < Kn; j += gridDim.x * blockDim.x) {
        const uint64_t g = keys[j] >> 31;
        if (j == 0 || (keys[j - 1] >> 31) != g) ranges[g].x = j;
        if (j == Kn - 1 || (keys[j + 1] >> 31) != g) ranges[g].y = j + 1;
    }
}

static int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

static int onesweep_blocks_per_sm() {
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_onesweep, SORT_THREADS, ONESWEEP_SMEM);
        if (occ <= 0) occ = 1;
    }
    return occ;
}

cudaError_t init_binning_attributes() {
    return cudaFuncSetAttribute(k_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ONESWEEP_SMEM);
}

int key_passes(int64_t gtiles) {
    int gbits = 1;
    while ((1ll << gbits) < gtiles) ++gbits;
    return (31 + gbits + 7) / 8;
}

cudaError_t launch_bin_sort(const queen_proj& proj, int n_views, int W, int H, queen_bins& bins, void* scratch,
                            const WsLayout& L, DevFlags* fl, cudaStream_t s, Prof* prof) {
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int64_t T = (int64_t)gx * gy;
    const int64_t count = (int64_t)n_views * proj.n_pad;
    const int64_t cap = bins.keys_cap;
    const int passes = key_passes(T * n_views);
    unsigned char* ws = static_cast<unsigned char*>(scratch);
    uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist);
    uint32_t* hist_excl = hist + MAX_PASSES * 256;
    unsigned long long* scan_lb = reinterpret_cast<unsigned long long*>(ws + L.scan_lb);
    uint32_t* sort_lb = reinterpret_cast<uint32_t*>(ws + L.sort_lb);
    const int64_t sort_tiles = (cap + SORT_TILE - 1) / SORT_TILE;
    const int64_t scan_tiles = (count + SCAN_TILE - 1) / SCAN_TILE;
    cudaError_t e;
    // reset tickets, histograms, look-back state, ranges
    prof->begin(ST_SCAN, s);
    if ((e = cudaMemsetAsync(fl->tickets, 0, sizeof(fl->tickets), s))) return e;
    if ((e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * MAX_PASSES * 256, s))) return e;
    if ((e = cudaMemsetAsync(scan_lb, 0, sizeof(unsigned long long) * (scan_tiles + 1), s))) return e;
    if ((e = cudaMemsetAsync(sort_lb, 0, sizeof(uint32_t) * 256 * (size_t)(sort_tiles + 1) * passes, s))) return e;
    if ((e = cudaMemsetAsync(bins.ranges, 0, sizeof(uint32_t) * 2 * (size_t)T * n_views, s))) return e;
    if ((e = cudaMemsetAsync(bins.K, 0, sizeof(uint32_t), s))) return e;
    if (scan_tiles > 0)
        k_scan_tiles<<<(unsigned)scan_tiles, SCAN_THREADS, 0, s>>>(proj.tiles, bins.offsets, count, scan_lb, fl, bins.K, cap);
    prof->end(s);
    prof->begin(ST_DUPLICATE, s);
    {
        const int64_t blocks = (count + 255) / 256;
        if (blocks > 0)
            k_duplicate<<<(unsigned)blocks, 256, 0, s>>>(proj.tiles, bins.offsets, reinterpret_cast<const short4*>(proj.rect),
                                                         proj.depth, count, proj.n_pad, gx, T, bins.keys, bins.vals, cap);
    }
    prof->end(s);
    const int sms = num_sms();
    prof->begin(ST_HIST, s);
    k_hist<<<sms * 4, 256, 0, s>>>(bins.keys, bins.K, cap, passes, hist);
    k_hist_scan<<<1, 32 * MAX_PASSES, 0, s>>>(hist, hist_excl, passes);
    prof->end(s, 2);
    uint64_t* ka = bins.keys;
    uint64_t* kb = bins.keys_alt;
    uint32_t* va = bins.vals;
    uint32_t* vb = bins.vals_alt;
    const int grid = sms * onesweep_blocks_per_sm();
    prof->begin(ST_SORT, s);
    for (int p = 0; p < passes; ++p) {
        k_onesweep<<<grid, SORT_THREADS, ONESWEEP_SMEM, s>>>(ka, va, kb, vb, bins.K, cap, 8 * p, hist_excl + p * 256,
                                                             sort_lb + (size_t)p * 256 * (sort_tiles + 1), &fl->tickets[p],
                                                             fl);
        uint64_t* tk = ka; ka = kb; kb = tk;
        uint32_t* tv = va; va = vb; vb = tv;
    }
    prof->end(s, passes);
    bins.sorted_in_alt = (passes & 1) ? 1 : 0;
    prof->begin(ST_RANGES, s);
    k_ranges<<<sms * 8, 256, 0, s>>>(ka, bins.K, cap, reinterpret_cast<uint2*>(bins.ranges));
    prof->end(s);
    return cudaGetLastError();
}

}  // namespace queen
