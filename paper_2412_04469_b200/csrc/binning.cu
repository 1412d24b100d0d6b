// K3-K6: binning for a batch of equally-sized views (BASELINE north_star: "duplication
// of Gaussians into 16x16 tiles, a radix sort on (tile, depth) keys, per-tile range
// extraction"; "warp-level scans and a custom onesweep radix sort").
//
// The sort is an LSD radix sort on the composite key (gt, depth) with gt = view*T +
// tile: LSD order processes the depth digits first and the tile digits last.  Every
// duplicate of a Gaussian carries the same depth, so the depth digits are sorted
// BEFORE duplication, on the M visible (view, Gaussian) pairs (M << K), and only the
// tile digits are sorted on the K duplicated entries, with 4-byte keys:
//   K3a k_vis_compact   decoupled look-back scan: visible pairs (tiles > 0) in (view,
//                       index) order -> (depth bits, flat index)            [M]
//   K5a k_onesweep32<8> x4  stable sort of the pairs by depth (31 bits)
//   K3b/K4 k_scan_dup   decoupled look-back scan of tiles touched in depth order fused
//                       with duplication: entry = (gt, Gaussian index), emitted for
//                       each pair ty-major, tx-minor; fused tile-digit histograms
//   K5b k_onesweep32<8|9> x2..3  stable sort of the entries by gt
//   K6  k_ranges        [first, last+1) of each gt
// Stability makes the final order (gt, depth, view, index) -> (gt, depth, index):
// identical to sorting the 96-bit (gt << 31 | depth, index) tuples (oracle: std::sort).
//
// onesweep pass: persistent CTAs take 4096-key tiles by atomic ticket (forward
// progress for the look-back), rank keys with warp match_any multisplit in key order
// (stable), publish per-digit tile counts, resolve global digit offsets by decoupled
// look-back, stage the tile in shared memory in digit order and write it out coalesced.
#include "queen_internal.cuh"

namespace queen {

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
    *reinterpret_cast<volatile unsigned long long*>(p) = v;
}
// look-back words: one 32-bit (flag | count) word each, so GPU-scope relaxed accesses suffice
// (volatile would compile to system-scope .STRONG.SYS accesses)
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr unsigned long long SCAN_AGG = 1ull << 62, SCAN_INC = 2ull << 62, SCAN_MASK = (1ull << 62) - 1;
constexpr uint32_t LB_AGG = 1u << 30, LB_INC = 2u << 30, LB_MASK = (1u << 30) - 1;
constexpr long long SPIN_LIMIT = 1ll << 24;
constexpr int SORT_WARPS = SORT_THREADS / 32;

enum : int { TK_DEPTH = 0, TK_TILE = 4, TK_VIS = 8, TK_DUP = 9 };

// Block-wide exclusive scan of one u32 per thread (256 threads); returns the exclusive
// prefix and the block total.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* s_w, uint32_t& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    uint32_t pre = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < SORT_WARPS; ++q) {
        const uint32_t s = s_w[q];
        pre += (q < w) ? s : 0u;
        tot += s;
    }
    total = tot;
    return pre + inc - x;
}

// Decoupled look-back over 64-bit aggregates (called by one thread).
__device__ unsigned long long lookback64(unsigned long long* lb, uint32_t tile, unsigned long long agg, DevFlags* fl) {
    unsigned long long prefix = 0;
    if (tile == 0) {
        st_volatile_u64(&lb[0], SCAN_INC | agg);
        return 0;
    }
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
    return prefix;
}

// ---------------------------------------------------------------------------
// K3a: visible (view, Gaussian) pairs, in flat-index order -> (depth bits, j)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(SORT_THREADS) k_vis_compact(const uint32_t* __restrict__ tiles,
                                                              const uint32_t* __restrict__ depth, int64_t count,
                                                              uint32_t* __restrict__ dkeys, uint32_t* __restrict__ dvals,
                                                              unsigned long long* lb, DevFlags* fl, uint32_t* M_out) {
    __shared__ uint32_t s_tile, s_w[SORT_WARPS];
    __shared__ unsigned long long s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(&fl->tickets[TK_VIS], 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t ntiles = (count + SORT_TILE - 1) / SORT_TILE;
    const int64_t base = (int64_t)tile * SORT_TILE + (int64_t)threadIdx.x * SORT_ITEMS;
    uint32_t vis = 0;  // bit e set <=> element base+e is visible
#pragma unroll
    for (int q = 0; q < SORT_ITEMS / 4; ++q) {
        if (base + 4 * q < count) {
            const uint4 t4 = __ldg(reinterpret_cast<const uint4*>(tiles + base + 4 * q));
            vis |= (t4.x ? 1u : 0u) << (4 * q) | (t4.y ? 2u : 0u) << (4 * q) | (t4.z ? 4u : 0u) << (4 * q) |
                   (t4.w ? 8u : 0u) << (4 * q);
        }
    }
    uint32_t total;
    const uint32_t excl = block_excl_scan(__popc(vis), s_w, total);
    if (threadIdx.x == 0) {
        s_prefix = lookback64(lb, tile, total, fl);
        if ((int64_t)tile == ntiles - 1) *M_out = (uint32_t)(s_prefix + total);
    }
    __syncthreads();
    uint64_t pos = s_prefix + excl;
    while (vis) {
        const int e = __ffs(vis) - 1;
        vis &= vis - 1;
        const int64_t j = base + e;
        dkeys[pos] = __ldg(depth + j);
        dvals[pos] = (uint32_t)j;
        ++pos;
    }
}

// ---------------------------------------------------------------------------
// K5: histograms of the depth digits (4 x 8 bits) of the M visible pairs
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_hist_depth(const uint32_t* __restrict__ keys, const uint32_t* count_ptr,
                                                    uint32_t* hist) {
    __shared__ uint32_t sh[DEPTH_PASSES * 256];
    for (int q = threadIdx.x; q < DEPTH_PASSES * 256; q += blockDim.x) sh[q] = 0;
    __syncthreads();
    const uint32_t n = *count_ptr;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint32_t k = keys[j];
#pragma unroll
        for (int p = 0; p < DEPTH_PASSES; ++p) atomicAdd(&sh[p * 256 + ((k >> (8 * p)) & 255u)], 1u);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < DEPTH_PASSES * 256; q += blockDim.x)
        if (sh[q]) atomicAdd(&hist[(q >> 8) * MAX_BINS + (q & 255)], sh[q]);  // per-pass stride MAX_BINS
}

// exclusive scan of each pass's digit counts (one warp per pass)
__global__ void k_hist_scan(const uint32_t* hist, uint32_t* excl, int passes, int bins) {
    const int p = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (p >= passes) return;
    const int per = bins / 32;
    uint32_t s = 0;
    for (int q = 0; q < per; ++q) s += hist[p * MAX_BINS + lane * per + q];
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    uint32_t run = x - s;
    for (int q = 0; q < per; ++q) {
        const uint32_t c = hist[p * MAX_BINS + lane * per + q];
        excl[p * MAX_BINS + lane * per + q] = run;
        run += c;
    }
}

// ---------------------------------------------------------------------------
// K5: one onesweep pass over (u32 key, u32 value) pairs
// ---------------------------------------------------------------------------
// Block of NT threads: exclusive scan of one u32 per thread; returns prefix, sets total.
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan_t(uint32_t x, uint32_t* s_w, uint32_t& total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    uint32_t pre = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
        const uint32_t s = s_w[q];
        pre += (q < w) ? s : 0u;
        tot += s;
    }
    total = tot;
    return pre + inc - x;
}

// onesweep configuration: NT threads x IT keys per thread = one 4096-key tile
template <int BITS>
struct Onesweep {
    static constexpr int NT = OS_THREADS, IT = OS_ITEMS, NW = NT / 32;
    static constexpr int TILE = NT * IT;
    static constexpr int BINS = 1 << BITS;
    static constexpr int DPT = BINS >= NT ? BINS / NT : 1;  // digits per thread (threads >= BINS idle)
    static constexpr size_t SMEM = (size_t)TILE * 4 * 2 + (size_t)NW * BINS * 4 + (size_t)BINS * 4 * 2;
};

template <int BITS>
__global__ void __launch_bounds__(Onesweep<BITS>::NT) k_onesweep32(const uint32_t* __restrict__ kin,
                                                                   const uint32_t* __restrict__ vin,
                                                                   uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                                   const uint32_t* count_ptr, uint32_t cap, int shift,
                                                                   const uint32_t* __restrict__ hist_excl, uint32_t* lb,
                                                                   uint32_t* ticket, DevFlags* fl) {
    using OS = Onesweep<BITS>;
    constexpr int NT = OS::NT, IT = OS::IT, NW = OS::NW, TILE = OS::TILE, BINS = OS::BINS, DPT = OS::DPT;
    constexpr uint32_t DMASK = BINS - 1;
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* sk = reinterpret_cast<uint32_t*>(smem);
    uint32_t* sv = sk + TILE;
    uint32_t* whist = sv + TILE;             // [warps][BINS]: counts, then exclusive-over-warps
    uint32_t* dstart = whist + NW * BINS;    // [BINS] tile-local exclusive digit start
    uint32_t* dbase = dstart + BINS;         // [BINS] global destination minus local start
    __shared__ uint32_t s_tile, s_w[NW];
    const uint32_t Kn = min(*count_ptr, cap);
    const uint32_t ntiles = (Kn + TILE - 1) / TILE;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const bool owns_digits = threadIdx.x * DPT < BINS;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
        for (int q = threadIdx.x; q < NW * BINS; q += NT) whist[q] = 0u;
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= ntiles) break;
        const uint32_t base = tile * TILE;
        uint32_t k[IT], val[IT], rk[IT];
#pragma unroll
        for (int j = 0; j < IT; ++j) {
            const uint32_t idx = base + w * (32 * IT) + j * 32 + lane;
            const bool ok = idx < Kn;
            k[j] = ok ? kin[idx] : 0u;
            val[j] = ok ? vin[idx] : 0u;
        }
        // warp multisplit in key order (stable): rank among this warp's earlier equal digits.
        // All MATCHes first (independent), then the short shared-memory chain.
        uint32_t peers[IT];
#pragma unroll
        for (int j = 0; j < IT; ++j) {
            const uint32_t idx = base + w * (32 * IT) + j * 32 + lane;
            rk[j] = idx < Kn ? ((k[j] >> shift) & DMASK) : (uint32_t)BINS;
            peers[j] = __match_any_sync(0xffffffffu, rk[j]);
        }
#pragma unroll
        for (int j = 0; j < IT; ++j) {
            const uint32_t d = rk[j];
            const uint32_t below = peers[j] & lt_mask;
            uint32_t prior = 0;
            if (d < (uint32_t)BINS) prior = whist[w * BINS + d];
            __syncwarp();
            if (below == 0 && d < (uint32_t)BINS) whist[w * BINS + d] = prior + __popc(peers[j]);
            __syncwarp();
            rk[j] = (prior + __popc(below)) | (d << 16);
        }
        __syncthreads();
        uint32_t cnt[DPT];
        uint32_t tsum = 0;
#pragma unroll
        for (int e = 0; e < DPT; ++e) {
            cnt[e] = 0;
            if (owns_digits) {
                const int d = threadIdx.x * DPT + e;
                uint32_t run = 0;
#pragma unroll
                for (int q = 0; q < NW; ++q) {
                    const uint32_t c = whist[q * BINS + d];
                    whist[q * BINS + d] = run;
                    run += c;
                }
                cnt[e] = run;
                tsum += run;
                st_volatile_u32(&lb[(size_t)tile * BINS + d], (tile == 0 ? LB_INC : LB_AGG) | run);
            }
        }
        uint32_t total;
        uint32_t excl = block_excl_scan_t<NT>(tsum, s_w, total);
        uint32_t lstart[DPT];
        if (owns_digits) {
#pragma unroll
            for (int e = 0; e < DPT; ++e) {
                lstart[e] = excl;
                dstart[threadIdx.x * DPT + e] = excl;
                excl += cnt[e];
            }
        }
        __syncthreads();
        // digit owners run the decoupled look-back first (the inclusive chain is the critical
        // path); meanwhile the other threads already scatter their keys into shared memory
        if (owns_digits) {
#pragma unroll
            for (int e = 0; e < DPT; ++e) {
                const int d = threadIdx.x * DPT + e;
                uint32_t prefix = 0;
                if (tile > 0) {
                    int64_t look = (int64_t)tile - 1;
                    long long spins = 0;
                    while (look >= 0) {
                        const uint32_t x = ld_volatile_u32(&lb[(size_t)look * BINS + d]);
                        const uint32_t f = x >> 30;
                        if (f == 0) {
                            if (++spins > SPIN_LIMIT) { raise_flag(fl, FLAG_TIMEOUT); break; }
                            continue;
                        }
                        prefix += x & LB_MASK;
                        if (f == 2) break;
                        --look;
                    }
                    st_volatile_u32(&lb[(size_t)tile * BINS + d], LB_INC | (prefix + cnt[e]));
                }
                dbase[d] = hist_excl[d] + prefix - lstart[e];
            }
        }
#pragma unroll
        for (int j = 0; j < IT; ++j) {
            const uint32_t d = rk[j] >> 16;
            if (d < (uint32_t)BINS) {
                const uint32_t pos = dstart[d] + whist[w * BINS + d] + (rk[j] & 0xffffu);
                sk[pos] = k[j];
                sv[pos] = val[j];
            }
        }
        __syncthreads();
        const uint32_t nvalid = min((uint32_t)TILE, Kn - base);
        for (uint32_t p = threadIdx.x; p < nvalid; p += NT) {
            const uint32_t key = sk[p];
            const uint32_t dest = dbase[(key >> shift) & DMASK] + p;
            kout[dest] = key;
            vout[dest] = sv[p];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// K3b + K4: offsets of the depth-sorted pairs (decoupled look-back) + duplication.
// Entry = (gt, Gaussian index), emitted for each pair ty-major, tx-minor.
// Phase 1 stages the block's 4096 pairs in shared memory (block-local offset, gt of the
// rect's first tile, Gaussian index, rect width) and adds the pair's tile rect to the
// per-view 2D difference array of tile counts (4 corner increments; k_tile_counts turns
// it into per-tile entry counts, i.e. the final ranges and the digit histograms).
// Phase 2: each warp emits a contiguous run of the block's entries, 32 at a time; every
// pair has >= 1 entry, so the pairs starting inside a 32-entry chunk are the next <= 31
// pairs: one shared load + redux.or + popc locates each lane's pair.  Stores coalesce.
// ---------------------------------------------------------------------------
constexpr size_t DUP_SMEM = (size_t)SORT_TILE * (4 + 4 + 4 + 2) + 16;

__global__ void __launch_bounds__(SORT_THREADS) k_scan_dup(const uint32_t* __restrict__ dvals, const uint32_t* count_ptr,
                                                           const short4* __restrict__ rect, int n_pad, int gx, int gy,
                                                           uint32_t T, uint32_t* __restrict__ keys,
                                                           uint32_t* __restrict__ vals, uint32_t cap,
                                                           unsigned long long* lb, DevFlags* fl, uint32_t* K_out,
                                                           int* __restrict__ diff) {
    extern __shared__ __align__(16) unsigned char dsm[];
    uint32_t* s_off = reinterpret_cast<uint32_t*>(dsm);       // [SORT_TILE + 1]
    uint32_t* s_base = s_off + SORT_TILE + 4;                // [SORT_TILE]
    uint32_t* s_i = s_base + SORT_TILE;                      // [SORT_TILE]
    uint16_t* s_wx = reinterpret_cast<uint16_t*>(s_i + SORT_TILE);
    __shared__ uint32_t s_tile, s_w[SORT_WARPS];
    __shared__ unsigned long long s_prefix;
    const uint32_t M = *count_ptr;
    const uint32_t ntiles = (M + SORT_TILE - 1) / SORT_TILE;
    if (threadIdx.x == 0) s_tile = atomicAdd(&fl->tickets[TK_DUP], 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) return;
    const uint32_t base = tile * SORT_TILE + threadIdx.x * SORT_ITEMS;
    const int dw = gx + 1, dplane = (gx + 1) * (gy + 1);
    uint32_t nt[SORT_ITEMS];
    uint32_t tsum = 0;
    // batch the dependent gathers: all 16 indices (4 x uint4), then all 16 rects, then use them
    uint32_t jj[SORT_ITEMS];
#pragma unroll
    for (int q4 = 0; q4 < SORT_ITEMS / 4; ++q4) {
        uint4 x = make_uint4(0, 0, 0, 0);
        if (base + 4 * q4 + 3 < M) x = __ldg(reinterpret_cast<const uint4*>(dvals + base + 4 * q4));
        else {
            if (base + 4 * q4 + 0 < M) x.x = __ldg(dvals + base + 4 * q4 + 0);
            if (base + 4 * q4 + 1 < M) x.y = __ldg(dvals + base + 4 * q4 + 1);
            if (base + 4 * q4 + 2 < M) x.z = __ldg(dvals + base + 4 * q4 + 2);
        }
        jj[4 * q4] = x.x; jj[4 * q4 + 1] = x.y; jj[4 * q4 + 2] = x.z; jj[4 * q4 + 3] = x.w;
    }
    short4 rr[SORT_ITEMS];
#pragma unroll
    for (int e = 0; e < SORT_ITEMS; ++e) rr[e] = base + e < M ? __ldg(rect + jj[e]) : make_short4(0, 0, 0, 0);
#pragma unroll
    for (int e = 0; e < SORT_ITEMS; ++e) {
        const uint32_t m = base + e;
        const int q = threadIdx.x * SORT_ITEMS + e;
        nt[e] = 0;
        if (m < M) {
            const uint32_t j = jj[e];
            const short4 r = rr[e];
            const uint32_t v = j / (uint32_t)n_pad;
            const uint32_t wx = (uint32_t)(r.z - r.x + 1), wy = (uint32_t)(r.w - r.y + 1);
            nt[e] = wx * wy;
            s_base[q] = v * T + (uint32_t)r.y * (uint32_t)gx + (uint32_t)r.x;
            s_i[q] = j - v * (uint32_t)n_pad;
            s_wx[q] = (uint16_t)wx;
            int* d = diff + (int64_t)v * dplane;
            atomicAdd(d + r.y * dw + r.x, 1);
            atomicAdd(d + r.y * dw + r.z + 1, -1);
            atomicAdd(d + (r.w + 1) * dw + r.x, -1);
            atomicAdd(d + (r.w + 1) * dw + r.z + 1, 1);
        }
        tsum += nt[e];
    }
    uint32_t total;
    const uint32_t excl = block_excl_scan(tsum, s_w, total);
    if (threadIdx.x == 0) {
        s_prefix = lookback64(lb, tile, total, fl);
        if (tile == ntiles - 1) {
            const unsigned long long K = s_prefix + total;
            if (K > cap) {
                raise_flag(fl, FLAG_CAPACITY);
                atomicMax(&fl->info, K);
            }
            // overflow: no entry list is produced (the tile sort sees 0 entries and every range is
            // [0,0)); QUEEN_ERR_CAPACITY carries the K needed.  K_out[2] = overflow flag.
            K_out[0] = K > cap ? 0u : (uint32_t)K;
            K_out[2] = K > cap ? 1u : 0u;
        }
        s_off[SORT_TILE] = total;
    }
    {
        uint32_t run = excl;
#pragma unroll
        for (int e = 0; e < SORT_ITEMS; ++e) {
            s_off[threadIdx.x * SORT_ITEMS + e] = run;
            run += nt[e];
        }
    }
    __syncthreads();
    const unsigned long long gbase = s_prefix;
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t nchunks = (total + 31) / 32;
    const uint32_t c0 = (uint32_t)(((uint64_t)nchunks * w) / SORT_WARPS);
    const uint32_t c1 = (uint32_t)(((uint64_t)nchunks * (w + 1)) / SORT_WARPS);
    if (c0 >= c1) return;
    // pair owning entry 32*c0 (binary search once; all lanes agree)
    int lo = 0;
    {
        const uint32_t p = 32 * c0;
        int hi = SORT_TILE;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_off[mid] <= p) lo = mid; else hi = mid;
        }
    }
    const uint32_t le_mask = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);
    for (uint32_t c = c0; c < c1; ++c) {
        const uint32_t p0 = 32 * c;
        const int cand = lo + (int)lane;
        const uint32_t o = cand <= SORT_TILE ? s_off[cand] : 0xffffffffu;
        const uint32_t sdel = o - p0;  // start of pair lo+lane relative to p0 (lanes >= 1 start after p0)
        const uint32_t bit = (lane > 0 && o > p0 && sdel < 32u) ? (1u << sdel) : 0u;
        const uint32_t starts = __reduce_or_sync(0xffffffffu, bit);
        const int e = lo + __popc(starts & le_mask);
        const uint32_t p = p0 + lane;
        if (p < total) {
            const uint32_t cc = p - s_off[e];
            const uint32_t wx = s_wx[e];
            const uint32_t row = cc / wx;
            const uint64_t dst = gbase + p;
            if (dst < cap) {
                keys[dst] = s_base[e] + row * (uint32_t)gx + (cc - row * wx);
                vals[dst] = s_i[e];
            }
        }
        const int e31 = __shfl_sync(0xffffffffu, e, 31);
        lo = e31 + ((e31 + 1 <= SORT_TILE && s_off[e31 + 1] == p0 + 32) ? 1 : 0);
    }
}

// Per-view 2D prefix sums of the tile-count difference arrays -> entries per global tile,
// their view-local exclusive starts, the tile-digit histograms of the coming tile sort,
// and per-view totals.  One block per view.
__global__ void __launch_bounds__(1024) k_tile_counts(const int* __restrict__ diff, int gx, int gy, uint32_t* counts,
                                                      uint32_t* lstart, uint32_t* view_tot, uint32_t* hist, int tpasses,
                                                      int tbits) {
    extern __shared__ int cs[];  // [(gy+1)][(gx+1)]
    __shared__ uint32_t sh[MAX_TILE_PASSES * MAX_BINS];
    __shared__ uint32_t s_w[32];
    const int v = blockIdx.x;
    const int dw = gx + 1, dplane = (gx + 1) * (gy + 1);
    const int T = gx * gy;
    for (int q = threadIdx.x; q < dplane; q += blockDim.x) cs[q] = diff[(int64_t)v * dplane + q];
    for (int q = threadIdx.x; q < tpasses * MAX_BINS; q += blockDim.x) sh[q] = 0;
    __syncthreads();
    for (int r = threadIdx.x; r < gy; r += blockDim.x) {  // prefix along x
        int run = 0;
        for (int x = 0; x < gx; ++x) { run += cs[r * dw + x]; cs[r * dw + x] = run; }
    }
    __syncthreads();
    for (int x = threadIdx.x; x < gx; x += blockDim.x) {  // prefix along y
        int run = 0;
        for (int r = 0; r < gy; ++r) { run += cs[r * dw + x]; cs[r * dw + x] = run; }
    }
    __syncthreads();
    // each thread: a contiguous chunk of tiles (row-major t) -> local exclusive starts
    const int per = (T + blockDim.x - 1) / blockDim.x;
    const int t0 = threadIdx.x * per, t1 = min(T, t0 + per);
    uint32_t csum = 0;
    for (int t = t0; t < t1; ++t) csum += (uint32_t)cs[(t / gx) * dw + (t % gx)];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = csum;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    uint32_t pre = 0, tot = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
        pre += q < w ? s_w[q] : 0u;
        tot += s_w[q];
    }
    uint32_t run = pre + inc - csum;
    const uint32_t dmask = (1u << tbits) - 1u;
    for (int t = t0; t < t1; ++t) {
        const uint32_t c = (uint32_t)cs[(t / gx) * dw + (t % gx)];
        const uint32_t g = (uint32_t)v * (uint32_t)T + (uint32_t)t;
        counts[g] = c;
        lstart[g] = run;
        run += c;
        if (c)
            for (int p = 0; p < tpasses; ++p) atomicAdd(&sh[p * MAX_BINS + ((g >> (p * tbits)) & dmask)], c);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < tpasses * MAX_BINS; q += blockDim.x)
        if (sh[q]) atomicAdd(&hist[q], sh[q]);
    if (threadIdx.x == 0) view_tot[v] = tot;
}

// ranges[gt] = view base + local start (view bases = exclusive scan of the <= 64 view
// totals); [0,0) for empty tiles and everywhere on capacity overflow (already flagged)
__global__ void __launch_bounds__(256) k_ranges_finalize(const uint32_t* __restrict__ counts,
                                                         const uint32_t* __restrict__ lstart,
                                                         const uint32_t* __restrict__ view_tot, int n_views, uint32_t T,
                                                         uint32_t cap, const uint32_t* Kd, uint2* __restrict__ ranges) {
    __shared__ unsigned long long s_base[QUEEN_MAX_VIEWS + 1];
    if (threadIdx.x == 0) {
        unsigned long long r = 0;
        for (int q = 0; q < n_views; ++q) { s_base[q] = r; r += view_tot[q]; }
    }
    __syncthreads();
    const bool overflow = Kd[2] != 0u;
    const uint64_t G = (uint64_t)n_views * T;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < G; g += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = counts[g];
        const unsigned long long st = s_base[g / T] + lstart[g], en = st + c;
        ranges[g] = (c && !overflow) ? make_uint2((uint32_t)(st < cap ? st : cap), (uint32_t)(en < cap ? en : cap))
                                     : make_uint2(0u, 0u);
    }
}

// launchers shared with the BUCKET binning mode (bucket.cu)
void launch_tile_counts(const int* diff, int gx, int gy, int n_views, uint32_t* counts, uint32_t* lstart,
                        uint32_t* view_tot, cudaStream_t s) {
    k_tile_counts<<<n_views, 1024, sizeof(int) * (size_t)(gx + 1) * (gy + 1), s>>>(diff, gx, gy, counts, lstart, view_tot,
                                                                                 nullptr, 0, 8);
}
void launch_ranges_finalize(const uint32_t* counts, const uint32_t* lstart, const uint32_t* view_tot, int n_views,
                            uint32_t T, uint32_t cap, const uint32_t* Kd, uint2* ranges, int grid, cudaStream_t s) {
    k_ranges_finalize<<<grid, 256, 0, s>>>(counts, lstart, view_tot, n_views, T, cap, Kd, ranges);
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

template <int BITS>
static int onesweep_grid() {
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_onesweep32<BITS>, Onesweep<BITS>::NT, Onesweep<BITS>::SMEM);
        if (occ <= 0) occ = 1;
    }
    return occ * num_sms();
}

cudaError_t init_binning_attributes() {
    cudaError_t e = cudaFuncSetAttribute(k_onesweep32<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Onesweep<8>::SMEM);
    if (e) return e;
    if ((e = cudaFuncSetAttribute(k_onesweep32<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Onesweep<9>::SMEM)))
        return e;
    if ((e = cudaFuncSetAttribute(k_scan_dup, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DUP_SMEM))) return e;
    return cudaFuncSetAttribute(k_tile_counts, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

template <int BITS>
static void onesweep(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout, const uint32_t* count,
                     uint32_t cap, int shift, const uint32_t* hist_excl, uint32_t* lb, uint32_t* ticket, DevFlags* fl,
                     cudaStream_t s) {
    k_onesweep32<BITS><<<onesweep_grid<BITS>(), Onesweep<BITS>::NT, Onesweep<BITS>::SMEM, s>>>(kin, vin, kout, vout, count, cap,
                                                                                         shift, hist_excl, lb, ticket, fl);
}

cudaError_t launch_bin_sort(const queen_proj& proj, int n_views, int W, int H, queen_bins& bins, void* scratch,
                            const WsLayout& L, DevFlags* fl, cudaStream_t s, Prof* prof) {
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int64_t T = (int64_t)gx * gy;
    const int64_t count = (int64_t)n_views * proj.n_pad;
    const uint32_t cap = (uint32_t)bins.keys_cap;
    const int gbits = tile_gbits(T * n_views);
    const int tbits = tile_digit_bits(gbits);
    const int tpasses = tile_passes(gbits);
    unsigned char* ws = static_cast<unsigned char*>(scratch);
    uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist);  // [depth 4 | tile 4][MAX_BINS] counts, then excl
    uint32_t* hist_excl = hist + (DEPTH_PASSES + MAX_TILE_PASSES) * MAX_BINS;
    unsigned long long* vis_lb = reinterpret_cast<unsigned long long*>(ws + L.vis_lb);
    unsigned long long* dup_lb = reinterpret_cast<unsigned long long*>(ws + L.dup_lb);
    uint32_t* depth_lb = reinterpret_cast<uint32_t*>(ws + L.depth_lb);
    uint32_t* tile_lb = reinterpret_cast<uint32_t*>(ws + L.tile_lb);
    uint32_t* dk[2] = {reinterpret_cast<uint32_t*>(ws + L.dkeys), reinterpret_cast<uint32_t*>(ws + L.dkeys_alt)};
    uint32_t* dv[2] = {reinterpret_cast<uint32_t*>(ws + L.dvals), reinterpret_cast<uint32_t*>(ws + L.dvals_alt)};
    const int64_t elem_tiles = (count + SORT_TILE - 1) / SORT_TILE;
    const int64_t os_elem_tiles = (count + OS_TILE - 1) / OS_TILE;
    const int64_t os_key_tiles = ((int64_t)cap + OS_TILE - 1) / OS_TILE;
    uint32_t* Kd = bins.K;      // [0] = K entries
    uint32_t* Md = bins.K + 1;  // [1] = M visible pairs
    cudaError_t e;
    prof->begin(ST_COMPACT, s);
    if ((e = cudaMemsetAsync(fl->tickets, 0, sizeof(fl->tickets), s))) return e;
    if ((e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (DEPTH_PASSES + MAX_TILE_PASSES) * MAX_BINS, s))) return e;
    if ((e = cudaMemsetAsync(vis_lb, 0, sizeof(unsigned long long) * (elem_tiles + 1), s))) return e;
    if ((e = cudaMemsetAsync(dup_lb, 0, sizeof(unsigned long long) * (elem_tiles + 1), s))) return e;
    if ((e = cudaMemsetAsync(depth_lb, 0, sizeof(uint32_t) * DEPTH_PASSES * 256 * (size_t)(os_elem_tiles + 1), s))) return e;
    if ((e = cudaMemsetAsync(tile_lb, 0, sizeof(uint32_t) * (size_t)tpasses * (1 << tbits) * (size_t)(os_key_tiles + 1), s)))
        return e;
    int* diff = reinterpret_cast<int*>(ws + L.diff);
    uint32_t* tcounts = reinterpret_cast<uint32_t*>(ws + L.counts);
    uint32_t* view_tot = reinterpret_cast<uint32_t*>(ws + L.view_tot);
    const size_t dplane = (size_t)(gx + 1) * (gy + 1);
    if ((e = cudaMemsetAsync(diff, 0, sizeof(int) * dplane * n_views, s))) return e;
    if ((e = cudaMemsetAsync(bins.K, 0, sizeof(uint32_t) * 4, s))) return e;
    if (elem_tiles > 0)
        k_vis_compact<<<(unsigned)elem_tiles, SORT_THREADS, 0, s>>>(proj.tiles, proj.depth, count, dk[0], dv[0], vis_lb,
                                                                     fl, Md);
    prof->end(s);
    // depth digits (LSD: least significant first) on the visible pairs
    prof->begin(ST_DEPTH_SORT, s);
    const int sms = num_sms();
    k_hist_depth<<<sms * 2, 256, 0, s>>>(dk[0], Md, hist);
    k_hist_scan<<<1, 32 * DEPTH_PASSES, 0, s>>>(hist, hist_excl, DEPTH_PASSES, 256);
    int cur = 0;
    for (int p = 0; p < DEPTH_PASSES; ++p) {
        onesweep<8>(dk[cur], dv[cur], dk[cur ^ 1], dv[cur ^ 1], Md, (uint32_t)count, 8 * p, hist_excl + p * MAX_BINS,
                    depth_lb + (size_t)p * 256 * (os_elem_tiles + 1), &fl->tickets[TK_DEPTH + p], fl, s);
        cur ^= 1;
    }
    prof->end(s, DEPTH_PASSES + 2);
    // offsets in depth order + duplication (+ tile-digit histograms)
    prof->begin(ST_DUPLICATE, s);
    uint32_t* thist = hist + DEPTH_PASSES * MAX_BINS;
    uint32_t* thist_excl = hist_excl + DEPTH_PASSES * MAX_BINS;
    if (elem_tiles > 0)
        k_scan_dup<<<(unsigned)elem_tiles, SORT_THREADS, DUP_SMEM, s>>>(dv[cur], Md,
                                                                         reinterpret_cast<const short4*>(proj.rect),
                                                                         proj.n_pad, gx, gy, (uint32_t)T, bins.keys,
                                                                         bins.vals, cap, dup_lb, fl, Kd, diff);
    prof->end(s);
    // per-tile entry counts -> ranges and tile-digit histograms
    prof->begin(ST_RANGES, s);
    k_tile_counts<<<n_views, 1024, sizeof(int) * dplane, s>>>(diff, gx, gy, tcounts, tcounts + T * n_views, view_tot, thist,
                                                               tpasses, tbits);
    k_ranges_finalize<<<sms * 2, 256, 0, s>>>(tcounts, tcounts + T * n_views, view_tot, n_views, (uint32_t)T, cap, Kd,
                                              reinterpret_cast<uint2*>(bins.ranges));
    prof->end(s, 2);
    // tile digits on the K entries
    prof->begin(ST_TILE_SORT, s);
    k_hist_scan<<<1, 32 * MAX_TILE_PASSES, 0, s>>>(thist, thist_excl, tpasses, 1 << tbits);
    uint32_t* ka = bins.keys;
    uint32_t* kb = bins.keys_alt;
    uint32_t* va = bins.vals;
    uint32_t* vb = bins.vals_alt;
    for (int p = 0; p < tpasses; ++p) {
        uint32_t* lbp = tile_lb + (size_t)p * (1 << tbits) * (os_key_tiles + 1);
        if (tbits == 9)
            onesweep<9>(ka, va, kb, vb, Kd, cap, 9 * p, thist_excl + p * MAX_BINS, lbp, &fl->tickets[TK_TILE + p], fl, s);
        else
            onesweep<8>(ka, va, kb, vb, Kd, cap, 8 * p, thist_excl + p * MAX_BINS, lbp, &fl->tickets[TK_TILE + p], fl, s);
        uint32_t* tk = ka; ka = kb; kb = tk;
        uint32_t* tv = va; va = vb; vb = tv;
    }
    prof->end(s, tpasses + 1);
    bins.sorted_in_alt = (tpasses & 1) ? 1 : 0;
    return cudaGetLastError();
}

}  // namespace queen
