// K3-K6: binning for a batch of equally-sized views (BASELINE north_star: "duplication
// of Gaussians into 16x16 tiles, a radix sort on (tile, depth) keys, per-tile range
// extraction"; "warp-level scans and a custom onesweep radix sort").  DESIGN.md §8.
//
// The entries are ordered by (gt, depth, index), gt = view*T + tile.  Every copy of a Gaussian
// carries the same depth, so the depth order is sorted once, on the M visible (view,
// Gaussian) pairs; the entries are then written directly at their final positions:
//       k_bin_init      the batch's tickets, histograms, look-back words, depth min/max
//   K3a k_slab_count    per slab of S consecutive elements of a view (one CTA): visible
//                       count, depth-digit histograms, and the slab's entries per tile via
//                       a shared-memory 2D difference array of tile rects -> counts[slab][t]
//       k_slab_sum      per view: entries per tile
//       k_view_scan_totals  per view: view-local tile starts; its last block: K, M, capacity
//                       check, slab offsets of the visible pairs
//       k_slab_compact  visible pairs in (view, index) order -> (depth bits, flat index) [M];
//                       also (K6) [first, last+1) of each gt from the per-tile counts, and its
//                       last block scans the depth-digit histograms
//   K5a k_onesweep32<9> x3 (+<8>)  stable sort of the pairs by relative depth (27 + 4 bits)
//   K4' k_piece_count / k_piece_colscan (+ bases) / k_piece_scatter: the pairs cut
//       into pieces per 16x8-tile bucket, each bucket's pieces in depth order
//   K5' k_emit_plan + k_emit: each bucket's entries written at their final positions
// The result equals sorting the 96-bit (gt << 31 | depth, index) tuples (oracle: std::sort).
//
// onesweep pass: persistent CTAs take 4096-key tiles by atomic ticket (forward
// progress for the look-back), rank keys with a warp multisplit in key order (stable;
// shared-memory match words), publish per-digit tile counts, resolve global digit offsets by
// decoupled look-back, stage the tile in shared memory in digit order and write it out
// coalesced.
#include <algorithm>

#include "queen_internal.cuh"

namespace queen {

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

constexpr uint32_t LB_AGG = 1u << 30, LB_INC = 2u << 30, LB_MASK = (1u << 30) - 1;
constexpr long long SPIN_LIMIT = 1ll << 24;
#ifndef QUEEN_LB_BATCH
#define QUEEN_LB_BATCH 4  // measured (round-1 tile sort, N3DV): 1 -> 420 us, 2 -> 388, 4 -> 390, 8 -> 408, 16 -> 450
#endif
constexpr int LB_BATCH = QUEEN_LB_BATCH;
#ifndef QUEEN_OS_MATCH_OR
#define QUEEN_OS_MATCH_OR 1  // warp match by shared atomicOr (measured, round-1 tile sort: 488 -> 417 us vs match.any)
#endif  // onesweep look-back predecessors loaded per round trip

// dynamic-tile tickets: depth passes 0..3, emission; last-block counters of k_view_scan_totals,
// k_slab_compact and k_piece_colscan
enum : int { TK_DEPTH = 0, TK_EMIT = 4, TK_VSCAN = 5, TK_COMPACT = 6, TK_COLSCAN = 7 };




// ---------------------------------------------------------------------------
// K3a: per-slab counting.  Each view's elements are cut into slabs of
// S consecutive indices (bin_plan); one CTA per slab:
//   * visible elements (tiles > 0) counted -> svis[slab];
//   * their depth digits (4 x 8 bits) histogrammed in shared memory -> hist (global adds);
//   * their tile rects added to a private shared-memory 2D difference array of per-tile
//     entry counts (4 shared atomics per element; measured ~11 lane-ops per clock per SM,
//     while REDs into one global plane serialise on hot corners), whose 2D prefix sum is
//     written densely as counts[slab][t].
// ---------------------------------------------------------------------------
constexpr int SLAB_THREADS = 512;
constexpr int SLAB_IT = 8;                             // consecutive elements per thread per round
constexpr int SLAB_ROUND = SLAB_THREADS * SLAB_IT;     // 4096 elements per round

// The 8 elements [i, i+8) of view row jb: tile counts, rects, depth bits (vector loads when
// the run is whole; n_pad % 4 == 0 keeps them 16-byte aligned), invalid ones get tiles = 0.
__device__ __forceinline__ void load8(const uint32_t* __restrict__ tiles, const short4* __restrict__ rect,
                                      const uint32_t* __restrict__ depth, int64_t jb, int i, int b, uint32_t (&nt)[8],
                                      short4 (&r)[8], uint32_t (&dk)[8], bool want_rect, bool want_depth) {
    if (i + 8 <= b) {
        const uint4 t0 = __ldg(reinterpret_cast<const uint4*>(tiles + jb + i));
        const uint4 t1 = __ldg(reinterpret_cast<const uint4*>(tiles + jb + i + 4));
        nt[0] = t0.x; nt[1] = t0.y; nt[2] = t0.z; nt[3] = t0.w; nt[4] = t1.x; nt[5] = t1.y; nt[6] = t1.z; nt[7] = t1.w;
        if (want_rect) {
            const uint4* rp = reinterpret_cast<const uint4*>(rect + jb + i);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 x = __ldg(rp + q);
                r[2 * q] = *reinterpret_cast<const short4*>(&x.x);
                r[2 * q + 1] = *reinterpret_cast<const short4*>(&x.z);
            }
        }
        if (want_depth) {
            const uint4 d0 = __ldg(reinterpret_cast<const uint4*>(depth + jb + i));
            const uint4 d1 = __ldg(reinterpret_cast<const uint4*>(depth + jb + i + 4));
            dk[0] = d0.x; dk[1] = d0.y; dk[2] = d0.z; dk[3] = d0.w; dk[4] = d1.x; dk[5] = d1.y; dk[6] = d1.z; dk[7] = d1.w;
        }
    } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const bool ok = i + e < b;
            nt[e] = ok ? tiles[jb + i + e] : 0u;
            if (want_rect) r[e] = ok ? rect[jb + i + e] : make_short4(0, 0, 0, 0);
            if (want_depth) dk[e] = ok ? depth[jb + i + e] : 0u;
        }
    }
}

__global__ void __launch_bounds__(SLAB_THREADS) k_slab_count(const uint32_t* __restrict__ tiles,
                                                             const short4* __restrict__ rect,
                                                             const uint32_t* __restrict__ depth, int n_pad, int S, int spv,
                                                             int gx, int gy, uint32_t* __restrict__ counts,
                                                             uint32_t* __restrict__ svis, uint32_t* __restrict__ dminmax) {
    extern __shared__ int cs[];  // [(gy+1)][(gx+1)] difference array -> 2D prefix
    __shared__ uint32_t s_vis, s_min, s_max;
    const int slab = blockIdx.x;
    const int v = slab / spv;
    const int a = (slab - v * spv) * S;
    const int b = min(a + S, n_pad);
    const int dw = gx + 1, dplane = (gx + 1) * (gy + 1);
    const int T = gx * gy;
    for (int q = threadIdx.x; q < dplane; q += blockDim.x) cs[q] = 0;
    if (threadIdx.x == 0) { s_vis = 0; s_min = 0xffffffffu; s_max = 0u; }
    __syncthreads();
    const int64_t jb = (int64_t)v * n_pad;
    uint32_t vis = 0, kmin = 0xffffffffu, kmax = 0u;
    for (int i = a + threadIdx.x * SLAB_IT; i < b; i += SLAB_ROUND) {
        uint32_t nt[8], dk[8];
        short4 r[8];
        load8(tiles, rect, depth, jb, i, b, nt, r, dk, true, true);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if (nt[e] == 0) continue;
            ++vis;
            kmin = min(kmin, dk[e]);
            kmax = max(kmax, dk[e]);
            atomicAdd(&cs[r[e].y * dw + r[e].x], 1);
            atomicAdd(&cs[r[e].y * dw + r[e].z + 1], -1);
            atomicAdd(&cs[(r[e].w + 1) * dw + r[e].x], -1);
            atomicAdd(&cs[(r[e].w + 1) * dw + r[e].z + 1], 1);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        vis += __shfl_down_sync(0xffffffffu, vis, o);
        kmin = min(kmin, __shfl_down_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_down_sync(0xffffffffu, kmax, o));
    }
    if ((threadIdx.x & 31) == 0 && vis) {
        atomicAdd(&s_vis, vis);
        atomicMin(&s_min, kmin);
        atomicMax(&s_max, kmax);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        svis[slab] = s_vis;
        if (s_vis) {
            atomicMin(&dminmax[0], s_min);
            atomicMax(&dminmax[1], s_max);
        }
    }
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
    uint32_t* out = counts + (int64_t)slab * T;
    for (int t = threadIdx.x; t < T; t += blockDim.x) out[t] = (uint32_t)cs[(t / gx) * dw + (t % gx)];
}

// Entries per tile = column sums of counts[slab][t] over the view's slabs (one thread per
// tile, grid = views x tile chunks).
__global__ void __launch_bounds__(256) k_slab_sum(const uint32_t* __restrict__ counts, int spv, int T,
                                                  uint32_t* __restrict__ tcounts) {
    const int v = blockIdx.y;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    const uint32_t* c0 = counts + (int64_t)v * spv * T + t;
    uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int q = 0;
    for (; q + 4 <= spv; q += 4) {
        s0 += c0[(int64_t)q * T];
        s1 += c0[(int64_t)(q + 1) * T];
        s2 += c0[(int64_t)(q + 2) * T];
        s3 += c0[(int64_t)(q + 3) * T];
    }
    for (; q < spv; ++q) s0 += c0[(int64_t)q * T];
    tcounts[(int64_t)v * T + t] = s0 + s1 + s2 + s3;
}

// Per-view block (1024 threads): view-local exclusive starts of the tile totals and the view total.
__device__ void view_scan_body(const uint32_t* __restrict__ tcounts, int T, uint32_t* lstart, uint32_t* view_tot) {
    __shared__ uint32_t s_w[32];
    const int v = blockIdx.x;
    const uint32_t* tc = tcounts + (int64_t)v * T;
    const int per = (T + blockDim.x - 1) / blockDim.x;
    const int t0 = threadIdx.x * per, t1 = min(T, t0 + per);
    uint32_t csum = 0;
    for (int t = t0; t < t1; ++t) csum += tc[t];
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
    for (int t = t0; t < t1; ++t) {
        lstart[(int64_t)v * T + t] = run;
        run += tc[t];
    }
    if (threadIdx.x == 0) view_tot[v] = tot;
}

__global__ void __launch_bounds__(1024) k_view_scan(const uint32_t* __restrict__ tcounts, int T, uint32_t* lstart,
                                                    uint32_t* view_tot) {
    view_scan_body(tcounts, T, lstart, view_tot);
}

// K, M, overflow flag; slab visible counts -> global exclusive offsets (in place).  Run by one
// block of 1024 threads: the last view block of k_view_scan, or k_totals.  view_tot is read
// through L2 (other blocks of the same launch wrote it).
__device__ void totals_body(const uint32_t* view_tot, int n_views, uint32_t* svis, int slabs, uint32_t cap,
                            uint32_t* Kd, DevFlags* fl) {
    __shared__ uint32_t s_w[32];
    __shared__ uint32_t s_carry;
    if (threadIdx.x == 0) {
        unsigned long long K = 0;
        for (int v = 0; v < n_views; ++v) K += __ldcg(view_tot + v);
        const bool over = K > cap;
        if (over) {
            raise_flag(fl, FLAG_CAPACITY);
            atomicMax(&fl->info, K);
        }
        // overflow: no entry list is produced (every range is [0,0)); QUEEN_ERR_CAPACITY
        // carries the K needed.  Kd[2] = overflow flag.
        Kd[0] = over ? 0u : (uint32_t)K;
        Kd[2] = over ? 1u : 0u;
        s_carry = 0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int b0 = 0; b0 < slabs; b0 += blockDim.x) {
        const int q = b0 + threadIdx.x;
        const uint32_t x = q < slabs ? svis[q] : 0u;
        uint32_t inc = x;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) s_w[w] = inc;
        __syncthreads();
        uint32_t pre = 0, tot = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            pre += k < w ? s_w[k] : 0u;
            tot += s_w[k];
        }
        const uint32_t carry = s_carry;
        if (q < slabs) svis[q] = carry + pre + inc - x;
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) Kd[1] = s_carry;  // M visible pairs
}

__global__ void __launch_bounds__(1024) k_totals(const uint32_t* __restrict__ view_tot, int n_views, uint32_t* svis,
                                                 int slabs, uint32_t cap, uint32_t* Kd, DevFlags* fl) {
    totals_body(view_tot, n_views, svis, slabs, cap, Kd, fl);
}

// k_view_scan, whose last block to finish then runs totals_body (one launch instead of two)
__global__ void __launch_bounds__(1024) k_view_scan_totals(const uint32_t* __restrict__ tcounts, int T,
                                                           uint32_t* lstart, uint32_t* view_tot, int n_views,
                                                           uint32_t* svis, int slabs, uint32_t cap, uint32_t* Kd,
                                                           DevFlags* fl, uint32_t* ticket) {
    view_scan_body(tcounts, T, lstart, view_tot);
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    totals_body(view_tot, n_views, svis, slabs, cap, Kd, fl);
}

// K3b: per slab, its visible elements in index order -> (depth bits, flat index) pairs at the
// slab's global offset.  Rounds of 4096 elements, 8 consecutive per thread (vector loads);
// block scan of the per-thread visible counts; pairs staged in shared memory in order and
// written out coalesced.
// (ranges_slice, hist_scan_body: defined below)
__device__ void ranges_slice(const uint32_t* __restrict__ counts, const uint32_t* __restrict__ lstart,
                             const uint32_t* __restrict__ view_tot, int n_views, uint32_t T, uint32_t cap,
                             const uint32_t* Kd, uint2* __restrict__ ranges, uint32_t* ohist);
__device__ void hist_scan_body(const uint32_t* hist, uint32_t* excl, int passes, int bins);

struct RangesArgs {  // k_ranges_finalize's work, done by k_slab_compact's blocks (grid-stride)
    const uint32_t* counts;
    const uint32_t* lstart;
    const uint32_t* view_tot;
    int n_views;
    uint32_t T, cap;
    const uint32_t* Kd;
    uint2* ranges;
    uint32_t* ocnt;  // blend-schedule class counts [ORDER_BINS] | cursors [ORDER_BINS]
};

// Also: every block finalises a slice of the tile ranges, and the last block to finish scans
// the depth digit histograms (k_ranges_finalize and k_hist_scan folded in: two launches fewer)
__global__ void __launch_bounds__(SLAB_THREADS) k_slab_compact(const uint32_t* __restrict__ tiles,
                                                               const uint32_t* __restrict__ depth, int n_pad, int S,
                                                               int spv, const uint32_t* __restrict__ soff,
                                                               const uint32_t* __restrict__ dminmax,
                                                               uint32_t* __restrict__ dkeys, uint32_t* __restrict__ dvals,
                                                               uint32_t* __restrict__ hist, uint32_t* __restrict__ hist_excl,
                                                               uint32_t* ticket, RangesArgs ra) {
    constexpr int NW = SLAB_THREADS / 32;
    __shared__ uint32_t s_w[NW];
    __shared__ uint32_t s_k[SLAB_ROUND], s_j[SLAB_ROUND];
    __shared__ uint32_t sh[DEPTH_PASSES * MAX_BINS];
    const int slab = blockIdx.x;
    const int v = slab / spv;
    const int a = (slab - v * spv) * S;
    const int b = min(a + S, n_pad);
    const int64_t jb = (int64_t)v * n_pad;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t kmin = dminmax[0];
    for (int q = threadIdx.x; q < DEPTH_PASSES * MAX_BINS; q += SLAB_THREADS) sh[q] = 0;
    uint32_t base = soff[slab];
    for (int i0 = a; i0 < b; i0 += SLAB_ROUND) {
        const int i = i0 + threadIdx.x * SLAB_IT;
        uint32_t nt[8], dk[8];
        short4 r[8];
        load8(tiles, nullptr, depth, jb, i, b, nt, r, dk, false, true);
        uint32_t c = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) c += nt[e] ? 1u : 0u;
        uint32_t inc = c;
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
            pre += q < w ? s_w[q] : 0u;
            tot += s_w[q];
        }
        uint32_t o = pre + inc - c;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if (nt[e]) {
                const uint32_t rk = dk[e] - kmin;  // relative depth key (order-preserving: keys >= kmin)
                s_k[o] = rk;
                s_j[o] = (uint32_t)(jb + i + e);
                ++o;
#pragma unroll
                for (int p = 0; p < DEPTH_PASSES; ++p)
                    atomicAdd(&sh[p * MAX_BINS + ((rk >> (DEPTH_BITS * p)) & (MAX_BINS - 1))], 1u);
            }
        }
        __syncthreads();
        for (uint32_t q = threadIdx.x; q < tot; q += SLAB_THREADS) {
            dkeys[base + q] = s_k[q];
            dvals[base + q] = s_j[q];
        }
        base += tot;
        __syncthreads();
    }
    for (int q = threadIdx.x; q < DEPTH_PASSES * MAX_BINS; q += SLAB_THREADS)
        if (sh[q]) atomicAdd(&hist[q], sh[q]);
    ranges_slice(ra.counts, ra.lstart, ra.view_tot, ra.n_views, ra.T, ra.cap, ra.Kd, ra.ranges, ra.ocnt);
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    hist_scan_body(hist, hist_excl, DEPTH_PASSES, MAX_BINS);
    if (threadIdx.x >= 32 * DEPTH_PASSES && threadIdx.x < 32 * DEPTH_PASSES + 32) {
        // blend schedule: each class's first position (exclusive scan, two classes per lane)
        const int l = threadIdx.x & 31;
        const uint32_t a = __ldcg(ra.ocnt + 2 * l), b = __ldcg(ra.ocnt + 2 * l + 1);
        uint32_t x = a + b;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (l >= o) x += y;
        }
        ra.ocnt[ORDER_BINS + 2 * l] = x - a - b;
        ra.ocnt[ORDER_BINS + 2 * l + 1] = x - b;
    }
}

// exclusive scan of each pass's digit counts (one warp per pass; threads past 32 * passes idle)
__device__ void hist_scan_body(const uint32_t* hist, uint32_t* excl, int passes, int bins) {
    const int p = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (p >= passes) return;
    const int per = bins / 32;
    uint32_t s = 0;
    for (int q = 0; q < per; ++q) s += __ldcg(hist + p * MAX_BINS + lane * per + q);
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    uint32_t run = x - s;
    for (int q = 0; q < per; ++q) {
        const uint32_t c = __ldcg(hist + p * MAX_BINS + lane * per + q);
        excl[p * MAX_BINS + lane * per + q] = run;
        run += c;
    }
}

__global__ void k_hist_scan(const uint32_t* hist, uint32_t* excl, int passes, int bins) {
    hist_scan_body(hist, excl, passes, bins);
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

// Pass mode: key + value in, key + value out (the depth passes over the visible pairs).
enum : int { OS_KV = 0 };

template <int BITS, int MODE>
__global__ void __launch_bounds__(Onesweep<BITS>::NT) k_onesweep32(const uint32_t* __restrict__ kin,
                                                                   const uint32_t* __restrict__ vin,
                                                                   uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                                   const uint32_t* count_ptr, uint32_t cap, int shift,
                                                                   int pshift, int ibits,
                                                                   const uint32_t* __restrict__ hist_excl, uint32_t* lb,
                                                                   uint32_t* ticket, DevFlags* fl,
                                                                   const uint32_t* __restrict__ triv) {
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
    // every key has digit 0: the stable pass is the identity -- nothing is written, and the
    // consumers (k_piece_count / k_piece_scatter) read the pass's input buffer instead
    if (triv && triv[0] == Kn) return;
    const bool owns_digits = threadIdx.x * DPT < BINS;
#if QUEEN_OS_MATCH_OR
    // warp match by shared-memory atomicOr (experiment knob): the per-warp match words live in
    // the staging buffer (free until the scatter), re-zeroed at the start of every tile
    static_assert(NW * BINS <= 2 * TILE, "match words must fit the staging buffer");
    uint32_t* wmatch = sk + w * BINS;
#endif
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
        // zero the per-warp histograms (and match words) with 16-byte stores
        for (int q = threadIdx.x; q < NW * BINS / 4; q += NT) {
            reinterpret_cast<uint4*>(whist)[q] = make_uint4(0u, 0u, 0u, 0u);
#if QUEEN_OS_MATCH_OR
            reinterpret_cast<uint4*>(sk)[q] = make_uint4(0u, 0u, 0u, 0u);
#endif
        }
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
#if QUEEN_OS_MATCH_OR
#pragma unroll
        for (int j = 0; j < IT; ++j) {
            const uint32_t idx = base + w * (32 * IT) + j * 32 + lane;
            rk[j] = idx < Kn ? ((k[j] >> shift) & DMASK) : (uint32_t)BINS;
            const bool ok = rk[j] < (uint32_t)BINS;
            const uint32_t inv = __ballot_sync(0xffffffffu, !ok);
            if (ok) atomicOr(&wmatch[rk[j]], 1u << lane);
            __syncwarp();
            peers[j] = ok ? wmatch[rk[j]] : inv;
            __syncwarp();
            if (ok && (peers[j] & lt_mask) == 0) wmatch[rk[j]] = 0u;
            __syncwarp();
        }
#else
#pragma unroll
        for (int j = 0; j < IT; ++j) {
            const uint32_t idx = base + w * (32 * IT) + j * 32 + lane;
            rk[j] = idx < Kn ? ((k[j] >> shift) & DMASK) : (uint32_t)BINS;
            peers[j] = __match_any_sync(0xffffffffu, rk[j]);
        }
#endif
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
                    // batched look-back: LB_BATCH predecessors per round trip (independent
                    // loads), consumed in order until an inclusive prefix or an unpublished
                    // tile (retried) -- the serial L2 latency chain shrinks ~LB_BATCH-fold
                    int64_t look = (int64_t)tile - 1;
                    long long spins = 0;
                    for (;;) {
                        uint32_t x[LB_BATCH];
#pragma unroll
                        for (int q = 0; q < LB_BATCH; ++q)
                            x[q] = look - q >= 0 ? ld_volatile_u32(&lb[(size_t)(look - q) * BINS + d]) : LB_INC;
                        int used = 0;
                        bool done = false, stall = false;
#pragma unroll
                        for (int q = 0; q < LB_BATCH; ++q) {
                            if (done || stall) continue;
                            const uint32_t f = x[q] >> 30;
                            if (f == 0) { stall = true; continue; }
                            prefix += x[q] & LB_MASK;
                            ++used;
                            if (f == 2) done = true;
                        }
                        if (done) break;
                        look -= used;
                        if (stall && ++spins > SPIN_LIMIT) { raise_flag(fl, FLAG_TIMEOUT); break; }
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
// K4'/K5': bucketed emission (replaces duplication + the tile radix passes).
// A bucket is a BK_W x BK_H block of one view's tiles.  A piece is (pair, bucket) for every
// bucket a visible pair's tile rect intersects.  With the pairs already in depth order
// (m = their rank), the final entry list is known position by position:
//   entry (tile t, pair m) -> ranges[t].first + #{pairs m' < m whose rect covers t}
// and every such count is local to t's bucket.  So:
//   k_piece_count   per chunk of g.ch depth-ordered pairs: pieces per bucket -> pcnt[b][chunk];
//                   the pairs' tile rects copied into m order for the scatter
//   k_piece_colscan per bucket: exclusive scan over chunks (in place) -> the bucket's
//                   (chunk, bucket) segment offsets and totals; its last block: bucket bases
//                   and emit-tile bases (ceil(total / em_e) tiles per bucket)
//   k_piece_scatter per chunk: each piece (Gaussian index, rect inside the bucket) into its
//                   (chunk, bucket) segment, in m order (per-warp cursors, match.any ranks)
//   k_emit_plan     per emit tile (whole segments of one bucket, ~em_e pieces): its bucket,
//                   piece range and segment range (binary searches); clears its look-back words
//   k_emit          per emit tile (one warp): entries per bucket tile, each tile's offset among
//                   the bucket's earlier emit tiles by decoupled look-back, then every entry's
//                   Gaussian index written at its final position -- rank among the round's
//                   earlier pieces = popc(R[ly] & C[lx] & lower lanes) from 24 coverage ballots
// The result is bit-identical to the sorted (gt, depth, index) order: a bucket's pieces are
// emitted in m order, and m order is (depth, view, index) order.
// ---------------------------------------------------------------------------
constexpr int PC_THREADS = 512;             // PC_CH / 8 pairs per thread
constexpr size_t PC_MAX_SMEM = 200 * 1024;  // per-chunk bucket counters: up to 51200 buckets per batch
constexpr int PS_MAX_WARPS = 8;
#ifndef QUEEN_PC_BUDGET
#define QUEEN_PC_BUDGET 16  // M words of per-(bucket, chunk) counts before the chunk size doubles (measured 4 / 16 / 64: Immersive bucket 0.53 / 0.41 / 0.46 ms, stress 7.2 / 6.1 / 6.6 ms)
#endif             // k_piece_scatter: chunks (warps) per CTA, fewer when VNB is large
#ifndef QUEEN_PC_CH0
#define QUEEN_PC_CH0 PC_CH  // starting chunk size (pairs), doubled up to 8 PC_CH by the budget rule
#endif


struct BucketGeo {
    int gx, gy, nbx, nby, NB, VNB;
    int T, n_pad;
    int CHS;  // row stride of pcnt ([bucket][chunk]): the chunk capacity
    int ch;   // depth-ordered pairs per chunk (a power-of-two multiple of PC_CH)
    int em_e; // nominal pieces per emit tile
    unsigned long long npad_magic;  // ceil(2^64 / n_pad): j / n_pad = umulhi64(j, magic), exact for j < 2^32
};

// view of a flat pair index j = v n_pad + i, without an integer division
__device__ __forceinline__ uint32_t view_of(uint32_t j, const BucketGeo& g) {
    return (uint32_t)__umul64hi((unsigned long long)j, g.npad_magic);
}

__device__ __forceinline__ const uint32_t* depth_order(const uint32_t* a, const uint32_t* b, const uint32_t* triv,
                                                       uint32_t M) {
    // the last depth pass is skipped (identity) when its digit histogram says so: its input holds the order
    return triv[0] == M ? a : b;
}

__device__ __forceinline__ uint32_t visible_pairs(const uint32_t* Kd) { return Kd[2] ? 0u : Kd[1]; }

struct OrderSched {  // the blend schedule built by k_piece_count (see launch_rasterize's order_pre)
    const uint2* ranges;
    uint32_t* cursor;  // per class: next position (starts from k_slab_compact's last block)
    uint32_t* order;   // [n_views * T] tile permutation
};

__global__ void __launch_bounds__(PC_THREADS) k_piece_count(const uint32_t* __restrict__ dva,
                                                            const uint32_t* __restrict__ dvb,
                                                            const uint32_t* __restrict__ triv,
                                                            const uint32_t* __restrict__ Kd,
                                                            const short4* __restrict__ rect, BucketGeo g,
                                                            uint32_t* __restrict__ pcnt, uint32_t* __restrict__ rlo,
                                                            uint32_t* __restrict__ rhi, OrderSched osched) {
    extern __shared__ uint32_t sc[];  // [VNB]
    {  // the blend schedule (tiles longest list first): slices of PC_THREADS tiles, grid-stride
        __shared__ uint32_t s_cnt[ORDER_BINS], s_at[ORDER_BINS];
        const uint32_t G = (uint32_t)g.VNB / (uint32_t)g.NB * (uint32_t)g.T;  // n_views * T
        for (uint32_t c0 = blockIdx.x * PC_THREADS; c0 < G; c0 += gridDim.x * PC_THREADS) {
            for (int q = threadIdx.x; q < ORDER_BINS; q += PC_THREADS) s_cnt[q] = 0u;
            __syncthreads();
            const uint32_t i = c0 + threadIdx.x;
            int cl = 0;
            uint32_t rank = 0;
            if (i < G) {
                cl = order_class(osched.ranges[i]);
                rank = atomicAdd(&s_cnt[cl], 1u);
            }
            __syncthreads();
            for (int q = threadIdx.x; q < ORDER_BINS; q += PC_THREADS)
                if (s_cnt[q]) s_at[q] = atomicAdd(&osched.cursor[q], s_cnt[q]);
            __syncthreads();
            if (i < G) osched.order[s_at[cl] + rank] = i;
            __syncthreads();
        }
    }
    const uint32_t M = visible_pairs(Kd);
    const uint32_t c = blockIdx.x;
    if ((uint64_t)c * g.ch >= M) return;
    const uint32_t* __restrict__ dvals = depth_order(dva, dvb, triv, Kd[1]);
    for (int b = threadIdx.x; b < g.VNB; b += PC_THREADS) sc[b] = 0u;
    __syncthreads();
#pragma unroll 2
    for (int e = 0; e < g.ch / PC_THREADS; ++e) {
        const uint32_t m = c * g.ch + e * PC_THREADS + threadIdx.x;
        if (m < M) {
            const uint32_t j = __ldg(dvals + m);
            const short4 r = __ldg(rect + j);
            // the pair's tile rect in m order, for the scatter's coalesced reads
            rlo[m] = (uint32_t)(uint16_t)r.x | ((uint32_t)(uint16_t)r.y << 16);
            rhi[m] = (uint32_t)(uint16_t)r.z | ((uint32_t)(uint16_t)r.w << 16);
            const int vb = (int)view_of(j, g) * g.NB;
            const int bx0 = r.x / BK_W, bx1 = r.z / BK_W, by0 = r.y / BK_H, by1 = r.w / BK_H;
            for (int by = by0; by <= by1; ++by)
                for (int bx = bx0; bx <= bx1; ++bx) atomicAdd(&sc[vb + by * g.nbx + bx], 1u);
        }
    }
    __syncthreads();
    // pcnt is bucket-major ([bucket][chunk], row stride g.CHS): each bucket's segment offsets are
    // contiguous for the column scan and the emit tiles' segment search
    for (int b = threadIdx.x; b < g.VNB; b += PC_THREADS) pcnt[(size_t)b * g.CHS + c] = sc[b];
}

// one block: bucket bases (exclusive scan of the totals) and emit-tile bases; meta[0] = pieces,
// meta[1] = emit tiles.  Run by the last block of k_piece_colscan (256 threads).
__device__ void piece_base_body(const uint32_t* ptotal, int VNB, uint32_t em_e, uint32_t* __restrict__ pbase,
                                uint32_t* __restrict__ ebase, uint32_t* __restrict__ meta, uint32_t* __restrict__ Kd) {
    constexpr int NWB = 8;  // warps of the 256-thread block
    __shared__ uint32_t s_w[NWB], s_e[NWB];
    __shared__ uint32_t s_carry, s_ecarry;
    if (threadIdx.x == 0) { s_carry = 0; s_ecarry = 0; }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int b0 = 0; b0 < VNB; b0 += blockDim.x) {
        const int b = b0 + threadIdx.x;
        const uint32_t x = b < VNB ? __ldcg(ptotal + b) : 0u;
        const uint32_t y = (x + em_e - 1) / em_e;
        uint32_t ix = x, iy = y;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t a = __shfl_up_sync(0xffffffffu, ix, o), c = __shfl_up_sync(0xffffffffu, iy, o);
            if (lane >= o) { ix += a; iy += c; }
        }
        if (lane == 31) { s_w[w] = ix; s_e[w] = iy; }
        __syncthreads();
        uint32_t px = 0, py = 0, tx = 0, ty = 0;
#pragma unroll
        for (int q = 0; q < NWB; ++q) {
            px += q < w ? s_w[q] : 0u;
            py += q < w ? s_e[q] : 0u;
            tx += s_w[q];
            ty += s_e[q];
        }
        const uint32_t cx = s_carry, cy = s_ecarry;
        if (b < VNB) {
            pbase[b] = cx + px + ix - x;
            ebase[b] = cy + py + iy - y;
        }
        __syncthreads();
        if (threadIdx.x == 0) { s_carry = cx + tx; s_ecarry = cy + ty; }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ebase[VNB] = s_ecarry;
        meta[0] = s_carry;
        meta[1] = s_ecarry;
        Kd[3] = s_carry;  // pieces P (evidence: bench's algorithmic bytes)
    }
}

// per bucket (one warp): exclusive scan of its pieces over the chunks (in place) and the total,
// 8 rounds of 32 chunks loaded at once; the last block to finish then computes the bucket and
// emit-tile bases (piece_base_body: one launch fewer)
constexpr int CS_ROUNDS = 8;
__global__ void __launch_bounds__(256) k_piece_colscan(uint32_t* __restrict__ pcnt, const uint32_t* __restrict__ Kd_in,
                                                       BucketGeo g, uint32_t* __restrict__ ptotal,
                                                       uint32_t* __restrict__ pbase, uint32_t* __restrict__ ebase,
                                                       uint32_t* __restrict__ meta, uint32_t* Kd,
                                                       uint32_t* ticket) {  // (Kd aliases Kd_in: [3] written, [1..2] read)
    const int b = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (b < g.VNB) {  // warp-uniform
        const uint32_t M = visible_pairs(Kd_in);
        const uint32_t nch = (M + g.ch - 1) / g.ch;
        uint32_t* row = pcnt + (size_t)b * g.CHS;
        uint32_t carry = 0;
        for (uint32_t c0 = 0; c0 < nch; c0 += 32 * CS_ROUNDS) {
            uint32_t xs[CS_ROUNDS];
#pragma unroll
            for (int u = 0; u < CS_ROUNDS; ++u) {
                const uint32_t c = c0 + 32 * u + lane;
                xs[u] = c < nch ? row[c] : 0u;
            }
#pragma unroll
            for (int u = 0; u < CS_ROUNDS; ++u) {
                const uint32_t c = c0 + 32 * u + lane;
                uint32_t inc = xs[u];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                if (c < nch) row[c] = carry + inc - xs[u];
                carry += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
        if (lane == 0) ptotal[b] = carry;
    }
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    piece_base_body(ptotal, g.VNB, (uint32_t)g.em_e, pbase, ebase, meta, Kd);
}

// bucket-local start of emit tile k of bucket b: the first (chunk, bucket) segment that starts
// at or after k * em_e (emit tiles hold whole segments), or the bucket total
// (also returns the chunk c whose segment starts there: off[c] = start, c = nch at the end).
// Both ends of a tile are searched in lockstep (independent loads in flight together).
__device__ __forceinline__ void emit_range(const uint32_t* row, uint32_t nch, uint32_t total, uint32_t k,
                                           uint32_t em_e, uint32_t& s0, uint32_t& c0, uint32_t& s1, uint32_t& c1) {
    const uint32_t wa = k * em_e, wb = (k + 1) * em_e;
    uint32_t la = 0, ha = nch, lb = 0, hb = nch;  // first c with off[c] >= want (off[nch] := total)
    while (la < ha || lb < hb) {
        const uint32_t ma = (la + ha) >> 1, mb = (lb + hb) >> 1;
        const uint32_t va = la < ha ? row[ma] : 0u, vb = lb < hb ? row[mb] : 0u;
        if (la < ha) { if (va >= wa) ha = ma; else la = ma + 1; }
        if (lb < hb) { if (vb >= wb) hb = mb; else lb = mb + 1; }
    }
    c0 = la;
    c1 = lb;
    s0 = la < nch ? row[la] : total;
    s1 = lb < nch ? row[lb] : total;
}

// one thread per emit tile: its bucket (binary search of the emit-tile bases), index k, pieces
// [s0, s0 + n) of the bucket, and its chunk segments [c0, c0 + nseg) -- all the searches in
// flight at once, before k_emit; also clears the tile's look-back words (only the NE tiles in
// use, not the capacity)
__global__ void __launch_bounds__(256) k_emit_plan(const uint32_t* __restrict__ pcnt, const uint32_t* __restrict__ ptotal,
                                                   const uint32_t* __restrict__ ebase,
                                                   const uint32_t* __restrict__ meta, const uint32_t* __restrict__ Kd,
                                                   BucketGeo g, uint4* __restrict__ plan, uint32_t* __restrict__ lb) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= meta[1]) return;
    const uint32_t nch = (visible_pairs(Kd) + g.ch - 1) / g.ch;
    uint32_t lo = 0, hi = (uint32_t)g.VNB;  // the last bucket b with ebase[b] <= t (non-empty: ebase[b+1] > t)
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(ebase + mid) <= t) lo = mid; else hi = mid;
    }
    const uint32_t b = lo;
    const uint32_t k = t - __ldg(ebase + b);
    const uint32_t tot = ptotal[b];
    const uint32_t* row = pcnt + (size_t)b * g.CHS;
    uint32_t s0, cA, s1, cB;
    emit_range(row, nch, tot, k, (uint32_t)g.em_e, s0, cA, s1, cB);
    plan[2 * (size_t)t] = make_uint4(b, k, s0, s1 - s0);
    plan[2 * (size_t)t + 1] = make_uint4(cA, cB - cA, 0u, 0u);
    uint4* lbt = reinterpret_cast<uint4*>(lb + (size_t)t * BK_T);  // the tile's look-back words, unpublished
#pragma unroll 8
    for (int q = 0; q < BK_T / 4; ++q) lbt[q] = make_uint4(0u, 0u, 0u, 0u);
}

// One CTA per chunk, its pairs split into wpc contiguous warp ranges.  Phase 1: each warp counts
// its pieces per bucket; the counts become per-warp cursors (chunk offset + earlier warps).
// Phase 2: each warp walks its pairs in m order with the pieces flattened 32 at a time
// ((pair, bucket row, bucket column) order); the pieces of one bucket in such a step come from
// distinct pairs in lane order, so match.any on the bucket gives each its rank.  Every (chunk,
// bucket) segment thus comes out in m order and the emission needs no sort.  A piece is stored as
// its Gaussian index (piece_gi) and its rect inside the bucket (piece_lr), so the emission streams
// them without gathers; the pairs' indices and rects are read in m order (k_piece_count wrote the
// rects there), 8 rounds of loads in flight per lane.
constexpr int PS_ROUNDS = 8;
__global__ void __launch_bounds__(PS_MAX_WARPS * 32) k_piece_scatter(const uint32_t* __restrict__ dva,
                                                                     const uint32_t* __restrict__ dvb,
                                                                     const uint32_t* __restrict__ triv,
                                                                     const uint32_t* __restrict__ Kd,
                                                                     const uint32_t* __restrict__ rlo,
                                                                     const uint32_t* __restrict__ rhi, BucketGeo g,
                                                                     const uint32_t* __restrict__ pcnt,
                                                                     const uint32_t* __restrict__ pbase,
                                                                     uint32_t* __restrict__ piece_gi,
                                                                     uint32_t* __restrict__ piece_lr) {
    extern __shared__ uint32_t ps_smem[];  // [wpc][VNB] counts, then cursors
    __shared__ uint32_t s_rcp[BK_W + 1];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpc = blockDim.x >> 5;
    const uint32_t M = visible_pairs(Kd);
    const uint32_t c = blockIdx.x;
    if ((uint64_t)c * g.ch >= M) return;  // block-uniform
    const uint32_t* __restrict__ dvals = depth_order(dva, dvb, triv, Kd[1]);
    uint32_t* cur = ps_smem + (size_t)w * g.VNB;
    for (int b = lane; b < g.VNB; b += 32) cur[b] = 0u;
    if (threadIdx.x <= BK_W) s_rcp[threadIdx.x] = threadIdx.x ? (65536u + threadIdx.x - 1) / threadIdx.x : 0u;
    const uint32_t span = g.ch / wpc;  // pairs per warp (multiple of 32 * PS_ROUNDS)
    const uint32_t m0 = c * g.ch + w * span;
    const uint32_t mend = min(M, m0 + span);
    __syncthreads();
    // phase 1: pieces per (warp, bucket)
    for (uint32_t mb = m0; mb < mend; mb += 32 * PS_ROUNDS) {
        uint32_t jv[PS_ROUNDS], lo[PS_ROUNDS], hi[PS_ROUNDS];
#pragma unroll
        for (int u = 0; u < PS_ROUNDS; ++u) {
            const uint32_t m = mb + 32 * u + lane;
            jv[u] = m < mend ? __ldg(dvals + m) : 0xffffffffu;
            lo[u] = m < mend ? __ldg(rlo + m) : 0u;
            hi[u] = m < mend ? __ldg(rhi + m) : 0u;
        }
#pragma unroll
        for (int u = 0; u < PS_ROUNDS; ++u) {
            if (jv[u] == 0xffffffffu) continue;
            const int vb = (int)view_of(jv[u], g) * g.NB;
            const int bx0 = (int)(lo[u] & 0xffffu) / BK_W, by0 = (int)(lo[u] >> 16) / BK_H;
            const int bx1 = (int)(hi[u] & 0xffffu) / BK_W, by1 = (int)(hi[u] >> 16) / BK_H;
            for (int by = by0; by <= by1; ++by)
                for (int bx = bx0; bx <= bx1; ++bx) atomicAdd(&cur[vb + by * g.nbx + bx], 1u);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < g.VNB; b += blockDim.x) {  // cursors: chunk offset + earlier warps
        uint32_t run = pbase[b] + pcnt[(size_t)b * g.CHS + c];
        for (int ww = 0; ww < wpc; ++ww) {
            const uint32_t x = ps_smem[(size_t)ww * g.VNB + b];
            ps_smem[(size_t)ww * g.VNB + b] = run;
            run += x;
        }
    }
    __syncthreads();
    // phase 2: the pieces in m order, flattened 32 at a time
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t le = lane == 31 ? 0xffffffffu : (2u << lane) - 1u;
    for (uint32_t mb = m0; mb < mend; mb += 32 * PS_ROUNDS) {
        uint32_t jv[PS_ROUNDS], lo[PS_ROUNDS], hi[PS_ROUNDS];
#pragma unroll
        for (int u = 0; u < PS_ROUNDS; ++u) {
            const uint32_t m = mb + 32 * u + lane;
            jv[u] = m < mend ? __ldg(dvals + m) : 0xffffffffu;
            lo[u] = m < mend ? __ldg(rlo + m) : 0u;
            hi[u] = m < mend ? __ldg(rhi + m) : 0u;
        }
#pragma unroll
        for (int u = 0; u < PS_ROUNDS; ++u) {
            const bool has = jv[u] != 0xffffffffu;
            const int bx0 = (int)(lo[u] & 0xffffu) / BK_W, by0 = (int)(lo[u] >> 16) / BK_H;
            const int bx1 = (int)(hi[u] & 0xffffu) / BK_W, by1 = (int)(hi[u] >> 16) / BK_H;
            const uint32_t np = has ? (uint32_t)((bx1 - bx0 + 1) * (by1 - by0 + 1)) : 0u;
            uint32_t incl = np;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const uint32_t excl = incl - np;
            const uint32_t NP = __shfl_sync(0xffffffffu, incl, 31);
            int pp = 0;  // pair of the step's first piece (lanes agree); pairs with pieces come first
            for (uint32_t e0 = 0; e0 < NP; e0 += 32) {
                // piece starts of pairs pp+1 .. inside (e0, e0 + 32): one redux.or
                const int cand = pp + lane + 1;
                const uint32_t st = __shfl_sync(0xffffffffu, excl, cand & 31);
                const uint32_t d = st - e0;
                const uint32_t bit = (cand < 32 && st > e0 && d < 32u) ? (1u << d) : 0u;
                const uint32_t starts = __reduce_or_sync(0xffffffffu, bit);
                const int p = pp + __popc(starts & le);
                const uint32_t e = e0 + lane;
                const bool valid = e < NP;
                // the pair's data from its lane
                const uint32_t pj = __shfl_sync(0xffffffffu, jv[u], p & 31);
                const uint32_t plo = __shfl_sync(0xffffffffu, lo[u], p & 31);
                const uint32_t phi = __shfl_sync(0xffffffffu, hi[u], p & 31);
                const uint32_t pst = __shfl_sync(0xffffffffu, excl, p & 31);
                int bk = -1 - lane;  // invalid lanes: keys no valid lane has
                uint32_t gi = 0, lrw = 0;
                if (valid) {
                    const int v = (int)view_of(pj, g);
                    const int tx0 = (int)(plo & 0xffffu), ty0 = (int)(plo >> 16);
                    const int tx1 = (int)(phi & 0xffffu), ty1 = (int)(phi >> 16);
                    const int qbx0 = tx0 / BK_W, qby0 = ty0 / BK_H, qbx1 = tx1 / BK_W;
                    const uint32_t bw = (uint32_t)(qbx1 - qbx0 + 1);
                    const uint32_t o = e - pst;
                    const uint32_t orow = (o * s_rcp[bw]) >> 16;  // exact: o < 4096
                    const int bx = qbx0 + (int)(o - orow * bw), by = qby0 + (int)orow;
                    bk = v * g.NB + by * g.nbx + bx;
                    gi = pj - (uint32_t)v * (uint32_t)g.n_pad;
                    const int tx0b = bx * BK_W, ty0b = by * BK_H;
                    const int lx0 = max(tx0 - tx0b, 0), lx1 = min(tx1 - tx0b, BK_W - 1);
                    const int ly0 = max(ty0 - ty0b, 0), ly1 = min(ty1 - ty0b, BK_H - 1);
                    lrw = (uint32_t)(lx0 | (lx1 << 4) | (ly0 << 8) | (ly1 << 11));
                }
                const uint32_t peers = __match_any_sync(0xffffffffu, bk);
                const uint32_t pos = valid ? cur[bk] + __popc(peers & lt) : 0u;
                __syncwarp();
                if (valid) {
                    piece_gi[pos] = gi;
                    piece_lr[pos] = lrw;
                    if ((peers & lt) == 0) cur[bk] += __popc(peers);  // the bucket's lowest lane
                }
                __syncwarp();
                const int p31 = __shfl_sync(0xffffffffu, p, 31);
                const uint32_t nst = __shfl_sync(0xffffffffu, excl, (p31 + 1) & 31);
                pp = p31 + ((p31 + 1 < 32 && nst == e0 + 32) ? 1 : 0);
            }
        }
    }
}

// Emission, one WARP per emit tile (its pieces: whole (chunk, bucket) segments in m order,
// streamed from piece_gi / piece_lr; no sort, no block barriers):
//   pass 1  entry counts per bucket tile (2D difference array over the 16 x 8 tiles);
//   then    each tile's offset among the bucket's earlier emit tiles by decoupled look-back
//           (4 tiles per lane), base = ranges[gt].first + offset;
//   pass 2  rounds of 32 pieces: an entry's rank among the round's earlier pieces on its tile is
//           popc(R[row] & C[column] & lower lanes) (row / column coverage ballots), so each tile's
//           entries are written in m order.
constexpr int EW_WARPS = 4;  // independent emit workers per CTA
struct EwSmem {
    int diff[(BK_H + 1) * (BK_W + 1)];
    uint32_t base[BK_T];   // final position of each bucket tile's next entry
    uint32_t R[BK_H], C[BK_W];  // the round's pieces covering each bucket row / column
};

__global__ void __launch_bounds__(EW_WARPS * 32) k_emit(const uint32_t* __restrict__ piece_gi,
                                                        const uint32_t* __restrict__ piece_lr,
                                                        const uint4* __restrict__ plan,
                                                        const uint32_t* __restrict__ pbase,
                                                        const uint32_t* __restrict__ meta,
                                                        const uint32_t* __restrict__ Kd,
                                                        const uint2* __restrict__ ranges, BucketGeo g,
                                                        uint32_t* __restrict__ vals, uint32_t* lb, uint32_t* ticket,
                                                        DevFlags* fl) {
    __shared__ EwSmem sm[EW_WARPS];
    const int lane = threadIdx.x & 31;
    EwSmem& S = sm[threadIdx.x >> 5];
    if (visible_pairs(Kd) == 0) return;
    const uint32_t NE = meta[1];
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(ticket, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= NE) break;
        const uint4 pa = plan[2 * (size_t)t];
        const uint32_t b = pa.x, k = pa.y, s0 = pa.z, n = pa.w;
        const int v = (int)b / g.NB;
        const int bl = (int)b - v * g.NB;
        const int by = bl / g.nbx, bx = bl - by * g.nbx;
        const int tx0b = bx * BK_W, ty0b = by * BK_H;
        const uint32_t* __restrict__ lrp = piece_lr + pbase[b] + s0;
        const uint32_t* __restrict__ gip = piece_gi + pbase[b] + s0;
        for (int q = lane; q < (BK_H + 1) * (BK_W + 1); q += 32) S.diff[q] = 0;
        __syncwarp();
        // pass 1: entries per bucket tile
        for (uint32_t q0 = 0; q0 < n; q0 += 32 * 8) {  // 8 loads in flight per lane
            uint32_t lrv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t q = q0 + 32 * u + lane;
                lrv[u] = q < n ? __ldg(lrp + q) : 0xffffffffu;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t lr = lrv[u];
                if (lr == 0xffffffffu) continue;
                const int lx0 = lr & 15, lx1 = (lr >> 4) & 15, ly0 = (lr >> 8) & 7, ly1 = (lr >> 11) & 7;
                atomicAdd(&S.diff[ly0 * (BK_W + 1) + lx0], 1);
                atomicAdd(&S.diff[ly0 * (BK_W + 1) + lx1 + 1], -1);
                atomicAdd(&S.diff[(ly1 + 1) * (BK_W + 1) + lx0], -1);
                atomicAdd(&S.diff[(ly1 + 1) * (BK_W + 1) + lx1 + 1], 1);
            }
        }
        __syncwarp();
        if (lane < BK_H) {
            int run = 0;
            for (int x = 0; x < BK_W; ++x) { run += S.diff[lane * (BK_W + 1) + x]; S.diff[lane * (BK_W + 1) + x] = run; }
        }
        __syncwarp();
        if (lane < BK_W) {
            int run = 0;
            for (int y = 0; y < BK_H; ++y) { run += S.diff[y * (BK_W + 1) + lane]; S.diff[y * (BK_W + 1) + lane] = run; }
        }
        __syncwarp();
        // look-back: tile lt = lane + 32 i (4 per lane); publish all four first
        uint32_t cnt[BK_T / 32], prefix[BK_T / 32];
#pragma unroll
        for (int i = 0; i < BK_T / 32; ++i) {
            const int lt = lane + 32 * i, ly = lt / BK_W, lx = lt - ly * BK_W;
            cnt[i] = (uint32_t)S.diff[ly * (BK_W + 1) + lx];
            prefix[i] = 0;
            st_volatile_u32(lb + (size_t)t * BK_T + lt, (k == 0 ? LB_INC : LB_AGG) | cnt[i]);
        }
        if (k > 0) {
#pragma unroll
            for (int i = 0; i < BK_T / 32; ++i) {
                const int lt = lane + 32 * i;
                int64_t look = (int64_t)t - 1;
                long long spins = 0;
                for (;;) {
                    const uint32_t x = ld_volatile_u32(lb + (size_t)look * BK_T + lt);
                    const uint32_t f = x >> 30;
                    if (f == 0) {
                        if (++spins > SPIN_LIMIT) { raise_flag(fl, FLAG_TIMEOUT); break; }
                        continue;
                    }
                    prefix[i] += x & LB_MASK;
                    if (f == 2) break;
                    --look;
                }
                st_volatile_u32(lb + (size_t)t * BK_T + lt, LB_INC | (prefix[i] + cnt[i]));
            }
        }
#pragma unroll
        for (int i = 0; i < BK_T / 32; ++i) {
            const int lt = lane + 32 * i, ly = lt / BK_W, lx = lt - ly * BK_W;
            const int ty = ty0b + ly, tx = tx0b + lx;
            const uint32_t gt = (uint32_t)v * (uint32_t)g.T + (uint32_t)(ty * g.gx + tx);
            S.base[lt] = (tx < g.gx && ty < g.gy) ? __ldg(&ranges[gt].x) + prefix[i] : 0u;
        }
        __syncwarp();
        // pass 2: rounds of 32 pieces in m order (lane = piece).  A piece covers the bucket tiles
        // rows x columns of its rect, so the round's pieces covering tile (ly, lx) are
        // R[ly] & C[lx] with R[ly] = ballot(piece covers row ly), C[lx] = ballot(covers column lx):
        // 24 ballots give every entry's rank among the round's earlier pieces -- popc(R & C & lower
        // lanes) -- with no atomics and no per-entry synchronisation.
        uint32_t lr_n = lane < n ? __ldg(lrp + lane) : 0u, gi_n = lane < n ? __ldg(gip + lane) : 0u;
        for (uint32_t q0 = 0; q0 < n; q0 += 32) {
            const uint32_t q = q0 + lane;
            const bool has = q < n;
            const uint32_t lr = lr_n, gi = gi_n;
            lr_n = q + 32 < n ? __ldg(lrp + q + 32) : 0u;  // next round's pieces, in flight meanwhile
            gi_n = q + 32 < n ? __ldg(gip + q + 32) : 0u;
            const uint32_t lx0 = lr & 15, lx1 = (lr >> 4) & 15, ly0 = (lr >> 8) & 7, ly1 = (lr >> 11) & 7;
            const uint32_t rm = has ? ((2u << ly1) - 1u) & ~((1u << ly0) - 1u) : 0u;  // rows covered
            const uint32_t cm = has ? ((2u << lx1) - 1u) & ~((1u << lx0) - 1u) : 0u;  // columns covered
#pragma unroll
            for (int y = 0; y < BK_H; ++y) {
                const uint32_t r = __ballot_sync(0xffffffffu, (rm >> y) & 1u);
                if (lane == 0) S.R[y] = r;
            }
#pragma unroll
            for (int x = 0; x < BK_W; ++x) {
                const uint32_t c = __ballot_sync(0xffffffffu, (cm >> x) & 1u);
                if (lane == 0) S.C[x] = c;
            }
            __syncwarp();
            if (has) {  // (flattening the entries over the lanes measured no faster: 208 vs 202 us)
                for (uint32_t ly = ly0; ly <= ly1; ++ly) {
                    const uint32_t rr = S.R[ly] & lt_mask;
                    for (uint32_t lx = lx0; lx <= lx1; ++lx)
                        vals[S.base[ly * BK_W + lx] + __popc(rr & S.C[lx])] = gi;
                }
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < BK_T / 32; ++i) {  // the round's entries per tile
                const int lt = lane + 32 * i;
                S.base[lt] += __popc(S.R[lt / BK_W] & S.C[lt % BK_W]);
            }
            __syncwarp();
        }
    }
}

// ranges[gt] = view base + local start (view bases = exclusive scan of the <= 64 view
// totals); [0,0) for empty tiles and everywhere on capacity overflow (already flagged).  Every
// block of the calling grid takes a grid-stride slice of the tiles.
__device__ void ranges_slice(const uint32_t* __restrict__ counts, const uint32_t* __restrict__ lstart,
                             const uint32_t* __restrict__ view_tot, int n_views, uint32_t T, uint32_t cap,
                             const uint32_t* Kd, uint2* __restrict__ ranges, uint32_t* ohist) {
    __shared__ unsigned long long s_base[QUEEN_MAX_VIEWS + 1];
    __shared__ uint32_t s_oh[ORDER_BINS];
    if (threadIdx.x == 0) {
        unsigned long long r = 0;
        for (int q = 0; q < n_views; ++q) { s_base[q] = r; r += view_tot[q]; }
    }
    for (int q = threadIdx.x; q < ORDER_BINS; q += blockDim.x) s_oh[q] = 0u;
    __syncthreads();
    const bool overflow = Kd[2] != 0u;
    const uint64_t G = (uint64_t)n_views * T;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < G; g += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = counts[g];
        const unsigned long long st = s_base[g / T] + lstart[g], en = st + c;
        const uint2 r = (c && !overflow) ? make_uint2((uint32_t)(st < cap ? st : cap), (uint32_t)(en < cap ? en : cap))
                                         : make_uint2(0u, 0u);
        ranges[g] = r;
        if (ohist) atomicAdd(&s_oh[order_class(r)], 1u);  // the blend schedule's class counts
    }
    if (ohist) {
        __syncthreads();
        for (int q = threadIdx.x; q < ORDER_BINS; q += blockDim.x)
            if (s_oh[q]) atomicAdd(&ohist[q], s_oh[q]);
    }
}

__global__ void __launch_bounds__(256) k_ranges_finalize(const uint32_t* __restrict__ counts,
                                                         const uint32_t* __restrict__ lstart,
                                                         const uint32_t* __restrict__ view_tot, int n_views, uint32_t T,
                                                         uint32_t cap, const uint32_t* Kd, uint2* __restrict__ ranges) {
    ranges_slice(counts, lstart, view_tot, n_views, T, cap, Kd, ranges, nullptr);
}

// one launch zeroing the binning's per-batch state: tickets, digit histograms, the depth
// passes' look-back words (uint4 stores), the depth min/max and the key counts
__global__ void __launch_bounds__(256) k_bin_init(DevFlags* fl, uint32_t* hist, int hist_words, uint4* lb,
                                                  size_t lb_vec, uint32_t* dminmax, uint32_t* K, uint32_t* ocnt) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < 16) fl->tickets[t] = 0u;
    if (ocnt && t < 2 * ORDER_BINS) ocnt[t] = 0u;  // blend-schedule class counts | cursors
    if (t < 4) K[t] = 0u;
    if (t == 0) { dminmax[0] = 0xffffffffu; dminmax[1] = 0u; }
    for (size_t q = t; q < (size_t)hist_words; q += (size_t)gridDim.x * blockDim.x) hist[q] = 0u;
    for (size_t q = t; q < lb_vec; q += (size_t)gridDim.x * blockDim.x) lb[q] = make_uint4(0u, 0u, 0u, 0u);
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

template <int BITS, int MODE>
static int onesweep_grid() {
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_onesweep32<BITS, MODE>, Onesweep<BITS>::NT,
                                                      Onesweep<BITS>::SMEM);
        if (occ <= 0) occ = 1;
    }
    return occ * num_sms();
}

template <int BITS, int MODE>
static cudaError_t onesweep_attr() {
    return cudaFuncSetAttribute(k_onesweep32<BITS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)Onesweep<BITS>::SMEM);
}

static int emit_grid() {
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_emit, EW_WARPS * 32, 0);
        if (occ <= 0) occ = 1;
    }
    return occ * num_sms();
}

cudaError_t init_binning_attributes() {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_piece_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PC_MAX_SMEM)) ||
        (e = cudaFuncSetAttribute(k_piece_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PC_MAX_SMEM)))
        return e;
    if ((e = onesweep_attr<8, OS_KV>()) || (e = onesweep_attr<9, OS_KV>())) return e;
    return cudaFuncSetAttribute(k_slab_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(int) * BIN_MAX_SMEM_WORDS));
}

template <int BITS, int MODE>
static void onesweep(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout, const uint32_t* count,
                     uint32_t cap, int shift, int pshift, int ibits, const uint32_t* hist_excl, uint32_t* lb,
                     uint32_t* ticket, DevFlags* fl, cudaStream_t s, const uint32_t* triv = nullptr) {
    k_onesweep32<BITS, MODE><<<onesweep_grid<BITS, MODE>(), Onesweep<BITS>::NT, Onesweep<BITS>::SMEM, s>>>(
        kin, vin, kout, vout, count, cap, shift, pshift, ibits, hist_excl, lb, ticket, fl, triv);
}


cudaError_t launch_bin_sort(const queen_proj& proj, int n_views, int W, int H, queen_bins& bins, void* scratch,
                            const WsLayout& L, DevFlags* fl, cudaStream_t s, Prof* prof, bool* order_ready) {
    if (order_ready) *order_ready = false;
    const int gx = (W + 15) / 16, gy = (H + 15) / 16;
    const int64_t T = (int64_t)gx * gy;
    const int64_t count = (int64_t)n_views * proj.n_pad;
    const uint32_t cap = (uint32_t)bins.keys_cap;
    const BinPlan bp = bin_plan(proj.n_pad, n_views, W, H);
    unsigned char* ws = static_cast<unsigned char*>(scratch);
    uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist);  // [depth 4 | tile 4][MAX_BINS] counts, then excl
    uint32_t* hist_excl = hist + DEPTH_PASSES * MAX_BINS;
    uint32_t* depth_lb = reinterpret_cast<uint32_t*>(ws + L.depth_lb);
    uint32_t* dk[2] = {reinterpret_cast<uint32_t*>(ws + L.dkeys), reinterpret_cast<uint32_t*>(ws + L.dkeys_alt)};
    uint32_t* dv[2] = {reinterpret_cast<uint32_t*>(ws + L.dvals), reinterpret_cast<uint32_t*>(ws + L.dvals_alt)};
    uint32_t* tcounts = reinterpret_cast<uint32_t*>(ws + L.counts);  // per-tile totals | view-local starts
    uint32_t* lstart = tcounts + T * n_views;
    uint32_t* view_tot = reinterpret_cast<uint32_t*>(ws + L.view_tot);
    uint32_t* scount = reinterpret_cast<uint32_t*>(ws + L.slab_counts);
    uint32_t* svis = reinterpret_cast<uint32_t*>(ws + L.slab_vis);
    const int64_t os_elem_tiles = (count + OS_TILE - 1) / OS_TILE;
    uint32_t* Kd = bins.K;      // [0] = K entries
    uint32_t* Md = bins.K + 1;  // [1] = M visible pairs
    const int sms = num_sms();
    const size_t dplane = (size_t)(gx + 1) * (gy + 1);
    cudaError_t e;
    prof->begin(ST_COMPACT, s);
    uint32_t* dminmax = reinterpret_cast<uint32_t*>(ws + L.dminmax);
    // the blend schedule (class counts | cursors | tile permutation) in the workspace's order
    // region: built by k_slab_compact (counts, cursors) and k_piece_count (permutation)
    uint32_t* ocnt = reinterpret_cast<uint32_t*>(ws + L.order);
    {  // one launch for the per-batch state (was six memsets)
        const size_t lb_vec = (size_t)DEPTH_PASSES * MAX_BINS * (size_t)(os_elem_tiles + 1) / 4;
        const unsigned blocks = (unsigned)std::max<size_t>(1, std::min<size_t>((size_t)sms * 4, (lb_vec + 255) / 256));
        k_bin_init<<<blocks, 256, 0, s>>>(fl, hist, DEPTH_PASSES * MAX_BINS, reinterpret_cast<uint4*>(depth_lb), lb_vec,
                                          dminmax, bins.K, ocnt);
    }
    // ranges: view base + local start per tile (the emission writes entries at their final
    // positions); finalised inside k_slab_compact
    RangesArgs ra{tcounts, lstart, view_tot, n_views, (uint32_t)T, cap, Kd, reinterpret_cast<uint2*>(bins.ranges), ocnt};
    if (bp.slabs > 0) {
        k_slab_count<<<(unsigned)bp.slabs, SLAB_THREADS, sizeof(int) * dplane, s>>>(
            proj.tiles, reinterpret_cast<const short4*>(proj.rect), proj.depth, proj.n_pad, (int)bp.S, (int)bp.spv, gx, gy,
            scount, svis, dminmax);
        k_slab_sum<<<dim3((unsigned)((T + 255) / 256), (unsigned)n_views), 256, 0, s>>>(scount, (int)bp.spv, (int)T,
                                                                                        tcounts);
        k_view_scan_totals<<<n_views, 1024, 0, s>>>(tcounts, (int)T, lstart, view_tot, n_views, svis, (int)bp.slabs, cap,
                                                    Kd, fl, &fl->tickets[TK_VSCAN]);
        k_slab_compact<<<(unsigned)bp.slabs, SLAB_THREADS, 0, s>>>(proj.tiles, proj.depth, proj.n_pad, (int)bp.S,
                                                                  (int)bp.spv, svis, dminmax, dk[0], dv[0], hist,
                                                                  hist_excl, &fl->tickets[TK_COMPACT], ra);
    } else {
        if ((e = cudaMemsetAsync(tcounts, 0, sizeof(uint32_t) * 2 * T * n_views, s))) return e;
        if ((e = cudaMemsetAsync(view_tot, 0, sizeof(uint32_t) * n_views, s))) return e;
        k_totals<<<1, 1024, 0, s>>>(view_tot, n_views, svis, 0, cap, Kd, fl);
        k_hist_scan<<<1, 32 * DEPTH_PASSES, 0, s>>>(hist, hist_excl, DEPTH_PASSES, MAX_BINS);
        k_ranges_finalize<<<sms * 2, 256, 0, s>>>(ra.counts, ra.lstart, ra.view_tot, n_views, (uint32_t)T, cap, Kd,
                                                  ra.ranges);
    }
    prof->end(s, bp.slabs > 0 ? 5 : 4);
    // depth digits (LSD: least significant first) on the visible pairs
    prof->begin(ST_DEPTH_SORT, s);
    // depth keys are relative to the batch's smallest visible depth (order-preserving, and the
    // range of a scene's depths fits 27 bits unless it spans > 2^27 ulps): three 9-bit passes,
    // then bits 27..31, which is skipped (no copy; the bucket kernels read the previous buffer)
    // whenever that digit is 0 for every key.  (The digit histograms' exclusive scans were done
    // by k_slab_compact's last block.)
    int cur = 0;
    for (int p = 0; p < DEPTH_PASSES; ++p) {
        uint32_t* lbp = depth_lb + (size_t)p * MAX_BINS * (os_elem_tiles + 1);
        if (p < DEPTH_PASSES - 1)
            onesweep<9, OS_KV>(dk[cur], dv[cur], dk[cur ^ 1], dv[cur ^ 1], Md, (uint32_t)count, DEPTH_BITS * p, 0, 32,
                               hist_excl + p * MAX_BINS, lbp, &fl->tickets[TK_DEPTH + p], fl, s);
        else
            onesweep<8, OS_KV>(dk[cur], dv[cur], dk[cur ^ 1], dv[cur ^ 1], Md, (uint32_t)count, DEPTH_BITS * p, 0, 32,
                               hist_excl + p * MAX_BINS, lbp, &fl->tickets[TK_DEPTH + p], fl, s, hist + p * MAX_BINS);
        cur ^= 1;
    }
    prof->end(s, DEPTH_PASSES);
    prof->begin(ST_RANGES, s);  // (folded into k_slab_compact: kept as an empty stage)
    prof->end(s, 0);
    // pieces (pair, bucket) bucketed in depth order, then emitted tile by tile
    BucketGeo bg;
    bg.gx = gx;
    bg.gy = gy;
    bg.nbx = (gx + BK_W - 1) / BK_W;
    bg.nby = (gy + BK_H - 1) / BK_H;
    bg.NB = bg.nbx * bg.nby;
    bg.VNB = bg.NB * n_views;
    bg.T = (int)T;
    bg.n_pad = proj.n_pad;
    // ceil(2^64 / n_pad) (n_pad >= 4): floor(j / n_pad) = umulhi64(j, magic) for every j < 2^32
    bg.npad_magic = ~0ull / (unsigned long long)proj.n_pad + 1ull;
    uint32_t* pcnt = reinterpret_cast<uint32_t*>(ws + L.pcnt);
    uint32_t* ptotal = reinterpret_cast<uint32_t*>(ws + L.pbuck);
    uint32_t* pbase = ptotal + bg.VNB;
    uint32_t* ebase = pbase + bg.VNB;  // [VNB + 1]
    uint32_t* meta = ebase + bg.VNB + 1;
    uint32_t* emit_lb = reinterpret_cast<uint32_t*>(ws + L.emit_lb);
    uint4* plan = reinterpret_cast<uint4*>(ws + L.eplan);                      // [etiles][2]
    // chunk size: 2048 pairs, doubled while the dense per-(bucket, chunk) counts would exceed
    // ~4 M words (batches of many views: Immersive's 46 views x 40 buckets)
    bg.ch = QUEEN_PC_CH0;
    while (bg.ch < 8 * PC_CH && (int64_t)bg.VNB * ((count + bg.ch - 1) / bg.ch) > ((int64_t)QUEEN_PC_BUDGET << 20)) bg.ch *= 2;
    const int64_t chunks = (count + bg.ch - 1) / bg.ch;
    bg.CHS = (int)chunks;
    bg.em_e = proj.n_pad > (1 << 20) ? 128 : 256;  // measured: stress (3 M) 128, N3DV / Immersive 256
    const int64_t etiles = ((int64_t)cap + bg.em_e - 1) / bg.em_e + bg.VNB + 1;
    const size_t vsm = sizeof(uint32_t) * (size_t)bg.VNB;
    const uint32_t* dlast_in = dv[cur ^ 1];   // input of the last depth pass
    const uint32_t* dlast_out = dv[cur];      // its output (unless it was skipped)
    const uint32_t* triv = hist + (DEPTH_PASSES - 1) * MAX_BINS;
    // the depth-key buffers are free after the depth sort: the pairs' rects in m order
    uint32_t* rlo = dk[0];
    uint32_t* rhi = dk[1];
    const short4* r4 = reinterpret_cast<const short4*>(proj.rect);
    if (8 * (size_t)bg.VNB > PC_MAX_SMEM) return cudaErrorInvalidConfiguration;  // > 25600 buckets: not reachable (<= 64 4K views)
    prof->begin(ST_BUCKET, s);
    if (chunks > 0) {
        const OrderSched os{reinterpret_cast<const uint2*>(bins.ranges), ocnt + ORDER_BINS, ocnt + 2 * ORDER_BINS};
        k_piece_count<<<(unsigned)chunks, PC_THREADS, vsm, s>>>(dlast_in, dlast_out, triv, Kd, r4, bg, pcnt, rlo, rhi, os);
        if (order_ready) *order_ready = bp.slabs > 0;
        k_piece_colscan<<<(unsigned)((bg.VNB + 7) / 8), 256, 0, s>>>(pcnt, Kd, bg, ptotal, pbase, ebase, meta, Kd,
                                                                     &fl->tickets[TK_COLSCAN]);
        // warps per chunk: each holds VNB cursors in shared memory
        int wpc = (int)std::max<int64_t>(1, std::min<int64_t>(PS_MAX_WARPS, (int64_t)PC_MAX_SMEM / (4 * (int64_t)bg.VNB)));
        while (wpc > 1 && (bg.ch / wpc) % (32 * PS_ROUNDS)) --wpc;
        k_piece_scatter<<<(unsigned)chunks, 32 * wpc, (size_t)wpc * 4 * bg.VNB, s>>>(
            dlast_in, dlast_out, triv, Kd, rlo, rhi, bg, pcnt, pbase, bins.keys_alt, bins.keys);
    }
    prof->end(s, chunks > 0 ? 3 : 0);
    prof->begin(ST_EMIT, s);
    if (chunks > 0)
        k_emit_plan<<<(unsigned)((etiles + 255) / 256), 256, 0, s>>>(pcnt, ptotal, ebase, meta, Kd, bg, plan,
                                                                     emit_lb);
    if (chunks > 0)
        k_emit<<<(unsigned)std::min<int64_t>(emit_grid(), (etiles + EW_WARPS - 1) / EW_WARPS), EW_WARPS * 32, 0, s>>>(bins.keys_alt, bins.keys, plan, pbase, meta, Kd,
                                                     reinterpret_cast<const uint2*>(bins.ranges), bg, bins.vals,
                                                     emit_lb, &fl->tickets[TK_EMIT], fl);
    prof->end(s, chunks > 0 ? 2 : 0);
    bins.sorted_in_alt = 0;
    return cudaGetLastError();
}

}  // namespace queen
