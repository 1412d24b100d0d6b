// Internal definitions of libqueen (sm_100a).  Not part of the C-ABI.
//
// Arithmetic contract: this library is compiled with -fmad=false -prec-div=true
// -prec-sqrt=true -ftz=false, so every `a * b + c` below is two roundings and every
// fmaf() is one, exactly as DESIGN.md "Arithmetic contract" specifies.  That is what
// makes projection records, tile rects, keys and skip decisions bit-identical to the
// CPU oracle (which is written independently from the same text).
#pragma once
#include <cstdint>
#include <cstddef>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/queen.h"

namespace queen {

// sticky device flags (bit i <-> error class)
enum : uint32_t {
    FLAG_INDEX = 1u << 0,
    FLAG_LATENT_RANGE = 1u << 1,
    FLAG_CAPACITY = 1u << 2,
    FLAG_NONFINITE = 1u << 3,
    FLAG_TIMEOUT = 1u << 4,
};

struct DevFlags {
    uint32_t flags;
    uint32_t pad;
    unsigned long long info;     // largest key count requested
    uint32_t tickets[16];        // per-launch dynamic tile counters (sort passes, scan)
    uint32_t pad2[12];
};
static_assert(sizeof(DevFlags) == 128, "DevFlags layout");

constexpr int MAX_PASSES = 8;
constexpr int SORT_TILE = 4096;  // workspace-capacity granularity (keys / elements)
constexpr int REC_WORDS = 12;
#ifndef QUEEN_OS_THREADS
#define QUEEN_OS_THREADS 512
#endif
#ifndef QUEEN_OS_ITEMS
#define QUEEN_OS_ITEMS 8
#endif
constexpr int OS_THREADS = QUEEN_OS_THREADS, OS_ITEMS = QUEEN_OS_ITEMS;  // onesweep pass CTA shape
constexpr int OS_TILE = OS_THREADS * OS_ITEMS;         // keys per onesweep tile
constexpr int64_t MAX_KEYS = (1ll << 30) - 1;  // look-back packs 30-bit counts

struct CamBatch {
    queen_camera cam[QUEEN_MAX_VIEWS];
};

// Binning plan: an LSD radix sort on (tile, depth) whose depth
// digits run BEFORE duplication, on the visible (view, Gaussian) pairs, and whose
// tile digits run after it on the duplicated entries:
//   depth passes : 4 x 8 bits over the 31 depth bits of the M visible pairs
//   tile passes  : ceil(gbits / TILE_DIGIT_BITS) x (8 or 9) bits over the K entries
constexpr int DEPTH_PASSES = 4;    // 3 x 9-bit digits of (depth - min depth), + bits 27..31
constexpr int DEPTH_BITS = 9;
constexpr int MAX_BINS = 512;


// Binning counts (binning.cu K3a): each view's elements are cut into slabs of S consecutive
// indices; one CTA per slab keeps the view's tile grid in shared memory as a difference
// array, and one CTA per view sums the slabs' tile counts in shared memory, so a view's tile
// grid must fit in BIN_MAX_SMEM_WORDS words: views up to 4K (241 x 136) qualify; larger
// ones are rejected with QUEEN_ERR_SHAPE.
constexpr int BIN_MAX_SMEM_WORDS = 48 * 1024;
struct BinPlan {
    bool ok;
    int64_t S, spv, slabs;  // slab size, slabs per view, slabs in the batch
};
#ifndef QUEEN_SLABS_PER_VIEW
#define QUEEN_SLABS_PER_VIEW 32
#endif
inline BinPlan bin_plan(int64_t n_pad, int64_t n_views, int W, int H) {
    const int64_t gx = (W + 15) / 16, gy = (H + 15) / 16;
    BinPlan p{};
    p.ok = (gx + 1) * (gy + 1) <= BIN_MAX_SMEM_WORDS;
    // ~32 slabs per view (S depends on n_pad only, so a smaller batch never needs more
    // slab-count space than the workspace was carved for), multiples of 1024 in [2048, 65536].
    // (~592 slabs per batch whatever its view count -- for the few-view batches of a multi-GPU
    // rank -- measured slower: 3-view N3DV batch, compact 58 -> 65 us.)
    (void)n_views;
    int64_t S = (n_pad + QUEEN_SLABS_PER_VIEW - 1) / QUEEN_SLABS_PER_VIEW;
    S = (S + 1023) / 1024 * 1024;
    S = S < 2048 ? 2048 : (S > 65536 ? 65536 : S);
    p.S = S;
    p.spv = n_pad > 0 ? (n_pad + S - 1) / S : 0;
    p.slabs = p.spv * n_views;
    return p;
}

// Bucketed emission (binning.cu K4'/K5'): buckets of BK_W x BK_H tiles of one view; the
// depth-ordered pairs are counted and scattered in chunks of PC_CH (or more); emit tiles hold
// ~g.em_e pieces.
constexpr int PC_CH = 2048;
constexpr int BK_W = 16, BK_H = 8, BK_T = BK_W * BK_H;
// emit-tile size: pieces per tile, chosen per batch (binning.cu: 256, or 128 above 1 M
// Gaussians); EM_E_MIN sizes the workspace.  Measured emit: N3DV 2048 ->
// 289 us, 512 -> 233 us, 256 -> 187 us, 128 -> 199 us; stress 512 -> 11.75 ms, 256 -> 9.75, 128 -> 8.23
constexpr int EM_E_MIN = 128;
inline int64_t buckets_per_view(int W, int H) {
    const int64_t gx = (W + 15) / 16, gy = (H + 15) / 16;
    return ((gx + BK_W - 1) / BK_W) * ((gy + BK_H - 1) / BK_H);
}

// Blend schedule (raster.cu): tiles launched longest list first, by list length classes of
// 32 entries (ORDER_BINS classes, the last open-ended), so the grid's tail holds short tiles.
constexpr int ORDER_BINS = 64;
// list-length class of a tile's range (0 = the longest lists)
__device__ __forceinline__ int order_class(uint2 r) {
    const uint32_t c = (r.y - r.x) >> 5;
    return ORDER_BINS - 1 - (int)(c < (uint32_t)(ORDER_BINS - 1) ? c : (uint32_t)(ORDER_BINS - 1));
}

// Workspace carve-up (bytes, 256-aligned) for (n_pad, n_views, W, H, keys_cap).
struct WsLayout {
    // scratch (bin_sort)
    size_t flags, hist, dminmax, depth_lb, dkeys, dkeys_alt, dvals, dvals_alt, counts, view_tot, slab_counts,
        slab_vis, select, pcnt, pbuck, emit_lb, eplan, order, total_scratch;
    // render_views / render_mask buffers
    size_t rec, depth, tiles, rect, keys, keys_alt, vals, vals_alt, ranges, K, mask_tmp, total;
    int64_t key_tiles, elem_tiles, os_key_tiles, os_elem_tiles, T, elems;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline WsLayout ws_layout(int32_t n_pad, int32_t n_views, int32_t W, int32_t H, int64_t keys_cap) {
    WsLayout L{};
    int64_t gx = (W + 15) / 16, gy = (H + 15) / 16;
    L.T = gx * gy;
    L.elems = (int64_t)n_pad * n_views;
    L.key_tiles = (keys_cap + SORT_TILE - 1) / SORT_TILE;
    L.elem_tiles = (L.elems + SORT_TILE - 1) / SORT_TILE;
    L.os_key_tiles = (keys_cap + OS_TILE - 1) / OS_TILE;
    L.os_elem_tiles = (L.elems + OS_TILE - 1) / OS_TILE;
    size_t o = 0;
    L.flags = o; o += align256(sizeof(DevFlags));
    L.hist = o; o += align256(sizeof(uint32_t) * DEPTH_PASSES * MAX_BINS * 2);
    L.dminmax = o; o += align256(sizeof(uint32_t) * 2);
    L.depth_lb = o; o += align256(sizeof(uint32_t) * DEPTH_PASSES * MAX_BINS * (L.os_elem_tiles + 1));
    L.dkeys = o; o += align256(sizeof(uint32_t) * L.elems);
    L.dkeys_alt = o; o += align256(sizeof(uint32_t) * L.elems);
    L.dvals = o; o += align256(sizeof(uint32_t) * L.elems);
    L.dvals_alt = o; o += align256(sizeof(uint32_t) * L.elems);
    L.counts = o; o += align256(sizeof(uint32_t) * 2 * (size_t)n_views * L.T);  // counts | local starts
    L.view_tot = o; o += align256(sizeof(uint32_t) * (size_t)n_views);
    const BinPlan bp = bin_plan(n_pad, n_views, W, H);
    L.slab_counts = o; o += align256(sizeof(uint32_t) * (size_t)(bp.ok ? bp.slabs : 0) * L.T);
    L.slab_vis = o; o += align256(sizeof(uint32_t) * (size_t)(bp.slabs + 1));
    L.select = o; o += align256((size_t)n_pad);  // render_mask: per-Gaussian subset flags
    {
        const int64_t vnb = (int64_t)n_views * buckets_per_view(W, H);
        const int64_t chunks = (L.elems + PC_CH - 1) / PC_CH;
        L.pcnt = o; o += align256(sizeof(uint32_t) * (size_t)(chunks * vnb));  // pieces per (chunk, bucket)
        L.pbuck = o; o += align256(sizeof(uint32_t) * (size_t)(3 * vnb + 8));  // totals | bases | emit-tile bases | meta
        const int64_t etiles = (keys_cap + EM_E_MIN - 1) / EM_E_MIN + vnb + 1;
        L.emit_lb = o; o += align256(sizeof(uint32_t) * BK_T * (size_t)etiles);  // emit-tile look-back
        L.eplan = o; o += align256(sizeof(uint32_t) * 9 * (size_t)etiles);       // emit-tile plans + buckets
    }
    L.order = o; o += align256(sizeof(uint32_t) * (2 * ORDER_BINS + (size_t)n_views * L.T));  // blend tile order
    L.total_scratch = o;
    L.rec = o; o += align256(sizeof(float) * REC_WORDS * L.elems);
    L.depth = o; o += align256(sizeof(uint32_t) * L.elems);
    L.tiles = o; o += align256(sizeof(uint32_t) * L.elems);
    L.rect = o; o += align256(sizeof(int16_t) * 4 * L.elems);
    L.keys = o; o += align256(sizeof(uint32_t) * keys_cap);
    L.keys_alt = o; o += align256(sizeof(uint32_t) * keys_cap);
    L.vals = o; o += align256(sizeof(uint32_t) * keys_cap);
    L.vals_alt = o; o += align256(sizeof(uint32_t) * keys_cap);
    L.ranges = o; o += align256(sizeof(uint32_t) * 2 * L.T * n_views);
    L.K = o; o += align256(sizeof(uint32_t) * 4);
    L.mask_tmp = o; o += align256((size_t)n_views * W * H);  // render_mask: row-dilated marks
    L.total = o;
    return L;
}

// every scratch region of `need` fits in the corresponding region of `have`
inline bool scratch_fits(const WsLayout& need, const WsLayout& have) {
    const size_t WsLayout::*r[] = {&WsLayout::flags,      &WsLayout::hist,        &WsLayout::dminmax,
                                   &WsLayout::depth_lb,   &WsLayout::dkeys,
                                   &WsLayout::dkeys_alt,  &WsLayout::dvals,       &WsLayout::dvals_alt,
                                   &WsLayout::counts,     &WsLayout::view_tot,    &WsLayout::slab_counts,
                                   &WsLayout::slab_vis,   &WsLayout::select,      &WsLayout::pcnt,
                                   &WsLayout::pbuck,      &WsLayout::emit_lb,     &WsLayout::eplan,
                                   &WsLayout::order,
                                   &WsLayout::total_scratch};
    for (size_t q = 0; q + 1 < sizeof(r) / sizeof(r[0]); ++q)
        if (need.*r[q + 1] - need.*r[q] > have.*r[q + 1] - have.*r[q]) return false;
    return true;
}

// ---------------------------------------------------------------------------
// det_exp / det_log:
// only IEEE + - * / fmaf rintf fminf fmaxf and bit casts, so results are identical
// on any IEEE-754 binary32 implementation.  Used for s = exp(log s),
// o = sigmoid(logit) and the gate sigmoid.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float det_exp(float x) {
    const float L2E = __int_as_float(0x3fb8aa3b);
    const float LN2_HI = __int_as_float(0x3f317200);
    const float LN2_LO = __int_as_float(0x35bfbe8e);
    x = fminf(fmaxf(x, -87.0f), 88.0f);
    float k = rintf(x * L2E);
    float r = fmaf(-k, LN2_HI, x);
    r = fmaf(-k, LN2_LO, r);
    float p = 1.0f / 5040.0f;
    p = fmaf(p, r, 1.0f / 720.0f);
    p = fmaf(p, r, 1.0f / 120.0f);
    p = fmaf(p, r, 1.0f / 24.0f);
    p = fmaf(p, r, 1.0f / 6.0f);
    p = fmaf(p, r, 0.5f);
    p = fmaf(p, r, 1.0f);
    p = fmaf(p, r, 1.0f);
    return p * __int_as_float((int)(k + 127.0f) << 23);
}

__device__ __forceinline__ float det_log(float y) {
    const float LN2_HI = __int_as_float(0x3f317200);
    const float LN2_LO = __int_as_float(0x35bfbe8e);
    uint32_t b = __float_as_uint(y);
    int e = (int)((b >> 23) & 255u) - 127;
    float m = __uint_as_float((b & 0x7fffffu) | 0x3f800000u);
    if (m > 1.41421356f) { m = m * 0.5f; e += 1; }
    float f = m - 1.0f;
    float s = f / (2.0f + f);
    float z = s * s;
    float R = fmaf(z, 2.0f / 9.0f, 2.0f / 7.0f);
    R = fmaf(z, R, 2.0f / 5.0f);
    R = fmaf(z, R, 2.0f / 3.0f);
    R = z * R;
    float hfsq = (0.5f * f) * f;
    float lnm = f - (hfsq - s * (hfsq + R));
    float ef = (float)e;
    return fmaf(ef, LN2_HI, fmaf(ef, LN2_LO, lnm));
}

__device__ __forceinline__ void raise_flag(DevFlags* fl, uint32_t bit) { atomicOr(&fl->flags, bit); }

// Can the record's alpha >= 1/255 region {p2 >= T2} reach a pixel centre of [x0,x1] x [y0,y1]?
// Conservative (false positives only cost time): p2 is a concave quadratic in (x, y), so its
// maximum over the rectangle is 0 if the centre (u, v) lies inside, else it sits on an edge,
// at the edge's 1D maximiser clamped to the edge.  The maximum is compared with T2 minus a
// slack of 1e-5 of the quadratic's magnitude over the bounding box (>> the few-ulp rounding
// of either evaluation).  Approximate division only moves the maximiser slightly, which
// lowers the edge value by a second-order amount (covered by the slack).
__device__ __forceinline__ bool touches(const float4& a, const float4& q, float x0, float x1, float y0, float y1) {
    if (a.x + a.z < x0 || a.x - a.z > x1 || a.y + a.w < y0 || a.y - a.w > y1) return false;
    if (a.x >= x0 && a.x <= x1 && a.y >= y0 && a.y <= y1) return true;
    const float A = q.x, B = q.y, C = q.z;
    const float iA = __fdividef(-0.5f * B, A), iC = __fdividef(-0.5f * B, C);
    const float dxl = a.x - x1, dxh = a.x - x0, dyl = a.y - y1, dyh = a.y - y0;
    float best = -INFINITY;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const float dy = e ? dyl : dyh;  // edge y = y0 (dy = v - y0) or y = y1
        const float dx = fminf(fmaxf(iA * dy, dxl), dxh);
        best = fmaxf(best, fmaf(A * dx, dx, fmaf(C * dy, dy, B * dx * dy)));
        const float ex = e ? dxl : dxh;  // edge x = x0 or x = x1
        const float ey = fminf(fmaxf(iC * ex, dyl), dyh);
        best = fmaxf(best, fmaf(A * ex, ex, fmaf(C * ey, ey, B * ex * ey)));
    }
    const float S = fabsf(A) * a.z * a.z + fabsf(B) * a.z * a.w + fabsf(C) * a.w * a.w;
    return best >= q.w - (1e-5f * S + 1e-6f);
}


// Stage profiler: CUDA events recorded on the launching stream at stage boundaries
// (enabled by queen_profile_enable; used by bench.py for per-kernel durations).
enum Stage { ST_APPLY = 0, ST_PROJECT, ST_COMPACT, ST_DEPTH_SORT, ST_BUCKET, ST_EMIT, ST_RANGES, ST_BLEND, ST_ENTROPY, ST_BLEND_ORDER, ST_COUNT };
struct Prof {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    struct Pending { int stage; size_t e0, e1; int launches; };
    std::vector<Pending> pending;
    double ms[ST_COUNT] = {0};
    long long launches[ST_COUNT] = {0};
    size_t open_ev = 0;
    int open_stage = -1;
    cudaEvent_t ev() {
        if (used == pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        return pool[used++];
    }
    // inside a stream capture the record must be an EXTERNAL event-record node, so every graph
    // replay re-records it (a plain record would only become a capture-internal dependency)
    static void record(cudaEvent_t e, cudaStream_t s) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cs);
        if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
        else cudaEventRecord(e, s);
    }
    // consecutive stages share their boundary event: begin() reuses the previous end() event
    // when nothing was profiled in between (halves the events, e.g. the nodes in a graph)
    // (a frame starts at the entropy decode, or at apply for uncoded packets: the chain breaks
    // there, so work enqueued between frames is never attributed to a stage)
    size_t last_end = SIZE_MAX;
    cudaStream_t last_stream = nullptr;
    int last_stage = -1;
    void begin(int stage, cudaStream_t s) {
        if (!on) return;
        const bool frame_start = stage == ST_ENTROPY || (stage == ST_APPLY && last_stage != ST_ENTROPY);
        if (!frame_start && last_end != SIZE_MAX && last_stream == s) {
            open_ev = last_end;
        } else {
            open_ev = used;
            record(ev(), s);
        }
        open_stage = stage;
    }
    void end(cudaStream_t s, int n_launches = 1) {
        if (!on || open_stage < 0) return;
        size_t e1 = used;
        record(ev(), s);
        pending.push_back({open_stage, open_ev, e1, n_launches});
        last_stage = open_stage;
        open_stage = -1;
        last_end = e1;
        last_stream = s;
    }
    void reset_chain() {
        last_end = SIZE_MAX;
        last_stage = -1;
    }
};

// host-side launchers (defined in the .cu files)
cudaError_t launch_decode_apply(const queen_packet& p, float* planes, float* resid_out, int8_t* q_out,
                                bool apply_attrs, bool apply_pos, DevFlags* fl, cudaStream_t s);
cudaError_t launch_gate_compact(const queen_packet& p, uint32_t* idx_out, float* val_out, int32_t* k_out,
                                void* scratch, DevFlags* fl, cudaStream_t s);
cudaError_t launch_coo_copy(const queen_packet& p, uint32_t* idx_out, float* val_out, int32_t* k_out, DevFlags* fl,
                            cudaStream_t s);
cudaError_t launch_project(const float* planes, int n, int n_pad, int deg, const CamBatch& cams, int n_views,
                           float* rec, uint32_t* depth, uint32_t* tiles, int16_t* rect, const uint8_t* select,
                           DevFlags* fl, cudaStream_t s);
cudaError_t launch_set_sh_rest(float* planes, int n, int n_pad, int deg, const int8_t* latents, int L,
                               const float* decoder, DevFlags* fl, cudaStream_t s);
// order_ready (optional out): true when the binning also wrote the blend's tile schedule into
// the workspace's order region (ws + L.order + 2 ORDER_BINS), for launch_rasterize's order_pre
cudaError_t launch_bin_sort(const queen_proj& proj, int n_views, int W, int H, queen_bins& bins, void* scratch,
                            const WsLayout& L, DevFlags* fl, cudaStream_t s, Prof* prof, bool* order_ready = nullptr);
enum : int { OUT_F32 = 0, OUT_MASK = 1, OUT_RGB8 = 2, OUT_F16 = 3, OUT_RGB10 = 4 };  // k_blend epilogues
#ifndef QUEEN_BLEND_TSUB
#define QUEEN_BLEND_TSUB 1  // blend transmittance T' = T - aT (aT = alpha T is formed anyway) instead of T (1 - alpha)
#endif
cudaError_t launch_rasterize(const float* rec, int n_pad, const uint32_t* ranges, const uint32_t* vals, int n_views,
                             int W, int H, float bg0, float bg1, float bg2, float* rgb_out, float* T_out,
                             uint8_t* out8, int out_mode, float mask_thresh, uint32_t* order_ws, cudaStream_t s,
                             int* n_launch = nullptr, Prof* prof = nullptr, int opts = 0,
                             const uint32_t* order_pre = nullptr);
// blend schedule: *order = longest-list-first permutation of the blocks gt tiles (in order_ws),
// or nullptr (grid order) when there is no scratch
cudaError_t launch_tile_order(const uint32_t* ranges, int64_t blocks, uint32_t* order_ws, cudaStream_t s,
                              const uint32_t** order, int opts = 0);
cudaError_t launch_select(const uint32_t* idx, int k, const int32_t* k_dev, int n, int n_pad, uint8_t* select,
                          DevFlags* fl, cudaStream_t s);
cudaError_t launch_dilate(uint8_t* marks, uint8_t* tmp, int n_views, int W, int H, int d, cudaStream_t s);
cudaError_t launch_blend_bwd(const float* rec, int n_pad, const uint32_t* ranges, const uint32_t* vals, int n_views,
                             int W, int H, float bg0, float bg1, float bg2, const float* gout, float* grec,
                             uint32_t* order_ws, cudaStream_t s);
cudaError_t launch_project_bwd(const float* planes, int n, int n_pad, int deg, const CamBatch& cams, int n_views,
                               const float* grec, float* gpl, cudaStream_t s);
cudaError_t launch_decode_bwd(const queen_packet& pk, const float* gA, float* gdec, float* glat, float* gla, float* gpre,
                              float* scratch, size_t scratch_floats, cudaStream_t s);
cudaError_t launch_densify(const float* src, int n_old, int np_src, const uint32_t* rem, int n_rem, const void* add,
                           int n_add, int P, float* dst, int np_dst, DevFlags* fl, cudaStream_t s);
cudaError_t launch_blend_counts(const float* rec, int n_pad, const uint32_t* ranges, const uint32_t* vals, int n_views,
                                int W, int H, long long* evaluated, long long* composited, cudaStream_t s);
cudaError_t init_kernel_attributes();

}  // namespace queen
