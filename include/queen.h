/*
 * queen.h -- C-ABI of libqueen: QUEEN's per-frame decode -> apply -> 3D-GS splat
 * hot path (arXiv 2412.04469), hand-written CUDA for sm_100a (B200).
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * R#n = DESIGN.md reading #n (where the paper is silent).
 *
 * Conventions shared by every call
 * ---------------------------------
 *  - Every function is extern "C", never throws, and returns a queen_status.
 *  - Pointers named *_dev, and every array member of the structs below, are DEVICE
 *    pointers on the ctx's device; camera arrays and queen_* structs themselves are
 *    HOST memory, read during the call only (cameras are copied into kernel
 *    parameters), so they may be freed as soon as the call returns.
 *  - All device buffers are caller-owned (torch tensors in the Python binding):
 *    contiguous, 16-byte aligned, n_pad % 4 == 0.  The library allocates NO device
 *    memory; its scratch lives in the caller-provided workspace (queen_set_workspace).
 *  - `stream` is a cudaStream_t passed as void*.  Calls only ENQUEUE work on it and
 *    return; nothing synchronises except queen_check.  Every call is capturable in a
 *    CUDA graph.
 *  - Host-detectable errors (null pointer, bad shape, bad degree, ...) are returned
 *    immediately and nothing is enqueued.  Device-detectable errors (bad COO index,
 *    latent out of range, key-capacity overflow, non-finite Gaussian) set sticky
 *    flags in the workspace that queen_check reports.
 *  - A queen_ctx is bound to one device and is not thread-safe.
 */
#ifndef QUEEN_H
#define QUEEN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t queen_status;
enum {
    QUEEN_OK = 0,
    QUEEN_ERR_INVALID_ARG = -1,   /* null pointer, bad enum, degree not in [0,3], ...        */
    QUEEN_ERR_SHAPE = -2,         /* n > n_pad, n_pad % 4, latent dims, view sizes differ   */
    QUEEN_ERR_INDEX = -3,         /* COO index >= n or not strictly increasing */
    QUEEN_ERR_LATENT_RANGE = -4,  /* rounded latent outside [-127, 127] (R#4)               */
    QUEEN_ERR_CAPACITY = -5,      /* keys needed > keys_cap; queen_check's info = keys needed */
    QUEEN_ERR_CUDA = -6,          /* a CUDA runtime call failed (see queen_last_error)      */
    QUEEN_ERR_TIMEOUT = -7,       /* a look-back spin exceeded its bound (should never fire) */
    QUEEN_WARN_NONFINITE = 1      /* a Gaussian had a non-finite attribute and was culled   */
};

enum { QUEEN_LAT_INT8 = 0, QUEEN_LAT_F32 = 1 };                 /* latent_kind */
enum { QUEEN_POS_COO = 0, QUEEN_POS_GATES = 1, QUEEN_POS_NONE = 2 }; /* pos_kind */
enum { QUEEN_MAX_VIEWS = 64, QUEEN_TILE = 16 };

typedef struct queen_ctx queen_ctx;

/* Gaussian attributes A = {p, q, s, o, h}, fp32 SoA,
 * planes[P][n_pad], P = 11 + 3B, B = (sh_degree+1)^2:
 *   rows 0-2 position xyz | 3-6 raw quaternion wxyz | 7-9 log-scale |
 *   10 opacity logit | 11 + 3b + ch SH coefficient b, channel ch.
 * Raw (pre-activation) storage: residuals add to raw values (R#1).  Columns
 * i >= n are padding and are never read or written. */
typedef struct {
    int32_t n, n_pad, sh_degree;
    float* planes;
} queen_gaussians;

/* One frame's residual packet R_t (Eq. 4).
 * Non-position categories c = (rot, scale, opacity, sh_dc, sh_rest) (R#2):
 *   M_c = (4, 3, 1, 3, 3(B-1)) residual rows, L_c = lat_dim[c] latent dims in [0,16]
 *   (0 = category absent; sh_rest must be 0 at degree 0).
 *   latents:  [sum L_c][n_pad] category-major, int8 (QUEEN_LAT_INT8, wire form) or
 *             fp32 trainer-state l_hat (QUEEN_LAT_F32), rounded half away from zero
 *             in-kernel (R#5).
 *   decoders: concatenation of row-major D_c (M_c x L_c), fp32 (Eq. 5).
 * Position:
 *   QUEEN_POS_COO:   pos_idx[k] strictly increasing u32, pos_val[3][k] fp32 (row stride k).
 *                    If k_dev != NULL the live count is min(*k_dev, k) read on the device
 *                    (packets broadcast over NCCL) and k is the capacity.
 *   QUEEN_POS_GATES: trainer state: log_alpha[n_pad], pos_pregate[3][n_pad] and the
 *                    hard-concrete hyperparameters (tau, gamma0, gamma1);
 *                    mask = log_alpha > tau ln(-gamma0/gamma1) (R#6).
 *   QUEEN_POS_NONE:  no position residual. */
typedef struct {
    int32_t n, n_pad, sh_degree;
    int32_t lat_dim[5];
    int32_t latent_kind;
    const void* latents;
    const float* decoders;
    int32_t pos_kind;
    int32_t k;
    const int32_t* k_dev;
    const uint32_t* pos_idx;
    const float* pos_val;
    const float* log_alpha;
    const float* pos_pregate;
    float tau, gamma0, gamma1;
} queen_packet;

/* Pinhole camera (intrinsics K, viewing transform W).  x_c = R p + t.
 * C = camera centre (-R^T t), limx/limy = 1.3 * tan(half FoV) (R#11), near_z = 0.2.
 * Pixel k is sampled at coordinate k (R#12).  96 bytes. */
typedef struct {
    float fx, fy, cx, cy;
    float R[9];
    float t[3];
    float C[3];
    float limx, limy, near_z;
    int32_t width, height;
} queen_camera;

/* Per-view projected records, each [n_views][n_pad]:
 *   rec   [..][12] fp32 = u, v, hx, hy | A2, B2, C2, T2 | o, r, g, b
 *         (A2,B2,C2 base-2 conic, T2 = log2(1/(255 o)); hx, hy = 1.0001 sqrt(2 ln(255 o) S'_xx|yy),
 *          the bounding box of the alpha >= 1/255 ellipse (R#13); all zero if culled)
 *   depth u32 = bits(z_c) (z_c > 0)          tiles u32 = #16x16 tiles touched
 *   rect  int16[4] = tx0, ty0, tx1, ty1 of [u +- ceil(hx)] x [v +- ceil(hy)] (inclusive) */
typedef struct {
    int32_t n_pad;
    float* rec;
    uint32_t* depth;
    uint32_t* tiles;
    int16_t* rect;
} queen_proj;

/* Binning buffers for one batch of equally-sized views (gt = view*T + tile, T = gx*gy).
 * The entries are the (16x16 tile, Gaussian) pairs, sorted by the composite key
 * (gt << 31 | depth bits) and then Gaussian index:
 *   vals (+ vals_alt ping-pong) [keys_cap] u32: the Gaussian index of each sorted entry
 *            (the entry's full sort key is (gt << 31) | proj.depth[view][val], gt = the
 *            range holding it); keys / keys_alt [keys_cap] u32: sort scratch
 *   ranges[n_views*T][2] u32  [first, last+1) of gt in the sorted entries, [0,0) if empty
 *   K (device u32[4])         [0] = entries K of the batch (0 if K > keys_cap: QUEEN_ERR_CAPACITY,
 *                             no entries, all ranges [0,0)), [1] = visible (view, Gaussian) pairs,
 *                             [2] = 1 on capacity overflow, [3] = pieces (visible pair x 16x8-tile
 *                             bucket) of the bucketed emission
 *   sorted_in_alt             OUT (host): 1 if the sorted result is in vals_alt (always 0: the
 *                             emission writes vals; keys / keys_alt / vals_alt are scratch) */
typedef struct {
    int64_t keys_cap;
    uint32_t* keys;
    uint32_t* keys_alt;
    uint32_t* vals;
    uint32_t* vals_alt;
    uint32_t* ranges;
    uint32_t* K;
    int32_t sorted_in_alt;
} queen_bins;

/* ---- context / workspace ------------------------------------------------ */
queen_status queen_create(int device, queen_ctx** out);
void queen_destroy(queen_ctx* ctx);
const char* queen_last_error(const queen_ctx* ctx);
const char* queen_version(void);

/* Bytes of device workspace for up to (n_pad, n_views <= QUEEN_MAX_VIEWS, width x
 * height, keys_cap < 2^30) -- covers queen_bin_sort's scratch and, for
 * queen_render_views, the proj / bins buffers it carves. */
queen_status queen_workspace_size(int32_t n_pad, int32_t n_views, int32_t width, int32_t height,
                                  int64_t keys_cap, size_t* bytes);
/* Hands the ctx a caller-owned device buffer (>= queen_workspace_size bytes, 256-B
 * aligned) and the shape it was sized for.  Zeroes the sticky flags (stream 0 order). */
queen_status queen_set_workspace(queen_ctx* ctx, void* dev_ptr, size_t bytes, int32_t n_pad, int32_t n_views,
                                 int32_t width, int32_t height, int64_t keys_cap);
/* Synchronises `stream`, returns the first sticky device error (or
 * QUEEN_WARN_NONFINITE, or QUEEN_OK) and clears the flags.  info_out (nullable)
 * receives the largest key count requested (for QUEEN_ERR_CAPACITY). */
queen_status queen_check(queen_ctx* ctx, void* stream, int64_t* info_out);

/* ---- the hot path ---------------------------------------------------------
 * queen_decode_residuals: UNFUSED decode (the test surface).  P:289-298, Eq. 5.
 *   resid_out  (nullable) fp32 [sum M_c][n_pad]: r_c = D_c float(l_c), row order =
 *              plane order 3.. (fmaf chain ascending k from +0, R#7)
 *   q_out      (nullable) int8 [sum L_c][n_pad]: rounded latents (a copy for INT8)
 *   coo_idx_out/coo_val_out/k_out (nullable together) u32 [n], fp32 [3][n] (row
 *              stride n), device int32: the position COO (gates -> mask -> ascending
 *              compaction, dp = g l_p; or a validated copy of the input COO). */
queen_status queen_decode_residuals(queen_ctx* ctx, const queen_packet* pkt, float* resid_out, int8_t* q_out,
                                    uint32_t* coo_idx_out, float* coo_val_out, int32_t* k_out, void* stream);
/* queen_apply_frame: FUSED a1-a5: A_{t-1} -> A_t in place (Eq. 4):
 * non-position planes += D_c float(round(l_c)); positions += COO / gated residual. */
queen_status queen_apply_frame(queen_ctx* ctx, queen_gaussians* scene, const queen_packet* pkt, void* stream);

/* queen_set_sh_rest: first-frame quantisation ("First-frame Quantization": only
 * frame 0's high-frequency SH coefficients, DC excluded, are learnably quantised).  Decodes them
 * ONCE and WRITES them (not added) into the scene:
 *   planes[14 + m][i] = sum_{k<L} decoder[m][k] * (float)latents[k][i]   (fmaf chain over
 *   ascending k from +0.0f, DESIGN R7), m = 3 (b - 1) + ch, b = 1 .. B-1, for i < n.
 * latents: device int8 [L][n_pad] (e.g. decoded by queen_entropy_decode); decoder: device fp32
 * row-major [3(B-1)][L]; scene->sh_degree 1..3; L in 1..16.  Other planes and columns >= n are
 * untouched.  Enqueue-only; no device-detectable errors. */
queen_status queen_set_sh_rest(queen_ctx* ctx, queen_gaussians* scene, const int8_t* latents, int32_t L,
                               const float* decoder, void* stream);
/* queen_project: a6-a7 for n_views cameras (Eq. 1 + SH colour).
 * `cams` is a HOST array of n_views cameras.  out arrays hold [n_views][n_pad]. */
queen_status queen_project(queen_ctx* ctx, const queen_gaussians* scene, const queen_camera* cams, int32_t n_views,
                           queen_proj* out, void* stream);
/* queen_bin_sort: a8-a11 for a batch of equally-sized views: the entries (gt, depth,
 * index) of every visible (view, Gaussian) x overlapped tile, ordered by gt then depth
 * then index (LSD onesweep radix sort on (gt, depth)), plus tile ranges.  Uses the
 * workspace scratch.  Outputs bit-exact.  The sorted index list is
 * bins->vals (or vals_alt when bins->sorted_in_alt is set on return); entry e belongs to
 * the gt whose range holds e.  keys / keys_alt are scratch (their content is unspecified on
 * return).  Views whose (ceil(W/16)+1)(ceil(H/16)+1) tile grid exceeds 48K words
 * (larger than 4K) are rejected with QUEEN_ERR_SHAPE. */
queen_status queen_bin_sort(queen_ctx* ctx, const queen_proj* proj, const queen_camera* cams, int32_t n_views,
                            queen_bins* bins, void* stream);
/* queen_rasterize: a12, Eq. 2: per pixel front-to-back over its tile's
 * range; skip a < 1/255 (p2 < T2), a = min(0.99, o 2^p2), stop after T < 1e-4.
 * rgb_out fp32 [n_views][3][H][W] = C + T bg;  T_out (nullable) fp32 [n_views][H][W].
 * When the context's workspace covers n_views x tiles, its scratch holds the blend schedule
 * (tiles launched longest list first; also used by queen_render_mask and
 * queen_rasterize_backward); otherwise tiles run in grid order.  Output is identical. */
queen_status queen_rasterize(queen_ctx* ctx, const queen_proj* proj, const queen_bins* bins, const queen_camera* cams,
                             int32_t n_views, const float bg[3], float* rgb_out, float* T_out, void* stream);
/* queen_render_views: project + bin_sort + rasterize with proj/bins carved from the
 * workspace (sized for >= these n_views/width/height/n_pad). */
queen_status queen_render_views(queen_ctx* ctx, const queen_gaussians* scene, const queen_camera* cams,
                                int32_t n_views, const float bg[3], float* rgb_out, float* T_out, void* stream);

/* Display-format variants (the streaming viewer's output): identical compositing, then
 * rgb8_out u8 [n_views][3][H][W] = round-half-even(clamp(C + T bg, 0, 1) * 255) in fp32;
 * T_out as above (nullable). */
queen_status queen_rasterize_rgb8(queen_ctx* ctx, const queen_proj* proj, const queen_bins* bins,
                                  const queen_camera* cams, int32_t n_views, const float bg[3], uint8_t* rgb8_out,
                                  float* T_out, void* stream);
queen_status queen_render_views_rgb8(queen_ctx* ctx, const queen_gaussians* scene, const queen_camera* cams,
                                     int32_t n_views, const float bg[3], uint8_t* rgb8_out, float* T_out, void* stream);
/* Half-precision variants (the streaming output that keeps the 2e-3 RGB bar: binary16 is within
 * 2^-11 of any value in [0, 1]): f16_out IEEE binary16 [n_views][3][H][W] = the fp32 output value
 * C + T bg rounded to nearest even (unclamped); T_out as above (nullable). */
queen_status queen_rasterize_f16(queen_ctx* ctx, const queen_proj* proj, const queen_bins* bins,
                                 const queen_camera* cams, int32_t n_views, const float bg[3], uint16_t* f16_out,
                                 float* T_out, void* stream);
queen_status queen_render_views_f16(queen_ctx* ctx, const queen_gaussians* scene, const queen_camera* cams,
                                    int32_t n_views, const float bg[3], uint16_t* f16_out, float* T_out, void* stream);
/* Packed 10-bit display variants (R10G10B10A2, the compact streaming output that keeps the 2e-3
 * RGB bar: 1/2 LSB = 4.9e-4): rgb10_out u32 [n_views][H][W], one word per pixel,
 * r | g << 10 | b << 20 | 3 << 30 with each channel round-half-even(clamp(C + T bg, 0, 1) * 1023)
 * in fp32 -- 4 bytes per pixel vs 6 for binary16 planar; T_out as above (nullable). */
queen_status queen_rasterize_rgb10(queen_ctx* ctx, const queen_proj* proj, const queen_bins* bins,
                                   const queen_camera* cams, int32_t n_views, const float bg[3], uint32_t* rgb10_out,
                                   float* T_out, void* stream);
queen_status queen_render_views_rgb10(queen_ctx* ctx, const queen_gaussians* scene, const queen_camera* cams,
                                      int32_t n_views, const float bg[3], uint32_t* rgb10_out, float* T_out,
                                      void* stream);

/* Debug / evidence: per-view blend work counters (evaluated and composited
 * (pixel, Gaussian) pairs, int64 device arrays [n_views]); same semantics as the
 * rasterizer, used only to compute the blend roofline. */
queen_status queen_blend_counts(queen_ctx* ctx, const queen_proj* proj, const queen_bins* bins,
                                const queen_camera* cams, int32_t n_views, int64_t* evaluated, int64_t* composited,
                                void* stream);

/* ---- NEXT #1: entropy-coded latents ----------
 * queen_entropy_encode (HOST, producer side): codes one category's latent matrix
 *   latents[L][n_pad] int8 (host memory; columns >= n ignored), flattened row-major,
 *   into the chunked 32-way interleaved rANS "QANS" stream written to `out` (host, capacity
 *   bytes).  *bytes = stream size; QUEEN_ERR_SHAPE if capacity is too small (nothing written).
 * queen_entropy_decode (DEVICE): decodes such a stream (device memory, stream_bytes long) back
 *   into latents_out[L][n_pad] int8 (device; columns >= n untouched), one warp per 8192-symbol
 *   chunk.  A stream too small for the header and chunk tables that (L, n) imply returns
 *   QUEEN_ERR_SHAPE.  A corrupt stream, one that does not match (L, n), or a chunk whose words
 *   lie outside stream_bytes sets QUEEN_ERR_INDEX (sticky; the mismatched category or chunk
 *   writes nothing, and no read or write leaves the stream or latents_out). */
queen_status queen_entropy_encode(const int8_t* latents, int32_t L, int32_t n, int32_t n_pad, void* out,
                                  size_t capacity, size_t* bytes);
queen_status queen_entropy_decode(queen_ctx* ctx, const void* stream_dev, int64_t stream_bytes, int32_t L, int32_t n,
                                  int32_t n_pad, int8_t* latents_out, void* stream);
/* queen_entropy_decode_frame: all five categories of a frame in ONE launch.  streams_dev
 * (HOST array of 5 device pointers, NULL where lat_dim[c] = 0), stream_bytes[5] (host; each
 * stream's size, the packet's ans_bytes), lat_dim[5] (host); output latents_out[sum L][n_pad]
 * int8 in category-major row order (the queen_packet layout).  Errors as queen_entropy_decode. */
queen_status queen_entropy_decode_frame(queen_ctx* ctx, const void* const* streams_dev, const int64_t* stream_bytes,
                                        const int32_t* lat_dim, int32_t n, int32_t n_pad, int8_t* latents_out,
                                        void* stream);

/* ---- NEXT #4: backward rasterizer (P:239-251 trains through Eq. 1-2) -----------------------
 * Gradients of L with respect to the inputs of the forward, holding its discrete decisions
 * (skip test, 0.99 clamp, composite-then-stop, culls, Jacobian clamp, max(0, .) on colour) at
 * the values the forward took (the derivative of the piece the input lies in).
 * queen_rasterize_backward: dL_drgb device fp32 [n_views][3][H][W] (gradient of L w.r.t. the
 *   queen_rasterize output C + T bg) -> grad_rec device fp32 [n_views][n_pad][9], per record:
 *   dL/du, dL/dv, dL/dA2, dL/dB2, dL/dC2, dL/do, dL/dr, dL/dg, dL/db (the queen_proj record
 *   words; A2/B2/C2 the base-2 conic of p2).  Overwritten (zeroed first).  Accumulated with
 *   float atomics: run-to-run differences at the rounding level.
 * queen_project_backward: grad_rec (as above, for the same cameras) -> grad_planes device fp32
 *   [11+3B][n_pad] = dL/d(raw attributes): position, raw quaternion (through its
 *   normalisation), log-scale, opacity logit, SH coefficients; views summed in order
 *   (deterministic); padding columns 0.  Overwritten.  cams: host array, <= QUEEN_MAX_VIEWS. */
queen_status queen_rasterize_backward(queen_ctx* ctx, const queen_proj* proj, const queen_bins* bins,
                                      const queen_camera* cams, int32_t n_views, const float bg[3], const float* dL_drgb,
                                      float* grad_rec, void* stream);
queen_status queen_project_backward(queen_ctx* ctx, const queen_gaussians* scene, const queen_camera* cams,
                                    int32_t n_views, const float* grad_rec, float* grad_planes, void* stream);
/* queen_decode_backward: the encode side of Eq. 4-5 and the gates.  grad_planes =
 *   dL/dA_t [11+3B][n_pad] (e.g. from queen_project_backward); outputs (each nullable, device fp32,
 *   overwritten):
 *   grad_decoders [ndec] (the packet's concatenated D_c layout): sum_i dL/dA[row][i] l[k][i],
 *     summed in a fixed order (deterministic);
 *   grad_latents [sum L][n_pad]: straight-through round: D_c^T dL/dr_c;
 *   grad_log_alpha [n_pad], grad_pregate [3][n_pad] (pos_kind GATES; zeros otherwise): on the
 *     forward's mask, dL/dl_p = g dL/dp and dL/dlog alpha = (l_p . dL/dp) dg/dlog alpha, 0 where
 *     g is clamped to 0 or 1 (deterministic gate, R#6).
 *   Uses the workspace's sort scratch for the decoder partial sums. */
queen_status queen_decode_backward(queen_ctx* ctx, const queen_packet* pkt, const float* grad_planes,
                                   float* grad_decoders, float* grad_latents, float* grad_log_alpha, float* grad_pregate,
                                   void* stream);

/* ---- NEXT #2: densification deltas (DESIGN reading R21) --------------------
 * queen_densify: dst = src without the Gaussians rem_idx (surviving columns keep their order)
 *   followed by n_add added Gaussians in order, whose attributes come as IEEE binary16 SoA
 *   add_attrs [11+3B][n_add] (host layout of the raw parameters, converted exactly to fp32).
 *   rem_idx: device u32 [n_rem], strictly increasing, each < src->n (else QUEEN_ERR_INDEX,
 *   sticky; dst contents undefined).  src and dst: same sh_degree, DISTINCT buffers (ping-pong);
 *   dst->n must equal src->n - n_rem + n_add <= dst->n_pad; dst padding columns are zeroed.
 *   Call after queen_apply_frame of the same frame (residuals refer to the pre-densification
 *   set). */
queen_status queen_densify(queen_ctx* ctx, const queen_gaussians* src, const uint32_t* rem_idx, int32_t n_rem,
                           const uint16_t* add_attrs, int32_t n_add, queen_gaussians* dst, void* stream);

/* ---- NEXT #3: masked / dynamic-subset rendering -----
 * queen_render_mask: renders ONLY the Gaussians listed in subset_idx (device u32 [k], strictly
 *   increasing, each < scene->n; when k_dev (device int32) is non-NULL the live count is
 *   min(*k_dev, k) -- e.g. a frame packet's gated COO indices, the "dynamic" set) for n_views
 *   equally-sized cameras; marks every pixel whose accumulated alpha 1 - T exceeds alpha_thresh
 *   (S:322-326 uses 1e-3; T by the same compositing rules as queen_rasterize, so with
 *   alpha_thresh < 1/255 a pixel is marked iff a subset Gaussian passes the 1/255 test there);
 *   then dilates the marks with a dilation x dilation square (48 in P:1262-1263): output pixel
 *   (x, y) is 1 iff a mark lies in [x - d/2, x - d/2 + d - 1] x [y - d/2, y - d/2 + d - 1],
 *   clipped at the borders (d = 1: no dilation).
 *   mask_out: device u8 [n_views][H][W], values 0/1.  Uses the workspace like
 *   queen_render_views (same sizing).  Invalid subset indices -> QUEEN_ERR_INDEX (sticky);
 *   dilation < 1, alpha_thresh outside [0,1), W > 12000 -> immediate error. */
queen_status queen_render_mask(queen_ctx* ctx, const queen_gaussians* scene, const uint32_t* subset_idx, int32_t k,
                               const int32_t* k_dev, const queen_camera* cams, int32_t n_views, float alpha_thresh,
                               int32_t dilation, uint8_t* mask_out, void* stream);

/* Makes `stream` wait until the binning (project + bin_sort) of the most recent
 * queen_render_views call on `ctx` has completed -- lets a renderer with several contexts
 * pipeline one batch's binning (memory/latency bound) under another batch's blend (ALU
 * bound).  Capturable; no host sync. */
queen_status queen_wait_binned(const queen_ctx* ctx, void* stream);

/* Makes `stream` wait until the projection of the most recent queen_render_views call on `ctx`
 * has completed.  The projection is the render's only read of the Gaussian SoA (the binning and
 * the blend read the projected records in the workspace), so the next frame's
 * queen_apply_frame (A_t -> A_{t+1}) may overwrite the SoA from then on while this
 * frame's binning and blend continue.  Capturable; no host sync. */
queen_status queen_wait_projected(const queen_ctx* ctx, void* stream);

/* Optional separate stream for the blend of queen_render_views[_rgb8] on `ctx` (NULL: the
 * call's stream, the default).  When set, the projection + binning run on the call's stream
 * and the blend on `stream` after them, so a renderer can give the (latency-bound) binning a
 * higher stream priority than the (ALU-bound) blend of another context; the next
 * queen_render_views on `ctx` waits for this blend before reusing the workspace.
 * queen_wait_rendered makes `stream` wait for the most recent blend that ran on a blend
 * stream of `ctx`.  Not for stream capture (the plain single-stream path is capturable). */
queen_status queen_set_blend_stream(queen_ctx* ctx, void* stream);
queen_status queen_wait_rendered(const queen_ctx* ctx, void* stream);

/* Stage profiler (evidence for bench.py): when enabled, every call records CUDA events
 * on its stream around each stage: 0 apply, 1 project, 2 compact (+resets), 3 depth sort,
 * 4 bucket (pieces counted and scattered into tile buckets), 5 emit (entries written in order), 6 ranges, 7 blend (k_blend alone), 8 entropy decode, 9 blend
 * order (the longest-list-first tile schedule built before the blend).  queen_profile_read
 * waits for the recorded events and returns per-stage summed milliseconds and kernel
 * launches (double[10], int64[10]), optionally resetting them.  Not capturable. */
queen_status queen_profile_enable(queen_ctx* ctx, int32_t enable);

/* Context options (test / experiment switches, set once per context, default 0):
 *   QUEEN_OPT_BLEND_NOMASK      k_blend without the per-warp record lists (per-thread box cull
 *                               only) -- the reference the exactness test of the lists compares to;
 *   QUEEN_OPT_BLEND_GRID_ORDER  blend tiles in grid order instead of longest-list-first.
 * Neither changes any output bit (both are tested).  Unknown bits -> QUEEN_ERR_INVALID_ARG. */
enum { QUEEN_OPT_BLEND_NOMASK = 1, QUEEN_OPT_BLEND_GRID_ORDER = 2 };
queen_status queen_set_options(queen_ctx* ctx, int32_t opts);
queen_status queen_profile_read(queen_ctx* ctx, double* ms, int64_t* launches, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* QUEEN_H */
