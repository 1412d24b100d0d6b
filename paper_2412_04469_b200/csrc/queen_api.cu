// libqueen C-ABI entry points (include/queen.h): argument validation, workspace
// carve-up, sticky-flag reporting and the per-frame orchestration
// (queen_render_views = project -> bin_sort -> rasterize, all enqueued, no host sync).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "queen_internal.cuh"

struct queen_ctx {
    int device = 0;
    void* ws = nullptr;
    size_t ws_bytes = 0;
    int32_t ws_n_pad = 0, ws_views = 0, ws_w = 0, ws_h = 0;
    const uint8_t* select = nullptr;  // set only while queen_render_mask projects its subset
    int64_t ws_keys = 0;
    queen::WsLayout L{};
    queen::Prof prof;
    cudaEvent_t binned = nullptr;     // recorded by queen_render_views after binning (queen_wait_binned)
    cudaEvent_t projected = nullptr;  // recorded after the projection: the last read of the SoA (queen_wait_projected)
    cudaEvent_t rendered = nullptr;     // recorded by queen_render_views after the blend
    cudaStream_t blend_stream = nullptr;  // queen_set_blend_stream: the blend's own stream
    bool blend_elsewhere = false;         // the most recent blend ran on blend_stream
    int32_t opts = 0;                     // queen_set_options (test / experiment switches)
    std::string err;
};

namespace queen {
float host_theta0(float tau, float g0, float g1) {
    // exact mask threshold on log alpha: g_tilde > 0 <=> log alpha > tau ln(-g0/g1) (R#6)
    return (float)((double)tau * std::log(-(double)g0 / (double)g1));
}
cudaError_t init_binning_attributes();
cudaError_t init_entropy_attributes();
size_t ans_encode(const int8_t* lat, int L, int n, int n_pad, std::vector<unsigned char>& out);
cudaError_t launch_ans_decode(const void* stream_dev, int64_t bytes, int L, int n, int n_pad, int8_t* out,
                              DevFlags* fl, cudaStream_t s);
cudaError_t launch_ans_decode_frame(const void* const streams[5], const int64_t bytes[5], const int L[5], int n,
                                    int n_pad, int8_t* out, DevFlags* fl, cudaStream_t s);
}  // namespace queen

using namespace queen;

static queen_status fail(queen_ctx* c, queen_status st, const char* msg) {
    if (c) c->err = msg;
    return st;
}
static queen_status cuda_fail(queen_ctx* c, cudaError_t e, const char* where) {
    if (c) c->err = std::string(where) + ": " + cudaGetErrorString(e);
    return QUEEN_ERR_CUDA;
}

extern "C" {

const char* queen_version(void) { return "libqueen 0.1 sm_100a"; }

queen_status queen_create(int device, queen_ctx** out) {
    if (!out) return QUEEN_ERR_INVALID_ARG;
    *out = nullptr;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return QUEEN_ERR_CUDA;
    if ((e = init_binning_attributes()) != cudaSuccess || (e = init_entropy_attributes()) != cudaSuccess)
        return QUEEN_ERR_CUDA;
    queen_ctx* c = new queen_ctx();
    c->device = device;
    if (cudaEventCreateWithFlags(&c->binned, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->projected, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->rendered, cudaEventDisableTiming) != cudaSuccess) {
        delete c;
        return QUEEN_ERR_CUDA;
    }
    *out = c;
    return QUEEN_OK;
}

void queen_destroy(queen_ctx* ctx) {
    if (!ctx) return;
    if (ctx->binned) cudaEventDestroy(ctx->binned);
    if (ctx->projected) cudaEventDestroy(ctx->projected);
    if (ctx->rendered) cudaEventDestroy(ctx->rendered);
    for (cudaEvent_t e : ctx->prof.pool) cudaEventDestroy(e);
    delete ctx;
}

queen_status queen_wait_binned(const queen_ctx* ctx, void* stream) {
    if (!ctx) return QUEEN_ERR_INVALID_ARG;
    return cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), ctx->binned, 0) == cudaSuccess ? QUEEN_OK
                                                                                                 : QUEEN_ERR_CUDA;
}

queen_status queen_wait_projected(const queen_ctx* ctx, void* stream) {
    if (!ctx) return QUEEN_ERR_INVALID_ARG;
    return cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), ctx->projected, 0) == cudaSuccess ? QUEEN_OK
                                                                                                    : QUEEN_ERR_CUDA;
}

queen_status queen_set_blend_stream(queen_ctx* ctx, void* stream) {
    if (!ctx) return QUEEN_ERR_INVALID_ARG;
    ctx->blend_stream = static_cast<cudaStream_t>(stream);
    return QUEEN_OK;
}

queen_status queen_wait_rendered(const queen_ctx* ctx, void* stream) {
    if (!ctx) return QUEEN_ERR_INVALID_ARG;
    return cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), ctx->rendered, 0) == cudaSuccess ? QUEEN_OK
                                                                                                   : QUEEN_ERR_CUDA;
}

const char* queen_last_error(const queen_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

queen_status queen_workspace_size(int32_t n_pad, int32_t n_views, int32_t width, int32_t height, int64_t keys_cap,
                                  size_t* bytes) {
    if (!bytes) return QUEEN_ERR_INVALID_ARG;
    if (n_pad < 0 || n_pad % 4 || n_views < 1 || n_views > QUEEN_MAX_VIEWS || width < 1 || height < 1 ||
        keys_cap < 1 || keys_cap > MAX_KEYS)
        return QUEEN_ERR_SHAPE;
    *bytes = ws_layout(n_pad, n_views, width, height, keys_cap).total;
    return QUEEN_OK;
}

queen_status queen_set_workspace(queen_ctx* ctx, void* dev_ptr, size_t bytes, int32_t n_pad, int32_t n_views,
                                 int32_t width, int32_t height, int64_t keys_cap) {
    if (!ctx || !dev_ptr) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null ctx/workspace");
    size_t need = 0;
    queen_status st = queen_workspace_size(n_pad, n_views, width, height, keys_cap, &need);
    if (st) return fail(ctx, st, "bad workspace shape");
    if (bytes < need) return fail(ctx, QUEEN_ERR_SHAPE, "workspace too small");
    if (reinterpret_cast<uintptr_t>(dev_ptr) % 256) return fail(ctx, QUEEN_ERR_INVALID_ARG, "workspace not 256-B aligned");
    ctx->ws = dev_ptr;
    ctx->ws_bytes = bytes;
    ctx->ws_n_pad = n_pad;
    ctx->ws_views = n_views;
    ctx->ws_w = width;
    ctx->ws_h = height;
    ctx->ws_keys = keys_cap;
    ctx->L = ws_layout(n_pad, n_views, width, height, keys_cap);
    cudaError_t e = cudaMemset(dev_ptr, 0, ctx->L.total_scratch);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "queen_set_workspace");
    return QUEEN_OK;
}

static DevFlags* flags_of(queen_ctx* c) { return reinterpret_cast<DevFlags*>(static_cast<unsigned char*>(c->ws) + c->L.flags); }

queen_status queen_check(queen_ctx* ctx, void* stream, int64_t* info_out) {
    if (!ctx || !ctx->ws) return fail(ctx, QUEEN_ERR_INVALID_ARG, "no workspace");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "queen_check sync");
    DevFlags h{};
    DevFlags* d = flags_of(ctx);
    e = cudaMemcpy(&h, d, sizeof(DevFlags), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "queen_check copy");
    if (info_out) *info_out = (int64_t)h.info;
    uint32_t zero[4] = {0, 0, 0, 0};
    e = cudaMemcpy(d, zero, 16, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "queen_check reset");
    if (h.flags & FLAG_INDEX) return fail(ctx, QUEEN_ERR_INDEX, "COO index out of range or not strictly increasing");
    if (h.flags & FLAG_LATENT_RANGE) return fail(ctx, QUEEN_ERR_LATENT_RANGE, "rounded latent outside [-127,127]");
    if (h.flags & FLAG_CAPACITY) return fail(ctx, QUEEN_ERR_CAPACITY, "key capacity exceeded (info = keys needed)");
    if (h.flags & FLAG_TIMEOUT) return fail(ctx, QUEEN_ERR_TIMEOUT, "look-back spin bound exceeded");
    if (h.flags & FLAG_NONFINITE) return fail(ctx, QUEEN_WARN_NONFINITE, "non-finite Gaussian culled");
    return QUEEN_OK;
}

static queen_status check_packet(queen_ctx* ctx, const queen_packet* p) {
    if (!p || !p->latents || !p->decoders) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null packet/latents/decoders");
    if (p->sh_degree < 0 || p->sh_degree > 3) return fail(ctx, QUEEN_ERR_INVALID_ARG, "sh_degree not in [0,3]");
    if (p->n < 0 || p->n > p->n_pad || p->n_pad % 4) return fail(ctx, QUEEN_ERR_SHAPE, "n > n_pad or n_pad % 4");
    for (int c = 0; c < 5; ++c)
        if (p->lat_dim[c] < 0 || p->lat_dim[c] > 16) return fail(ctx, QUEEN_ERR_SHAPE, "lat_dim outside [0,16]");
    if (p->sh_degree == 0 && p->lat_dim[4] != 0) return fail(ctx, QUEEN_ERR_SHAPE, "sh_rest latent dim must be 0 at degree 0");
    if (p->latent_kind != QUEEN_LAT_INT8 && p->latent_kind != QUEEN_LAT_F32) return fail(ctx, QUEEN_ERR_INVALID_ARG, "latent_kind");
    if (p->pos_kind == QUEEN_POS_COO) {
        if (p->k < 0 || (p->k > 0 && (!p->pos_idx || !p->pos_val))) return fail(ctx, QUEEN_ERR_INVALID_ARG, "bad COO");
    } else if (p->pos_kind == QUEEN_POS_GATES) {
        if (!p->log_alpha || !p->pos_pregate) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null gates");
        if (!(p->tau > 0.f) || !(p->gamma0 < 0.f) || !(p->gamma1 > 1.f)) return fail(ctx, QUEEN_ERR_INVALID_ARG, "gate hyperparameters");
    } else if (p->pos_kind != QUEEN_POS_NONE) {
        return fail(ctx, QUEEN_ERR_INVALID_ARG, "pos_kind");
    }
    return QUEEN_OK;
}

queen_status queen_decode_residuals(queen_ctx* ctx, const queen_packet* pkt, float* resid_out, int8_t* q_out,
                                    uint32_t* coo_idx_out, float* coo_val_out, int32_t* k_out, void* stream) {
    if (!ctx || !ctx->ws) return fail(ctx, QUEEN_ERR_INVALID_ARG, "no ctx/workspace");
    if (queen_status st = check_packet(ctx, pkt)) return st;
    const bool coo_out = coo_idx_out || coo_val_out || k_out;
    if (coo_out && !(coo_idx_out && coo_val_out && k_out)) return fail(ctx, QUEEN_ERR_INVALID_ARG, "COO outputs go together");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DevFlags* fl = flags_of(ctx);
    cudaError_t e = cudaSuccess;
    if (resid_out || q_out) e = launch_decode_apply(*pkt, nullptr, resid_out, q_out, false, false, fl, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "decode");
    if (coo_out) {
        if (pkt->pos_kind == QUEEN_POS_GATES) {
            // scratch for block counts: the depth-key buffer (not in use concurrently)
            void* scratch = static_cast<unsigned char*>(ctx->ws) + ctx->L.dkeys;
            size_t need = sizeof(uint32_t) * ((pkt->n + 1023) / 1024 + 1);
            if (need > ctx->L.dkeys_alt - ctx->L.dkeys) return fail(ctx, QUEEN_ERR_SHAPE, "workspace too small for gate compaction");
            e = launch_gate_compact(*pkt, coo_idx_out, coo_val_out, k_out, scratch, fl, s);
        } else if (pkt->pos_kind == QUEEN_POS_COO) {
            e = launch_coo_copy(*pkt, coo_idx_out, coo_val_out, k_out, fl, s);
        } else {
            e = cudaMemsetAsync(k_out, 0, sizeof(int32_t), s);
        }
        if (e != cudaSuccess) return cuda_fail(ctx, e, "decode positions");
    }
    return QUEEN_OK;
}

queen_status queen_apply_frame(queen_ctx* ctx, queen_gaussians* scene, const queen_packet* pkt, void* stream) {
    if (!ctx || !ctx->ws) return fail(ctx, QUEEN_ERR_INVALID_ARG, "no ctx/workspace");
    if (!scene || !scene->planes) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null scene");
    if (queen_status st = check_packet(ctx, pkt)) return st;
    if (scene->n != pkt->n || scene->n_pad != pkt->n_pad || scene->sh_degree != pkt->sh_degree)
        return fail(ctx, QUEEN_ERR_SHAPE, "scene / packet shape mismatch");
    ctx->prof.begin(ST_APPLY, static_cast<cudaStream_t>(stream));
    cudaError_t e = launch_decode_apply(*pkt, scene->planes, nullptr, nullptr, true, true, flags_of(ctx),
                                        static_cast<cudaStream_t>(stream));
    ctx->prof.end(static_cast<cudaStream_t>(stream), 1);  // decode + apply + gates / COO scatter: one launch
    if (e != cudaSuccess) return cuda_fail(ctx, e, "apply");
    return QUEEN_OK;
}

queen_status queen_set_sh_rest(queen_ctx* ctx, queen_gaussians* scene, const int8_t* latents, int32_t L,
                               const float* decoder, void* stream) {
    if (!ctx) return QUEEN_ERR_INVALID_ARG;
    if (!scene || !scene->planes || !latents || !decoder) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null args");
    if (scene->sh_degree < 1 || scene->sh_degree > 3) return fail(ctx, QUEEN_ERR_INVALID_ARG, "sh_degree must be 1..3 (SH-rest exists)");
    if (L < 1 || L > 16) return fail(ctx, QUEEN_ERR_INVALID_ARG, "latent dim must be 1..16");
    if (scene->n < 0 || scene->n > scene->n_pad || scene->n_pad % 4) return fail(ctx, QUEEN_ERR_SHAPE, "n <= n_pad, n_pad % 4 == 0");
    ctx->prof.begin(ST_APPLY, static_cast<cudaStream_t>(stream));
    cudaError_t e = launch_set_sh_rest(scene->planes, scene->n, scene->n_pad, scene->sh_degree, latents, L, decoder,
                                       flags_of(ctx), static_cast<cudaStream_t>(stream));
    ctx->prof.end(static_cast<cudaStream_t>(stream), 1);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "set_sh_rest");
    return QUEEN_OK;
}

static queen_status check_cams(queen_ctx* ctx, const queen_camera* cams, int32_t n_views, bool same_size) {
    if (!cams || n_views < 1) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null cams / n_views < 1");
    for (int v = 0; v < n_views; ++v) {
        const queen_camera& c = cams[v];
        if (!(c.fx > 0.f) || !(c.fy > 0.f) || !(c.near_z > 0.f) || c.width < 1 || c.height < 1)
            return fail(ctx, QUEEN_ERR_INVALID_ARG, "camera: fx, fy, near must be > 0");
        if (c.width > 16 * 32767 || c.height > 16 * 32767) return fail(ctx, QUEEN_ERR_SHAPE, "image too large");
        for (int r = 0; r < 3; ++r)
            for (int q = 0; q < 3; ++q) {
                double d = 0;
                for (int m = 0; m < 3; ++m) d += (double)c.R[r * 3 + m] * c.R[q * 3 + m];
                if (std::fabs(d - (r == q ? 1.0 : 0.0)) > 1e-6) return fail(ctx, QUEEN_ERR_INVALID_ARG, "camera R not orthonormal (1e-6)");
            }
        if (same_size && (c.width != cams[0].width || c.height != cams[0].height))
            return fail(ctx, QUEEN_ERR_SHAPE, "views of a batch must share width/height");
    }
    return QUEEN_OK;
}

queen_status queen_project(queen_ctx* ctx, const queen_gaussians* scene, const queen_camera* cams, int32_t n_views,
                           queen_proj* out, void* stream) {
    if (!ctx || !ctx->ws) return fail(ctx, QUEEN_ERR_INVALID_ARG, "no ctx/workspace");
    if (!scene || !scene->planes || !out || !out->rec || !out->depth || !out->tiles || !out->rect)
        return fail(ctx, QUEEN_ERR_INVALID_ARG, "null scene/proj");
    if (scene->sh_degree < 0 || scene->sh_degree > 3) return fail(ctx, QUEEN_ERR_INVALID_ARG, "sh_degree");
    if (scene->n < 0 || scene->n > scene->n_pad || scene->n_pad % 4 || out->n_pad != scene->n_pad)
        return fail(ctx, QUEEN_ERR_SHAPE, "n / n_pad");
    if (queen_status st = check_cams(ctx, cams, n_views, false)) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ctx->prof.begin(ST_PROJECT, s);
    for (int v0 = 0; v0 < n_views; v0 += QUEEN_MAX_VIEWS) {
        const int nv = n_views - v0 < (int)QUEEN_MAX_VIEWS ? n_views - v0 : (int)QUEEN_MAX_VIEWS;
        CamBatch cb;
        std::memset(&cb, 0, sizeof(cb));
        std::memcpy(cb.cam, cams + v0, sizeof(queen_camera) * nv);
        const int64_t o = (int64_t)v0 * scene->n_pad;
        cudaError_t e = launch_project(scene->planes, scene->n, scene->n_pad, scene->sh_degree, cb, nv, out->rec + o * REC_WORDS,
                                       out->depth + o, out->tiles + o, out->rect + o * 4, ctx->select, flags_of(ctx), s);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "project");
    }
    ctx->prof.end(s, (n_views + QUEEN_MAX_VIEWS - 1) / QUEEN_MAX_VIEWS);
    return QUEEN_OK;
}

// order_ready (render paths): set when the binning also built the blend's tile schedule
static queen_status bin_sort_impl(queen_ctx* ctx, const queen_proj* proj, const queen_camera* cams, int32_t n_views,
                                  queen_bins* bins, void* stream, bool* order_ready) {
    if (order_ready) *order_ready = false;
    if (!ctx || !ctx->ws) return fail(ctx, QUEEN_ERR_INVALID_ARG, "no ctx/workspace");
    if (!proj || !bins || !bins->keys || !bins->keys_alt || !bins->vals || !bins->vals_alt || !bins->ranges || !bins->K)
        return fail(ctx, QUEEN_ERR_INVALID_ARG, "null proj/bins");
    if (queen_status st = check_cams(ctx, cams, n_views, true)) return st;
    const int W = cams[0].width, H = cams[0].height;
    const int64_t T = (int64_t)((W + 15) / 16) * ((H + 15) / 16);
    if (bins->keys_cap < 1 || bins->keys_cap > MAX_KEYS) return fail(ctx, QUEEN_ERR_SHAPE, "keys_cap outside [1, 2^30)");
    if (T * n_views >= (1ll << 31)) return fail(ctx, QUEEN_ERR_SHAPE, "too many tiles in one batch");
    if (!bin_plan(proj->n_pad, n_views, W, H).ok)
        return fail(ctx, QUEEN_ERR_SHAPE, "view too large: its (gx+1)(gy+1) tile grid exceeds 48K words (> 4K views)");
    // scratch must cover this batch
    WsLayout need = ws_layout(proj->n_pad, n_views, W, H, bins->keys_cap);
    if (need.key_tiles > ctx->L.key_tiles || need.elem_tiles > ctx->L.elem_tiles || need.elems > ctx->L.elems ||
        !scratch_fits(need, ctx->L))
        return fail(ctx, QUEEN_ERR_SHAPE, "workspace scratch too small for this batch");
    cudaError_t e = launch_bin_sort(*proj, n_views, W, H, *bins, ctx->ws, ctx->L, flags_of(ctx),
                                    static_cast<cudaStream_t>(stream), &ctx->prof, order_ready);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "bin_sort");
    return QUEEN_OK;
}

queen_status queen_bin_sort(queen_ctx* ctx, const queen_proj* proj, const queen_camera* cams, int32_t n_views,
                            queen_bins* bins, void* stream) {
    return bin_sort_impl(ctx, proj, cams, n_views, bins, stream, nullptr);
}

// workspace scratch for the blend schedule (tile order), if the workspace covers this call
static uint32_t* order_scratch(queen_ctx* ctx, int32_t n_views, int W, int H) {
    if (!ctx->ws) return nullptr;
    const int64_t T = (int64_t)((W + 15) / 16) * ((H + 15) / 16);
    if ((int64_t)n_views * T > (int64_t)ctx->ws_views * ctx->L.T) return nullptr;
    return reinterpret_cast<uint32_t*>(static_cast<unsigned char*>(ctx->ws) + ctx->L.order);
}

static queen_status rasterize_impl(queen_ctx* ctx, const queen_proj* proj, const queen_bins* bins,
                                   const queen_camera* cams, int32_t n_views, const float bg[3], float* rgb_out,
                                   float* T_out, uint8_t* rgb8_out, void* stream, int alt_mode = OUT_RGB8,
                                   bool order_ready = false) {
    if (!ctx) return QUEEN_ERR_INVALID_ARG;
    if (!proj || !bins || !(rgb_out || rgb8_out) || !bg) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null args");
    if (queen_status st = check_cams(ctx, cams, n_views, true)) return st;
    const uint32_t* vals = bins->sorted_in_alt ? bins->vals_alt : bins->vals;
    int nl = 1;
    uint32_t* ows = order_scratch(ctx, n_views, cams[0].width, cams[0].height);
    cudaError_t e = launch_rasterize(proj->rec, proj->n_pad, bins->ranges, vals, n_views, cams[0].width, cams[0].height,
                                     bg[0], bg[1], bg[2], rgb_out, T_out, rgb8_out, rgb8_out ? alt_mode : OUT_F32, 0.f,
                                     ows, static_cast<cudaStream_t>(stream), &nl, &ctx->prof, ctx->opts,
                                     (order_ready && ows) ? ows + 2 * ORDER_BINS : nullptr);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "rasterize");
    return QUEEN_OK;
}

queen_status queen_rasterize(queen_ctx* ctx, const queen_proj* proj, const queen_bins* bins, const queen_camera* cams,
                             int32_t n_views, const float bg[3], float* rgb_out, float* T_out, void* stream) {
    if (ctx && !rgb_out) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null rgb_out");
    return rasterize_impl(ctx, proj, bins, cams, n_views, bg, rgb_out, T_out, nullptr, stream);
}

queen_status queen_rasterize_f16(queen_ctx* ctx, const queen_proj* proj, const queen_bins* bins,
                                 const queen_camera* cams, int32_t n_views, const float bg[3], uint16_t* f16_out,
                                 float* T_out, void* stream) {
    if (ctx && !f16_out) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null f16_out");
    return rasterize_impl(ctx, proj, bins, cams, n_views, bg, nullptr, T_out, reinterpret_cast<uint8_t*>(f16_out), stream,
                          OUT_F16);
}

queen_status queen_rasterize_rgb10(queen_ctx* ctx, const queen_proj* proj, const queen_bins* bins,
                                 const queen_camera* cams, int32_t n_views, const float bg[3], uint32_t* rgb10_out,
                                 float* T_out, void* stream) {
    if (ctx && !rgb10_out) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null rgb10_out");
    return rasterize_impl(ctx, proj, bins, cams, n_views, bg, nullptr, T_out, reinterpret_cast<uint8_t*>(rgb10_out), stream,
                          OUT_RGB10);
}

queen_status queen_rasterize_rgb8(queen_ctx* ctx, const queen_proj* proj, const queen_bins* bins,
                                  const queen_camera* cams, int32_t n_views, const float bg[3], uint8_t* rgb8_out,
                                  float* T_out, void* stream) {
    if (ctx && !rgb8_out) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null rgb8_out");
    return rasterize_impl(ctx, proj, bins, cams, n_views, bg, nullptr, T_out, rgb8_out, stream);
}

queen_status queen_blend_counts(queen_ctx* ctx, const queen_proj* proj, const queen_bins* bins,
                                const queen_camera* cams, int32_t n_views, int64_t* evaluated, int64_t* composited,
                                void* stream) {
    if (!ctx) return QUEEN_ERR_INVALID_ARG;
    if (!proj || !bins || !evaluated || !composited) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null args");
    if (queen_status st = check_cams(ctx, cams, n_views, true)) return st;
    const uint32_t* vals = bins->sorted_in_alt ? bins->vals_alt : bins->vals;
    cudaError_t e = launch_blend_counts(proj->rec, proj->n_pad, bins->ranges, vals, n_views, cams[0].width,
                                        cams[0].height, reinterpret_cast<long long*>(evaluated),
                                        reinterpret_cast<long long*>(composited), static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "blend_counts");
    return QUEEN_OK;
}

queen_status queen_set_options(queen_ctx* ctx, int32_t opts) {
    if (!ctx) return QUEEN_ERR_INVALID_ARG;
    if (opts & ~(QUEEN_OPT_BLEND_NOMASK | QUEEN_OPT_BLEND_GRID_ORDER)) return fail(ctx, QUEEN_ERR_INVALID_ARG, "unknown option bits");
    ctx->opts = opts;
    return QUEEN_OK;
}

queen_status queen_profile_enable(queen_ctx* ctx, int32_t enable) {
    if (!ctx) return QUEEN_ERR_INVALID_ARG;
    ctx->prof.on = enable != 0;
    ctx->prof.reset_chain();
    return QUEEN_OK;
}

queen_status queen_profile_read(queen_ctx* ctx, double* ms, int64_t* launches, int32_t reset) {
    if (!ctx || !ms || !launches) return QUEEN_ERR_INVALID_ARG;
    Prof& P = ctx->prof;
    if (!P.pending.empty()) {
        cudaError_t e = cudaEventSynchronize(P.pool[P.pending.back().e1]);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "queen_profile_read");
        for (auto& q : P.pending) {
            float t = 0.f;
            e = cudaEventElapsedTime(&t, P.pool[q.e0], P.pool[q.e1]);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "queen_profile_read elapsed");
            P.ms[q.stage] += t;
            P.launches[q.stage] += q.launches;
        }
        P.pending.clear();
        P.used = 0;
        P.reset_chain();
    }
    for (int i = 0; i < ST_COUNT; ++i) {
        ms[i] = P.ms[i];
        launches[i] = P.launches[i];
        if (reset) { P.ms[i] = 0; P.launches[i] = 0; }
    }
    return QUEEN_OK;
}

queen_status queen_entropy_encode(const int8_t* latents, int32_t L, int32_t n, int32_t n_pad, void* out,
                                  size_t capacity, size_t* bytes) {
    if (!latents || !bytes || L < 0 || L > 16 || n < 0 || n > n_pad) return QUEEN_ERR_INVALID_ARG;
    std::vector<unsigned char> buf;
    const size_t need = ans_encode(latents, L, n, n_pad, buf);
    *bytes = need;
    if (!out || capacity < need) return QUEEN_ERR_SHAPE;
    std::memcpy(out, buf.data(), need);
    return QUEEN_OK;
}

queen_status queen_entropy_decode(queen_ctx* ctx, const void* stream_dev, int64_t stream_bytes, int32_t L, int32_t n,
                                  int32_t n_pad, int8_t* latents_out, void* stream) {
    if (!ctx || !ctx->ws) return fail(ctx, QUEEN_ERR_INVALID_ARG, "no ctx/workspace");
    if (!stream_dev || !latents_out || L < 0 || L > 16 || n < 0 || n > n_pad) return fail(ctx, QUEEN_ERR_INVALID_ARG, "entropy decode args");
    ctx->prof.begin(ST_ENTROPY, static_cast<cudaStream_t>(stream));
    cudaError_t e = launch_ans_decode(stream_dev, stream_bytes, L, n, n_pad, latents_out, flags_of(ctx),
                                      static_cast<cudaStream_t>(stream));
    ctx->prof.end(static_cast<cudaStream_t>(stream), 1);
    if (e == cudaErrorInvalidValue) return fail(ctx, QUEEN_ERR_SHAPE, "entropy stream smaller than its header and chunk tables");
    if (e != cudaSuccess) return cuda_fail(ctx, e, "entropy decode");
    return QUEEN_OK;
}

queen_status queen_entropy_decode_frame(queen_ctx* ctx, const void* const* streams_dev, const int64_t* stream_bytes,
                                        const int32_t* lat_dim, int32_t n, int32_t n_pad, int8_t* latents_out,
                                        void* stream) {
    if (!ctx || !ctx->ws) return fail(ctx, QUEEN_ERR_INVALID_ARG, "no ctx/workspace");
    if (!streams_dev || !stream_bytes || !lat_dim || !latents_out || n < 0 || n > n_pad)
        return fail(ctx, QUEEN_ERR_INVALID_ARG, "entropy frame args");
    const void* s5[5];
    int L5[5];
    int64_t b5[5];
    for (int c = 0; c < 5; ++c) {
        if (lat_dim[c] < 0 || lat_dim[c] > 16 || (lat_dim[c] > 0 && !streams_dev[c])) return fail(ctx, QUEEN_ERR_INVALID_ARG, "entropy frame category");
        s5[c] = streams_dev[c];
        L5[c] = lat_dim[c];
        b5[c] = stream_bytes[c];
    }
    ctx->prof.begin(ST_ENTROPY, static_cast<cudaStream_t>(stream));
    cudaError_t e = launch_ans_decode_frame(s5, b5, L5, n, n_pad, latents_out, flags_of(ctx),
                                            static_cast<cudaStream_t>(stream));
    ctx->prof.end(static_cast<cudaStream_t>(stream), 1);
    if (e == cudaErrorInvalidValue) return fail(ctx, QUEEN_ERR_SHAPE, "entropy stream smaller than its header and chunk tables");
    if (e != cudaSuccess) return cuda_fail(ctx, e, "entropy decode frame");
    return QUEEN_OK;
}

static queen_status render_impl(queen_ctx* ctx, const queen_gaussians* scene, const queen_camera* cams, int32_t n_views,
                                const float bg[3], float* rgb_out, float* T_out, uint8_t* rgb8_out, void* stream,
                                int alt_mode = OUT_RGB8) {
    if (!ctx || !ctx->ws) return fail(ctx, QUEEN_ERR_INVALID_ARG, "no ctx/workspace");
    if (!scene || !(rgb_out || rgb8_out) || !bg) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null args");
    if (queen_status st = check_cams(ctx, cams, n_views, true)) return st;
    if (scene->n_pad > ctx->ws_n_pad || n_views > ctx->ws_views || cams[0].width > ctx->ws_w || cams[0].height > ctx->ws_h)
        return fail(ctx, QUEEN_ERR_SHAPE, "workspace was sized for a smaller batch");
    unsigned char* ws = static_cast<unsigned char*>(ctx->ws);
    const WsLayout& L = ctx->L;
    queen_proj pj;
    pj.n_pad = scene->n_pad;
    pj.rec = reinterpret_cast<float*>(ws + L.rec);
    pj.depth = reinterpret_cast<uint32_t*>(ws + L.depth);
    pj.tiles = reinterpret_cast<uint32_t*>(ws + L.tiles);
    pj.rect = reinterpret_cast<int16_t*>(ws + L.rect);
    queen_bins b;
    b.keys_cap = ctx->ws_keys;
    b.keys = reinterpret_cast<uint32_t*>(ws + L.keys);
    b.keys_alt = reinterpret_cast<uint32_t*>(ws + L.keys_alt);
    b.vals = reinterpret_cast<uint32_t*>(ws + L.vals);
    b.vals_alt = reinterpret_cast<uint32_t*>(ws + L.vals_alt);
    b.ranges = reinterpret_cast<uint32_t*>(ws + L.ranges);
    b.K = reinterpret_cast<uint32_t*>(ws + L.K);
    b.sorted_in_alt = 0;
    cudaStream_t bs = ctx->blend_stream;
    // after a blend on a separate stream, that blend must be done before the binning overwrites
    // the workspace (the rendered event is only ever recorded on a separate blend stream, never
    // inside a capture of the plain path)
    if (ctx->blend_elsewhere && cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), ctx->rendered, 0) != cudaSuccess)
        return cuda_fail(ctx, cudaGetLastError(), "wait rendered event");
    ctx->blend_elsewhere = bs != nullptr;
    if (queen_status st = queen_project(ctx, scene, cams, n_views, &pj, stream)) return st;
    if (cudaEventRecord(ctx->projected, static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return cuda_fail(ctx, cudaGetLastError(), "record projected event");
    bool ord = false;
    if (queen_status st = bin_sort_impl(ctx, &pj, cams, n_views, &b, stream, &ord)) return st;
    if (cudaEventRecord(ctx->binned, static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return cuda_fail(ctx, cudaGetLastError(), "record binned event");
    if (!bs) return rasterize_impl(ctx, &pj, &b, cams, n_views, bg, rgb_out, T_out, rgb8_out, stream, alt_mode, ord);
    if (cudaStreamWaitEvent(bs, ctx->binned, 0) != cudaSuccess) return cuda_fail(ctx, cudaGetLastError(), "blend wait");
    queen_status st = rasterize_impl(ctx, &pj, &b, cams, n_views, bg, rgb_out, T_out, rgb8_out, bs, alt_mode, ord);
    if (!st && cudaEventRecord(ctx->rendered, bs) != cudaSuccess)
        return cuda_fail(ctx, cudaGetLastError(), "record rendered event");
    return st;
}

queen_status queen_render_views(queen_ctx* ctx, const queen_gaussians* scene, const queen_camera* cams, int32_t n_views,
                                const float bg[3], float* rgb_out, float* T_out, void* stream) {
    if (ctx && !rgb_out) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null rgb_out");
    return render_impl(ctx, scene, cams, n_views, bg, rgb_out, T_out, nullptr, stream);
}

queen_status queen_render_views_f16(queen_ctx* ctx, const queen_gaussians* scene, const queen_camera* cams,
                                    int32_t n_views, const float bg[3], uint16_t* f16_out, float* T_out, void* stream) {
    if (ctx && !f16_out) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null f16_out");
    return render_impl(ctx, scene, cams, n_views, bg, nullptr, T_out, reinterpret_cast<uint8_t*>(f16_out), stream, OUT_F16);
}

queen_status queen_render_views_rgb10(queen_ctx* ctx, const queen_gaussians* scene, const queen_camera* cams,
                                    int32_t n_views, const float bg[3], uint32_t* rgb10_out, float* T_out, void* stream) {
    if (ctx && !rgb10_out) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null rgb10_out");
    return render_impl(ctx, scene, cams, n_views, bg, nullptr, T_out, reinterpret_cast<uint8_t*>(rgb10_out), stream, OUT_RGB10);
}

queen_status queen_render_views_rgb8(queen_ctx* ctx, const queen_gaussians* scene, const queen_camera* cams,
                                     int32_t n_views, const float bg[3], uint8_t* rgb8_out, float* T_out, void* stream) {
    if (ctx && !rgb8_out) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null rgb8_out");
    return render_impl(ctx, scene, cams, n_views, bg, nullptr, T_out, rgb8_out, stream);
}

queen_status queen_rasterize_backward(queen_ctx* ctx, const queen_proj* proj, const queen_bins* bins,
                                      const queen_camera* cams, int32_t n_views, const float bg[3], const float* dL_drgb,
                                      float* grad_rec, void* stream) {
    if (!ctx) return QUEEN_ERR_INVALID_ARG;
    if (!proj || !bins || !bg || !dL_drgb || !grad_rec) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null args");
    if (queen_status st = check_cams(ctx, cams, n_views, true)) return st;
    const uint32_t* vals = bins->sorted_in_alt ? bins->vals_alt : bins->vals;
    cudaError_t e = launch_blend_bwd(proj->rec, proj->n_pad, bins->ranges, vals, n_views, cams[0].width, cams[0].height,
                                     bg[0], bg[1], bg[2], dL_drgb, grad_rec,
                                     order_scratch(ctx, n_views, cams[0].width, cams[0].height),
                                     static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "rasterize_backward");
    return QUEEN_OK;
}

queen_status queen_project_backward(queen_ctx* ctx, const queen_gaussians* scene, const queen_camera* cams,
                                    int32_t n_views, const float* grad_rec, float* grad_planes, void* stream) {
    if (!ctx) return QUEEN_ERR_INVALID_ARG;
    if (!scene || !scene->planes || !grad_rec || !grad_planes) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null args");
    if (scene->sh_degree < 0 || scene->sh_degree > 3) return fail(ctx, QUEEN_ERR_INVALID_ARG, "sh_degree");
    if (scene->n < 0 || scene->n > scene->n_pad || scene->n_pad % 4) return fail(ctx, QUEEN_ERR_SHAPE, "n / n_pad");
    if (n_views > (int32_t)QUEEN_MAX_VIEWS) return fail(ctx, QUEEN_ERR_SHAPE, "n_views > QUEEN_MAX_VIEWS");
    if (queen_status st = check_cams(ctx, cams, n_views, false)) return st;
    CamBatch cb;
    std::memset(&cb, 0, sizeof(cb));
    std::memcpy(cb.cam, cams, sizeof(queen_camera) * n_views);
    cudaError_t e = launch_project_bwd(scene->planes, scene->n, scene->n_pad, scene->sh_degree, cb, n_views, grad_rec,
                                       grad_planes, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "project_backward");
    return QUEEN_OK;
}

queen_status queen_decode_backward(queen_ctx* ctx, const queen_packet* pkt, const float* grad_planes,
                                   float* grad_decoders, float* grad_latents, float* grad_log_alpha, float* grad_pregate,
                                   void* stream) {
    if (!ctx || !ctx->ws) return fail(ctx, QUEEN_ERR_INVALID_ARG, "no ctx/workspace");
    if (queen_status st = check_packet(ctx, pkt)) return st;
    if (!grad_planes) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null grad_planes");
    if ((grad_log_alpha || grad_pregate) && pkt->pos_kind == QUEEN_POS_GATES && (!pkt->log_alpha || !pkt->pos_pregate))
        return fail(ctx, QUEEN_ERR_INVALID_ARG, "gate gradients need log_alpha and pos_pregate");
    float* scratch = reinterpret_cast<float*>(static_cast<unsigned char*>(ctx->ws) + ctx->L.dkeys);
    const size_t sfloats = (ctx->L.counts - ctx->L.dkeys) / sizeof(float);
    cudaError_t e = launch_decode_bwd(*pkt, grad_planes, grad_decoders, grad_latents, grad_log_alpha, grad_pregate,
                                      scratch, sfloats, static_cast<cudaStream_t>(stream));
    if (e == cudaErrorInvalidValue) return fail(ctx, QUEEN_ERR_SHAPE, "workspace too small for the decoder gradient");
    if (e != cudaSuccess) return cuda_fail(ctx, e, "decode_backward");
    return QUEEN_OK;
}

queen_status queen_densify(queen_ctx* ctx, const queen_gaussians* src, const uint32_t* rem_idx, int32_t n_rem,
                           const uint16_t* add_attrs, int32_t n_add, queen_gaussians* dst, void* stream) {
    if (!ctx || !ctx->ws) return fail(ctx, QUEEN_ERR_INVALID_ARG, "no ctx/workspace");
    if (!src || !dst || !src->planes || !dst->planes) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null scene");
    if (src->planes == dst->planes) return fail(ctx, QUEEN_ERR_INVALID_ARG, "src and dst must be distinct buffers");
    if (n_rem < 0 || n_add < 0 || (n_rem > 0 && !rem_idx) || (n_add > 0 && !add_attrs))
        return fail(ctx, QUEEN_ERR_INVALID_ARG, "bad removal / addition lists");
    if (src->sh_degree != dst->sh_degree || src->sh_degree < 0 || src->sh_degree > 3)
        return fail(ctx, QUEEN_ERR_INVALID_ARG, "sh_degree");
    if (src->n < 0 || src->n > src->n_pad || n_rem > src->n) return fail(ctx, QUEEN_ERR_SHAPE, "src n / n_rem");
    if (dst->n != src->n - n_rem + n_add || dst->n > dst->n_pad || dst->n_pad % 4)
        return fail(ctx, QUEEN_ERR_SHAPE, "dst n must be src n - n_rem + n_add <= dst n_pad (n_pad % 4 == 0)");
    const int B = (src->sh_degree + 1) * (src->sh_degree + 1);
    cudaError_t e = launch_densify(src->planes, src->n, src->n_pad, rem_idx, n_rem, add_attrs, n_add, 11 + 3 * B,
                                   dst->planes, dst->n_pad, flags_of(ctx), static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "densify");
    return QUEEN_OK;
}

queen_status queen_render_mask(queen_ctx* ctx, const queen_gaussians* scene, const uint32_t* subset_idx, int32_t k,
                               const int32_t* k_dev, const queen_camera* cams, int32_t n_views, float alpha_thresh,
                               int32_t dilation, uint8_t* mask_out, void* stream) {
    if (!ctx || !ctx->ws) return fail(ctx, QUEEN_ERR_INVALID_ARG, "no ctx/workspace");
    if (!scene || !scene->planes || !mask_out) return fail(ctx, QUEEN_ERR_INVALID_ARG, "null scene/mask_out");
    if (k < 0 || (k > 0 && !subset_idx)) return fail(ctx, QUEEN_ERR_INVALID_ARG, "bad subset");
    if (dilation < 1 || !(alpha_thresh >= 0.f && alpha_thresh < 1.f))
        return fail(ctx, QUEEN_ERR_INVALID_ARG, "dilation >= 1 and alpha_thresh in [0,1) required");
    if (queen_status st = check_cams(ctx, cams, n_views, true)) return st;
    const int W = cams[0].width, H = cams[0].height;
    if (scene->n_pad > ctx->ws_n_pad || n_views > ctx->ws_views || W > ctx->ws_w || H > ctx->ws_h)
        return fail(ctx, QUEEN_ERR_SHAPE, "workspace was sized for a smaller batch");
    if (W > 12000) return fail(ctx, QUEEN_ERR_SHAPE, "mask rows wider than 12000 pixels");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    unsigned char* ws = static_cast<unsigned char*>(ctx->ws);
    const WsLayout& L = ctx->L;
    uint8_t* sel = reinterpret_cast<uint8_t*>(ws + L.select);
    cudaError_t e = launch_select(subset_idx, k, k_dev, scene->n, scene->n_pad, sel, flags_of(ctx), s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "render_mask select");
    queen_proj pj;
    pj.n_pad = scene->n_pad;
    pj.rec = reinterpret_cast<float*>(ws + L.rec);
    pj.depth = reinterpret_cast<uint32_t*>(ws + L.depth);
    pj.tiles = reinterpret_cast<uint32_t*>(ws + L.tiles);
    pj.rect = reinterpret_cast<int16_t*>(ws + L.rect);
    queen_bins b;
    b.keys_cap = ctx->ws_keys;
    b.keys = reinterpret_cast<uint32_t*>(ws + L.keys);
    b.keys_alt = reinterpret_cast<uint32_t*>(ws + L.keys_alt);
    b.vals = reinterpret_cast<uint32_t*>(ws + L.vals);
    b.vals_alt = reinterpret_cast<uint32_t*>(ws + L.vals_alt);
    b.ranges = reinterpret_cast<uint32_t*>(ws + L.ranges);
    b.K = reinterpret_cast<uint32_t*>(ws + L.K);
    b.sorted_in_alt = 0;
    ctx->select = sel;
    queen_status st = queen_project(ctx, scene, cams, n_views, &pj, stream);
    ctx->select = nullptr;
    if (st) return st;
    if ((st = queen_bin_sort(ctx, &pj, cams, n_views, &b, stream))) return st;
    const uint32_t* vals = b.sorted_in_alt ? b.vals_alt : b.vals;
    ctx->prof.begin(ST_BLEND, s);
    int nl = 1;
    e = launch_rasterize(pj.rec, pj.n_pad, b.ranges, vals, n_views, W, H, 0.f, 0.f, 0.f, nullptr, nullptr, mask_out,
                         OUT_MASK, alpha_thresh, order_scratch(ctx, n_views, W, H), s, &nl, nullptr, ctx->opts);
    if (e == cudaSuccess) e = launch_dilate(mask_out, reinterpret_cast<uint8_t*>(ws + L.mask_tmp), n_views, W, H, dilation, s);
    ctx->prof.end(s, nl + (dilation > 1 ? 2 : 0));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "render_mask");
    return QUEEN_OK;
}

}  // extern "C"
