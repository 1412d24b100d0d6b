// K1 / K1b: fused residual decode + apply (Eq. 4-5) and the
// position step (hard-concrete gate P:329-336, COO P:1389-1390).
//
// One coalesced, vectorised pass over the Gaussian SoA, split into work groups of rows so
// that every thread has all of its loads in flight at once (below).  The decoders sit in
// shared memory and are read as warp-uniform broadcasts.  HBM-bound: bytes per Gaussian =
// sum L_c (int8) + 2*4*sum M_c (fp32 read+write), K1.
#include "queen_internal.cuh"

namespace queen {

#ifndef QUEEN_DA_MINB
#define QUEEN_DA_MINB 4  // min resident blocks per SM (register cap: 64)
#endif
#ifndef QUEEN_DA_ROWS
#define QUEEN_DA_ROWS 4  // measured N3DV apply (L2 flushed): 8 rows x 2 blocks 57 us, 6 x 3 45 us, 4 x 4 41 us
#endif
// Gaussian blocks per grid super-tile: group-major over all blocks while a category's latent rows
// stay in L2 anyway; super-tiles of 512 blocks once they do not (measured, apply stage with L2
// flushed: stress 590 -> 516 us with 128, 506 us with 512; N3DV 42.8 us group-major vs 44.1
// with 128, 47.4 with 32)
#ifndef QUEEN_DA_SUPER
#define QUEEN_DA_SUPER 512  // measured (round 2, stress apply): 64 0.533, 128 0.516, 256 0.510, 512 0.506, 1024 0.510, 1536 0.522 ms
#endif
inline int da_super(int n) { return n > (1 << 20) ? QUEEN_DA_SUPER : 1 << 30; }
constexpr int DA_ROWS = QUEEN_DA_ROWS;      // attribute rows per work group (all loads in flight at once)
constexpr int DA_MAX_GROUPS = 5 + (4 + 3 + 1 + 3 + 45 + DA_ROWS - 1) / DA_ROWS + 1;  // worst case at degree 3, + gates

// One work group = rows [m0, m1) of category c (m1 - m0 <= DA_ROWS, balanced runs), or the gated position
// rows (c = 5).  The grid is (Gaussian blocks) x (groups) (+ the fused COO scatter blocks).
// A thread owns 4 consecutive Gaussians of one group (16-byte attribute accesses, 512 B per
// warp and row) and issues ALL of its loads -- the category's latent rows (<= 16 char4) and
// its <= DA_ROWS attribute rows -- before using any: one memory round trip per thread.
// Latents stay packed (one register per 4 Gaussians) and the decode runs k-outermost, so 64
// registers suffice for 4 resident blocks per SM.  (One thread walking all 56 rows was a chain of ~20
// dependent round trips in a single wave at 24 % occupancy: latency-bound at ~25 % of HBM.)
struct DecodeParams {
    int n, n_pad;
    int lat[5], M[5], lat_row0[5], dec_off[5], out_row0[5];
    int ndec;
    int ngroups;
    int g_c[DA_MAX_GROUPS], g_m0[DA_MAX_GROUPS], g_m1[DA_MAX_GROUPS];
    int xblocks;                 // Gaussian blocks per group
    int sx;                      // Gaussian blocks per grid super-tile
    int coo_k;                   // COO capacity (entries); 0 = no fused scatter
    const int32_t* coo_kdev;
    const uint32_t* coo_idx;
    const float* coo_val;
    const void* latents;
    const float* decoders;
    float* planes;
    float* resid_out;
    int8_t* q_out;
    const float* log_alpha;
    const float* pregate;
    float tau, g0, g1, theta0;
    DevFlags* fl;
};

// hard-concrete gate value: g = min(1, max(0, sigmoid(la/tau)(g1-g0)+g0))
__device__ __forceinline__ float gate_value(float la, float tau, float g0, float g1) {
    float ghat = 1.0f / (1.0f + det_exp((-la) / tau));
    float gt = fmaf(ghat, g1 - g0, g0);
    return fminf(1.0f, fmaxf(0.0f, gt));
}

// a5: p[I_k] += E_p[k] for entry j of the COO position residual; validates
// the index: idx < n and strictly increasing, else QUEEN_ERR_INDEX and skip.
__device__ __forceinline__ void coo_entry(float* planes, int n, int64_t n_pad, const uint32_t* idx, const float* val,
                                          int kcap, int j, DevFlags* fl) {
    const uint32_t i = idx[j];
    if (i >= (uint32_t)n || (j > 0 && i <= idx[j - 1])) {
        raise_flag(fl, FLAG_INDEX);
        return;
    }
    const float v0 = val[j], v1 = val[(int64_t)kcap + j], v2 = val[2 * (int64_t)kcap + j];
    planes[i] = planes[i] + v0;
    planes[n_pad + i] = planes[n_pad + i] + v1;
    planes[2 * n_pad + i] = planes[2 * n_pad + i] + v2;
}

template <bool F32, bool APPLY, bool GATES, bool SET = false>
__global__ void __launch_bounds__(256, QUEEN_DA_MINB) k_decode_apply(DecodeParams p) {
    extern __shared__ float sdec[];
    // grid: super-tiles of p.sx Gaussian blocks (da_super); inside one, group-major.  Every group
    // of a category re-reads the category's latent rows, which then come from L2 (a super-tile's
    // latents are <= sx * 1024 * 16 B), while the concurrent blocks still stream one plane at a
    // time.  (Fully gid-fastest was slower: N3DV 41 -> 49 us, stress 573 -> 628 us.)
    if ((int)blockIdx.x >= p.ngroups * p.xblocks) {
        // fused COO scatter blocks (COO mode: the decode groups never touch position rows)
        int k = p.coo_k;
        if (p.coo_kdev) k = min(max(*p.coo_kdev, 0), p.coo_k);
        const int j = (blockIdx.x - p.ngroups * p.xblocks) * blockDim.x + threadIdx.x;
        if (j < k) coo_entry(p.planes, p.n, p.n_pad, p.coo_idx, p.coo_val, p.coo_k, j, p.fl);
        return;
    }
    const int sx = min(p.sx, p.xblocks);
    const int sup = (int)blockIdx.x / (p.ngroups * sx);
    const int rem = (int)blockIdx.x - sup * p.ngroups * sx;
    const int width = min(sx, p.xblocks - sup * sx);  // Gaussian blocks in this super-tile
    const int gid = rem / width;
    const int xb = sup * sx + (rem - gid * width);
    const int c = p.g_c[gid];
    const int64_t np = p.n_pad;
    const int i0 = (xb * blockDim.x + threadIdx.x) * 4;
    if (c == 5) {
        if (!(GATES && APPLY) || i0 >= p.n) return;
        // a4 fused: dp = g l_p for log alpha > theta0 (R#6), p += dp
        const bool l1 = i0 + 1 < p.n, l2 = i0 + 2 < p.n, l3 = i0 + 3 < p.n;
        const float4 la = __ldg(reinterpret_cast<const float4*>(p.log_alpha + i0));
        float4 lp[3], pv[3];
#pragma unroll
        for (int dd = 0; dd < 3; ++dd) {
            lp[dd] = __ldg(reinterpret_cast<const float4*>(p.pregate + (int64_t)dd * np + i0));
            pv[dd] = *reinterpret_cast<const float4*>(p.planes + (int64_t)dd * np + i0);
        }
        const float lav[4] = {la.x, la.y, la.z, la.w};
        const bool live[4] = {true, l1, l2, l3};
        float g[4];
        bool on[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            on[j] = live[j] && (lav[j] > p.theta0);
            g[j] = on[j] ? gate_value(lav[j], p.tau, p.g0, p.g1) : 0.0f;
        }
#pragma unroll
        for (int dd = 0; dd < 3; ++dd) {
            float4 v = pv[dd];
            if (on[0]) v.x = v.x + g[0] * lp[dd].x;
            if (on[1]) v.y = v.y + g[1] * lp[dd].y;
            if (on[2]) v.z = v.z + g[2] * lp[dd].z;
            if (on[3]) v.w = v.w + g[3] * lp[dd].w;
            *reinterpret_cast<float4*>(p.planes + (int64_t)dd * np + i0) = v;
        }
        return;
    }
    const int L = p.lat[c];
    const int m0 = p.g_m0[gid], R = p.g_m1[gid] - m0;
    const int dbase = p.dec_off[c] + m0 * L;
    for (int j = threadIdx.x; j < R * L; j += blockDim.x) sdec[j] = p.decoders[dbase + j];
    __syncthreads();
    if (i0 >= p.n) return;
    const bool l1 = i0 + 1 < p.n, l2 = i0 + 2 < p.n, l3 = i0 + 3 < p.n;
    const int row0 = p.out_row0[c] + m0;
    if (L == 0) {
        if (p.resid_out)
            for (int m = 0; m < R; ++m)
                *reinterpret_cast<float4*>(p.resid_out + (int64_t)(row0 + m) * np + i0) = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
    const bool write_q = p.q_out && m0 == 0;  // one group per category writes the rounded latents
    bool bad = false;
    // the group's latents (4 Gaussians packed per register) and attribute rows, all loads issued
    // before any is used: one memory round trip per thread
    uint32_t q4[16];
    float4 av[DA_ROWS];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        if (k < L) {
            const int64_t off = (int64_t)(p.lat_row0[c] + k) * np + i0;
            if (F32) {
                // a1: l = round(l_hat), half away from zero (R#5); |l| <= 127 (R#4)
                float4 lh = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(p.latents) + off));
                float r0 = roundf(lh.x), r1 = roundf(lh.y), r2 = roundf(lh.z), r3 = roundf(lh.w);
                if (!(r0 >= -127.f && r0 <= 127.f)) { bad = true; r0 = r0 < 0.f ? -127.f : 127.f; }
                if (l1 && !(r1 >= -127.f && r1 <= 127.f)) { bad = true; r1 = r1 < 0.f ? -127.f : 127.f; }
                if (l2 && !(r2 >= -127.f && r2 <= 127.f)) { bad = true; r2 = r2 < 0.f ? -127.f : 127.f; }
                if (l3 && !(r3 >= -127.f && r3 <= 127.f)) { bad = true; r3 = r3 < 0.f ? -127.f : 127.f; }
                r1 = fminf(fmaxf(r1, -127.f), 127.f);
                r2 = fminf(fmaxf(r2, -127.f), 127.f);
                r3 = fminf(fmaxf(r3, -127.f), 127.f);
                const char4 c4 = make_char4((signed char)(int)r0, (signed char)(int)r1, (signed char)(int)r2,
                                            (signed char)(int)r3);
                q4[k] = *reinterpret_cast<const uint32_t*>(&c4);
            } else {
                q4[k] = __ldg(reinterpret_cast<const uint32_t*>(static_cast<const int8_t*>(p.latents) + off));
            }
            if (write_q) *reinterpret_cast<uint32_t*>(p.q_out + off) = q4[k];
        }
    }
    if (APPLY && !SET) {
#pragma unroll
        for (int u = 0; u < DA_ROWS; ++u)
            if (u < R) av[u] = *reinterpret_cast<const float4*>(p.planes + (int64_t)(3 + row0 + u) * np + i0);
    }
    // a2: r = D_c[m] . float(l), fmaf chain ascending k from +0 (R#7); k outermost, so
    // only one latent column is unpacked at a time
    float4 r[DA_ROWS];
#pragma unroll
    for (int u = 0; u < DA_ROWS; ++u) r[u] = make_float4(+0.0f, +0.0f, +0.0f, +0.0f);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        if (k < L) {
            const uint32_t w4 = q4[k];
            const float f0 = (float)(int8_t)(w4 & 0xffu), f1 = (float)(int8_t)((w4 >> 8) & 0xffu);
            const float f2 = (float)(int8_t)((w4 >> 16) & 0xffu), f3 = (float)(int8_t)(w4 >> 24);
#pragma unroll
            for (int u = 0; u < DA_ROWS; ++u) {
                if (u < R) {
                    const float w = sdec[u * L + k];
                    r[u].x = fmaf(w, f0, r[u].x);
                    r[u].y = fmaf(w, f1, r[u].y);
                    r[u].z = fmaf(w, f2, r[u].z);
                    r[u].w = fmaf(w, f3, r[u].w);
                }
            }
        }
    }
#pragma unroll
    for (int u = 0; u < DA_ROWS; ++u) {
        if (u >= R) break;
        const int row = row0 + u;
        if (p.resid_out) *reinterpret_cast<float4*>(p.resid_out + (int64_t)row * np + i0) = r[u];
        if (SET) {
            // first-frame "set" decode: A_0 = D . float(l), written, not added
            float4 v = *reinterpret_cast<const float4*>(&r[u]);
            if (!l1 || !l2 || !l3) {  // ragged tail: keep the padding columns as they are
                const float4 o = *reinterpret_cast<const float4*>(p.planes + (int64_t)(3 + row) * np + i0);
                if (!l1) v.y = o.y;
                if (!l2) v.z = o.z;
                if (!l3) v.w = o.w;
            }
            *reinterpret_cast<float4*>(p.planes + (int64_t)(3 + row) * np + i0) = v;
        } else if (APPLY) {
            // a3: A_t = A_{t-1} + r, separate add (R#7)
            float4 v = av[u];
            v.x = v.x + r[u].x;
            if (l1) v.y = v.y + r[u].y;
            if (l2) v.z = v.z + r[u].z;
            if (l3) v.w = v.w + r[u].w;
            *reinterpret_cast<float4*>(p.planes + (int64_t)(3 + row) * np + i0) = v;
        }
    }
    if (bad) raise_flag(p.fl, FLAG_LATENT_RANGE);
}

// a5: p[I_k] += E_p[k] for the COO position residual; validates the
// indices: idx < n and strictly increasing, else QUEEN_ERR_INDEX and skip.
__global__ void __launch_bounds__(256) k_coo_scatter(float* planes, int n, int n_pad, const uint32_t* idx,
                                                     const float* val, int kcap, const int32_t* kdev, DevFlags* fl,
                                                     uint32_t* idx_out, float* val_out, int32_t* k_out, int out_stride,
                                                     bool apply) {
    int k = kcap;
    if (kdev) k = min(max(*kdev, 0), kcap);
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j == 0 && k_out) *k_out = k;
    if (j >= k) return;
    const uint32_t i = idx[j];
    if (i >= (uint32_t)n || (j > 0 && i <= idx[j - 1])) {
        raise_flag(fl, FLAG_INDEX);
        return;
    }
    const float v0 = val[j], v1 = val[(int64_t)kcap + j], v2 = val[2 * (int64_t)kcap + j];
    if (apply) {
        planes[i] = planes[i] + v0;
        planes[(int64_t)n_pad + i] = planes[(int64_t)n_pad + i] + v1;
        planes[2 * (int64_t)n_pad + i] = planes[2 * (int64_t)n_pad + i] + v2;
    }
    if (idx_out) {
        idx_out[j] = i;
        val_out[j] = v0;
        val_out[(int64_t)out_stride + j] = v1;
        val_out[2 * (int64_t)out_stride + j] = v2;
    }
}

// ---- gate -> mask -> ascending COO compaction (decode_residuals, trainer state) ----
constexpr int GC_THREADS = 256, GC_ITEMS = 4, GC_TILE = GC_THREADS * GC_ITEMS;

__global__ void __launch_bounds__(GC_THREADS) k_gate_count(const float* la, int n, float theta0, uint32_t* counts) {
    __shared__ uint32_t warp_sum[GC_THREADS / 32];
    const int base = blockIdx.x * GC_TILE + threadIdx.x * GC_ITEMS;
    uint32_t c = 0;
    for (int j = 0; j < GC_ITEMS; ++j) c += (base + j < n && la[base + j] > theta0) ? 1u : 0u;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int w = 0; w < GC_THREADS / 32; ++w) s += warp_sum[w];
        counts[blockIdx.x] = s;
    }
}

// single block: exclusive scan of nb block counts -> offsets; writes total to k_out
__global__ void __launch_bounds__(1024) k_gate_scan(uint32_t* counts, int nb, int32_t* k_out) {
    __shared__ uint32_t carry;
    __shared__ uint32_t wsum[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += 1024) {
        const int j = base + threadIdx.x;
        uint32_t v = j < nb ? counts[j] : 0u;
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if ((threadIdx.x & 31) >= o) x += y;
        }
        if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
        __syncthreads();
        if (threadIdx.x < 32) {
            uint32_t w = wsum[threadIdx.x];
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (threadIdx.x >= o) w += y;
            }
            wsum[threadIdx.x] = w;
        }
        __syncthreads();
        const uint32_t incl = x + ((threadIdx.x >> 5) ? wsum[(threadIdx.x >> 5) - 1] : 0u);
        if (j < nb) counts[j] = carry + incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) *k_out = (int32_t)carry;
}

__global__ void __launch_bounds__(GC_THREADS) k_gate_write(const float* la, const float* pregate, int n, int n_pad,
                                                           float theta0, float tau, float g0, float g1,
                                                           const uint32_t* offsets, uint32_t* idx_out, float* val_out,
                                                           int out_stride) {
    __shared__ uint32_t wsum[GC_THREADS / 32];
    const int base = blockIdx.x * GC_TILE + threadIdx.x * GC_ITEMS;
    bool m[GC_ITEMS];
    uint32_t c = 0;
    for (int j = 0; j < GC_ITEMS; ++j) {
        m[j] = base + j < n && la[base + j] > theta0;
        c += m[j];
    }
    uint32_t x = c;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    uint32_t pre = 0;
    for (int q = 0; q < w; ++q) pre += wsum[q];
    uint32_t pos = offsets[blockIdx.x] + pre + x - c;
    for (int j = 0; j < GC_ITEMS; ++j) {
        if (!m[j]) continue;
        const int i = base + j;
        const float g = gate_value(la[i], tau, g0, g1);
        idx_out[pos] = (uint32_t)i;
        for (int d = 0; d < 3; ++d) val_out[(int64_t)d * out_stride + pos] = g * pregate[(int64_t)d * n_pad + i];
        ++pos;
    }
}

// ---------------------------------------------------------------------------
static void fill_params(const queen_packet& pk, DecodeParams& p) {
    const int B = (pk.sh_degree + 1) * (pk.sh_degree + 1);
    const int Mc[5] = {4, 3, 1, 3, 3 * (B - 1)};
    int lr = 0, dof = 0, orow = 0;
    for (int c = 0; c < 5; ++c) {
        p.lat[c] = pk.lat_dim[c];
        p.M[c] = Mc[c];
        p.lat_row0[c] = lr;
        p.dec_off[c] = dof;
        p.out_row0[c] = orow;
        lr += pk.lat_dim[c];
        dof += Mc[c] * pk.lat_dim[c];
        orow += Mc[c];
    }
    p.ndec = dof;
    p.n = pk.n;
    p.n_pad = pk.n_pad;
    p.latents = pk.latents;
    p.decoders = pk.decoders;
}

float host_theta0(float tau, float g0, float g1);

cudaError_t launch_decode_apply(const queen_packet& pk, float* planes, float* resid_out, int8_t* q_out,
                                bool apply_attrs, bool apply_pos, DevFlags* fl, cudaStream_t s) {
    DecodeParams p{};
    fill_params(pk, p);
    p.planes = planes;
    p.resid_out = resid_out;
    p.q_out = q_out;
    p.fl = fl;
    p.log_alpha = pk.log_alpha;
    p.pregate = pk.pos_pregate;
    p.tau = pk.tau;
    p.g0 = pk.gamma0;
    p.g1 = pk.gamma1;
    p.theta0 = host_theta0(pk.tau, pk.gamma0, pk.gamma1);
    const bool f32 = pk.latent_kind == QUEEN_LAT_F32;
    const bool gates = apply_pos && pk.pos_kind == QUEEN_POS_GATES;
    // work groups: each category's rows in balanced runs of <= DA_ROWS, then the gated positions
    int ng = 0, max_dec = 1;
    for (int c = 0; c < 5; ++c) {
        const int M = p.M[c], parts = (M + DA_ROWS - 1) / DA_ROWS;
        for (int q = 0; q < parts; ++q) {
            p.g_c[ng] = c;
            p.g_m0[ng] = (int)((int64_t)M * q / parts);
            p.g_m1[ng] = (int)((int64_t)M * (q + 1) / parts);
            max_dec = max(max_dec, (p.g_m1[ng] - p.g_m0[ng]) * p.lat[c]);
            ++ng;
        }
    }
    if (gates && apply_attrs) {
        p.g_c[ng] = 5; p.g_m0[ng] = 0; p.g_m1[ng] = 3;
        ++ng;
    }
    p.ngroups = ng;
    const int threads = 256;
    p.xblocks = (pk.n + 4 * threads - 1) / (4 * threads);
    p.sx = da_super(pk.n);
    const bool coo = apply_attrs && apply_pos && pk.pos_kind == QUEEN_POS_COO && pk.k > 0;
    int coo_blocks = 0;
    if (coo) {
        p.coo_k = pk.k;
        p.coo_kdev = pk.k_dev;
        p.coo_idx = pk.pos_idx;
        p.coo_val = pk.pos_val;
        coo_blocks = (pk.k + threads - 1) / threads;
    }
    const int64_t blocks = (int64_t)p.xblocks * ng + coo_blocks;
    const size_t smem = sizeof(float) * (size_t)max_dec;
    if (blocks > 0) {
        if (apply_attrs) {
            if (f32) {
                if (gates) k_decode_apply<true, true, true><<<(unsigned)blocks, threads, smem, s>>>(p);
                else k_decode_apply<true, true, false><<<(unsigned)blocks, threads, smem, s>>>(p);
            } else {
                if (gates) k_decode_apply<false, true, true><<<(unsigned)blocks, threads, smem, s>>>(p);
                else k_decode_apply<false, true, false><<<(unsigned)blocks, threads, smem, s>>>(p);
            }
        } else {
            if (f32) k_decode_apply<true, false, false><<<(unsigned)blocks, threads, smem, s>>>(p);
            else k_decode_apply<false, false, false><<<(unsigned)blocks, threads, smem, s>>>(p);
        }
    }
    if (apply_pos && !apply_attrs && pk.pos_kind == QUEEN_POS_COO && pk.k > 0) {
        const int kb = (pk.k + 255) / 256;
        k_coo_scatter<<<kb, 256, 0, s>>>(planes, pk.n, pk.n_pad, pk.pos_idx, pk.pos_val, pk.k, pk.k_dev, fl, nullptr,
                                         nullptr, nullptr, 0, true);
    }
    return cudaGetLastError();
}

// First-frame quantisation: frame 0's high-frequency SH coefficients (SH-rest,
// excluding DC) are stored as integer latents + a decoder and decoded ONCE, written absolutely:
// planes[14 + m][i] = sum_k D[m][k] float(l[k][i]) (fmaf chain ascending k from +0, R#7),
// m = 3 (b - 1) + ch.  Same kernel as the frame residuals (category 4 groups only, SET mode).
cudaError_t launch_set_sh_rest(float* planes, int n, int n_pad, int deg, const int8_t* latents, int L,
                               const float* decoder, DevFlags* fl, cudaStream_t s) {
    queen_packet pk{};
    pk.n = n;
    pk.n_pad = n_pad;
    pk.sh_degree = deg;
    pk.lat_dim[4] = L;
    pk.latent_kind = QUEEN_LAT_INT8;
    pk.latents = latents;
    pk.decoders = decoder;
    DecodeParams p{};
    fill_params(pk, p);
    p.planes = planes;
    p.fl = fl;
    const int M = p.M[4], parts = (M + DA_ROWS - 1) / DA_ROWS;
    int ng = 0, max_dec = 1;
    for (int q = 0; q < parts; ++q) {
        p.g_c[ng] = 4;
        p.g_m0[ng] = (int)((int64_t)M * q / parts);
        p.g_m1[ng] = (int)((int64_t)M * (q + 1) / parts);
        max_dec = max(max_dec, (p.g_m1[ng] - p.g_m0[ng]) * L);
        ++ng;
    }
    p.ngroups = ng;
    const int threads = 256;
    p.xblocks = (n + 4 * threads - 1) / (4 * threads);
    p.sx = da_super(n);
    const int64_t blocks = (int64_t)p.xblocks * ng;
    if (blocks > 0 && M > 0)
        k_decode_apply<false, true, false, true><<<(unsigned)blocks, threads, sizeof(float) * (size_t)max_dec, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_coo_copy(const queen_packet& pk, uint32_t* idx_out, float* val_out, int32_t* k_out, DevFlags* fl,
                            cudaStream_t s) {
    if (pk.k <= 0) {
        cudaMemsetAsync(k_out, 0, sizeof(int32_t), s);
        return cudaGetLastError();
    }
    const int kb = (pk.k + 255) / 256;
    k_coo_scatter<<<kb, 256, 0, s>>>(nullptr, pk.n, pk.n_pad, pk.pos_idx, pk.pos_val, pk.k, pk.k_dev, fl, idx_out,
                                     val_out, k_out, pk.n, false);
    return cudaGetLastError();
}

cudaError_t launch_gate_compact(const queen_packet& pk, uint32_t* idx_out, float* val_out, int32_t* k_out,
                                void* scratch, DevFlags* fl, cudaStream_t s) {
    (void)fl;
    const float th0 = host_theta0(pk.tau, pk.gamma0, pk.gamma1);
    const int nb = (pk.n + GC_TILE - 1) / GC_TILE;
    uint32_t* counts = static_cast<uint32_t*>(scratch);
    if (nb == 0) {
        cudaMemsetAsync(k_out, 0, sizeof(int32_t), s);
        return cudaGetLastError();
    }
    k_gate_count<<<nb, GC_THREADS, 0, s>>>(pk.log_alpha, pk.n, th0, counts);
    k_gate_scan<<<1, 1024, 0, s>>>(counts, nb, k_out);
    k_gate_write<<<nb, GC_THREADS, 0, s>>>(pk.log_alpha, pk.pos_pregate, pk.n, pk.n_pad, th0, pk.tau, pk.gamma0,
                                           pk.gamma1, counts, idx_out, val_out, pk.n);
    return cudaGetLastError();
}

}  // namespace queen
