// K1 / K1b: fused residual decode + apply (Eq. 4-5) and the
// position step (hard-concrete gate P:329-336, COO P:1389-1390).
//
// One coalesced, vectorised pass over the Gaussian SoA: each thread owns 4
// consecutive Gaussians, so every latent row is one 4-byte char4 load and every
// attribute row one 16-byte float4 load + store per thread (a warp moves 128 B of
// latents and 512 B of attributes per row).  The decoders (<= 896 floats) sit in
// shared memory and are read as warp-uniform broadcasts.  HBM-bound: bytes per
// Gaussian = sum L_c (int8) + 2*4*sum M_c (fp32 read+write), K1.
#include "queen_internal.cuh"

namespace queen {

constexpr int DA_CHUNK = 4;  // attribute rows per batch of loads (rows in flight per warp)

struct DecodeParams {
    int n, n_pad;
    int lat[5], M[5], lat_row0[5], dec_off[5], out_row0[5];
    int ndec;
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

template <bool F32, bool APPLY, bool GATES>
__global__ void __launch_bounds__(256) k_decode_apply(DecodeParams p) {
    extern __shared__ float sdec[];
    for (int j = threadIdx.x; j < p.ndec; j += blockDim.x) sdec[j] = p.decoders[j];
    __syncthreads();
    const int i0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i0 >= p.n) return;
    const bool l1 = i0 + 1 < p.n, l2 = i0 + 2 < p.n, l3 = i0 + 3 < p.n;
    const int64_t np = p.n_pad;
    bool bad = false;
#pragma unroll 1
    for (int c = 0; c < 5; ++c) {
        const int L = p.lat[c], M = p.M[c];
        if (L == 0) {
            if (p.resid_out)
                for (int m = 0; m < M; ++m)
                    *reinterpret_cast<float4*>(p.resid_out + (int64_t)(p.out_row0[c] + m) * np + i0) =
                        make_float4(0.f, 0.f, 0.f, 0.f);
            continue;
        }
        float ql[16][4];
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
                    ql[k][0] = r0; ql[k][1] = r1; ql[k][2] = r2; ql[k][3] = r3;
                    if (p.q_out)
                        *reinterpret_cast<char4*>(p.q_out + off) =
                            make_char4((signed char)(int)r0, (signed char)(int)r1, (signed char)(int)r2,
                                       (signed char)(int)r3);
                } else {
                    char4 q4 = __ldg(reinterpret_cast<const char4*>(static_cast<const int8_t*>(p.latents) + off));
                    ql[k][0] = (float)q4.x; ql[k][1] = (float)q4.y; ql[k][2] = (float)q4.z; ql[k][3] = (float)q4.w;
                    if (p.q_out) *reinterpret_cast<char4*>(p.q_out + off) = q4;
                }
            }
        }
        // rows in chunks of DA_CHUNK: the chunk's attribute loads are issued together (memory-
        // level parallelism: DA_CHUNK x 512 B in flight per warp instead of one row at a time)
#pragma unroll 1
        for (int m0 = 0; m0 < M; m0 += DA_CHUNK) {
            float4 av[DA_CHUNK];
            if (APPLY) {
#pragma unroll
                for (int u = 0; u < DA_CHUNK; ++u)
                    if (m0 + u < M)
                        av[u] = *reinterpret_cast<const float4*>(p.planes + (int64_t)(3 + p.out_row0[c] + m0 + u) * np + i0);
            }
#pragma unroll
            for (int u = 0; u < DA_CHUNK; ++u) {
                const int m = m0 + u;
                if (m >= M) break;
                // a2: r = D_c[m] . float(l), fmaf chain ascending k from +0 (R#7)
                const float* d = sdec + p.dec_off[c] + m * L;
                float r0 = +0.0f, r1 = +0.0f, r2 = +0.0f, r3 = +0.0f;
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    if (k < L) {
                        const float w = d[k];
                        r0 = fmaf(w, ql[k][0], r0);
                        r1 = fmaf(w, ql[k][1], r1);
                        r2 = fmaf(w, ql[k][2], r2);
                        r3 = fmaf(w, ql[k][3], r3);
                    }
                }
                const int row = p.out_row0[c] + m;
                if (p.resid_out)
                    *reinterpret_cast<float4*>(p.resid_out + (int64_t)row * np + i0) = make_float4(r0, r1, r2, r3);
                if (APPLY) {
                    // a3: A_t = A_{t-1} + r, separate add (R#7)
                    float4 v = av[u];
                    v.x = v.x + r0;
                    if (l1) v.y = v.y + r1;
                    if (l2) v.z = v.z + r2;
                    if (l3) v.w = v.w + r3;
                    *reinterpret_cast<float4*>(p.planes + (int64_t)(3 + row) * np + i0) = v;
                }
            }
        }
    }
    if (GATES && APPLY) {
        // a4 fused: dp = g l_p for log alpha > theta0 (R#6), p += dp
        const float4 la = __ldg(reinterpret_cast<const float4*>(p.log_alpha + i0));
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
            const float4 lp = __ldg(reinterpret_cast<const float4*>(p.pregate + (int64_t)dd * np + i0));
            float4* a = reinterpret_cast<float4*>(p.planes + (int64_t)dd * np + i0);
            float4 v = *a;
            if (on[0]) v.x = v.x + g[0] * lp.x;
            if (on[1]) v.y = v.y + g[1] * lp.y;
            if (on[2]) v.z = v.z + g[2] * lp.z;
            if (on[3]) v.w = v.w + g[3] * lp.w;
            *a = v;
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
    const int groups = (pk.n + 3) / 4;
    const int threads = 256;
    const int blocks = (groups + threads - 1) / threads;
    const size_t smem = sizeof(float) * (size_t)(p.ndec > 0 ? p.ndec : 1);
    if (blocks > 0) {
        if (apply_attrs) {
            if (f32) {
                if (gates) k_decode_apply<true, true, true><<<blocks, threads, smem, s>>>(p);
                else k_decode_apply<true, true, false><<<blocks, threads, smem, s>>>(p);
            } else {
                if (gates) k_decode_apply<false, true, true><<<blocks, threads, smem, s>>>(p);
                else k_decode_apply<false, true, false><<<blocks, threads, smem, s>>>(p);
            }
        } else {
            if (f32) k_decode_apply<true, false, false><<<blocks, threads, smem, s>>>(p);
            else k_decode_apply<false, false, false><<<blocks, threads, smem, s>>>(p);
        }
    }
    if (apply_pos && pk.pos_kind == QUEEN_POS_COO && pk.k > 0) {
        const int kb = (pk.k + 255) / 256;
        k_coo_scatter<<<kb, 256, 0, s>>>(planes, pk.n, pk.n_pad, pk.pos_idx, pk.pos_val, pk.k, pk.k_dev, fl, nullptr,
                                         nullptr, nullptr, 0, true);
    }
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
