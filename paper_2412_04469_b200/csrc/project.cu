// K2: multi-view projection (Eq. 1) + SH colour.
//
// One thread per Gaussian reads its attributes ONCE (11 + 3B planes, coalesced
// per plane) and loops over every view of the batch, so the SoA is streamed from
// HBM once per frame instead of once per view.  Cameras arrive by value in the
// kernel parameters (<= 64 x 96 B).  Output per (view, Gaussian): a 48-byte blend
// record (3 x float4, coalesced), depth bits, tiles touched and the tile rect.
// Arithmetic follows DESIGN.md "Arithmetic contract" line by line (no FMA
// contraction; fmaf only where written) so every field is bit-identical to the
// oracle's.
#include "queen_internal.cuh"

namespace queen {

__device__ __forceinline__ void sh_basis(int deg, float x, float y, float z, float* Y) {
    // 3D-GS real SH constants / signs (R#10), degree <= 3
    const float C0 = 0.28209479177387814f;
    const float C1 = 0.4886025119029199f;
    Y[0] = C0;
    if (deg < 1) return;
    Y[1] = -C1 * y;
    Y[2] = C1 * z;
    Y[3] = -C1 * x;
    if (deg < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    Y[4] = 1.0925484305920792f * xy;
    Y[5] = -1.0925484305920792f * yz;
    Y[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
    Y[7] = -1.0925484305920792f * xz;
    Y[8] = 0.5462742152960396f * (xx - yy);
    if (deg < 3) return;
    Y[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    Y[10] = 2.890611442640554f * xy * z;
    Y[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
    Y[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    Y[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
    Y[14] = 1.445305721320277f * z * (xx - yy);
    Y[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
}

template <int DEG>
__global__ void __launch_bounds__(128) k_project(const float* __restrict__ planes, int n, int n_pad, const CamBatch cams,
                                                 int n_views, float4* __restrict__ rec, uint32_t* __restrict__ depth,
                                                 uint32_t* __restrict__ tiles, short4* __restrict__ rect,
                                                 const uint8_t* __restrict__ select, DevFlags* fl) {
    constexpr int B = (DEG + 1) * (DEG + 1);
    constexpr int P = 11 + 3 * B;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_pad) return;
    const int64_t np = n_pad;
    if (i >= n) {  // padding columns: zero records, zero tiles
        for (int v = 0; v < n_views; ++v) {
            const int64_t o = (int64_t)v * np + i;
            rec[o * 3 + 0] = rec[o * 3 + 1] = rec[o * 3 + 2] = make_float4(0.f, 0.f, 0.f, 0.f);
            depth[o] = 0u;
            tiles[o] = 0u;
            rect[o] = make_short4(0, 0, 0, 0);
        }
        return;
    }
    float a[P];
#pragma unroll
    for (int p = 0; p < P; ++p) a[p] = __ldg(planes + (int64_t)p * np + i);
    // 0. non-finite input -> cull + QUEEN_WARN_NONFINITE (before any fminf/fmaxf)
    bool finite = true;
#pragma unroll
    for (int p = 0; p < P; ++p) finite = finite && isfinite(a[p]);
    // view-independent part: normalised quaternion, R(q) S, Sigma, opacity
    float S[9], o = 0.f, e2 = 0.f;
    // render_mask: Gaussians outside the requested subset are culled like invisible ones
    bool live = finite && (select == nullptr || select[i] != 0);
    if (live) {
        float qw = a[3], qx = a[4], qy = a[5], qz = a[6];
        const float n2 = fmaf(qw, qw, fmaf(qx, qx, fmaf(qy, qy, qz * qz)));
        live = n2 > 0.0f;
        const float inv = 1.0f / sqrtf(n2);
        qw = qw * inv; qx = qx * inv; qy = qy * inv; qz = qz * inv;
        const float s0 = det_exp(a[7]), s1 = det_exp(a[8]), s2 = det_exp(a[9]);
        float Rq[9];
        Rq[0] = 1.0f - 2.0f * fmaf(qy, qy, qz * qz);
        Rq[1] = 2.0f * (qx * qy - qw * qz);
        Rq[2] = 2.0f * (qx * qz + qw * qy);
        Rq[3] = 2.0f * (qx * qy + qw * qz);
        Rq[4] = 1.0f - 2.0f * fmaf(qx, qx, qz * qz);
        Rq[5] = 2.0f * (qy * qz - qw * qx);
        Rq[6] = 2.0f * (qx * qz - qw * qy);
        Rq[7] = 2.0f * (qy * qz + qw * qx);
        Rq[8] = 1.0f - 2.0f * fmaf(qx, qx, qy * qy);
        float Mm[9];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            Mm[j * 3 + 0] = Rq[j * 3 + 0] * s0;
            Mm[j * 3 + 1] = Rq[j * 3 + 1] * s1;
            Mm[j * 3 + 2] = Rq[j * 3 + 2] * s2;
        }
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = j; k < 3; ++k) {
                const float v = fmaf(Mm[j * 3 + 0], Mm[k * 3 + 0], fmaf(Mm[j * 3 + 1], Mm[k * 3 + 1], Mm[j * 3 + 2] * Mm[k * 3 + 2]));
                S[j * 3 + k] = v;
                S[k * 3 + j] = v;
            }
        o = 1.0f / (1.0f + det_exp(-a[10]));
        live = live && (255.0f * o > 1.0f);
        if (live) e2 = 2.0f * det_log(255.0f * o);
    }
    const float px = a[0], py = a[1], pz = a[2];
    for (int v = 0; v < n_views; ++v) {
        const queen_camera& c = cams.cam[v];
        const int64_t oidx = (int64_t)v * np + i;
        float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0, r2 = r0;
        uint32_t dbits = 0u, nt = 0u;
        short4 rc = make_short4(0, 0, 0, 0);
        bool ok = live;
        float xc = 0.f, yc = 0.f, zc = 1.f;
        if (ok) {
            const float* Rw = c.R;
            xc = fmaf(Rw[0], px, fmaf(Rw[1], py, fmaf(Rw[2], pz, c.t[0])));
            yc = fmaf(Rw[3], px, fmaf(Rw[4], py, fmaf(Rw[5], pz, c.t[1])));
            zc = fmaf(Rw[6], px, fmaf(Rw[7], py, fmaf(Rw[8], pz, c.t[2])));
            ok = zc > c.near_z;
        }
        float a2 = 0.f, b2 = 0.f, c2 = 0.f, sxx = 0.f, syy = 0.f, tx = 0.f, ty = 0.f;
        if (ok) {
            const float* Rw = c.R;
            const float iz = 1.0f / zc;  // one reciprocal of z_c (DESIGN "Arithmetic contract")
            tx = xc * iz;
            ty = yc * iz;
            const float j00 = c.fx * iz;
            const float j02 = -(c.fx * fminf(c.limx, fmaxf(-c.limx, tx))) * iz;
            const float j11 = c.fy * iz;
            const float j12 = -(c.fy * fminf(c.limy, fmaxf(-c.limy, ty))) * iz;
            float A[6];
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                A[m] = fmaf(j00, Rw[m], j02 * Rw[6 + m]);
                A[3 + m] = fmaf(j11, Rw[3 + m], j12 * Rw[6 + m]);
            }
            float Bm[6];
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int m = 0; m < 3; ++m)
                    Bm[r * 3 + m] = fmaf(A[r * 3 + 0], S[m], fmaf(A[r * 3 + 1], S[3 + m], A[r * 3 + 2] * S[6 + m]));
            float sa = fmaf(Bm[0], A[0], fmaf(Bm[1], A[1], Bm[2] * A[2]));
            const float sb = fmaf(Bm[0], A[3], fmaf(Bm[1], A[4], Bm[2] * A[5]));
            float sc = fmaf(Bm[3], A[3], fmaf(Bm[4], A[4], Bm[5] * A[5]));
            sa = sa + 0.3f;
            sc = sc + 0.3f;
            const float det = fmaf(sa, sc, -(sb * sb));
            ok = det > 0.0f;
            if (ok) {
                const float idet = 1.0f / det;
                a2 = sc * idet;   // conic xx
                b2 = -sb * idet;  // conic xy
                c2 = sa * idet;   // conic yy
                sxx = sa;         // Sigma'_xx (incl. the 0.3 dilation)
                syy = sc;
            }
        }
        if (ok) {
            // opacity-aware extent (R#13): tight bounding box of d^T S'^-1 d <= e2, 1e-4 slack
            const float hx = 1.0001f * sqrtf(e2 * sxx);
            const float hy = 1.0001f * sqrtf(e2 * syy);
            const float rx = ceilf(hx), ry = ceilf(hy);
            const float u = fmaf(c.fx, tx, c.cx);
            const float vv = fmaf(c.fy, ty, c.cy);
            const int gx = (c.width + 15) / 16, gy = (c.height + 15) / 16;
            const float ftx0 = fminf(fmaxf(ceilf(((u - rx) - 15.0f) * 0.0625f), 0.0f), (float)gx);
            const float ftx1 = fminf(fmaxf(floorf((u + rx) * 0.0625f), -1.0f), (float)(gx - 1));
            const float fty0 = fminf(fmaxf(ceilf(((vv - ry) - 15.0f) * 0.0625f), 0.0f), (float)gy);
            const float fty1 = fminf(fmaxf(floorf((vv + ry) * 0.0625f), -1.0f), (float)(gy - 1));
            const int tx0 = (int)ftx0, tx1 = (int)ftx1, ty0 = (int)fty0, ty1 = (int)fty1;
            nt = (tx0 <= tx1 && ty0 <= ty1) ? (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1)) : 0u;
            const float L2E = 1.4426950408889634f;
            r0 = make_float4(u, vv, hx, hy);
            r1 = make_float4((-0.5f * a2) * L2E, (-b2) * L2E, (-0.5f * c2) * L2E, -(0.5f * e2) * L2E);
            // colour: dir = (p - C)/|p - C|, rgb = max(0, sum Y_b h_b + 0.5) (R#8, R#10)
            float dx = px - c.C[0], dy = py - c.C[1], dz = pz - c.C[2];
            const float dn = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
            const float idn = 1.0f / dn;
            dx = dx * idn; dy = dy * idn; dz = dz * idn;
            float Y[16];
            sh_basis(DEG, dx, dy, dz, Y);
            float rgb[3];
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                float acc = Y[0] * a[11 + ch];
#pragma unroll
                for (int b = 1; b < B; ++b) acc = fmaf(Y[b], a[11 + 3 * b + ch], acc);
                rgb[ch] = fmaxf(0.0f, acc + 0.5f);
            }
            r2 = make_float4(o, rgb[0], rgb[1], rgb[2]);
            dbits = __float_as_uint(zc);
            rc = make_short4((short)tx0, (short)ty0, (short)tx1, (short)ty1);
        }
        rec[oidx * 3 + 0] = r0;
        rec[oidx * 3 + 1] = r1;
        rec[oidx * 3 + 2] = r2;
        depth[oidx] = dbits;
        tiles[oidx] = nt;
        rect[oidx] = rc;
    }
    if (!finite) raise_flag(fl, FLAG_NONFINITE);
}

cudaError_t launch_project(const float* planes, int n, int n_pad, int deg, const CamBatch& cams, int n_views,
                           float* rec, uint32_t* depth, uint32_t* tiles, int16_t* rect, const uint8_t* select,
                           DevFlags* fl, cudaStream_t s) {
    const int threads = 128;
    const int blocks = (n_pad + threads - 1) / threads;
    if (blocks == 0) return cudaSuccess;
    float4* r = reinterpret_cast<float4*>(rec);
    short4* rc = reinterpret_cast<short4*>(rect);
    switch (deg) {
        case 0: k_project<0><<<blocks, threads, 0, s>>>(planes, n, n_pad, cams, n_views, r, depth, tiles, rc, select, fl); break;
        case 1: k_project<1><<<blocks, threads, 0, s>>>(planes, n, n_pad, cams, n_views, r, depth, tiles, rc, select, fl); break;
        case 2: k_project<2><<<blocks, threads, 0, s>>>(planes, n, n_pad, cams, n_views, r, depth, tiles, rc, select, fl); break;
        default: k_project<3><<<blocks, threads, 0, s>>>(planes, n, n_pad, cams, n_views, r, depth, tiles, rc, select, fl); break;
    }
    return cudaGetLastError();
}

}  // namespace queen
