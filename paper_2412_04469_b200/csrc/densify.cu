// NEXT #2: densification deltas in the stream.  The paper applies the 3D-GS
// densification stage at every time-step but does not say how a decoder
// reproduces it; the stream carries, per frame, the indices of removed Gaussians and the full
// attributes of added ones (DESIGN reading R21, after SPEC's codec additions/removals
// sections).  queen_densify builds A'_t = (A_t without the removed columns, order kept)
// followed by the additions, into a second SoA buffer:
//   k_densify_keep  one thread per source column: removed iff it is in the sorted list
//                   (binary search); kept columns move to i - #(removed < i), all planes
//   k_densify_add   one thread per destination column >= kept count: additions (binary16 ->
//                   fp32, exact) then zero padding
#include <cuda_fp16.h>

#include "queen_internal.cuh"

namespace queen {

__global__ void __launch_bounds__(256) k_densify_keep(const float* __restrict__ src, int n_old, int np_src,
                                                      const uint32_t* __restrict__ rem, int n_rem, int P,
                                                      float* __restrict__ dst, int np_dst, DevFlags* fl) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_rem && (rem[i] >= (uint32_t)n_old || (i > 0 && rem[i] <= rem[i - 1]))) raise_flag(fl, FLAG_INDEX);
    if (i >= n_old) return;
    // c = #(rem < i): first position with rem[pos] >= i
    int lo = 0, hi = n_rem;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (rem[mid] < (uint32_t)i) lo = mid + 1; else hi = mid;
    }
    if (lo < n_rem && rem[lo] == (uint32_t)i) return;  // removed
    const int j = i - lo;
    // a valid list puts every kept column below n_old - n_rem; a bad one (duplicate, unsorted or
    // out-of-range entries, already flagged above) must not write into the additions or past
    // the destination's n_pad
    if (j >= n_old - n_rem) return;
    for (int p = 0; p < P; ++p) dst[(int64_t)p * np_dst + j] = src[(int64_t)p * np_src + i];
}

__global__ void __launch_bounds__(256) k_densify_add(const __half* __restrict__ add, int n_add, int n_kept, int P,
                                                     float* __restrict__ dst, int np_dst) {
    const int c = n_kept + blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= np_dst) return;
    const int a = c - n_kept;
    for (int p = 0; p < P; ++p)
        dst[(int64_t)p * np_dst + c] = a < n_add ? __half2float(add[(int64_t)p * n_add + a]) : 0.0f;
}

cudaError_t launch_densify(const float* src, int n_old, int np_src, const uint32_t* rem, int n_rem, const void* add,
                           int n_add, int P, float* dst, int np_dst, DevFlags* fl, cudaStream_t s) {
    const int nk = n_old > n_rem ? n_old : n_rem;
    if (nk > 0)
        k_densify_keep<<<(nk + 255) / 256, 256, 0, s>>>(src, n_old, np_src, rem, n_rem, P, dst, np_dst, fl);
    const int n_kept = n_old - n_rem;
    const int tail = np_dst - n_kept;
    if (tail > 0)
        k_densify_add<<<(tail + 255) / 256, 256, 0, s>>>(static_cast<const __half*>(add), n_add, n_kept, P, dst, np_dst);
    return cudaGetLastError();
}

}  // namespace queen
