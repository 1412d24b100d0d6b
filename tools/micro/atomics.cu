// Microbenchmark: shared-memory atomic throughput on sm_100a (design input for binning).
//   mode 0: each lane adds to bin (lane*stride + it) % BINS   (conflict-free when stride=1)
//   mode 1: random bins (hash)                               (bank conflicts + address conflicts)
//   mode 2: all lanes same bin                                (full conflict)
//   mode 3: warp-aggregated same bin (match_any + one add)
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE, int BINS>
__global__ void k_atoms(unsigned* out, int iters) {
    __shared__ unsigned h[BINS];
    for (int i = threadIdx.x; i < BINS; i += blockDim.x) h[i] = 0;
    __syncthreads();
    unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
    for (int it = 0; it < iters; ++it) {
        unsigned b;
        if (MODE == 0) b = (threadIdx.x + it) % BINS;
        else if (MODE == 1) { x = x * 1664525u + 1013904223u; b = (x >> 16) % BINS; }
        else b = it % BINS;
        if (MODE == 3) {
            unsigned m = __match_any_sync(0xffffffffu, b);
            if ((threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(&h[b], __popc(m));
        } else {
            atomicAdd(&h[b], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < BINS; i += blockDim.x) atomicAdd(&out[i], h[i]);
}

template <int MODE, int BINS>
float run(unsigned* out, int blocks, int threads, int iters) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    k_atoms<MODE, BINS><<<blocks, threads>>>(out, iters);
    cudaEventRecord(a);
    k_atoms<MODE, BINS><<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double lane_ops = (double)blocks * threads * iters;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("mode %d bins %5d: %.3f ms  %.2f lane-atomics/clk/SM\n", MODE, BINS, ms, lane_ops / cyc / sms);
    return ms;
}

// global RED contention: N updates spread over `addrs` addresses
__global__ void k_red(int* d, int addrs, int iters) {
    unsigned x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
    for (int it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
        atomicAdd(d + (x >> 8) % addrs, 1);
    }
}

int main() {
    unsigned* out; cudaMalloc(&out, 1 << 20);
    int blocks = 148 * 8, threads = 256, iters = 1024;
    run<0, 512>(out, blocks, threads, iters);
    run<1, 512>(out, blocks, threads, iters);
    run<1, 8192>(out, blocks, threads, iters);
    run<2, 512>(out, blocks, threads, iters);
    run<3, 512>(out, blocks, threads, iters);
    int* d; cudaMalloc(&d, 64 << 20);
    for (int addrs : {1024, 16384, 112000, 1 << 22}) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        k_red<<<148 * 8, 256>>>(d, addrs, 64);
        cudaEventRecord(a);
        k_red<<<148 * 8, 256>>>(d, addrs, 64);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("global RED over %8d addrs: %.3f ms  %.2f G/s\n", addrs, ms, 148.0 * 8 * 256 * 64 / ms / 1e6);
    }
    return 0;
}
