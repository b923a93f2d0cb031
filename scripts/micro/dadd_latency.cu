// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro/dadd_latency scripts/micro/dadd_latency.cu
// Measured (B200, round 1): 1 warp/SMSP x 1 chain = 21 % of the FP64 pipe (add latency ~9 cycles);
// 1 warp/SMSP x 4 chains = 86 %, x 9 chains = 92 %; 4 warps/SMSP x 9 chains = 99 %.
// FP64 add latency / per-warp issue on B200: W warps per SM, K independent
// __dadd_rn chains per thread.  adds/s per SM vs (W, K) shows how much ILP a
// warp needs to keep the FP64 pipe busy (the accumulate kernel has CPL = 9).
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void chains(double* out, int iters, double step) {
    double a[K];
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < K; ++k) a[k] = __dadd_rn(a[k], step);
    }
    double r = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) r += a[k];
    if (r == 1.2345) out[blockIdx.x] = r;
}

template <int K>
void run(int warps_per_sm, double* out) {
    int sms = 148, iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    chains<K><<<sms, 32 * warps_per_sm>>>(out, 100, 1e-9);
    cudaEventRecord(a);
    chains<K><<<sms, 32 * warps_per_sm>>>(out, iters, 1e-9);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double adds = double(sms) * 32 * warps_per_sm * K * iters;
    printf("warps/SM %2d chains %2d: %.3e adds/s (%.1f%% of 64/SM/clk at 1.965 GHz)\n", warps_per_sm, K, adds / (ms * 1e-3),
           100.0 * adds / (ms * 1e-3) / (148 * 64 * 1.965e9));
}

int main() {
    double* out;
    cudaMalloc(&out, 4096 * sizeof(double));
    for (int w : {4, 8, 16, 24}) {
        run<1>(w, out);
        run<2>(w, out);
        run<4>(w, out);
        run<9>(w, out);
        run<18>(w, out);
    }
    return 0;
}
