// Microbenchmark: does a predicated-off DADD cost FP64 pipe time on sm_100a?
//   plain:  per step 8 independent __dadd_rn (8 chains)
//   pred:   per step, per chain: @p add a / @!p add b  (16 issued, 8 effective)
//   sel:    per step, per chain: v = p ? a : b (2 SEL) then add (select form)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pred_dadd pred_dadd.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, int iters, double a, double b) {
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = threadIdx.x * 1e-9 + j;
    const unsigned key = (threadIdx.x * 2654435761u) >> 7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const unsigned ck = (key + 97u * j + 13u * it) & 0xffffu;
            if (MODE == 0) {
                acc[j] = __dadd_rn(acc[j], a);
            } else if (MODE == 1) {
                asm volatile("{\n .reg .pred p;\n setp.le.u32 p, %1, 32768;\n @p add.rn.f64 %0, %0, %2;\n @!p add.rn.f64 %0, %0, %3;\n}"
                             : "+d"(acc[j]) : "r"(ck), "d"(a), "d"(b));
            } else {
                const double v = ck <= 32768u ? a : b;
                acc[j] = __dadd_rn(acc[j], v);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
        for (int mode = 0; mode < 3; ++mode) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, threads>>>(out, iters, 1.5, 2.5);
            if (mode == 1) k<1><<<blocks, threads>>>(out, iters, 1.5, 2.5);
            if (mode == 2) k<2><<<blocks, threads>>>(out, iters, 1.5, 2.5);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double adds = double(blocks) * threads * iters * 8;
            printf("mode %s: %.3f ms, %.3e effective adds/s\n", mode == 0 ? "plain" : (mode == 1 ? "pred " : "sel  "), ms,
                   adds / (ms * 1e-3));
        }
    }
    return 0;
}
