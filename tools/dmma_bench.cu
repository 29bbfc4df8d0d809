// Micro-benchmark: FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput alone and concurrent with DFMA.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH, int FMA>
__global__ void k(double *out, int iters, double x) {
    double acc[CH][2];
    double f[FMA > 0 ? FMA : 1];
    for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-3 + i;
    for (int i = 0; i < FMA; ++i) f[i] = i;
    double a = x, b = x * 0.5;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) dmma(acc[i][0], acc[i][1], a, b);
#pragma unroll
        for (int i = 0; i < FMA; ++i) f[i] = fma(f[i], x, b);
    }
    double s = 0;
    for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
    for (int i = 0; i < FMA; ++i) s += f[i];
    if (s == 1.2345) out[0] = s;
}
template <int CH, int FMA>
void run(int warps, double *d) {
    int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<CH, FMA><<<148, warps * 32>>>(d, 10, 1.0000001);
    cudaEventRecord(e0);
    k<CH, FMA><<<148, warps * 32>>>(d, iters, 1.0000001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double mma_flops = 148.0 * warps * (double)iters * CH * (8 * 8 * 4 * 2);  // per warp-level mma
    double fma_flops = 148.0 * warps * 32 * (double)iters * FMA * 2;
    printf("warps %2d chains %d fma/iter %d : DMMA %.2f TFLOP/s + DFMA %.2f TFLOP/s = %.2f\n", warps, CH, FMA,
           mma_flops / (ms * 1e-3) / 1e12, fma_flops / (ms * 1e-3) / 1e12, (mma_flops + fma_flops) / (ms * 1e-3) / 1e12);
}
int main() {
    double *d;
    cudaMalloc(&d, 64);
    run<4, 0>(8, d);
    run<8, 0>(8, d);
    run<8, 0>(16, d);
    run<4, 4>(8, d);
    run<4, 8>(8, d);
    run<8, 8>(16, d);
    run<2, 8>(16, d);
    return 0;
}
