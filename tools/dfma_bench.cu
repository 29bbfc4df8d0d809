// Micro-benchmark: DFMA throughput per SM vs warps per SM and independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void k(double *out, int iters, double b, double c) {
    double a[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += a[i];
    if (s == 1.2345) out[0] = s;
}
template <int ILP>
void run(int warps, double *d) {
    int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<ILP><<<148, warps * 32>>>(d, 10, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    k<ILP><<<148, warps * 32>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = 148.0 * warps * 32 * (double)iters * ILP;
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double per_clk_sm = ops / (ms * 1e-3) / 148 / (clk * 1e3);
    printf("warps/SM %2d ILP %d : %.1f DFMA/clk/SM (%.2f TFLOP/s)\n", warps, ILP, per_clk_sm, ops * 2 / (ms * 1e-3) / 1e12);
}
int main() {
    double *d;
    cudaMalloc(&d, 64);
    for (int w : {1, 2, 4, 8, 12, 16, 32}) {
        run<1>(w, d);
        run<2>(w, d);
        run<4>(w, d);
        run<8>(w, d);
    }
    return 0;
}
