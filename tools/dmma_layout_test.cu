// Verifies the m8n8k4 f64 fragment layout assumed by the pass kernel:
// A[r][k]: lane (r = lane>>2, k = lane&3); B[k][n]: lane (k = lane&3, n = lane>>2);
// D[r][n]: lane (r = lane>>2, n = 2(lane&3) + i).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(const double *A, const double *B, double *D) {
    int lane = threadIdx.x, r = lane >> 2, c = lane & 3;
    double a = A[r * 4 + c];
    double b = B[c * 8 + r];
    double d0 = 0, d1 = 0;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    D[r * 8 + 2 * c] = d0;
    D[r * 8 + 2 * c + 1] = d1;
}
int main() {
    double hA[32], hB[32], hD[64], ref[64];
    for (int i = 0; i < 32; ++i) { hA[i] = 1.0 + i * 0.37; hB[i] = -2.0 + i * 0.11; }
    for (int r = 0; r < 8; ++r)
        for (int n = 0; n < 8; ++n) {
            double s = 0;
            for (int kk = 0; kk < 4; ++kk) s += hA[r * 4 + kk] * hB[kk * 8 + n];
            ref[r * 8 + n] = s;
        }
    double *dA, *dB, *dD;
    cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dD, 512);
    cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dA, dB, dD);
    cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
    printf("max err %.3e %s\n", err, err < 1e-12 ? "LAYOUT OK" : "LAYOUT MISMATCH");
    return 0;
}
