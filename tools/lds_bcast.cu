// Shared-memory wavefronts of one warp-wide 16-byte load by address pattern
// (ncu: l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum): does a
// warp-uniform LDS.128 (a broadcast) cost 1 wavefront?  mode 0: all lanes one
// address; 1: two addresses (lane bit 0); 2: two addresses (lane bit 4);
// 3: 32 distinct consecutive (4 wavefronts ideal).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double2 *out, int mode, int iters) {
    __shared__ double2 s[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s[i] = make_double2(i, -i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int idx = mode == 0 ? 5 : mode == 1 ? (lane & 1) : mode == 2 ? ((lane >> 4) & 1) : lane;
    double2 acc = make_double2(0, 0);
    for (int it = 0; it < iters; ++it) {
        double2 v;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(&s[(idx + it * 0) & 255])));
        acc.x += v.x;
        acc.y += v.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    double2 *o;
    cudaMalloc(&o, 1 << 20);
    for (int m = 0; m < 4; ++m) {
        k<<<1, 32>>>(o, m, 1000);
        cudaDeviceSynchronize();
    }
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
