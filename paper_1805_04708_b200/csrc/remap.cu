// remap.cu -- data movement of the all-to-all remap.
//
// A remap swaps m global bits g_i with m local bits l_i at once (planner op
// QSIM_OP_REMAP).  In block terms: the shard holding global value phi owns,
// for every value t of its l bits, the block B(t) = {x : x[l_i] = t_i}; after
// the remap, block B(t) of shard phi holds what was block B(phi[j]) of the
// shard phi' = phi with its j bits (j_i = g_i - nl) replaced by t -- a
// pairwise swap of equal blocks between shards that differ only in the j
// bits (block B(t) itself stays when t = phi[j]).  Every shard trades
// 2^nl (1 - 2^-m) amplitudes, once, instead of m pairwise half-shard swaps
// (PAPER.md:384-392 swaps one bit at a time).
//
// Kernels: k_blockswap (loopback: both blocks on this device, swapped in
// place), k_pack / k_unpack (NCCL: a block's chunk to / from a contiguous
// staging slot).  All move 16-byte vectors when the lowest l bit leaves runs
// of >= 16 bytes (E always; A when l_0 >= 3), else single elements.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace qsim {

static int rm_num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// insert the m block bits (positions pos[0] < pos[1] < ..., values from v) into w
__device__ __forceinline__ uint64_t rm_ins(uint64_t w, const RemapBlock &b, uint32_t v) {
    for (int i = 0; i < b.m; ++i) {
        const int p = b.pos[i];
        w = ((w >> p) << (p + 1)) | (w & ((1ull << p) - 1ull)) | ((uint64_t)((v >> i) & 1u) << p);
    }
    return w;
}

template <typename T>
__global__ void __launch_bounds__(256) k_blockswap(T *__restrict__ a, T *__restrict__ b, uint64_t n,
                                                   const __grid_constant__ RemapBlock blk, uint32_t va, uint32_t vb) {
    for (uint64_t x = (uint64_t)blockIdx.x * 256 + threadIdx.x; x < n; x += (uint64_t)gridDim.x * 256) {
        const uint64_t ia = rm_ins(x, blk, va), ib = rm_ins(x, blk, vb);
        const T ta = a[ia], tb = b[ib];
        a[ia] = tb;
        b[ib] = ta;
    }
}
template <typename T>
__global__ void __launch_bounds__(256) k_pack(const T *__restrict__ src, T *__restrict__ out, uint64_t base, uint64_t n,
                                              const __grid_constant__ RemapBlock blk, uint32_t v) {
    for (uint64_t x = (uint64_t)blockIdx.x * 256 + threadIdx.x; x < n; x += (uint64_t)gridDim.x * 256)
        out[x] = src[rm_ins(base + x, blk, v)];
}
template <typename T>
__global__ void __launch_bounds__(256) k_unpack(T *__restrict__ dst, const T *__restrict__ in, uint64_t base, uint64_t n,
                                                const __grid_constant__ RemapBlock blk, uint32_t v) {
    for (uint64_t x = (uint64_t)blockIdx.x * 256 + threadIdx.x; x < n; x += (uint64_t)gridDim.x * 256)
        dst[rm_ins(base + x, blk, v)] = in[x];
}

// all partners at once: slot p of out (count elements each) <- block v[p] of src
template <typename T>
__global__ void __launch_bounds__(256) k_pack_multi(const T *__restrict__ src, T *__restrict__ out, uint64_t base,
                                                    uint64_t count, const __grid_constant__ RemapBlock blk,
                                                    const __grid_constant__ RemapVals vals) {
    const uint64_t total = count * (uint64_t)vals.n;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < total; i += (uint64_t)gridDim.x * 256) {
        const uint64_t p = i / count, x = i - p * count;
        out[i] = src[rm_ins(base + x, blk, vals.v[p])];
    }
}
template <typename T>
__global__ void __launch_bounds__(256) k_unpack_multi(T *__restrict__ dst, const T *__restrict__ in, uint64_t base,
                                                      uint64_t count, const __grid_constant__ RemapBlock blk,
                                                      const __grid_constant__ RemapVals vals) {
    const uint64_t total = count * (uint64_t)vals.n;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < total; i += (uint64_t)gridDim.x * 256) {
        const uint64_t p = i / count, x = i - p * count;
        dst[rm_ins(base + x, blk, vals.v[p])] = in[i];
    }
}

static int rm_grid(uint64_t n) {
    const uint64_t cap = (uint64_t)rm_num_sms() * 8, need = (n + 255) / 256;
    return (int)(need < cap ? (need ? need : 1) : cap);
}

// vector view: 16-byte units when every block bit is at or above the unit's
// element count (shift = log2(16 / elem))
static bool rm_vec(const RemapBlock &b, size_t elem, RemapBlock &vb, int &shift) {
    shift = elem == 16 ? 0 : elem == 8 ? 1 : elem == 4 ? 2 : elem == 2 ? 3 : 4;
    if (b.pos[0] < shift) return false;
    vb = b;
    for (int i = 0; i < b.m; ++i) vb.pos[i] = b.pos[i] - shift;
    return true;
}

void launch_blockswap(void *a, void *b, uint64_t nblock, const RemapBlock &blk, uint32_t va, uint32_t vb,
                      size_t elem, cudaStream_t s) {
    RemapBlock v;
    int sh;
    if (rm_vec(blk, elem, v, sh)) {
        const uint64_t n = nblock >> sh;
        k_blockswap<uint4><<<rm_grid(n), 256, 0, s>>>((uint4 *)a, (uint4 *)b, n, v, va, vb);
    } else if (elem == 2) {
        k_blockswap<uint16_t><<<rm_grid(nblock), 256, 0, s>>>((uint16_t *)a, (uint16_t *)b, nblock, blk, va, vb);
    } else {
        k_blockswap<double2><<<rm_grid(nblock), 256, 0, s>>>((double2 *)a, (double2 *)b, nblock, blk, va, vb);
    }
}

void launch_pack(const void *src, void *out, uint64_t base, uint64_t count, const RemapBlock &blk, uint32_t v,
                 size_t elem, cudaStream_t s) {
    RemapBlock vb;
    int sh;
    if (rm_vec(blk, elem, vb, sh) && ((base | count) & ((1ull << sh) - 1)) == 0) {
        const uint64_t n = count >> sh;
        k_pack<uint4><<<rm_grid(n), 256, 0, s>>>((const uint4 *)src, (uint4 *)out, base >> sh, n, vb, v);
    } else if (elem == 2) {
        k_pack<uint16_t><<<rm_grid(count), 256, 0, s>>>((const uint16_t *)src, (uint16_t *)out, base, count, blk, v);
    } else {
        k_pack<double2><<<rm_grid(count), 256, 0, s>>>((const double2 *)src, (double2 *)out, base, count, blk, v);
    }
}

void launch_unpack(void *dst, const void *in, uint64_t base, uint64_t count, const RemapBlock &blk, uint32_t v,
                   size_t elem, cudaStream_t s) {
    RemapBlock vb;
    int sh;
    if (rm_vec(blk, elem, vb, sh) && ((base | count) & ((1ull << sh) - 1)) == 0) {
        const uint64_t n = count >> sh;
        k_unpack<uint4><<<rm_grid(n), 256, 0, s>>>((uint4 *)dst, (const uint4 *)in, base >> sh, n, vb, v);
    } else if (elem == 2) {
        k_unpack<uint16_t><<<rm_grid(count), 256, 0, s>>>((uint16_t *)dst, (const uint16_t *)in, base, count, blk, v);
    } else {
        k_unpack<double2><<<rm_grid(count), 256, 0, s>>>((double2 *)dst, (const double2 *)in, base, count, blk, v);
    }
}

void launch_pack_multi(const void *src, void *out, uint64_t base, uint64_t count, const RemapBlock &blk,
                       const RemapVals &vals, size_t elem, cudaStream_t s) {
    RemapBlock vb;
    int sh;
    if (rm_vec(blk, elem, vb, sh) && ((base | count) & ((1ull << sh) - 1)) == 0) {
        const uint64_t n = count >> sh;
        k_pack_multi<uint4><<<rm_grid(n * vals.n), 256, 0, s>>>((const uint4 *)src, (uint4 *)out, base >> sh, n, vb,
                                                                  vals);
    } else if (elem == 2) {
        k_pack_multi<uint16_t><<<rm_grid(count * vals.n), 256, 0, s>>>((const uint16_t *)src, (uint16_t *)out, base,
                                                                         count, blk, vals);
    } else {
        k_pack_multi<double2><<<rm_grid(count * vals.n), 256, 0, s>>>((const double2 *)src, (double2 *)out, base,
                                                                        count, blk, vals);
    }
}

void launch_unpack_multi(void *dst, const void *in, uint64_t base, uint64_t count, const RemapBlock &blk,
                         const RemapVals &vals, size_t elem, cudaStream_t s) {
    RemapBlock vb;
    int sh;
    if (rm_vec(blk, elem, vb, sh) && ((base | count) & ((1ull << sh) - 1)) == 0) {
        const uint64_t n = count >> sh;
        k_unpack_multi<uint4><<<rm_grid(n * vals.n), 256, 0, s>>>((uint4 *)dst, (const uint4 *)in, base >> sh, n, vb,
                                                                    vals);
    } else if (elem == 2) {
        k_unpack_multi<uint16_t><<<rm_grid(count * vals.n), 256, 0, s>>>((uint16_t *)dst, (const uint16_t *)in, base,
                                                                           count, blk, vals);
    } else {
        k_unpack_multi<double2><<<rm_grid(count * vals.n), 256, 0, s>>>((double2 *)dst, (const double2 *)in, base,
                                                                          count, blk, vals);
    }
}

}  // namespace qsim
