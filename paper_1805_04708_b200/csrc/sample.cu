// sample.cu -- GENERATE EVENTS (App. B): draw basis states
// from |a|^2 by inverse-CDF sampling in LOGICAL index order.
//
// 1. p[L] = |a(phys(L))|^2 for every logical index L (one pass over each shard,
//    decoded for A);
// 2. a tree of block sums (1024 children per node, fixed summation order);
// 3. one warp per event: u_k = (splitmix64(seed + k) >> 11) 2^-53, target
//    t = u_k * total; descend the tree, at each level scanning the 1024 children
//    of the current node with a warp prefix sum and taking the first child whose
//    running sum exceeds the remaining target.
// Deterministic for a given state, seed and count.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "internal.h"
#include "kernels.h"
#include "kernels_a.h"

namespace qsim {

constexpr int FANOUT = 1024;

__device__ __forceinline__ uint64_t phys_to_logical_s(uint64_t phys, const int *inv, int nq) {
    uint64_t L = 0;
    for (int b = 0; b < nq; ++b)
        if ((phys >> b) & 1ull) L |= 1ull << inv[b];
    return L;
}

__global__ void k_prob_logical_e(const double2 *__restrict__ a, uint64_t n, uint64_t base,
                                 const int *__restrict__ inv, int nq, double *__restrict__ p) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double2 v = a[i];
        p[phys_to_logical_s(base | i, inv, nq)] = fma(v.x, v.x, v.y * v.y);
    }
}

// A: |decode(code)|^2 = r(b0)^2 (cos^2 + sin^2 = 1 up to rounding; computed as the decoded value's square)
__global__ void k_prob_logical_a(const uint16_t *__restrict__ a, uint64_t n, uint64_t base,
                                 const int *__restrict__ inv, int nq, const ATabData *__restrict__ t,
                                 double *__restrict__ p) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = a[i];
        const int b0i = (int)(c & 0xffu) ^ 0x80, b1i = (int)((c >> 8) & 0xffu) ^ 0x80;
        const double r = t->r[b0i];
        const double zr = r * t->cth[b1i], zi = r * t->sth[b1i];
        p[phys_to_logical_s(base | i, inv, nq)] = fma(zr, zr, zi * zi);
    }
}

// s[j] = sum of x[j*FANOUT .. (j+1)*FANOUT) (fixed-order tree reduction; missing tail = 0)
__global__ void __launch_bounds__(256) k_block_sums(const double *__restrict__ x, uint64_t n, double *__restrict__ s) {
    const uint64_t j = blockIdx.x;
    const uint64_t b = j * FANOUT;
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < FANOUT / 256; ++k) {
        const uint64_t i = b + threadIdx.x * (FANOUT / 256) + k;
        v += (i < n) ? x[i] : 0.0;
    }
    __shared__ double red[256];
    red[threadIdx.x] = v;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) s[j] = red[0];
}

__device__ __forceinline__ uint64_t splitmix64_d(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

struct TreeLevels {
    const double *lv[8];  // lv[0] = p (finest), lv[nlev-1] = root level (<= FANOUT entries)
    uint64_t len[8];
    int nlev;
};

// One warp per event.
__global__ void __launch_bounds__(256) k_sample(const __grid_constant__ TreeLevels T, double total, uint64_t seed,
                                                uint64_t nsamp, uint64_t *__restrict__ out) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t k = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (k >= nsamp) return;
    const double u = (double)(splitmix64_d(seed + k) >> 11) * (1.0 / 9007199254740992.0);
    double t = u * total;
    uint64_t node = 0;  // index of the current node within its level (root level: single implicit node)
    for (int lev = T.nlev - 1; lev >= 0; --lev) {
        const double *x = T.lv[lev];
        const uint64_t first = node * FANOUT;
        // each lane takes 32 consecutive children
        double part[32];
        double lsum = 0.0;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            const uint64_t i = first + lane * 32 + c;
            part[c] = (i < T.len[lev]) ? x[i] : 0.0;
            lsum += part[c];
        }
        // exclusive warp scan of lane sums
        double incl = lsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += y;
        }
        const double excl = incl - lsum;
        // first lane whose inclusive sum exceeds t (last lane with any mass if none does)
        const unsigned ball = __ballot_sync(0xffffffffu, incl > t);
        const unsigned nz = __ballot_sync(0xffffffffu, lsum > 0.0);
        const int sel = ball ? (__ffs(ball) - 1) : (nz ? (31 - __clz(nz)) : 31);
        const double base_sum = __shfl_sync(0xffffffffu, excl, sel);
        int child = 31;
        if ((int)lane == sel) {
            double run = excl;
            child = -1;
            int lastnz = 31;
            for (int c = 0; c < 32; ++c) {
                if (part[c] > 0.0) lastnz = c;
                run += part[c];
                if (run > t && child < 0) child = c;
            }
            if (child < 0) child = lastnz;
        }
        child = __shfl_sync(0xffffffffu, child, sel);
        double before = 0.0;
        if ((int)lane == sel) {
            before = excl;
            for (int c = 0; c < child; ++c) before += part[c];
        }
        before = __shfl_sync(0xffffffffu, before, sel);
        (void)base_sum;
        t -= before;
        node = first + (uint64_t)sel * 32 + (uint64_t)child;
    }
    if (lane == 0) out[k] = node;
}

int sample_logical(void *const *shard_amps, const uint64_t *shard_base, int nshards, int nl, int nq, const int *inv_host,
                   int enc, const ATables *at, uint64_t nsamp, uint64_t seed, uint64_t *out_host, cudaStream_t s,
                   void *nccl_comm) {
    const uint64_t dim = 1ull << nq;
    std::vector<void *> bufs;
    auto cleanup = [&]() {
        for (void *b : bufs) cudaFree(b);
    };
    auto alloc = [&](size_t bytes) -> void * {
        void *p = nullptr;
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        bufs.push_back(p);
        return p;
    };
    double *p = (double *)alloc(dim * sizeof(double));
    int *d_inv = (int *)alloc(nq * sizeof(int));
    uint64_t *d_out = (uint64_t *)alloc((nsamp ? nsamp : 1) * sizeof(uint64_t));
    if (!p || !d_inv || !d_out) {
        cleanup();
        set_error("qsim_sample: cannot allocate the 8 B x 2^N probability array");
        return QSIM_ENOMEM;
    }
    cudaMemcpyAsync(d_inv, inv_host, nq * sizeof(int), cudaMemcpyHostToDevice, s);
    if (nccl_comm) cudaMemsetAsync(p, 0, dim * sizeof(double), s);  // the other ranks' entries stay 0 here
    const uint64_t nshard_amps = 1ull << nl;
    const int grid = 148 * 8;
    for (int r = 0; r < nshards; ++r) {
        if (enc == QSIM_ENC_FP64)
            k_prob_logical_e<<<grid, 256, 0, s>>>((const double2 *)shard_amps[r], nshard_amps, shard_base[r], d_inv, nq,
                                                  p);
        else
            k_prob_logical_a<<<grid, 256, 0, s>>>((const uint16_t *)shard_amps[r], nshard_amps, shard_base[r], d_inv,
                                                  nq, at->d[at->cur], p);
    }
    // NCCL transport: each rank filled its own shard's entries (zeros elsewhere,
    // the array was cleared); the sum is the whole distribution, exactly, on
    // every rank -- which then draws the same samples from the same seed
    if (nccl_comm &&
        ncclAllReduce(p, p, dim, ncclFloat64, ncclSum, (ncclComm_t)nccl_comm, s) != ncclSuccess) {
        cleanup();
        set_error("qsim_sample: ncclAllReduce of the probabilities failed");
        return QSIM_ECOMM;
    }
    TreeLevels T{};
    T.lv[0] = p;
    T.len[0] = dim;
    T.nlev = 1;
    while (T.len[T.nlev - 1] > (uint64_t)FANOUT) {
        const uint64_t n = T.len[T.nlev - 1];
        const uint64_t m = (n + FANOUT - 1) / FANOUT;
        double *lv = (double *)alloc(m * sizeof(double));
        if (!lv || T.nlev >= 8) {
            cleanup();
            set_error("qsim_sample: tree allocation failed");
            return QSIM_ENOMEM;
        }
        k_block_sums<<<(unsigned)m, 256, 0, s>>>(T.lv[T.nlev - 1], n, lv);
        T.lv[T.nlev] = lv;
        T.len[T.nlev] = m;
        T.nlev++;
    }
    // total = sum of the root level, in the same order the sampler scans it
    double *d_tot = (double *)alloc(sizeof(double));
    if (!d_tot) {
        cleanup();
        return QSIM_ENOMEM;
    }
    k_block_sums<<<1, 256, 0, s>>>(T.lv[T.nlev - 1], T.len[T.nlev - 1], d_tot);
    double total = 0.0;
    cudaMemcpyAsync(&total, d_tot, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) {
        cleanup();
        set_error("qsim_sample: CUDA error");
        return QSIM_ECUDA;
    }
    if (!(total > 0.0)) {
        cleanup();
        set_error("qsim_sample: zero norm");
        return QSIM_EZERONORM;
    }
    if (nsamp) {
        const uint64_t threads = nsamp * 32;
        k_sample<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(T, total, seed, nsamp, d_out);
        cudaMemcpyAsync(out_host, d_out, nsamp * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
    }
    cudaError_t e = cudaStreamSynchronize(s);
    cleanup();
    if (e != cudaSuccess) {
        set_error(std::string("qsim_sample: ") + cudaGetErrorString(e));
        return QSIM_ECUDA;
    }
    return QSIM_OK;
}

// ---- SHORBOX (App. B) ---------------------------------
__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) {
    return (uint64_t)(((unsigned __int128)a * b) % m);
}
__device__ __forceinline__ uint64_t powmod(uint64_t y, uint64_t x, uint64_t m) {
    uint64_t r = 1 % m, b = y % m;
    while (x) {
        if (x & 1) r = mulmod(r, b, m);
        b = mulmod(b, b, m);
        x >>= 1;
    }
    return r;
}
// E: a(phys) = 2^{-nx/2} iff f == y^x mod G for the logical index x + 2^nx f
__global__ void k_shorbox_e(double2 *__restrict__ a, uint64_t n, uint64_t base, const int *__restrict__ inv, int nq,
                            int nx, uint64_t G, uint64_t y, double amp) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t L = phys_to_logical_s(base | i, inv, nq);
        const uint64_t x = L & ((1ull << nx) - 1ull), f = L >> nx;
        a[i] = make_double2((f == powmod(y, x, G)) ? amp : 0.0, 0.0);
    }
}
// A: the same state as codes: (b0, b1) = (0, 0) -> r0 = r1 = 2^{-nx/2} (degenerate bounds), or
// (127, 0) when nx = 0 (a basis state), special zero elsewhere
__global__ void k_shorbox_a(uint16_t *__restrict__ a, uint64_t n, uint64_t base, const int *__restrict__ inv, int nq,
                            int nx, uint64_t G, uint64_t y, uint16_t code) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t L = phys_to_logical_s(base | i, inv, nq);
        const uint64_t x = L & ((1ull << nx) - 1ull), f = L >> nx;
        a[i] = (f == powmod(y, x, G)) ? code : (uint16_t)0x0080u;  // 0x0080 = (b0 -128, b1 0)
    }
}
int shorbox(void *const *shard_amps, const uint64_t *shard_base, int nshards, int nl, int nq, const int *inv_host,
            int enc, int nx, uint64_t G, uint64_t y, cudaStream_t s) {
    int *d_inv = nullptr;
    if (cudaMalloc(&d_inv, nq * sizeof(int)) != cudaSuccess) return QSIM_ENOMEM;
    cudaMemcpyAsync(d_inv, inv_host, nq * sizeof(int), cudaMemcpyHostToDevice, s);
    const double amp = ldexp(1.0, -nx / 2) * ((nx & 1) ? 0.70710678118654752440 : 1.0);
    for (int r = 0; r < nshards; ++r) {
        if (enc == QSIM_ENC_FP64)
            k_shorbox_e<<<148 * 8, 256, 0, s>>>((double2 *)shard_amps[r], 1ull << nl, shard_base[r], d_inv, nq, nx, G, y,
                                                amp);
        else
            k_shorbox_a<<<148 * 8, 256, 0, s>>>((uint16_t *)shard_amps[r], 1ull << nl, shard_base[r], d_inv, nq, nx, G,
                                                y, (uint16_t)(nx == 0 ? 0x007Fu : 0x0000u));
    }
    cudaError_t e = cudaStreamSynchronize(s);
    cudaFree(d_inv);
    if (e != cudaSuccess) {
        set_error(std::string("shorbox: ") + cudaGetErrorString(e));
        return QSIM_ECUDA;
    }
    return QSIM_OK;
}

}  // namespace qsim
