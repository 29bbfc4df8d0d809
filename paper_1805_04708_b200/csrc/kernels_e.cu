// kernels_e.cu -- sm_100a kernels for the E (complex fp64) state vector.
//
// Every kernel is HBM-bound: a 1-qubit gate is 14 fp64
// flops per 32 bytes moved.  Design points:
//  * 16-byte amplitudes (double2) move with 128-bit loads/stores.
//  * sweeps: each thread handles 4 groups per iteration (all loads issued
//    before the first FMA) in a grid sized to a multiple of the 148 SMs.
//  * fused pass: a tile of 2^K amplitudes spanning qubits 0..4 (512 B
//    contiguous runs) plus up to 7 arbitrary higher qubits is staged in
//    shared memory with cp.async, every gate of a run whose target lies in
//    the tile is applied there (16 amplitudes per thread in registers per
//    stage), and the tile is written back: one HBM pass for the whole run
//    (the "combining ... to multi-qubit gates" of PAPER.md:787-790).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "internal.h"
#include "kernels.h"

namespace qsim {

static int g_num_sms = 0;
static int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

__device__ __forceinline__ uint64_t insert_zero(uint64_t w, int p) {
    uint64_t lo = w & ((1ull << p) - 1ull);
    return ((w >> p) << (p + 1)) | lo;
}

// complex helpers: r = u0 * x + u1 * y
__device__ __forceinline__ double2 cmad2(double u0r, double u0i, double2 x, double u1r, double u1i, double2 y) {
    double2 r;
    r.x = fma(u0r, x.x, fma(-u0i, x.y, fma(u1r, y.x, -u1i * y.y)));
    r.y = fma(u0r, x.y, fma(u0i, x.x, fma(u1r, y.y, u1i * y.x)));
    return r;
}
__device__ __forceinline__ double2 cmul(double ur, double ui, double2 x) {
    double2 r;
    r.x = fma(ur, x.x, -ui * x.y);
    r.y = fma(ur, x.y, ui * x.x);
    return r;
}

// ============================================================================
// single-gate sweep
// ============================================================================
constexpr int SWEEP_THREADS = 256;
constexpr int SWEEP_ILP = 4;

template <int CLS, int TOUCH>
__global__ void __launch_bounds__(SWEEP_THREADS) k_sweep_e(const __grid_constant__ SweepParams p) {
    double2 *__restrict__ a = reinterpret_cast<double2 *>(p.a);
    const uint64_t tb = 1ull << p.t;
    const uint64_t stride = (uint64_t)gridDim.x * SWEEP_THREADS * SWEEP_ILP;
    for (uint64_t w0 = (uint64_t)blockIdx.x * SWEEP_THREADS * SWEEP_ILP + threadIdx.x; w0 < p.nitems; w0 += stride) {
        uint64_t i0[SWEEP_ILP];
        double2 x[SWEEP_ILP], y[SWEEP_ILP];
        bool ok[SWEEP_ILP];
#pragma unroll
        for (int k = 0; k < SWEEP_ILP; ++k) {
            uint64_t w = w0 + (uint64_t)k * SWEEP_THREADS;
            ok[k] = w < p.nitems;
            uint64_t i = w;
            for (int q = 0; q < p.nins; ++q) i = insert_zero(i, p.ins[q]);
            i0[k] = i | p.cmask;
            if (ok[k]) {
                if (TOUCH & 1) x[k] = a[i0[k]];
                if (TOUCH & 2) y[k] = a[i0[k] | tb];
            }
        }
#pragma unroll
        for (int k = 0; k < SWEEP_ILP; ++k) {
            if (!ok[k]) continue;
            if (CLS == CLS_DENSE) {
                double2 nx = cmad2(p.u[0], p.u[1], x[k], p.u[2], p.u[3], y[k]);
                double2 ny = cmad2(p.u[4], p.u[5], x[k], p.u[6], p.u[7], y[k]);
                a[i0[k]] = nx;
                a[i0[k] | tb] = ny;
            } else if (CLS == CLS_ANTI) {
                double2 nx = cmul(p.u[2], p.u[3], y[k]);
                double2 ny = cmul(p.u[4], p.u[5], x[k]);
                a[i0[k]] = nx;
                a[i0[k] | tb] = ny;
            } else {  // diagonal
                if (TOUCH & 1) a[i0[k]] = cmul(p.u[0], p.u[1], x[k]);
                if (TOUCH & 2) a[i0[k] | tb] = cmul(p.u[6], p.u[7], y[k]);
            }
        }
    }
}

// k-qubit dense matrix (qsim_apply_matrix, k = 1..3): every group of 2^k
// amplitudes that differ only in the k physical bits, matrix index bit
// (k-1-b) <-> physical bit phys[b] (qubits[0] the most significant, reading
// A14), y = U x with U row-major 2^k x 2^k complex.
template <int K>
__global__ void __launch_bounds__(256) k_matk_e(const __grid_constant__ MatKParams p) {
    constexpr int M = 1 << K;
    double2 *__restrict__ a = reinterpret_cast<double2 *>(p.a);
    for (uint64_t w = (uint64_t)blockIdx.x * 256 + threadIdx.x; w < p.ngroups; w += (uint64_t)gridDim.x * 256) {
        uint64_t base = w;
        for (int b = 0; b < K; ++b) base = insert_zero(base, p.sorted[b]);
        uint64_t idx[M];
        double2 x[M];
#pragma unroll
        for (int m = 0; m < M; ++m) {
            uint64_t i = base;
#pragma unroll
            for (int b = 0; b < K; ++b)
                if ((m >> (K - 1 - b)) & 1) i |= 1ull << p.phys[b];
            idx[m] = i;
            x[m] = a[i];
        }
#pragma unroll
        for (int r = 0; r < M; ++r) {
            double yr = 0.0, yi = 0.0;
#pragma unroll
            for (int c = 0; c < M; ++c) {
                const double ur = p.u[2 * (r * M + c)], ui = p.u[2 * (r * M + c) + 1];
                yr = fma(ur, x[c].x, fma(-ui, x[c].y, yr));
                yi = fma(ur, x[c].y, fma(ui, x[c].x, yi));
            }
            a[idx[r]] = make_double2(yr, yi);
        }
    }
}

void launch_matk_e(const MatKParams &p, cudaStream_t s) {
    uint64_t cap = (uint64_t)num_sms() * 8, need = (p.ngroups + 255) / 256;
    const int grid = (int)(need < cap ? (need ? need : 1) : cap);
    if (p.k == 1)
        k_matk_e<1><<<grid, 256, 0, s>>>(p);
    else if (p.k == 2)
        k_matk_e<2><<<grid, 256, 0, s>>>(p);
    else
        k_matk_e<3><<<grid, 256, 0, s>>>(p);
}

static int sweep_grid(uint64_t nitems) {
    uint64_t per = (uint64_t)SWEEP_THREADS * SWEEP_ILP;
    uint64_t need = (nitems + per - 1) / per;
    uint64_t cap = (uint64_t)num_sms() * 8;  // 8 x 256 threads per SM resident
    return (int)(need < cap ? (need ? need : 1) : cap);
}

void launch_sweep_e(const SweepParams &p, cudaStream_t s) {
    int grid = sweep_grid(p.nitems);
    if (p.cls == CLS_DENSE)
        k_sweep_e<CLS_DENSE, 3><<<grid, SWEEP_THREADS, 0, s>>>(p);
    else if (p.cls == CLS_ANTI)
        k_sweep_e<CLS_ANTI, 3><<<grid, SWEEP_THREADS, 0, s>>>(p);
    else if (p.touch == 1)
        k_sweep_e<CLS_DIAG, 1><<<grid, SWEEP_THREADS, 0, s>>>(p);
    else if (p.touch == 2)
        k_sweep_e<CLS_DIAG, 2><<<grid, SWEEP_THREADS, 0, s>>>(p);
    else
        k_sweep_e<CLS_DIAG, 3><<<grid, SWEEP_THREADS, 0, s>>>(p);
}

__global__ void __launch_bounds__(SWEEP_THREADS) k_scale_e(const __grid_constant__ ScaleParams p) {
    double2 *__restrict__ a = reinterpret_cast<double2 *>(p.a);
    const uint64_t stride = (uint64_t)gridDim.x * SWEEP_THREADS;
    for (uint64_t w = (uint64_t)blockIdx.x * SWEEP_THREADS + threadIdx.x; w < p.nitems; w += stride) {
        uint64_t i = w;
        for (int q = 0; q < p.nins; ++q) i = insert_zero(i, p.ins[q]);
        i |= p.cmask;
        a[i] = cmul(p.f[0], p.f[1], a[i]);
    }
}

void launch_scale_e(const ScaleParams &p, cudaStream_t s) {
    int grid = sweep_grid(p.nitems * SWEEP_ILP / 4 + 1);
    k_scale_e<<<grid, SWEEP_THREADS, 0, s>>>(p);
}

// ============================================================================
// exchange-fused gate: (kept half slice, received slice) -> both slots
// ============================================================================
template <int MODE, int CLS>
__global__ void __launch_bounds__(SWEEP_THREADS) k_xchg_e(const __grid_constant__ XchgParams p) {
    double2 *__restrict__ own = reinterpret_cast<double2 *>(p.own);
    const double2 *__restrict__ stg = reinterpret_cast<const double2 *>(p.stage);
    const uint64_t lb = 1ull << p.l;
    const uint64_t stride = (uint64_t)gridDim.x * SWEEP_THREADS;
    for (uint64_t k = (uint64_t)blockIdx.x * SWEEP_THREADS + threadIdx.x; k < p.n; k += stride) {
        const uint64_t i0 = insert_zero(p.p0 + k, p.l);
        const uint64_t i1 = i0 | lb;
        const double2 r = stg[k];
        if (MODE == 0) {
            own[p.b ? i0 : i1] = r;
            continue;
        }
        const double2 kept = own[p.b ? i1 : i0];
        double2 x = p.b ? r : kept, y = p.b ? kept : r;
        if (((p.shard_base | i0) & p.cmask) == p.cmask) {
            if (CLS == CLS_DENSE) {
                double2 nx = cmad2(p.u[0], p.u[1], x, p.u[2], p.u[3], y);
                double2 ny = cmad2(p.u[4], p.u[5], x, p.u[6], p.u[7], y);
                x = nx;
                y = ny;
            } else if (CLS == CLS_ANTI) {
                double2 nx = cmul(p.u[2], p.u[3], y);
                double2 ny = cmul(p.u[4], p.u[5], x);
                x = nx;
                y = ny;
            } else {
                x = cmul(p.u[0], p.u[1], x);
                y = cmul(p.u[6], p.u[7], y);
            }
        }
        own[i0] = x;
        own[i1] = y;
    }
}

void launch_xchg_e(const XchgParams &p, cudaStream_t s) {
    int grid = sweep_grid(p.n / SWEEP_ILP + 1);
    if (p.mode == 0)
        k_xchg_e<0, CLS_DENSE><<<grid, SWEEP_THREADS, 0, s>>>(p);
    else if (p.cls == CLS_DENSE)
        k_xchg_e<1, CLS_DENSE><<<grid, SWEEP_THREADS, 0, s>>>(p);
    else if (p.cls == CLS_ANTI)
        k_xchg_e<1, CLS_ANTI><<<grid, SWEEP_THREADS, 0, s>>>(p);
    else
        k_xchg_e<1, CLS_DIAG><<<grid, SWEEP_THREADS, 0, s>>>(p);
}

// ============================================================================
// reductions (a10): deterministic two-level (fixed grid, fixed order)
// ============================================================================
constexpr int RED_THREADS = 256;
int red_blocks() { return num_sms() * 2; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Each warp walks segments of 256 amplitudes: lane = qubits 0..4, j = qubits
// 5..7, segment index = qubits >= 8.  partials: [block][RED_SLOTS].
__global__ void __launch_bounds__(RED_THREADS) k_probs_e(const double2 *__restrict__ a, int nl, double *partials) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t n = 1ull << nl;
    const uint64_t nseg = n >> 8;
    const uint64_t gwarp = (uint64_t)blockIdx.x * (RED_THREADS / 32) + warp;
    const uint64_t nwarps = (uint64_t)gridDim.x * (RED_THREADS / 32);
    double tot_lane = 0.0, pj[3] = {0.0, 0.0, 0.0}, phigh = 0.0;  // phigh: qubit 8 + lane
    for (uint64_t sgi = gwarp; sgi < nseg; sgi += nwarps) {
        const double2 *seg = a + (sgi << 8);
        double2 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = seg[lane + 32 * j];
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            double m = fma(v[j].x, v[j].x, v[j].y * v[j].y);
            t += m;
            if (j & 1) pj[0] += m;
            if (j & 2) pj[1] += m;
            if (j & 4) pj[2] += m;
        }
        tot_lane += t;
        double seg_tot = warp_sum(t);
        if (8 + lane < nl && ((sgi >> lane) & 1ull)) phigh += seg_tot;
    }
    __shared__ double sm[RED_THREADS / 32][RED_SLOTS];
    // per-warp vector: [0] total, [1+q] p1 of qubit q
    double tot = warp_sum(tot_lane);
    double pq[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) pq[q] = warp_sum((lane >> q) & 1 ? tot_lane : 0.0);
    double p5 = warp_sum(pj[0]), p6 = warp_sum(pj[1]), p7 = warp_sum(pj[2]);
    if (lane == 0) {
        sm[warp][0] = tot;
        for (int q = 0; q < 5; ++q) sm[warp][1 + q] = pq[q];
        sm[warp][6] = p5;
        sm[warp][7] = p6;
        sm[warp][8] = p7;
    }
    sm[warp][9 + lane] = phigh;                               // qubit 8 + lane
    if (41 + lane < RED_SLOTS) sm[warp][41 + lane] = 0.0;     // unused slots
    __syncwarp();
    __syncthreads();
    if (threadIdx.x < RED_SLOTS) {
        double s = 0.0;
        for (int w = 0; w < RED_THREADS / 32; ++w) s += sm[w][threadIdx.x];
        partials[(size_t)blockIdx.x * RED_SLOTS + threadIdx.x] = s;
    }
}

// small shards (< 256 amplitudes never happen: nl >= 9); final fixed-order sum
__global__ void k_final_sum(const double *partials, int nblocks, int nslots, double *out) {
    int s = threadIdx.x;
    if (s >= nslots) return;
    double acc = 0.0;
    for (int b = 0; b < nblocks; ++b) acc += partials[(size_t)b * nslots + s];
    out[s] = acc;
}

void launch_probs_e(const void *a, int nl, double *partials, double *out, cudaStream_t s) {
    int nb = red_blocks();
    k_probs_e<<<nb, RED_THREADS, 0, s>>>(reinterpret_cast<const double2 *>(a), nl, partials);
    k_final_sum<<<1, RED_SLOTS, 0, s>>>(partials, nb, RED_SLOTS, out);
}

__global__ void __launch_bounds__(RED_THREADS) k_pairdot_e(const double2 *__restrict__ a, int nl, int q,
                                                           double *partials) {
    const uint64_t npairs = 1ull << (nl - 1);
    const uint64_t qb = 1ull << q;
    double sr = 0.0, si = 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * RED_THREADS;
    for (uint64_t w = (uint64_t)blockIdx.x * RED_THREADS + threadIdx.x; w < npairs; w += stride) {
        uint64_t i0 = insert_zero(w, q);
        double2 x = a[i0], y = a[i0 | qb];
        sr = fma(x.x, y.x, fma(x.y, y.y, sr));  // Re conj(x) y
        si = fma(x.x, y.y, fma(-x.y, y.x, si)); // Im conj(x) y
    }
    __shared__ double sm[2][RED_THREADS / 32];
    sr = warp_sum(sr);
    si = warp_sum(si);
    if ((threadIdx.x & 31) == 0) {
        sm[0][threadIdx.x >> 5] = sr;
        sm[1][threadIdx.x >> 5] = si;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        double s = 0.0;
        for (int w = 0; w < RED_THREADS / 32; ++w) s += sm[threadIdx.x][w];
        partials[(size_t)blockIdx.x * 2 + threadIdx.x] = s;
    }
}

void launch_pairdot_e(const void *a, int nl, int q, double *partials, double *out, cudaStream_t s) {
    int nb = red_blocks();
    k_pairdot_e<<<nb, RED_THREADS, 0, s>>>(reinterpret_cast<const double2 *>(a), nl, q, partials);
    k_final_sum<<<1, 32, 0, s>>>(partials, nb, 2, out);
}

__global__ void __launch_bounds__(RED_THREADS) k_dot_e(const double2 *__restrict__ x, const double2 *__restrict__ y,
                                                       uint64_t n, double *partials) {
    double sr = 0.0, si = 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * RED_THREADS;
    for (uint64_t i = (uint64_t)blockIdx.x * RED_THREADS + threadIdx.x; i < n; i += stride) {
        double2 u = x[i], v = y[i];
        sr = fma(u.x, v.x, fma(u.y, v.y, sr));
        si = fma(u.x, v.y, fma(-u.y, v.x, si));
    }
    __shared__ double sm[2][RED_THREADS / 32];
    sr = warp_sum(sr);
    si = warp_sum(si);
    if ((threadIdx.x & 31) == 0) {
        sm[0][threadIdx.x >> 5] = sr;
        sm[1][threadIdx.x >> 5] = si;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        double s = 0.0;
        for (int w = 0; w < RED_THREADS / 32; ++w) s += sm[threadIdx.x][w];
        partials[(size_t)blockIdx.x * 2 + threadIdx.x] = s;
    }
}

void launch_dot_e(const void *x, const void *y, uint64_t n, double *partials, double *out, cudaStream_t s) {
    int nb = red_blocks();
    k_dot_e<<<nb, RED_THREADS, 0, s>>>(reinterpret_cast<const double2 *>(x), reinterpret_cast<const double2 *>(y), n,
                                       partials);
    k_final_sum<<<1, 32, 0, s>>>(partials, nb, 2, out);
}

// max |a|^2 and min of the non-zero |a|^2 (the magnitude range of the state:
// SURVEY.md §8(d) "value distributions", the A bounds' E counterpart).
// Non-negative doubles order like their bit patterns, so the block results
// merge with integer atomics (order-independent, exact).
__global__ void __launch_bounds__(RED_THREADS) k_absrange_e(const double2 *__restrict__ a, uint64_t n,
                                                            unsigned long long *out) {
    double mx = 0.0, mn = INFINITY;
    const uint64_t stride = (uint64_t)gridDim.x * RED_THREADS;
    for (uint64_t i = (uint64_t)blockIdx.x * RED_THREADS + threadIdx.x; i < n; i += stride) {
        double2 v = a[i];
        double m = fma(v.x, v.x, v.y * v.y);
        mx = fmax(mx, m);
        if (m > 0.0) mn = fmin(mn, m);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&out[1], (unsigned long long)__double_as_longlong(mx));
        atomicMin(&out[0], (unsigned long long)__double_as_longlong(mn));
    }
}

void launch_absrange_e(const void *a, uint64_t n, void *out_u64x2, cudaStream_t s) {
    k_absrange_e<<<red_blocks(), RED_THREADS, 0, s>>>(reinterpret_cast<const double2 *>(a), n,
                                                      reinterpret_cast<unsigned long long *>(out_u64x2));
}

__global__ void k_collapse_e(double2 *__restrict__ a, uint64_t n, int q, int keep, double f) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        int bit = (int)((i >> q) & 1ull);
        double2 v = a[i];
        if (bit != keep) {
            v.x = 0.0;
            v.y = 0.0;
        } else {
            v.x *= f;
            v.y *= f;
        }
        a[i] = v;
    }
}
void launch_collapse_e(void *a, uint64_t n, int q, int keep, double f, cudaStream_t s) {
    k_collapse_e<<<sweep_grid(n / SWEEP_ILP + 1), SWEEP_THREADS, 0, s>>>(reinterpret_cast<double2 *>(a), n, q, keep,
                                                                         f);
}
__global__ void k_scale_all_e(double2 *__restrict__ a, uint64_t n, double f) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        double2 v = a[i];
        v.x *= f;
        v.y *= f;
        a[i] = v;
    }
}
void launch_scale_all_e(void *a, uint64_t n, double f, cudaStream_t s) {
    k_scale_all_e<<<sweep_grid(n / SWEEP_ILP + 1), SWEEP_THREADS, 0, s>>>(reinterpret_cast<double2 *>(a), n, f);
}

__global__ void k_gather_e(const double2 *__restrict__ a, const uint64_t *__restrict__ off, uint64_t m,
                           double2 *__restrict__ out) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x)
        out[k] = a[off[k]];
}
__global__ void k_scatter_e(double2 *__restrict__ a, const uint64_t *__restrict__ off, uint64_t m,
                            const double2 *__restrict__ in) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x)
        a[off[k]] = in[k];
}
void launch_gather_e(const void *a, const uint64_t *off, uint64_t m, void *out, cudaStream_t s) {
    if (!m) return;
    k_gather_e<<<sweep_grid(m / SWEEP_ILP + 1), SWEEP_THREADS, 0, s>>>(reinterpret_cast<const double2 *>(a), off, m,
                                                                       reinterpret_cast<double2 *>(out));
}
void launch_scatter_e(void *a, const uint64_t *off, uint64_t m, const void *in, cudaStream_t s) {
    if (!m) return;
    k_scatter_e<<<sweep_grid(m / SWEEP_ILP + 1), SWEEP_THREADS, 0, s>>>(reinterpret_cast<double2 *>(a), off, m,
                                                                        reinterpret_cast<const double2 *>(in));
}

__device__ __forceinline__ uint64_t phys_to_logical(uint64_t phys, const int *inv, int nq) {
    uint64_t L = 0;
    for (int b = 0; b < nq; ++b)
        if ((phys >> b) & 1ull) L |= 1ull << inv[b];
    return L;
}
__global__ void k_to_logical_e(const double2 *__restrict__ a, uint64_t n, uint64_t base, const int *__restrict__ inv,
                               int nq, double2 *__restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[phys_to_logical(base | i, inv, nq)] = a[i];
}
__global__ void k_from_logical_e(double2 *__restrict__ a, uint64_t n, uint64_t base, const int *__restrict__ inv,
                                 int nq, const double2 *__restrict__ in) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = in[phys_to_logical(base | i, inv, nq)];
}
void launch_to_logical_e(const void *a, uint64_t n, uint64_t base, const int *inv, int nq, void *out,
                         cudaStream_t s) {
    k_to_logical_e<<<sweep_grid(n / SWEEP_ILP + 1), SWEEP_THREADS, 0, s>>>(reinterpret_cast<const double2 *>(a), n,
                                                                           base, inv, nq,
                                                                           reinterpret_cast<double2 *>(out));
}
void launch_from_logical_e(void *a, uint64_t n, uint64_t base, const int *inv, int nq, const void *in,
                           cudaStream_t s) {
    k_from_logical_e<<<sweep_grid(n / SWEEP_ILP + 1), SWEEP_THREADS, 0, s>>>(reinterpret_cast<double2 *>(a), n,
                                                                             base, inv, nq,
                                                                             reinterpret_cast<const double2 *>(in));
}

}  // namespace qsim
