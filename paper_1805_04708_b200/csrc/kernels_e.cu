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
// fused tile pass
// ============================================================================
__device__ __forceinline__ uint32_t swz(uint32_t x) { return x ^ (((x >> 3) ^ (x >> 6) ^ (x >> 9)) & 7u); }

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// In-place pair updates.  Each output's final FMA is the last use of exactly
// one input, so the register allocator can write every output over its own
// input: no register copies at the gate-dispatch merge points (the loop over a
// stage's gates is a runtime switch).
//   x' = u00 x + u01 y,  y' = u10 x + u11 y   (u = {u00r,u00i,u01r,u01i,u10r,u10i,u11r,u11i})
__device__ __forceinline__ void pair_dense(double2 &x, double2 &y, const double (&u)[8]) {
    const double p0 = fma(u[2], y.x, fma(-u[1], x.y, -u[3] * y.y));  // x'.re - u00r x.re
    const double p1 = fma(u[2], y.y, fma(u[1], x.x, u[3] * y.x));    // x'.im - u00r x.im
    const double p2 = fma(u[4], x.x, fma(-u[5], x.y, -u[7] * y.y));  // y'.re - u11r y.re
    const double p3 = fma(u[4], x.y, fma(u[5], x.x, u[7] * y.x));    // y'.im - u11r y.im
    x.x = fma(u[0], x.x, p0);
    x.y = fma(u[0], x.y, p1);
    y.x = fma(u[6], y.x, p2);
    y.y = fma(u[6], y.y, p3);
}
__device__ __forceinline__ void amp_phase(double2 &x, double ur, double ui) {
    const double p = -ui * x.y, q = ui * x.x;
    x.x = fma(ur, x.x, p);
    x.y = fma(ur, x.y, q);
}

// Gate table entry as staged in shared memory (one LDS.128 per complex entry).
struct SmGate {
    double2 u[4];        // u00, u01, u10, u11
    uint64_t cmask_out;
    uint64_t tmask_out;
    int32_t kind, slot, cslot, op;
};

// Gate application on the NS = 2^R register-resident amplitudes of one group.
// `f` is the group's slot-flip mask: register j holds the amplitude of
// logical slot j ^ f.  An uncontrolled X / CNOT-like swap on slot S is applied
// as f ^= 2^S (no data moves); later gates of the stage select conjugated
// coefficients for flipped slots and the stage's store XORs f into the
// (GF(2)-linear) smem address.  Every update is in place, so the register
// allocator never copies the amplitudes at the gate-dispatch merge points.
// FULL: no control inside the register set.
template <int NS, int S, bool FULL>
__device__ __forceinline__ void pg_dense(double2 (&v)[NS], const SmGate &g, int cslot, uint32_t f) {
    // flipped target slot: registers hold (y, x): apply X U X (complex entry c -> c ^ 3)
    const int cx = ((f >> S) & 1u) ? 3 : 0;
    const double2 e0 = g.u[0 ^ cx], e1 = g.u[1 ^ cx], e2 = g.u[2 ^ cx], e3 = g.u[3 ^ cx];
    const double u[8] = {e0.x, e0.y, e1.x, e1.y, e2.x, e2.y, e3.x, e3.y};
#pragma unroll
    for (int j = 0; j < NS; ++j) {
        if (j & (1 << S)) continue;
        if (!FULL && (((uint32_t)j ^ f) & cslot) != (uint32_t)cslot) continue;
        pair_dense(v[j], v[j | (1 << S)], u);
    }
}
// diagonal on slot S: logical bit 0 -> a0, logical bit 1 -> a1
template <int NS, int S, bool FULL>
__device__ __forceinline__ void pg_phase(double2 (&v)[NS], double2 a0, double2 a1, int cslot, uint32_t f) {
    const bool fl = (f >> S) & 1u;
    const double2 c0 = fl ? a1 : a0;  // registers with bit S = 0
    const double2 c1 = fl ? a0 : a1;  // registers with bit S = 1
#pragma unroll
    for (int j = 0; j < NS; ++j) {
        if (!FULL && (((uint32_t)j ^ f) & cslot) != (uint32_t)cslot) continue;
        if (j & (1 << S))
            amp_phase(v[j], c1.x, c1.y);
        else
            amp_phase(v[j], c0.x, c0.y);
    }
}
template <int NS>
__device__ __forceinline__ void pg_diag_out(double2 (&v)[NS], double2 c, int cslot, uint32_t f, bool full) {
    if (full) {
#pragma unroll
        for (int j = 0; j < NS; ++j) amp_phase(v[j], c.x, c.y);
    } else {
#pragma unroll
        for (int j = 0; j < NS; ++j)
            if ((((uint32_t)j ^ f) & cslot) == (uint32_t)cslot) amp_phase(v[j], c.x, c.y);
    }
}

// one gate on slot S (compile time) of a group; sub = op % 6
template <int NS, int S>
__device__ __forceinline__ void pg_slot(double2 (&v)[NS], const SmGate &g, int sub, int cs, uint32_t &f) {
    switch (sub) {
        case 0: pg_dense<NS, S, true>(v, g, cs, f); break;
        case 1: pg_dense<NS, S, false>(v, g, cs, f); break;
        case 2: pg_phase<NS, S, true>(v, g.u[0], g.u[3], cs, f); break;
        case 3: pg_phase<NS, S, false>(v, g.u[0], g.u[3], cs, f); break;
        case 4:  // x' = u01 y, y' = u10 x: flip slot S, then bit 0 gets u01, bit 1 gets u10
            f ^= 1u << S;
            pg_phase<NS, S, true>(v, g.u[1], g.u[2], 0, f);
            break;
        default: f ^= 1u << S; break;  // 5: uncontrolled in-register swap = slot flip
    }
}

// D = A B + C for one m8n8k4 f64 tile (A: lane (r = lane>>2, k = lane&3);
// B: lane (k = lane&3, n = lane>>2); D: lane (r, n = 2 (lane&3) + {0,1})).
__device__ __forceinline__ void dmma_first(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%4};\n"
                 : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(0.0));
}
__device__ __forceinline__ void dmma_acc(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// Shared memory of one CTA: the tile (2^K double2, XOR-swizzled), the
// two-level deposit tables of the high tile bits, the gate table, and per
// stage the swizzled base address of every register group.
struct PassSmemLayout {
    size_t tile, depA, depB, depJ, gates, gx, fbt, total;
};
__host__ __device__ inline PassSmemLayout pass_layout(int K, int R, int nstages) {
    PassSmemLayout L;
    L.tile = 0;
    L.depA = ((size_t)1 << K) * 16;
    L.depB = L.depA + 32 * 8;
    L.depJ = L.depB + 32 * 8;
    L.gates = L.depJ + 32 * 8;
    L.gx = L.gates + PASS_MAX_GATES * sizeof(SmGate);
    L.fbt = L.gx + (size_t)nstages * ((size_t)1 << (K - R)) * 2;
    L.total = L.fbt + (size_t)nstages * 8 * 2;
    return L;
}

template <int R, int MINB>
__global__ void __launch_bounds__(PASS_THREADS, MINB) k_pass_e(const __grid_constant__ PassParams p) {
    constexpr int NS = 1 << R;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int K = p.K;
    const PassSmemLayout L = pass_layout(K, R, p.nstages);
    double2 *tile = reinterpret_cast<double2 *>(smem_raw + L.tile);
    uint64_t *depA = reinterpret_cast<uint64_t *>(smem_raw + L.depA);  // high tile bits 0..4
    uint64_t *depB = reinterpret_cast<uint64_t *>(smem_raw + L.depB);  // high tile bits 5..
    SmGate *gates = reinterpret_cast<SmGate *>(smem_raw + L.gates);
    uint16_t *gx = reinterpret_cast<uint16_t *>(smem_raw + L.gx);
    uint16_t *fbt = reinterpret_cast<uint16_t *>(smem_raw + L.fbt);
    const uint32_t tsize = 1u << K;
    const int h = K - PASS_LOW;
    const uint32_t ngroups = tsize >> R;
    const uint32_t tid = threadIdx.x;
    // ---- one-time setup per CTA ----
    if (tid < 64) {
        const int lo = tid < 32 ? 0 : 5;
        const uint32_t hi = tid & 31u;
        uint64_t m = 0;
        for (int i = 0; i < 5 && lo + i < h; ++i)
            if (hi & (1u << i)) m |= 1ull << p.high_q[lo + i];
        (tid < 32 ? depA : depB)[hi] = m;
    }
    for (int gi = tid; gi < PASS_MAX_GATES; gi += PASS_THREADS) {
        const PassGate &g = p.g[gi];
        SmGate sg;
        for (int c = 0; c < 4; ++c) sg.u[c] = make_double2(g.u[2 * c], g.u[2 * c + 1]);
        sg.cmask_out = g.cmask_out;
        sg.tmask_out = g.tmask_out;
        sg.kind = g.kind;
        sg.slot = g.slot;
        sg.cslot = g.cslot;
        sg.op = g.op;
        gates[gi] = sg;
    }
    for (int s = 0; s < p.nstages; ++s) {
        const PassStage &st = p.st[s];
        if (st.type == 1) {  // pair stage: thread base address (lane, warp bits) + fragment basis
            uint32_t xl = 0;
            for (int i = 0; i < 7; ++i) xl |= ((tid >> i) & 1u) << st.mbits[i];
            gx[s * ngroups + tid] = (uint16_t)swz(xl);
            if (tid < 8) fbt[s * 8 + tid] = (tid < 5 && 7 + (int)tid < K) ? (uint16_t)swz(1u << st.mbits[7 + tid]) : 0;
            continue;
        }
        for (uint32_t grp = tid; grp < ngroups; grp += PASS_THREADS) {
            uint32_t x0 = 0;
            for (int i = 0; i < K - R; ++i) x0 |= ((grp >> i) & 1u) << st.gbits[i];
            gx[s * ngroups + grp] = (uint16_t)swz(x0);
        }
    }
    __syncthreads();
    double2 *__restrict__ a = reinterpret_cast<double2 *>(p.a);
    constexpr uint32_t LOWM = (1u << PASS_LOW) - 1u;
    auto dep = [&](uint32_t hi) -> uint64_t { return depA[hi & 31u] | depB[hi >> 5]; };
    static_assert(PASS_THREADS == 128, "load/store addressing assumes x = tid + 128 j");
    const uint32_t njt = tsize >> 7;  // elements per thread in the load / store loops
    const uint32_t s_tid = swz(tid);
    const uint64_t d_tid = (tid & LOWM) | dep(tid >> PASS_LOW);
    uint64_t *depJ = reinterpret_cast<uint64_t *>(smem_raw + L.depJ);  // dep(16 j): high tile bits >= 4
    for (uint32_t j = tid; j < njt; j += PASS_THREADS) depJ[j] = dep(j << (7 - PASS_LOW));
    __syncthreads();

    for (uint64_t T = blockIdx.x; T < p.ntiles; T += gridDim.x) {
        // base: insert zeros at the tile's qubits (0..PASS_LOW-1 and high_q ascending)
        uint64_t base = T << PASS_LOW;
        for (int i = 0; i < h; ++i) base = insert_zero(base, p.high_q[i]);
        // ---- load the tile (coalesced 128 B runs) ----
        // x = tid + 128 j: swz and the deposit are GF(2)-linear on disjoint
        // bits, so address = a[(base | d_tid) + depJ[j]] and smem = s_tid ^ swz(128 j).
        const double2 *pt = a + (base | d_tid);
        if (!p.noio) {
#pragma unroll 8
            for (uint32_t j = 0; j < njt; ++j) cp_async16(&tile[s_tid ^ swz(j << 7)], pt + depJ[j]);
        }
        cp_async_wait_all();
        __syncthreads();
        // ---- stages ----
        for (int s = 0; s < p.nstages; ++s) {
            const PassStage &st = p.st[s];
            if (st.type == 1) {
                // ---- tensor-core pair stage: amp' = G amp on the quad (lane bits 0,1) ----
                // Real 8x8 form: k = c <-> Re(in_c), k = 4 + c <-> Im(in_c);
                // n = 2c' <-> Re(out_c'), n = 2c' + 1 <-> Im(out_c').  A lane holds
                // amp c of item r as (A chunk 0, A chunk 1) and receives amp'_c as (d0, d1).
                // Per-thread base address and fragment-bit basis come from the
                // per-CTA tables built at kernel start (GF(2)-linear swizzle).
                const uint32_t sl = gx[s * ngroups + tid];
                const uint16_t *fbs = fbt + s * 8;
                const uint32_t fb0 = fbs[0], fb1 = fbs[1], fb2 = fbs[2], fb3 = fbs[3], fb4 = fbs[4];
                const uint32_t off[8] = {0u, fb0, fb1, fb0 ^ fb1, fb2, fb0 ^ fb2, fb1 ^ fb2, fb0 ^ fb1 ^ fb2};
                const uint32_t c = tid & 3u, nn = (tid & 31u) >> 2;
                const double2 gcc = p.op4[st.opi][(nn >> 1) * 4 + c];  // G[c'][c]
                const double b0 = (nn & 1u) ? gcc.y : gcc.x;            // B[c][n]
                const double b1 = (nn & 1u) ? gcc.x : -gcc.y;           // B[4 + c][n]
                const uint32_t nch = 1u << (K - 10);                     // chunks of 8 fragments
                for (uint32_t ch = 0; ch < nch; ++ch) {
                    const uint32_t cb = sl ^ ((ch & 1u) ? fb3 : 0u) ^ ((ch & 2u) ? fb4 : 0u);
                    double2 v8[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) v8[j] = tile[cb ^ off[j]];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        double d0, d1;
                        dmma_first(d0, d1, v8[j].x, b0);
                        dmma_acc(d0, d1, v8[j].y, b1);
                        v8[j] = make_double2(d0, d1);
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) tile[cb ^ off[j]] = v8[j];
                }
                __syncthreads();
                continue;
            }
            // swz is linear over GF(2): swz(x0 | slot bits) = swz(x0) ^ xor of swz(slot bit)
            uint32_t sb[R];
#pragma unroll
            for (int r = 0; r < R; ++r) sb[r] = swz(1u << st.rbits[r]);
            const int g0 = st.first_gate, g1 = st.first_gate + st.ngates;
            const bool nf = st.needs_full;
            for (uint32_t grp = tid; grp < ngroups; grp += PASS_THREADS) {
                const uint32_t sx0 = gx[s * ngroups + grp];
                uint64_t full0 = 0;
                if (nf) {
                    const uint32_t x0 = swz(sx0);  // swz is an involution
                    full0 = p.shard_base | base | (x0 & LOWM) | dep(x0 >> PASS_LOW);
                }
                double2 v[NS];
#pragma unroll
                for (int j = 0; j < NS; ++j) {
                    uint32_t xs = sx0;
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        if (j & (1 << r)) xs ^= sb[r];
                    v[j] = tile[xs];
                }
                uint32_t f = 0;
                // software-pipelined dispatch: the next gate's descriptor is
                // loaded while the current gate's FMA block runs
                int op_n = g0 < g1 ? gates[g0].op : 0;
                int cs_n = g0 < g1 ? gates[g0].cslot : 0;
                uint64_t cm_n = g0 < g1 ? gates[g0].cmask_out : 0;
                for (int gi = g0; gi < g1; ++gi) {
                    const SmGate &g = gates[gi];
                    const int op = op_n, cs = cs_n;
                    const uint64_t cm = cm_n;
                    if (gi + 1 < g1) {
                        op_n = gates[gi + 1].op;
                        cs_n = gates[gi + 1].cslot;
                        cm_n = gates[gi + 1].cmask_out;
                    }
                    if ((full0 & cm) != cm) continue;
                    switch (op) {
#define PG_OPS(S)                                                                            \
    case (S) * 6 + 0: pg_dense<NS, (S), true>(v, g, cs, f); break;                           \
    case (S) * 6 + 1: pg_dense<NS, (S), false>(v, g, cs, f); break;                          \
    case (S) * 6 + 2: pg_phase<NS, (S), true>(v, g.u[0], g.u[3], cs, f); break;              \
    case (S) * 6 + 3: pg_phase<NS, (S), false>(v, g.u[0], g.u[3], cs, f); break;             \
    case (S) * 6 + 4:                                                                        \
        f ^= 1u << (S);                                                                      \
        pg_phase<NS, (S), true>(v, g.u[1], g.u[2], 0, f);                                    \
        break;                                                                               \
    case (S) * 6 + 5: f ^= 1u << (S); break;
                        PG_OPS(0)
                        PG_OPS(1)
                        PG_OPS(2)
                        PG_OPS(3)
#undef PG_OPS
                        default:
                            if (op >= 6 * R) {  // diagonal gate whose target is outside the registers
                                const bool bit = (full0 & g.tmask_out) != 0;
                                pg_diag_out<NS>(v, bit ? g.u[3] : g.u[0], cs, f, op == 6 * R);
                            } else if constexpr (R > 4) {
                                pg_slot<NS, (R > 4 ? 4 : 0)>(v, g, op - 24, cs, f);
                            }
                            break;
                    }
                }
                // register j holds logical slot j ^ f: store to swz(x0 | slots(j ^ f))
                uint32_t sxf = sx0;
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (f & (1u << r)) sxf ^= sb[r];
#pragma unroll
                for (int j = 0; j < NS; ++j) {
                    uint32_t xs = sxf;
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        if (j & (1 << r)) xs ^= sb[r];
                    tile[xs] = v[j];
                }
            }
            __syncthreads();
        }
        // ---- store the tile ----
        double2 *ps = a + (base | d_tid);
        if (!p.noio) {
#pragma unroll 8
            for (uint32_t j = 0; j < njt; ++j) ps[depJ[j]] = tile[s_tid ^ swz(j << 7)];
        }
        __syncthreads();
    }
}

static size_t pass_smem(int K, int R, int nstages) { return pass_layout(K, R, nstages).total; }


static bool g_pass_attr = false;
// CTAs per SM of the R = 4 kernel: 3 (164 registers, K = 12 tiles), or 4 / 5
// (register-capped, K = 11 tiles) -- selected with QSIM_PASS_OCC for tuning.
static int pass_occ() {
    static int occ = 0;
    if (!occ) {
        const char *e = getenv("QSIM_PASS_OCC");
        occ = e ? atoi(e) : 3;
        if (occ < 3 || occ > 5) occ = 3;
    }
    return occ;
}
int pass_e_max_k() { return pass_occ() == 3 ? 12 : 11; }
int pass_e_max_grid(int R) { return num_sms() * (R >= 5 ? 2 : pass_occ()); }

void launch_pass_e(const PassParams &p, int grid, cudaStream_t s) {
    if (!g_pass_attr) {
        cudaFuncSetAttribute(k_pass_e<4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pass_smem(PASS_MAX_K, 4, PASS_MAX_STAGES));
        cudaFuncSetAttribute(k_pass_e<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pass_smem(PASS_MAX_K, 4, PASS_MAX_STAGES));
        cudaFuncSetAttribute(k_pass_e<4, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pass_smem(PASS_MAX_K, 4, PASS_MAX_STAGES));
        cudaFuncSetAttribute(k_pass_e<5, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pass_smem(PASS_MAX_K, 5, PASS_MAX_STAGES));
        g_pass_attr = true;
    }
    if (p.R >= 5)
        k_pass_e<5, 2><<<grid, PASS_THREADS, pass_smem(p.K, 5, p.nstages), s>>>(p);
    else if (pass_occ() == 4)
        k_pass_e<4, 4><<<grid, PASS_THREADS, pass_smem(p.K, 4, p.nstages), s>>>(p);
    else if (pass_occ() == 5)
        k_pass_e<4, 5><<<grid, PASS_THREADS, pass_smem(p.K, 4, p.nstages), s>>>(p);
    else
        k_pass_e<4, 3><<<grid, PASS_THREADS, pass_smem(p.K, 4, p.nstages), s>>>(p);
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
