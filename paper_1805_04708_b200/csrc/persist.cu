// persist.cu -- the "single persistent kernel" mode of SURVEY.md §8(d) config 1
// (latency-bound small states, N <= 16): ONE launch applies a whole circuit.
// The state lives in the distributed shared memory of a thread-block cluster
// (16 CTAs where the device allows the non-portable size, else 8; CTA r holds
// amplitudes [r 2^(n-c), (r+1) 2^(n-c)), c = log2 of the cluster size).
//
// The gates are cut into phases: maximal runs of gates whose targets lie in a
// set Q of K qubits (controls anywhere).  In a phase every thread loads
// groups of 2^K amplitudes -- the amplitudes that differ only in the Q bits --
// into registers, applies all of the phase's gates there (Eq. NUM2,
// (a_i0, a_i1) <- U (a_i0, a_i1) for the pairs whose control
// bits are 1; a control outside Q is one test per group), and stores them
// back; one barrier per phase instead of one per gate.  A phase whose Q holds
// a cluster-select bit reads and writes other CTAs' blocks through DSMEM
// between two cluster barriers; a phase on local bits only needs the CTA's
// own barrier.  No host work between gates and no HBM traffic between them.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <vector>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace qsim {

#ifndef PC_THREADS_DEF
#define PC_THREADS_DEF 256
#endif
constexpr int PC_THREADS = PC_THREADS_DEF;

// kind of a gate: 0 dense, 1 diagonal (u01 = u10 = 0), 2 anti-diagonal (u00 = u11 = 0);
// the dropped terms are exact zeros, so every kind evaluates the general formula's value
template <int K, int M>
__device__ __forceinline__ void pc_apply(double2 (&v)[1 << K], const PersistOp &op) {
    const double u0r = op.u[0], u0i = op.u[1], u1r = op.u[2], u1i = op.u[3];
    const double u2r = op.u[4], u2i = op.u[5], u3r = op.u[6], u3i = op.u[7];
    const uint32_t cin = op.cin;
    if (op.kind == 1) {
#pragma unroll
        for (int k = 0; k < (1 << (K - 1)); ++k) {
            const int j0 = ((k >> M) << (M + 1)) | (k & ((1 << M) - 1)), j1 = j0 | (1 << M);
            if (((uint32_t)j0 & cin) != cin) continue;
            const double2 x = v[j0], y = v[j1];
            v[j0] = make_double2(fma(u0r, x.x, -u0i * x.y), fma(u0r, x.y, u0i * x.x));
            v[j1] = make_double2(fma(u3r, y.x, -u3i * y.y), fma(u3r, y.y, u3i * y.x));
        }
    } else if (op.kind == 2) {
#pragma unroll
        for (int k = 0; k < (1 << (K - 1)); ++k) {
            const int j0 = ((k >> M) << (M + 1)) | (k & ((1 << M) - 1)), j1 = j0 | (1 << M);
            if (((uint32_t)j0 & cin) != cin) continue;
            const double2 x = v[j0], y = v[j1];
            v[j0] = make_double2(fma(u1r, y.x, -u1i * y.y), fma(u1r, y.y, u1i * y.x));
            v[j1] = make_double2(fma(u2r, x.x, -u2i * x.y), fma(u2r, x.y, u2i * x.x));
        }
    } else {
#pragma unroll
        for (int k = 0; k < (1 << (K - 1)); ++k) {
            const int j0 = ((k >> M) << (M + 1)) | (k & ((1 << M) - 1)), j1 = j0 | (1 << M);
            if (((uint32_t)j0 & cin) != cin) continue;
            const double2 x = v[j0], y = v[j1];
            v[j0] = make_double2(fma(u0r, x.x, fma(-u0i, x.y, fma(u1r, y.x, -u1i * y.y))),
                                 fma(u0r, x.y, fma(u0i, x.x, fma(u1r, y.y, u1i * y.x))));
            v[j1] = make_double2(fma(u2r, x.x, fma(-u2i, x.y, fma(u3r, y.x, -u3i * y.y))),
                                 fma(u2r, x.y, fma(u2i, x.x, fma(u3r, y.y, u3i * y.x))));
        }
    }
}

template <int K>
__global__ void __launch_bounds__(PC_THREADS) k_persist_e(double2 *__restrict__ a, int n, int lcs,
                                                          const PersistPhase *__restrict__ ph, int nph,
                                                          const PersistOp *__restrict__ ops, int nops) {
    constexpr int R = 1 << K;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) double2 pc_sh[];
    const int rank = (int)cluster.block_rank();
    const int cs = 1 << lcs;
    const int lb = n - lcs;  // local bits of a CTA's block
    const uint32_t S = 1u << lb;
    double2 *mine = pc_sh;
    PersistOp *os = reinterpret_cast<PersistOp *>(pc_sh + S);  // the records, staged once
    PersistPhase *ps = reinterpret_cast<PersistPhase *>(os + nops);
    for (uint32_t j = threadIdx.x; j < S; j += PC_THREADS) mine[j] = a[(size_t)rank * S + j];
    for (int k = threadIdx.x; k < nops * (int)(sizeof(PersistOp) / 8); k += PC_THREADS)
        reinterpret_cast<double *>(os)[k] = reinterpret_cast<const double *>(ops)[k];
    for (int k = threadIdx.x; k < nph * (int)(sizeof(PersistPhase) / 8); k += PC_THREADS)
        reinterpret_cast<double *>(ps)[k] = reinterpret_cast<const double *>(ph)[k];
    cluster.sync();
    const uint32_t G = 1u << (n - K), gpc = G / cs;  // groups, per CTA
    bool prev_remote = true;                         // the staging above counts as remote
    for (int p = 0; p < nph; ++p) {
        const PersistPhase P = ps[p];
        const bool remote = P.remote != 0;
        if (remote || prev_remote)
            cluster.sync();
        else
            __syncthreads();
        prev_remote = remote;
        uint32_t off[R];  // member offsets of a group: the Q bits of j
#pragma unroll
        for (int j = 0; j < R; ++j) {
            uint32_t o = 0;
#pragma unroll
            for (int b = 0; b < K; ++b)
                if ((j >> b) & 1) o |= 1u << P.q[b];
            off[j] = o;
        }
        for (uint32_t gi = (uint32_t)rank * gpc + threadIdx.x; gi < (uint32_t)(rank + 1) * gpc; gi += PC_THREADS) {
            uint32_t base = gi;  // zeros inserted at the Q positions (ascending)
#pragma unroll
            for (int b = 0; b < K; ++b) {
                const uint32_t q = P.q[b];
                base = ((base >> q) << (q + 1)) | (base & ((1u << q) - 1u));
            }
            double2 v[R];
            if (!remote) {  // the group lies in this CTA's block
                const uint32_t lo = base & (S - 1u);
#pragma unroll
                for (int j = 0; j < R; ++j) v[j] = mine[lo | off[j]];
            } else {
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const uint32_t i = base | off[j];
                    v[j] = *cluster.map_shared_rank(mine + (i & (S - 1u)), (int)(i >> lb));
                }
            }
            for (int g = P.g0; g < P.g0 + P.ng; ++g) {
                const PersistOp &op = os[g];
                if ((base & op.cout) != op.cout) continue;
                switch (op.m) {
                    case 0: pc_apply<K, 0>(v, op); break;
                    case 1: pc_apply<K, 1>(v, op); break;
                    case 2: pc_apply<K, 2>(v, op); break;
                    default:
                        if (K > 3) pc_apply<K, (K > 3 ? 3 : 0)>(v, op);
                        break;
                }
            }
            if (!remote) {
                const uint32_t lo = base & (S - 1u);
#pragma unroll
                for (int j = 0; j < R; ++j) mine[lo | off[j]] = v[j];
            } else {
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const uint32_t i = base | off[j];
                    *cluster.map_shared_rank(mine + (i & (S - 1u)), (int)(i >> lb)) = v[j];
                }
            }
        }
    }
    cluster.sync();
    for (uint32_t j = threadIdx.x; j < S; j += PC_THREADS) a[(size_t)rank * S + j] = mine[j];
}

// Phases (host).  Gates on disjoint qubit sets commute, so the host may
// reorder them: each qubit keeps the queue of its gates (target and
// controls) in program order, and a gate is ready when it heads the queues
// of all its qubits.  A phase takes ready gates whose target is in its set Q
// (<= K qubits) or can join it.  Remote phases (Q holding a cluster-select
// bit) cost DSMEM traffic and cluster barriers, so a phase stays local while
// a ready gate with a local target exists, and a remote phase then takes the
// ready remote gates first -- batching them.  A closed Q is padded with the
// lowest unused qubits and sorted; each gate becomes an op in the phase's
// coordinates (target position m, controls inside Q as a group-index mask,
// controls outside as a full-index mask).  The reordering changes only the
// rounding order (products of commuting 2x2 factors).
static int kind_of(const double *u) {
    if (u[2] == 0.0 && u[3] == 0.0 && u[4] == 0.0 && u[5] == 0.0) return 1;
    if (u[0] == 0.0 && u[1] == 0.0 && u[6] == 0.0 && u[7] == 0.0) return 2;
    return 0;
}
int persist_plan(const PersistGate *g, int ngates, int n, int K, int lcs, std::vector<PersistPhase> &ph,
                 std::vector<PersistOp> &ops) {
    ph.clear();
    ops.clear();
    const int lb = n - lcs;
    std::vector<std::vector<int>> qq(n);  // per qubit: its gates in program order
    std::vector<size_t> head(n, 0);
    auto touches = [&](int k) { return g[k].cmask | (1u << g[k].t); };
    for (int k = 0; k < ngates; ++k)
        for (int b = 0; b < n; ++b)
            if ((touches(k) >> b) & 1u) qq[b].push_back(k);
    auto ready = [&](int k) {
        const uint32_t m = touches(k);
        for (int b = 0; b < n; ++b)
            if (((m >> b) & 1u) && (head[b] >= qq[b].size() || qq[b][head[b]] != k)) return false;
        return true;
    };
    int left = ngates;
    std::vector<int> Q, sel;
    while (left > 0) {
        Q.clear();
        sel.clear();
        // the phase is local if some ready gate has a local target
        bool remote_phase = true;
        for (int b = 0; b < n && remote_phase; ++b)
            if (head[b] < qq[b].size()) {
                const int k = qq[b][head[b]];
                if (g[k].t < lb && ready(k)) remote_phase = false;
            }
        for (;;) {
            // the next gate: ready, target in Q (lowest program index), else one that can
            // join Q (remote targets first in a remote phase, none in a local one)
            int best = -1, bestjoin = -1;
            for (int b = 0; b < n; ++b) {
                if (head[b] >= qq[b].size()) continue;
                const int k = qq[b][head[b]];
                if (!ready(k)) continue;
                const int t = g[k].t;
                const bool inq = std::find(Q.begin(), Q.end(), t) != Q.end();
                if (inq) {
                    if (best < 0 || k < best) best = k;
                } else if ((int)Q.size() < K && (remote_phase || t < lb)) {
                    const bool pref = remote_phase ? t >= lb : true;
                    const bool bpref = bestjoin >= 0 && (remote_phase ? g[bestjoin].t >= lb : true);
                    if (bestjoin < 0 || (pref && !bpref) || (pref == bpref && k < bestjoin)) bestjoin = k;
                }
            }
            const int k = best >= 0 ? best : bestjoin;
            if (k < 0) break;
            if (best < 0) Q.push_back(g[k].t);
            sel.push_back(k);
            const uint32_t m = touches(k);
            for (int b = 0; b < n; ++b)
                if ((m >> b) & 1u) ++head[b];
            --left;
        }
        if (sel.empty()) return -1;  // cannot happen: the lowest unscheduled gate is always ready
        std::vector<int> q = Q;
        for (int b = 0; (int)q.size() < K && b < n; ++b)
            if (std::find(q.begin(), q.end(), b) == q.end()) q.push_back(b);
        std::sort(q.begin(), q.end());
        PersistPhase P{};
        uint32_t qm = 0;
        for (int b = 0; b < K; ++b) {
            P.q[b] = (uint8_t)q[b];
            qm |= 1u << q[b];
            if (q[b] >= lb) P.remote = 1;
        }
        P.g0 = (int32_t)ops.size();
        for (int k : sel) {
            PersistOp o{};
            for (int i = 0; i < 8; ++i) o.u[i] = g[k].u[i];
            o.kind = (uint8_t)kind_of(g[k].u);
            for (int b = 0; b < K; ++b) {
                if (q[b] == g[k].t) o.m = (uint8_t)b;
                if ((g[k].cmask >> q[b]) & 1u) o.cin |= (uint8_t)(1u << b);
            }
            o.cout = g[k].cmask & ~qm;
            ops.push_back(o);
        }
        P.ng = (int32_t)(ops.size() - P.g0);
        ph.push_back(P);
    }
    return 0;
}

template <int K>
static int launch_k(void *a, int n, int lcs, const PersistPhase *ph, int nph, const PersistOp *ops, int nops,
                    cudaStream_t s) {
    const size_t smem = (sizeof(double2) << (n - lcs)) + (size_t)nops * sizeof(PersistOp) +
                        (size_t)nph * sizeof(PersistPhase);
    static std::atomic<uint64_t> attr_devs{0};  // the >48 KiB opt-in and the 16-CTA cluster are per device
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_devs.load() & bit)) {
        if (cudaFuncSetAttribute(k_persist_e<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) !=
                cudaSuccess ||
            cudaFuncSetAttribute(k_persist_e<K>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            cudaGetLastError();
            return -1;
        }
        attr_devs.fetch_or(bit);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1u << lcs);
    cfg.blockDim = dim3(PC_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1u << lcs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_persist_e<K>, reinterpret_cast<double2 *>(a), n, lcs, ph, nph, ops, nops) !=
        cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return 0;
}

// the cluster size this device runs (16 if a 16-CTA cluster with the largest
// block fits, else 8); cached per device
int persist_lcs() {
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    const int c = cache[dev & 63].load();
    if (c) return c;
    int lcs = 3;
    if (cudaFuncSetAttribute(k_persist_e<4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
        cudaFuncSetAttribute(k_persist_e<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) ==
            cudaSuccess) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(PC_THREADS);
        cfg.dynamicSmemBytes = 200 * 1024;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, k_persist_e<4>, &cfg) == cudaSuccess && nc > 0) lcs = 4;
    }
    cudaGetLastError();
    cache[dev & 63].store(lcs);
    return lcs;
}

// K = 4 (16-amplitude groups) when each CTA still has a full block of groups,
// else 3
int persist_k(int n, int lcs) { return (n - 4 - lcs >= 8) ? 4 : 3; }

int launch_persist_e(void *a, int n, int lcs, int K, const PersistPhase *ph, int nph, const PersistOp *ops,
                     int nops, cudaStream_t s) {
    if (n < PERSIST_MIN_N || n > PERSIST_MAX_N || nops > PERSIST_MAX_GATES || nph > nops) return -1;
    if ((K != 3 && K != 4) || n - lcs < K) return -1;
    return K == 4 ? launch_k<4>(a, n, lcs, ph, nph, ops, nops, s) : launch_k<3>(a, n, lcs, ph, nph, ops, nops, s);
}

}  // namespace qsim
