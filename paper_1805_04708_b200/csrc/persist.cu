// persist.cu -- the "single persistent kernel" mode of SURVEY.md §8(d) config 1
// (latency-bound small states, N <= 16): ONE launch applies a whole circuit.
// The state lives in the distributed shared memory of a thread-block cluster
// of 8 CTAs (CTA r holds amplitudes [r 2^(n-3), (r+1) 2^(n-3)), up to 128 KiB
// each); every gate is one sweep over the pairs (Eq. NUM2, PAPER.md:285-307:
// (a_i0, a_i1) <- U (a_i0, a_i1) for the pairs whose control bits are 1)
// followed by a barrier.  A target inside a CTA's block pairs local
// amplitudes (a CTA barrier suffices between such gates); a target among the
// top 3 bits pairs a CTA with its partner CTA through DSMEM (the CTA with the
// bit clear updates both) between two cluster barriers.  No host work between
// gates and no HBM traffic between them.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace qsim {

constexpr int PC_CTAS = 8;  // portable cluster size
constexpr int PC_THREADS = 512;

__global__ void __cluster_dims__(PC_CTAS, 1, 1) __launch_bounds__(PC_THREADS)
    k_persist_e(double2 *__restrict__ a, int n, const PersistGate *__restrict__ g, int ngates) {
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) double2 pc_sh[];
    const int rank = (int)cluster.block_rank();
    const int lb = n - 3;  // local bits of a CTA's block
    const uint32_t S = 1u << lb;
    double2 *mine = pc_sh;
    PersistGate *gs = reinterpret_cast<PersistGate *>(pc_sh + S);  // the gate records, staged once
    for (uint32_t j = threadIdx.x; j < S; j += PC_THREADS) mine[j] = a[(size_t)rank * S + j];
    for (int k = threadIdx.x; k < ngates * (int)(sizeof(PersistGate) / 8); k += PC_THREADS)
        reinterpret_cast<double *>(gs)[k] = reinterpret_cast<const double *>(g)[k];
    cluster.sync();
    bool synced = true;  // the cluster has synchronised since the last gate
    for (int k = 0; k < ngates; ++k) {
        const PersistGate &G = gs[k];
        const int t = G.t;
        // a gate on a cluster-select bit reads / writes a partner CTA's block: the
        // whole cluster must be done with the previous gate; a local gate only
        // needs this CTA done with it
        if (t >= lb && !synced) cluster.sync();
        const double u0r = G.u[0], u0i = G.u[1], u1r = G.u[2], u1i = G.u[3];
        const double u2r = G.u[4], u2i = G.u[5], u3r = G.u[6], u3i = G.u[7];
        const uint32_t cmask = G.cmask;
        double2 *p0, *p1;
        uint32_t base, npairs, q0;
        if (t < lb) {
            p0 = p1 = mine;
            base = (uint32_t)rank * S;
            npairs = S >> 1;
            q0 = 0;
        } else {
            // the CTA pair (r, r | bit) shares the S pairs: each takes half, with its own
            // block on one side of every pair and the partner's on the other
            const int cb = t - lb;
            const int lo = rank & ~(1 << cb), hi = rank | (1 << cb);
            p0 = cluster.map_shared_rank(mine, lo);
            p1 = cluster.map_shared_rank(mine, hi);
            base = (uint32_t)lo * S;
            npairs = S >> 1;
            q0 = (rank >> cb) & 1 ? S >> 1 : 0;
        }
        for (uint32_t q = threadIdx.x; q < npairs; q += PC_THREADS) {
            uint32_t j0, j1;
            if (t < lb) {
                j0 = ((q >> t) << (t + 1)) | (q & ((1u << t) - 1u));
                j1 = j0 | (1u << t);
            } else {
                j0 = j1 = q0 + q;
            }
            const uint32_t i0 = base | j0;  // full index of the |0> member (controls tested on it)
            if ((i0 & cmask) != cmask) continue;
            const double2 x = p0[j0], y = p1[j1];
            double2 nx, ny;
            nx.x = fma(u0r, x.x, fma(-u0i, x.y, fma(u1r, y.x, -u1i * y.y)));
            nx.y = fma(u0r, x.y, fma(u0i, x.x, fma(u1r, y.y, u1i * y.x)));
            ny.x = fma(u2r, x.x, fma(-u2i, x.y, fma(u3r, y.x, -u3i * y.y)));
            ny.y = fma(u2r, x.y, fma(u2i, x.x, fma(u3r, y.y, u3i * y.x)));
            p0[j0] = nx;
            p1[j1] = ny;
        }
        if (t >= lb) {
            cluster.sync();  // the partner's block is written: visible before anyone's next gate
            synced = true;
        } else {
            __syncthreads();
            synced = false;
        }
    }
    cluster.sync();
    for (uint32_t j = threadIdx.x; j < S; j += PC_THREADS) a[(size_t)rank * S + j] = mine[j];
}

int launch_persist_e(void *a, int n, const PersistGate *g, int ngates, cudaStream_t s) {
    if (n < PERSIST_MIN_N || n > PERSIST_MAX_N || ngates > PERSIST_MAX_GATES) return -1;
    const size_t smem = (sizeof(double2) << n) / PC_CTAS + (size_t)ngates * sizeof(PersistGate);
    static std::atomic<uint64_t> attr_devs{0};  // the >48 KiB opt-in is per device
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_devs.load() & bit)) {
        if (cudaFuncSetAttribute(k_persist_e, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)((sizeof(double2) << PERSIST_MAX_N) / PC_CTAS +
                                       PERSIST_MAX_GATES * sizeof(PersistGate))) != cudaSuccess)
            return -1;
        attr_devs.fetch_or(bit);
    }
    k_persist_e<<<PC_CTAS, PC_THREADS, smem, s>>>(reinterpret_cast<double2 *>(a), n, g, ngates);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace qsim
