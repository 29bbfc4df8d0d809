// kernels.h -- device kernel parameter blocks and launchers (internal).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace qsim {

// ---- single-gate sweep (a3, a4, a5) ------------------------------------------
// Enumerates the 2^(nl-1-nlc) amplitude groups of one gate: insert a 0 bit at
// every sorted position of {target} U local controls, OR in the local control
// mask (all controls 1), then pair i0 with i1 = i0 | 2^t (Eq. NUM2).
struct SweepParams {
    void *a;                // shard base (double2 for E)
    uint64_t nitems;        // number of groups
    uint64_t cmask;         // local control bits (set after insertion)
    int32_t ins[3];         // sorted insertion positions
    int32_t nins;
    int32_t t;              // target bit (local)
    int32_t cls;            // CLS_DENSE / CLS_DIAG / CLS_ANTI
    int32_t touch;          // DIAG: 3 = both halves, 2 = only i1 (u00 == 1), 1 = only i0 (u11 == 1)
    int32_t pad;
    double u[8];
};
void launch_sweep_e(const SweepParams &p, cudaStream_t s);

// Multiply every amplitude whose local control bits are set by `f` (a diagonal
// gate whose target is a global bit: the factor is uniform on the shard).
struct ScaleParams {
    void *a;
    uint64_t nitems;
    uint64_t cmask;
    int32_t ins[2];
    int32_t nins;
    int32_t pad;
    double f[2];
};
void launch_scale_e(const ScaleParams &p, cudaStream_t s);

// ---- k-qubit dense matrix (qsim_apply_matrix) ---------------------------------
struct MatKParams {
    void *a;
    uint64_t ngroups;   // 2^(nl - k)
    int32_t k;
    int32_t phys[3];    // physical bit of matrix index bit k-1-b (qubits[b])
    int32_t sorted[3];  // the same bits ascending (zero insertion)
    int32_t pad;
    double u[128];      // 2^k x 2^k complex, row-major interleaved
};
void launch_matk_e(const MatKParams &p, cudaStream_t s);

// ---- exchange-fused gate (a7) ------------------------------------------------
struct XchgParams {
    void *own;             // this shard
    const void *stage;     // received chunk (partner's half-shard slice)
    uint64_t p0;           // first half-index of the chunk
    uint64_t n;            // amplitudes in the chunk
    uint64_t shard_base;   // full physical index of local 0 (after the swap)
    uint64_t cmask;        // full-index control mask
    int32_t l;             // victim bit (now holds the gate's target)
    int32_t b;             // this shard's value of the exchanged global bit = slot it keeps
    int32_t mode;          // 0 = copy only (pure swap), 1 = apply gate on arrival
    int32_t cls;
    double u[8];
};
void launch_xchg_e(const XchgParams &p, cudaStream_t s);

// ---- all-to-all remap (remap.cu, NEXT-1 (i)) ---------------------------------
// A block of a shard: the elements whose local bits pos[0] < ... < pos[m-1]
// equal the bits of a value v (bit i of v at pos[i]); element x of the block
// is the x-th such index in increasing order.
struct RemapBlock {
    int32_t m;
    int32_t pos[8];
};
// swap block va of shard a with block vb of shard b (same device), nblock elements each
void launch_blockswap(void *a, void *b, uint64_t nblock, const RemapBlock &blk, uint32_t va, uint32_t vb,
                      size_t elem, cudaStream_t s);
// elements [base, base + count) of block v of src -> out[0 .. count), and back
void launch_pack(const void *src, void *out, uint64_t base, uint64_t count, const RemapBlock &blk, uint32_t v,
                 size_t elem, cudaStream_t s);
void launch_unpack(void *dst, const void *in, uint64_t base, uint64_t count, const RemapBlock &blk, uint32_t v,
                   size_t elem, cudaStream_t s);
// every partner in one launch: slot p (count elements) <-> block vals.v[p]
struct RemapVals {
    int32_t n;
    uint32_t v[7];
};
void launch_pack_multi(const void *src, void *out, uint64_t base, uint64_t count, const RemapBlock &blk,
                       const RemapVals &vals, size_t elem, cudaStream_t s);
void launch_unpack_multi(void *dst, const void *in, uint64_t base, uint64_t count, const RemapBlock &blk,
                         const RemapVals &vals, size_t elem, cudaStream_t s);

// ---- single persistent kernel (config 1, persist.cu) ---------------------------
struct PersistGate {
    double u[8];
    int32_t t;       // physical target bit
    uint32_t cmask;  // physical control bits (full index)
};
constexpr int PERSIST_MIN_N = 4, PERSIST_MAX_N = 16;  // 2^(N-c) amplitudes per CTA of a 2^c-CTA cluster
constexpr int PERSIST_MAX_GATES = 1024;  // records staged in each CTA's shared memory (<= 88 KiB)
// one gate of a phase, in the phase's group coordinates (persist.cu)
struct PersistOp {
    double u[8];
    uint32_t cout;  // control bits outside the phase's qubits (full index)
    uint8_t m;      // target: its position in the phase's sorted qubit list
    uint8_t cin;    // controls among the phase's qubits (group-index mask)
    uint8_t kind;   // 0 dense, 1 diagonal, 2 anti-diagonal
    uint8_t pad;
};
struct PersistPhase {
    uint8_t q[4];   // the phase's K qubits, ascending
    int32_t g0, ng; // its ops [g0, g0 + ng)
    int32_t remote; // a qubit is a cluster-select bit
};
static_assert(sizeof(PersistOp) == 72 && sizeof(PersistPhase) == 16, "record layout");
int persist_lcs();                // log2 of the cluster size this device runs (4 or 3)
int persist_k(int n, int lcs);    // qubits per phase (4 or 3)
int persist_plan(const PersistGate *g, int ngates, int n, int K, int lcs, std::vector<PersistPhase> &ph,
                 std::vector<PersistOp> &ops);
int launch_persist_e(void *a, int n, int lcs, int K, const PersistPhase *ph, int nph, const PersistOp *ops,
                     int nops, cudaStream_t s);

// ---- reductions (a10) ---------------------------------------------------------
// Per-shard: out[0] = sum |a|^2, out[1 + q] = sum_{bit q = 1} |a|^2 for local q.
constexpr int RED_SLOTS = 64;
int red_blocks();
void launch_probs_e(const void *a, int nl, double *partials, double *out, cudaStream_t s);
// S = sum_{i: bit q = 0} conj(a_i) a_{i | 2^q}  (out[0] = re, out[1] = im)
void launch_pairdot_e(const void *a, int nl, int q, double *partials, double *out, cudaStream_t s);
// S = sum_i conj(x_i) y_i over two shards (global-qubit pairs in loopback mode)
void launch_absrange_e(const void *a, uint64_t n, void *out_u64x2, cudaStream_t s);
void launch_dot_e(const void *x, const void *y, uint64_t n, double *partials, double *out, cudaStream_t s);
// Collapse: zero amplitudes whose bit q != keep, scale the others by f.
void launch_collapse_e(void *a, uint64_t n, int q, int keep, double f, cudaStream_t s);
void launch_scale_all_e(void *a, uint64_t n, double f, cudaStream_t s);

// Gather a[off[k]] -> out[k]; scatter in[k] -> a[off[k]] (double2 each)
void launch_gather_e(const void *a, const uint64_t *off, uint64_t m, void *out, cudaStream_t s);
void launch_scatter_e(void *a, const uint64_t *off, uint64_t m, const void *in, cudaStream_t s);
// Permute a shard into logical order: out[logical(shard_base | i)] = a[i]
void launch_to_logical_e(const void *a, uint64_t n, uint64_t shard_base, const int *inv_dev, int nq, void *out,
                         cudaStream_t s);
void launch_from_logical_e(void *a, uint64_t n, uint64_t shard_base, const int *inv_dev, int nq, const void *in,
                           cudaStream_t s);

}  // namespace qsim
