// lpass.h -- the relabelling tile pass.
//
// One HBM pass over the shard applies a run of gates whose targets lie in a
// tile of K qubits (K <= 12: the 3 lowest local qubits, 128 B contiguous runs,
// plus up to 9 higher ones).  Compared with a gate-by-gate sweep (Eq. NUM2,
// PAPER.md:285-299) the pass reorganises the arithmetic, never the result
// (identical up to fp reassociation):
//
//  * Tile relabelling.  The tile lives in shared memory at "physical"
//    positions p; logical tile index x (bit i = tile qubit i) sits at
//    p = M x XOR b with M an invertible GF(2) matrix and b a vector.  A
//    CNOT / X on tile qubits (the permutation gates of PAPER.md:442-444) only
//    updates M (in-tile control) or b (no control, or controls outside the
//    tile: b gains the vector on the tiles whose control bits are 1): no
//    amplitude moves.  The store at the end of the pass reads logical x from
//    p = M x XOR b, so the shard leaves the pass in logical order.
//  * Register stages.  A stage holds R = 4 (or 5) tile qubits Q in registers:
//    thread groups of 2^R amplitudes are cosets p0 XOR span(M e_q, q in Q).
//    Register j holds logical slot sigma(j) = A (j XOR g) of Q, where A is a
//    host-known R x R GF(2) matrix (in-stage CNOTs) and g a per-group runtime
//    vector (X gates, flips conditioned on qubits outside the registers).
//  * Shear decomposition of a dense 2x2 U (unitary):
//        U = Dl . cos(theta) [[1, -t], [t, 1]] . Dr,   |t| <= 1,
//    Dl, Dr diagonal (when |u01| > |u00|, U = X . V and V is decomposed).  A
//    shear costs 2 fp64 FMAs per amplitude instead of 8 for a general 2x2
//    product; all diagonal factors (Dl, Dr, cos(theta), phase gates, CPHASE)
//    are merged on the host into one 2^R-entry table per flush and applied
//    with one complex multiply per amplitude.  If a gate's decomposition does
//    not reproduce U to 1e-14 the gate is applied as a general 2x2 (DENSE op).
//
// The host compiler (lpass_compile.cpp, pure C++) turns a gate list into an
// LPassParams program; the kernel (lpass.cu) interprets it.  Only the kernel
// touches amplitudes.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#ifdef __CUDACC__
#define LP_HD __host__ __device__
#else
#define LP_HD
#endif

namespace qsim {

constexpr int LP_LOW = 3;           // tile bits 0..2 = local qubits 0..2
constexpr int LP_MAX_K = 12;        // 2^12 amplitudes x 16 B = 64 KiB of shared memory
constexpr int LP_MIN_K = 9;
constexpr int LP_THREADS = 128;
constexpr int LP_MAX_STAGES = 24;
constexpr int LP_MAX_OPS = 192;
constexpr int LP_MAX_EVENTS = 16;
constexpr int LP_MAX_COEF = 1024;   // doubles of diagonal tables (staged in shared memory)
constexpr int LP_MAX_SC = 512;      // scalar coefficients (shear t / a, 2x2 matrices; read from constant memory)
constexpr int LP_MAX_PASS_GATES = 96;

// op codes: v-indexed types use code = type * 16 + vsel (SHEAR / SHEARU: any
// pair vector of weight <= 2; CSHEAR / DENSE / CSWAP: weight 1, vsel < R)
enum : uint8_t {
    LOP_SHEAR = 0,   // shear on the register pair vector v, per-pair orientation
    LOP_SHEARU = 1,  // shear, orientation uniform over the pairs
    LOP_CSHEAR = 2,  // shear restricted to pairs whose in-register controls are 1
    LOP_DENSE = 3,   // general 2x2 (optionally controlled)
    LOP_CSWAP = 4,   // swap the pair when its in-register controls are 1 (data move)
    LOP_NVT = 5,
};
constexpr uint8_t LOP_CODE_DIAGT = 250;  // v[j] *= T[j ^ g]
constexpr uint8_t LOP_CODE_FLIP = 251;   // g ^= gvec
// ROUND: v[j] *= T[j ^ g] (T at coef, 2^R complex), then for every register bit
// r in gvec (ascending) a lifted shear on the pairs (j0, j0 | 2^r) with
// (t_r, a_r) = coef[2^(R+1) + 2k], coef[2^(R+1) + 2k + 1]:
//   logical x += a y;  y += t x     (x = bit-r-0 member of sigma, a = -t / (1 + t^2))
// which with the factor diag(1, 1 + t^2) already in T is exactly the shear
// [[1, -t], [t, 1]]  (L D U factorisation; in place, no register copies).
// Register j0 holds the logical-1 member iff bit r of g is set.
constexpr uint8_t LOP_CODE_ROUND = 252;
constexpr uint8_t LF_COND = 1;           // op applies only where (xq & tmask) == tval && (full & omask) == oval

// number of register pair vectors with weight 1 or 2 (the v-indexed op variants)
LP_HD constexpr int lp_nv(int R) { return R + R * (R - 1) / 2; }
// the vsel-th vector: singles e_0..e_{R-1}, then pairs (a < b) in lexicographic order
LP_HD constexpr int lp_vec(int R, int vsel) {
    if (vsel < R) return 1 << vsel;
    int k = vsel - R;
    for (int a = 0; a < R; ++a)
        for (int b = a + 1; b < R; ++b) {
            if (k == 0) return (1 << a) | (1 << b);
            --k;
        }
    return 0;
}

struct LOp {
    // 8-byte header (read by the kernel as one 64-bit constant load)
    uint8_t code;
    uint8_t flags;
    uint8_t rowS;      // row S of A: bit S of sigma(j) = par(rowS & (j ^ g))
    uint8_t gvec;      // FLIP: A^-1 e_t;  ROUND: register bits sheared
    uint16_t coef;     // DIAGT / ROUND: table offset in coef[]; SHEAR*/DENSE: offset in sc[]
    uint8_t nctl;      // in-register controls (CSHEAR / DENSE / CSWAP); DIAGT / ROUND: table variants
    uint8_t pad0;
    uint32_t pm;       // bit j = par(rowS & j) (SHEARU: bit 0 = the uniform parity; ROUND: offset in sc[])
    uint32_t pmc[2];   // the same for each in-register control row
                       // DIAGT / ROUND: up to 2 pre-flips applied before the op:
                       // bit 16 valid, bits 8-15 condition code (tile bit b -> b,
                       // full-index bit b -> 64 + b, 255 = always), bits 0-7 gvec
    uint8_t rowc[2];
    uint16_t pad1;
    uint16_t tmask, tval;  // condition on the group's logical tile bits outside the registers
    uint32_t pad2;
    uint64_t omask, oval;  // condition on the full index bits outside the tile (tile base | shard base)
};
static_assert(sizeof(LOp) == 48, "LOp layout");

struct LStage {
    uint16_t reg_phys[5];  // swizzled position of register slot r (S M_s e_{q_r})
    uint16_t grp_phys[8];  // swizzled position of group bit i (S M_s e_{q'_i})
    uint16_t grp_log[8];   // logical tile bit of group bit i (1 << q'_i)
    uint16_t y_static;     // M_s^-1 b_static (logical tile bits)
    uint16_t qmask;        // logical tile bits held in registers
    uint8_t qbit[5];       // logical tile bit of register slot r
    uint8_t needs_xq;      // some op tests tile bits outside the registers
    uint16_t first_op, nops;
    uint32_t ev_mask;      // events that happened before this stage
    uint16_t y_ev[LP_MAX_EVENTS];  // M_s^-1 v_e
};

struct LPassParams {
    void *a;
    uint64_t shard_base;   // full physical index of local amplitude 0 (rank bits)
    uint64_t ntiles;
    int32_t nl, K, R, nstages, nevents, ncoef, noio, pad;
    int32_t high_q[LP_MAX_K];          // tile bit LP_LOW + i <-> local qubit (ascending)
    uint16_t scol[LP_MAX_K];           // load: swizzled position of logical tile bit i
    uint16_t smcol[LP_MAX_K];          // store: S M_final e_i
    uint16_t sb_static;                // store: S b_static_final
    uint16_t pad2[3];
    uint16_t sv_ev[LP_MAX_EVENTS];     // store: S v_e
    uint64_t ev_full[LP_MAX_EVENTS];   // event e happens on tiles whose full-index bits ev_full[e] are all 1
    LStage st[LP_MAX_STAGES];
    LOp op[LP_MAX_OPS];
    double coef[LP_MAX_COEF];  // diagonal tables, 2^(R+1) doubles each, table-aligned
    double sc[LP_MAX_SC];
    int32_t nsc, pad3;
};

// A gate of the run in PHYSICAL bit positions (after the planner's qubit map):
// target t, controls ctl[0..nctl) (local < nl, global >= nl), U as in qsim.h.
struct LGate {
    int32_t t, nctl, ctl[2];
    double u[8];
};

struct LCompileStats {
    int stages = 0, ops = 0, diagt = 0, shears = 0, dense = 0, flips = 0, relabels = 0, events = 0, cswaps = 0,
        tile_free = 0, carried = 0, deferred = 0;
};

// Compile gates[0..ng) (all non-diagonal targets inside the tile) into `p`.
// tile_q[i] = local qubit of tile bit i (tile_q[i] = i for i < LP_LOW; the
// rest ascending).  Returns 0 on success, 1 if the run does not fit the
// program limits (the caller shortens the run), -1 on an internal error
// (message in *err).  Fills every field of p except a, shard_base, noio.
//
// With `deferred` non-null, a stage's final pending diagonal that factorises
// over the register qubits is not flushed: its 1-qubit factors are carried to
// the next stage that holds the qubit (absorbed into that stage's first
// table), and whatever is still carried when the pass ends is returned as
// 1-qubit diagonal gates (local qubits) that the caller must apply right
// after the pass, before any remaining gate (they are the last operations of
// the pass on their qubits, so this order is the circuit's).
int lpass_compile(const LGate *gates, int ng, int nl, int K, int R, const int *tile_q, int max_coef,
                  LPassParams &p, LCompileStats *stats, std::string *err, std::vector<LGate> *deferred = nullptr);

// ---- host scheduler: a run of gates -> passes (and single-gate sweeps) ----
// Callbacks of lpass_run: the runtime launches kernels, the CPU emulator
// (tools/lpass_emu.cpp) interprets the same programs.
struct LPassSink {
    virtual ~LPassSink() {}
    // one pass over the shard; ids[k] = index of the k-th pass gate in the
    // caller's list, or -1 for a synthetic (deferred) diagonal
    virtual int pass(const LPassParams &p, const LCompileStats &cs, const std::vector<int> &ids) = 0;
    virtual int sweep(const LGate &g, int id) = 0;  // one gate alone
    virtual double gate_bytes(const LGate &g) = 0;  // algorithmic bytes of the gate alone
};
struct LRunConfig {
    int nl = 0, K = 0, R = 4, max_coef = 0;
    bool defer = true;        // carry / defer diagonals across stages and passes
    double pass_bytes = 0.0;  // bytes of one pass (read + write of the shard)
};
// Greedy commutation-aware pass formation: each pass takes, in order, every
// pending gate that commutes with all skipped earlier ones and whose
// non-diagonal target fits the tile (K - LP_LOW qubits above the 3 lowest),
// up to LP_MAX_PASS_GATES; a program that does not fit gives back its last
// gates; a pass that would move more bytes than its gates alone runs as
// sweeps.  Deferred diagonals are re-queued at the front of the pending
// list; the pass that holds every pending gate defers nothing.  Returns 0 or
// the first nonzero callback / compile code (-1 with *err on internal errors).
int lpass_run(const LGate *gates, int ng, const LRunConfig &cfg, LPassSink &sink, std::string *err);

// ---- device side (lpass.cu) ----
int lpass_max_coef(int R);        // coefficient pool that fits the kernel's shared memory budget
int lpass_ctas_per_sm(int R);
size_t lpass_smem_bytes(int K, int ncoef);
void launch_lpass_e(const LPassParams &p, struct CUstream_st *stream);  // grid = min(ntiles, CTAs/SM x SMs)

}  // namespace qsim
