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

#include "lpass_types.h"

namespace qsim {

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
// grid = min(ntiles, CTAs/SM x SMs); returns 1 if a run-time specialised (NVRTC) kernel ran, 0 the interpreter
int launch_lpass_e(const LPassParams &p, struct CUstream_st *stream);
void lpass_jit_sync();      // wait for every queued specialisation
void lpass_jit_shutdown();  // stop and join the compile threads (before process exit)
// CUDA source of the kernel specialised to this program (R register qubits,
// minb CTAs per SM, nt threads per CTA, ng register groups per thread at
// once): lp_body with literal stages and ops
// (lpass_dev.cuh)
std::string lpass_jit_source(const LPassParams &p, int R, int minb, int nt = LP_THREADS, int ng = 1);
void lpass_launch_counts(long long *jit, long long *interp);  // specialised (NVRTC) / interpreter launches so far

}  // namespace qsim
