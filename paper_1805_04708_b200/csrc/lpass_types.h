// lpass_types.h -- the relabelling pass program (constants, LOp, LStage,
// LPassParams): shared by the host compiler (lpass_compile.cpp), the CUDA
// kernel (lpass_dev.cuh) and the run-time specialised kernels compiled with
// NVRTC (lpass.cu), so it includes nothing NVRTC lacks.
#pragma once

#ifndef __CUDACC_RTC__
#include <cstddef>
#include <cstdint>
#endif

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
// DIAG1: a (conditional) diagonal that depends on one logical register slot S
// only: v[j] *= T[b], b = par(rowS & (j ^ g)) (pm: bit j = par(rowS & j)),
// T = (T0, T1) complex at sc[coef .. coef + 4) -- no 2^R table in the pool;
// gvec bit 0 set: T0 == 1 exactly (controlled phases), only the b = 1 half moves
constexpr uint8_t LOP_CODE_DIAG1 = 253;
// PHASES: adjacent controlled phases on one logical register slot S, each
// under one condition bit outside the registers: per group the product
// c = prod_k (bit_k ? e_k : 1) over the nctl terms at sc[coef + 3k] = (code,
// re, im) (code: tile bit b -> b, full-index bit b -> 64 + b), then v[j] *= c
// where par(rowS & (j ^ g)) = 1 -- one complex multiply per term per group
// instead of per amplitude (the QFT's CPHASE ladders).  Terms on full-index
// bits come first; when pmc[1] = m > 0 their product is formed once per tile
// into coef[pmc[0] .. pmc[0] + 2) (shared memory) and the group starts from it
constexpr uint8_t LOP_CODE_PHASES = 254;
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
    int32_t nl, K, R, nstages, nevents, ncoef, noio;
    int32_t nops_ph;                   // ops [0, nops_ph) hold every PHASES op with hoisted terms
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
    int32_t nsc;
    // tile scalars: nts terms (omask, oval as bit patterns, re, im) at sc[ts_off];
    // the product of the terms with (full & omask) == oval multiplies the tile at
    // its store (formed per tile into coef[ts_slot .. ts_slot + 2))
    int32_t nts, ts_off, ts_slot;
};

}  // namespace qsim
