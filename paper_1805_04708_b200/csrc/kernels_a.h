// kernels_a.h -- A-variant (adaptive 2-byte polar code, §4.1) kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

struct qsim_state;

namespace qsim {

struct Shard;
struct PlanOp;

// Decode / encode tables for one pair of bounds (r0, r1).  All values are
// computed on the host in fp64 with the same expressions as PAPER.md:449-453.
struct ATabData {
    double r[256];      // magnitude of b0 (index b0 + 128): 0 for -128, 1 for 127, (b0+127)(r1-r0)/253 + r0
    double thr[256];    // thr[c] = (r0 + (c + 0.5)(r1 - r0)/253)^2, c = 0..252: boundary between codes c, c+1
    double cth[256];    // cos(pi b1 / 128), index b1 + 128
    double sth[256];    // sin(pi b1 / 128)
    double cb[260];     // cos((k + 0.5) pi / 128), index k + 129, k = -129..128
    double sb[260];
    double r0, r1, scale;  // scale = 253 / (r1 - r0) (0 if degenerate)
    int32_t degenerate;    // r1 == r0
    int32_t pad;
};

// fp32 copies of the decode tables for the dense-gate fast path (kernels_a.cu
// "certified fp32"), replicated so that a warp's 32 random lookups never
// share a shared-memory bank: rf[raw b0][lane], cs[raw b1][lane & 15] (a
// 64-bit load serves 16 lanes per wavefront).  Indexed by the raw code byte
// (two's-complement int8), so no bias is added at lookup.
struct AFTab {
    float rf[256][32];
    float cs[256][16][2];
};
static_assert(sizeof(AFTab) == 65536, "AFTab is 64 KiB (one CTA's dynamic shared memory)");

struct ATables {
    ATabData *d[2] = {nullptr, nullptr};
    AFTab *f[2] = {nullptr, nullptr};  // fp32 tables of d[0] / d[1]
    ATabData *h = nullptr;  // pinned host staging
    AFTab *hf = nullptr;
    unsigned long long *gext = nullptr;  // k_bounds_a: the gate's exact (min, max) |z'|^2 bits, grid-wide
    int cur = 0;
};
int atables_alloc(ATables **out);
void atables_free(ATables *t);
int atables_set(ATables *t, double r0, double r1, cudaStream_t s);       // current = next = (r0, r1)
int atables_set_next(ATables *t, double r0, double r1, cudaStream_t s);  // tables for the encode bounds
int atables_commit_next(ATables *t, cudaStream_t s);                     // next becomes current

// A run of diagonal gates that follows a dense gate, applied to the dense
// gate's output codes as they are stored: the same integer b1 steps the
// diagonal sweeps add (exact; k_diag_run_a semantics), so the run costs no
// extra pass.  Per code of a 16-code unit the step is base[j] (gates whose
// target and controls are all unit-internal bits) + the scalar gates (every
// bit outside the unit: one value per unit) + the mixed gates (a unit-index
// condition selecting a per-code pattern).
constexpr int A_EPI_MAX_SCALAR = 48, A_EPI_MAX_MIXED = 4;
struct AEpiScalar {
    uint64_t cext;  // local control bits (all outside the unit)
    int16_t t;      // local target bit outside the unit, or -1: the constant step k0
    int8_t k0, k1;  // b1 steps for target bit 0 / 1
    int32_t pad;
};
struct AEpiMixed {
    uint64_t cext;       // local control bits outside the unit
    int16_t t;           // local target bit outside the unit (selects pat[1]), or -1 (pat[0])
    int16_t pad[3];
    int8_t pat[2][16];   // per code of the unit
};
struct AEpilogue {
    int32_t nscalar, nmixed;
    int8_t base[16];
    AEpiScalar s[A_EPI_MAX_SCALAR];
    AEpiMixed m[A_EPI_MAX_MIXED];
};

struct AGateParams {
    void *a;              // uint16 codes: low byte b0, high byte b1
    uint64_t shard_base;  // full physical index of local 0
    uint64_t cmask;       // full-index control mask
    int32_t nl;
    int32_t t;            // target physical bit (local unless diagonal)
    int32_t cls;
    int32_t pad;
    double u[8];
    // filled by the dense launchers: fp32 copy of U, and the magnitude
    // coefficients of the bounds screen (k_bounds_a): A >= B >= 0 bound
    // max(|u00|, |u11|), max(|u01|, |u10|) from above, a / b their nominal values
    float uf[8];
    float kf[16];  // packed fp32x2 coefficient pairs of a_gate_f2 (a_dense_params, per matrix class)
    float mA, mB, ma, mb;
    // lazy bounds (reading R-A25): codes are written to aout (out of place,
    // nullptr = in place); an output magnitude outside [r0 - d, r1 + d] sets *oor
    void *aout;
    int32_t *oor;
    int32_t has_epi;  // the following diagonal run applied at store (AEpilogue)
    int32_t pad2;
    AEpilogue epi;
};
struct ACollapseParams {
    void *a;
    uint64_t n;
    uint64_t shard_base;
    int32_t bit;  // physical bit measured
    int32_t keep; // outcome kept
    double f;     // 1/sqrt(p_kept)
};

void launch_init_a(void *a, uint64_t n, bool first, cudaStream_t s);
// phase 1 of a dense gate: acc = (min |z'|^2, -max |z'|^2) over intermediates (+inf/+inf if none),
// merged into acc unless `first` (several shards on one device); ncclMin-reducible across ranks
void launch_bounds_a(const AGateParams &p, const ATables *t, double *partials, double *acc, bool first,
                     cudaStream_t s);
// the next tables (r, thr, r0, r1, scale) built on the device from acc (no host round trip)
void launch_tables_next(const double *acc, ATables *t, cudaStream_t s);
void a_bounds_debug_print();  // debug build (-DQSIM_ABND_DEBUG): screen counters of k_bounds_a
// phase 2: decode (current tables), apply, encode (next tables)
void launch_apply_a(const AGateParams &p, const ATables *t, cudaStream_t s);
// the lazy policy's one pass (reading R-A25): decode, apply, encode with the CURRENT
// tables into p.aout, *p.oor |= some intermediate output left [r0 - d, r1 + d]
void launch_apply_a_lazy(const AGateParams &p, const ATables *t, cudaStream_t s);
// exact bounds, fp32 arithmetic without certification (reading R-A26; QSIM_A_POLICY_FP32)
void launch_apply_a_fp32(const AGateParams &p, const ATables *t, cudaStream_t s);
// diagonal / anti-diagonal gates: b1 shifts and code moves, bounds unchanged
void launch_fast_a(const AGateParams &p, const ATables *t, cudaStream_t s);
// A run of consecutive diagonal gates in one sweep: each gate's b1 step
// round(128 arg(u)/pi) per value of its target bit, added under its local
// controls (global targets / controls resolved per shard by the caller into
// constant steps / dropped gates) -- the same integers, summed mod 256, the
// gates add one by one (exact).
constexpr int A_MAX_DIAG_RUN = 48;
struct ADiagRunGate {
    uint32_t cmask;   // local control bits
    int16_t t;        // local target bit, or -1: constant step k0 for the whole shard
    int8_t k0, k1;    // b1 steps for target bit 0 / 1
};
struct ADiagRunParams {
    void *a;
    uint64_t n;       // codes in the shard
    int32_t ngates, pad;
    ADiagRunGate g[A_MAX_DIAG_RUN];
};
void launch_diag_run_a(const ADiagRunParams &p, cudaStream_t s);
int a_phase_steps(double ur, double ui);
void launch_xchg_a(const struct XchgParams &p, const ATables *t, cudaStream_t s);
// collapse phase 1: out = (min |z'|^2, -max |z'|^2)
void launch_collapse_bounds_a(const ACollapseParams &p, const ATables *t, double *partials, double *out,
                              cudaStream_t s);
void launch_collapse_apply_a(const ACollapseParams &p, const ATables *t, cudaStream_t s);

void launch_probs_a(const void *a, int nl, const ATables *t, double *partials, double *out, cudaStream_t s);
void launch_pairdot_a(const void *a, int nl, int q, const ATables *t, double *partials, double *out,
                      cudaStream_t s);
void launch_dot_a(const void *x, const void *y, uint64_t n, const ATables *t, double *partials, double *out,
                  cudaStream_t s);
// <x|y> over n amplitudes; tx / ty: the A tables of an A side, nullptr for an E side
void launch_overlap(const void *x, const ATables *tx, const void *y, const ATables *ty, uint64_t n, double *partials,
                    double *out, cudaStream_t s);
void launch_gather_a(const void *a, const uint64_t *off, uint64_t m, const ATables *t, double *out, cudaStream_t s);
void launch_to_logical_a(const void *a, uint64_t n, uint64_t base, const int *inv, int nq, const ATables *t,
                         void *out, cudaStream_t s);
void launch_codes_to_logical_a(const void *a, uint64_t n, uint64_t base, const int *inv, int nq, void *out,
                               cudaStream_t s);
void launch_codes_from_logical_a(void *a, uint64_t n, uint64_t base, const int *inv, int nq, const void *in,
                                 cudaStream_t s);

int sample_logical(void *const *shard_amps, const uint64_t *shard_base, int nshards, int nl, int nq, const int *inv_host,
                   int enc, const ATables *at, uint64_t nsamp, uint64_t seed, uint64_t *out_host, cudaStream_t s,
                   void *nccl_comm = nullptr);  // NCCL: all-reduce the distribution over the ranks' shards

int shorbox(void *const *shard_amps, const uint64_t *shard_base, int nshards, int nl, int nq, const int *inv_host,
            int enc, int nx, uint64_t G, uint64_t y, cudaStream_t s);

void fill_agate(AGateParams &p, const qsim_state *s, const Shard &sh, const PlanOp &o, const double *u);
int measure_collapse_a(qsim_state *s, int b, int out, double f);

}  // namespace qsim
