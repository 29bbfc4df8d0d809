/*
 * qsim.h -- C-ABI of the B200-native JUQCS hot path (arXiv:1805.04708).
 *
 * The library applies single-qubit and controlled (2-/3-qubit) gate matrices
 * to a 2^N-amplitude wave function stored either as complex fp64 ("E",
 * PAPER.md:113-121, 440) or in the paper's adaptive 2-byte polar code ("A",
 * PAPER.md §4.1), sharded over P = 2^k shards by the top k
 * physical index bits (§3.2).  All device work runs in
 * the library's own sm_100a kernels; there is no CPU fallback: a call that
 * needs the GPU fails with QSIM_ECUDA when no device is usable.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Qubit j is bit j of the basis index, qubit 0 least significant
 *    (PAPER.md:255-258).  All qubit and amplitude indices at this boundary are
 *    LOGICAL; the internal qubit map is never visible.
 *  - A 2x2 gate matrix U is 8 doubles, row-major, interleaved (re, im):
 *    {u00r,u00i,u01r,u01i,u10r,u10i,u11r,u11i}; row = output |0>,|1> of the
 *    target.  It is applied to every amplitude pair (a(..0_t..), a(..1_t..))
 *    whose control bits are all 1 (Eq. NUM2; groups of
 *    4/8 for CNOT/TOFFOLI-like gates, App. B
 *    PAPER.md:1300-1363).  U is copied at call time.
 *  - Ownership: the qsim_state handle owns all device memory and streams it
 *    creates; the caller owns every host array passed in or out.
 *  - Synchronisation: apply_* calls are stream-ordered and may return before
 *    the GPU finishes; every read-out call (norm, probabilities,
 *    expectations, measure, get_*) and qsim_sync are synchronous.
 *  - Threading: a handle must not be used from two threads at once.
 *  - Errors: every int-returning function returns QSIM_OK (0) or a negative
 *    QSIM_E* code and sets a thread-local message read by qsim_last_error().
 *    A failed call leaves the state unchanged unless the code is QSIM_ECUDA /
 *    QSIM_ECOMM (device or communicator failure: the state is undefined).
 */
#ifndef QSIM_H
#define QSIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------- */
#define QSIM_OK 0
#define QSIM_EINVAL (-1)       /* bad argument: qubit out of range, duplicates, N outside [2,63], ... */
#define QSIM_ENOMEM (-2)       /* device allocation failed; message states the bytes needed */
#define QSIM_ECUDA (-3)        /* CUDA runtime error or no usable device */
#define QSIM_ECOMM (-4)        /* NCCL error */
#define QSIM_EZERONORM (-5)    /* projection with norm^2 < 1e-14 */
#define QSIM_ENOTUNITARY (-6)  /* ||U^dagger U - I||_max > 1e-10 */
#define QSIM_EUNSUPPORTED (-7) /* valid request this build does not implement */

/* ---- encodings ------------------------------------ */
#define QSIM_ENC_FP64 0      /* E: 16 B/amplitude, interleaved (re, im) fp64 */
#define QSIM_ENC_ADAPTIVE2 1 /* A: 2 B/amplitude, byte 0 = b0 (magnitude), byte 1 = b1 (angle) */

/* ---- transports for sharded states (§3.2, 370-402) ----------- */
#define QSIM_TRANSPORT_LOCAL 0 /* all nshards shards live on this process's device ("loopback"):
                                  the exchange of a global-qubit gate is a device-to-device copy */
#define QSIM_TRANSPORT_NCCL 1  /* one process per GPU; this process owns shard `rank`;
                                  the exchange is NCCL send/recv over NVLink */
#define QSIM_TRANSPORT_DEVICES 2 /* one process drives nshards GPUs (devices `device`.. `device` + P - 1,
                                  `device` = -1 meaning 0): shard r on device r, an in-process NCCL
                                  communicator, one host thread per device running each call on its
                                  shard -- the NCCL code path with every rank in this process */

/* ---- gate records ---------------------------------------------------- */
#define QSIM_GATE_U 0    /* controlled 2x2 gate: target, controls[0..ncontrols-1], u */
#define QSIM_GATE_SWAP 1 /* SWAP(target, target2): a relabelling of the qubit map, moves 0 bytes */

typedef struct qsim_state qsim_state; /* opaque; owns all device memory of one process */

typedef struct qsim_gate {
    int32_t kind;        /* QSIM_GATE_U or QSIM_GATE_SWAP */
    int32_t target;      /* logical target qubit, 0..N-1 */
    int32_t target2;     /* SWAP only: second qubit; ignored otherwise */
    int32_t ncontrols;   /* 0, 1 or 2 */
    int32_t controls[2]; /* logical control qubits, distinct from target and each other */
    double u[8];         /* U as described above (ignored for SWAP) */
} qsim_gate;             /* 88 bytes, no padding */

typedef struct qsim_config {
    int32_t n_qubits;    /* N, 2 <= N <= 63 (QUBITS) */
    int32_t encoding;    /* QSIM_ENC_* */
    int32_t nshards;     /* P = 2^k >= 1; N - k >= 10 local qubits required */
    int32_t transport;   /* QSIM_TRANSPORT_* (ignored when nshards == 1) */
    int32_t rank;        /* NCCL: this process's shard index, 0..P-1 */
    int32_t device;      /* CUDA device ordinal to use; -1 = current device */
    const uint8_t *nccl_id; /* NCCL: 128-byte ncclUniqueId from qsim_nccl_unique_id on rank 0 */
    int64_t chunk_bytes; /* exchange chunk per transfer; 0 = default (2^{N-3}/P B in
                            total, i.e. 2^{N-4}/P per buffer of a double buffer, capped at 512 MiB) */
    int32_t fuse;        /* 1 = fuse runs of gates into shared-memory tile passes (default), 0 = one sweep per gate */
    int32_t a_policy;    /* A encoding: when (r0, r1) are updated ("need to be updated"):
                            QSIM_A_POLICY_EXACT (0, default): exact bounds of every dense gate's output
                            (reading R-A4; two passes, 6 B/amp); QSIM_A_POLICY_LAZY (1): kept while the
                            outputs stay within one step of them, exact rescale when one leaves (reading
                            R-A25; one out-of-place pass of 4 B/amp in range, a second code buffer);
                            QSIM_A_POLICY_FP32 (2): exact bounds, the decode / apply / encode in fp32
                            without the certified fp64 fallback (reading R-A26, SURVEY 8(f) NEXT-4 "fp32
                            decode/apply"): codes within one step of the fp64 reference's */
} qsim_config;
#define QSIM_A_POLICY_EXACT 0
#define QSIM_A_POLICY_LAZY 1
#define QSIM_A_POLICY_FP32 2

/* Counters since creation (or the last qsim_reset_stats). Bytes are ALGORITHMIC
 * bytes (SURVEY.md §8(d) byte-accounting rule), summed over the shards this
 * process owns. */
typedef struct qsim_stats {
    int64_t gates;            /* gate records applied (SWAPs included) */
    int64_t kernels;          /* device kernels launched by the library */
    int64_t sweeps;           /* single-gate sweep launches */
    int64_t passes;           /* fused tile-pass launches */
    int64_t fused_gates;      /* gates applied inside fused passes */
    int64_t exchanges;        /* global<->local swap exchanges (a7) */
    double hbm_bytes;         /* algorithmic HBM bytes of sweeps + passes + exchange kernels */
    double gate_bytes;        /* sum over gates of the per-gate algorithmic bytes had each run alone */
    double exchange_bytes;    /* bytes sent per direction by this process's shards */
    int64_t stages;           /* register stages summed over fused passes */
    int64_t jit_passes;       /* fused passes run by a run-time specialised kernel (the rest interpreted) */
    int64_t a_rescales;       /* A: dense gates that (re)computed the bounds (every dense gate for the exact
                                 policy; the out-of-range ones for the lazy policy) */
    int64_t a_dense;          /* A: dense gates applied */
} qsim_stats;

/* ---- lifetime ---------------------------------------------------------- */

/* Create |0...0> (Eq. appa0) with N qubits in `encoding`,
 * sharded over `ngpus` GPUs driven by this process: shard r on device r
 * (QSIM_TRANSPORT_DEVICES; ngpus = 1: the current device).  The top
 * log2(ngpus) qubits are global.  Every other call takes
 * the handle as for one GPU; read-outs are collective and return one result.
 * Use qsim_create_ex for one process per GPU (QSIM_TRANSPORT_NCCL) or for
 * several shards on one device (QSIM_TRANSPORT_LOCAL, "loopback").
 * *out receives the handle.  Errors: EINVAL (N, ngpus not a power of two or
 * more than the visible GPUs, fewer than 10 local qubits), ENOMEM (message
 * has the byte count), ECUDA, ECOMM. */
int qsim_create(int n_qubits, int encoding, int ngpus, qsim_state **out);

/* Full configuration (see qsim_config).  For QSIM_TRANSPORT_NCCL every rank
 * calls this collectively with the same n_qubits/encoding/nshards/nccl_id. */
int qsim_create_ex(const qsim_config *cfg, qsim_state **out);

/* Free all device memory and the communicator.  NULL is a no-op. */
int qsim_destroy(qsim_state *s);

/* Rank 0 of a QSIM_TRANSPORT_NCCL job calls this and broadcasts the 128
 * bytes to the other ranks (e.g. over torch.distributed). ECOMM on failure. */
int qsim_nccl_unique_id(uint8_t out[128]);

/* ---- gates (a2-a8) -------------------------------------------------------- */

/* Apply U to logical `target` iff all `controls` are 1 (Eq. NUM2 with
 * controls).  A gate whose target sits on a global
 * (shard-index) bit is preceded by a half-shard swap exchange that moves the
 * qubit to a local bit; diagonal gates never exchange.
 * Errors: EINVAL (qubit outside [0,N), duplicates, ncontrols > 2),
 * ENOTUNITARY. */
int qsim_apply_gate(qsim_state *s, const double u[8], int target, const int *controls, int ncontrols);

/* A k-qubit unitary U (k = 1..3: SPEC's apply_two / apply_three) on logical
 * qubits[0..k): U is 2^k x 2^k complex, row-major, interleaved (re, im);
 * qubits[0] is the MOST significant bit of the matrix index (reading A14),
 * i.e. U[r][c] maps basis state c to r with bit (k-1-b) of r/c = qubit b.
 * Global qubits of the set are first brought to local bits by half-shard
 * swap exchanges; one sweep over the shard (32 B per
 * amplitude).  E encoding only (A: QSIM_EUNSUPPORTED).  Errors: EINVAL (k,
 * range, duplicates, non-finite), ENOTUNITARY (||U^dagger U - I||_max > 1e-10). */
int qsim_apply_matrix(qsim_state *s, const double *U, const int *qubits, int k);

/* SWAP(q1, q2) as a qubit-map relabelling (0 bytes moved).  EINVAL. */
int qsim_apply_swap(qsim_state *s, int q1, int q2);

/* Apply `ngates` records in order.  Consecutive local gates are fused into
 * shared-memory tile passes (one HBM pass for many gates, the "combining
 * ... to multi-qubit gates" of PAPER.md:787-790); the result equals applying
 * them one by one up to floating-point reassociation (E) or is the same
 * per-gate A computation (A gates are never fused).  All records are
 * validated before any is applied; EINVAL / ENOTUNITARY name the index. */
int qsim_apply_circuit(qsim_state *s, const qsim_gate *gates, size_t ngates);

/* The whole circuit in ONE kernel launch (the
 * latency-bound small states): the state lives in the distributed shared
 * memory of an 8-CTA thread-block cluster, each gate is one sweep over the
 * pairs (Eq. NUM2 with controls) followed by a cluster
 * barrier; SWAP records relabel the qubit map.  One launch per 1024 gate
 * records.  E encoding, one shard on one device, 4 <= N <= 16 (EINVAL /
 * EUNSUPPORTED otherwise).  Same results as
 * qsim_apply_circuit up to fp reassociation.  Stream-ordered like
 * qsim_apply_circuit. */
int qsim_apply_circuit_persistent(qsim_state *s, const qsim_gate *gates, size_t ngates);

/* ---- read-out (a10, a11) ------------------------------------------------- */

/* Sum_i |a_i|^2 (Eq. STAT1), decoded amplitudes for A. */
int qsim_norm(qsim_state *s, double *norm2);

/* out[0] + i out[1] = <a|b> = sum_x conj(a_x) b_x over the logical basis
 * (decoded amplitudes for an A side), e.g. the fidelity |<A|E>|^2 / (<A|A><E|E>)
 * of an A run against an E run of the same circuit (SURVEY.md §8(d) config 4,
 * BASELINE north_star "fidelity against fp64 reported").  Both handles must
 * live in this process on the same device with the same N and shard count,
 * the loopback transport, and the same qubit map and shard labels (as two
 * runs of one circuit have): QSIM_EUNSUPPORTED otherwise.  Synchronous. */
int qsim_overlap(qsim_state *a, qsim_state *b, double *out);

/* Magnitude range of an E state: *max = max_x |a_x|, *min_nonzero = min over
 * the x with a_x != 0 of |a_x| (0 if the state is all zero) -- the fp64
 * counterpart of the A bounds r0 / r1, used to report the
 * value distribution of the workloads.  A device reduction
 * (exact: min / max are order-independent); all-reduced over NCCL ranks.
 * QSIM_EUNSUPPORTED for the A encoding (its range is (r0, r1), qsim_get_codes).
 * Synchronous. */
int qsim_magnitude_range(qsim_state *s, double *min_nonzero, double *max);

/* p1[n] = P(qubit n = 1) = sum over |a(..1_n..)|^2, n = 0..N-1,
 * not renormalised.  p1 has N entries. */
int qsim_probabilities(qsim_state *s, double *p1);

/* BEGIN MEASUREMENT: q[3n+0..2] = <Qx(n)>, <Qy(n)>, <Qz(n)>
 * with <Qa(n)> = <psi|(1 - sigma^a_n)|psi> / (2 <psi|psi>), i.e. of the
 * normalised state (Eq. STAT1; matters for A, whose encoding drifts the norm).
 * q has 3N entries.  May move
 * global qubits to local bits (a relabelling; the logical state is unchanged). */
int qsim_expectations(qsim_state *s, double *q);

/* Projective measurement M of `qubit`: p0 = P(0)/norm^2,
 * outcome 0 iff u < p0, then the other half is zeroed and the kept half is
 * scaled by 1/sqrt(p_kept) (E) or re-encoded (A).  qsim_measure derives u
 * from `seed` with splitmix64: x = splitmix64(seed), u = (x >> 11) * 2^-53.
 * p0_out may be NULL.  EZERONORM if the kept half has norm^2 < 1e-14. */
int qsim_measure(qsim_state *s, int qubit, uint64_t seed, int *outcome);
int qsim_measure_u(qsim_state *s, int qubit, double u, int *outcome, double *p0_out);

/* GENERATE EVENTS (App. B): draw `nsamples` basis states
 * (LOGICAL indices, written to out[0..nsamples)) from |a|^2, without changing
 * the state.  Event k uses u_k = (splitmix64(seed + k) >> 11) * 2^-53 and is the
 * smallest logical index L with cumsum_{L' <= L} |a_L'|^2 > u_k * norm^2
 * (inverse CDF in logical order).  Needs 8 B x 2^N of scratch (N <= 34);
 * for the NCCL transport every rank calls it collectively: the ranks'
 * probability masses are all-reduced into the full distribution and every
 * rank draws the same events.  EZERONORM for a zero state. */
int qsim_sample(qsim_state *s, size_t nsamples, uint64_t seed, uint64_t *out);

/* SHORBOX n_x G y (App. B; §5.4):
 * replace the state by 2^{-nx/2} sum_{x=0}^{2^nx - 1} |x>|y^x mod G>, the
 * x-register on logical qubits 0..nx-1 and the f-register on nx..N-1 (the
 * logical index is x + 2^nx f).  Direct preparation: no gates, no exchange.
 * EINVAL unless 0 <= nx < N, 2 <= G <= 2^(N-nx) and 1 <= y < G. */
int qsim_prepare_shorbox(qsim_state *s, int nx, uint64_t G, uint64_t y);

/* Set the logical -> physical qubit map (pos[q] = physical bit of logical
 * qubit q, a permutation of 0..N-1): BIT ASSIGNMENT (App. B, PAPER.md:
 * 1424-1449), a performance choice that leaves results unchanged when issued
 * on |0...0> (right after qsim_create / qsim_reset); on another state it
 * relabels the qubits.  EINVAL unless pos is a permutation. */
int qsim_set_qubit_map(qsim_state *s, const int *pos);

/* ---- the assembler-like instruction language (App. B) --
 * qsim_asm_parse compiles a program text (host only, no GPU): one instruction
 * per line, '!' starts a comment, mnemonics case-insensitive; QUBITS N first;
 * BIT ASSIGNMENT and DEPOLARIZING CHANNEL before the first gate; gates I H X Y
 * Z S S+ T T+ U1 U2 U3 +X -X +Y -Y R CNOT U TOFFOLI with the matrices of
 * App. B; BEGIN MEASUREMENT, GENERATE EVENTS, M, SHORBOX, CLEAR, SET, EXIT.
 * Errors: EINVAL with "line L: ..." in qsim_last_error().  qsim_asm_run
 * executes it on a fresh state (encoding; ngpus shards on the current device,
 * QSIM_TRANSPORT_LOCAL): runs of gates
 * go to qsim_apply_circuit; BEGIN MEASUREMENT appends the 3N expectations of
 * qsim_expectations to the result; M n appends (n, outcome) drawn by
 * qsim_measure with seed = seed + (measurement index); GENERATE EVENTS draws
 * with qsim_sample (its own seed if > 0, else `seed`) and ends the run;
 * EXIT measures qubits 0..N-1 and ends the run; the depolarising channel
 * inserts X/Y/Z after every gate (reading R-B11).  The result object owns its
 * arrays; qsim_asm_result_get copies min(cap, count) items into buf and
 * returns the full count. */
typedef struct qsim_asm qsim_asm;
typedef struct qsim_asm_result qsim_asm_result;
#define QSIM_ASM_GATE 0        /* `gate` holds the record */
#define QSIM_ASM_MEASURE_ALL 1 /* BEGIN MEASUREMENT */
#define QSIM_ASM_EVENTS 2      /* GENERATE EVENTS args[0] = events, args[1] = seed */
#define QSIM_ASM_M 3           /* M args[0] */
#define QSIM_ASM_SHORBOX 4     /* args = nx, G, y */
#define QSIM_ASM_CLEAR 5       /* args[0] = qubit */
#define QSIM_ASM_SET 6         /* args[0] = qubit */
#define QSIM_ASM_EXIT 7
typedef struct qsim_asm_op {
    int32_t type;    /* QSIM_ASM_* */
    int32_t line;    /* source line */
    int64_t args[3];
    qsim_gate gate;  /* QSIM_ASM_GATE */
} qsim_asm_op;
#define QSIM_ASM_R_TABLES 0   /* double: 3N per BEGIN MEASUREMENT (<Qx>,<Qy>,<Qz> per qubit) */
#define QSIM_ASM_R_OUTCOMES 1 /* int32 pairs (qubit, outcome) per measured qubit */
#define QSIM_ASM_R_EVENTS 2   /* uint64 logical basis indices */
int qsim_asm_parse(const char *text, qsim_asm **out);
int qsim_asm_info(const qsim_asm *a, int *n_qubits, int64_t *nops, int *perm /* N, nullable */,
                  double *depol /* 4: p_x, p_y, p_z, seed; nullable */);
int qsim_asm_get_op(const qsim_asm *a, int64_t i, qsim_asm_op *op);
void qsim_asm_destroy(qsim_asm *a);
int qsim_asm_run(const qsim_asm *a, int encoding, int ngpus, uint64_t seed, qsim_asm_result **out);
int qsim_asm_result_get(const qsim_asm_result *r, int what, void *buf, int64_t cap, int64_t *count);
void qsim_asm_result_destroy(qsim_asm_result *r);

/* ---- auxiliary-variable method (§4.2) -------------
 * Stateless: no qsim_state, no 2^N vector.  out[2k], out[2k+1] = <y_k|psi>
 * (re, im) for the LOGICAL indices y_k = idx[k] (< 2^N), psi = the gate list
 * applied to |0...0> (Eq. appa0), by
 *     <y|psi> = 2^{-P} sum_{s_1..s_P = +-1} prod_j <y_j| W_j(s) |0>_j   (Eq. appa7)
 * where every CNOT is H_t U_ct(pi) H_t and every controlled phase
 * U_ct(a) (Eq. appa4) becomes a sum over one auxiliary variable by the
 * discrete Hubbard-Stratonovich identity, cos 2x = e^{ia/2} (Eqs. appa5-6).
 * Gates: single-qubit gates, and one-control gates whose 2x2 is diagonal or
 * anti-diagonal (reading R-B9: diag(1, d0) on the control and U_ct(arg
 * d1/d0), then a CNOT for the anti-diagonal case).  abs_sum (nullable, m
 * doubles) receives 2^{-P} sum_s |term_s|: the HS terms are not bounded by
 * 1 (x is complex), so the rounding error of the sum scales with it.  Runs on
 * the current CUDA device; work O(2^P (number of qubits with variables) m).
 * Errors: EINVAL (N outside [2,63], bad qubits / indices), EUNSUPPORTED
 * (SWAP records, two controls, a controlled dense 2x2, P > 40, more than 2^20
 * values on one qubit), ECUDA. */
int qsim_aux_amplitudes(int n_qubits, const qsim_gate *gates, size_t ngates, const uint64_t *idx, size_t m,
                        double *out, double *abs_sum);
/* Number P of auxiliary variables of a gate list (host only, no GPU). */
int qsim_aux_num_vars(int n_qubits, const qsim_gate *gates, size_t ngates, int *P);

/* CLEAR (value 0) / SET (value 1) of App. B: project
 * `qubit` onto |value> and renormalise.  EZERONORM if the projected state has
 * norm^2 < 1e-14 ("fails if the projection results in a state with amplitude
 * zero"); the state is then unchanged. */
int qsim_project(qsim_state *s, int qubit, int value);

/* Amplitudes at `n` LOGICAL basis indices (each < 2^N), written as
 * out[2k] = re, out[2k+1] = im (decoded for A).  For NCCL every rank
 * calls it collectively and receives all n values. */
int qsim_get_amplitudes(qsim_state *s, const uint64_t *logical_idx, size_t n, double *out);

/* Whole state in logical order (2^N complex, interleaved), for tests at
 * small N (N <= 30).  get: E or A (decoded); set: E only (A: EUNSUPPORTED). */
int qsim_get_state(qsim_state *s, double *out);
int qsim_set_state(qsim_state *s, const double *amps);

/* The A state's current bounds (r0, r1) (min / max |z| over
 * the intermediate amplitudes; (0.5, 0.5) before any exists, reading R-A8),
 * without reading the codes.  QSIM_EUNSUPPORTED for E.  Synchronous. */
int qsim_get_bounds(qsim_state *s, double *r0, double *r1);

/* A only: raw codes in logical order (2^N pairs (b0, b1) as int8) and the
 * magnitude bounds r0 <= r1.  EUNSUPPORTED for E. */
int qsim_get_codes(qsim_state *s, int8_t *codes, double *r0, double *r1);
int qsim_set_codes(qsim_state *s, const int8_t *codes, double r0, double r1);

/* ---- plumbing --------------------------------------------------------- */

/* Re-initialise to |0...0> (Eq. appa0) and reset the qubit map; keeps all
 * allocations (so a benchmark step can start from the method's input state). */
int qsim_reset(qsim_state *s);

/* Re-initialise to the basis state |x> (logical index x, bit q = qubit q,
 * PAPER.md:255-258): a(x) = 1, every other amplitude 0 -- the state X on the
 * set bits of x makes from |0...0>, prepared without a pass over the state
 * beyond the reset (config 5's input |x>).  Resets the qubit map like
 * qsim_reset.  EINVAL unless x < 2^N or while a graph capture is open. */
int qsim_reset_basis(qsim_state *s, uint64_t x);

/* Per-kernel-class timing: while enabled, every library kernel launch is
 * bracketed by CUDA events on the launching stream.  qsim_profile_read
 * synchronises, aggregates the finished records per class into out[0..max)
 * (*nout = classes written), and clears them.  Bytes are algorithmic bytes. */
#define QSIM_K_PASS 0      /* fused tile pass (E) */
#define QSIM_K_SWEEP 1     /* single-gate sweep (E) */
#define QSIM_K_XCHG 2      /* exchange-fused gate / swap copy (E and A) */
#define QSIM_K_A_BOUNDS 3  /* A phase 1: post-gate bounds */
#define QSIM_K_A_APPLY 4   /* A phase 2: decode-apply-encode */
#define QSIM_K_A_FAST 5    /* A permutation / phase gates */
#define QSIM_K_NUM 6
typedef struct qsim_kernel_profile {
    int32_t kind;
    int32_t pad;
    int64_t launches;
    double ms;     /* summed event durations */
    double bytes;  /* summed algorithmic bytes */
    double flops;  /* summed algorithmic fp64 flops (14 per amplitude of a dense
                      gate, 6 per touched amplitude of a phase gate, 0 for permutations) */
} qsim_kernel_profile;
int qsim_profile(qsim_state *s, int enable);
int qsim_profile_read(qsim_state *s, qsim_kernel_profile *out, int max, int *nout);

/* Wait for all work of this handle. */
int qsim_sync(qsim_state *s);

/* The fused pass runs a compiled gate program either in the interpreter
 * kernel or in a kernel specialised to that program (NVRTC, sm_100a, cached
 * per program shape, compiled in background threads; the two run the same
 * device functions, so results do not depend on which ran).  This call
 * waits until every specialisation queued so far has been compiled (or has
 * failed: such programs keep running interpreted).  QSIM_LPASS_JIT = 0 / 1
 * (default) / 2 selects off / background / compile-at-first-launch. */
int qsim_jit_sync(void);

/* Stop the compile threads of the specialisations and wait for their
 * in-flight compiles; later passes run interpreted.  Call it before the
 * process exits while compiles may be running (the Python binding registers
 * it with atexit): exit handlers must not wait for threads that may need the
 * dynamic loader. */
int qsim_jit_shutdown(void);

/* ---- CUDA graphs of a gate sequence (the
 * latency-bound N=14 circuit with "per-gate launch, a CUDA Graph, and a
 * single persistent kernel") ----------------------------------------------
 * qsim_graph_begin starts capturing every launch this handle makes on its
 * stream (nothing runs); the gate calls that follow (qsim_apply_gate /
 * qsim_apply_circuit) are planned and compiled on the host as usual;
 * qsim_graph_end stops the capture and instantiates the graph (*out, owned
 * by the caller, freed with qsim_graph_destroy).  qsim_graph_launch replays
 * it on the handle's stream: the same kernels with the same parameters,
 * i.e. the captured gate sequence applied again to the CURRENT state, with
 * no host planning.  Valid only when the captured sequence leaves the
 * logical->physical qubit map and the shard labels unchanged (so a replay
 * sees the layout the capture saw); otherwise qsim_graph_end returns
 * QSIM_EUNSUPPORTED and the state is in an unspecified (but allocated)
 * condition -- call qsim_reset.  E encoding and the loopback transport only
 * (the A encoding synchronises with the host for its bounds; NCCL uses a
 * second stream): QSIM_EUNSUPPORTED otherwise.  Read-out calls between
 * begin and end return QSIM_EINVAL.  Profiling records are not taken while
 * capturing. */
typedef struct qsim_graph qsim_graph;
int qsim_graph_begin(qsim_state *s);
int qsim_graph_end(qsim_state *s, qsim_graph **out);
int qsim_graph_launch(qsim_state *s, qsim_graph *g);
int qsim_graph_destroy(qsim_graph *g);

/* The cudaStream_t (as void*) the library launches shard `shard`'s kernels
 * on (shard index local to this process), for event timing by the caller. */
void *qsim_stream(qsim_state *s, int shard);

int qsim_get_stats(qsim_state *s, qsim_stats *out);
int qsim_reset_stats(qsim_state *s);

/* Logical qubit -> physical bit map (N ints); bits >= N - log2(P) are global. */
int qsim_get_qubit_map(qsim_state *s, int *pos);

/* Thread-local message of the last failed call ("" if none). */
const char *qsim_last_error(void);

/* ---- planner (host only; callable without a GPU) ---------------------------
 * The exchange/remap plan the executor follows (a2, a7): for testing the
 * sharded path's host logic on CPU.  An op is either
 *   QSIM_OP_EXCHANGE: swap physical global bit `g` with local bit `l`
 *     (the shards holding global bits G and G ^ 2^(g-nl) trade half-shards;
 *     qubit map updated),
 *   QSIM_OP_GATE: gate on physical bits (target `l`, controls) with class
 *     0 = dense, 1 = diagonal, 2 = anti-diagonal, 3 = identity (skipped), or
 *   QSIM_OP_RELABEL: an anti-diagonal gate (X, CNOT, Toffoli, Y, ...) whose
 *     target `l` and controls are all global bits: its phase part runs as a
 *     diagonal gate and its permutation part only relabels which shard holds
 *     which global bits -- no data moves (PAPER.md:389-392 does this for
 *     SWAP; CNOT "can be implemented without having to exchange data",
 *     P:395-400), or
 *   QSIM_OP_REMAP: one (global bit `g`, local bit `l`) pair of a
 *     simultaneous swap of m >= 2 global bits with m local bits (SURVEY.md
 *     §8(f) NEXT-1 (i)); the m consecutive REMAP ops with the same
 *     gate_index form ONE all-to-all: every shard trades 2^nl (1 - 2^-m)
 *     amplitudes with the 2^m - 1 shards that differ from it in those global
 *     bits, instead of m pairwise half-shard exchanges (m/2 of a shard).  The
 *     planner emits it when the gate that needs a global target is followed,
 *     within 2N gates, by non-diagonal gates on other global targets.
 * Ownership: qsim_plan_create allocates *out, qsim_plan_destroy frees it. */
#define QSIM_OP_EXCHANGE 0
#define QSIM_OP_GATE 1
#define QSIM_OP_RELABEL 2
#define QSIM_OP_REMAP 3
typedef struct qsim_plan qsim_plan;
typedef struct qsim_plan_op {
    int32_t type;        /* QSIM_OP_* */
    int32_t g;           /* EXCHANGE / REMAP: global physical bit */
    int32_t l;           /* EXCHANGE / REMAP: local victim bit; GATE: physical target bit */
    int32_t cls;         /* GATE: matrix class */
    int32_t ncontrols;   /* GATE */
    int32_t controls[2]; /* GATE: physical control bits */
    int32_t gate_index;  /* GATE: index of the record in the input list */
} qsim_plan_op;

int qsim_plan_create(int n_qubits, int nshards, const int *initial_map, const qsim_gate *gates, size_t ngates,
                     qsim_plan **out);
int64_t qsim_plan_num_ops(const qsim_plan *p);
int qsim_plan_get_op(const qsim_plan *p, int64_t i, qsim_plan_op *op);
int qsim_plan_final_map(const qsim_plan *p, int *pos);
void qsim_plan_destroy(qsim_plan *p);

#ifdef __cplusplus
}
#endif
#endif /* QSIM_H */
