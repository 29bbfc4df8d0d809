/*
 * qsim_oracle.c -- ORACLE: TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU state-vector simulator written from
 * /root/reference/PAPER.md (arXiv:1805.04708, "Massively parallel quantum
 * computer simulator, eleven years later").  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this file.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_1805_04708_b200/csrc) and neither side includes the other.
 *
 * Conventions (all from the paper):
 *  - state: 2^N complex amplitudes a(i), stored interleaved (re, im) in fp64
 *    ("two 8-byte floating point numbers to encode one complex
 *    amplitude"; Eq. STAT2).
 *  - qubit j is bit j of the basis index i, qubit 0 rightmost
 *    (PAPER.md:255-258).
 *  - a single-qubit gate U on qubit t updates every pair
 *    (a(*..0_t..*), a(*..1_t..*)) by the 2x2 matrix U (Eq. NUM2,
 *    PAPER.md:285-299); a controlled gate updates only the pairs whose control
 *    bits are all 1 (groups of 4 / 8; App. B CNOT, U(k),
 *    TOFFOLI: PAPER.md:1300-1363).
 *  - U is given row-major as {u00r,u00i,u01r,u01i,u10r,u10i,u11r,u11i};
 *    row = output |0>,|1> of the target.
 *
 * The A ("adaptive", 2 bytes per amplitude) functions follow PAPER.md §4.1
 * (lines 446-460) step by step; the readings of the points the paper leaves
 * open are DESIGN.md readings R-A3..R-A11.
 *
 * Parity pins for every function live in tests/test_oracle_*.py (marked
 * "not gpu").  Build: gcc -O2 -fopenmp -shared -fPIC (see oracle/__init__.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_PI 3.14159265358979323846

/* ------------------------------------------------------------------------ */
/* E: exact complex fp64 state                                               */
/* ------------------------------------------------------------------------ */

/* |0...0> (Eq. appa0): a(0)=1, all others 0. */
void oracle_e_init(double *a, int n)
{
    uint64_t dim = (uint64_t)1 << n;
    memset(a, 0, sizeof(double) * 2 * dim);
    a[0] = 1.0;
}

/* Eq. NUM2 generalised to controls:
 * for every i with bit t = 0 and all control bits = 1, j = i | 2^t,
 * (a_i, a_j) <- (u00 a_i + u01 a_j, u10 a_i + u11 a_j). */
int oracle_e_apply(double *a, int n, const double *u, int t, const int *ctrl, int nctrl)
{
    uint64_t dim = (uint64_t)1 << n;
    uint64_t tbit = (uint64_t)1 << t;
    uint64_t cmask = 0;
    for (int k = 0; k < nctrl; ++k) cmask |= (uint64_t)1 << ctrl[k];
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < (int64_t)dim; ++i) {
        uint64_t ii = (uint64_t)i;
        if (ii & tbit) continue;
        if ((ii & cmask) != cmask) continue;
        uint64_t j = ii | tbit;
        double xr = a[2 * ii], xi = a[2 * ii + 1];
        double yr = a[2 * j], yi = a[2 * j + 1];
        a[2 * ii]     = u[0] * xr - u[1] * xi + u[2] * yr - u[3] * yi;
        a[2 * ii + 1] = u[0] * xi + u[1] * xr + u[2] * yi + u[3] * yr;
        a[2 * j]      = u[4] * xr - u[5] * xi + u[6] * yr - u[7] * yi;
        a[2 * j + 1]  = u[4] * xi + u[5] * xr + u[6] * yi + u[7] * yr;
    }
    return 0;
}

/* SWAP(q1,q2): exchange a(i) and a(i ^ 2^q1 ^ 2^q2) for every i with
 * bit q1 = 1 and bit q2 = 0 (the two-qubit permutation used by the QFT's
 * final qubit reversal). */
int oracle_e_swap(double *a, int n, int q1, int q2)
{
    uint64_t dim = (uint64_t)1 << n;
    uint64_t b1 = (uint64_t)1 << q1, b2 = (uint64_t)1 << q2;
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < (int64_t)dim; ++i) {
        uint64_t ii = (uint64_t)i;
        if (!(ii & b1) || (ii & b2)) continue;
        uint64_t j = ii ^ b1 ^ b2;
        double tr = a[2 * ii], ti = a[2 * ii + 1];
        a[2 * ii] = a[2 * j];
        a[2 * ii + 1] = a[2 * j + 1];
        a[2 * j] = tr;
        a[2 * j + 1] = ti;
    }
    return 0;
}

/* A circuit: arrays of gate records.  kind[g] = 0: controlled 2x2 gate
 * (target[g], ctrl[2g..2g+nctrl[g]-1], u[8g..8g+7]); kind[g] = 1: SWAP of
 * target[g] and target2[g]. */
int oracle_e_run(double *a, int n, int64_t ngates, const int32_t *kind, const int32_t *target,
                 const int32_t *target2, const int32_t *nctrl, const int32_t *ctrl, const double *u)
{
    for (int64_t g = 0; g < ngates; ++g) {
        if (kind[g] == 1) {
            oracle_e_swap(a, n, target[g], target2[g]);
        } else {
            int c[2] = {ctrl[2 * g], ctrl[2 * g + 1]};
            oracle_e_apply(a, n, u + 8 * g, target[g], c, nctrl[g]);
        }
    }
    return 0;
}

/* Eq. STAT1: sum_i |a_i|^2, accumulated in long double. */
double oracle_e_norm2(const double *a, int n)
{
    uint64_t dim = (uint64_t)1 << n;
    long double s = 0.0L;
    for (uint64_t i = 0; i < dim; ++i) s += (long double)a[2 * i] * a[2 * i] + (long double)a[2 * i + 1] * a[2 * i + 1];
    return (double)s;
}

/* BEGIN MEASUREMENT (App. B):
 *   <Qx(n)> = <(1 - sigma^x_n)>/2, <Qy(n)> = <(1 - sigma^y_n)>/2,
 *   <Qz(n)> = <(1 - sigma^z_n)>/2 = P(qubit n = 1).
 * With S_n = sum_{i: bit n = 0} conj(a_i) a_{i|2^n}:
 *   <sigma^x_n> = 2 Re S_n, <sigma^y_n> = 2 Im S_n,
 *   <sigma^z_n> = sum |a(bit n = 0)|^2 - sum |a(bit n = 1)|^2.
 * Output q[3n+0..2] = <Qx(n)>, <Qy(n)>, <Qz(n)> of the normalised state
 * (divided by sum |a|^2; reading R-B7). */
void oracle_e_expectations(const double *a, int n, double *q)
{
    uint64_t dim = (uint64_t)1 << n;
    for (int k = 0; k < n; ++k) {
        uint64_t b = (uint64_t)1 << k;
        long double sr = 0.0L, si = 0.0L, p0 = 0.0L, p1 = 0.0L;
        for (uint64_t i = 0; i < dim; ++i) {
            long double m = (long double)a[2 * i] * a[2 * i] + (long double)a[2 * i + 1] * a[2 * i + 1];
            if (i & b) {
                p1 += m;
            } else {
                uint64_t j = i | b;
                long double xr = a[2 * i], xi = a[2 * i + 1], yr = a[2 * j], yi = a[2 * j + 1];
                /* conj(x) * y */
                sr += xr * yr + xi * yi;
                si += xr * yi - xi * yr;
                p0 += m;
            }
        }
        /* expectation values of the normalised state (Eq. STAT1; reading R-B7:
         * the A encoding does not preserve the norm, R-A11) */
        long double nrm = p0 + p1;
        q[3 * k + 0] = (double)((nrm - 2.0L * sr) / (2.0L * nrm));
        q[3 * k + 1] = (double)((nrm - 2.0L * si) / (2.0L * nrm));
        q[3 * k + 2] = (double)((nrm - (p0 - p1)) / (2.0L * nrm));
    }
}

/* p1[n] = sum_{bit n = 1} |a_i|^2. */
void oracle_e_probabilities(const double *a, int n, double *p1)
{
    uint64_t dim = (uint64_t)1 << n;
    for (int k = 0; k < n; ++k) {
        uint64_t b = (uint64_t)1 << k;
        long double s = 0.0L;
        for (uint64_t i = 0; i < dim; ++i)
            if (i & b) s += (long double)a[2 * i] * a[2 * i] + (long double)a[2 * i + 1] * a[2 * i + 1];
        p1[k] = (double)s;
    }
}

/* M (App. B): compute p0, p1; outcome 0 iff u < p0
 * (u uniform in [0,1), drawn by the caller); project onto the outcome and
 * rescale the kept half by 1/sqrt(p_outcome) (renormalisation: SURVEY.md
 * K10 / §8(a) a10).  p0 here is normalised by the state's norm so that the
 * draw is a probability.  Returns the outcome, or -5 if the kept half has
 * norm^2 < 1e-14 ("fails if ... amplitude zero"). */
int oracle_e_measure(double *a, int n, int qubit, double u_draw, double *p0_out)
{
    uint64_t dim = (uint64_t)1 << n;
    uint64_t b = (uint64_t)1 << qubit;
    long double s0 = 0.0L, s1 = 0.0L;
    for (uint64_t i = 0; i < dim; ++i) {
        long double m = (long double)a[2 * i] * a[2 * i] + (long double)a[2 * i + 1] * a[2 * i + 1];
        if (i & b) s1 += m; else s0 += m;
    }
    double p0 = (double)(s0 / (s0 + s1));
    if (p0_out) *p0_out = p0;
    int outcome = (u_draw < p0) ? 0 : 1;
    long double keep = outcome ? s1 : s0;
    if (keep < 1e-14L) return -5;
    double scale = (double)(1.0L / sqrtl(keep));
    for (uint64_t i = 0; i < dim; ++i) {
        int bit = (i & b) ? 1 : 0;
        if (bit != outcome) {
            a[2 * i] = 0.0;
            a[2 * i + 1] = 0.0;
        } else {
            a[2 * i] *= scale;
            a[2 * i + 1] *= scale;
        }
    }
    return outcome;
}

/* SHORBOX n_x G y (App. B; §5.4):
 * 2^{-n_x/2} sum_{x=0}^{2^{n_x}-1} |x>|y^x mod G>, the x-register on qubits
 * 0..n_x-1 and the f-register above it: a(x + 2^{n_x} f) = 2^{-n_x/2} iff
 * f = y^x mod G (sum limit: reading A21).  Replaces the state. */
void oracle_e_shorbox(double *a, int n, int nx, uint64_t G, uint64_t y)
{
    uint64_t dim = (uint64_t)1 << n;
    memset(a, 0, sizeof(double) * 2 * dim);
    double amp = pow(2.0, -0.5 * nx);
    uint64_t f = 1 % G; /* y^0 mod G */
    for (uint64_t x = 0; x < ((uint64_t)1 << nx); ++x) {
        uint64_t i = x + (f << nx);
        a[2 * i] = amp;
        f = (f * y) % G;
    }
}

/* GENERATE EVENTS (App. B): for each caller-drawn
 * u_k in [0,1), the smallest index L with sum_{L' <= L} |a_L'|^2 > u_k * total
 * (inverse CDF over the basis index order; cumulative sums in long double). */
void oracle_e_sample(const double *a, int n, const double *u, int64_t nsamp, uint64_t *out)
{
    uint64_t dim = (uint64_t)1 << n;
    long double *cum = (long double *)malloc(sizeof(long double) * dim);
    long double run = 0.0L;
    for (uint64_t i = 0; i < dim; ++i) {
        run += (long double)a[2 * i] * a[2 * i] + (long double)a[2 * i + 1] * a[2 * i + 1];
        cum[i] = run;
    }
    for (int64_t k = 0; k < nsamp; ++k) {
        long double t = (long double)u[k] * run;
        uint64_t lo = 0, hi = dim - 1; /* first i with cum[i] > t */
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo) / 2;
            if (cum[mid] > t) hi = mid; else lo = mid + 1;
        }
        out[k] = lo;
    }
    free(cum);
}

/* CLEAR / SET (App. B): the projector |v><v| on qubit n,
 * followed by renormalisation; returns -5 if the projected norm^2 < 1e-14
 * ("fails if the projection results in a state with amplitude zero"), leaving
 * the state unchanged. */
int oracle_e_project(double *a, int n, int qubit, int value)
{
    uint64_t dim = (uint64_t)1 << n;
    uint64_t b = (uint64_t)1 << qubit;
    long double keep = 0.0L;
    for (uint64_t i = 0; i < dim; ++i)
        if (((i & b) ? 1 : 0) == value) keep += (long double)a[2 * i] * a[2 * i] + (long double)a[2 * i + 1] * a[2 * i + 1];
    if (keep < 1e-14L) return -5;
    double scale = (double)(1.0L / sqrtl(keep));
    for (uint64_t i = 0; i < dim; ++i) {
        if (((i & b) ? 1 : 0) != value) {
            a[2 * i] = 0.0;
            a[2 * i + 1] = 0.0;
        } else {
            a[2 * i] *= scale;
            a[2 * i + 1] *= scale;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* A: adaptive 2-byte polar encoding, §4.1             */
/* Codes are stored interleaved: code[2i] = b0 (magnitude), code[2i+1] = b1   */
/* (angle).                                                                  */
/* ------------------------------------------------------------------------ */

#define ORACLE_EPS0 1e-12 /* reading R-A5: |z| < EPS0 is the special r = 0 */
#define ORACLE_EPS1 1e-12 /* reading R-A5: |z| > 1-EPS1 is the special r = 1 */

/* round half away from zero (reading R-A6). */
static double round_half_away(double x)
{
    return (x >= 0.0) ? floor(x + 0.5) : -floor(-x + 0.5);
}

/* theta = pi b1/128; r = 0 if b0 = -128; r = 1 if b0 = 127;
 * else r = (b0+127)(r1-r0)/253 + r0.  z = r e^{i theta}. */
void oracle_a_decode(int b0, int b1, double r0, double r1, double *zr, double *zi)
{
    double r;
    if (b0 == -128) r = 0.0;
    else if (b0 == 127) r = 1.0;
    else r = (double)(b0 + 127) * (r1 - r0) / 253.0 + r0;
    double th = ORACLE_PI * (double)b1 / 128.0;
    *zr = r * cos(th);
    *zi = r * sin(th);
}

/* 0 = special zero, 1 = special one, 2 = intermediate (readings R-A3, R-A5). */
static int a_class(double m)
{
    if (m < ORACLE_EPS0) return 0;
    if (m > 1.0 - ORACLE_EPS1) return 1;
    return 2;
}

/* Inverse of the decode map with round-half-away (readings R-A6, R-A7). */
void oracle_a_encode(double zr, double zi, double r0, double r1, int *b0_out, int *b1_out)
{
    double m = hypot(zr, zi);
    int cls = a_class(m);
    int b0, b1;
    if (cls == 0) {
        *b0_out = -128;
        *b1_out = 0;
        return;
    }
    if (cls == 1) {
        b0 = 127;
    } else if (r1 > r0) {
        double k = round_half_away((m - r0) * 253.0 / (r1 - r0)) - 127.0;
        if (k < -127.0) k = -127.0;
        if (k > 126.0) k = 126.0;
        b0 = (int)k;
    } else {
        b0 = 0; /* r0 == r1: every code in [-127,126] decodes to r0 (R-A7) */
    }
    double kb = round_half_away(128.0 * atan2(zi, zr) / ORACLE_PI);
    if (kb >= 128.0) kb = -128.0; /* theta = pi wraps to b1 = -128 */
    b1 = (int)kb;
    *b0_out = b0;
    *b1_out = b1;
}

/* Bounds (reading R-A3/R-A8): r0 = min, r1 = max of |z| over
 * the intermediate amplitudes; (0.5, 0.5) sentinel if there are none.
 * z is an interleaved complex fp64 vector of length dim. */
void oracle_a_bounds(const double *z, uint64_t dim, double *r0_out, double *r1_out)
{
    double r0 = INFINITY, r1 = -INFINITY;
    /* min / max are exact and order-independent: the reduction gives the
     * same bits for any thread count */
#pragma omp parallel for schedule(static) reduction(min : r0) reduction(max : r1)
    for (uint64_t i = 0; i < dim; ++i) {
        double m = hypot(z[2 * i], z[2 * i + 1]);
        if (a_class(m) != 2) continue;
        if (m < r0) r0 = m;
        if (m > r1) r1 = m;
    }
    if (r0 > r1) {
        r0 = 0.5;
        r1 = 0.5;
    }
    *r0_out = r0;
    *r1_out = r1;
}

/* |0...0> in A: b0 = 127, b1 = 0 at index 0; special zero elsewhere; bounds
 * start at the sentinel (reading R-A8). */
void oracle_a_init(int8_t *code, int n, double *r0, double *r1)
{
    uint64_t dim = (uint64_t)1 << n;
    for (uint64_t i = 0; i < dim; ++i) {
        code[2 * i] = -128;
        code[2 * i + 1] = 0;
    }
    code[0] = 127;
    code[1] = 0;
    *r0 = 0.5;
    *r1 = 0.5;
}

/* Decode every amplitude into an fp64 vector (step 1 of SURVEY.md §8(c) A). */
void oracle_a_decode_state(const int8_t *code, int n, double r0, double r1, double *z)
{
    uint64_t dim = (uint64_t)1 << n;
#pragma omp parallel for schedule(static)
    for (uint64_t i = 0; i < dim; ++i) oracle_a_decode(code[2 * i], code[2 * i + 1], r0, r1, &z[2 * i], &z[2 * i + 1]);
}

/* Steps 3-4: new exact bounds of z, then re-encode every amplitude. */
void oracle_a_encode_state(const double *z, int n, int8_t *code, double *r0, double *r1)
{
    uint64_t dim = (uint64_t)1 << n;
    oracle_a_bounds(z, dim, r0, r1);
#pragma omp parallel for schedule(static)
    for (uint64_t i = 0; i < dim; ++i) {
        int b0, b1;
        oracle_a_encode(z[2 * i], z[2 * i + 1], *r0, *r1, &b0, &b1);
        code[2 * i] = (int8_t)b0;
        code[2 * i + 1] = (int8_t)b1;
    }
}

/* One gate in A, reading R-A4 (exact bounds per gate): decode all, apply the
 * E rule in fp64, recompute exact bounds over the whole state, re-encode all.
 * work: caller-provided scratch of 2*2^n doubles.  No fast paths. */
int oracle_a_apply(int8_t *code, int n, double *r0, double *r1, const double *u, int t, const int *ctrl,
                   int nctrl, double *work)
{
    oracle_a_decode_state(code, n, *r0, *r1, work);
    oracle_e_apply(work, n, u, t, ctrl, nctrl);
    oracle_a_encode_state(work, n, code, r0, r1);
    return 0;
}

int oracle_a_swap(int8_t *code, int n, double *r0, double *r1, int q1, int q2, double *work)
{
    oracle_a_decode_state(code, n, *r0, *r1, work);
    oracle_e_swap(work, n, q1, q2);
    oracle_a_encode_state(work, n, code, r0, r1);
    return 0;
}

int oracle_a_run(int8_t *code, int n, double *r0, double *r1, int64_t ngates, const int32_t *kind,
                 const int32_t *target, const int32_t *target2, const int32_t *nctrl, const int32_t *ctrl,
                 const double *u, double *work)
{
    for (int64_t g = 0; g < ngates; ++g) {
        if (kind[g] == 1) {
            oracle_a_swap(code, n, r0, r1, target[g], target2[g], work);
        } else {
            int c[2] = {ctrl[2 * g], ctrl[2 * g + 1]};
            oracle_a_apply(code, n, r0, r1, u + 8 * g, target[g], c, nctrl[g], work);
        }
    }
    return 0;
}

/* ---- A with lazy ("lagged") bounds: SURVEY.md §8(f) NEXT-4, the policy
 * variant of PAPER.md:455-456 ("the values of r0 and r1 need to be updated")
 * that updates them only when the circuit leaves the current range, reading
 * R-A25 (SPEC's lazy rescale):
 *   decode all with (r0, r1); apply the gate in fp64; if every intermediate
 *   output magnitude m (reading R-A3/R-A5 classification) lies in
 *   [r0 - d, r1 + d], d = (r1 - r0)/253 the magnitude step, encode with the
 *   SAME (r0, r1) (a magnitude within one step outside the range clamps to
 *   the nearest end code); otherwise recompute r0, r1 exactly over the whole
 *   state (oracle_a_bounds) and encode with them -- the exact policy's step.
 * Returns 1 when the gate rescaled, 0 when it kept the bounds.  work: 2*2^n
 * doubles of scratch.  No fast paths. */
static int oracle_a_in_range(const double *z, uint64_t dim, double r0, double r1)
{
    const double d = (r1 - r0) / 253.0;
    int in = 1;
#pragma omp parallel for schedule(static) reduction(&& : in)
    for (uint64_t i = 0; i < dim; ++i) {
        const double m = hypot(z[2 * i], z[2 * i + 1]);
        if (a_class(m) != 2) continue;
        in = in && (m >= r0 - d) && (m <= r1 + d);
    }
    return in;
}

static void oracle_a_encode_with(const double *z, int n, int8_t *code, double r0, double r1)
{
    uint64_t dim = (uint64_t)1 << n;
#pragma omp parallel for schedule(static)
    for (uint64_t i = 0; i < dim; ++i) {
        int b0, b1;
        oracle_a_encode(z[2 * i], z[2 * i + 1], r0, r1, &b0, &b1);
        code[2 * i] = (int8_t)b0;
        code[2 * i + 1] = (int8_t)b1;
    }
}

int oracle_a_apply_lazy(int8_t *code, int n, double *r0, double *r1, const double *u, int t, const int *ctrl,
                        int nctrl, double *work)
{
    uint64_t dim = (uint64_t)1 << n;
    oracle_a_decode_state(code, n, *r0, *r1, work);
    oracle_e_apply(work, n, u, t, ctrl, nctrl);
    if (oracle_a_in_range(work, dim, *r0, *r1)) {
        oracle_a_encode_with(work, n, code, *r0, *r1);
        return 0;
    }
    oracle_a_encode_state(work, n, code, r0, r1);
    return 1;
}

/* a circuit under the lazy policy; SWAP records rescale like gates (their
 * outputs are the inputs, always in range); returns the number of rescales */
int64_t oracle_a_run_lazy(int8_t *code, int n, double *r0, double *r1, int64_t ngates, const int32_t *kind,
                          const int32_t *target, const int32_t *target2, const int32_t *nctrl, const int32_t *ctrl,
                          const double *u, double *work)
{
    int64_t rescales = 0;
    for (int64_t g = 0; g < ngates; ++g) {
        if (kind[g] == 1) {
            oracle_a_decode_state(code, n, *r0, *r1, work);
            oracle_e_swap(work, n, target[g], target2[g]);
            if (oracle_a_in_range(work, (uint64_t)1 << n, *r0, *r1)) {
                oracle_a_encode_with(work, n, code, *r0, *r1);
            } else {
                oracle_a_encode_state(work, n, code, r0, r1);
                ++rescales;
            }
        } else {
            int c[2] = {ctrl[2 * g], ctrl[2 * g + 1]};
            rescales += oracle_a_apply_lazy(code, n, r0, r1, u + 8 * g, target[g], c, nctrl[g], work);
        }
    }
    return rescales;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* thread count of the OpenMP loops (timing harness: SURVEY.md §8(d) times the
 * oracle on 1 thread and on all cores); no effect on the results */
void oracle_set_num_threads(int n)
{
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    omp_set_num_threads(n);
#else
    (void)n;
#endif
}
