// kernels_a.cu -- sm_100a kernels for the A variant: the paper's adaptive
// 2-byte polar encoding (§4.1) fused into the sweeps.
//
// Storage: one uint16 per amplitude, low byte b0 (magnitude code), high byte
// b1 (angle code): theta = pi b1 / 128; r = 0 (b0 = -128), 1 (b0 = 127), else
// (b0 + 127)(r1 - r0)/253 + r0.
//
// Dense gates follow reading R-A4 (exact bounds per gate): phase 1 decodes,
// applies the gate and reduces min/max |z'|^2 over the intermediate
// magnitudes (read-only, 2 B/amp); the host turns them into (r0, r1) (global
// over all shards); phase 2 decodes, applies and encodes with those bounds
// (4 B/amp).  Both phases use the same device functions, so the
// zero/one/intermediate classification agrees bit for bit.
//
// Decode is a table lookup (tables built on the host with the paper's
// expressions).  Encode avoids fp64 sqrt/atan2: an fp32 candidate code is
// corrected against exact fp64 boundaries (squared-magnitude thresholds and
// boundary-direction cross products), so the code equals the fp64 rounding of
// the definition except at exact ties.
//
// Permutation and phase gates never decode: anti-diagonal gates move codes and
// add round(128 arg(u)/pi) to b1, diagonal gates add it in place (PAPER.md:
// 442-444, 459-460: "very little" extra cost for X / CNOT).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.h"
#include "kernels.h"
#include "kernels_a.h"

namespace qsim {

// reading R-A5: |z| < 1e-12 is the special 0, |z| > 1 - 1e-12 the special 1 (compared squared)
#define A_ZERO2 1e-24
#define A_ONE2 ((1.0 - 1e-12) * (1.0 - 1e-12))

static int a_num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// ---------------------------------------------------------------- tables (host)
static void fill_tables(ATabData &t, double r0, double r1) {
    const double PI = 3.14159265358979323846;
    for (int i = 0; i < 256; ++i) {
        int b0 = i - 128;
        if (b0 == -128)
            t.r[i] = 0.0;
        else if (b0 == 127)
            t.r[i] = 1.0;
        else
            t.r[i] = (double)(b0 + 127) * (r1 - r0) / 253.0 + r0;
        double th = PI * (double)b0 / 128.0;  // i - 128 doubles as b1 here
        t.cth[i] = std::cos(th);
        t.sth[i] = std::sin(th);
    }
    for (int c = 0; c < 256; ++c) {
        double m = r0 + ((double)c + 0.5) * (r1 - r0) / 253.0;
        t.thr[c] = (c < 253) ? m * m : INFINITY;
    }
    for (int k = -129; k <= 130; ++k) {
        double beta = ((double)k + 0.5) * PI / 128.0;
        t.cb[k + 129] = std::cos(beta);
        t.sb[k + 129] = std::sin(beta);
    }
    t.r0 = r0;
    t.r1 = r1;
    t.degenerate = !(r1 > r0);
    t.scale = t.degenerate ? 0.0 : 253.0 / (r1 - r0);
}

int atables_alloc(ATables **out) {
    auto *t = new ATables();
    if (cudaMalloc(&t->d[0], sizeof(ATabData)) != cudaSuccess || cudaMalloc(&t->d[1], sizeof(ATabData)) != cudaSuccess ||
        cudaMallocHost(&t->h, sizeof(ATabData)) != cudaSuccess) {
        cudaGetLastError();
        atables_free(t);
        set_error("A tables allocation failed");
        return QSIM_ENOMEM;
    }
    *out = t;
    return QSIM_OK;
}

void atables_free(ATables *t) {
    if (!t) return;
    if (t->d[0]) cudaFree(t->d[0]);
    if (t->d[1]) cudaFree(t->d[1]);
    if (t->h) cudaFreeHost(t->h);
    delete t;
}

static int upload(ATables *t, int which, double r0, double r1, cudaStream_t s) {
    if (cudaStreamSynchronize(s) != cudaSuccess) return QSIM_ECUDA;  // h is reused
    fill_tables(*t->h, r0, r1);
    if (cudaMemcpyAsync(t->d[which], t->h, sizeof(ATabData), cudaMemcpyHostToDevice, s) != cudaSuccess) {
        set_error("A tables upload failed");
        return QSIM_ECUDA;
    }
    if (cudaStreamSynchronize(s) != cudaSuccess) return QSIM_ECUDA;
    return QSIM_OK;
}

int atables_set(ATables *t, double r0, double r1, cudaStream_t s) {
    int rc = upload(t, t->cur, r0, r1, s);
    if (rc) return rc;
    return upload(t, 1 - t->cur, r0, r1, s);
}
int atables_set_next(ATables *t, double r0, double r1, cudaStream_t s) { return upload(t, 1 - t->cur, r0, r1, s); }
int atables_commit_next(ATables *t, cudaStream_t s) {
    (void)s;
    t->cur = 1 - t->cur;
    return QSIM_OK;
}
static const ATabData *tcur(const ATables *t) { return t->d[t->cur]; }
static const ATabData *tnext(const ATables *t) { return t->d[1 - t->cur]; }

// ---------------------------------------------------------------- device side
struct ASm {
    double r[256];    // decode (current bounds)
    double thr[256];  // encode thresholds (next bounds)
    double2 cs[256];  // (cos, sin)(pi b1 / 128), one 128-bit load per decode
    double cb[260], sb[260];
    double r0n, scalen;
    int degn;
    float mmargin;  // magnitude-candidate margin (steps) below which the fp64 check is skipped
    float scalef, r0s;  // fp32 253/(r1-r0) and r0 * that (next bounds), for the candidate
};

__device__ void load_asm(ASm &sm, const ATabData *__restrict__ cur, const ATabData *__restrict__ nxt) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        sm.r[i] = cur->r[i];
        sm.thr[i] = nxt->thr[i];
        sm.cs[i] = make_double2(cur->cth[i], cur->sth[i]);
    }
    for (int i = threadIdx.x; i < 260; i += blockDim.x) {
        sm.cb[i] = cur->cb[i];
        sm.sb[i] = cur->sb[i];
    }
    if (threadIdx.x == 0) {
        sm.r0n = nxt->r0;
        sm.scalen = nxt->scale;
        sm.degn = nxt->degenerate;
        // fp32 candidate error in steps: |d tf| <= (eps32 (|m| + r0) + |m - m_f|) * scale,
        // bounded by 4e-7 * (r1 + r0) * scale + 1e-3; above 0.5 -> always check
        const double e = 6e-7 * (nxt->r1 + nxt->r0) * nxt->scale + 1e-4;
        sm.mmargin = (float)(e < 0.49 ? e : 0.5);
        sm.scalef = (float)nxt->scale;
        sm.r0s = (float)(nxt->r0 * nxt->scale);
    }
    __syncthreads();
}

__device__ __forceinline__ double2 a_decode(const ASm &sm, uint32_t code) {
    const int b0i = (int)(code & 0xffu) ^ 0x80;  // int8 b0 + 128
    const int b1i = (int)((code >> 8) & 0xffu) ^ 0x80;
    const double r = sm.r[b0i];
    const double2 cs = sm.cs[b1i];
    return make_double2(r * cs.x, r * cs.y);
}

__device__ __forceinline__ double a_m2(double2 z) { return fma(z.x, z.x, z.y * z.y); }

__device__ __forceinline__ uint32_t pack(int b0, int b1) { return (uint32_t)(b0 & 0xff) | ((uint32_t)(b1 & 0xff) << 8); }

// fp32 atan2 candidate in units of the b1 step (128/pi per radian): octant
// reduction + the odd minimax polynomial of Abramowitz & Stegun 4.4.49
// (|error| <= 1e-5 rad = 4e-4 steps).
__device__ __forceinline__ float atan2_steps(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    const float t = __fdividef(mn, mx);
    const float s = t * t;
    float p = fmaf(fmaf(fmaf(fmaf(0.0208351f, s, -0.0851330f), s, 0.1801410f), s, -0.3302995f), s, 0.9998660f) * t;
    if (ay > ax) p = 1.57079632679f - p;
    if (x < 0.f) p = 3.14159265359f - p;
    if (y < 0.f) p = -p;
    return p * 40.74366543152521f;  // 128 / pi
}

// Angle code: round half away from zero of 128 atan2(y, x) / pi, computed in
// fp64 terms.  The fp32 candidate is exact unless it lies within A_MARGIN
// steps of a rounding boundary; only then the exact fp64 boundary-direction
// cross products decide (ties away from zero, reading R-A6).  Candidate error:
// polynomial <= 4e-4 steps + fp32 rounding ~3e-6 steps, so 1e-3 is safe; a
// small margin keeps the (divergent) fp64 path rare per warp.
#define A_MARGIN 1e-3f
__device__ __forceinline__ int a_angle_code(const ASm &sm, double2 z) {
    const float af = atan2_steps((float)z.y, (float)z.x);
    int k = __float2int_rn(af);
    const float fr = af - (float)k;
    k = max(-128, min(128, k));
    if (fabsf(fr) > 0.5f - A_MARGIN) {
        // upper boundary of code k: beta = (k + 0.5) pi / 128 (index k + 129)
        double cu = z.y * sm.cb[k + 129] - z.x * sm.sb[k + 129];
        if ((k >= 0) ? (cu >= 0.0) : (cu > 0.0)) {
            k += 1;
        } else {
            double cl = z.y * sm.cb[k + 128] - z.x * sm.sb[k + 128];  // beta = (k - 0.5) pi / 128
            if ((k > 0) ? (cl < 0.0) : (cl <= 0.0)) k -= 1;
        }
        k = max(-128, min(128, k));
    }
    return (k == 128) ? -128 : k;
}

// Encode with the NEXT bounds (PAPER.md:449-453 inverted; readings R-A3, R-A5..R-A7).
// Magnitude: fp32 candidate, exact fp64 squared-threshold check only near a
// rounding boundary (sm.mmargin steps, derived from the fp32 error bound).
__device__ __forceinline__ uint32_t a_encode(const ASm &sm, double2 z) {
    const double m2 = a_m2(z);
    if (m2 < A_ZERO2) return pack(-128, 0);
    int b0;
    if (m2 > A_ONE2) {
        b0 = 127;
    } else if (sm.degn) {
        b0 = 0;
    } else {
        const float mf = sqrtf((float)m2);
        const float tf = (mf - (float)sm.r0n) * (float)sm.scalen;
        int c = __float2int_rn(tf);
        const float fr = tf - (float)c;
        c = max(0, min(253, c));
        if (fabsf(fr) > 0.5f - sm.mmargin) {
            if (c < 253 && m2 >= sm.thr[c])
                c += 1;
            else if (c > 0 && m2 < sm.thr[c - 1])
                c -= 1;
        }
        b0 = c - 127;
    }
    return pack(b0, a_angle_code(sm, z));
}

__device__ __forceinline__ void a_gate(const double *u, int cls, double2 &x, double2 &y) {
    if (cls == CLS_DENSE) {
        double2 nx, ny;
        nx.x = fma(u[0], x.x, fma(-u[1], x.y, fma(u[2], y.x, -u[3] * y.y)));
        nx.y = fma(u[0], x.y, fma(u[1], x.x, fma(u[2], y.y, u[3] * y.x)));
        ny.x = fma(u[4], x.x, fma(-u[5], x.y, fma(u[6], y.x, -u[7] * y.y)));
        ny.y = fma(u[4], x.y, fma(u[5], x.x, fma(u[6], y.y, u[7] * y.x)));
        x = nx;
        y = ny;
    }
}

__device__ __forceinline__ uint64_t a_ins0(uint64_t w, int p) {
    return ((w >> p) << (p + 1)) | (w & ((1ull << p) - 1ull));
}

__device__ __forceinline__ bool is_inter(double m2) { return m2 >= A_ZERO2 && m2 <= A_ONE2; }

// A unit = 16 codes = 8 pairs.  LOWT (t < 4): 16 contiguous codes, pairs
// (k, k | 2^t); else: 8 contiguous codes at the i0 run and 8 at the i1 run.
template <bool LOWT>
__device__ __forceinline__ void unit_load(const uint16_t *__restrict__ a, uint64_t u, int t, uint32_t (&c)[16],
                                          uint64_t &s0) {
    uint4 v0, v1;
    if (LOWT) {
        s0 = u << 4;
        v0 = *reinterpret_cast<const uint4 *>(a + s0);
        v1 = *reinterpret_cast<const uint4 *>(a + s0 + 8);
    } else {
        s0 = a_ins0(u << 3, t);
        v0 = *reinterpret_cast<const uint4 *>(a + s0);
        v1 = *reinterpret_cast<const uint4 *>(a + (s0 | (1ull << t)));
    }
    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        c[2 * k] = w[k] & 0xffffu;
        c[2 * k + 1] = w[k] >> 16;
    }
}
template <bool LOWT>
__device__ __forceinline__ void unit_store(uint16_t *__restrict__ a, uint64_t s0, int t, const uint32_t (&c)[16]) {
    uint4 v0, v1;
    v0.x = c[0] | (c[1] << 16);
    v0.y = c[2] | (c[3] << 16);
    v0.z = c[4] | (c[5] << 16);
    v0.w = c[6] | (c[7] << 16);
    v1.x = c[8] | (c[9] << 16);
    v1.y = c[10] | (c[11] << 16);
    v1.z = c[12] | (c[13] << 16);
    v1.w = c[14] | (c[15] << 16);
    if (LOWT) {
        *reinterpret_cast<uint4 *>(a + s0) = v0;
        *reinterpret_cast<uint4 *>(a + s0 + 8) = v1;
    } else {
        *reinterpret_cast<uint4 *>(a + s0) = v0;
        *reinterpret_cast<uint4 *>(a + (s0 | (1ull << t))) = v1;
    }
}
// pair k of a unit: slots (j0, j1) and the local index of j0
template <bool LOWT>
__device__ __forceinline__ void pair_slots(int k, int t, uint64_t s0, int &j0, int &j1, uint64_t &i0) {
    if (LOWT) {
        // k-th index in 0..15 with bit t clear
        int lo = k & ((1 << t) - 1);
        j0 = ((k >> t) << (t + 1)) | lo;
        j1 = j0 | (1 << t);
        i0 = s0 + (uint64_t)j0;
    } else {
        j0 = k;
        j1 = k + 8;
        i0 = s0 + (uint64_t)k;
    }
}

constexpr int A_THREADS = 256;

static int a_grid(uint64_t units) {
    uint64_t cap = (uint64_t)a_num_sms() * 8;
    uint64_t need = (units + A_THREADS - 1) / A_THREADS;
    return (int)(need < cap ? (need ? need : 1) : cap);
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum_a(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------- dense gates
// A unit = 16 codes = 8 pairs, one per thread per iteration.  TL = 0..3: the
// target is bit TL of 16 contiguous codes (pairs (j, j | 2^TL)); TL = 4: the
// target t >= 4 is a runtime bit, the unit is 8 contiguous codes at s0 and 8
// at s0 | 2^t (pairs (k, k + 8)).  All register indexing is compile-time.
// Controls: a pair is selected iff its full index has every cmask bit; the
// unit's low bits (0..3, resp. 0..2) are the only ones that differ inside a
// unit, so the test is (hi part of the unit) && ((slot & cl) == cl).
template <int TL>
struct AUnit {
    static constexpr int LOWB = TL < 4 ? 4 : 3;
    __device__ static __forceinline__ int j0(int k) { return TL < 4 ? (((k >> TL) << (TL + 1)) | (k & ((1 << TL) - 1))) : k; }
    __device__ static __forceinline__ int j1(int k) { return TL < 4 ? (j0(k) | (1 << TL)) : k + 8; }
    __device__ static __forceinline__ uint64_t s0(uint64_t u, int t) { return TL < 4 ? (u << 4) : a_ins0(u << 3, t); }
    __device__ static __forceinline__ void load(const uint16_t *__restrict__ a, uint64_t s0, int t, uint32_t (&c)[16]) {
        const uint4 v0 = __ldcs(reinterpret_cast<const uint4 *>(a + s0));
        const uint4 v1 = __ldcs(reinterpret_cast<const uint4 *>(a + (TL < 4 ? s0 + 8 : (s0 | (1ull << t)))));
        const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            c[2 * k] = w[k] & 0xffffu;
            c[2 * k + 1] = w[k] >> 16;
        }
    }
    __device__ static __forceinline__ void store(uint16_t *__restrict__ a, uint64_t s0, int t, const uint32_t (&c)[16]) {
        uint4 v0, v1;
        v0.x = c[0] | (c[1] << 16);
        v0.y = c[2] | (c[3] << 16);
        v0.z = c[4] | (c[5] << 16);
        v0.w = c[6] | (c[7] << 16);
        v1.x = c[8] | (c[9] << 16);
        v1.y = c[10] | (c[11] << 16);
        v1.z = c[12] | (c[13] << 16);
        v1.w = c[14] | (c[15] << 16);
        __stcs(reinterpret_cast<uint4 *>(a + s0), v0);
        __stcs(reinterpret_cast<uint4 *>(a + (TL < 4 ? s0 + 8 : (s0 | (1ull << t)))), v1);
    }
};

// Matrix classes of a dense U for the A kernels (host: a_ukind): 0 general,
// 1 every entry real (H, Ry), 2 real diagonal and imaginary off-diagonal (Rx).
// The class formulas are the general one with its exactly-zero terms dropped
// (fma(0, b, c) = c, fma(a, b, +-0) = a b rounded once), so the fp64 results
// are the same bits.
template <int UK>
__device__ __forceinline__ void a_gate2k(const double (&u)[8], double2 &x, double2 &y) {
    const double2 x0 = x, y0 = y;
    if (UK == 1) {
        x.x = fma(u[0], x0.x, u[2] * y0.x);
        x.y = fma(u[0], x0.y, u[2] * y0.y);
        y.x = fma(u[4], x0.x, u[6] * y0.x);
        y.y = fma(u[4], x0.y, u[6] * y0.y);
    } else {
        x.x = fma(u[0], x0.x, -(u[3] * y0.y));
        x.y = fma(u[0], x0.y, u[3] * y0.x);
        y.x = fma(-u[5], x0.y, u[6] * y0.x);
        y.y = fma(u[5], x0.x, u[6] * y0.y);
    }
}
template <int UK>
__device__ __forceinline__ void a_gate_fk(const float (&u)[8], float2 &x, float2 &y) {
    const float2 x0 = x, y0 = y;
    if (UK == 1) {
        x.x = fmaf(u[0], x0.x, u[2] * y0.x);
        x.y = fmaf(u[0], x0.y, u[2] * y0.y);
        y.x = fmaf(u[4], x0.x, u[6] * y0.x);
        y.y = fmaf(u[4], x0.y, u[6] * y0.y);
    } else {
        x.x = fmaf(u[0], x0.x, -(u[3] * y0.y));
        x.y = fmaf(u[0], x0.y, u[3] * y0.x);
        y.x = fmaf(-u[5], x0.y, u[6] * y0.x);
        y.y = fmaf(u[5], x0.x, u[6] * y0.y);
    }
}

__device__ __forceinline__ void a_gate2(const double (&u)[8], double2 &x, double2 &y) {
    const double2 x0 = x, y0 = y;
    x.x = fma(u[0], x0.x, fma(-u[1], x0.y, fma(u[2], y0.x, -u[3] * y0.y)));
    x.y = fma(u[0], x0.y, fma(u[1], x0.x, fma(u[2], y0.y, u[3] * y0.x)));
    y.x = fma(u[4], x0.x, fma(-u[5], x0.y, fma(u[6], y0.x, -u[7] * y0.y)));
    y.y = fma(u[4], x0.y, fma(u[5], x0.x, fma(u[6], y0.y, u[7] * y0.x)));
}

// hi words of A_ZERO2 = 1e-24 and A_ONE2 = (1 - 1e-12)^2: an m2 >= A_ZERO2 has
// hi(m2) >= A_ZHI, an m2 <= A_ONE2 has hi(m2) <= A_OHI (m2 >= 0: hi words order
// like the values); the fast paths below only ever widen to the exact tests.
#define A_ZHI 0x3af357c2u
#define A_OHI 0x3fefffffu

// Running exact min / max of the intermediate m2 = |z|^2 (reading R-A4/R-A5)
// with a hi-word pre-filter: a value can change mn (mx) only if its hi word is
// <= hi(mn) (>= hi(mx)) and it can be intermediate; only those take the exact
// fp64 path.
struct ABnd {
    double mn, mx;
    uint32_t mnh, mxh;
    __device__ __forceinline__ void init() {
        mn = INFINITY;
        mx = -INFINITY;
        mnh = 0x7ff00000u;
        mxh = 0u;
    }
    __device__ __forceinline__ void add(double m2) {
        const uint32_t h = (uint32_t)__double2hiint(m2);
        const bool cand = ((h <= mnh) & (h >= A_ZHI)) | ((h >= mxh) & (h <= A_OHI));
        if (cand) {
            if (m2 >= A_ZERO2 && m2 <= A_ONE2) {
                if (m2 < mn) {
                    mn = m2;
                    mnh = h;
                }
                if (m2 > mx) {
                    mx = m2;
                    mxh = h;
                }
            }
        }
    }
};


// ---- fp32 fast path with a certified fallback ------------------------------
// The dense A gate decides codes and bounds from fp32 copies of the decode
// tables, of U and of the gate arithmetic, together with a rigorous bound on
// how far each fp32 output can be from the fp64 reference (a_decode, a_gate2,
// a_m2 -- the functions the fallback and the oracle's definition use).  A code
// (or a bounds candidate) is committed from fp32 only when that bound proves
// the fp64 reference decides the same way; otherwise the pair is recomputed in
// fp64 exactly as before.  So the result is the fp64 reference's, bit for bit,
// while most pairs cost fp32 (FMA pipe) instead of fp64 + conversions.
//
// Error bound (u = 2^-24): the fp32 decode has |zf - z| <= 3u r per component
// (table value r, cos / sin and the product each rounded once); one output
// component is 4 products summed by an fma chain, with |Re u_ij| + |Im u_ij|
// <= sqrt2: sum_j sqrt2 (3u + u) r_j for the inputs and coefficients plus 4
// roundings of partial sums <= 4u sqrt2 (r0 + r1) -- in all <= 11.4u (r0 + r1)
// = 6.8e-7 (r0 + r1).  A_KF = 1e-6 > that, so per output component
// |xf - x| <= E = A_KF (r0 + r1) with r the pair's decoded magnitudes.
#define A_KF 1e-6f
struct ASmF {
    float rf[256];
    float2 csf[256];
    float scalef, r0s, r0f;
};
__device__ __forceinline__ void load_asmf(ASmF &f, const ASm &sm) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        f.rf[i] = (float)sm.r[i];
        f.csf[i] = make_float2((float)sm.cs[i].x, (float)sm.cs[i].y);
    }
    if (threadIdx.x == 0) {
        f.scalef = (float)sm.scalen;
        f.r0s = (float)(sm.r0n * sm.scalen);
        f.r0f = (float)sm.r0n;
    }
    __syncthreads();
}
__device__ __forceinline__ float2 a_decode_f(const ASmF &f, uint32_t code, float &r) {
    r = f.rf[(code & 0xffu) ^ 0x80u];
    const float2 cs = f.csf[((code >> 8) & 0xffu) ^ 0x80u];
    return make_float2(r * cs.x, r * cs.y);
}
__device__ __forceinline__ void a_gate_f(const float (&u)[8], float2 &x, float2 &y) {
    const float2 x0 = x, y0 = y;
    x.x = fmaf(u[0], x0.x, fmaf(-u[1], x0.y, fmaf(u[2], y0.x, -u[3] * y0.y)));
    x.y = fmaf(u[0], x0.y, fmaf(u[1], x0.x, fmaf(u[2], y0.y, u[3] * y0.x)));
    y.x = fmaf(u[4], x0.x, fmaf(-u[5], x0.y, fmaf(u[6], y0.x, -u[7] * y0.y)));
    y.y = fmaf(u[4], x0.y, fmaf(u[5], x0.x, fmaf(u[6], y0.y, u[7] * y0.x)));
}
template <int UK>
__device__ __forceinline__ void a_gate2u(const double (&u)[8], double2 &x, double2 &y) {
    if (UK == 0)
        a_gate2(u, x, y);
    else
        a_gate2k<UK>(u, x, y);
}
template <int UK>
__device__ __forceinline__ void a_gate_fu(const float (&u)[8], float2 &x, float2 &y) {
    if (UK == 0)
        a_gate_f(u, x, y);
    else
        a_gate_fk<UK>(u, x, y);
}

// nearest integer of t (|t| < 2^22) without the conversion unit: k and t - k
__device__ __forceinline__ int a_rnd(float t, float &fr) {
    const float m = t + 12582912.0f;  // 1.5 * 2^23
    fr = t - (m - 12582912.0f);
    return __float_as_int(m) - 0x4B400000;
}
// The code of one fp32 output x (component error bound E); ok = false when
// the fp32 value cannot decide it.  Branch-free.
__device__ __forceinline__ uint32_t a_encode_f(const ASm &sm, const ASmF &f, float2 x, float E, bool &ok) {
    const float m2f = fmaf(x.x, x.x, x.y * x.y);
    const float rs = rsqrtf(m2f);
    const float mf = m2f > 0.f ? m2f * rs : 0.f;
    const float Em = fmaf(1.4143f, E, 4e-7f * mf);  // | |z| - mf |
    const bool zero = mf + Em < 0.99999e-12f;    // certainly the special zero (reading R-A5)
    // certainly intermediate, and the direction known to within 1 %
    const bool inter = (mf - Em > 1.00001e-12f) & (mf + Em < 0.999999f) & (Em < 0.01f * mf);
    float fr;
    const float tf = fminf(fmaxf(fmaf(mf, f.scalef, -f.r0s), -2.f), 256.f);
    const int c = a_rnd(tf, fr);
    const float errm = fmaf(Em + 1.2e-7f * (mf + f.r0f), f.scalef, 2e-5f);
    const bool okm = sm.degn || (fabsf(fr) < 0.5f - errm);
    const int b0 = sm.degn ? 0 : max(0, min(253, c)) - 127;
    float fa;
    int k = a_rnd(atan2_steps(x.y, x.x), fa);
    // direction error <= sqrt(2) E / |z| (|z| >= 0.99 mf) rad, polynomial 1e-5 rad + fp32 rounding
    const float erra = fmaf(1.4143f * 1.0102f * 40.7437f, E * rs, 6e-4f);
    const bool oka = fabsf(fa) < 0.5f - erra;
    k = max(-128, min(128, k));
    ok = zero | (inter & okm & oka);
    return zero ? pack(-128, 0) : pack(b0, k == 128 ? -128 : k);
}

// fp64 reference for the pairs of a unit whose fp32 decision failed (rare;
// out of line so the hot loop stays small), then the unit's store.  Only
// scalars cross the call (the fp32 codes packed two per word, the gate from
// the kernel parameters; the input codes are reloaded -- this thread has not
// stored the unit yet), so the hot loop keeps its arrays in registers.
template <int TL, int UK>
__device__ __noinline__ void a_unit_exact_store(const ASm &sm, const double *u, uint16_t *a, uint64_t s0, int t,
                                                uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t w4,
                                                uint32_t w5, uint32_t w6, uint32_t w7, uint32_t fail, uint32_t selm) {
    double uu[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) uu[i] = u[i];
    const uint32_t w[8] = {w0, w1, w2, w3, w4, w5, w6, w7};
    uint32_t c[16], nc[16];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        nc[2 * k] = w[k] & 0xffffu;
        nc[2 * k + 1] = w[k] >> 16;
    }
    AUnit<TL>::load(a, s0, t, c);
    for (int k = 0; k < 8; ++k) {
        if (!((fail >> k) & 1u)) continue;
        const int j0 = AUnit<TL>::j0(k), j1 = AUnit<TL>::j1(k);
        double2 x = a_decode(sm, c[j0]), y = a_decode(sm, c[j1]);
        if ((selm >> k) & 1u) a_gate2u<UK>(uu, x, y);
        nc[j0] = a_encode(sm, x);
        nc[j1] = a_encode(sm, y);
    }
    AUnit<TL>::store(a, s0, t, nc);
}

template <int TL, bool CTRL, int UK>
__global__ void __launch_bounds__(A_THREADS) k_bounds_a(const __grid_constant__ AGateParams p,
                                                        const ATabData *__restrict__ cur,
                                                        const ATabData *__restrict__ nxt, double *partials) {
    using U = AUnit<TL>;
    __shared__ ASm sm;
    load_asm(sm, cur, nxt);
    const uint16_t *a = reinterpret_cast<const uint16_t *>(p.a);
    const uint64_t units = (p.nl >= 4) ? (1ull << (p.nl - 4)) : 1ull;
    const uint64_t lowm = (1ull << U::LOWB) - 1ull;
    const uint64_t chi = p.cmask & ~lowm;
    const uint32_t cl = (uint32_t)(p.cmask & lowm);
    double u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) u[i] = p.u[i];
    ABnd b;
    b.init();
    for (uint64_t v = (uint64_t)blockIdx.x * A_THREADS + threadIdx.x; v < units; v += (uint64_t)gridDim.x * A_THREADS) {
        uint32_t c[16];
        const uint64_t s0 = U::s0(v, p.t);
        U::load(a, s0, p.t, c);
        const bool hi_ok = !CTRL || (((p.shard_base | s0) & chi) == chi);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int j0 = U::j0(k), j1 = U::j1(k);
            double2 x = a_decode(sm, c[j0]), y = a_decode(sm, c[j1]);
            const int off = TL < 4 ? j0 : k;
            if (!CTRL || (hi_ok && ((uint32_t)off & cl) == cl)) a_gate2u<UK>(u, x, y);
            b.add(a_m2(x));
            b.add(a_m2(y));
        }
    }
    __shared__ double red[2][A_THREADS / 32];
    const double mn = warp_min(b.mn), mx = warp_max(b.mx);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = mn;
        red[1][threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a0 = INFINITY, a1 = -INFINITY;
        for (int w = 0; w < A_THREADS / 32; ++w) {
            a0 = fmin(a0, red[0][w]);
            a1 = fmax(a1, red[1][w]);
        }
        partials[2 * blockIdx.x] = a0;
        partials[2 * blockIdx.x + 1] = a1;
    }
}

// merge the per-block partials into acc = (min m2, -max m2) (first shard:
// overwrite), the form one ncclAllReduce(ncclMin) combines across ranks
__global__ void k_minmax_final(const double *partials, int nb, double *acc, int first) {
    __shared__ double r0[32], r1[32];
    double a0 = INFINITY, a1 = -INFINITY;
    for (int i = threadIdx.x; i < nb; i += 32) {
        a0 = fmin(a0, partials[2 * i]);
        a1 = fmax(a1, partials[2 * i + 1]);
    }
    r0[threadIdx.x] = a0;
    r1[threadIdx.x] = a1;
    __syncwarp();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 32; ++w) {
            a0 = fmin(a0, r0[w]);
            a1 = fmax(a1, r1[w]);
        }
        if (first) {
            acc[0] = a0;
            acc[1] = -a1;
        } else {
            acc[0] = fmin(acc[0], a0);
            acc[1] = fmin(acc[1], -a1);
        }
    }
}

// next tables from acc = (min m2, -max m2): r0 = sqrt(min), r1 = sqrt(max), or
// the sentinel 0.5 when no magnitude is intermediate (reading R-A8).  The same
// expressions as fill_tables on the host, with explicit IEEE roundings (no
// FMA contraction), so device- and host-built tables are bit-identical.
__global__ void k_tables_next(const double *acc, ATabData *t) {
    const double mn = acc[0], mx = -acc[1];
    const bool none = !(mn <= mx);
    const double r0 = none ? 0.5 : __dsqrt_rn(mn), r1 = none ? 0.5 : __dsqrt_rn(mx);
    const double d = __dsub_rn(r1, r0);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        const int b0 = i - 128;
        t->r[i] = b0 == -128 ? 0.0 : b0 == 127 ? 1.0 : __dadd_rn(__ddiv_rn(__dmul_rn((double)(b0 + 127), d), 253.0), r0);
        if (i < 253) {
            const double m = __dadd_rn(r0, __ddiv_rn(__dmul_rn((double)i + 0.5, d), 253.0));
            t->thr[i] = __dmul_rn(m, m);
        } else {
            t->thr[i] = INFINITY;
        }
    }
    if (threadIdx.x == 0) {
        t->r0 = r0;
        t->r1 = r1;
        t->degenerate = !(r1 > r0);
        t->scale = !(r1 > r0) ? 0.0 : __ddiv_rn(253.0, d);
    }
}

template <int TL, bool CTRL, int UK>
static void launch_bounds_tl(const AGateParams &p, const ATables *t, double *partials, int grid, cudaStream_t s) {
    k_bounds_a<TL, CTRL, UK><<<grid, A_THREADS, 0, s>>>(p, tcur(t), tnext(t), partials);
}
template <int TL, int UK>
static void launch_bounds_c(const AGateParams &p, const ATables *t, double *partials, int grid, cudaStream_t s) {
    if (p.cmask)
        launch_bounds_tl<TL, true, UK>(p, t, partials, grid, s);
    else
        launch_bounds_tl<TL, false, UK>(p, t, partials, grid, s);
}
template <int UK>
static void launch_bounds_k(const AGateParams &p, const ATables *t, double *partials, int grid, cudaStream_t s) {
    switch (p.t < 4 ? p.t : 4) {
        case 0: launch_bounds_c<0, UK>(p, t, partials, grid, s); break;
        case 1: launch_bounds_c<1, UK>(p, t, partials, grid, s); break;
        case 2: launch_bounds_c<2, UK>(p, t, partials, grid, s); break;
        case 3: launch_bounds_c<3, UK>(p, t, partials, grid, s); break;
        default: launch_bounds_c<4, UK>(p, t, partials, grid, s); break;
    }
}
// matrix class of U (see a_gate2k)
static int a_ukind(const double *u) {
    if (u[1] == 0.0 && u[3] == 0.0 && u[5] == 0.0 && u[7] == 0.0) return 1;
    if (u[1] == 0.0 && u[7] == 0.0 && u[2] == 0.0 && u[4] == 0.0) return 2;
    return 0;
}

void launch_bounds_a(const AGateParams &p, const ATables *t, double *partials, double *acc, bool first,
                     cudaStream_t s) {
    const uint64_t units = (p.nl >= 4) ? (1ull << (p.nl - 4)) : 1ull;
    int grid = a_grid(units);
    if (grid > 2 * a_num_sms() * 4) grid = 2 * a_num_sms() * 4;  // partials capacity
    switch (a_ukind(p.u)) {
        case 1: launch_bounds_k<1>(p, t, partials, grid, s); break;
        case 2: launch_bounds_k<2>(p, t, partials, grid, s); break;
        default: launch_bounds_k<0>(p, t, partials, grid, s); break;
    }
    k_minmax_final<<<1, 32, 0, s>>>(partials, grid, acc, first ? 1 : 0);
}

void launch_tables_next(const double *acc, ATables *t, cudaStream_t s) {
    k_tables_next<<<1, 256, 0, s>>>(acc, t->d[1 - t->cur]);
}

template <int TL, bool CTRL, int UK>
__global__ void __launch_bounds__(A_THREADS) k_apply_a(const __grid_constant__ AGateParams p,
                                                       const ATabData *__restrict__ cur,
                                                       const ATabData *__restrict__ nxt) {
    using U = AUnit<TL>;
    __shared__ ASm sm;
    load_asm(sm, cur, nxt);
    uint16_t *a = reinterpret_cast<uint16_t *>(p.a);
    const uint64_t units = (p.nl >= 4) ? (1ull << (p.nl - 4)) : 1ull;
    const uint64_t lowm = (1ull << U::LOWB) - 1ull;
    const uint64_t chi = p.cmask & ~lowm;
    const uint32_t cl = (uint32_t)(p.cmask & lowm);
    __shared__ ASmF f;
    load_asmf(f, sm);
    float uf[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) uf[i] = (float)p.u[i];
    for (uint64_t v = (uint64_t)blockIdx.x * A_THREADS + threadIdx.x; v < units; v += (uint64_t)gridDim.x * A_THREADS) {
        uint32_t c[16];
        const uint64_t s0 = U::s0(v, p.t);
        U::load(a, s0, p.t, c);
        const bool hi_ok = !CTRL || (((p.shard_base | s0) & chi) == chi);
        uint32_t nc[16], fail = 0, selm = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int j0 = U::j0(k), j1 = U::j1(k);
            const int off = TL < 4 ? j0 : k;
            const bool sel = !CTRL || (hi_ok && ((uint32_t)off & cl) == cl);
            selm |= (uint32_t)sel << k;
            float ra, rb;
            float2 xf = a_decode_f(f, c[j0], ra), yf = a_decode_f(f, c[j1], rb);
            if (sel) a_gate_fu<UK>(uf, xf, yf);
            const float E = A_KF * (ra + rb);
            bool okx, oky;
            nc[j0] = a_encode_f(sm, f, xf, E, okx);
            nc[j1] = a_encode_f(sm, f, yf, E, oky);
            fail |= (uint32_t)!(okx && oky) << k;
        }
        if (fail)
            a_unit_exact_store<TL, UK>(sm, p.u, a, s0, p.t, nc[0] | (nc[1] << 16), nc[2] | (nc[3] << 16),
                                       nc[4] | (nc[5] << 16), nc[6] | (nc[7] << 16), nc[8] | (nc[9] << 16),
                                       nc[10] | (nc[11] << 16), nc[12] | (nc[13] << 16), nc[14] | (nc[15] << 16),
                                       fail, selm);
        else
            U::store(a, s0, p.t, nc);
    }
}

template <int TL, int UK>
static void launch_apply_c(const AGateParams &p, const ATables *t, int grid, cudaStream_t s) {
    if (p.cmask)
        k_apply_a<TL, true, UK><<<grid, A_THREADS, 0, s>>>(p, tcur(t), tnext(t));
    else
        k_apply_a<TL, false, UK><<<grid, A_THREADS, 0, s>>>(p, tcur(t), tnext(t));
}
template <int UK>
static void launch_apply_k(const AGateParams &p, const ATables *t, int grid, cudaStream_t s) {
    switch (p.t < 4 ? p.t : 4) {
        case 0: launch_apply_c<0, UK>(p, t, grid, s); break;
        case 1: launch_apply_c<1, UK>(p, t, grid, s); break;
        case 2: launch_apply_c<2, UK>(p, t, grid, s); break;
        case 3: launch_apply_c<3, UK>(p, t, grid, s); break;
        default: launch_apply_c<4, UK>(p, t, grid, s); break;
    }
}

void launch_apply_a(const AGateParams &p, const ATables *t, cudaStream_t s) {
    const uint64_t units = (p.nl >= 4) ? (1ull << (p.nl - 4)) : 1ull;
    const int grid = a_grid(units);
    switch (a_ukind(p.u)) {
        case 1: launch_apply_k<1>(p, t, grid, s); break;
        case 2: launch_apply_k<2>(p, t, grid, s); break;
        default: launch_apply_k<0>(p, t, grid, s); break;
    }
}

// ---------------------------------------------------------------- fast paths
static int phase_steps(double ur, double ui) {
    // round half away from zero of 128 arg(u) / pi (the b1 grid of PAPER.md:449)
    const double PI = 3.14159265358979323846;
    double x = 128.0 * std::atan2(ui, ur) / PI;
    double k = (x >= 0.0) ? std::floor(x + 0.5) : -std::floor(-x + 0.5);
    return (int)k;
}

__device__ __forceinline__ uint32_t shift_b1(uint32_t code, int k) {
    if ((code & 0xffu) == 0x80u) return code;  // special zero keeps b1 = 0
    int b1 = (int)(int8_t)(code >> 8);
    b1 = ((b1 + k + 128) & 255) - 128;
    return (code & 0xffu) | ((uint32_t)(b1 & 0xff) << 8);
}

struct AFastParams {
    void *a;
    uint64_t shard_base;
    uint64_t cmask;
    uint64_t n;  // codes in the shard
    int32_t nl, t, cls;
    int32_t k0, k1;  // DIAG: b1 steps for bit 0 / 1; ANTI: k0 = steps of u01, k1 = steps of u10
};

// Diagonal gates visit only the 16-byte vectors (8 codes) that hold touched
// codes: the touched set is "control bits = 1" plus, when one diagonal entry
// has no phase step (CPHASE, S, T, Z ...: k0 = 0), "target bit = 1" -- the
// fixed bits at or above bit 3 are inserted into the vector index (like the E
// sweep), those below bit 3 select lanes.  b1 += k (mod 256) for the
// touched codes, the special zero keeps b1 = 0; b0 never changes.
struct ADiagParams {
    void *a;
    uint64_t nvec;      // vectors visited
    uint64_t orv;       // vector-index bits fixed to 1
    int32_t ins[4];     // vector-index positions of the fixed bits (ascending)
    int32_t nins;
    uint32_t lowmask, lowval;  // fixed bits of the lane index (code bits 0..2)
    int32_t tlow;       // target bit < 3 (lane bit), else -1
    int32_t tvec;       // target bit >= 3 and not fixed: vector-index bit, else -1
    int32_t tconst;     // target bit value when it is neither (fixed or global)
    int32_t k0, k1;
};
__device__ __forceinline__ uint32_t shift_b1_fast(uint32_t code, uint32_t k8) {
    const uint32_t moved = (code & 0xffu) | ((code + k8) & 0xff00u);
    return (code & 0xffu) == 0x80u ? code : moved;
}
__global__ void __launch_bounds__(A_THREADS) k_diag_a(const __grid_constant__ ADiagParams p) {
    uint16_t *a = reinterpret_cast<uint16_t *>(p.a);
    const uint32_t k08 = (uint32_t)p.k0 << 8, k18 = (uint32_t)p.k1 << 8;
    for (uint64_t w = (uint64_t)blockIdx.x * A_THREADS + threadIdx.x; w < p.nvec; w += (uint64_t)gridDim.x * A_THREADS) {
        uint64_t v = w;
        for (int q = 0; q < p.nins; ++q) v = a_ins0(v, p.ins[q]);
        v |= p.orv;
        uint4 x = __ldcs(reinterpret_cast<const uint4 *>(a + (v << 3)));
        uint32_t ws[4] = {x.x, x.y, x.z, x.w};
        const uint32_t tv = p.tvec >= 0 ? (uint32_t)(v >> p.tvec) & 1u : (uint32_t)p.tconst;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (((uint32_t)j & p.lowmask) != p.lowval) continue;
            const uint32_t bit = p.tlow >= 0 ? ((uint32_t)j >> p.tlow) & 1u : tv;
            const uint32_t k8 = bit ? k18 : k08;
            const uint32_t c = (j & 1) ? (ws[j >> 1] >> 16) : (ws[j >> 1] & 0xffffu);
            const uint32_t n = shift_b1_fast(c, k8);
            ws[j >> 1] = (j & 1) ? ((ws[j >> 1] & 0xffffu) | (n << 16)) : ((ws[j >> 1] & 0xffff0000u) | n);
        }
        x.x = ws[0];
        x.y = ws[1];
        x.z = ws[2];
        x.w = ws[3];
        __stcs(reinterpret_cast<uint4 *>(a + (v << 3)), x);
    }
}

template <bool LOWT>
__global__ void __launch_bounds__(A_THREADS) k_anti_a(const __grid_constant__ AFastParams p) {
    uint16_t *a = reinterpret_cast<uint16_t *>(p.a);
    const uint64_t units = (p.nl >= 4) ? (1ull << (p.nl - 4)) : 1ull;
    for (uint64_t u = (uint64_t)blockIdx.x * A_THREADS + threadIdx.x; u < units; u += (uint64_t)gridDim.x * A_THREADS) {
        uint32_t c[16];
        uint64_t s0;
        unit_load<LOWT>(a, u, p.t, c, s0);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            int j0, j1;
            uint64_t i0;
            pair_slots<LOWT>(k, p.t, s0, j0, j1, i0);
            if (((p.shard_base | i0) & p.cmask) != p.cmask) continue;
            uint32_t x = c[j0], y = c[j1];
            c[j0] = shift_b1(y, p.k0);  // a0' = u01 a1
            c[j1] = shift_b1(x, p.k1);  // a1' = u10 a0
        }
        unit_store<LOWT>(a, s0, p.t, c);
    }
}

void launch_fast_a(const AGateParams &g, const ATables *t, cudaStream_t s) {
    (void)t;
    AFastParams p{};
    p.a = g.a;
    p.shard_base = g.shard_base;
    p.cmask = g.cmask;
    p.n = std::max<uint64_t>(1ull << g.nl, 256);  // shards are padded to >= 256 codes (zero specials)
    p.nl = g.nl;
    p.t = g.t;
    p.cls = g.cls;
    if (g.cls == CLS_DIAG) {
        const int k0 = phase_steps(g.u[0], g.u[1]), k1 = phase_steps(g.u[6], g.u[7]);
        const int nl = g.nl >= 3 ? g.nl : 3;  // shards are padded to >= 256 codes (zero specials)
        const uint64_t lmask = (nl >= 64) ? ~0ull : ((1ull << nl) - 1ull);
        uint64_t fixed = g.cmask & lmask, val = fixed;  // global controls: checked by the caller
        ADiagParams d{};
        d.a = g.a;
        d.k0 = k0;
        d.k1 = k1;
        d.tlow = d.tvec = -1;
        if (g.t >= g.nl) {  // global target: one step for the whole shard
            d.tconst = (int)((g.shard_base >> g.t) & 1ull);
            if ((d.tconst ? k1 : k0) == 0) return;
        } else if (k0 == 0 || k1 == 0) {  // only one value of the target bit moves
            if (k0 == 0 && k1 == 0) return;
            fixed |= 1ull << g.t;
            if (k1 != 0) val |= 1ull << g.t;
            d.tconst = k1 != 0 ? 1 : 0;
        } else if (g.t < 3) {
            d.tlow = g.t;
        } else {
            d.tconst = 0;
        }
        d.lowmask = (uint32_t)(fixed & 7u);
        d.lowval = (uint32_t)(val & 7u);
        int nf = 0;
        for (int b = 3; b < nl; ++b)
            if ((fixed >> b) & 1ull) {
                d.ins[nf++] = b - 3;
                if ((val >> b) & 1ull) d.orv |= 1ull << (b - 3);
            }
        d.nins = nf;
        if (g.t >= 3 && g.t < nl && !((fixed >> g.t) & 1ull)) {
            d.tvec = g.t - 3;  // bit of the (inserted) vector index
        }
        d.nvec = (1ull << (nl - 3)) >> nf;
        k_diag_a<<<a_grid(d.nvec), A_THREADS, 0, s>>>(d);
        return;
    } else {
        p.k0 = phase_steps(g.u[2], g.u[3]);
        p.k1 = phase_steps(g.u[4], g.u[5]);
        if (g.t < 4)
            k_anti_a<true><<<a_grid(p.n >> 4), A_THREADS, 0, s>>>(p);
        else
            k_anti_a<false><<<a_grid(p.n >> 4), A_THREADS, 0, s>>>(p);
    }
}

// a run of diagonal gates: per code, the sum of the gates' b1 steps (mod 256)
__global__ void __launch_bounds__(A_THREADS) k_diag_run_a(const __grid_constant__ ADiagRunParams p) {
    uint16_t *a = reinterpret_cast<uint16_t *>(p.a);
    const uint64_t nvec = p.n >> 3;
    for (uint64_t v = (uint64_t)blockIdx.x * A_THREADS + threadIdx.x; v < nvec; v += (uint64_t)gridDim.x * A_THREADS) {
        uint4 w = __ldcs(reinterpret_cast<const uint4 *>(a + (v << 3)));
        uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        const uint32_t hi = (uint32_t)(v << 3);  // local index bits >= 3 of the 8 codes (bits < 32 suffice:
                                                  // the gates' local bits are < 32 -- checked by the caller)
        uint32_t sh[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int gi = 0; gi < p.ngates; ++gi) {
            const ADiagRunGate g = p.g[gi];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t idx = hi | (uint32_t)j;
                const bool on = (idx & g.cmask) == g.cmask;
                const bool bit = g.t >= 0 && ((idx >> g.t) & 1u);
                sh[j] += on ? (uint32_t)(int)(bit ? g.k1 : g.k0) : 0u;
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t c = (j & 1) ? (ws[j >> 1] >> 16) : (ws[j >> 1] & 0xffffu);
            const uint32_t n = shift_b1_fast(c, (sh[j] & 0xffu) << 8);
            ws[j >> 1] = (j & 1) ? ((ws[j >> 1] & 0xffffu) | (n << 16)) : ((ws[j >> 1] & 0xffff0000u) | n);
        }
        w.x = ws[0];
        w.y = ws[1];
        w.z = ws[2];
        w.w = ws[3];
        __stcs(reinterpret_cast<uint4 *>(a + (v << 3)), w);
    }
}

void launch_diag_run_a(const ADiagRunParams &p, cudaStream_t s) {
    k_diag_run_a<<<a_grid(p.n >> 3), A_THREADS, 0, s>>>(p);
}
int a_phase_steps(double ur, double ui) { return phase_steps(ur, ui); }

// exchange for A: codes move; a diagonal / anti-diagonal gate is applied on arrival
struct AXParams {
    void *own;
    const void *stage;
    uint64_t p0, n, shard_base, cmask;
    int32_t l, b, mode, cls, k0, k1;
};
__global__ void __launch_bounds__(A_THREADS) k_xchg_a(const __grid_constant__ AXParams p) {
    uint16_t *own = reinterpret_cast<uint16_t *>(p.own);
    const uint16_t *stg = reinterpret_cast<const uint16_t *>(p.stage);
    const uint64_t lb = 1ull << p.l;
    for (uint64_t k = (uint64_t)blockIdx.x * A_THREADS + threadIdx.x; k < p.n; k += (uint64_t)gridDim.x * A_THREADS) {
        const uint64_t i0 = a_ins0(p.p0 + k, p.l);
        const uint64_t i1 = i0 | lb;
        uint32_t r = stg[k];
        if (p.mode == 0) {
            own[p.b ? i0 : i1] = (uint16_t)r;
            continue;
        }
        uint32_t kept = own[p.b ? i1 : i0];
        uint32_t x = p.b ? r : kept, y = p.b ? kept : r;
        if (((p.shard_base | i0) & p.cmask) == p.cmask) {
            if (p.cls == CLS_ANTI) {
                uint32_t nx = shift_b1(y, p.k0), ny = shift_b1(x, p.k1);
                x = nx;
                y = ny;
            } else {
                x = shift_b1(x, p.k0);
                y = shift_b1(y, p.k1);
            }
        }
        own[i0] = (uint16_t)x;
        own[i1] = (uint16_t)y;
    }
}
void launch_xchg_a(const XchgParams &x, const ATables *t, cudaStream_t s) {
    (void)t;
    AXParams p{};
    p.own = x.own;
    p.stage = x.stage;
    p.p0 = x.p0;
    p.n = x.n;
    p.shard_base = x.shard_base;
    p.cmask = x.cmask;
    p.l = x.l;
    p.b = x.b;
    p.mode = x.mode;
    p.cls = x.cls;
    if (x.mode == 1) {
        if (x.cls == CLS_ANTI) {
            p.k0 = phase_steps(x.u[2], x.u[3]);
            p.k1 = phase_steps(x.u[4], x.u[5]);
        } else {
            p.k0 = phase_steps(x.u[0], x.u[1]);
            p.k1 = phase_steps(x.u[6], x.u[7]);
        }
    }
    k_xchg_a<<<a_grid(x.n / 4 + 1), A_THREADS, 0, s>>>(p);
}

// ---------------------------------------------------------------- collapse (measure)
template <bool APPLY>
__global__ void __launch_bounds__(A_THREADS) k_collapse_a(const __grid_constant__ ACollapseParams p,
                                                          const ATabData *__restrict__ cur,
                                                          const ATabData *__restrict__ nxt, double *partials) {
    __shared__ ASm sm;
    load_asm(sm, cur, nxt);
    uint16_t *a = reinterpret_cast<uint16_t *>(p.a);
    double mn = INFINITY, mx = -INFINITY;
    const uint64_t nvec = p.n >> 3;
    for (uint64_t v = (uint64_t)blockIdx.x * A_THREADS + threadIdx.x; v < nvec; v += (uint64_t)gridDim.x * A_THREADS) {
        uint4 w = *reinterpret_cast<uint4 *>(a + (v << 3));
        uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        uint32_t outc[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint64_t full = p.shard_base | ((v << 3) + k);
            uint32_t c = (k & 1) ? (ws[k >> 1] >> 16) : (ws[k >> 1] & 0xffffu);
            double2 z = a_decode(sm, c);
            if ((int)((full >> p.bit) & 1ull) != p.keep) {
                z.x = 0.0;
                z.y = 0.0;
            } else {
                z.x *= p.f;
                z.y *= p.f;
            }
            if (APPLY) {
                outc[k] = a_encode(sm, z);
            } else {
                double m2 = a_m2(z);
                if (is_inter(m2)) {
                    mn = fmin(mn, m2);
                    mx = fmax(mx, m2);
                }
            }
        }
        if (APPLY) {
            w.x = outc[0] | (outc[1] << 16);
            w.y = outc[2] | (outc[3] << 16);
            w.z = outc[4] | (outc[5] << 16);
            w.w = outc[6] | (outc[7] << 16);
            *reinterpret_cast<uint4 *>(a + (v << 3)) = w;
        }
    }
    if (APPLY) return;
    __shared__ double red[2][A_THREADS / 32];
    mn = warp_min(mn);
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = mn;
        red[1][threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a0 = INFINITY, a1 = -INFINITY;
        for (int w2 = 0; w2 < A_THREADS / 32; ++w2) {
            a0 = fmin(a0, red[0][w2]);
            a1 = fmax(a1, red[1][w2]);
        }
        partials[2 * blockIdx.x] = a0;
        partials[2 * blockIdx.x + 1] = a1;
    }
}
void launch_collapse_bounds_a(const ACollapseParams &p, const ATables *t, double *partials, double *out,
                              cudaStream_t s) {
    int grid = a_grid(p.n >> 3);
    if (grid > 2 * a_num_sms() * 4) grid = 2 * a_num_sms() * 4;
    k_collapse_a<false><<<grid, A_THREADS, 0, s>>>(p, tcur(t), tnext(t), partials);
    k_minmax_final<<<1, 32, 0, s>>>(partials, grid, out, 1);  // out = (min, -max)
}
void launch_collapse_apply_a(const ACollapseParams &p, const ATables *t, cudaStream_t s) {
    k_collapse_a<true><<<a_grid(p.n >> 3), A_THREADS, 0, s>>>(p, tcur(t), tnext(t), nullptr);
}

__global__ void k_init_a(uint16_t *a, uint64_t n, int first) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = (first && i == 0) ? (uint16_t)pack(127, 0) : (uint16_t)pack(-128, 0);
}
void launch_init_a(void *a, uint64_t n, bool first, cudaStream_t s) {
    k_init_a<<<a_grid(n / 8 + 1), A_THREADS, 0, s>>>(reinterpret_cast<uint16_t *>(a), n, first ? 1 : 0);
}

// ---------------------------------------------------------------- reductions on decoded values
__global__ void __launch_bounds__(256) k_probs_a(const uint16_t *__restrict__ a, int nl,
                                                 const ATabData *__restrict__ cur, double *partials) {
    __shared__ ASm sm;
    load_asm(sm, cur, cur);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t n = 1ull << nl;
    const uint64_t nseg = n >> 8;
    const uint64_t gwarp = (uint64_t)blockIdx.x * 8 + warp;
    const uint64_t nwarps = (uint64_t)gridDim.x * 8;
    double tot_lane = 0.0, pj[3] = {0.0, 0.0, 0.0}, phigh = 0.0;
    for (uint64_t sgi = gwarp; sgi < nseg; sgi += nwarps) {
        const uint16_t *seg = a + (sgi << 8);
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            double2 z = a_decode(sm, seg[lane + 32 * j]);
            double m = fma(z.x, z.x, z.y * z.y);
            t += m;
            if (j & 1) pj[0] += m;
            if (j & 2) pj[1] += m;
            if (j & 4) pj[2] += m;
        }
        tot_lane += t;
        double seg_tot = warp_sum_a(t);
        if (8 + lane < nl && ((sgi >> lane) & 1ull)) phigh += seg_tot;
    }
    __shared__ double smr[8][RED_SLOTS];
    double tot = warp_sum_a(tot_lane);
    double pq[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) pq[q] = warp_sum_a((lane >> q) & 1 ? tot_lane : 0.0);
    double p5 = warp_sum_a(pj[0]), p6 = warp_sum_a(pj[1]), p7 = warp_sum_a(pj[2]);
    if (lane == 0) {
        smr[warp][0] = tot;
        for (int q = 0; q < 5; ++q) smr[warp][1 + q] = pq[q];
        smr[warp][6] = p5;
        smr[warp][7] = p6;
        smr[warp][8] = p7;
    }
    smr[warp][9 + lane] = phigh;
    if (41 + lane < RED_SLOTS) smr[warp][41 + lane] = 0.0;
    __syncthreads();
    if (threadIdx.x < RED_SLOTS) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += smr[w][threadIdx.x];
        partials[(size_t)blockIdx.x * RED_SLOTS + threadIdx.x] = s;
    }
}
__global__ void k_final_sum_a(const double *partials, int nblocks, int nslots, double *out) {
    int s = threadIdx.x;
    if (s >= nslots) return;
    double acc = 0.0;
    for (int b = 0; b < nblocks; ++b) acc += partials[(size_t)b * nslots + s];
    out[s] = acc;
}
void launch_probs_a(const void *a, int nl, const ATables *t, double *partials, double *out, cudaStream_t s) {
    int nb = red_blocks();
    k_probs_a<<<nb, 256, 0, s>>>(reinterpret_cast<const uint16_t *>(a), nl, tcur(t), partials);
    k_final_sum_a<<<1, RED_SLOTS, 0, s>>>(partials, nb, RED_SLOTS, out);
}

__global__ void __launch_bounds__(256) k_pairdot_a(const uint16_t *__restrict__ a, int nl, int q,
                                                   const ATabData *__restrict__ cur, double *partials) {
    __shared__ ASm sm;
    load_asm(sm, cur, cur);
    const uint64_t npairs = 1ull << (nl - 1);
    const uint64_t qb = 1ull << q;
    double sr = 0.0, si = 0.0;
    for (uint64_t w = (uint64_t)blockIdx.x * 256 + threadIdx.x; w < npairs; w += (uint64_t)gridDim.x * 256) {
        uint64_t i0 = a_ins0(w, q);
        double2 x = a_decode(sm, a[i0]), y = a_decode(sm, a[i0 | qb]);
        sr = fma(x.x, y.x, fma(x.y, y.y, sr));
        si = fma(x.x, y.y, fma(-x.y, y.x, si));
    }
    __shared__ double red[2][8];
    sr = warp_sum_a(sr);
    si = warp_sum_a(si);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = sr;
        red[1][threadIdx.x >> 5] = si;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        double s2 = 0.0;
        for (int w = 0; w < 8; ++w) s2 += red[threadIdx.x][w];
        partials[(size_t)blockIdx.x * 2 + threadIdx.x] = s2;
    }
}
void launch_pairdot_a(const void *a, int nl, int q, const ATables *t, double *partials, double *out,
                      cudaStream_t s) {
    int nb = red_blocks();
    k_pairdot_a<<<nb, 256, 0, s>>>(reinterpret_cast<const uint16_t *>(a), nl, q, tcur(t), partials);
    k_final_sum_a<<<1, 32, 0, s>>>(partials, nb, 2, out);
}

__global__ void __launch_bounds__(256) k_dot_a(const uint16_t *__restrict__ x, const uint16_t *__restrict__ y,
                                               uint64_t n, const ATabData *__restrict__ cur, double *partials) {
    __shared__ ASm sm;
    load_asm(sm, cur, cur);
    double sr = 0.0, si = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256) {
        double2 u = a_decode(sm, x[i]), v = a_decode(sm, y[i]);
        sr = fma(u.x, v.x, fma(u.y, v.y, sr));
        si = fma(u.x, v.y, fma(-u.y, v.x, si));
    }
    __shared__ double red[2][8];
    sr = warp_sum_a(sr);
    si = warp_sum_a(si);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = sr;
        red[1][threadIdx.x >> 5] = si;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        double s2 = 0.0;
        for (int w = 0; w < 8; ++w) s2 += red[threadIdx.x][w];
        partials[(size_t)blockIdx.x * 2 + threadIdx.x] = s2;
    }
}
void launch_dot_a(const void *x, const void *y, uint64_t n, const ATables *t, double *partials, double *out,
                  cudaStream_t s) {
    int nb = red_blocks();
    k_dot_a<<<nb, 256, 0, s>>>(reinterpret_cast<const uint16_t *>(x), reinterpret_cast<const uint16_t *>(y), n,
                               tcur(t), partials);
    k_final_sum_a<<<1, 32, 0, s>>>(partials, nb, 2, out);
}

// <x|y> = sum conj(x_i) y_i over one shard pair, each side E (complex fp64)
// or A (decoded with its own current tables): the fidelity of an A run
// against an E run of the same circuit.
struct AOvSm {
    double r[2][256];
    double2 cs[2][256];
};
template <bool XA, bool YA>
__global__ void __launch_bounds__(256) k_overlap(const void *__restrict__ xv, const void *__restrict__ yv, uint64_t n,
                                                 const ATabData *__restrict__ tx, const ATabData *__restrict__ ty,
                                                 double *partials) {
    __shared__ AOvSm sm;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        if (XA) {
            sm.r[0][i] = tx->r[i];
            sm.cs[0][i] = make_double2(tx->cth[i], tx->sth[i]);
        }
        if (YA) {
            sm.r[1][i] = ty->r[i];
            sm.cs[1][i] = make_double2(ty->cth[i], ty->sth[i]);
        }
    }
    __syncthreads();
    double sr = 0.0, si = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256) {
        double2 u, v;
        if (XA) {
            const uint32_t c = reinterpret_cast<const uint16_t *>(xv)[i];
            const double r = sm.r[0][(c & 0xffu) ^ 0x80u];
            const double2 e = sm.cs[0][((c >> 8) & 0xffu) ^ 0x80u];
            u = make_double2(r * e.x, r * e.y);
        } else {
            u = reinterpret_cast<const double2 *>(xv)[i];
        }
        if (YA) {
            const uint32_t c = reinterpret_cast<const uint16_t *>(yv)[i];
            const double r = sm.r[1][(c & 0xffu) ^ 0x80u];
            const double2 e = sm.cs[1][((c >> 8) & 0xffu) ^ 0x80u];
            v = make_double2(r * e.x, r * e.y);
        } else {
            v = reinterpret_cast<const double2 *>(yv)[i];
        }
        sr = fma(u.x, v.x, fma(u.y, v.y, sr));
        si = fma(u.x, v.y, fma(-u.y, v.x, si));
    }
    __shared__ double red[2][8];
    sr = warp_sum_a(sr);
    si = warp_sum_a(si);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = sr;
        red[1][threadIdx.x >> 5] = si;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        double s2 = 0.0;
        for (int w = 0; w < 8; ++w) s2 += red[threadIdx.x][w];
        partials[(size_t)blockIdx.x * 2 + threadIdx.x] = s2;
    }
}
void launch_overlap(const void *x, const ATables *tx, const void *y, const ATables *ty, uint64_t n, double *partials,
                    double *out, cudaStream_t s) {
    const int nb = red_blocks();
    const ATabData *dx = tx ? tcur(tx) : nullptr, *dy = ty ? tcur(ty) : nullptr;
    if (tx && ty)
        k_overlap<true, true><<<nb, 256, 0, s>>>(x, y, n, dx, dy, partials);
    else if (tx)
        k_overlap<true, false><<<nb, 256, 0, s>>>(x, y, n, dx, dy, partials);
    else if (ty)
        k_overlap<false, true><<<nb, 256, 0, s>>>(x, y, n, dx, dy, partials);
    else
        k_overlap<false, false><<<nb, 256, 0, s>>>(x, y, n, dx, dy, partials);
    k_final_sum_a<<<1, 32, 0, s>>>(partials, nb, 2, out);
}

__global__ void __launch_bounds__(256) k_gather_a(const uint16_t *__restrict__ a, const uint64_t *__restrict__ off,
                                                  uint64_t m, const ATabData *__restrict__ cur, double2 *out) {
    __shared__ ASm sm;
    load_asm(sm, cur, cur);
    for (uint64_t k = (uint64_t)blockIdx.x * 256 + threadIdx.x; k < m; k += (uint64_t)gridDim.x * 256)
        out[k] = a_decode(sm, a[off[k]]);
}
void launch_gather_a(const void *a, const uint64_t *off, uint64_t m, const ATables *t, double *out, cudaStream_t s) {
    if (!m) return;
    k_gather_a<<<a_grid(m), 256, 0, s>>>(reinterpret_cast<const uint16_t *>(a), off, m, tcur(t),
                                         reinterpret_cast<double2 *>(out));
}

__device__ __forceinline__ uint64_t phys_to_logical_a(uint64_t phys, const int *inv, int nq) {
    uint64_t L = 0;
    for (int b = 0; b < nq; ++b)
        if ((phys >> b) & 1ull) L |= 1ull << inv[b];
    return L;
}
__global__ void __launch_bounds__(256) k_to_logical_a(const uint16_t *__restrict__ a, uint64_t n, uint64_t base,
                                                      const int *__restrict__ inv, int nq,
                                                      const ATabData *__restrict__ cur, double2 *out) {
    __shared__ ASm sm;
    load_asm(sm, cur, cur);
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256)
        out[phys_to_logical_a(base | i, inv, nq)] = a_decode(sm, a[i]);
}
void launch_to_logical_a(const void *a, uint64_t n, uint64_t base, const int *inv, int nq, const ATables *t,
                         void *out, cudaStream_t s) {
    k_to_logical_a<<<a_grid(n), 256, 0, s>>>(reinterpret_cast<const uint16_t *>(a), n, base, inv, nq, tcur(t),
                                             reinterpret_cast<double2 *>(out));
}
__global__ void k_codes_to_logical(const uint16_t *__restrict__ a, uint64_t n, uint64_t base,
                                   const int *__restrict__ inv, int nq, uint16_t *out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[phys_to_logical_a(base | i, inv, nq)] = a[i];
}
__global__ void k_codes_from_logical(uint16_t *a, uint64_t n, uint64_t base, const int *__restrict__ inv, int nq,
                                     const uint16_t *__restrict__ in) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = in[phys_to_logical_a(base | i, inv, nq)];
}
void launch_codes_to_logical_a(const void *a, uint64_t n, uint64_t base, const int *inv, int nq, void *out,
                               cudaStream_t s) {
    k_codes_to_logical<<<a_grid(n), 256, 0, s>>>(reinterpret_cast<const uint16_t *>(a), n, base, inv, nq,
                                                 reinterpret_cast<uint16_t *>(out));
}
void launch_codes_from_logical_a(void *a, uint64_t n, uint64_t base, const int *inv, int nq, const void *in,
                                 cudaStream_t s) {
    k_codes_from_logical<<<a_grid(n), 256, 0, s>>>(reinterpret_cast<uint16_t *>(a), n, base, inv, nq,
                                                   reinterpret_cast<const uint16_t *>(in));
}

}  // namespace qsim
