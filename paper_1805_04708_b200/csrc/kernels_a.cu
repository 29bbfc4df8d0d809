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
#include <atomic>
#include <cmath>
#include <cstring>
#include <cstdio>

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

static void fill_ftab(AFTab &f, const ATabData &t) {
    for (int raw = 0; raw < 256; ++raw) {
        const int i = (int)(int8_t)(uint8_t)raw + 128;  // table index of the code byte
        const float r = (float)t.r[i], c = (float)t.cth[i], sn = (float)t.sth[i];
        for (int l = 0; l < 32; ++l) f.rf[raw][l] = r;
        for (int l = 0; l < 16; ++l) {
            f.cs[raw][l][0] = c;
            f.cs[raw][l][1] = sn;
        }
    }
}

int atables_alloc(ATables **out) {
    auto *t = new ATables();
    if (cudaMalloc(&t->d[0], sizeof(ATabData)) != cudaSuccess || cudaMalloc(&t->d[1], sizeof(ATabData)) != cudaSuccess ||
        cudaMalloc(&t->f[0], sizeof(AFTab)) != cudaSuccess || cudaMalloc(&t->f[1], sizeof(AFTab)) != cudaSuccess ||
        cudaMalloc(&t->gext, 2 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMallocHost(&t->h, sizeof(ATabData)) != cudaSuccess || cudaMallocHost(&t->hf, sizeof(AFTab)) != cudaSuccess) {
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
    for (int k = 0; k < 2; ++k) {
        if (t->d[k]) cudaFree(t->d[k]);
        if (t->f[k]) cudaFree(t->f[k]);
    }
    if (t->gext) cudaFree(t->gext);
    if (t->h) cudaFreeHost(t->h);
    if (t->hf) cudaFreeHost(t->hf);
    delete t;
}

static int upload(ATables *t, int which, double r0, double r1, cudaStream_t s) {
    if (cudaStreamSynchronize(s) != cudaSuccess) return QSIM_ECUDA;  // h is reused
    fill_tables(*t->h, r0, r1);
    fill_ftab(*t->hf, *t->h);
    if (cudaMemcpyAsync(t->d[which], t->h, sizeof(ATabData), cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(t->f[which], t->hf, sizeof(AFTab), cudaMemcpyHostToDevice, s) != cudaSuccess) {
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
static const AFTab *fcur(const ATables *t) { return t->f[t->cur]; }

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
    // local index of code j of the unit at s0
    __device__ static __forceinline__ uint64_t pos(uint64_t s0, int t, int j) {
        return TL < 4 ? s0 + (uint64_t)j : (j < 8 ? s0 + (uint64_t)j : (s0 | (1ull << t)) + (uint64_t)(j - 8));
    }
    __device__ static __forceinline__ void load_raw(const uint16_t *__restrict__ a, uint64_t s0, int t, uint4 &v0,
                                                    uint4 &v1) {
        v0 = __ldcs(reinterpret_cast<const uint4 *>(a + s0));
        v1 = __ldcs(reinterpret_cast<const uint4 *>(a + (TL < 4 ? s0 + 8 : (s0 | (1ull << t)))));
    }
    __device__ static __forceinline__ void unpack(const uint4 &v0, const uint4 &v1, uint32_t (&c)[16]) {
        const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            c[2 * k] = w[k] & 0xffffu;
            c[2 * k + 1] = w[k] >> 16;
        }
    }
    __device__ static __forceinline__ void load(const uint16_t *__restrict__ a, uint64_t s0, int t, uint32_t (&c)[16]) {
        uint4 v0, v1;
        load_raw(a, s0, t, v0, v1);
        unpack(v0, v1, c);
    }
    __device__ static __forceinline__ void store(uint16_t *__restrict__ a, uint64_t s0, int t, const uint32_t (&c)[16]) {
        uint4 v0, v1;  // low halves of c[] (upper bits ignored)
        v0.x = __byte_perm(c[0], c[1], 0x5410);
        v0.y = __byte_perm(c[2], c[3], 0x5410);
        v0.z = __byte_perm(c[4], c[5], 0x5410);
        v0.w = __byte_perm(c[6], c[7], 0x5410);
        v1.x = __byte_perm(c[8], c[9], 0x5410);
        v1.y = __byte_perm(c[10], c[11], 0x5410);
        v1.z = __byte_perm(c[12], c[13], 0x5410);
        v1.w = __byte_perm(c[14], c[15], 0x5410);
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


// ---- certified fp32 fast path -------------------------------------------------
// The dense A gate decides codes and bounds from fp32 copies of the decode
// tables, of U and of the gate arithmetic, together with a rigorous bound on
// how far each fp32 output can be from the fp64 reference (a_decode, a_gate2,
// a_m2 / a_encode -- the functions of the fallback, which follow the oracle's
// definition).  A code (or a bounds candidate) is committed from fp32 only when
// that bound proves the fp64 reference decides the same way; otherwise the
// pair is recomputed in fp64.  So the result is the fp64 reference's, bit for
// bit, while almost every pair costs fp32 arithmetic only.
//
// Error bound (u = 2^-24): the fp32 decode has |zf - z| <= 3u r per component
// (table value r, cos / sin and the product each rounded once); one output
// component is 4 products summed by an fma chain, with |Re u_ij| + |Im u_ij|
// <= sqrt2: sum_j sqrt2 (3u + u) r_j for the inputs and coefficients plus 4
// roundings of partial sums <= 4u sqrt2 (ra + rb) -- in all <= 11.4u (ra + rb)
// = 6.8e-7 (ra + rb).  A_KF = 1e-6 > that, so per output component
// |xf - x| <= E = A_KF (ra + rb) with ra, rb the pair's decoded magnitudes.
//
// Lookups: the fp32 tables (AFTab, 64 KiB of dynamic shared memory) hold one
// copy per lane, so a warp's 32 random codes never share a bank (the shared
// 256-entry tables cost ~5 wavefronts per lookup on random codes).
#define A_KF 1e-6f

template <int UK>
__device__ __forceinline__ void a_gate2u(const double (&u)[8], double2 &x, double2 &y) {
    if (UK == 0)
        a_gate2(u, x, y);
    else
        a_gate2k<UK>(u, x, y);
}
__device__ __forceinline__ void a_gate_f(const float (&u)[8], float2 &x, float2 &y) {
    const float2 x0 = x, y0 = y;
    x.x = fmaf(u[0], x0.x, fmaf(-u[1], x0.y, fmaf(u[2], y0.x, -u[3] * y0.y)));
    x.y = fmaf(u[0], x0.y, fmaf(u[1], x0.x, fmaf(u[2], y0.y, u[3] * y0.x)));
    y.x = fmaf(u[4], x0.x, fmaf(-u[5], x0.y, fmaf(u[6], y0.x, -u[7] * y0.y)));
    y.y = fmaf(u[4], x0.y, fmaf(u[5], x0.x, fmaf(u[6], y0.y, u[7] * y0.x)));
}
template <int UK>
__device__ __forceinline__ void a_gate_fu(const float (&u)[8], float2 &x, float2 &y) {
    if (UK == 0)
        a_gate_f(u, x, y);
    else
        a_gate_fk<UK>(u, x, y);
}

__device__ __forceinline__ float2 f2s(float v) { return make_float2(v, v); }

// The fp32 gate on Blackwell's packed fp32x2 instructions (FFMA2 / FMUL2, a
// scalar operand broadcast to both halves): the outputs come out as
// RE = (Re x', Re y'), IM = (Im x', Im y') -- the layout a_encode_f2 takes --
// from the decoded inputs A = x, B = y.  Each component is the same sum of at
// most 4 products by an fma chain as a_gate_f (the error bound A_KF covers
// any order); the coefficient pairs kf come from a_dense_params:
//   UK 0: RE = (u0,u4) A.x + (-u1,-u5) A.y + (u2,u6) B.x + (-u3,-u7) B.y,
//         IM = (u1,u5) A.x + (u0,u4) A.y + (u3,u7) B.x + (u2,u6) B.y;
//   UK 1: RE = (u0,u4) A.x + (u2,u6) B.x, IM = (u0,u4) A.y + (u2,u6) B.y;
//   UK 2: RE = (u0,-u5) (A.x,A.y) + (-u3,u6) (B.y,B.x),
//         IM = (u0,u5) (A.y,A.x) + (u3,u6) (B.x,B.y).
template <int UK>
__device__ __forceinline__ void a_gate_f2(const float (&k)[16], float2 A, float2 B, float2 &RE, float2 &IM) {
    const float2 k0 = make_float2(k[0], k[1]), k1 = make_float2(k[2], k[3]);
    const float2 k2 = make_float2(k[4], k[5]), k3 = make_float2(k[6], k[7]);
    if (UK == 0) {
        const float2 k4 = make_float2(k[8], k[9]), k5 = make_float2(k[10], k[11]);
        const float2 k6 = make_float2(k[12], k[13]), k7 = make_float2(k[14], k[15]);
        RE = __ffma2_rn(k3, f2s(B.y), __ffma2_rn(k2, f2s(B.x), __ffma2_rn(k1, f2s(A.y), __fmul2_rn(k0, f2s(A.x)))));
        IM = __ffma2_rn(k7, f2s(B.y), __ffma2_rn(k6, f2s(B.x), __ffma2_rn(k5, f2s(A.y), __fmul2_rn(k4, f2s(A.x)))));
    } else if (UK == 1) {
        RE = __ffma2_rn(k2, f2s(B.x), __fmul2_rn(k0, f2s(A.x)));
        IM = __ffma2_rn(k2, f2s(B.y), __fmul2_rn(k0, f2s(A.y)));
    } else {
        RE = __ffma2_rn(k0, A, __fmul2_rn(k1, make_float2(B.y, B.x)));
        IM = __ffma2_rn(k2, make_float2(A.y, A.x), __fmul2_rn(k3, B));
    }
}

// the fp32 tables of this thread's lane in shared memory
struct AFLane {
    const float *rf;   // rf[raw * 32]
    const float2 *cs;  // cs[raw * 16]
    __device__ __forceinline__ float2 decode(uint32_t code, float &r) const {
        r = rf[(code & 0xffu) * 32u];
        const float2 c = cs[((code >> 8) & 0xffu) * 16u];
        return make_float2(r * c.x, r * c.y);
    }
    // the byte offsets of both tables are raw * 128
    __device__ __forceinline__ float mag(uint32_t code) const {
        return *reinterpret_cast<const float *>(reinterpret_cast<const char *>(rf) +
                                                (__byte_perm(code, 0u, 0x4440) << 7));
    }
    __device__ __forceinline__ float2 cs2(uint32_t code) const {
        return *reinterpret_cast<const float2 *>(reinterpret_cast<const char *>(cs) +
                                                 (__byte_perm(code, 0u, 0x4441) << 7));
    }
    // the same values as decode (one FMUL2)
    __device__ __forceinline__ float2 decode2(uint32_t code, float &r) const {
        r = mag(code);
        return __fmul2_rn(f2s(r), cs2(code));
    }
};
extern __shared__ __align__(16) unsigned char a_dsm[];
// stage the fp32 tables (64 KiB, L2-resident) in shared memory
__device__ __forceinline__ AFLane load_aflane(const AFTab *__restrict__ f) {
    const uint4 *src = reinterpret_cast<const uint4 *>(f);
    uint4 *dst = reinterpret_cast<uint4 *>(a_dsm);
    for (int i = threadIdx.x; i < (int)(sizeof(AFTab) / 16); i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const AFTab *t = reinterpret_cast<const AFTab *>(a_dsm);
    AFLane L;
    L.rf = &t->rf[0][lane];
    L.cs = reinterpret_cast<const float2 *>(&t->cs[0][lane & 15][0]);
    return L;
}

// The fp64 reference tables read from global memory (the fallback path is
// rare; the dense kernels keep shared memory for the fp32 tables).  Same
// values and the same arithmetic as ASm / a_decode / a_encode.
struct AGlob {
    const ATabData *cur, *nxt;
    float mmargin;
    __device__ void init(const ATabData *c, const ATabData *n) {
        cur = c;
        nxt = n;
        const double e = 6e-7 * (__ldg(&n->r1) + __ldg(&n->r0)) * __ldg(&n->scale) + 1e-4;
        mmargin = (float)(e < 0.49 ? e : 0.5);
    }
    __device__ __forceinline__ double2 decode(uint32_t code) const {
        const int b0i = (int)(code & 0xffu) ^ 0x80, b1i = (int)((code >> 8) & 0xffu) ^ 0x80;
        const double r = __ldg(&cur->r[b0i]);
        return make_double2(r * __ldg(&cur->cth[b1i]), r * __ldg(&cur->sth[b1i]));
    }
    __device__ uint32_t encode(double2 z) const {
        const double m2 = a_m2(z);
        if (m2 < A_ZERO2) return pack(-128, 0);
        int b0;
        if (m2 > A_ONE2) {
            b0 = 127;
        } else if (__ldg(&nxt->degenerate)) {
            b0 = 0;
        } else {
            const float mf = sqrtf((float)m2);
            const float tf = (mf - (float)__ldg(&nxt->r0)) * (float)__ldg(&nxt->scale);
            int c = __float2int_rn(tf);
            const float fr = tf - (float)c;
            c = max(0, min(253, c));
            if (fabsf(fr) > 0.5f - mmargin) {
                if (c < 253 && m2 >= __ldg(&nxt->thr[c]))
                    c += 1;
                else if (c > 0 && m2 < __ldg(&nxt->thr[c - 1]))
                    c -= 1;
            }
            b0 = c - 127;
        }
        // angle: the same decision as a_angle_code
        const float af = atan2_steps((float)z.y, (float)z.x);
        int k = __float2int_rn(af);
        const float fr = af - (float)k;
        k = max(-128, min(128, k));
        if (fabsf(fr) > 0.5f - A_MARGIN) {
            const double cu = z.y * __ldg(&nxt->cb[k + 129]) - z.x * __ldg(&nxt->sb[k + 129]);
            if ((k >= 0) ? (cu >= 0.0) : (cu > 0.0)) {
                k += 1;
            } else {
                const double cl = z.y * __ldg(&nxt->cb[k + 128]) - z.x * __ldg(&nxt->sb[k + 128]);
                if ((k > 0) ? (cl < 0.0) : (cl <= 0.0)) k -= 1;
            }
            k = max(-128, min(128, k));
        }
        return pack(b0, (k == 128) ? -128 : k);
    }
};

// Encode constants of the next bounds (per thread, from nxt): t = mf s1 + s0
// is the fp32 magnitude coordinate (b0 + 127); its distance to the fp64
// reference's is at most (5.2e-7 |z| + sqrt2 E) scale + C0 steps (candidate
// mf: 4e-7 mf + sqrt2 E from |zf - z|; s1, s0 and the roundings: 6e-8 (mf +
// r0) scale + 253 * 2^-24 + slack).  Degenerate bounds (r0 = r1): t = 127
// exactly, the code every intermediate gets.
struct AEncF {
    float s1, s0, kS, kE, C0;
    __device__ void init(const ATabData *n) {
        const double sc = __ldg(&n->scale), r0 = __ldg(&n->r0);
        if (__ldg(&n->degenerate)) {
            s1 = 0.f;
            s0 = 127.f;
            kS = kE = C0 = 0.f;
        } else {
            s1 = (float)sc;
            s0 = (float)(-r0 * sc);
            kS = (float)(5.2e-7 * sc);
            kE = (float)(1.4143 * sc);
            C0 = (float)(1.2e-7 * r0 * sc + 5e-5);
        }
    }
};

// fp32 atan(w) in units of 2 b1 steps (256/pi per radian) for |w| <= 1: odd
// polynomial of degree 13 (least-squares minimax fit, |error| <= 3e-5 steps
// in fp32 evaluation); used on the half angle w = tan(theta / 2).
__device__ __forceinline__ float atan_2steps(float w) {
    const float s = w * w;
    float p = fmaf(0.5550681352615356f, s, -2.7382962703704834f);
    p = fmaf(p, s, 6.488292694091797f);
    p = fmaf(p, s, -10.783480644226074f);
    p = fmaf(p, s, 16.14085578918457f);
    p = fmaf(p, s, -27.149433135986328f);
    p = fmaf(p, s, 81.48701477050781f);
    return p * w;
}

// raw MUFU approximations, flush-to-zero (no denormal rescaling): an output
// with |z|^2 < 2^-126 gives rs = inf, mf = NaN and fails certification (the
// fp64 fallback decides it), far below the intermediate range |z| >= 1e-12
__device__ __forceinline__ float a_rsqrt(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float a_rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

#define A_MAGIC 12582912.0f  // 1.5 * 2^23: x + A_MAGIC holds round(x) in its low mantissa bits

// One fp32 output z of a pair with magnitudes ra + rb = S -> a 16-bit code
// candidate; ok = the error bounds prove the fp64 reference gives the same
// code.  Magnitude: t = mf scale - r0 scale is the coordinate b0 + 127; the
// exact t lies in [0, 253] (r0, r1 are the exact extremes of these very
// outputs), so round(t) needs no clamp; byte (c + 129) & 0xff = c - 127.  Its
// certification takes the pair's limit limm = 0.5 - ((5.2e-7 S + sqrt2 E)
// scale + C0) (|z| <= S).  Angle: theta = 2 atan(y / (|z| + |x|)), reflected
// for x < 0, in steps; k = round half away (exact ties fall back); byte
// k & 0xff (k = 128 wraps to -128, reading R-A6).  Its error: 73 E / |z|
// steps from E (valid while E / |z| <= 0.141; above, 73 E rs > 0.5 fails) +
// 2e-4 for the polynomial and the roundings.  A passing angle test also
// proves |z| > 0.99 mf >= 1.445e-4 S, so S > 7e-9 (checked per pair) rules
// out the special zero.
template <bool LAZY>
__device__ __forceinline__ uint32_t a_encode_f(const AEncF &ce, float2 z, float errm, float KE, float eS, bool &ok,
                                              bool &oor) {
    const float m2 = fmaf(z.x, z.x, z.y * z.y);
    const float rs = a_rsqrt(m2);
    const float mf = m2 > 0.f ? m2 * rs : 0.f;
    float t = fmaf(mf, ce.s1, ce.s0);
    bool edge = false;
    // |z| certainly below 1e-12: the special zero; certainly above: intermediate (reading R-A5)
    const bool zero = fmaf(mf, 1.0000005f, eS) < 0.99999e-12f;
    const bool inter = fmaf(mf, 0.9999995f, -eS) > 1.00001e-12f;
    if (LAZY) {
        // kept bounds: one step (1 in t) of slack on each side, clamped to the end codes;
        // certainly outside -> rescale; within errm of the slack's edge -> fp64 decides
        oor = inter & ((t < -1.f - errm) | (t > 254.f + errm));
        edge = (fabsf(t + 1.f) <= errm) | (fabsf(t - 254.f) <= errm);
        t = fminf(fmaxf(t, 0.f), 253.f);
    }
    const float tm = t + (A_MAGIC + 129.f);
    const float frm = t - (tm - (A_MAGIC + 129.f));
    const float w = z.y * a_rcp(mf + fabsf(z.x));
    const float p = atan_2steps(w);
    const float q = (z.x < 0.f) ? copysignf(128.f, z.y) - p : p;
    const float ta = q + A_MAGIC;
    const float fra = q - (ta - A_MAGIC);
    ok = zero | (inter & !edge & (fabsf(frm) < 0.5f - errm) & (fmaf(KE, rs, fabsf(fra)) < 0.4998f));
    return zero ? 0x0080u : __byte_perm(__float_as_uint(tm), __float_as_uint(ta), 0x0040);
}

// The same encode for the two outputs of a pair at once, on Blackwell's
// packed fp32x2 instructions (FFMA2 / FADD2 / FMUL2: two IEEE round-to-nearest
// operations per issue, the same results bit for bit as the scalar ones above,
// so the certification is unchanged); lane .x = output x, .y = output y.
__device__ __forceinline__ float2 atan_2steps2(float2 w) {
    const float2 s = __fmul2_rn(w, w);
    float2 p = __ffma2_rn(f2s(0.5550681352615356f), s, f2s(-2.7382962703704834f));
    p = __ffma2_rn(p, s, f2s(6.488292694091797f));
    p = __ffma2_rn(p, s, f2s(-10.783480644226074f));
    p = __ffma2_rn(p, s, f2s(16.14085578918457f));
    p = __ffma2_rn(p, s, f2s(-27.149433135986328f));
    p = __ffma2_rn(p, s, f2s(81.48701477050781f));
    return __fmul2_rn(p, w);
}
// FAST (the fp32 arithmetic variant, reading R-A26): the same fp32 values,
// no certification -- the magnitude coordinate clamped to the end codes, the
// special zero decided in fp32 (|zf| < 1e-12); the codes differ from the fp64
// reference's only where the fp32 error (~1e-6 relative) crosses a rounding
// boundary, i.e. by one step.
template <bool LAZY, bool FAST = false>
__device__ __forceinline__ void a_encode_f2(const AEncF &ce, float2 re, float2 im, float errm, float KE, float eS,
                                            uint32_t &cx, uint32_t &cy, bool &okx, bool &oky, bool &ox, bool &oy) {
    const float2 m2 = __ffma2_rn(re, re, __fmul2_rn(im, im));
    // rsqrt of max(m2, 1e-37): mf = |z| for m2 >= 1e-37, 0 for m2 = 0, and below
    // sqrt(m2) < 3.2e-19 otherwise -- all of those certify as the special zero
    // (|z| <= 3.2e-19 + eS < 1e-12 whenever mf + eS passes the zero test)
    const float2 rs = make_float2(a_rsqrt(fmaxf(m2.x, 1e-37f)), a_rsqrt(fmaxf(m2.y, 1e-37f)));
    const float2 mf = __fmul2_rn(m2, rs);
    float2 t = __ffma2_rn(mf, f2s(ce.s1), f2s(ce.s0));
    bool zerox, zeroy, interx, intery;
    if (FAST) {
        zerox = mf.x < 1e-12f;
        zeroy = mf.y < 1e-12f;
        interx = !zerox;
        intery = !zeroy;
        t.x = fminf(fmaxf(t.x, 0.f), 253.f);
        t.y = fminf(fmaxf(t.y, 0.f), 253.f);
    } else {
        const float2 zt = __ffma2_rn(mf, f2s(1.0000005f), f2s(eS));
        const float2 it = __ffma2_rn(mf, f2s(0.9999995f), f2s(-eS));
        zerox = zt.x < 0.99999e-12f;
        zeroy = zt.y < 0.99999e-12f;
        interx = it.x > 1.00001e-12f;
        intery = it.y > 1.00001e-12f;
    }
    bool edgex = false, edgey = false;
    if (LAZY) {
        ox = interx & ((t.x < -1.f - errm) | (t.x > 254.f + errm));
        oy = intery & ((t.y < -1.f - errm) | (t.y > 254.f + errm));
        edgex = (fabsf(t.x + 1.f) <= errm) | (fabsf(t.x - 254.f) <= errm);
        edgey = (fabsf(t.y + 1.f) <= errm) | (fabsf(t.y - 254.f) <= errm);
        t.x = fminf(fmaxf(t.x, 0.f), 253.f);
        t.y = fminf(fmaxf(t.y, 0.f), 253.f);
    }
    const float2 tm = __fadd2_rn(t, f2s(A_MAGIC + 129.f));
    const float2 frm = __fadd2_rn(t, __ffma2_rn(tm, f2s(-1.f), f2s(A_MAGIC + 129.f)));  // t - (tm - M), exact
    const float2 den = __fadd2_rn(mf, make_float2(fabsf(re.x), fabsf(re.y)));
    const float2 w = __fmul2_rn(im, make_float2(a_rcp(den.x), a_rcp(den.y)));
    const float2 p = atan_2steps2(w);
    const float2 q = make_float2((re.x < 0.f) ? copysignf(128.f, im.x) - p.x : p.x,
                                 (re.y < 0.f) ? copysignf(128.f, im.y) - p.y : p.y);
    const float2 ta = __fadd2_rn(q, f2s(A_MAGIC));
    const float2 fra = __fadd2_rn(q, __ffma2_rn(ta, f2s(-1.f), f2s(A_MAGIC)));  // q - (ta - M), exact
    if (FAST) {
        okx = oky = true;
    } else {
        const float2 ka = __ffma2_rn(f2s(KE), rs, make_float2(fabsf(fra.x), fabsf(fra.y)));
        okx = zerox | (interx & !edgex & (fabsf(frm.x) < 0.5f - errm) & (ka.x < 0.4998f));
        oky = zeroy | (intery & !edgey & (fabsf(frm.y) < 0.5f - errm) & (ka.y < 0.4998f));
    }
    cx = zerox ? 0x0080u : __byte_perm(__float_as_uint(tm.x), __float_as_uint(ta.x), 0x0040);
    cy = zeroy ? 0x0080u : __byte_perm(__float_as_uint(tm.y), __float_as_uint(ta.y), 0x0040);
}

// b1 += k8 >> 8 (mod 256) except for the special zero, which keeps b1 = 0
// (a diagonal gate's phase step); b0 never changes
__device__ __forceinline__ uint32_t shift_b1_fast(uint32_t code, uint32_t k8) {
    const uint32_t moved = (code & 0xffu) | ((code + k8) & 0xff00u);
    return (code & 0xffu) == 0x80u ? code : moved;
}

// The following diagonal run (AEpilogue): the summed b1 step of code j of the
// unit at s0 -- the same sum k_diag_run_a forms per code.  The scalar part is
// one value per unit.
__device__ __forceinline__ uint32_t a_epi_scalar(const AEpilogue &e, uint64_t s0) {
    uint32_t acc = 0;
#pragma unroll 1
    for (int g = 0; g < e.nscalar; ++g) {
        const AEpiScalar x = e.s[g];
        const bool on = (s0 & x.cext) == x.cext;
        const bool b = x.t >= 0 && ((s0 >> x.t) & 1ull);
        acc += on ? (uint32_t)(int)(b ? x.k1 : x.k0) : 0u;
    }
    return acc;
}
// the queue path (rare): the steps of the pair's two codes, sh0 | sh1 << 8
__device__ __noinline__ uint32_t a_epi_pair(const AEpilogue *e, uint64_t s0, int j0, int j1) {
    const uint32_t acc = a_epi_scalar(*e, s0);
    uint32_t s[2] = {acc + (uint32_t)(int)e->base[j0], acc + (uint32_t)(int)e->base[j1]};
#pragma unroll 1
    for (int g = 0; g < e->nmixed; ++g) {
        const AEpiMixed &m = e->m[g];
        if ((s0 & m.cext) != m.cext) continue;
        const int sel = m.t >= 0 ? (int)((s0 >> m.t) & 1ull) : 0;
        s[0] += (uint32_t)(int)m.pat[sel][j0];
        s[1] += (uint32_t)(int)m.pat[sel][j1];
    }
    return (s[0] & 0xffu) | ((s[1] & 0xffu) << 8);
}
__device__ __forceinline__ void a_epi_apply(const AEpilogue &e, uint64_t s0, uint32_t (&nc)[16]) {
    const uint32_t acc = a_epi_scalar(e, s0);
    uint32_t sh[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) sh[j] = acc + (uint32_t)(int)e.base[j];
#pragma unroll 1
    for (int g = 0; g < e.nmixed; ++g) {
        const AEpiMixed &m = e.m[g];
        if ((s0 & m.cext) != m.cext) continue;
        const int sel = m.t >= 0 ? (int)((s0 >> m.t) & 1ull) : 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) sh[j] += (uint32_t)(int)m.pat[sel][j];
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) nc[j] = shift_b1_fast(nc[j], (sh[j] & 0xffu) << 8);
}

// Pairs whose fp32 decision failed go to a per-warp queue; the fp64 reference
// (AGlob: the same arithmetic as a_decode / a_gate2 / a_encode) recomputes
// them 32 at a time, one pair per lane, after their units' provisional
// stores -- instead of stalling the whole warp for every unit with a failing
// pair.  Entry: the pair's first code index i0 (bit 63: the gate applies),
// the input codes (c0 | c1 << 16); the second code is at i0 + 2^t; the
// epilogue's b1 steps of the two codes (sh0 | sh1 << 8).
struct AFail {
    uint64_t i0;
    uint32_t codes, sh;
};
constexpr int A_QN = 32;
template <int UK, bool LAZY>
__device__ __noinline__ void a_flush(const AGateParams *pp, const ATabData *cur, const ATabData *nxt,
                                     const AFail *q, int n) {
    __syncwarp();  // the queued units' provisional stores and the entries are visible
    const int lane = threadIdx.x & 31;
    if (lane < n) {
        AGlob g;
        g.init(cur, nxt);
        const AFail e = q[lane];
        const uint64_t i0 = e.i0 & ~(1ull << 63);
        double2 x = g.decode(e.codes & 0xffffu), y = g.decode(e.codes >> 16);
        if (e.i0 >> 63) {
            double u[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) u[i] = pp->u[i];
            a_gate2u<UK>(u, x, y);
        }
        if (LAZY) {  // reading R-A25: outside [r0 - d, r1 + d] -> the gate rescales
            const double r0 = __ldg(&cur->r0), r1 = __ldg(&cur->r1), d = (r1 - r0) / 253.0;
            const double lo = r0 - d, hi = r1 + d;
            const double mx = a_m2(x), my = a_m2(y);
            const bool ox = is_inter(mx) && (mx < (lo > 0.0 ? lo * lo : 0.0) || mx > hi * hi);
            const bool oy = is_inter(my) && (my < (lo > 0.0 ? lo * lo : 0.0) || my > hi * hi);
            if (ox || oy) atomicOr(pp->oor, 1);
        }
        uint16_t *a = reinterpret_cast<uint16_t *>(pp->aout ? pp->aout : pp->a);
        a[i0] = (uint16_t)shift_b1_fast(g.encode(x), (e.sh & 0xffu) << 8);
        a[i0 + (1ull << pp->t)] = (uint16_t)shift_b1_fast(g.encode(y), e.sh & 0xff00u);
    }
    __syncwarp();  // the queue is free again
}

constexpr int A_DENSE_MINB = 2;  // CTAs per SM of the dense kernels (64 KiB of tables each)

// Phase 1 (reading R-A4): exact min / max of the intermediate |z'|^2 of the
// gate's output, through screens of increasing cost:
//  0. magnitudes only (fp32 table ra, rb): rigorous bounds on both outputs
//       hi = A max(ra, rb) + B min(ra, rb) >= |u_j0| ra + |u_j1| rb >= |z'_j|,
//       lo = min(|a ra - b rb|, |b ra - a rb|) - 3e-6 (ra + rb) <= |z'_j|
//     (reverse triangle inequality; a = |u00| ~ |u11|, b = |u01| ~ |u10| for
//     a unitary U, the margins cover fp32 rounding and the 1e-10 unitarity
//     tolerance); a pair passes when [lo, hi] lies inside the running
//     [min |z'|, max |z'|];
//  1. fp32 decode + gate + |z'| with the certified bound ||z'f| - |z'|| <=
//     sqrt2 E (E = A_KF (ra + rb) per component) and the fp32 rounding of
//     the magnitude (4e-7 relative): a pair passes when both outputs provably
//     lie inside the running [min, max] of the intermediate |z'| (and so are
//     intermediate themselves) or are certainly below 1e-12 (special zero);
//  2. otherwise (a new extreme, or a tie with one: the structured workload
//     states have massive exact ties at the extremes), the pair's class --
//     raw b0 of both codes, the b1 difference mod 256, whether the gate
//     applies -- is looked up in a per-warp cache; a class not found there
//     goes to a per-warp queue, evaluated in the same iteration, one class
//     per lane, updating the warp's exact min / max, which it shares with the
//     grid through two atomics (min / max of the fp64 bit patterns).
// The value of a class is |z'_j|^2 evaluated in fp64 in the frame of the
// first input: z'_j = u_j0 ra + u_j1 rb e^{i pi (b1b - b1a)/128} (reading
// R-A24: the gate output up to the common phase e^{i pi b1a/128}, which
// |.|^2 does not see; it differs from the per-amplitude fp64 evaluation by
// rounding only, ~1e-16 (ra + rb)).  So the bounds are a deterministic
// function of the set of classes present -- independent of the sharding and
// of the evaluation order -- and the structured workload states, with
// massive exact ties at the extremes, cost one evaluation per class.
// A pair that passes a screen provably lies inside [min, max] and is
// intermediate, so it cannot change the result.
__device__ unsigned long long g_abnd_dbg[5];  // debug: screen-1 candidates, screen-2 candidates, queued, flushes
struct ACand {
    uint32_t key;  // b0a | b0b << 8 | ((b1b - b1a) & 0xff) << 16 | sel << 24 (raw code bytes)
};
constexpr int A_BOUNDS_MINB = 3;
constexpr int A_DEDUP = 256;  // per-warp direct-mapped cache of queued class keys
template <int UK>
__device__ __forceinline__ void a_bounds_flush(const AGateParams &p, const ATabData *__restrict__ cur,
                                               const ACand *q, int n, double &mn, double &mx, float &tlo,
                                               float &thi, unsigned long long *gext) {
    __syncwarp();
    const int lane = threadIdx.x & 31;
    if (lane < n) {
        const uint32_t key = q[lane].key;
        const int b0a = (int)(key & 0xffu) ^ 0x80, b0b = (int)((key >> 8) & 0xffu) ^ 0x80;
        const int dl = (int)((key >> 16) & 0xffu) ^ 0x80;  // (b1b - b1a) as a table index
        const double ra = __ldg(&cur->r[b0a]), rb = __ldg(&cur->r[b0b]);
        double ma, mb;
        if (key >> 24) {
            const double yr = rb * __ldg(&cur->cth[dl]), yi = rb * __ldg(&cur->sth[dl]);
            // z'_0 = u00 ra + u01 y, z'_1 = u10 ra + u11 y (y = rb e^{i pi d / 128})
            const double x0r = fma(p.u[0], ra, fma(p.u[2], yr, -p.u[3] * yi));
            const double x0i = fma(p.u[1], ra, fma(p.u[2], yi, p.u[3] * yr));
            const double x1r = fma(p.u[4], ra, fma(p.u[6], yr, -p.u[7] * yi));
            const double x1i = fma(p.u[5], ra, fma(p.u[6], yi, p.u[7] * yr));
            ma = fma(x0r, x0r, x0i * x0i);
            mb = fma(x1r, x1r, x1i * x1i);
        } else {  // unselected: the inputs themselves
            ma = ra * ra;
            mb = rb * rb;
        }
        if (is_inter(ma)) {
            mn = fmin(mn, ma);
            mx = fmax(mx, ma);
        }
        if (is_inter(mb)) {
            mn = fmin(mn, mb);
            mx = fmax(mx, mb);
        }
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    // share with the grid: exact extremes found by other warps tighten this warp's
    // thresholds (non-negative doubles order like their bit patterns)
    if (lane == 0) {
        const unsigned long long omn = atomicMin(&gext[0], (unsigned long long)__double_as_longlong(mn));
        const unsigned long long omx =
            atomicMax(&gext[1], (unsigned long long)__double_as_longlong(mx > 0.0 ? mx : 0.0));
        mn = fmin(mn, __longlong_as_double((long long)omn));
        if (omx) mx = fmax(mx, __longlong_as_double((long long)omx));
    }
    mn = __shfl_sync(0xffffffffu, mn, 0);
    mx = __shfl_sync(0xffffffffu, mx, 0);
    // fp32 thresholds on |z|: tlo >= sqrt(mn), thi <= sqrt(mx) (directed roundings)
    tlo = mn == INFINITY ? INFINITY : __double2float_ru(__dsqrt_ru(mn));
    thi = mx == -INFINITY ? -INFINITY : __double2float_rd(__dsqrt_rd(mx));
    __syncwarp();
}

template <int TL, bool CTRL, int UK>
__global__ void __launch_bounds__(A_THREADS, A_BOUNDS_MINB) k_bounds_a(const __grid_constant__ AGateParams p,
                                                                       const ATabData *__restrict__ cur,
                                                                       const AFTab *__restrict__ fcur,
                                                                       double *partials, unsigned long long *gext) {
    using U = AUnit<TL>;
    const AFLane L = load_aflane(fcur);
    const int lane = threadIdx.x & 31;
    __shared__ ACand qall[A_THREADS / 32][A_QN];
    __shared__ uint32_t dall[A_THREADS / 32][A_DEDUP];
    ACand *q = qall[threadIdx.x >> 5];
    uint32_t *dd = dall[threadIdx.x >> 5];
    for (int i = lane; i < A_DEDUP; i += 32) dd[i] = ~0u;  // no key (keys < 2^25)
    __syncwarp();
    int qn = 0;  // warp-uniform
    const uint16_t *a = reinterpret_cast<const uint16_t *>(p.a);
    const uint64_t units = (p.nl >= 4) ? (1ull << (p.nl - 4)) : 1ull;
    const uint64_t lowm = (1ull << U::LOWB) - 1ull;
    const uint64_t chi = p.cmask & ~lowm;
    const uint32_t cl = (uint32_t)(p.cmask & lowm);
    float uf[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) uf[i] = p.uf[i];
    double mn = INFINITY, mx = -INFINITY;  // exact, warp-wide
    float tlo = INFINITY, thi = -INFINITY;
    const uint32_t lt = (1u << lane) - 1u;
    // the next unit's codes are loaded one iteration ahead (the loop is latency-bound
    // on its loads otherwise: few warps per scheduler, a dependent chain per unit)
    const uint64_t stride = (uint64_t)gridDim.x * A_THREADS;
    uint4 w0 = make_uint4(0, 0, 0, 0), w1 = w0;
    {
        const uint64_t v = (uint64_t)blockIdx.x * A_THREADS + threadIdx.x;
        if (v < units) U::load_raw(a, U::s0(v, p.t), p.t, w0, w1);
    }
    for (uint64_t vb = (uint64_t)blockIdx.x * A_THREADS + (threadIdx.x & ~31u); vb < units; vb += stride) {
        const uint64_t v = vb + (uint64_t)lane;
        uint32_t c[16], keys[8];
        uint32_t candm = 0;
        if (v < units) {
            const uint64_t s0 = U::s0(v, p.t);
            U::unpack(w0, w1, c);
            if (v + stride < units) U::load_raw(a, U::s0(v + stride, p.t), p.t, w0, w1);
            const bool hi_ok = !CTRL || (((p.shard_base | s0) & chi) == chi);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int j0 = U::j0(k), j1 = U::j1(k);
                const int off = TL < 4 ? j0 : k;
                const bool sel = !CTRL || (hi_ok && ((uint32_t)off & cl) == cl);
                const float ra = L.mag(c[j0]), rb = L.mag(c[j1]);
                const float S = ra + rb;
                const float eS = 1.4145e-6f * S;
                // screen 0, magnitudes only: hi >= |z'_j| >= lo for both outputs
                float hi, lo;
                if (!CTRL || sel) {
                    hi = fmaf(p.mA, fmaxf(ra, rb), p.mB * fminf(ra, rb));
                    // (ma ra - mb rb, mb ra - ma rb) on one FFMA2
                    const float2 T = __ffma2_rn(make_float2(p.ma, p.mb), f2s(ra),
                                                __fmul2_rn(make_float2(-p.mb, -p.ma), f2s(rb)));
                    lo = fminf(fabsf(T.x), fabsf(T.y));
                } else {  // unselected: |z'| = (ra, rb); a zero code stays the exact zero special
                    hi = fmaxf(ra, rb);
                    lo = fminf(ra == 0.f ? INFINITY : ra, rb == 0.f ? INFINITY : rb);
                }
                bool cand = (S > 0.f) & ((fmaf(-3e-6f, S, lo) < tlo) | (hi > thi));
                if (cand) {  // screen 1, fp32 gate: |z'| within sqrt2 E of |z'f|, mf within 4e-7 mf
                    const float2 A = __fmul2_rn(f2s(ra), L.cs2(c[j0])), B = __fmul2_rn(f2s(rb), L.cs2(c[j1]));
                    float2 RE = make_float2(A.x, B.x), IM = make_float2(A.y, B.y);
                    if (sel) a_gate_f2<UK>(p.kf, A, B, RE, IM);
                    const float2 m2 = __ffma2_rn(RE, RE, __fmul2_rn(IM, IM));
                    // as a_encode_f2: mf = |z'f| for m2 >= 1e-37, else below 3.2e-19 (certainly zero)
                    const float2 mf2 = __fmul2_rn(
                        m2, make_float2(a_rsqrt(fmaxf(m2.x, 1e-37f)), a_rsqrt(fmaxf(m2.y, 1e-37f))));
                    const float mfx = mf2.x, mfy = mf2.y;
                    // a certainly-zero output (|z'| < 1e-12, reading R-A5) is no intermediate:
                    // not a min candidate (the A states of the workloads hold many amplitudes
                    // at the 1e-12 floor, whose products straddle it)
                    float lx = fmaf(mfx, 1.0000005f, eS) < 0.99999e-12f ? INFINITY : mfx;
                    float ly = fmaf(mfy, 1.0000005f, eS) < 0.99999e-12f ? INFINITY : mfy;
                    if (CTRL && !sel) {
                        lx = ra == 0.f ? INFINITY : lx;
                        ly = rb == 0.f ? INFINITY : ly;
                    }
                    cand = (fminf(lx, ly) * 0.9999995f < tlo + eS) | (fmaxf(mfx, mfy) * 1.0000005f > thi - eS);
                }
#ifdef QSIM_ABND_DEBUG
                if (cand) atomicAdd(&g_abnd_dbg[1], 1ull);
#endif
                if (cand) {  // one evaluation per class: a class in the warp's cache is done
                    const uint32_t ca = c[j0], cb = c[j1];
                    const uint32_t key = (ca & 0xffu) | ((cb & 0xffu) << 8) |
                                         ((((cb >> 8) - (ca >> 8)) & 0xffu) << 16) | ((uint32_t)sel << 24);
                    const uint32_t slot = (key * 2654435761u) >> 24;
                    if (dd[slot] != key) {
                        dd[slot] = key;
                        candm |= 1u << k;
                        keys[k] = key;
                    }
                }
            }
        }
        if (__any_sync(0xffffffffu, candm != 0)) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const bool f = (candm >> k) & 1u;
                const uint32_t key = keys[k];
                const uint32_t bal = __ballot_sync(0xffffffffu, f);
                if (bal) {
                    const int tot = __popc(bal);
                    if (qn + tot > A_QN) {
                        a_bounds_flush<UK>(p, cur, q, qn, mn, mx, tlo, thi, gext);
                        qn = 0;
                    }
                    if (f) {
#ifdef QSIM_ABND_DEBUG
                        atomicAdd(&g_abnd_dbg[2], 1ull);
#endif
                        q[qn + __popc(bal & lt)].key = key;
                    }
                    qn += tot;
                }
            }
            // evaluate now: the thresholds must follow (a class found in the cache is not
            // queued again, so waiting for a full queue would leave them stale)
            if (qn) {
                a_bounds_flush<UK>(p, cur, q, qn, mn, mx, tlo, thi, gext);
                qn = 0;
            }
        }
    }
    if (qn) a_bounds_flush<UK>(p, cur, q, qn, mn, mx, tlo, thi, gext);
    __shared__ double red[2][A_THREADS / 32];
    if (lane == 0) {
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
__global__ void k_tables_next(const double *acc, ATabData *t, AFTab *f) {
    const double mn = acc[0], mx = -acc[1];
    const bool none = !(mn <= mx);
    const double r0 = none ? 0.5 : __dsqrt_rn(mn), r1 = none ? 0.5 : __dsqrt_rn(mx);
    const double d = __dsub_rn(r1, r0);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        const int b0 = i - 128;
        const double ri =
            b0 == -128 ? 0.0 : b0 == 127 ? 1.0 : __dadd_rn(__ddiv_rn(__dmul_rn((double)(b0 + 127), d), 253.0), r0);
        t->r[i] = ri;
        const float rf = __double2float_rn(ri);  // fp32 copy (fill_ftab), one per lane
        float *row = f->rf[(i - 128) & 0xff];
        for (int l = 0; l < 32; ++l) row[l] = rf;
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

// 64 KiB of dynamic shared memory (the fp32 tables): opted in once per device
// and kernel instantiation
static bool a_dense_attr(const void *kern, std::atomic<uint64_t> &devs) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (devs.load() & bit) return true;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(AFTab)) != cudaSuccess)
        return false;
    devs.fetch_or(bit);
    return true;
}

template <int TL, bool CTRL, int UK>
static void launch_bounds_tl(const AGateParams &p, const ATables *t, double *partials, int grid, cudaStream_t s) {
    static std::atomic<uint64_t> attr{0};
    a_dense_attr((const void *)k_bounds_a<TL, CTRL, UK>, attr);
    k_bounds_a<TL, CTRL, UK><<<grid, A_THREADS, sizeof(AFTab), s>>>(p, tcur(t), fcur(t), partials, t->gext);
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
// fp32 copy of U and the magnitude coefficients of the bounds screen
static int a_ukind(const double *u);
static AGateParams a_dense_params(const AGateParams &p0) {
    AGateParams p = p0;
    for (int i = 0; i < 8; ++i) p.uf[i] = (float)p.u[i];
    {  // a_gate_f2's coefficient pairs
        const float *u = p.uf;
        float *k = p.kf;
        switch (a_ukind(p.u)) {
            case 1: {
                const float v[8] = {u[0], u[4], 0.f, 0.f, u[2], u[6], 0.f, 0.f};
                for (int i = 0; i < 8; ++i) k[i] = v[i];
                break;
            }
            case 2: {
                const float v[8] = {u[0], -u[5], -u[3], u[6], u[0], u[5], u[3], u[6]};
                for (int i = 0; i < 8; ++i) k[i] = v[i];
                break;
            }
            default: {
                const float v[16] = {u[0], u[4], -u[1], -u[5], u[2], u[6], -u[3], -u[7],
                                     u[1], u[5], u[0], u[4], u[3], u[7], u[2], u[6]};
                for (int i = 0; i < 16; ++i) k[i] = v[i];
            }
        }
    }
    const double m00 = std::hypot(p.u[0], p.u[1]), m01 = std::hypot(p.u[2], p.u[3]);
    const double m10 = std::hypot(p.u[4], p.u[5]), m11 = std::hypot(p.u[6], p.u[7]);
    const double A = std::max(m00, m11) * (1.0 + 1e-6), B = std::max(m01, m10) * (1.0 + 1e-6);
    p.mA = (float)std::max(A, B);
    p.mB = (float)std::min(A, B);
    p.ma = (float)m00;
    p.mb = (float)m01;
    return p;
}
// persistent grid: MINB CTAs per SM (capped by the work and by the partials' capacity)
static int a_dense_grid(uint64_t units, int minb = A_DENSE_MINB) {
    const uint64_t cap = (uint64_t)a_num_sms() * minb;
    const uint64_t need = (units + A_THREADS - 1) / A_THREADS;
    return (int)(need < cap ? (need ? need : 1) : cap);
}

void a_bounds_debug_print() {
#ifdef QSIM_ABND_DEBUG
    unsigned long long h[4];
    cudaMemcpyFromSymbol(h, g_abnd_dbg, sizeof(h));
    fprintf(stderr, "abnd: min-cands %llu cands %llu queued %llu tiny(<1e-3 S) %llu\n", h[0], h[1], h[2], h[3]);
    unsigned long long z[5] = {0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_abnd_dbg, z, sizeof(z));
#endif
}
void launch_bounds_a(const AGateParams &p0, const ATables *t, double *partials, double *acc, bool first,
                     cudaStream_t s) {
    const AGateParams p = a_dense_params(p0);
    if (first) {  // the gate's running extremes shared by the grid: (+inf, 0) as bit patterns
        static const unsigned long long init[2] = {0x7ff0000000000000ull, 0ull};
        cudaMemcpyAsync(t->gext, init, sizeof(init), cudaMemcpyHostToDevice, s);
    }
    const uint64_t units = (p.nl >= 4) ? (1ull << (p.nl - 4)) : 1ull;
    const int grid = a_dense_grid(units, A_BOUNDS_MINB);
    switch (a_ukind(p.u)) {
        case 1: launch_bounds_k<1>(p, t, partials, grid, s); break;
        case 2: launch_bounds_k<2>(p, t, partials, grid, s); break;
        default: launch_bounds_k<0>(p, t, partials, grid, s); break;
    }
    k_minmax_final<<<1, 32, 0, s>>>(partials, grid, acc, first ? 1 : 0);
}

void launch_tables_next(const double *acc, ATables *t, cudaStream_t s) {
    k_tables_next<<<1, 256, 0, s>>>(acc, t->d[1 - t->cur], t->f[1 - t->cur]);
}

// Phase 2: decode (current tables), apply, encode (next tables) -- fp32 with
// the certified fallback per failing pair (the warp queue, a_flush).  The
// grid-stride loop is warp-uniform (lanes past the end idle) so that the
// queue's votes see the whole warp.
// MODE 0: exact bounds, certified; 1: lazy (reading R-A25); 2: exact bounds, fp32 arithmetic (R-A26)
template <int TL, bool CTRL, int UK, int MODE>
__global__ void __launch_bounds__(A_THREADS, A_DENSE_MINB) k_apply_a(const __grid_constant__ AGateParams p,
                                                                     const ATabData *__restrict__ cur,
                                                                     const ATabData *__restrict__ nxt,
                                                                     const AFTab *__restrict__ fcur) {
    using U = AUnit<TL>;
    constexpr bool LAZY = MODE == 1, FAST = MODE == 2;
    const AFLane L = load_aflane(fcur);
    __shared__ AFail qall[A_THREADS / 32][A_QN];
    const int lane = threadIdx.x & 31;
    AFail *q = qall[threadIdx.x >> 5];
    int qn = 0;  // warp-uniform
    AEncF ce;
    ce.init(nxt);  // LAZY: nxt = cur (the kept bounds)
    uint16_t *a = reinterpret_cast<uint16_t *>(p.a);
    uint16_t *ao = reinterpret_cast<uint16_t *>(p.aout ? p.aout : p.a);
    bool oor_any = false;
    const uint64_t units = (p.nl >= 4) ? (1ull << (p.nl - 4)) : 1ull;
    const uint64_t lowm = (1ull << U::LOWB) - 1ull;
    const uint64_t chi = p.cmask & ~lowm;
    const uint32_t cl = (uint32_t)(p.cmask & lowm);
    float uf[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) uf[i] = p.uf[i];
    const uint32_t lt = (1u << lane) - 1u;
    // the next unit's codes are loaded one iteration ahead (as in k_bounds_a)
    const uint64_t stride = (uint64_t)gridDim.x * A_THREADS;
    uint4 w0 = make_uint4(0, 0, 0, 0), w1 = w0;
    {
        const uint64_t v = (uint64_t)blockIdx.x * A_THREADS + threadIdx.x;
        if (v < units) U::load_raw(a, U::s0(v, p.t), p.t, w0, w1);
    }
    for (uint64_t vb = (uint64_t)blockIdx.x * A_THREADS + (threadIdx.x & ~31u); vb < units; vb += stride) {
        if (LAZY) {  // an output left the kept range somewhere: this pass is discarded, stop early
            int f = lane == 0 ? *reinterpret_cast<volatile int32_t *>(p.oor) : 0;
            if (__shfl_sync(0xffffffffu, f, 0)) break;
        }
        const uint64_t v = vb + (uint64_t)lane;
        uint32_t fail = 0, selm = 0;
        uint32_t c[16];
        uint64_t s0 = 0;
        if (v < units) {
            s0 = U::s0(v, p.t);
            U::unpack(w0, w1, c);
            if (v + stride < units) U::load_raw(a, U::s0(v + stride, p.t), p.t, w0, w1);
            const bool hi_ok = !CTRL || (((p.shard_base | s0) & chi) == chi);
            uint32_t nc[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int j0 = U::j0(k), j1 = U::j1(k);
                const int off = TL < 4 ? j0 : k;
                const bool sel = !CTRL || (hi_ok && ((uint32_t)off & cl) == cl);
                selm |= (uint32_t)sel << k;
                float ra, rb;
#ifdef QSIM_A_SCALAR_ENCODE
                float2 x = L.decode(c[j0], ra), y = L.decode(c[j1], rb);
                if (sel) a_gate_fu<UK>(uf, x, y);
#else
                const float2 A = L.decode2(c[j0], ra), B = L.decode2(c[j1], rb);
                float2 RE = make_float2(A.x, B.x), IM = make_float2(A.y, B.y);
                if (sel) a_gate_f2<UK>(p.kf, A, B, RE, IM);
#endif
                const float S = ra + rb;
                const float E = A_KF * S;
                const float errm = fmaf(S, ce.kS, fmaf(E, ce.kE, ce.C0)), KE = 73.f * E;
                const float eS = 1.4145f * E;
                bool okx, oky, ox = false, oy = false;
                uint32_t cx, cy;
#ifdef QSIM_A_SCALAR_ENCODE
                cx = a_encode_f<LAZY>(ce, x, errm, KE, eS, okx, ox);
                cy = a_encode_f<LAZY>(ce, y, errm, KE, eS, oky, oy);
#else
                a_encode_f2<LAZY, FAST>(ce, RE, IM, errm, KE, eS, cx, cy, okx, oky, ox, oy);
#endif
                if (LAZY) oor_any |= (ox & (!CTRL || sel)) | (oy & (!CTRL || sel));
                if (CTRL) {  // an unselected zero code stays the exact zero special
                    const bool zx = (ra == 0.f) & !sel, zy = (rb == 0.f) & !sel;
                    cx = zx ? 0x0080u : cx;
                    cy = zy ? 0x0080u : cy;
                    okx |= zx;
                    oky |= zy;
                }
                // |z'| <= ra + rb < 0.999: never the special one; else fp64 decides
                const bool ok = okx & oky & (S < 0.999f);
                nc[j0] = cx;
                nc[j1] = cy;
                fail |= (uint32_t)!ok << k;
            }
            if (p.has_epi) a_epi_apply(p.epi, s0, nc);
            U::store(ao, s0, p.t, nc);  // provisional for the failing pairs
        }
        if (LAZY && __any_sync(0xffffffffu, oor_any)) {
            if (lane == 0) atomicOr(p.oor, 1);
            break;
        }
        if (__any_sync(0xffffffffu, fail != 0)) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const bool f = (fail >> k) & 1u;
                const uint32_t bal = __ballot_sync(0xffffffffu, f);
                if (bal) {
                    const int tot = __popc(bal);
                    if (qn + tot > A_QN) {
                        a_flush<UK, LAZY>(&p, cur, nxt, q, qn);
                        qn = 0;
                    }
                    if (f) {
                        AFail e;
                        e.i0 = U::pos(s0, p.t, U::j0(k)) | ((uint64_t)((selm >> k) & 1u) << 63);
                        e.codes = __byte_perm(c[U::j0(k)], c[U::j1(k)], 0x5410);
                        e.sh = 0;
                        if (p.has_epi) e.sh = a_epi_pair(&p.epi, s0, U::j0(k), U::j1(k));
                        q[qn + __popc(bal & lt)] = e;
                    }
                    qn += tot;
                }
            }
        }
    }
    if (qn) a_flush<UK, LAZY>(&p, cur, nxt, q, qn);
}

template <int TL, bool CTRL, int UK, int MODE>
static void launch_apply_tl(const AGateParams &p, const ATables *t, int grid, cudaStream_t s) {
    static std::atomic<uint64_t> attr{0};
    a_dense_attr((const void *)k_apply_a<TL, CTRL, UK, MODE>, attr);
    // LAZY: encode with the current tables (the kept bounds)
    k_apply_a<TL, CTRL, UK, MODE><<<grid, A_THREADS, sizeof(AFTab), s>>>(p, tcur(t), MODE == 1 ? tcur(t) : tnext(t),
                                                                         fcur(t));
}
template <int TL, int UK, int MODE>
static void launch_apply_c(const AGateParams &p, const ATables *t, int grid, cudaStream_t s) {
    if (p.cmask)
        launch_apply_tl<TL, true, UK, MODE>(p, t, grid, s);
    else
        launch_apply_tl<TL, false, UK, MODE>(p, t, grid, s);
}
template <int UK, int MODE>
static void launch_apply_k(const AGateParams &p, const ATables *t, int grid, cudaStream_t s) {
    switch (p.t < 4 ? p.t : 4) {
        case 0: launch_apply_c<0, UK, MODE>(p, t, grid, s); break;
        case 1: launch_apply_c<1, UK, MODE>(p, t, grid, s); break;
        case 2: launch_apply_c<2, UK, MODE>(p, t, grid, s); break;
        case 3: launch_apply_c<3, UK, MODE>(p, t, grid, s); break;
        default: launch_apply_c<4, UK, MODE>(p, t, grid, s); break;
    }
}
template <int MODE>
static void launch_apply_any(const AGateParams &p0, const ATables *t, cudaStream_t s) {
    const AGateParams p = a_dense_params(p0);
    const uint64_t units = (p.nl >= 4) ? (1ull << (p.nl - 4)) : 1ull;
    const int grid = a_dense_grid(units);
    switch (a_ukind(p.u)) {
        case 1: launch_apply_k<1, MODE>(p, t, grid, s); break;
        case 2: launch_apply_k<2, MODE>(p, t, grid, s); break;
        default: launch_apply_k<0, MODE>(p, t, grid, s); break;
    }
}
void launch_apply_a(const AGateParams &p, const ATables *t, cudaStream_t s) { launch_apply_any<0>(p, t, s); }
void launch_apply_a_fp32(const AGateParams &p, const ATables *t, cudaStream_t s) { launch_apply_any<2>(p, t, s); }
void launch_apply_a_lazy(const AGateParams &p, const ATables *t, cudaStream_t s) { launch_apply_any<1>(p, t, s); }

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
    // ANTI: units visited = units with every local control above the unit's own bits = 1:
    // unit index bits fixed to 1 (ascending positions), the visited count
    int32_t ins[2], nins;
    uint64_t nvis;
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

// Permutation gates move codes: only the units whose
// control bits above the unit's own code bits are all 1 are visited (those
// bits are inserted into the unit index, like the E sweep's control
// insertion); controls inside a unit are tested per pair.
template <bool LOWT>
__global__ void __launch_bounds__(A_THREADS) k_anti_a(const __grid_constant__ AFastParams p) {
    uint16_t *a = reinterpret_cast<uint16_t *>(p.a);
    for (uint64_t w = (uint64_t)blockIdx.x * A_THREADS + threadIdx.x; w < p.nvis; w += (uint64_t)gridDim.x * A_THREADS) {
        uint64_t u = w;
        for (int q = 0; q < p.nins; ++q) u = a_ins0(u, p.ins[q]) | (1ull << p.ins[q]);
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
        // local controls above the unit bits become fixed unit-index bits
        const bool lowt = g.t < 4;
        const int lowb = lowt ? 4 : 3;
        const uint64_t units = p.n >> 4;
        int ub[2], nu = 0;
        for (int b = lowb; b < g.nl && b < 64; ++b)
            if (b != g.t && ((g.cmask >> b) & 1ull)) ub[nu++] = lowt ? b - 4 : (b < g.t ? b - 3 : b - 4);
        p.nins = nu;
        for (int q = 0; q < nu; ++q) p.ins[q] = ub[q];  // ascending
        p.nvis = units >> nu;
        if (lowt)
            k_anti_a<true><<<a_grid(p.nvis), A_THREADS, 0, s>>>(p);
        else
            k_anti_a<false><<<a_grid(p.nvis), A_THREADS, 0, s>>>(p);
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
