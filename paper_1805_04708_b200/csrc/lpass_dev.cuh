// lpass_dev.cuh -- device code of the relabelling tile pass (lpass.h): the
// op semantics (exactly those of the host emulator tools/lpass_emu.cpp) and
// the kernel body.  Included by lpass.cu (the interpreter kernel) and, as
// source text, by the run-time specialised kernels NVRTC compiles (lpass.cu,
// lpass_jit_*): both run the same device functions.
#pragma once

#include "lpass_types.h"

namespace qsim {

__device__ __forceinline__ uint64_t lp_ins0(uint64_t w, int p) {
    return ((w >> p) << (p + 1)) | (w & ((1ull << p) - 1ull));
}
__device__ __forceinline__ uint32_t lp_par(uint32_t x) { return __popc(x) & 1u; }
__host__ __device__ constexpr int lp_ctz5(int i) { return (i & 1) ? 0 : (i & 2) ? 1 : (i & 4) ? 2 : (i & 8) ? 3 : 4; }
__host__ __device__ constexpr int lp_hibit(int v) { return v >= 16 ? 4 : v >= 8 ? 3 : v >= 4 ? 2 : v >= 2 ? 1 : 0; }

__device__ __forceinline__ void lp_cp_async16(void *smem, const void *gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void lp_cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
// bring a 128-byte run into L2 ahead of its cp.async (no completion to wait for)
__device__ __forceinline__ void lp_prefetch_l2_128(const void *gmem) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;\n" ::"l"(gmem) : "memory");
}

// 16-byte shared-memory access of one amplitude (register stages).  Explicit
// v2.f64: from C++ the compiler splits some stages' double2 accesses into two
// 8-byte halves (LDS.64 / STS.64 pairs, twice the wavefronts -- measured); the
// asm is volatile so it stays between the stage's __syncthreads.
#ifndef LP_STAGE_ASM
#define LP_STAGE_ASM 1
#endif
// LP_CHECK (QSIM_LPASS_CHECK=1, specialised kernels): bounds checks of every
// shared-memory and HBM address the pass forms -- tile slots, table and slot
// reads in the coefficient pool, the tile's runs in the shard; a violation
// prints and traps (the pool has no compute-sanitizer; PAPER-independent)
#ifndef LP_CHECK
#define LP_CHECK 0
#endif
#if LP_CHECK
#define LP_ASSERT(c)                                                                                       \
    do {                                                                                                   \
        if (!(c)) {                                                                                        \
            printf("lpass check failed: %s (block %d thread %d)\n", #c, (int)blockIdx.x, (int)threadIdx.x); \
            __trap();                                                                                      \
        }                                                                                                  \
    } while (0)
#else
#define LP_ASSERT(c) \
    do {             \
    } while (0)
#endif
#ifndef LP_PREFETCH
#define LP_PREFETCH 0  // L2 prefetch of the next tile (QSIM_LPASS_PREFETCH=1): measured slower, off
#endif
__device__ __forceinline__ double2 lp_lds16(uint32_t sa) {
#if LP_STAGE_ASM
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(sa));
    return v;
#else
    extern __shared__ __align__(16) unsigned char smem_raw[];
    return *reinterpret_cast<const double2 *>(smem_raw + (sa - (uint32_t)__cvta_generic_to_shared(smem_raw)));
#endif
}
__device__ __forceinline__ void lp_sts16(uint32_t sa, const double2 &v) {
#if LP_STAGE_ASM
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(sa), "d"(v.x), "d"(v.y));
#else
    extern __shared__ __align__(16) unsigned char smem_raw[];
    *reinterpret_cast<double2 *>(smem_raw + (sa - (uint32_t)__cvta_generic_to_shared(smem_raw))) = v;
#endif
}

// x' = x - t y, y' = y + t x  (2 FMAs per amplitude component)
__device__ __forceinline__ void lp_shear_pair(double2 &x, double2 &y, double t) {
    const double2 x0 = x;
    x.x = fma(-t, y.x, x.x);
    x.y = fma(-t, y.y, x.y);
    y.x = fma(t, x0.x, y.x);
    y.y = fma(t, x0.y, y.y);
}

template <int NS, int V>
__device__ __forceinline__ void lp_shearu(double2 (&v)[NS], double te) {
    constexpr int HB = lp_hibit(V);
#pragma unroll
    for (int j0 = 0; j0 < NS; ++j0) {
        if (j0 & (1 << HB)) continue;
        lp_shear_pair(v[j0], v[j0 ^ V], te);
    }
}
template <int NS, int V>
__device__ __forceinline__ void lp_shear(double2 (&v)[NS], double t, uint32_t pm, uint32_t gp) {
    constexpr int HB = lp_hibit(V);
    const uint32_t q = pm ^ (gp ? 0xffffffffu : 0u);
#pragma unroll
    for (int j0 = 0; j0 < NS; ++j0) {
        if (j0 & (1 << HB)) continue;
        const double te = ((q >> j0) & 1u) ? -t : t;
        lp_shear_pair(v[j0], v[j0 ^ V], te);
    }
}
// per-pair control predicate: all in-register controls of sigma(j0) are 1
__device__ __forceinline__ uint32_t lp_ctl_mask(const LOp &o, uint32_t g) {
    uint32_t m = 0xffffffffu;
    const int nc = o.nctl;
    if (nc > 0) m &= o.pmc[0] ^ (lp_par(o.rowc[0] & g) ? 0xffffffffu : 0u);
    if (nc > 1) m &= o.pmc[1] ^ (lp_par(o.rowc[1] & g) ? 0xffffffffu : 0u);
    return m;  // bit j0 = 1 iff the pair at j0 is selected
}
template <int NS, int V>
__device__ __forceinline__ void lp_cshear(double2 (&v)[NS], double t, uint32_t pm, uint32_t gp, uint32_t cm) {
    constexpr int HB = lp_hibit(V);
    const uint32_t q = pm ^ (gp ? 0xffffffffu : 0u);
#pragma unroll
    for (int j0 = 0; j0 < NS; ++j0) {
        if (j0 & (1 << HB)) continue;
        double te = ((q >> j0) & 1u) ? -t : t;
        te = ((cm >> j0) & 1u) ? te : 0.0;
        lp_shear_pair(v[j0], v[j0 ^ V], te);
    }
}
template <int NS, int V>
__device__ __forceinline__ void lp_dense(double2 (&v)[NS], const double2 *u, uint32_t pm, uint32_t gp, uint32_t cm) {
    constexpr int HB = lp_hibit(V);
    const uint32_t q = pm ^ (gp ? 0xffffffffu : 0u);
    const double2 a = u[0], b = u[1], c = u[2], d = u[3];
#pragma unroll
    for (int j0 = 0; j0 < NS; ++j0) {
        if (j0 & (1 << HB)) continue;
        if (!((cm >> j0) & 1u)) continue;
        // register j0 holds the logical-1 member when the bit is set: apply X U X
        const bool s = (q >> j0) & 1u;
        const double2 e00 = s ? d : a, e01 = s ? c : b, e10 = s ? b : c, e11 = s ? a : d;
        const double2 x = v[j0], y = v[j0 ^ V];
        v[j0] = make_double2(e00.x * x.x - e00.y * x.y + e01.x * y.x - e01.y * y.y,
                             e00.x * x.y + e00.y * x.x + e01.x * y.y + e01.y * y.x);
        v[j0 ^ V] = make_double2(e10.x * x.x - e10.y * x.y + e11.x * y.x - e11.y * y.y,
                                 e10.x * x.y + e10.y * x.x + e11.x * y.y + e11.y * y.x);
    }
}
template <int NS, int V>
__device__ __forceinline__ void lp_cswap(double2 (&v)[NS], uint32_t cm) {
    constexpr int HB = lp_hibit(V);
#pragma unroll
    for (int j0 = 0; j0 < NS; ++j0) {
        if (j0 & (1 << HB)) continue;
        const bool s = (cm >> j0) & 1u;
        const double2 x = v[j0], y = v[j0 ^ V];
        v[j0] = s ? y : x;
        v[j0 ^ V] = s ? x : y;
    }
}

struct LPSmem {
    size_t tile, cpool, total;
};
// tables sit right after the tile: both offsets are multiples of a table's
// size (2^R x 16 B), so entry j ^ g of a table is at (base + g*16) ^ (j*16)
__host__ __device__ inline LPSmem lp_smem(int K, int ncoef) {
    LPSmem L;
    L.tile = 0;
    L.cpool = ((size_t)1 << K) * 16;
    L.total = L.cpool + (size_t)((ncoef + 1) & ~1) * 8;
    return L;
}

// lifted shear on register bit r (L D U factorisation, D already applied by
// the table): logical x += a y; y += t x -- every FMA writes its own input
template <int NS, int RB, bool FLIP>
__device__ __forceinline__ void lp_lift(double2 (&v)[NS], double t, double a) {
    // all x updates first, then all y updates: dependent FMAs NS/2 apart
#pragma unroll
    for (int j0 = 0; j0 < NS; ++j0) {
        if (j0 & (1 << RB)) continue;
        double2 &x = FLIP ? v[j0 | (1 << RB)] : v[j0];
        const double2 &y = FLIP ? v[j0] : v[j0 | (1 << RB)];
        x.x = fma(a, y.x, x.x);
        x.y = fma(a, y.y, x.y);
    }
#pragma unroll
    for (int j0 = 0; j0 < NS; ++j0) {
        if (j0 & (1 << RB)) continue;
        const double2 &x = FLIP ? v[j0 | (1 << RB)] : v[j0];
        double2 &y = FLIP ? v[j0] : v[j0 | (1 << RB)];
        y.x = fma(t, x.x, y.x);
        y.y = fma(t, x.y, y.y);
    }
}

// v[j] *= T[j ^ g]; tb = byte offset of the table in shared memory + 16 g
template <int NS>
__device__ __forceinline__ void lp_table(double2 (&v)[NS], const unsigned char *smem, uint32_t tb) {
    // chunks of 8 entries: bounded register pressure, loads still ahead of the math
    constexpr int CH = NS < 8 ? NS : 8;
#pragma unroll
    for (int j0 = 0; j0 < NS; j0 += CH) {
        double2 c[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) c[j] = *reinterpret_cast<const double2 *>(smem + (tb ^ (uint32_t)((j0 + j) << 4)));
#pragma unroll
        for (int j = 0; j < CH; ++j) {
            const double p = c[j].y * v[j0 + j].y, q = c[j].y * v[j0 + j].x;
            v[j0 + j].x = fma(c[j].x, v[j0 + j].x, -p);
            v[j0 + j].y = fma(c[j].x, v[j0 + j].y, q);
        }
    }
}

// tile load (cp.async) / store of the NJ = 2^(K-7) elements of this thread:
// logical x = tid + NT j, j in Gray-code order (one column changes per step)
// (slim, glo, ghi: the tile's shared-memory bytes and the shard's byte range, LP_CHECK only)
template <int NJ>
__device__ __forceinline__ void lp_tile_load(unsigned char *smem, const char *gp, uint32_t so, const uint32_t *s_hi,
                                             const uint64_t *d_hi, uint32_t slim = 0, const char *glo = nullptr,
                                             const char *ghi = nullptr) {
    uint64_t dj = 0;
#pragma unroll
    for (int i = 0; i < NJ; ++i) {
        if (i) {
            so ^= s_hi[lp_ctz5(i)];
            dj ^= d_hi[lp_ctz5(i)];
        }
        LP_ASSERT(so + 16u <= slim && gp + dj >= glo && gp + dj + 16 <= ghi);
        lp_cp_async16(smem + so, gp + dj);
    }
}
template <int NJ>
__device__ __forceinline__ void lp_tile_store(const unsigned char *smem, char *gp, uint32_t mo, const uint32_t *m_hi,
                                              const uint64_t *d_hi, uint32_t slim = 0, const char *glo = nullptr,
                                              const char *ghi = nullptr) {
    uint64_t dj = 0;
#pragma unroll
    for (int i = 0; i < NJ; ++i) {
        if (i) {
            mo ^= m_hi[lp_ctz5(i)];
            dj ^= d_hi[lp_ctz5(i)];
        }
        LP_ASSERT(mo + 16u <= slim && gp + dj >= glo && gp + dj + 16 <= ghi);
        *reinterpret_cast<double2 *>(gp + dj) = *reinterpret_cast<const double2 *>(smem + mo);
    }
}
// the same, every amplitude times the tile scalar c (LPassParams::nts)
template <int NJ>
__device__ __forceinline__ void lp_tile_store_scaled(const unsigned char *smem, char *gp, uint32_t mo,
                                                     const uint32_t *m_hi, const uint64_t *d_hi, double2 c,
                                                     uint32_t slim = 0, const char *glo = nullptr,
                                                     const char *ghi = nullptr) {
    uint64_t dj = 0;
#pragma unroll
    for (int i = 0; i < NJ; ++i) {
        if (i) {
            mo ^= m_hi[lp_ctz5(i)];
            dj ^= d_hi[lp_ctz5(i)];
        }
        LP_ASSERT(mo + 16u <= slim && gp + dj >= glo && gp + dj + 16 <= ghi);
        const double2 v = *reinterpret_cast<const double2 *>(smem + mo);
        const double pp = c.y * v.y, qq = c.y * v.x;
        *reinterpret_cast<double2 *>(gp + dj) = make_double2(fma(c.x, v.x, -pp), fma(c.x, v.y, qq));
    }
}

// table variant offset (bytes in shared memory) of a group: the group's
// values of up to 2 condition bits select among the op's consecutive tables
template <int R>
__device__ __forceinline__ uint32_t lp_toff(uint64_t h, const LOp &o, uint32_t xq, uint64_t full, uint32_t cpool_off) {
    uint32_t toff = cpool_off + (uint32_t)((h >> 32) & 0xffffu) * 8u;
    const uint32_t nv = (uint32_t)(h >> 48) & 0xffu;
    if (nv) {
#pragma unroll
        for (int i = 0; i < 2; ++i)
            if (i < (int)nv) {
                const uint32_t c = o.rowc[i];
                const uint32_t bit = c < 64 ? (xq >> c) & 1u : (uint32_t)(full >> (c - 64)) & 1u;
                toff += bit << (i + R + 4);
            }
    }
    return toff;
}

// flips folded into a table op (compiler): g ^= gvec where the condition bit is 1
__device__ __forceinline__ void lp_preflip(uint32_t &g, const LOp &o, uint32_t xq, uint64_t full) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const uint32_t f = o.pmc[k];
        if (!(f >> 16)) break;
        const uint32_t c = (f >> 8) & 255u;
        const uint32_t bit = c == 255u ? 1u : c < 64u ? (xq >> c) & 1u : (uint32_t)(full >> (c - 64u)) & 1u;
        g ^= bit ? (f & 255u) : 0u;
    }
}

// the lifted shears of a ROUND op on the register bits in mask (ascending),
// coefficients (t, a) pairs at sp
template <int R>
__device__ __forceinline__ void lp_lifts(double2 (&v)[1 << R], uint32_t g, uint32_t mask, const double *sp) {
    constexpr int NS = 1 << R;
    int k = 0;
#define LP_ROUND_BIT(RB)                                                          \
    if constexpr ((RB) < R) {                                                     \
        if ((mask >> (RB)) & 1u) {                                                \
            const double t = sp[2 * k], aa = sp[2 * k + 1];                       \
            ++k;                                                                  \
            if ((g >> (RB)) & 1u)                                                 \
                lp_lift<NS, ((RB) < R ? (RB) : 0), true>(v, t, aa);               \
            else                                                                  \
                lp_lift<NS, ((RB) < R ? (RB) : 0), false>(v, t, aa);              \
        }                                                                         \
    }
    LP_ROUND_BIT(0) LP_ROUND_BIT(1) LP_ROUND_BIT(2) LP_ROUND_BIT(3) LP_ROUND_BIT(4)
#undef LP_ROUND_BIT
}

// One op of the stage program on one register group (v, g: its register
// values and flip vector; xq: its logical tile bits outside the registers).
template <int R>
__device__ __forceinline__ void lp_op1(double2 (&v)[1 << R], uint32_t &g, uint32_t xq, uint64_t full, uint64_t h,
                                       const LOp &o, const LPassParams &p, const unsigned char *smem_raw,
                                       uint32_t cpool_off) {
    constexpr int NS = 1 << R;
    const uint32_t code = (uint32_t)h & 0xffu;
    const uint32_t coef = (uint32_t)(h >> 32) & 0xffffu;
    if ((h >> 8) & LF_COND) {
        if (((xq & o.tmask) != o.tval) || ((full & o.omask) != o.oval)) return;
    }
    if (code == LOP_CODE_ROUND || code == LOP_CODE_DIAGT) lp_preflip(g, o, xq, full);
    const uint32_t toff = lp_toff<R>(h, o, xq, full, cpool_off);
    LP_ASSERT(!(code == LOP_CODE_ROUND || code == LOP_CODE_DIAGT) ||
              (toff >= cpool_off && toff + (uint32_t)NS * 16u <= cpool_off + (uint32_t)p.ncoef * 8u));
    if (code == LOP_CODE_ROUND) {
        lp_table<NS>(v, smem_raw, toff | (g << 4));
        lp_lifts<R>(v, g, (uint32_t)(h >> 24) & 0xffu, p.sc + o.pm);
        return;
    }
    if (code == LOP_CODE_DIAGT) {
        lp_table<NS>(v, smem_raw, toff | (g << 4));
        return;
    }
    if (code == LOP_CODE_FLIP) {
        g ^= (uint32_t)(h >> 24) & 0xffu;
        return;
    }
    if (code == LOP_CODE_PHASES) {
        const double *T = p.sc + coef;
        const int nt = (int)((h >> 48) & 0xffu);
        double cr = 1.0, ci = 0.0;
        const int nf = (int)o.pmc[1];  // leading full-index-bit terms: this tile's product (lp_body)
        if (nf) {
            LP_ASSERT(o.pmc[0] * 8u + 16u <= (uint32_t)p.ncoef * 8u && nf <= nt);
            const double2 c = *reinterpret_cast<const double2 *>(smem_raw + cpool_off + o.pmc[0] * 8u);
            cr = c.x;
            ci = c.y;
        }
        for (int k = nf; k < nt; ++k) {
            const int c = (int)T[3 * k];
            const uint32_t bit = c < 64 ? (xq >> c) & 1u : (uint32_t)(full >> (c - 64)) & 1u;
            if (bit) {
                const double er = T[3 * k + 1], ei = T[3 * k + 2];
                const double nr = fma(cr, er, -ci * ei);
                ci = fma(cr, ei, ci * er);
                cr = nr;
            }
        }
        const uint32_t gp = lp_par(((uint32_t)(h >> 16) & 0xffu) & g);
        const uint32_t want = gp ? 0u : 1u;
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            if (((o.pm >> j) & 1u) != want) continue;
            const double pp = ci * v[j].y, qq = ci * v[j].x;
            v[j].x = fma(cr, v[j].x, -pp);
            v[j].y = fma(cr, v[j].y, qq);
        }
        return;
    }
    if (code == LOP_CODE_DIAG1) {
        const uint32_t gp = lp_par(((uint32_t)(h >> 16) & 0xffu) & g);
        const double *T = p.sc + coef;
        const double t0r = T[0], t0i = T[1], t1r = T[2], t1i = T[3];
        if ((h >> 24) & 1u) {  // T0 == 1: multiply the half with b = 1 only (uniform branch on gp)
            const uint32_t want = gp ? 0u : 1u;
#pragma unroll
            for (int j = 0; j < NS; ++j) {
                if (((o.pm >> j) & 1u) != want) continue;
                const double pp = t1i * v[j].y, qq = t1i * v[j].x;
                v[j].x = fma(t1r, v[j].x, -pp);
                v[j].y = fma(t1r, v[j].y, qq);
            }
            return;
        }
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            const bool b = (((o.pm >> j) & 1u) ^ gp) != 0;
            const double cr = b ? t1r : t0r, ci = b ? t1i : t0i;
            const double pp = ci * v[j].y, qq = ci * v[j].x;
            v[j].x = fma(cr, v[j].x, -pp);
            v[j].y = fma(cr, v[j].y, qq);
        }
        return;
    }
    const uint32_t gp = lp_par(((uint32_t)(h >> 16) & 0xffu) & g);
    switch (code) {
#define LP_V_CASES(VS)                                                                                    \
    case LOP_SHEARU * 16 + (VS):                                                                          \
        if constexpr ((VS) < lp_nv(R)) {                                                                  \
            const double t = p.sc[coef];                                                                  \
            lp_shearu<NS, lp_vec(R, (VS))>(v, ((o.pm ^ gp) & 1u) ? -t : t);                               \
        }                                                                                                 \
        break;                                                                                            \
    case LOP_SHEAR * 16 + (VS):                                                                           \
        if constexpr ((VS) < lp_nv(R)) lp_shear<NS, lp_vec(R, (VS))>(v, p.sc[coef], o.pm, gp);             \
        break;
#define LP_W1_CASES(VS)                                                                                   \
    case LOP_CSHEAR * 16 + (VS):                                                                          \
        if constexpr ((VS) < R) lp_cshear<NS, (1 << (VS))>(v, p.sc[coef], o.pm, gp, lp_ctl_mask(o, g));    \
        break;                                                                                            \
    case LOP_DENSE * 16 + (VS):                                                                           \
        if constexpr ((VS) < R)                                                                           \
            lp_dense<NS, (1 << (VS))>(v, reinterpret_cast<const double2 *>(p.sc + coef), o.pm, gp,        \
                      lp_ctl_mask(o, g));                                                 \
        break;                                                                                            \
    case LOP_CSWAP * 16 + (VS):                                                                           \
        if constexpr ((VS) < R) lp_cswap<NS, (1 << (VS))>(v, lp_ctl_mask(o, g));                          \
        break;
        LP_V_CASES(0) LP_V_CASES(1) LP_V_CASES(2) LP_V_CASES(3) LP_V_CASES(4)
        LP_V_CASES(5) LP_V_CASES(6) LP_V_CASES(7) LP_V_CASES(8) LP_V_CASES(9)
        LP_V_CASES(10) LP_V_CASES(11) LP_V_CASES(12) LP_V_CASES(13) LP_V_CASES(14)
        LP_W1_CASES(0) LP_W1_CASES(1) LP_W1_CASES(2) LP_W1_CASES(3) LP_W1_CASES(4)
#undef LP_V_CASES
#undef LP_W1_CASES
        default:
            break;
    }
}

// Per-tile context of the stage loop.
struct LpTile {
    unsigned char *smem_raw;
    uint64_t full;    // full physical index of the tile's base
    uint32_t fired;   // events of this tile
    uint32_t cpool_off;
};

// One register stage: every group of 2^R amplitudes (a coset of the stage's
// register basis) is loaded from shared memory, `ops(v, g, xq, full, p,
// smem, cpool_off)` applies the stage's ops, and it is stored back.  KK: the
// tile width when known at compile time (0: p.K); NT: threads per CTA.
template <int R, int KK, class Ops, int NT = LP_THREADS, int G = 1>
__device__ __forceinline__ void lp_stage(const LPassParams &p, const LpTile &t, const LStage &st, const Ops &ops) {
    constexpr int NS = 1 << R;
    const int K = KK ? KK : p.K;
    constexpr int TB = NT == 256 ? 8 : 7;  // group bits held by the thread index
    const uint32_t tid = threadIdx.x;
    const uint32_t ngroups = 1u << (K - R);
    unsigned char *smem_raw = t.smem_raw;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
    uint32_t y = st.y_static;
    // static event indices (a literal stage keeps only its events, no indexed array)
#pragma unroll
    for (int e = 0; e < LP_MAX_EVENTS; ++e)
        if ((st.ev_mask >> e) & 1u)
            if ((t.fired >> e) & 1u) y ^= st.y_ev[e];
    uint32_t g0 = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) g0 |= ((y >> st.qbit[r]) & 1u) << r;
    const uint32_t yrest = y & ~(uint32_t)st.qmask;
    uint32_t rp[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rp[r] = (uint32_t)st.reg_phys[r] << 4;
    const bool nxq = st.needs_xq;
    // group bits 0..TB-1 = this thread's index: their address / logical parts
    // once per stage; bits >= TB per group below
    uint32_t a0t = 0, xqt = yrest;
#pragma unroll
    for (int i = 0; i < TB; ++i)
        if (i < K - R && ((tid >> i) & 1u)) {
            a0t ^= (uint32_t)st.grp_phys[i] << 4;
            xqt ^= st.grp_log[i];
        }
    if constexpr (G == 2) {
        // two register groups per thread, every op applied to both (independent
        // work for the scheduler to interleave); needs ngroups == 2 NT
        uint32_t a0[2], xq[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            a0[k] = a0t;
            xq[k] = nxq ? xqt : yrest;
            if (k) {
                a0[k] ^= (uint32_t)st.grp_phys[TB] << 4;
                if (nxq) xq[k] ^= st.grp_log[TB];
            }
        }
        double2 v0[NS], v1[NS];
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            uint32_t ad = 0;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (j & (1 << r)) ad ^= rp[r];
            LP_ASSERT((a0[0] ^ ad) + 16u <= (16u << K) && (a0[1] ^ ad) + 16u <= (16u << K));
            v0[j] = lp_lds16(sbase + (a0[0] ^ ad));
            v1[j] = lp_lds16(sbase + (a0[1] ^ ad));
        }
        uint32_t g_0 = g0, g_1 = g0;
        ops(v0, g_0, xq[0], t.full, p, smem_raw, t.cpool_off);
        ops(v1, g_1, xq[1], t.full, p, smem_raw, t.cpool_off);
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            uint32_t ad = 0;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (j & (1 << r)) ad ^= rp[r];
            lp_sts16(sbase + (a0[0] ^ ad), v0[j]);
            lp_sts16(sbase + (a0[1] ^ ad), v1[j]);
        }
        __syncthreads();
        return;
    }
    for (uint32_t grp = tid; grp < ngroups; grp += NT) {
        uint32_t a0 = a0t, xq = nxq ? xqt : yrest;
        for (int i = TB; i < K - R; ++i)
            if ((grp >> i) & 1u) {
                a0 ^= (uint32_t)st.grp_phys[i] << 4;
                if (nxq) xq ^= st.grp_log[i];
            }
        double2 v[NS];
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            uint32_t ad = a0;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (j & (1 << r)) ad ^= rp[r];
            LP_ASSERT(ad + 16u <= (16u << K));
            v[j] = lp_lds16(sbase + ad);
        }
        uint32_t g = g0;
        ops(v, g, xq, t.full, p, smem_raw, t.cpool_off);
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            uint32_t ad = a0;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (j & (1 << r)) ad ^= rp[r];
            lp_sts16(sbase + ad, v[j]);
        }
    }
    __syncthreads();
}

// The pass kernel body.  `stages(t)` runs the register stages of one tile
// (lp_stage per stage): the interpreter (lpass.cu) walks p.st / p.op, a
// run-time specialised kernel (NVRTC) calls lp_stage with literal stages and
// ops.  Everything else -- tile load / store, addressing -- is this code.
template <int R, int KK, class Stages, int NT = LP_THREADS>
__device__ __forceinline__ void lp_body(const LPassParams &p, const Stages &stages) {
    constexpr int TB = NT == 256 ? 8 : 7;  // tile bits held by the thread index
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int K = KK ? KK : p.K;
    const LPSmem L = lp_smem(K, p.ncoef);
    double *cpool = reinterpret_cast<double *>(smem_raw + L.cpool);
    const uint32_t tid = threadIdx.x;
    // ---- one-time setup per CTA ----
    for (int i = tid; i < p.ncoef; i += NT) cpool[i] = p.coef[i];
    // load / store addressing: logical x = tid + NT j; smem byte offset of x
    // at load = XOR of scol over its bits (store: smcol, plus S b); HBM offset
    // = deposit of its bits.  Bits 0..TB-1 are this thread's, the rest come from j.
    uint32_t s_tid = 0, m_tid = 0;
    uint64_t d_tid = tid & 7u;
#pragma unroll
    for (int i = 0; i < TB; ++i)
        if ((tid >> i) & 1u) {
            s_tid ^= (uint32_t)p.scol[i] << 4;
            m_tid ^= (uint32_t)p.smcol[i] << 4;
            if (i >= LP_LOW) d_tid |= 1ull << p.high_q[i - LP_LOW];
        }
    uint32_t s_hi[5], m_hi[5];
    uint64_t d_hi[5];
#pragma unroll
    for (int b = 0; b < 5; ++b) {
        const bool on = TB + b < K;
        s_hi[b] = on ? (uint32_t)p.scol[TB + b] << 4 : 0u;
        m_hi[b] = on ? (uint32_t)p.smcol[TB + b] << 4 : 0u;
        d_hi[b] = on ? (16ull << p.high_q[TB + b - LP_LOW]) : 0ull;  // bytes
    }
    __syncthreads();
    double2 *__restrict__ a = reinterpret_cast<double2 *>(p.a);
#if LP_CHECK  // the tile's shared-memory bytes, the shard's bytes
#define LP_LIMS , (uint32_t)L.cpool, reinterpret_cast<const char *>(a), reinterpret_cast<const char *>(a + (1ull << p.nl))
#else
#define LP_LIMS
#endif

    for (uint64_t T = blockIdx.x; T < p.ntiles; T += gridDim.x) {
        uint64_t base = T << LP_LOW;
        for (int i = 0; i < K - LP_LOW; ++i) base = lp_ins0(base, p.high_q[i]);
        LpTile t;
        t.smem_raw = smem_raw;
        t.full = p.shard_base | base;
        t.cpool_off = (uint32_t)L.cpool;
        t.fired = 0;
        for (int e = 0; e < p.nevents; ++e)
            if ((t.full & p.ev_full[e]) == p.ev_full[e]) t.fired |= 1u << e;
        // ---- load the tile: logical x = tid + 128 j at S x ----
        if (!p.noio) {
            const char *gp = reinterpret_cast<const char *>(a + (base | d_tid));
            switch (K - TB) {
                case 5: lp_tile_load<32>(smem_raw, gp, s_tid, s_hi, d_hi LP_LIMS); break;
                case 4: lp_tile_load<16>(smem_raw, gp, s_tid, s_hi, d_hi LP_LIMS); break;
                case 3: lp_tile_load<8>(smem_raw, gp, s_tid, s_hi, d_hi LP_LIMS); break;
                case 2: lp_tile_load<4>(smem_raw, gp, s_tid, s_hi, d_hi LP_LIMS); break;
                default: lp_tile_load<2>(smem_raw, gp, s_tid, s_hi, d_hi LP_LIMS); break;
            }
        }
        // ---- per-tile products of the PHASES terms on full-index bits (op slots
        // in the coefficient pool; read after the barrier below) ----
        for (int i = (int)tid; i < p.nops_ph; i += NT) {
            const LOp &o = p.op[i];
            if (o.code != LOP_CODE_PHASES || !o.pmc[1]) continue;
            const double *T = p.sc + o.coef;
            double cr = 1.0, ci = 0.0;
            for (int k = 0; k < (int)o.pmc[1]; ++k) {
                const int c = (int)T[3 * k];
                if ((t.full >> (c - 64)) & 1u) {
                    const double er = T[3 * k + 1], ei = T[3 * k + 2];
                    const double nr = fma(cr, er, -ci * ei);
                    ci = fma(cr, ei, ci * er);
                    cr = nr;
                }
            }
            LP_ASSERT(o.pmc[0] * 8u + 16u <= (uint32_t)p.ncoef * 8u && T + 3 * o.pmc[1] <= p.sc + p.nsc);
            *reinterpret_cast<double2 *>(smem_raw + L.cpool + o.pmc[0] * 8u) = make_double2(cr, ci);
        }
        // ---- the tile scalar (conditional scalars on full-index bits, applied at the store) ----
        if (p.nts && tid == 0) {
            double cr = 1.0, ci = 0.0;
            for (int k = 0; k < p.nts; ++k) {
                const double *T = p.sc + p.ts_off + 4 * k;
                const uint64_t m = (uint64_t)__double_as_longlong(T[0]), v = (uint64_t)__double_as_longlong(T[1]);
                if ((t.full & m) == v) {
                    const double er = T[2], ei = T[3];
                    const double nr = fma(cr, er, -ci * ei);
                    ci = fma(cr, ei, ci * er);
                    cr = nr;
                }
            }
            LP_ASSERT((uint32_t)p.ts_slot * 8u + 16u <= (uint32_t)p.ncoef * 8u && p.ts_off + 4 * p.nts <= p.nsc);
            *reinterpret_cast<double2 *>(smem_raw + L.cpool + (uint32_t)p.ts_slot * 8u) = make_double2(cr, ci);
        }
        lp_cp_async_wait_all();
        __syncthreads();
        // ---- L2 prefetch of this CTA's next tile: its HBM reads overlap this
        // tile's stages, and its cp.async loads then hit L2 (one thread per
        // 128-byte run: the threads with logical bits 0..2 = 0) ----
        if (LP_PREFETCH && !p.noio && T + gridDim.x < p.ntiles) {
            // the runs are (thread bits 3.., j bits); thread tid takes the runs of the
            // j with j % 8 == tid % 8, i.e. 2^(K-TB)/8 of them
            uint64_t nb = (T + gridDim.x) << LP_LOW;
            for (int i = 0; i < K - LP_LOW; ++i) nb = lp_ins0(nb, p.high_q[i]);
            const char *gp = reinterpret_cast<const char *>(a + (nb | (d_tid & ~7ull)));
            const int nj = 1 << (K - TB);
            for (int j = (int)(tid & 7u); j < nj; j += 8) {
                uint64_t dj = 0;
#pragma unroll
                for (int b = 0; b < 5; ++b)
                    if ((j >> b) & 1) dj ^= d_hi[b];
                lp_prefetch_l2_128(gp + dj);
            }
        }
        // ---- register stages ----
        stages(t);
        // ---- store: logical x = tid + 128 j from S (M x ^ b) ----
        uint32_t sbt = p.sb_static;
        for (uint32_t m = t.fired; m; m &= m - 1) sbt ^= p.sv_ev[__ffs(m) - 1];
        double2 tsc = make_double2(1.0, 0.0);
        if (p.nts) tsc = *reinterpret_cast<const double2 *>(smem_raw + L.cpool + (uint32_t)p.ts_slot * 8u);
        if (!p.noio) {
            char *gp = reinterpret_cast<char *>(a + (base | d_tid));
            const uint32_t mo = m_tid ^ (sbt << 4);
            if (tsc.x == 1.0 && tsc.y == 0.0) {
                switch (K - TB) {
                    case 5: lp_tile_store<32>(smem_raw, gp, mo, m_hi, d_hi LP_LIMS); break;
                    case 4: lp_tile_store<16>(smem_raw, gp, mo, m_hi, d_hi LP_LIMS); break;
                    case 3: lp_tile_store<8>(smem_raw, gp, mo, m_hi, d_hi LP_LIMS); break;
                    case 2: lp_tile_store<4>(smem_raw, gp, mo, m_hi, d_hi LP_LIMS); break;
                    default: lp_tile_store<2>(smem_raw, gp, mo, m_hi, d_hi LP_LIMS); break;
                }
            } else {
                switch (K - TB) {
                    case 5: lp_tile_store_scaled<32>(smem_raw, gp, mo, m_hi, d_hi, tsc LP_LIMS); break;
                    case 4: lp_tile_store_scaled<16>(smem_raw, gp, mo, m_hi, d_hi, tsc LP_LIMS); break;
                    case 3: lp_tile_store_scaled<8>(smem_raw, gp, mo, m_hi, d_hi, tsc LP_LIMS); break;
                    case 2: lp_tile_store_scaled<4>(smem_raw, gp, mo, m_hi, d_hi, tsc LP_LIMS); break;
                    default: lp_tile_store_scaled<2>(smem_raw, gp, mo, m_hi, d_hi, tsc LP_LIMS); break;
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace qsim
