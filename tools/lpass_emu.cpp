// lpass_emu.cpp -- TEST INFRASTRUCTURE for the relabelling-pass compiler.
//
// Compiles random gate runs with lpass_compile() and interprets the program
// on the CPU with the exact semantics of the k_lpass_e kernel (lpass.cu),
// then compares with applying the same gates one by one (Eq. NUM2 with
// controls) on the full 2^n state.  It checks the host
// compiler's bookkeeping (relabelling, register addressing, diagonal merging,
// shear decomposition, conditions); it is not linked into libqsim and is never
// on a product path.  Usage: lpass_emu [ncases] [seed]; exit code 1 on failure.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../paper_1805_04708_b200/csrc/lpass.h"

using namespace qsim;
using cd = std::complex<double>;

static inline uint64_t ins0(uint64_t w, int p) { return ((w >> p) << (p + 1)) | (w & ((1ull << p) - 1ull)); }
static inline int par(uint32_t x) { return __builtin_popcount(x) & 1; }

// ---- reference: one gate at a time on the full state (physical index) ----
static void apply_direct(std::vector<cd> &a, int n, const LGate &g) {
    uint64_t cm = 0;
    for (int c = 0; c < g.nctl; ++c) cm |= 1ull << g.ctl[c];
    const uint64_t tb = 1ull << g.t;
    const cd u00(g.u[0], g.u[1]), u01(g.u[2], g.u[3]), u10(g.u[4], g.u[5]), u11(g.u[6], g.u[7]);
    for (uint64_t i = 0; i < (1ull << n); ++i) {
        if ((i & tb) || (i & cm) != cm) continue;
        const cd x = a[i], y = a[i | tb];
        a[i] = u00 * x + u01 * y;
        a[i | tb] = u10 * x + u11 * y;
    }
}

// ---- the kernel's semantics, transcribed ----
static void emu_pass(const LPassParams &p, cd *a) {
    const int K = p.K, R = p.R, NS = 1 << R;
    const uint32_t ngroups = 1u << (K - R);
    std::vector<cd> tile(1u << K);
    for (uint64_t T = 0; T < p.ntiles; ++T) {
        uint64_t base = T << LP_LOW;
        for (int i = 0; i < K - LP_LOW; ++i) base = ins0(base, p.high_q[i]);
        const uint64_t full = p.shard_base | base;
        uint32_t fired = 0;
        for (int e = 0; e < p.nevents; ++e)
            if ((full & p.ev_full[e]) == p.ev_full[e]) fired |= 1u << e;
        auto dep = [&](uint32_t x) {
            uint64_t l = x & 7u;
            for (int i = 0; i < K - LP_LOW; ++i)
                if ((x >> (LP_LOW + i)) & 1) l |= 1ull << p.high_q[i];
            return l;
        };
        for (uint32_t x = 0; x < (1u << K); ++x) {
            uint32_t ad = 0;
            for (int i = 0; i < K; ++i)
                if ((x >> i) & 1) ad ^= p.scol[i];
            tile[ad] = a[base | dep(x)];
        }
        for (int s = 0; s < p.nstages; ++s) {
            const LStage &st = p.st[s];
            uint32_t y = st.y_static;
            for (int e = 0; e < p.nevents; ++e)
                if (((fired & st.ev_mask) >> e) & 1) y ^= st.y_ev[e];
            uint32_t g0 = 0;
            for (int r = 0; r < R; ++r) g0 |= ((y >> st.qbit[r]) & 1u) << r;
            const uint32_t yrest = y & ~(uint32_t)st.qmask;
            for (uint32_t grp = 0; grp < ngroups; ++grp) {
                uint32_t a0 = 0, xq = yrest;
                for (int i = 0; i < K - R; ++i)
                    if ((grp >> i) & 1) {
                        a0 ^= st.grp_phys[i];
                        xq ^= st.grp_log[i];
                    }
                uint32_t off[32];
                cd v[32];
                for (int j = 0; j < NS; ++j) {
                    off[j] = a0;
                    for (int r = 0; r < R; ++r)
                        if ((j >> r) & 1) off[j] ^= st.reg_phys[r];
                    v[j] = tile[off[j]];
                }
                uint32_t g = g0;
                for (int oi = st.first_op; oi < st.first_op + st.nops; ++oi) {
                    const LOp &o = p.op[oi];
                    if ((o.flags & LF_COND) && (((xq & o.tmask) != o.tval) || ((full & o.omask) != o.oval))) continue;
                    if (o.code == LOP_CODE_ROUND || o.code == LOP_CODE_DIAGT)
                        for (int k = 0; k < 2; ++k) {  // pre-flips folded into the table op
                            const uint32_t f = o.pmc[k];
                            if (!(f >> 16)) continue;
                            const uint32_t c = (f >> 8) & 255u;
                            const uint32_t bit =
                                c == 255 ? 1u : c < 64 ? (xq >> c) & 1u : (uint32_t)((full >> (c - 64)) & 1u);
                            if (bit) g ^= f & 255u;
                        }
                    uint32_t toff = o.coef;  // table variant selected by the group's condition bits
                    if (o.code == LOP_CODE_ROUND || o.code == LOP_CODE_DIAGT)
                        for (int i = 0; i < o.nctl; ++i) {
                            const int c = o.rowc[i];
                            const uint32_t bit = c < 64 ? (xq >> c) & 1u : (uint32_t)((full >> (c - 64)) & 1u);
                            toff += bit << (i + R + 1);
                        }
                    if (o.code == LOP_CODE_DIAGT) {
                        for (int j = 0; j < NS; ++j) {
                            const uint32_t k = j ^ g;
                            v[j] *= cd(p.coef[toff + 2 * k], p.coef[toff + 2 * k + 1]);
                        }
                        continue;
                    }
                    if (o.code == LOP_CODE_ROUND) {
                        for (int j = 0; j < NS; ++j) {
                            const uint32_t k = j ^ g;
                            v[j] *= cd(p.coef[toff + 2 * k], p.coef[toff + 2 * k + 1]);
                        }
                        int ns = 0;
                        for (int r = 0; r < R; ++r) {
                            if (!((o.gvec >> r) & 1)) continue;
                            const double t = p.sc[o.pm + 2 * ns], aa = p.sc[o.pm + 2 * ns + 1];
                            ++ns;
                            const bool flip = (g >> r) & 1;
                            for (int j0 = 0; j0 < NS; ++j0) {
                                if ((j0 >> r) & 1) continue;
                                cd &x = flip ? v[j0 | (1 << r)] : v[j0];
                                cd &yy = flip ? v[j0] : v[j0 | (1 << r)];
                                x += aa * yy;
                                yy += t * x;
                            }
                        }
                        continue;
                    }
                    if (o.code == LOP_CODE_FLIP) {
                        g ^= o.gvec;
                        continue;
                    }
                    if (o.code == LOP_CODE_PHASES) {
                        cd c(1.0, 0.0);
                        for (int k = 0; k < o.nctl; ++k) {
                            const int cc = (int)p.sc[o.coef + 3 * k];
                            const uint32_t bit =
                                cc < 64 ? (xq >> cc) & 1u : (uint32_t)((full >> (cc - 64)) & 1u);
                            if (bit) c *= cd(p.sc[o.coef + 3 * k + 1], p.sc[o.coef + 3 * k + 2]);
                        }
                        const int gp = __builtin_popcount(o.rowS & g) & 1;
                        for (int j = 0; j < NS; ++j)
                            if (((o.pm >> j) & 1) ^ gp) v[j] *= c;
                        continue;
                    }
                    if (o.code == LOP_CODE_DIAG1) {
                        const int gp = __builtin_popcount(o.rowS & g) & 1;
                        const cd t0(p.sc[o.coef], p.sc[o.coef + 1]), t1(p.sc[o.coef + 2], p.sc[o.coef + 3]);
                        for (int j = 0; j < NS; ++j) v[j] *= ((((o.pm >> j) & 1) ^ gp) ? t1 : t0);
                        continue;
                    }
                    const int type = o.code >> 4, V = lp_vec(R, o.code & 15);
                    const int hb = 31 - __builtin_clz((unsigned)V);
                    const uint32_t gp = par(o.rowS & g);
                    uint32_t gpc[2] = {0, 0};
                    for (int k = 0; k < o.nctl; ++k) gpc[k] = par(o.rowc[k] & g);
                    for (int j0 = 0; j0 < NS; ++j0) {
                        if ((j0 >> hb) & 1) continue;
                        const int j1 = j0 ^ V;
                        bool ok = true;
                        for (int k = 0; k < o.nctl; ++k) ok = ok && (((o.pmc[k] >> j0) ^ gpc[k]) & 1u);
                        const uint32_t sgn = (type == LOP_SHEARU) ? ((o.pm ^ gp) & 1u) : (((o.pm >> j0) ^ gp) & 1u);
                        if (type == LOP_SHEAR || type == LOP_SHEARU || type == LOP_CSHEAR) {
                            double t = p.sc[o.coef];
                            if (sgn) t = -t;
                            if (!ok) t = 0.0;
                            const cd x = v[j0], yy = v[j1];
                            v[j0] = x - t * yy;
                            v[j1] = yy + t * x;
                        } else if (type == LOP_DENSE) {
                            if (!ok) continue;
                            const double *u = &p.sc[o.coef];
                            const cd u00(u[0], u[1]), u01(u[2], u[3]), u10(u[4], u[5]), u11(u[6], u[7]);
                            cd &x = sgn ? v[j1] : v[j0];
                            cd &yy = sgn ? v[j0] : v[j1];
                            const cd nx = u00 * x + u01 * yy, ny = u10 * x + u11 * yy;
                            x = nx;
                            yy = ny;
                        } else if (type == LOP_CSWAP) {
                            if (ok) std::swap(v[j0], v[j1]);
                        }
                    }
                }
                for (int j = 0; j < NS; ++j) tile[off[j]] = v[j];
            }
        }
        uint32_t sbt = p.sb_static;
        for (int e = 0; e < p.nevents; ++e)
            if ((fired >> e) & 1) sbt ^= p.sv_ev[e];
        cd tsc(1.0, 0.0);  // the tile scalar (LPassParams::nts), applied at the store
        for (int k = 0; k < p.nts; ++k) {
            const double *T = p.sc + p.ts_off + 4 * k;
            uint64_t m, v;
            std::memcpy(&m, &T[0], 8);
            std::memcpy(&v, &T[1], 8);
            if ((full & m) == v) tsc *= cd(T[2], T[3]);
        }
        for (uint32_t x = 0; x < (1u << K); ++x) {
            uint32_t ad = sbt;
            for (int i = 0; i < K; ++i)
                if ((x >> i) & 1) ad ^= p.smcol[i];
            a[base | dep(x)] = tsc == cd(1.0, 0.0) ? tile[ad] : tile[ad] * tsc;
        }
    }
}

// ---- random gates ----
struct Rng {
    std::mt19937_64 r;
    explicit Rng(uint64_t s) : r(s) {}
    double uni() { return std::uniform_real_distribution<double>(0.0, 1.0)(r); }
    int below(int n) { return (int)(r() % (uint64_t)n); }
};

static void random_u2(Rng &rng, double *u) {
    const double a = 2 * M_PI * rng.uni(), b = 2 * M_PI * rng.uni(), c = M_PI * rng.uni(), d = 2 * M_PI * rng.uni();
    const cd e = std::polar(1.0, a);
    const cd m00 = e * std::polar(std::cos(c / 2), -(b + d) / 2), m01 = -e * std::polar(std::sin(c / 2), -(b - d) / 2),
             m10 = e * std::polar(std::sin(c / 2), (b - d) / 2), m11 = e * std::polar(std::cos(c / 2), (b + d) / 2);
    const cd m[4] = {m00, m01, m10, m11};
    for (int k = 0; k < 4; ++k) {
        u[2 * k] = m[k].real();
        u[2 * k + 1] = m[k].imag();
    }
}

static void set_u(double *u, cd a, cd b, cd c, cd d) {
    const cd m[4] = {a, b, c, d};
    for (int k = 0; k < 4; ++k) {
        u[2 * k] = m[k].real();
        u[2 * k + 1] = m[k].imag();
    }
}

// ---- whole circuits through the host scheduler lpass_run (the runtime's loop) ----
struct EmuSink : LPassSink {
    std::vector<cd> *st;
    int n, nl, nglob;
    long passes = 0, sweeps = 0, synth = 0, hoisted = 0, tscal = 0;
    int pass(const LPassParams &p0, const LCompileStats &, const std::vector<int> &ids) override {
        static LPassParams p;
        p = p0;
        // per-tile hoisting: PHASES ops with full-index-bit terms, tile-scalar terms
        for (int i = 0; i < p.nops_ph; ++i)
            if (p.op[i].code == LOP_CODE_PHASES) hoisted += p.op[i].pmc[1];
        tscal += p.nts;
        for (int sh = 0; sh < (1 << nglob); ++sh) {
            p.shard_base = (uint64_t)sh << nl;
            emu_pass(p, st->data() + ((size_t)sh << nl));
        }
        ++passes;
        for (int id : ids) synth += id < 0;
        return 0;
    }
    int sweep(const LGate &g, int) override {
        apply_direct(*st, n, g);
        ++sweeps;
        return 0;
    }
    double gate_bytes(const LGate &g) override {
        const bool diag = g.u[2] == 0 && g.u[3] == 0 && g.u[4] == 0 && g.u[5] == 0;
        return std::ldexp(32.0, nl - g.nctl) * (diag ? 0.5 : 1.0);
    }
};

static int run_circuits(int ncases, uint64_t seed) {
    Rng rng(seed);
    double worst = 0.0;
    long passes = 0, sweeps = 0, synth = 0, gates = 0, hoisted = 0, tscal = 0;
    for (int cs = 0; cs < ncases; ++cs) {
        const int nl = 12 + rng.below(3), nglob = rng.below(2), n = nl + nglob;
        const int K = std::min(LP_MAX_K, nl), R = (cs % 3 == 2) ? 5 : 4;
        std::vector<LGate> gs;
        const int layered = cs % 2;
        const int ng = layered ? 0 : 60 + rng.below(200);
        if (layered) {  // config-2 shape: U on every qubit, CNOTs on a random matching
            for (int l = 0; l < 6; ++l) {
                for (int q = 0; q < nl; ++q) {  // global targets go through the exchange, not a pass
                    LGate g{};
                    g.t = q;
                    random_u2(rng, g.u);
                    gs.push_back(g);
                }
                std::vector<int> perm(n);
                for (int i = 0; i < n; ++i) perm[i] = i;
                for (int i = n - 1; i > 0; --i) std::swap(perm[i], perm[rng.below(i + 1)]);
                for (int i = 0; i + 1 < n; i += 2) {
                    LGate g{};
                    g.t = perm[i + 1];
                    g.nctl = 1;
                    g.ctl[0] = perm[i];
                    set_u(g.u, 0, 1, 1, 0);
                    if (g.t < nl) gs.push_back(g);  // global targets need the exchange, not a pass
                }
            }
        }
        for (int k = 0; k < ng; ++k) {  // config-1 shape: random kinds, qubits without replacement
            LGate g{};
            const int kind = rng.below(12);
            std::vector<int> qs(n);
            for (int i = 0; i < n; ++i) qs[i] = i;
            for (int i = n - 1; i > 0; --i) std::swap(qs[i], qs[rng.below(i + 1)]);
            const double th = 2 * M_PI * rng.uni();
            int nc = kind == 9 || kind == 10 ? 1 : kind == 11 ? 2 : 0;
            for (int c = 0; c < nc; ++c) g.ctl[c] = qs[1 + c];
            g.nctl = nc;
            g.t = qs[0];
            switch (kind) {
                case 0: set_u(g.u, M_SQRT1_2, M_SQRT1_2, M_SQRT1_2, -M_SQRT1_2); break;
                case 1: set_u(g.u, 0, 1, 1, 0); break;
                case 2: set_u(g.u, 0, cd(0, -1), cd(0, 1), 0); break;
                case 3: set_u(g.u, 1, 0, 0, -1); break;
                case 4: set_u(g.u, 1, 0, 0, cd(0, 1)); break;
                case 5: set_u(g.u, 1, 0, 0, std::polar(1.0, M_PI / 4)); break;
                case 6: set_u(g.u, std::polar(1.0, -th / 2), 0, 0, std::polar(1.0, th / 2)); break;
                case 7: set_u(g.u, std::cos(th / 2), cd(0, -std::sin(th / 2)), cd(0, -std::sin(th / 2)), std::cos(th / 2)); break;
                case 8: random_u2(rng, g.u); break;
                case 9: set_u(g.u, 0, 1, 1, 0); break;
                case 10: set_u(g.u, 1, 0, 0, std::polar(1.0, th)); break;
                default: set_u(g.u, 0, 1, 1, 0); break;
            }
            const bool diag = g.u[2] == 0 && g.u[3] == 0 && g.u[4] == 0 && g.u[5] == 0;
            if (!diag && g.t >= nl) continue;  // global non-diagonal targets go through the exchange
            gs.push_back(g);
        }
        if (cs % 5 == 4) {  // QFT-like ladders: PHASES ops mixing tile-bit and full-index-bit terms
            for (int j = nl - 1; j >= 0; --j) {
                LGate h{};
                h.t = j;
                set_u(h.u, M_SQRT1_2, M_SQRT1_2, M_SQRT1_2, -M_SQRT1_2);
                gs.push_back(h);
                for (int m = n - 1; m >= 0; --m) {
                    if (m == j) continue;
                    LGate g{};
                    g.t = j;
                    g.nctl = 1;
                    g.ctl[0] = m;
                    set_u(g.u, 1, 0, 0, std::polar(1.0, 2 * M_PI * rng.uni()));
                    gs.push_back(g);
                }
            }
        }
        std::vector<cd> a(1ull << n), b;
        for (auto &z : a) z = cd(rng.uni() - 0.5, rng.uni() - 0.5);
        b = a;
        for (const LGate &g : gs) apply_direct(a, n, g);
        EmuSink sink;
        sink.st = &b;
        sink.n = n;
        sink.nl = nl;
        sink.nglob = nglob;
        LRunConfig cfg;
        cfg.nl = nl;
        cfg.K = K;
        cfg.R = R;
        cfg.max_coef = R == 4 ? 960 : LP_MAX_COEF;
        cfg.defer = (cs % 4) != 3;
        cfg.pass_bytes = std::ldexp(32.0, nl);
        std::string err;
        const int rc = lpass_run(gs.data(), (int)gs.size(), cfg, sink, &err);
        if (rc) {
            printf("FAIL circuit %d: lpass_run rc=%d %s\n", cs, rc, err.c_str());
            return 1;
        }
        double e = 0.0;
        for (size_t i = 0; i < a.size(); ++i) e = std::max(e, std::abs(a[i] - b[i]));
        worst = std::max(worst, e);
        passes += sink.passes;
        sweeps += sink.sweeps;
        synth += sink.synth;
        hoisted += sink.hoisted;
        tscal += sink.tscal;
        gates += (long)gs.size();
        if (e > 1e-12) {
            printf("FAIL circuit %d: nl=%d nglob=%d R=%d layered=%d gates=%zu err=%.3e\n", cs, nl, nglob, R, layered,
                   gs.size(), e);
            return 1;
        }
    }
    printf("ok circuits=%d gates=%ld passes=%ld sweeps=%ld synthetic=%ld hoisted=%ld tile_scalars=%ld worst=%.3e\n",
           ncases, gates, passes, sweeps, synth, hoisted, tscal, worst);
    return 0;
}

// compile-only statistics of a gate file (t nctl c0 c1 u0..u7 per line) at nl
// local qubits: the program the runtime would launch, without a state
struct StatSink : LPassSink {
    long passes = 0, sweeps = 0, stages = 0, ops = 0, tables = 0, shears = 0, flips = 0, relabels = 0,
         tile_free = 0, events = 0, wf_ideal = 0, wf = 0;
    int nl = 30;
    int pass(const LPassParams &p, const LCompileStats &cs, const std::vector<int> &) override {
        ++passes;
        // shared-memory wavefronts of one warp's stage load (16-byte elements:
        // a wavefront serves each 16-byte bank group once)
        for (int s = 0; s < p.nstages; ++s) {
            int cnt[8][32] = {};
            int nb[8] = {};
            for (int lane = 0; lane < 32; ++lane) {
                uint32_t a = 0;
                for (int i = 0; i < 5 && i < p.K - p.R; ++i)
                    if ((lane >> i) & 1) a ^= p.st[s].grp_phys[i];
                bool seen = false;
                for (int k = 0; k < nb[a & 7]; ++k) seen |= cnt[a & 7][k] == (int)a;
                if (!seen) cnt[a & 7][nb[a & 7]++] = (int)a;
            }
            int mx = 0;
            for (int b = 0; b < 8; ++b) mx = std::max(mx, nb[b]);
            wf += mx;
            wf_ideal += 4;
        }
        stages += cs.stages;
        ops += cs.ops;
        tables += cs.diagt;
        shears += cs.shears;
        flips += cs.flips;
        relabels += cs.relabels;
        tile_free += cs.tile_free;
        events += cs.events;
        return 0;
    }
    int sweep(const LGate &, int) override {
        ++sweeps;
        return 0;
    }
    double gate_bytes(const LGate &g) override {
        const bool diag = g.u[2] == 0 && g.u[3] == 0 && g.u[4] == 0 && g.u[5] == 0;
        return std::ldexp(32.0, nl - g.nctl) * (diag ? 0.5 : 1.0);
    }
};

static int stats_file(const char *path, int nl, int R) {
    FILE *f = fopen(path, "r");
    if (!f) return 2;
    std::vector<LGate> gs;
    LGate g{};
    while (fscanf(f, "%d %d %d %d %lf %lf %lf %lf %lf %lf %lf %lf", &g.t, &g.nctl, &g.ctl[0], &g.ctl[1], &g.u[0],
                  &g.u[1], &g.u[2], &g.u[3], &g.u[4], &g.u[5], &g.u[6], &g.u[7]) == 12)
        gs.push_back(g);
    fclose(f);
    StatSink sink;
    sink.nl = nl;
    LRunConfig cfg;
    cfg.nl = nl;
    cfg.K = std::min(getenv("QSIM_LPASS_K") ? atoi(getenv("QSIM_LPASS_K")) : LP_MAX_K, nl);
    cfg.R = R;
    cfg.max_coef = R == 4 ? 960 : LP_MAX_COEF;
    cfg.pass_bytes = std::ldexp(32.0, nl);
    std::string err;
    if (lpass_run(gs.data(), (int)gs.size(), cfg, sink, &err)) {
        printf("error %s\n", err.c_str());
        return 1;
    }
    printf("gates=%zu passes=%ld sweeps=%ld stages=%ld ops=%ld tables=%ld shears=%ld flips=%ld relabels=%ld "
           "tile_free=%ld events=%ld stage_wavefronts=%ld/%ld\n",
           gs.size(), sink.passes, sink.sweeps, sink.stages, sink.ops, sink.tables, sink.shears, sink.flips,
           sink.relabels, sink.tile_free, sink.events, sink.wf, sink.wf_ideal);
    return 0;
}

// the CUDA sources of the specialised kernels of a gate file's passes
// (lpass_jit_source), one file per pass: jit_<k>.cu in outdir
struct SrcSink : LPassSink {
    std::string dir;
    int R = 4, k = 0, maxn = 1 << 30, nt = 128;
    int pass(const LPassParams &p, const LCompileStats &, const std::vector<int> &) override {
        if (k >= maxn) return 0;
        const int minb = p.R == 5 ? 2 : (p.R == 4 && p.K <= 11) ? 4 : 3;
        const std::string src = nt == 256 ? lpass_jit_source(p, p.R, 2, 256) : lpass_jit_source(p, p.R, minb);
        FILE *f = fopen((dir + "/jit_" + std::to_string(k++) + ".cu").c_str(), "w");
        if (!f) return 1;
        fputs(src.c_str(), f);
        fclose(f);
        return 0;
    }
    int sweep(const LGate &, int) override { return 0; }
    double gate_bytes(const LGate &) override { return 1e30; }
};

static int jit_sources(const char *path, int nl, const char *dir, int maxn) {
    FILE *f = fopen(path, "r");
    if (!f) return 2;
    std::vector<LGate> gs;
    LGate g{};
    while (fscanf(f, "%d %d %d %d %lf %lf %lf %lf %lf %lf %lf %lf", &g.t, &g.nctl, &g.ctl[0], &g.ctl[1], &g.u[0],
                  &g.u[1], &g.u[2], &g.u[3], &g.u[4], &g.u[5], &g.u[6], &g.u[7]) == 12)
        gs.push_back(g);
    fclose(f);
    SrcSink sink;
    sink.dir = dir;
    sink.maxn = maxn;
    if (getenv("QSIM_LPASS_NT") && atoi(getenv("QSIM_LPASS_NT")) == 256) sink.nt = 256;
    LRunConfig cfg;
    cfg.nl = nl;
    cfg.K = std::min(LP_MAX_K, nl);
    cfg.R = 4;
    cfg.max_coef = 960;
    cfg.pass_bytes = std::ldexp(32.0, nl);
    std::string err;
    if (lpass_run(gs.data(), (int)gs.size(), cfg, sink, &err)) {
        printf("error %s\n", err.c_str());
        return 1;
    }
    printf("ok sources=%d\n", sink.k);
    return 0;
}

int main(int argc, char **argv) {
    if (argc > 4 && std::string(argv[1]) == "jitsrc")
        return jit_sources(argv[2], atoi(argv[3]), argv[4], argc > 5 ? atoi(argv[5]) : 1 << 30);
    if (argc > 3 && std::string(argv[1]) == "stats") return stats_file(argv[2], atoi(argv[3]), argc > 4 ? atoi(argv[4]) : 4);
    const int ncases = argc > 1 ? atoi(argv[1]) : 300;
    const uint64_t seed = argc > 2 ? strtoull(argv[2], nullptr, 10) : 1;
    if (argc > 3 && std::string(argv[3]) == "run") return run_circuits(ncases, seed);
    Rng rng(seed);
    double worst = 0.0;
    long tot_carried = 0, tot_deferred = 0, tot_gates = 0, tot_stages = 0, tot_ops = 0, tot_shear = 0, tot_dense = 0, tot_free = 0, tot_short = 0;
    static LPassParams p;
    for (int cs = 0; cs < ncases; ++cs) {
        const int R = (cs % 3 == 2) ? 5 : 4;
        const int K = LP_MIN_K + rng.below(LP_MAX_K - LP_MIN_K + 1);
        const int nl = K + rng.below(3);
        const int nglob = rng.below(3);
        const int n = nl + nglob;
        // tile: qubits 0..2 plus K-3 random higher local qubits
        std::vector<int> hi;
        for (int q = LP_LOW; q < nl; ++q) hi.push_back(q);
        for (size_t i = hi.size(); i > 1; --i) std::swap(hi[i - 1], hi[rng.below((int)i)]);
        hi.resize(K - LP_LOW);
        std::sort(hi.begin(), hi.end());
        std::vector<int> tq = {0, 1, 2};
        for (int q : hi) tq.push_back(q);
        std::vector<char> in_tile(n, 0);
        for (int q : tq) in_tile[q] = 1;
        // gates
        const int style = rng.below(4);  // 0: config-2-like layers, 1..3: random mixes
        int ng = 1 + rng.below(LP_MAX_PASS_GATES);
        std::vector<LGate> gs;
        auto pick_tile = [&]() { return tq[rng.below(K)]; };
        auto pick_any = [&]() { return rng.below(n); };
        for (int k = 0; k < ng; ++k) {
            LGate g{};
            const int kind = (style == 0) ? (rng.below(3) < 2 ? 8 : 9) : rng.below(15);
            g.t = pick_tile();
            auto add_ctl = [&](bool tile_only) {
                for (int tries = 0; tries < 50; ++tries) {
                    const int c = tile_only ? pick_tile() : pick_any();
                    bool dup = c == g.t;
                    for (int j = 0; j < g.nctl; ++j) dup = dup || g.ctl[j] == c;
                    if (!dup) {
                        g.ctl[g.nctl++] = c;
                        return;
                    }
                }
            };
            const double th = 2 * M_PI * rng.uni();
            switch (kind) {
                case 0: set_u(g.u, M_SQRT1_2, M_SQRT1_2, M_SQRT1_2, -M_SQRT1_2); break;  // H
                case 1: set_u(g.u, 0, 1, 1, 0); break;                                    // X
                case 2: set_u(g.u, 0, cd(0, -1), cd(0, 1), 0); break;                     // Y
                case 3: set_u(g.u, 1, 0, 0, -1); g.t = pick_any(); break;                 // Z anywhere
                case 4: set_u(g.u, 1, 0, 0, std::polar(1.0, th)); g.t = pick_any(); add_ctl(false); break;  // CPHASE
                case 5: set_u(g.u, std::polar(1.0, -th / 2), 0, 0, std::polar(1.0, th / 2)); g.t = pick_any(); break;  // Rz
                case 6: set_u(g.u, std::cos(th / 2), cd(0, -std::sin(th / 2)), cd(0, -std::sin(th / 2)), std::cos(th / 2)); break;  // Rx
                case 7: random_u2(rng, g.u); add_ctl(false); break;  // controlled U
                case 8: random_u2(rng, g.u); break;                  // U
                case 9: set_u(g.u, 0, 1, 1, 0); add_ctl(style == 0); break;  // CNOT
                case 10: set_u(g.u, 0, 1, 1, 0); add_ctl(false); add_ctl(false); break;  // Toffoli
                case 11: random_u2(rng, g.u); add_ctl(false); add_ctl(false); break;     // CCU
                case 12: set_u(g.u, 0, std::polar(1.0, th), std::polar(1.0, 0.3), 0); add_ctl(false); break;  // controlled anti
                case 14:  // a unitary off by 1e-11 (accepted by the API, fails the 1e-14 shear reconstruction)
                    random_u2(rng, g.u);
                    g.u[0] += 1e-11;
                    if (rng.below(2)) add_ctl(false);
                    break;
                default: {  // swapped dense (|u01| > |u00|)
                    const double c = std::cos(1.2), s = std::sin(1.2);
                    set_u(g.u, c * std::polar(1.0, th), -s, s * std::polar(1.0, th), c);
                    break;
                }
            }
            gs.push_back(g);
        }
        // compile (shorten like the runtime when the program does not fit)
        std::string err;
        LCompileStats stt;
        int rc;
        std::vector<LGate> dfr;
        const bool defer = (cs % 2) == 1;
        while ((rc = lpass_compile(gs.data(), (int)gs.size(), nl, K, R, tq.data(), LP_MAX_COEF, p, &stt, &err,
                                   defer ? &dfr : nullptr)) == 1) {
            gs.pop_back();
            ++tot_short;
        }
        if (rc != 0) {
            printf("case %d: compile error: %s\n", cs, err.c_str());
            return 1;
        }
        // random state
        std::vector<cd> a(1ull << n), b;
        for (auto &z : a) z = cd(rng.uni() - 0.5, rng.uni() - 0.5);
        b = a;
        for (const LGate &g : gs) apply_direct(a, n, g);
        for (int sh = 0; sh < (1 << nglob); ++sh) {
            p.shard_base = (uint64_t)sh << nl;
            emu_pass(p, b.data() + ((size_t)sh << nl));
        }
        for (const LGate &g : dfr) apply_direct(b, n, g);  // deferred diagonals right after the pass
        tot_carried += stt.carried;
        tot_deferred += (long)dfr.size();
        double e = 0.0;
        for (size_t i = 0; i < a.size(); ++i) e = std::max(e, std::abs(a[i] - b[i]));
        worst = std::max(worst, e);
        tot_gates += (long)gs.size();
        tot_stages += stt.stages;
        tot_ops += stt.ops;
        tot_shear += stt.shears;
        tot_dense += stt.dense;
        tot_free += stt.tile_free;
        if (e > 1e-12) {
            printf("FAIL case %d: K=%d R=%d nl=%d nglob=%d style=%d gates=%zu err=%.3e\n", cs, K, R, nl, nglob, style,
                   gs.size(), e);
            return 1;
        }
    }
    printf("ok cases=%d gates=%ld stages=%ld ops=%ld shears=%ld dense=%ld tile_free=%ld carried=%ld deferred=%ld "
           "shortened=%ld worst=%.3e\n",
           ncases, tot_gates, tot_stages, tot_ops, tot_shear, tot_dense, tot_free, tot_carried, tot_deferred, tot_short,
           worst);
    return 0;
}
