// lpass_compile.cpp -- host compiler of the relabelling tile pass (lpass.h).
//
// Input: a run of gates in circuit order (physical bit positions), the tile
// (K local qubits), the register width R.  Output: an LPassParams program:
// per register stage the register / group addressing, and a list of ops
// (shears, general 2x2, controlled swaps, flips, diagonal-table multiplies).
//
// Correctness argument (the result equals applying the gates one after the
// other, Eq. NUM2 PAPER.md:285-299 with controls PAPER.md:302-307):
//  * gates are only reordered across gates they commute with (every shared
//    qubit acted on diagonally by both: controls and diagonal targets);
//  * a dense U is replaced by the product Dl . cos . shear(t) . Dr (checked
//    entry by entry against U, else applied as a general 2x2);
//  * diagonal factors are accumulated in a table P over the register slots
//    and flushed before any non-diagonal op on a slot P depends on; a
//    permutation of the slots (X, CNOT, Toffoli on register qubits) commutes
//    with P after conjugation (P' = P o pi^-1);
//  * CNOT / X relabel the tile (M, b of lpass.h); every later address is
//    computed from the current (M, b), and the final store undoes them.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lpass.h"

namespace qsim {
namespace {

using cd = std::complex<double>;

inline int par(uint32_t x) { return __builtin_popcount(x) & 1; }

enum { GC_IDENT, GC_DIAG, GC_ANTI, GC_DENSE };

int gclass(const double *u) {
    const bool off0 = u[2] == 0.0 && u[3] == 0.0 && u[4] == 0.0 && u[5] == 0.0;
    const bool dia0 = u[0] == 0.0 && u[1] == 0.0 && u[6] == 0.0 && u[7] == 0.0;
    if (off0) return (u[0] == 1.0 && u[1] == 0.0 && u[6] == 1.0 && u[7] == 0.0) ? GC_IDENT : GC_DIAG;
    if (dia0) return GC_ANTI;
    return GC_DENSE;
}

struct GInfo {
    int cls = GC_IDENT;
    bool pure = false;  // anti-diagonal with u01 = u10 = 1 (X, CNOT, Toffoli)
    int tt = -1;        // target tile bit (-1: outside the tile)
    uint64_t tfull = 0; // target as a full-index mask
    int nci = 0;
    int ci[2] = {-1, -1};  // controls inside the tile (tile bits)
    uint64_t om = 0;       // controls outside the tile (full-index mask)
    uint64_t xq = 0, zq = 0;
    const double *u = nullptr;
};

// Tile relabelling state: logical tile index x sits at physical p = M x ^ b,
// b = b_static ^ (v_e of every event e that fired on this tile).
struct TileState {
    int K = 0;
    uint16_t col[LP_MAX_K];  // M e_i
    uint16_t row[LP_MAX_K];  // row i of M^-1
    uint16_t b_static = 0;
    std::vector<uint64_t> ev_full;
    std::vector<uint16_t> ev_v;
    void init(int K_) {
        K = K_;
        for (int i = 0; i < K; ++i) col[i] = row[i] = (uint16_t)(1u << i);
        b_static = 0;
        ev_full.clear();
        ev_v.clear();
    }
    // CNOT(c -> t) on logical tile bits: M <- M L, L = I + e_t e_c^T
    void relabel(int c, int t) {
        col[c] ^= col[t];
        row[t] ^= row[c];
    }
    uint16_t logical(uint16_t p) const {
        uint16_t x = 0;
        for (int i = 0; i < K; ++i)
            if (par(row[i] & p)) x |= (uint16_t)(1u << i);
        return x;
    }
};

enum PKind { PK_DIAGM, PK_DIAGC, PK_SHEAR, PK_DENSE, PK_RELABEL, PK_FLIPU, PK_FLIPC, PK_CSWAP };

struct Prim {
    int kind = PK_DIAGM;
    int S = -1;   // non-diagonal target slot
    int cs = 0;   // in-register control slots
    int rc = -1;  // RELABEL control slot
    uint16_t tmask = 0, tval = 0;
    uint64_t omask = 0, oval = 0;
    double t = 0.0;
    double u[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    std::vector<cd> tab;  // diagonal over the 2^R logical slot values
    int fl_ctl = -1;      // FLIPC: in-tile control (tile bit) -> tile-level relabel
    uint64_t fl_om = 0;   // FLIPC: out-of-tile controls -> tile-level event
    int xs = 0, zs = 0;
    bool cond() const { return tmask != 0 || omask != 0; }
};

inline bool prim_conflict(const Prim &a, const Prim &b) { return (a.xs & (b.xs | b.zs)) || (a.zs & b.xs); }

// tile-level replay of the stage's relabels / flips (in emission order)
struct Replay {
    int kind;  // PK_RELABEL, PK_FLIPU, PK_FLIPC
    int c_tbit, t_tbit;
    uint64_t om;
};

struct StageRec {
    int Q[5];
    uint16_t col[LP_MAX_K], row[LP_MAX_K];
    uint16_t b_static;
    int nev;
    int op0, nops;
    bool needs_xq;
    uint32_t flip_ctl;  // tile bits that condition an in-stage flip (keep them warp-uniform)
};

struct Compiler {
    const LGate *gates;
    int ng, nl, K, R, NS, NV, max_coef;
    int tbit_of[64];
    std::vector<GInfo> G;
    TileState ts;
    std::vector<LOp> ops;
    std::vector<double> coef;
    std::vector<StageRec> stages;
    LCompileStats st;
    std::string err;
    int vidx[32];  // register pair vector -> vsel (-1 if weight > 2)

    // carried 1-qubit diagonals (per logical tile bit) and scalar
    bool allow_carry = false;
    bool has_carry[LP_MAX_K] = {false};
    cd carry[LP_MAX_K][2];
    cd carry_scalar = cd(1.0, 0.0);
    std::vector<LGate> out_deferred;  // uncontrolled diagonals on qubits outside the tile

    bool is_free(const GInfo &g) const {
        if (!g.pure || g.tt < 0) return false;
        // a carried diagonal on the target commutes with an uncontrolled X only
        if (has_carry[g.tt] && !(g.nci == 0 && g.om == 0)) return false;
        if (g.nci == 1 && g.om == 0) return true;
        if (g.nci == 0 && g.om == 0) return true;
        if (g.nci == 0 && (int)ts.ev_v.size() < LP_MAX_EVENTS) return true;
        return false;
    }
    void apply_free(const GInfo &g) {
        if (g.nci == 1)
            ts.relabel(g.ci[0], g.tt);
        else if (g.om == 0) {
            ts.b_static ^= ts.col[g.tt];
            if (has_carry[g.tt]) std::swap(carry[g.tt][0], carry[g.tt][1]);  // D X = X D'
        }
        else {
            ts.ev_full.push_back(g.om);
            ts.ev_v.push_back(ts.col[g.tt]);
        }
        st.tile_free++;
    }

    std::vector<double> sc;
    int add_table(const double *v, int n, bool reuse = false) {  // n = 2^(R+1): tables stay aligned to their size
        if (reuse)  // an identical table already in the pool (bitwise): share it
            for (int at = 0; at + n <= (int)coef.size(); at += n)
                if (std::memcmp(coef.data() + at, v, sizeof(double) * (size_t)n) == 0) return at;
        if ((int)coef.size() + n > max_coef) return -1;
        const int at = (int)coef.size();
        coef.insert(coef.end(), v, v + n);
        return at;
    }
    int add_sc(const double *v, int n) {
        if ((int)sc.size() + n > LP_MAX_SC) return -1;
        const int at = (int)sc.size();
        sc.insert(sc.end(), v, v + n);
        return at;
    }

    int run();
    int compile_stage(const std::vector<int> &take, const int *Q);
    // stage register sets: greedy lookahead (LPASS_LOOKAHEAD=1, default) with a
    // score penalty per in-stage flip (LPASS_FLIP_PENALTY), or first-come (0).
    // With the specialised kernels (no op dispatch) the lookahead's fewer
    // stages win: QFT N=32 835 -> 775 ms, config 3 N=33 1426 -> 1396 ms,
    // config 2 equal (it measured slower with the interpreter)
    int lookahead = 1, flip_penalty = 2;
};

// Build the register-stage prims of one gate.  `slot_of` maps tile bit -> slot.
struct PrimBuilder {
    int R, NS;
    const int *slot_of;
    int nev_avail;  // events still available for FLIPC on out-of-tile controls
    std::vector<Prim> *out;

    void ctl_split(const GInfo &g, int &cs, uint16_t &tm, uint64_t &om) const {
        cs = 0;
        tm = 0;
        om = g.om;
        for (int k = 0; k < g.nci; ++k) {
            const int s = slot_of[g.ci[k]];
            if (s >= 0)
                cs |= 1 << s;
            else
                tm |= (uint16_t)(1u << g.ci[k]);
        }
    }
    std::vector<cd> diag_table(int S, int cs, cd d0, cd d1) const {
        std::vector<cd> tab(NS, cd(1.0, 0.0));
        for (int s = 0; s < NS; ++s) {
            if ((s & cs) != cs) continue;
            tab[s] = (S >= 0) ? (((s >> S) & 1) ? d1 : d0) : d0;
        }
        return tab;
    }
    // diagonal diag(d0, d1) on the target of g (controls of g)
    void diag(const GInfo &g, cd d0, cd d1) {
        int cs;
        uint16_t tm;
        uint64_t om;
        ctl_split(g, cs, tm, om);
        const int S = (g.tt >= 0) ? slot_of[g.tt] : -1;
        if (S >= 0) {
            if (d0 == cd(1.0, 0.0) && d1 == cd(1.0, 0.0)) return;
            Prim p;
            p.kind = (tm || om) ? PK_DIAGC : PK_DIAGM;
            p.tab = diag_table(S, cs, d0, d1);
            p.tmask = p.tval = tm;
            p.omask = p.oval = om;
            p.zs = cs | (1 << S);
            out->push_back(p);
            return;
        }
        // target outside the registers: one conditional table per target value
        for (int b = 0; b < 2; ++b) {
            const cd d = b ? d1 : d0;
            if (d == cd(1.0, 0.0)) continue;
            Prim p;
            p.kind = PK_DIAGC;
            p.tab = diag_table(-1, cs, d, d);
            p.tmask = p.tval = tm;
            p.omask = p.oval = om;
            if (g.tt >= 0) {
                p.tmask |= (uint16_t)(1u << g.tt);
                if (b) p.tval |= (uint16_t)(1u << g.tt);
            } else {
                p.omask |= g.tfull;
                if (b) p.oval |= g.tfull;
            }
            p.zs = cs;
            out->push_back(p);
        }
    }
    // controlled X on slot S (the permutation part of an anti-diagonal gate)
    void xpart(const GInfo &g, int S) {
        int cs;
        uint16_t tm;
        uint64_t om;
        ctl_split(g, cs, tm, om);
        const int nin = __builtin_popcount(cs), nout = __builtin_popcount(tm);
        Prim p;
        p.S = S;
        p.xs = 1 << S;
        if (nin == 0 && nout == 0 && om == 0) {
            p.kind = PK_FLIPU;
        } else if (nin == 1 && nout == 0 && om == 0) {
            p.kind = PK_RELABEL;
            p.rc = __builtin_ctz(cs);
            p.zs = cs;
        } else if (nin == 0 && nout == 1 && om == 0) {
            p.kind = PK_FLIPC;
            p.tmask = p.tval = tm;
            p.fl_ctl = __builtin_ctz(tm);
        } else if (nin == 0 && nout == 0 && om != 0 && nev_avail > 0) {
            p.kind = PK_FLIPC;
            p.omask = p.oval = om;
            p.fl_om = om;
            --nev_avail;
        } else {
            p.kind = PK_CSWAP;
            p.cs = cs;
            p.zs = cs;
            p.tmask = p.tval = tm;
            p.omask = p.oval = om;
        }
        out->push_back(p);
    }
    void gate(const GInfo &g) {
        const double *u = g.u;
        if (g.cls == GC_IDENT) return;
        if (g.cls == GC_DIAG) {
            diag(g, cd(u[0], u[1]), cd(u[6], u[7]));
            return;
        }
        const int S = slot_of[g.tt];
        if (g.cls == GC_ANTI) {
            // U = X . diag(u10, u01)
            diag(g, cd(u[4], u[5]), cd(u[2], u[3]));
            xpart(g, S);
            return;
        }
        // dense: U = X^s V, V = Dl . c . shear(t) . Dr
        const cd u00(u[0], u[1]), u01(u[2], u[3]), u10(u[4], u[5]), u11(u[6], u[7]);
        const bool swapped = std::abs(u01) > std::abs(u00);
        const cd a = swapped ? u10 : u00, b = swapped ? u11 : u01, c = swapped ? u00 : u10,
                 d = swapped ? u01 : u11;
        const double ma = std::abs(a), mb = std::abs(b);
        bool ok = ma > 0.0 && mb > 0.0;
        cd l0, l1, r1;
        double t = 0.0;
        if (ok) {
            l0 = a / ma;
            r1 = -b * std::conj(l0) / mb;
            l1 = c / mb;
            t = mb / ma;
            const cd dl0 = l0 * ma, dl1 = l1 * ma;
            const cd R00 = dl0, R01 = -dl0 * t * r1, R10 = dl1 * t, R11 = dl1 * r1;
            const double e = std::max(std::max(std::abs(R00 - a), std::abs(R01 - b)),
                                      std::max(std::abs(R10 - c), std::abs(R11 - d)));
            ok = e <= 1e-14 && t <= 1.0;
            if (ok) {
                int cs;
                uint16_t tm;
                uint64_t om;
                ctl_split(g, cs, tm, om);
                diag(g, cd(1.0, 0.0), r1);
                Prim p;
                p.kind = PK_SHEAR;
                p.S = S;
                p.cs = cs;
                p.t = t;
                p.tmask = p.tval = tm;
                p.omask = p.oval = om;
                p.xs = 1 << S;
                p.zs = cs;
                out->push_back(p);
                diag(g, dl0, dl1);
                if (swapped) xpart(g, S);
                return;
            }
        }
        int cs;
        uint16_t tm;
        uint64_t om;
        ctl_split(g, cs, tm, om);
        Prim p;
        p.kind = PK_DENSE;
        p.S = S;
        p.cs = cs;
        std::memcpy(p.u, u, sizeof(p.u));
        p.tmask = p.tval = tm;
        p.omask = p.oval = om;
        p.xs = 1 << S;
        p.zs = cs;
        out->push_back(p);
    }
};

int Compiler::compile_stage(const std::vector<int> &take, const int *Q) {
    int slot_of[LP_MAX_K];
    for (int i = 0; i < LP_MAX_K; ++i) slot_of[i] = -1;
    for (int r = 0; r < R; ++r) slot_of[Q[r]] = r;
    std::vector<Prim> prims;
    PrimBuilder pb{R, NS, slot_of, LP_MAX_EVENTS - (int)ts.ev_v.size(), &prims};
    for (int k : take) pb.gate(G[k]);

    StageRec sr;
    for (int r = 0; r < R; ++r) sr.Q[r] = Q[r];
    std::memcpy(sr.col, ts.col, sizeof(sr.col));
    std::memcpy(sr.row, ts.row, sizeof(sr.row));
    sr.b_static = ts.b_static;
    sr.nev = (int)ts.ev_v.size();
    sr.op0 = (int)ops.size();
    sr.needs_xq = false;
    sr.flip_ctl = 0;

    uint8_t Arow[5], Ainv[5];
    for (int r = 0; r < R; ++r) Arow[r] = Ainv[r] = (uint8_t)(1u << r);
    const bool absorb_carry = true;  // carried factors of the register qubits start the pending diagonal
    // Pending diagonal: one table over the logical register slots per value
    // of up to 2 single-bit conditions (tile bit b -> code b, full-index bit b
    // -> code 64 + b).  A flip conditioned on one such bit conjugates only the
    // variants where the bit is 1, so it needs no flush; the kernel selects
    // the variant per group.
    std::vector<std::vector<cd>> PV(1, std::vector<cd>(NS, cd(1.0, 0.0)));
    int pv_n = 0, pv_code[2] = {0, 0};
    std::vector<Replay> replay;
    if (absorb_carry) {
        for (int r = 0; r < R; ++r)
            if (has_carry[Q[r]]) {
                for (int sg = 0; sg < NS; ++sg) PV[0][sg] *= carry[Q[r]][(sg >> r) & 1];
                has_carry[Q[r]] = false;
            }
        if (carry_scalar != cd(1.0, 0.0)) {
            for (int sg = 0; sg < NS; ++sg) PV[0][sg] *= carry_scalar;
            carry_scalar = cd(1.0, 0.0);
        }
    }

    auto suppP = [&]() {
        int m = 0;
        for (const auto &P : PV)
            for (int r = 0; r < R; ++r)
                for (int s = 0; s < NS; ++s)
                    if (P[s] != P[s ^ (1 << r)]) {
                        m |= 1 << r;
                        break;
                    }
        return m;
    };
    auto isI = [&]() {
        for (const auto &P : PV)
            for (int s = 0; s < NS; ++s)
                if (P[s] != cd(1.0, 0.0)) return false;
        return true;
    };
    auto reset_P = [&]() {
        PV.assign(1, std::vector<cd>(NS, cd(1.0, 0.0)));
        pv_n = 0;
    };
    // conjugate every variant (selected by vmask over variant indices) by a slot permutation
    auto conj_P = [&](auto perm, uint32_t vsel_bits, uint32_t vsel_val) {
        for (size_t vi = 0; vi < PV.size(); ++vi) {
            if ((vi & vsel_bits) != vsel_val) continue;
            std::vector<cd> Q2(NS);
            for (int s = 0; s < NS; ++s) Q2[s] = PV[vi][perm(s)];
            PV[vi].swap(Q2);
        }
    };
    auto A_apply = [&](int k) {  // A k
        int x = 0;
        for (int r = 0; r < R; ++r)
            if (par(Arow[r] & k)) x |= 1 << r;
        return x;
    };
    auto pmask = [&](uint8_t row) {
        uint32_t m = 0;
        for (int j = 0; j < NS; ++j)
            if (par(row & j)) m |= 1u << j;
        return m;
    };
    auto set_cond = [&](LOp &o, const Prim &p) {
        if (p.cond()) {
            o.flags |= LF_COND;
            o.tmask = p.tmask;
            o.tval = p.tval;
            o.omask = p.omask;
            o.oval = p.oval;
            if (p.tmask) sr.needs_xq = true;
        }
    };
    auto table_at = [&](const std::vector<cd> &T, bool reuse) -> int {
        std::vector<double> buf(2 * NS);
        for (int k = 0; k < NS; ++k) {
            const cd e = T[A_apply(k)];
            buf[2 * k] = e.real();
            buf[2 * k + 1] = e.imag();
        }
        return add_table(buf.data(), 2 * NS, reuse);
    };
    // the pending tables (all variants, consecutive); fills the variant fields of o
    auto pending_tables = [&](LOp &o) -> int {
        int first = -1;
        for (const auto &P : PV) {
            const int at = table_at(P, PV.size() == 1);  // variants must stay consecutive
            if (at < 0) return -1;
            if (first < 0) first = at;
        }
        o.coef = (uint16_t)first;
        o.nctl = (uint8_t)pv_n;
        for (int i = 0; i < pv_n; ++i) {
            o.rowc[i] = (uint8_t)pv_code[i];
            if (pv_code[i] < 64) sr.needs_xq = true;
        }
        return 0;
    };
    auto emit_table = [&](const std::vector<cd> &T, const Prim *cp) -> int {
        const int at = table_at(T, true);
        if (at < 0) return 1;
        LOp o{};
        o.code = LOP_CODE_DIAGT;
        o.coef = (uint16_t)at;
        if (cp) set_cond(o, *cp);
        ops.push_back(o);
        st.diagt++;
        return 0;
    };
    auto flush_P = [&]() -> int {
        LOp o{};
        o.code = LOP_CODE_DIAGT;
        if (pending_tables(o)) return 1;
        ops.push_back(o);
        st.diagt++;
        reset_P();
        return 0;
    };
    // a shear that can join a ROUND: unconditional, uncontrolled, and slot S
    // maps to a single register bit r both ways (A e_r = e_S), so its pairs are
    // (j0, j0 | 2^r) and the orientation is bit r of g.  Returns r or -1.
    auto round_bit = [&](const Prim &p) -> int {
        if (p.kind != PK_SHEAR || p.cs || p.cond()) return -1;
        const int v = Ainv[p.S];
        if (__builtin_popcount(v) != 1 || Arow[p.S] != v) return -1;
        return __builtin_ctz(v);
    };
    auto emit_v = [&](int type, const Prim &p, int coef_at) -> int {
        const int v = Ainv[p.S];
        const int vsel = vidx[v];
        if (vsel < 0) {
            err = "internal: register pair vector of weight > 2";
            return -1;
        }
        LOp o{};
        o.rowS = Arow[p.S];
        o.pm = pmask(Arow[p.S]);
        if (type == LOP_SHEAR && p.cs == 0) {
            const int hb = 31 - __builtin_clz((unsigned)v);
            int first = -1;
            bool uni = true;
            for (int j = 0; j < NS; ++j) {
                if ((j >> hb) & 1) continue;
                const int b = (o.pm >> j) & 1;
                if (first < 0)
                    first = b;
                else if (b != first)
                    uni = false;
            }
            if (uni) {
                type = LOP_SHEARU;
                o.pm = (uint32_t)first;
            }
        }
        if (type == LOP_SHEAR && p.cs) type = LOP_CSHEAR;
        int k = 0;
        for (int c = 0; c < R; ++c)
            if ((p.cs >> c) & 1) {
                o.rowc[k] = Arow[c];
                o.pmc[k] = pmask(Arow[c]);
                ++k;
            }
        o.nctl = (uint8_t)k;
        o.code = (uint8_t)(type * 16 + vsel);
        o.coef = (uint16_t)coef_at;
        set_cond(o, p);
        ops.push_back(o);
        return 0;
    };

    const int n = (int)prims.size();
    std::vector<char> done(n, 0);
    int ndone = 0;
    auto ready = [&](int k) {
        for (int j = 0; j < k; ++j)
            if (!done[j] && prim_conflict(prims[j], prims[k])) return false;
        return true;
    };
    while (ndone < n) {
        bool progress = true;
        while (progress) {
            progress = false;
            for (int k = 0; k < n; ++k) {
                if (done[k] || !ready(k)) continue;
                Prim &p = prims[k];
                const int sp = suppP();
                bool emitted = true;
                switch (p.kind) {
                    case PK_DIAGM:
                        for (auto &P : PV)
                            for (int s = 0; s < NS; ++s) P[s] *= p.tab[s];
                        break;
                    case PK_DIAGC: {
                        // a conditional diagonal on one logical slot (CPHASE / controlled
                        // phase with its control outside the registers): two coefficients
                        // in sc, no 2^R table in the coefficient pool
                        int S1 = -1;
                        for (int b = 0; b < R && S1 < 0; ++b) {
                            bool ok1 = true;
                            for (int sv = 0; sv < NS && ok1; ++sv)
                                ok1 = p.tab[sv] == p.tab[((sv >> b) & 1) ? (1 << b) : 0];
                            if (ok1) S1 = b;
                        }
                        // T0 = 1 under one condition bit (= 1): a PHASES term, merged into the
                        // previous op when that is a PHASES op on the same slot whose terms end
                        // the scalar array
                        int pcode = -1;
                        if (S1 >= 0 && p.tab[0] == cd(1.0, 0.0)) {
                            if (p.tmask && !p.omask && __builtin_popcount(p.tmask) == 1 && p.tval == p.tmask)
                                pcode = __builtin_ctz(p.tmask);
                            else if (!p.tmask && p.omask && __builtin_popcountll(p.omask) == 1 && p.oval == p.omask)
                                pcode = 64 + __builtin_ctzll(p.omask);
                        }
                        if (pcode >= 0) {
                            const double term[3] = {(double)pcode, p.tab[1 << S1].real(), p.tab[1 << S1].imag()};
                            LOp *last = ops.size() > (size_t)sr.op0 ? &ops.back() : nullptr;
                            if (last && last->code == LOP_CODE_PHASES && last->rowS == Arow[S1] && last->nctl < 255 &&
                                (int)sc.size() == last->coef + 3 * last->nctl) {
                                if (add_sc(term, 3) < 0) return 1;
                                last->nctl++;
                            } else {
                                const int at = add_sc(term, 3);
                                if (at < 0) return 1;
                                LOp o{};
                                o.code = LOP_CODE_PHASES;
                                o.rowS = Arow[S1];
                                o.pm = pmask(Arow[S1]);
                                o.coef = (uint16_t)at;
                                o.nctl = 1;
                                ops.push_back(o);
                            }
                            if (pcode < 64) sr.needs_xq = true;
                            st.diagt++;
                            break;
                        }
                        if (S1 >= 0) {
                            const double tv[4] = {p.tab[0].real(), p.tab[0].imag(), p.tab[1 << S1].real(),
                                                  p.tab[1 << S1].imag()};
                            const int at = add_sc(tv, 4);
                            if (at < 0) return 1;
                            LOp o{};
                            o.code = LOP_CODE_DIAG1;
                            o.rowS = Arow[S1];
                            o.pm = pmask(Arow[S1]);
                            o.coef = (uint16_t)at;
                            o.gvec = (uint8_t)(p.tab[0] == cd(1.0, 0.0) ? 1 : 0);
                            set_cond(o, p);
                            ops.push_back(o);
                            st.diagt++;
                            break;
                        }
                        const int rc = emit_table(p.tab, &p);
                        if (rc) return rc;
                        break;
                    }
                    case PK_SHEAR:
                    case PK_DENSE: {
                        if ((sp >> p.S) & 1) {
                            emitted = false;
                            break;
                        }
                        if (p.kind == PK_SHEAR && round_bit(p) >= 0) {  // joins the next ROUND
                            emitted = false;
                            break;
                        }
                        int at;
                        if (p.kind == PK_SHEAR) {
                            at = add_sc(&p.t, 1);
                            st.shears++;
                        } else {
                            at = add_sc(p.u, 8);
                            st.dense++;
                        }
                        if (at < 0) return 1;
                        const int rc = emit_v(p.kind == PK_SHEAR ? LOP_SHEAR : LOP_DENSE, p, at);
                        if (rc) return rc;
                        break;
                    }
                    case PK_CSWAP: {
                        if (p.cond() && ((sp >> p.S) & 1)) {
                            emitted = false;
                            break;
                        }
                        const int rc = emit_v(LOP_CSWAP, p, 0);
                        if (rc) return rc;
                        st.cswaps++;
                        if (!p.cond())
                            conj_P([&](int s) { return ((s & p.cs) == p.cs) ? s ^ (1 << p.S) : s; }, 0, 0);
                        break;
                    }
                    case PK_RELABEL: {
                        conj_P([&](int s) { return s ^ (((s >> p.rc) & 1) << p.S); }, 0, 0);
                        Arow[p.S] ^= Arow[p.rc];
                        Ainv[p.rc] ^= Ainv[p.S];
                        replay.push_back({PK_RELABEL, Q[p.rc], Q[p.S], 0});
                        st.relabels++;
                        break;
                    }
                    case PK_FLIPU:
                    case PK_FLIPC: {
                        if (p.kind == PK_FLIPC && ((sp >> p.S) & 1)) {
                            // a single-bit condition becomes a variant of the pending diagonal
                            int code = -1;
                            if (p.fl_ctl >= 0)
                                code = p.fl_ctl;
                            else if (__builtin_popcountll(p.fl_om) == 1)
                                code = 64 + __builtin_ctzll(p.fl_om);
                            int vi = -1;
                            for (int i = 0; i < pv_n; ++i)
                                if (pv_code[i] == code) vi = i;
                            if (code < 0 || (vi < 0 && pv_n >= 2)) {
                                emitted = false;
                                break;
                            }
                            if (vi < 0) {
                                const size_t nv = PV.size();
                                for (size_t k2 = 0; k2 < nv; ++k2) PV.push_back(PV[k2]);
                                vi = pv_n;
                                pv_code[pv_n++] = code;
                            }
                            conj_P([&](int s) { return s ^ (1 << p.S); }, 1u << vi, 1u << vi);
                        }
                        LOp o{};
                        o.code = LOP_CODE_FLIP;
                        o.gvec = Ainv[p.S];
                        set_cond(o, p);
                        ops.push_back(o);
                        st.flips++;
                        if (p.kind == PK_FLIPU) {
                            conj_P([&](int s) { return s ^ (1 << p.S); }, 0, 0);
                            replay.push_back({PK_FLIPU, -1, Q[p.S], 0});
                        } else {
                            replay.push_back({PK_FLIPC, p.fl_ctl, Q[p.S], p.fl_om});
                            if (p.fl_ctl >= 0) sr.flip_ctl |= 1u << p.fl_ctl;
                        }
                        break;
                    }
                }
                if (emitted) {
                    done[k] = 1;
                    ++ndone;
                    progress = true;
                }
            }
        }
        if (ndone < n) {
            // ROUND: flush P together with every ready shear that can join
            std::vector<int> rs;
            uint32_t mask = 0;
            for (int k = 0; k < n; ++k)
                if (!done[k] && ready(k) && round_bit(prims[k]) >= 0) {
                    rs.push_back(k);
                    mask |= 1u << round_bit(prims[k]);
                }
            if (!rs.empty()) {
                double par_sc[2 * 5];
                for (int r = 0; r < R; ++r) {
                    if (!((mask >> r) & 1)) continue;
                    for (int k : rs) {
                        const Prim &p = prims[k];
                        if (round_bit(p) != r) continue;
                        const double s1 = 1.0 + p.t * p.t;  // L D U: D = diag(1, 1 + t^2) on logical 1
                        for (auto &P : PV)
                            for (int sg = 0; sg < NS; ++sg)
                                if ((sg >> p.S) & 1) P[sg] *= s1;
                    }
                }
                int ns = 0;
                for (int r = 0; r < R; ++r)
                    for (int k : rs)
                        if (round_bit(prims[k]) == r) {
                            par_sc[2 * ns] = prims[k].t;
                            par_sc[2 * ns + 1] = -prims[k].t / (1.0 + prims[k].t * prims[k].t);
                            ++ns;
                        }
                LOp o{};
                o.code = LOP_CODE_ROUND;
                const int sa = add_sc(par_sc, 2 * ns);
                if (pending_tables(o) || sa < 0) return 1;
                o.gvec = (uint8_t)mask;
                o.pm = (uint32_t)sa;
                ops.push_back(o);
                st.diagt++;
                st.shears += ns;
                for (int k : rs) {
                    done[k] = 1;
                    ++ndone;
                }
                reset_P();
                continue;
            }
            if (isI()) {
                err = "internal: stage scheduler made no progress";
                return -1;
            }
            if (flush_P()) return 1;
        }
    }
    if (!isI()) {
        // carry a product-form pending diagonal instead of flushing it
        bool carried = false;
        if (allow_carry && pv_n == 0 && std::abs(PV[0][0]) > 0.0) {
            const std::vector<cd> &P = PV[0];
            const cd p0 = P[0];
            cd ratio[5];
            for (int r = 0; r < R; ++r) ratio[r] = P[1 << r] / p0;
            bool ok = true;
            for (int sg = 0; sg < NS && ok; ++sg) {
                cd pred = p0;
                for (int r = 0; r < R; ++r)
                    if ((sg >> r) & 1) pred *= ratio[r];
                ok = std::abs(pred - P[sg]) <= 1e-14 * std::abs(P[sg]);
            }
            if (ok) {
                carry_scalar *= p0;
                for (int r = 0; r < R; ++r) {
                    if (ratio[r] == cd(1.0, 0.0)) continue;
                    const int q = Q[r];
                    carry[q][0] = cd(1.0, 0.0);
                    carry[q][1] = ratio[r];
                    has_carry[q] = true;
                    st.carried++;
                }
                carried = true;
            }
        }
        if (!carried && flush_P()) return 1;
    }
    if ((int)ops.size() > LP_MAX_OPS) return 1;
    // fold FLIP ops into the table op that follows them (<= 2 per op): a flip
    // only updates the group's vector g, so applying it right before the next
    // op is the same program with one dispatch less
    {
        std::vector<LOp> merged;
        std::vector<LOp> pend;
        for (int i = sr.op0; i < (int)ops.size(); ++i) {
            const LOp &o = ops[i];
            int code = -1;
            if (o.code == LOP_CODE_FLIP) {
                if (!(o.flags & LF_COND))
                    code = 255;
                else if (o.tmask && !o.omask && __builtin_popcount(o.tmask) == 1 && o.tval == o.tmask)
                    code = __builtin_ctz(o.tmask);
                else if (!o.tmask && o.omask && __builtin_popcountll(o.omask) == 1 && o.oval == o.omask)
                    code = 64 + __builtin_ctzll(o.omask);
            }
            if (code >= 0 && pend.size() < 2) {
                LOp f = o;
                f.pm = (uint32_t)code;  // stash
                pend.push_back(f);
                continue;
            }
            const bool table = (o.code == LOP_CODE_DIAGT || o.code == LOP_CODE_ROUND) && !(o.flags & LF_COND);
            if (table && !pend.empty()) {
                LOp t = o;
                for (size_t k = 0; k < pend.size(); ++k)
                    t.pmc[k] = (1u << 16) | (pend[k].pm << 8) | pend[k].gvec;
                merged.push_back(t);
                pend.clear();
                continue;
            }
            for (const LOp &f : pend) {  // no table op next: keep them as ops
                LOp x = f;
                x.pm = 0;
                merged.push_back(x);
            }
            pend.clear();
            if (code >= 0) {  // a third flip in a row
                LOp f = o;
                f.pm = (uint32_t)code;
                pend.push_back(f);
                continue;
            }
            merged.push_back(o);
        }
        // flips after the stage's last table op: g is not read again -- the
        // tile-level relabelling (replay below) carries their effect
        ops.resize(sr.op0);
        ops.insert(ops.end(), merged.begin(), merged.end());
    }
    sr.nops = (int)ops.size() - sr.op0;
    stages.push_back(sr);
    // tile-level effect of the stage's relabels and flips
    for (const Replay &x : replay) {
        if (x.kind == PK_RELABEL) {
            ts.relabel(x.c_tbit, x.t_tbit);
        } else if (x.kind == PK_FLIPU) {
            ts.b_static ^= ts.col[x.t_tbit];
        } else if (x.c_tbit >= 0) {
            ts.relabel(x.c_tbit, x.t_tbit);
        } else {
            ts.ev_full.push_back(x.om);
            ts.ev_v.push_back(ts.col[x.t_tbit]);
        }
    }
    return 0;
}

int Compiler::run() {
    NS = 1 << R;
    NV = lp_nv(R);
    for (int v = 0; v < 32; ++v) vidx[v] = -1;
    for (int k = 0; k < NV; ++k) vidx[lp_vec(R, k)] = k;
    ts.init(K);
    std::vector<int> rem;
    for (int k = 0; k < ng; ++k) rem.push_back(k);
    while (!rem.empty()) {
        // (1) permutation gates at tile level (free: M / b updates)
        {
            uint64_t bx = 0, bz = 0;
            std::vector<int> left;
            for (int k : rem) {
                const GInfo &g = G[k];
                const bool conflict = (g.xq & (bx | bz)) || (g.zq & bx);
                if (!conflict && g.cls == GC_IDENT) continue;
                if (!conflict && is_free(g)) {
                    apply_free(g);
                    continue;
                }
                bx |= g.xq;
                bz |= g.zq;
                left.push_back(k);
            }
            rem.swap(left);
        }
        if (rem.empty()) break;
        if ((int)stages.size() >= LP_MAX_STAGES) return 1;
        // (2) one register stage: every remaining gate that commutes with the
        // skipped ones and whose non-diagonal target fits the R register slots.
        // scan(): the selection for a given initial register set; with grow,
        // gates may claim free slots first-come; dry runs change no state.
        struct Scan {
            int Q[5];
            int nq = 0;
            int slot_of[LP_MAX_K];
            uint32_t used_out = 0;
            std::vector<int> take, left;
            bool carried_any = false;
            int score = 0;
        };
        auto scan = [&](const int *Qi, int nqi, bool grow, bool dry, Scan &S) {
            int *Q = S.Q;
            int &nq = S.nq;
            int *slot_of = S.slot_of;
            uint32_t &used_out = S.used_out;
            std::vector<int> &take = S.take, &left = S.left;
            bool &carried_any = S.carried_any;
            nq = 0;
            for (int i = 0; i < LP_MAX_K; ++i) slot_of[i] = -1;
            for (int i = 0; i < nqi; ++i) {
                Q[nq] = Qi[i];
                slot_of[Qi[i]] = nq++;
            }
            uint8_t ainv[5];
            for (int r = 0; r < R; ++r) ainv[r] = (uint8_t)(1u << r);
            int nev_avail = LP_MAX_EVENTS - (int)ts.ev_v.size();
            used_out = 0;  // tile bits the stage tests outside the registers (conditions)
            std::vector<Prim> tmp;
            uint64_t bx = 0, bz = 0;
            for (int k : rem) {
                const GInfo &g = G[k];
                bool ok = !((g.xq & (bx | bz)) || (g.zq & bx));
                // an uncontrolled 1-qubit diagonal on a qubit outside the registers
                // commutes with the whole stage: carry it (or defer it out of the
                // pass when its qubit is not in the tile) -- no op, no table
                if (ok && allow_carry && g.cls == GC_DIAG && g.nci == 0 && g.om == 0 &&
                    (g.tt < 0 || slot_of[g.tt] < 0)) {
                    carried_any = true;
                    if (dry) continue;
                    const cd d0(g.u[0], g.u[1]), d1(g.u[6], g.u[7]);
                    if (g.tt >= 0) {
                        if (!has_carry[g.tt]) {
                            carry[g.tt][0] = carry[g.tt][1] = cd(1.0, 0.0);
                            has_carry[g.tt] = true;
                        }
                        carry[g.tt][0] *= d0;
                        carry[g.tt][1] *= d1;
                    } else {
                        LGate x{};
                        x.t = gates[k].t;
                        std::memcpy(x.u, g.u, sizeof(x.u));
                        out_deferred.push_back(x);
                    }
                    st.carried++;
                    carried_any = true;
                    continue;
                }
                int added = -1;
                // a diagonal gate takes a free register slot for its (tile) target:
                // then it merges into the stage's table instead of needing its own
                if (ok && grow && g.cls == GC_DIAG && g.tt >= 0 && slot_of[g.tt] < 0 && nq < R &&
                    !((used_out >> g.tt) & 1)) {
                    Q[nq] = g.tt;
                    slot_of[g.tt] = nq;
                    added = nq++;
                }
                if (ok && (g.cls == GC_ANTI || g.cls == GC_DENSE) && slot_of[g.tt] < 0) {
                    // a new register qubit: not for a free permutation (done at tile
                    // level), not a bit already tested outside the registers, room left
                    if (!grow || (is_free(g) && !take.empty()) || nq >= R || ((used_out >> g.tt) & 1))
                        ok = false;
                    else {
                        Q[nq] = g.tt;
                        slot_of[g.tt] = nq;
                        added = nq++;
                    }
                }
                uint32_t uo = used_out;
                if (ok) {
                    for (int c = 0; c < g.nci; ++c)
                        if (slot_of[g.ci[c]] < 0) uo |= 1u << g.ci[c];
                    if (g.cls == GC_DIAG && g.tt >= 0 && slot_of[g.tt] < 0) uo |= 1u << g.tt;
                    if (__builtin_popcount(uo) + R > K) ok = false;  // padding must find untested bits
                }
                int nev2 = nev_avail;
                uint8_t ainv2[5];
                std::memcpy(ainv2, ainv, sizeof(ainv2));
                if (ok) {
                    // the prims this gate becomes: every register pair vector must have weight <= 2
                    tmp.clear();
                    PrimBuilder pb{R, NS, slot_of, nev_avail, &tmp};
                    pb.gate(g);
                    nev2 = pb.nev_avail;
                    for (const Prim &p : tmp) {
                        // shears take pair vectors of weight <= 2; the rare controlled
                        // ops (general 2x2, controlled shear / swap) weight 1
                        const bool w1 = p.kind == PK_DENSE || p.kind == PK_CSWAP || (p.kind == PK_SHEAR && p.cs);
                        if (p.kind == PK_SHEAR && vidx[ainv2[p.S]] < 0) ok = false;
                        if (w1 && __builtin_popcount(ainv2[p.S]) != 1) ok = false;
                        if (p.kind == PK_RELABEL) ainv2[p.rc] ^= ainv2[p.S];
                    }
                }
                if (ok) {
                    take.push_back(k);
                    S.score += g.cls == GC_DENSE ? 4 : (g.cls == GC_ANTI ? 1 : 0);
                    if (g.cls == GC_ANTI && g.tt >= 0 && slot_of[g.tt] >= 0) {  // an in-stage flip costs an op
                        bool inq = false;
                        for (int c = 0; c < g.nci; ++c) inq = inq || slot_of[g.ci[c]] >= 0;
                        if (!inq && (g.nci > 0 || g.om)) S.score -= flip_penalty;
                    }
                    used_out = uo;
                    nev_avail = nev2;
                    std::memcpy(ainv, ainv2, sizeof(ainv));
                } else {
                    if (added >= 0) {
                        slot_of[Q[added]] = -1;
                        --nq;
                    }
                    bx |= g.xq;
                    bz |= g.zq;
                    left.push_back(k);
                }
            }
        };
        // register set by greedy lookahead: add the tile qubit that lets the
        // stage take the most gates (dense gates weigh most: they share tables)
        int Qsel[5];
        int nsel = 0;
        if (lookahead) {
            Scan base;
            scan(Qsel, 0, false, true, base);
            int best_score = base.score;
            uint32_t cand = 0;
            for (int k : rem)
                if ((G[k].cls == GC_DENSE || G[k].cls == GC_ANTI) && G[k].tt >= 0) cand |= 1u << G[k].tt;
            while (nsel < R) {
                int best = -1;
                for (int c = 0; c < K; ++c) {
                    if (!((cand >> c) & 1)) continue;
                    bool in = false;
                    for (int i = 0; i < nsel; ++i) in = in || Qsel[i] == c;
                    if (in) continue;
                    Qsel[nsel] = c;
                    Scan tr;
                    scan(Qsel, nsel + 1, false, true, tr);
                    if (tr.score > best_score) {
                        best_score = tr.score;
                        best = c;
                    }
                }
                if (best < 0) break;
                Qsel[nsel++] = best;
            }
        }
        Scan S;
        scan(Qsel, nsel, true, false, S);
        {
            // a permutation gate the tile level can apply for free (is_free) that
            // no later gate of the stage depends on goes back to the remaining
            // gates: it is then a relabelling after the stage, not an in-stage
            // flip (one op per group, and divergent flip vectors)
            std::vector<int> keep, back;
            uint64_t lx = 0, lz = 0;  // qubits used by the later kept gates
            for (int i = (int)S.take.size() - 1; i >= 0; --i) {
                const int k = S.take[i];
                const GInfo &g = G[k];
                const bool later_dep = (g.xq & (lx | lz)) || (g.zq & lx);
                if (g.pure && is_free(g) && !later_dep && !(g.nci == 1 && S.slot_of[g.ci[0]] >= 0)) {
                    back.push_back(k);
                    continue;
                }
                keep.push_back(k);
                lx |= g.xq;
                lz |= g.zq;
            }
            if (!back.empty()) {
                std::reverse(keep.begin(), keep.end());
                S.take.swap(keep);
                S.left.insert(S.left.end(), back.begin(), back.end());
                std::sort(S.left.begin(), S.left.end());
            }
        }
        int *Q = S.Q;
        int &nq = S.nq;
        int *slot_of = S.slot_of;
        const uint32_t used_out = S.used_out;
        std::vector<int> &take = S.take, &left = S.left;
        const bool carried_any = S.carried_any;
        if (take.empty()) {
            if (carried_any) {
                rem.swap(left);
                continue;
            }
            err = "internal: no gate fits a register stage";
            return -1;
        }
        // pad the register set with tile bits the stage does not test
        for (int b = 0; nq < R && b < K; ++b)
            if (slot_of[b] < 0 && !((used_out >> b) & 1)) {
                Q[nq] = b;
                slot_of[b] = nq++;
            }
        const int rc = compile_stage(take, Q);
        if (rc) return rc;
        rem.swap(left);
    }
    return 0;
}

// Low-3-bit rank of a set of vectors (bank groups of 16-byte elements).
int rank3(const uint16_t *v, int n) {
    int basis[3] = {0, 0, 0};
    int r = 0;
    for (int i = 0; i < n; ++i) {
        int x = v[i] & 7;
        for (int b = 2; b >= 0; --b) {
            if (!((x >> b) & 1)) continue;
            if (!basis[b]) {
                basis[b] = x;
                ++r;
                break;
            }
            x ^= basis[b];
        }
    }
    return r;
}

}  // namespace

int lpass_compile(const LGate *gates, int ng, int nl, int K, int R, const int *tile_q, int max_coef,
                  LPassParams &p, LCompileStats *stats, std::string *err, std::vector<LGate> *deferred) {
    if (K < LP_MIN_K || K > LP_MAX_K || K > nl || (R != 4 && R != 5) || ng > LP_MAX_PASS_GATES ||
        max_coef > LP_MAX_COEF) {
        if (err) *err = "lpass_compile: bad arguments";
        return -1;
    }
    Compiler c;
    c.gates = gates;
    c.ng = ng;
    c.nl = nl;
    c.K = K;
    c.R = R;
    c.max_coef = max_coef;
    c.allow_carry = deferred != nullptr;
    // the lookahead costs host time per stage: worth it when a pass is long
    // (2^(nl-K) >= 1024 tiles); small states keep first-come register sets
    c.lookahead = nl - K >= 10 ? 1 : 0;
    if (const char *e = getenv("LPASS_LOOKAHEAD")) c.lookahead = atoi(e);
    if (const char *e = getenv("LPASS_FLIP_PENALTY")) c.flip_penalty = atoi(e);
    for (int q = 0; q < 64; ++q) c.tbit_of[q] = -1;
    for (int i = 0; i < K; ++i) c.tbit_of[tile_q[i]] = i;
    c.G.resize(ng);
    for (int k = 0; k < ng; ++k) {
        const LGate &x = gates[k];
        GInfo &g = c.G[k];
        g.u = x.u;
        g.cls = gclass(x.u);
        g.pure = g.cls == GC_ANTI && x.u[2] == 1.0 && x.u[3] == 0.0 && x.u[4] == 1.0 && x.u[5] == 0.0;
        g.tt = (x.t < nl) ? c.tbit_of[x.t] : -1;
        g.tfull = 1ull << x.t;
        if ((g.cls == GC_ANTI || g.cls == GC_DENSE) && g.tt < 0) {
            if (err) *err = "lpass_compile: non-diagonal target outside the tile";
            return -1;
        }
        for (int j = 0; j < x.nctl; ++j) {
            const int q = x.ctl[j];
            if (q < nl && c.tbit_of[q] >= 0)
                g.ci[g.nci++] = c.tbit_of[q];
            else
                g.om |= 1ull << q;
            g.zq |= 1ull << q;
        }
        if (g.cls == GC_DIAG)
            g.zq |= 1ull << x.t;
        else if (g.cls != GC_IDENT)
            g.xq |= 1ull << x.t;
        if (g.cls == GC_IDENT) g.zq = g.xq = 0;
    }
    int rc = c.run();
    if (rc == 0 && (int)c.coef.size() > max_coef) rc = 1;
    int p_ts_off = 0, p_nts = 0, p_ts_slot = 0;
    if (rc) {
        if (err) *err = c.err;
        return rc;
    }
    // Per-tile hoisting (values that are the same for every group of a tile).
    // (1) Conditional scalars (a DIAG1 with T0 == T1 whose condition is on
    // full-index bits only: a CPHASE with both qubits outside the tile) commute
    // with every op of the pass: they become one product per tile (terms
    // (omask, oval, e) in sc, formed in lp_body into a coefficient-pool slot)
    // applied at the tile store, and the op a no-op (FLIP with gvec 0).
    // the per-tile products are formed serially while the tile loads: worth it
    // when a pass has many tiles (>= 1024, as the lookahead); on small,
    // latency-bound passes it measured 2 us slower per config-1 circuit
    // (LPASS_HOIST=1 / 0 forces it on / off)
    static const int hoist_env = getenv("LPASS_HOIST") ? atoi(getenv("LPASS_HOIST")) : -1;
    const bool hoist = hoist_env < 0 ? nl - K >= 10 : hoist_env != 0;
    std::vector<size_t> ts_ops;
    for (size_t i = 0; i < c.ops.size() && hoist; ++i) {
        const LOp &o = c.ops[i];
        if (o.code != LOP_CODE_DIAG1 || !(o.flags & LF_COND) || o.tmask || !o.omask) continue;
        const double *T = &c.sc[o.coef];
        if (T[0] == T[2] && T[1] == T[3]) ts_ops.push_back(i);
    }
    if (!ts_ops.empty() && (int)c.sc.size() + 4 * (int)ts_ops.size() <= LP_MAX_SC &&
        (int)((c.coef.size() + 1) & ~(size_t)1) + 2 <= max_coef) {  // else they stay DIAG1 ops
        p_ts_off = (int)c.sc.size();
        p_nts = (int)ts_ops.size();
        for (size_t i : ts_ops) {
            LOp &o = c.ops[i];
            double term[4];
            std::memcpy(&term[0], &o.omask, 8);
            std::memcpy(&term[1], &o.oval, 8);
            term[2] = c.sc[o.coef];
            term[3] = c.sc[o.coef + 1];
            c.sc.insert(c.sc.end(), term, term + 4);
            o.code = LOP_CODE_FLIP;
            o.flags = 0;
            o.gvec = 0;
        }
        if (c.coef.size() & 1) c.coef.push_back(0.0);
        p_ts_slot = (int)c.coef.size();
        c.coef.push_back(1.0);
        c.coef.push_back(0.0);
    }
    // (2) PHASES terms conditioned on full-index bits (outside the tile): move
    // them to the front of the op's term list (stable; the phases commute) and
    // give the op a 2-double slot at the end of the coefficient pool, which the
    // kernel fills once per tile (lp_body); the op then multiplies only its
    // tile-bit terms per group.  pmc[0] = slot offset in coef (doubles),
    // pmc[1] = number of hoisted terms.
    int nops_ph = 0;
    for (size_t i = 0; i < c.ops.size() && hoist; ++i) {
        LOp &o = c.ops[i];
        if (o.code != LOP_CODE_PHASES) continue;
        std::vector<double> full_t, tile_t;
        for (int k = 0; k < o.nctl; ++k) {
            std::vector<double> &dst = c.sc[o.coef + 3 * k] >= 64.0 ? full_t : tile_t;
            for (int j = 0; j < 3; ++j) dst.push_back(c.sc[o.coef + 3 * k + j]);
        }
        if (full_t.empty() || (int)((c.coef.size() + 1) & ~(size_t)1) + 2 > max_coef) continue;
        if (c.coef.size() & 1) c.coef.push_back(0.0);  // 16-byte aligned slot
        const size_t nfull = full_t.size() / 3;
        for (double x : tile_t) full_t.push_back(x);
        std::memcpy(&c.sc[o.coef], full_t.data(), full_t.size() * sizeof(double));
        o.pmc[0] = (uint32_t)c.coef.size();
        o.pmc[1] = (uint32_t)nfull;
        c.coef.push_back(1.0);
        c.coef.push_back(0.0);
        nops_ph = (int)i + 1;
    }
    if (deferred) {
        // still-carried diagonals: the caller applies them right after the pass
        deferred->clear();
        cd scal = c.carry_scalar;
        for (int q = 0; q < K; ++q) {
            if (!c.has_carry[q]) continue;
            LGate g{};
            g.t = tile_q[q];
            const cd d0 = c.carry[q][0] * scal, d1 = c.carry[q][1] * scal;
            scal = cd(1.0, 0.0);
            g.u[0] = d0.real();
            g.u[1] = d0.imag();
            g.u[6] = d1.real();
            g.u[7] = d1.imag();
            deferred->push_back(g);
        }
        for (const LGate &x : c.out_deferred) deferred->push_back(x);
        if (scal != cd(1.0, 0.0)) {
            LGate g{};
            g.t = tile_q[0];
            g.u[0] = g.u[6] = scal.real();
            g.u[1] = g.u[7] = scal.imag();
            deferred->push_back(g);
        }
        c.st.deferred = (int)deferred->size();
    }
    // ---- swizzle: S p = p ^ (sum over high bits i of p of stuff[i]) in the low 3 bits.
    // Loads read logical x at S x (conflict-free: S e_i = e_i for i < 3); the
    // store reads S (M_f x ^ b): choose stuff so S M_f e_0..2 have independent bank bits.
    uint16_t stuff[LP_MAX_K] = {0};
    auto Sw = [&](uint16_t x) {
        uint16_t y = x;
        for (int i = LP_LOW; i < K; ++i)
            if ((x >> i) & 1) y ^= stuff[i];
        return y;
    };
    uint32_t lcg = 12345u;
    for (int attempt = 0; attempt < 256; ++attempt) {
        for (int i = LP_LOW; i < K; ++i) {
            if (attempt == 0) {
                stuff[i] = (uint16_t)(1u << (i % 3));
            } else {
                lcg = lcg * 1664525u + 1013904223u;
                stuff[i] = (uint16_t)((lcg >> 13) & 7u);
            }
        }
        uint16_t v[3];
        for (int i = 0; i < 3; ++i) v[i] = Sw(c.ts.col[i]);
        if (rank3(v, 3) == 3) break;
    }
    std::memset(&p, 0, sizeof(p));
    p.nl = nl;
    p.K = K;
    p.R = R;
    p.ntiles = 1ull << (nl - K);
    for (int i = LP_LOW; i < K; ++i) p.high_q[i - LP_LOW] = tile_q[i];
    for (int i = 0; i < K; ++i) {
        p.scol[i] = Sw((uint16_t)(1u << i));
        p.smcol[i] = Sw(c.ts.col[i]);
    }
    p.sb_static = Sw(c.ts.b_static);
    p.nevents = (int)c.ts.ev_v.size();
    for (int e = 0; e < p.nevents; ++e) {
        p.sv_ev[e] = Sw(c.ts.ev_v[e]);
        p.ev_full[e] = c.ts.ev_full[e];
    }
    p.nstages = (int)c.stages.size();
    for (int s = 0; s < p.nstages; ++s) {
        const StageRec &sr = c.stages[s];
        LStage &ls = p.st[s];
        uint16_t qm = 0;
        for (int r = 0; r < R; ++r) {
            ls.reg_phys[r] = Sw(sr.col[sr.Q[r]]);
            ls.qbit[r] = (uint8_t)sr.Q[r];
            qm |= (uint16_t)(1u << sr.Q[r]);
        }
        ls.qmask = qm;
        // group bits: three with independent bank bits first (conflict-free
        // quarter warps), then the other lane bits; bits that condition an
        // in-stage flip go to the warp / loop positions (>= 5) when possible so
        // that g -- and the orientation of later shears -- stays warp-uniform
        std::vector<int> rest, gb;
        for (int b = 0; b < K; ++b)
            if (!((qm >> b) & 1) && !((sr.flip_ctl >> b) & 1)) rest.push_back(b);
        for (int b = 0; b < K; ++b)
            if (!((qm >> b) & 1) && ((sr.flip_ctl >> b) & 1)) rest.push_back(b);
        uint16_t chosen[3];
        int nch = 0;
        for (size_t k = 0; k < rest.size() && nch < 3;) {
            chosen[nch] = Sw(sr.col[rest[k]]);
            if (rank3(chosen, nch + 1) == nch + 1) {
                gb.push_back(rest[k]);
                rest.erase(rest.begin() + k);
                ++nch;
            } else {
                ++k;
            }
        }
        for (int b : rest) gb.push_back(b);
        // positions 3, 4 (lane bits): prefer bits that do not condition flips
        for (int pos = 3; pos < 5 && pos < (int)gb.size(); ++pos)
            if ((sr.flip_ctl >> gb[pos]) & 1)
                for (int k = 5; k < (int)gb.size(); ++k)
                    if (!((sr.flip_ctl >> gb[k]) & 1)) {
                        std::swap(gb[pos], gb[k]);
                        break;
                    }
        for (int i = 0; i < K - R; ++i) {
            ls.grp_phys[i] = Sw(sr.col[gb[i]]);
            ls.grp_log[i] = (uint16_t)(1u << gb[i]);
        }
        TileState tsn;
        tsn.K = K;
        std::memcpy(tsn.row, sr.row, sizeof(tsn.row));
        ls.y_static = tsn.logical(sr.b_static);
        ls.ev_mask = (sr.nev >= 32) ? 0xffffffffu : ((1u << sr.nev) - 1u);
        for (int e = 0; e < sr.nev; ++e) ls.y_ev[e] = tsn.logical(c.ts.ev_v[e]);
        ls.needs_xq = sr.needs_xq ? 1 : 0;
        ls.first_op = (uint16_t)sr.op0;
        ls.nops = (uint16_t)sr.nops;
    }
    p.ncoef = (int)c.coef.size();
    p.nsc = (int)c.sc.size();
    p.nops_ph = nops_ph;
    p.nts = p_nts;
    p.ts_off = p_ts_off;
    p.ts_slot = p_ts_slot;
    std::memcpy(p.op, c.ops.data(), c.ops.size() * sizeof(LOp));
    std::memcpy(p.coef, c.coef.data(), c.coef.size() * sizeof(double));
    std::memcpy(p.sc, c.sc.data(), c.sc.size() * sizeof(double));
    c.st.stages = p.nstages;
    c.st.ops = (int)c.ops.size();
    c.st.events = p.nevents;
    if (stats) *stats = c.st;
    return 0;
}

int lpass_run(const LGate *gates, int ng, const LRunConfig &cfg, LPassSink &sink, std::string *err) {
    const int K = cfg.K, nl = cfg.nl, hmax = K - LP_LOW;
    struct Item {
        LGate g;
        int id;
        uint64_t xq, zq;
        bool needs_reg;
    };
    auto mk = [&](const LGate &g, int id) {
        Item it{g, id, 0, 0, false};
        const int cls = gclass(g.u);
        if (cls == GC_DIAG)
            it.zq |= 1ull << g.t;
        else if (cls != GC_IDENT)
            it.xq |= 1ull << g.t;
        for (int c = 0; c < g.nctl; ++c) it.zq |= 1ull << g.ctl[c];
        if (cls == GC_IDENT) it.xq = it.zq = 0;
        it.needs_reg = cls == GC_ANTI || cls == GC_DENSE;
        return it;
    };
    std::vector<Item> pend;
    for (int k = 0; k < ng; ++k) pend.push_back(mk(gates[k], k));
    static thread_local LPassParams prog;
    std::vector<LGate> lg, dfr;
    std::vector<int> sel, ids;
    // Greedy pass selection: every pending gate (in order) that commutes with
    // all skipped earlier ones and whose non-diagonal target fits the tile's
    // hmax free qubits (first come, first served), qubits in `forbid` never
    // joining the tile.  Score: dense / permutation gates 1, others 0.3.
    static const double w_other = getenv("LPASS_W") ? atof(getenv("LPASS_W")) : 0.3;
    static const int best_impr = getenv("LPASS_BEST") ? atoi(getenv("LPASS_BEST")) : 0;
    static const bool pairs_ok = getenv("LPASS_PAIRS") ? atoi(getenv("LPASS_PAIRS")) != 0 : true;
    // score of the plain greedy pass over the gates not in `skip` (the pass
    // that would follow): the search's two-pass lookahead
    auto next_score = [&](const std::vector<char> &skip) {
        std::vector<int> hi;
        uint64_t bx = 0, bz = 0;
        double score = 0.0;
        int nsel = 0;
        for (size_t k = 0; k < pend.size() && nsel < LP_MAX_PASS_GATES; ++k) {
            if (skip[k]) continue;
            const Item &it = pend[k];
            bool ok = !((it.xq & (bx | bz)) || (it.zq & bx));
            if (ok && it.needs_reg) {
                const int t = it.g.t;
                if (t >= LP_LOW && std::find(hi.begin(), hi.end(), t) == hi.end()) {
                    if ((int)hi.size() >= hmax)
                        ok = false;
                    else
                        hi.push_back(t);
                }
                if (ok && it.g.nctl == 1) {
                    const int c = it.g.ctl[0];
                    if (c >= LP_LOW && c < nl && (int)hi.size() < hmax &&
                        std::find(hi.begin(), hi.end(), c) == hi.end())
                        hi.push_back(c);
                }
            }
            if (ok) {
                ++nsel;
                score += it.needs_reg ? 1.0 : w_other;
            } else {
                bx |= it.xq;
                bz |= it.zq;
            }
        }
        return score;
    };
    static const double beta = getenv("LPASS_SCORE2") ? atof(getenv("LPASS_SCORE2")) : 0.75;
    auto select1 = [&](uint64_t forbid, std::vector<int> &sel_, std::vector<int> &high_, std::vector<char> &done_) {
        done_.assign(pend.size(), 0);
        high_.clear();
        sel_.clear();
        auto in_high = [&](int q) { return std::find(high_.begin(), high_.end(), q) != high_.end(); };
        uint64_t bx = 0, bz = 0;
        double score = 0.0;
        for (size_t k = 0; k < pend.size() && (int)sel_.size() < LP_MAX_PASS_GATES; ++k) {
            const Item &it = pend[k];
            bool ok = !((it.xq & (bx | bz)) || (it.zq & bx));
            if (ok && it.needs_reg) {
                const int t = it.g.t;
                if (t >= LP_LOW && !in_high(t)) {
                    if ((int)high_.size() >= hmax || ((forbid >> t) & 1ull))
                        ok = false;
                    else
                        high_.push_back(t);
                }
                // a local control in the tile makes a CNOT a tile relabelling
                if (ok && it.g.nctl == 1) {
                    const int c = it.g.ctl[0];
                    if (c >= LP_LOW && c < nl && (int)high_.size() < hmax && !in_high(c) && !((forbid >> c) & 1ull))
                        high_.push_back(c);
                }
            }
            if (ok) {
                done_[k] = 1;
                sel_.push_back((int)k);
                score += it.needs_reg ? 1.0 : w_other;
            } else {
                bx |= it.xq;
                bz |= it.zq;
            }
        }
        return score;
    };
    auto select = [&](uint64_t forbid, std::vector<int> &sel_, std::vector<int> &high_, std::vector<char> &done_) {
        const double s1 = select1(forbid, sel_, high_, done_);
        return beta > 0.0 ? s1 + beta * next_score(done_) : s1;
    };
    // the search costs host time per pass: small states (< 1024 tiles) skip it
    static const int search_env = getenv("LPASS_SEARCH") ? atoi(getenv("LPASS_SEARCH")) : -1;
    const int search = search_env >= 0 ? search_env : (nl - K >= 10 ? 3 : 0);
    while (!pend.empty()) {
        std::vector<char> done;
        std::vector<int> high;
        double best = select(0, sel, high, done);
        // local search over the tile's qubits: keep one of them out when that
        // lets more gates into the pass (a qubit whose gates come early but
        // block many others), a few rounds
        uint64_t forbid = 0;
        for (int round = 0; round < search; ++round) {
            bool improved = false;
            const std::vector<int> h0 = high;
            uint64_t fbest = forbid;
            for (int q : h0) {
                std::vector<int> s2, h2;
                std::vector<char> d2;
                const uint64_t f = (best_impr ? forbid : fbest) | (1ull << q);
                const double sc = select(f, s2, h2, d2);
                if (sc > best + 1e-9) {
                    best = sc;
                    sel.swap(s2);
                    high.swap(h2);
                    done.swap(d2);
                    fbest = f;
                    improved = true;
                }
            }
            forbid = fbest;
            if (!improved && pairs_ok) {  // no single exclusion helps: try pairs
                for (size_t a = 0; a < h0.size() && !improved; ++a)
                    for (size_t b2 = a + 1; b2 < h0.size(); ++b2) {
                        std::vector<int> s2, h2;
                        std::vector<char> d2;
                        const uint64_t f = forbid | (1ull << h0[a]) | (1ull << h0[b2]);
                        const double sc = select(f, s2, h2, d2);
                        if (sc > best + 1e-9) {
                            best = sc;
                            sel.swap(s2);
                            high.swap(h2);
                            done.swap(d2);
                            fbest = f;
                            improved = true;
                        }
                    }
                forbid = fbest;
            }
            if (!improved) break;
        }
        if (getenv("LPASS_TRACE")) fprintf(stderr, "lpass_run: pending %zu, pass %zu\n", pend.size(), sel.size());
        LCompileStats cs;
        int rc = 1;
        bool deferred_ok = false;
        while (rc == 1 && !sel.empty()) {
            std::vector<int> hq;
            for (int k : sel)
                if (pend[k].needs_reg && pend[k].g.t >= LP_LOW && std::find(hq.begin(), hq.end(), pend[k].g.t) == hq.end())
                    hq.push_back(pend[k].g.t);
            for (int q : high)  // controls pulled into the tile, while they fit
                if ((int)hq.size() < hmax && std::find(hq.begin(), hq.end(), q) == hq.end()) hq.push_back(q);
            for (int q = LP_LOW; (int)hq.size() < hmax && q < nl; ++q)
                if (std::find(hq.begin(), hq.end(), q) == hq.end()) hq.push_back(q);
            std::sort(hq.begin(), hq.end());
            int tq[LP_MAX_K];
            for (int i = 0; i < LP_LOW; ++i) tq[i] = i;
            for (int i = 0; i < hmax; ++i) tq[LP_LOW + i] = hq[i];
            lg.clear();
            for (int k : sel) lg.push_back(pend[k].g);
            int nreal = 0;
            for (int k : sel) nreal += pend[k].id >= 0;
            // progress: the pass holding every pending gate, or no circuit gate, defers nothing
            deferred_ok = cfg.defer && sel.size() != pend.size() && nreal > 0;
            std::string e2;
            rc = lpass_compile(lg.data(), (int)lg.size(), nl, K, cfg.R, tq, cfg.max_coef, prog, &cs, &e2,
                               deferred_ok ? &dfr : nullptr);
            if (rc < 0) {
                if (err) *err = e2;
                return -1;
            }
            if (rc == 1) {
                done[sel.back()] = 0;
                sel.pop_back();
            }
        }
        if (!deferred_ok) dfr.clear();
        double sweep_bytes = 0.0;
        for (int k : sel) sweep_bytes += sink.gate_bytes(pend[k].g);
        if (rc == 0 && sel.size() >= 2 && cfg.pass_bytes < sweep_bytes) {
            ids.clear();
            for (int k : sel) ids.push_back(pend[k].id);
            const int r2 = sink.pass(prog, cs, ids);
            if (r2) return r2;
        } else {
            dfr.clear();
            for (int k : sel) {
                const int r2 = sink.sweep(pend[k].g, pend[k].id);
                if (r2) return r2;
            }
        }
        std::vector<Item> next;
        for (const LGate &g : dfr)
            if (gclass(g.u) != GC_IDENT) next.push_back(mk(g, -1));
        for (size_t k = 0; k < pend.size(); ++k)
            if (!done[k]) next.push_back(pend[k]);
        pend.swap(next);
    }
    return 0;
}

// The specialised kernel: the tile's stages in order, each an lp_stage call
// with the stage as a literal LStage and a functor holding its ops as literal
// LOps (lp_op1 folds to straight-line code); the tile width is a template
// constant.
std::string lpass_jit_source(const LPassParams &p, int R, int minb, int nt, int ng) {
    std::string s;
    s.reserve(8192);
    s += "#include \"lpass_dev.cuh\"\n";
    char buf[640];
    for (int st = 0; st < p.nstages; ++st) {
        snprintf(buf, sizeof buf,
                 "template <int R>\nstruct JitOps%d {\n  __device__ __forceinline__ void operator()(double2 (&v)[1 << R], "
                 "uint32_t &g, uint32_t xq, uint64_t full, const qsim::LPassParams &p, const unsigned char *smem, "
                 "uint32_t cpool_off) const {\n",
                 st);
        s += buf;
        for (int i = p.st[st].first_op; i < p.st[st].first_op + p.st[st].nops; ++i) {
            // the whole op as a literal: conditions, parities, pre-flips and
            // coefficient offsets fold into the code
            const LOp &o = p.op[i];
            uint64_t h;
            std::memcpy(&h, &o, 8);
            snprintf(buf, sizeof buf,
                     "    { constexpr qsim::LOp o{%u, %u, %u, %u, %u, %u, %u, %uu, {%uu, %uu}, {%u, %u}, 0, %u, %u, 0, "
                     "0x%llxull, 0x%llxull};\n",
                     o.code, o.flags, o.rowS, o.gvec, o.coef, o.nctl, o.pad0, o.pm, o.pmc[0], o.pmc[1], o.rowc[0],
                     o.rowc[1], o.tmask, o.tval, (unsigned long long)o.omask, (unsigned long long)o.oval);
            s += buf;
            snprintf(buf, sizeof buf, "      qsim::lp_op1<R>(v, g, xq, full, 0x%016llxull, o, p, smem, cpool_off); }\n",
                     (unsigned long long)h);
            s += buf;
        }
        s += "  }\n};\n";
    }
    s += "struct JitStages {\n  const qsim::LPassParams &p;\n  __device__ __forceinline__ void operator()(const "
         "qsim::LpTile &t) const {\n";
    for (int st = 0; st < p.nstages; ++st) {
        const LStage &S = p.st[st];
        std::string ev = "{";
        for (int e = 0; e < LP_MAX_EVENTS; ++e) ev += std::to_string(S.y_ev[e]) + (e + 1 < LP_MAX_EVENTS ? "," : "}");
        snprintf(buf, sizeof buf,
                 "    { constexpr qsim::LStage S{{%u,%u,%u,%u,%u}, {%u,%u,%u,%u,%u,%u,%u,%u}, {%u,%u,%u,%u,%u,%u,%u,%u}, "
                 "%u, %u, {%u,%u,%u,%u,%u}, %u, %u, %u, %uu, ",
                 S.reg_phys[0], S.reg_phys[1], S.reg_phys[2], S.reg_phys[3], S.reg_phys[4], S.grp_phys[0],
                 S.grp_phys[1], S.grp_phys[2], S.grp_phys[3], S.grp_phys[4], S.grp_phys[5], S.grp_phys[6],
                 S.grp_phys[7], S.grp_log[0], S.grp_log[1], S.grp_log[2], S.grp_log[3], S.grp_log[4], S.grp_log[5],
                 S.grp_log[6], S.grp_log[7], S.y_static, S.qmask, S.qbit[0], S.qbit[1], S.qbit[2], S.qbit[3],
                 S.qbit[4], S.needs_xq, S.first_op, S.nops, S.ev_mask);
        s += buf;
        s += ev + "};\n";
        snprintf(buf, sizeof buf, "      qsim::lp_stage<%d, %d, JitOps%d<%d>, %d, %d>(p, t, S, JitOps%d<%d>{}); }\n", R,
                 p.K, st, R, nt, ng, st, R);
        s += buf;
    }
    s += "  }\n};\n";
    snprintf(buf, sizeof buf,
             "extern \"C\" __global__ void __launch_bounds__(%d, %d) k_lpass_jit(const __grid_constant__ "
             "qsim::LPassParams p) { qsim::lp_body<%d, %d, JitStages, %d>(p, JitStages{p}); }\n",
             nt, minb, R, p.K, nt);
    s += buf;
    return s;
}

}  // namespace qsim
