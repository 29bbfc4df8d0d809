// planner.cpp -- host-side gate classification and the global/local plan
// (SURVEY.md §8(a) rows a2 and a7).
//
// The state is split over P = 2^k shards by the top k physical index bits
// (§3.2, 374-379).  A gate whose target sits on a global bit "needs
// to exchange data between compute nodes"; as in JUQCS the
// exchange is implemented "by swapping nonlocal qubits and local ones and
// keeping track of these swaps by updating the permutation of the N bit
// indices".  Swaps are never undone ("defers swaps").
// Diagonal gates never exchange: their phase depends only on index bits,
// rank bits included.  Controls on global bits become a per-shard predicate.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>

#include "internal.h"

namespace qsim {

int32_t classify(const double u[8]) {
    bool off0 = u[2] == 0.0 && u[3] == 0.0 && u[4] == 0.0 && u[5] == 0.0;
    bool diag0 = u[0] == 0.0 && u[1] == 0.0 && u[6] == 0.0 && u[7] == 0.0;
    if (off0) {
        if (u[0] == 1.0 && u[1] == 0.0 && u[6] == 1.0 && u[7] == 0.0) return CLS_IDENT;
        return CLS_DIAG;
    }
    if (diag0) return CLS_ANTI;
    return CLS_DENSE;
}

static bool is_unitary(const double u[8], double tol) {
    // U^dagger U - I, U = [[a, b], [c, d]]
    double ar = u[0], ai = u[1], br = u[2], bi = u[3], cr = u[4], ci = u[5], dr = u[6], di = u[7];
    double m00 = ar * ar + ai * ai + cr * cr + ci * ci - 1.0;
    double m11 = br * br + bi * bi + dr * dr + di * di - 1.0;
    // (U^dag U)_01 = conj(a) b + conj(c) d
    double m01r = ar * br + ai * bi + cr * dr + ci * di;
    double m01i = ar * bi - ai * br + cr * di - ci * dr;
    return std::fabs(m00) <= tol && std::fabs(m11) <= tol && std::fabs(m01r) <= tol && std::fabs(m01i) <= tol;
}

int validate_gates(int n, const qsim_gate *gates, size_t ngates, bool check_unitary) {
    for (size_t g = 0; g < ngates; ++g) {
        const qsim_gate &q = gates[g];
        auto bad = [&](const char *why) {
            set_error("gate " + std::to_string(g) + ": " + why);
            return QSIM_EINVAL;
        };
        if (q.target < 0 || q.target >= n) return bad("target out of range");
        if (q.kind == QSIM_GATE_SWAP) {
            if (q.target2 < 0 || q.target2 >= n) return bad("target2 out of range");
            if (q.target2 == q.target) return bad("SWAP of a qubit with itself");
            continue;
        }
        if (q.kind != QSIM_GATE_U) return bad("unknown kind");
        if (q.ncontrols < 0 || q.ncontrols > 2) return bad("ncontrols must be 0..2");
        for (int c = 0; c < q.ncontrols; ++c) {
            if (q.controls[c] < 0 || q.controls[c] >= n) return bad("control out of range");
            if (q.controls[c] == q.target) return bad("control equals target");
        }
        if (q.ncontrols == 2 && q.controls[0] == q.controls[1]) return bad("duplicate controls");
        for (int k = 0; k < 8; ++k)
            if (!std::isfinite(q.u[k])) return bad("non-finite matrix entry");
        if (check_unitary && !is_unitary(q.u, 1e-10)) {
            set_error("gate " + std::to_string(g) + ": ||U^dagger U - I||_max > 1e-10");
            return QSIM_ENOTUNITARY;
        }
    }
    return QSIM_OK;
}

void Planner::init(int n_, int nshards, const int *initial_map) {
    n = n_;
    int k = 0;
    while ((1 << k) < nshards) ++k;
    nl = n - k;
    pos.assign(n, 0);
    inv.assign(n, 0);
    for (int q = 0; q < n; ++q) pos[q] = initial_map ? initial_map[q] : q;
    for (int q = 0; q < n; ++q) inv[pos[q]] = q;
}

void Planner::swap_bits(int a, int b) {
    int qa = inv[a], qb = inv[b];
    inv[a] = qb;
    inv[b] = qa;
    pos[qa] = b;
    pos[qb] = a;
}

// Victim local bit for an exchange (reading R-A17: any choice gives the same
// logical state; it is a performance choice).  Candidates are the top 8 local
// bits (so exchanged halves are long contiguous runs), excluding the bits the
// current gate uses.  With lookahead, pick the one whose logical qubit is next
// needed as a non-diagonal target furthest in the future (Belady); else the
// highest candidate.
int Planner::choose_victim(const qsim_gate *gates, size_t ngates, size_t cur, const int *avoid, int navoid,
                           bool lookahead, bool wide) {
    // candidates: the top 8 local bits for a pairwise exchange (its half-shard
    // slot is contiguous in runs of 2^l amplitudes: the NCCL chunks); an
    // all-to-all remap packs its blocks, so its victims may come from every
    // local bit >= min(QSIM_VICTIM_FLOOR = 12, nl - 8): Belady then finds
    // qubits the coming gates do not need (config 3, N = 36 / P = 8: 15.6 ->
    // 11.9 shard-equivalents of exchange per GPU)
    static const int floor_bit = getenv("QSIM_VICTIM_FLOOR") ? atoi(getenv("QSIM_VICTIM_FLOOR")) : 12;
    int lo = wide ? std::min(floor_bit, nl - 8) : nl - 8;
    if (lo < 0) lo = 0;
    int best = -1;
    int64_t best_next = -1;
    for (int l = nl - 1; l >= lo; --l) {
        bool skip = false;
        for (int a = 0; a < navoid; ++a)
            if (avoid[a] == l) skip = true;
        if (skip) continue;
        int64_t next = std::numeric_limits<int64_t>::max();
        if (lookahead) {
            int q = inv[l];
            for (size_t g = cur + 1; g < ngates; ++g) {
                const qsim_gate &x = gates[g];
                if (x.kind == QSIM_GATE_SWAP) {
                    if (x.target == q || x.target2 == q) break;  // relabelled: stop tracking (rare)
                    continue;
                }
                if (x.target == q && classify(x.u) != CLS_DIAG && classify(x.u) != CLS_IDENT) {
                    next = (int64_t)g;
                    break;
                }
            }
        }
        if (next > best_next) {
            best_next = next;
            best = l;
        }
        if (!lookahead) break;
    }
    if (best < 0) {  // every candidate is used by the gate: take any other local bit
        for (int l = nl - 1; l >= 0 && best < 0; --l) {
            bool skip = false;
            for (int a = 0; a < navoid; ++a)
                if (avoid[a] == l) skip = true;
            if (!skip) best = l;
        }
    }
    return best;
}

void Planner::plan(const qsim_gate *gates, size_t ngates, std::vector<PlanOp> &ops, bool lookahead) {
    for (size_t g = 0; g < ngates; ++g) {
        const qsim_gate &x = gates[g];
        if (x.kind == QSIM_GATE_SWAP) {  // relabel only: 0 bytes
            swap_bits(pos[x.target], pos[x.target2]);
            continue;
        }
        int32_t cls = classify(x.u);
        if (cls == CLS_IDENT) continue;
        int pt = pos[x.target];
        if (pt >= nl && cls == CLS_ANTI && relabel_global) {
            // a permutation gate on global bits only: relabel the shards (no exchange)
            bool all_global = true;
            for (int c = 0; c < x.ncontrols; ++c) all_global = all_global && pos[x.controls[c]] >= nl;
            if (all_global) {
                PlanOp r{};
                r.type = QSIM_OP_RELABEL;
                r.l = pt;
                r.cls = cls;
                r.nctrl = x.ncontrols;
                r.ctrl[0] = x.ncontrols > 0 ? pos[x.controls[0]] : -1;
                r.ctrl[1] = x.ncontrols > 1 ? pos[x.controls[1]] : -1;
                r.gate_index = (int32_t)g;
                ops.push_back(r);
                continue;
            }
        }
        if (pt >= nl && cls != CLS_DIAG) {
            int avoid[2 + 64];
            int navoid = 0;
            for (int c = 0; c < x.ncontrols; ++c)
                if (pos[x.controls[c]] < nl) avoid[navoid++] = pos[x.controls[c]];
            // NEXT-1 (i): the other global bits that non-diagonal gates will
            // target within the next 2N gates join this exchange as one
            // all-to-all (m bits: 1 - 2^-m of a shard per GPU instead of m/2)
            int gl[64];
            int m = 0;
            gl[m++] = pt;
            if (remap && n - nl >= 2) {
                const size_t end = std::min(ngates, g + 1 + 2 * (size_t)n);
                for (size_t h = g + 1; h < end && m < std::min(n - nl, kRemapMaxBits); ++h) {
                    const qsim_gate &y = gates[h];
                    if (y.kind == QSIM_GATE_SWAP) break;  // relabels: stop looking (rare)
                    const int32_t yc = classify(y.u);
                    if (yc == CLS_DIAG || yc == CLS_IDENT) continue;
                    const int py = pos[y.target];
                    if (py < nl) continue;
                    bool allg = yc == CLS_ANTI && relabel_global;  // would relabel: no data moves
                    for (int c = 0; c < y.ncontrols && allg; ++c) allg = pos[y.controls[c]] >= nl;
                    if (allg) continue;
                    bool dup = false;
                    for (int i = 0; i < m; ++i) dup = dup || gl[i] == py;
                    if (!dup) gl[m++] = py;
                }
            }
            static const int remap_min = getenv("QSIM_REMAP_MIN") ? atoi(getenv("QSIM_REMAP_MIN")) : 2;
            if (remap && m >= remap_min && n - nl >= 1) {
                int lv[64];
                for (int i = 0; i < m; ++i) {
                    lv[i] = choose_victim(gates, ngates, g, avoid, navoid, lookahead, true);
                    avoid[navoid++] = lv[i];
                }
                for (int i = 0; i < m; ++i) {
                    PlanOp e{};
                    e.type = QSIM_OP_REMAP;
                    e.g = gl[i];
                    e.l = lv[i];
                    e.gate_index = (int32_t)g;
                    ops.push_back(e);
                }
                for (int i = 0; i < m; ++i) swap_bits(gl[i], lv[i]);
                pt = pos[x.target];
            } else {
            int l = choose_victim(gates, ngates, g, avoid, navoid, lookahead);
            PlanOp e{};
            e.type = QSIM_OP_EXCHANGE;
            e.g = pt;
            e.l = l;
            e.gate_index = (int32_t)g;
            ops.push_back(e);
            swap_bits(pt, l);
            pt = l;
            }
        }
        PlanOp o{};
        o.type = QSIM_OP_GATE;
        o.l = pt;
        o.cls = cls;
        o.nctrl = x.ncontrols;
        for (int c = 0; c < x.ncontrols; ++c) o.ctrl[c] = pos[x.controls[c]];
        o.ctrl[1] = x.ncontrols > 1 ? o.ctrl[1] : -1;
        if (x.ncontrols == 0) o.ctrl[0] = -1;
        o.gate_index = (int32_t)g;
        ops.push_back(o);
    }
}

}  // namespace qsim

// ---- C-ABI planner entry points (callable without a GPU) -------------------
extern "C" {

int qsim_plan_create(int n_qubits, int nshards, const int *initial_map, const qsim_gate *gates, size_t ngates,
                     qsim_plan **out) {
    if (!out || n_qubits < 2 || n_qubits > 63 || nshards < 1 || (nshards & (nshards - 1))) {
        qsim::set_error("qsim_plan_create: bad n_qubits / nshards / out");
        return QSIM_EINVAL;
    }
    int rc = qsim::validate_gates(n_qubits, gates, ngates, true);
    if (rc) return rc;
    auto *p = new qsim_plan();
    p->pl.init(n_qubits, nshards, initial_map);
    if (p->pl.nl < 1) {
        delete p;
        qsim::set_error("qsim_plan_create: no local qubits");
        return QSIM_EINVAL;
    }
    p->pl.remap = getenv("QSIM_NO_REMAP") == nullptr;  // same switch as qsim_create
    p->pl.plan(gates, ngates, p->ops, true);
    *out = p;
    return QSIM_OK;
}

int64_t qsim_plan_num_ops(const qsim_plan *p) { return p ? (int64_t)p->ops.size() : -1; }

int qsim_plan_get_op(const qsim_plan *p, int64_t i, qsim_plan_op *op) {
    if (!p || !op || i < 0 || i >= (int64_t)p->ops.size()) {
        qsim::set_error("qsim_plan_get_op: bad index");
        return QSIM_EINVAL;
    }
    const qsim::PlanOp &o = p->ops[(size_t)i];
    op->type = o.type;
    op->g = o.g;
    op->l = o.l;
    op->cls = o.cls;
    op->ncontrols = o.nctrl;
    op->controls[0] = o.ctrl[0];
    op->controls[1] = o.ctrl[1];
    op->gate_index = o.gate_index;
    return QSIM_OK;
}

int qsim_plan_final_map(const qsim_plan *p, int *pos) {
    if (!p || !pos) return QSIM_EINVAL;
    for (int q = 0; q < p->pl.n; ++q) pos[q] = p->pl.pos[q];
    return QSIM_OK;
}

void qsim_plan_destroy(qsim_plan *p) { delete p; }

int qsim_aux_num_vars(int n_qubits, const qsim_gate *gates, size_t ngates, int *P) {
    if (!P || (ngates && !gates) || n_qubits < 2 || n_qubits > 63) {
        qsim::set_error("qsim_aux_num_vars: bad arguments");
        return QSIM_EINVAL;
    }
    int rc = qsim::validate_gates(n_qubits, gates, ngates, true);
    if (rc) return rc;
    return qsim::aux_num_vars(n_qubits, gates, ngates, P);
}
}
