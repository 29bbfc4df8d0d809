// asm.cpp -- the JUQCS assembler-like instruction language (App. B,
// lines 1104-1532): a host parser and a runner that
// drives the C-ABI (runs of gates -> qsim_apply_circuit, then the measurement
// and preparation instructions).
//
// Readings:
//  * '!' starts a comment to the end of the line (App. C: "Removing `!' from
//    the second line instructs ..."); mnemonics are case-insensitive.
//  * BIT ASSIGNMENT p_0 .. p_{N-1}: logical qubit j is stored at physical bit
//    p_j (R-B10) -- the initial qubit map; results are unchanged.
//  * DEPOLARIZING CHANNEL: after every gate operation, for every
//    qubit j, one draw u = splitmix64(seed ^ (2^32 g + j)) >> 11 * 2^-53 (g =
//    gate counter) selects X if u < p_x, Y if u < p_x + p_y, Z if u < p_x +
//    p_y + p_z, else nothing (R-B11: the three are exclusive, as the constraint
//    p_x + p_y + p_z <= 1 suggests).  SEED <= 0 uses the run's seed.
//  * M n: outcome from qsim_measure with seed = run seed + (index of the M /
//    EXIT measurement, counted from 0); EXIT measures qubits 0..N-1 in order
//    and stops; GENERATE EVENTS "destroys the state ... force[s] QC to exit"
//    (P:1386-1388): the run stops after it.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "internal.h"

struct qsim_asm {
    int n = 0;
    std::vector<int> perm;         // BIT ASSIGNMENT (empty: identity)
    double depol[4] = {0, 0, 0, 0};  // p_x, p_y, p_z, seed
    std::vector<qsim_asm_op> ops;
};

struct qsim_asm_result {
    int n = 0;
    std::vector<double> tables;      // 3N per BEGIN MEASUREMENT: <Qx>, <Qy>, <Qz> interleaved per qubit
    std::vector<int32_t> outcomes;   // (qubit, outcome) per M
    std::vector<uint64_t> events;    // GENERATE EVENTS (logical indices)
};

namespace {

using qsim::set_error;

std::string upper(std::string s) {
    for (char &c : s) c = (char)std::toupper((unsigned char)c);
    return s;
}

bool to_int(const std::string &t, int64_t &v) {
    if (t.empty()) return false;
    char *e = nullptr;
    v = std::strtoll(t.c_str(), &e, 10);
    return e && *e == 0;
}
bool to_double(const std::string &t, double &v) {
    if (t.empty()) return false;
    char *e = nullptr;
    v = std::strtod(t.c_str(), &e);
    return e && *e == 0 && std::isfinite(v);
}

void set_u(qsim_gate &g, double a0, double a1, double b0, double b1, double c0, double c1, double d0, double d1) {
    const double u[8] = {a0, a1, b0, b1, c0, c1, d0, d1};
    std::memcpy(g.u, u, sizeof(u));
}
void set_phase(qsim_gate &g, double ang) { set_u(g, 1, 0, 0, 0, 0, 0, std::cos(ang), std::sin(ang)); }

uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

}  // namespace

extern "C" {

int qsim_asm_parse(const char *text, qsim_asm **out) {
    if (!text || !out) {
        set_error("qsim_asm_parse: null argument");
        return QSIM_EINVAL;
    }
    auto a = new qsim_asm();
    std::istringstream in(text);
    std::string raw;
    int lineno = 0;
    bool seen_gate = false;
    auto fail = [&](const std::string &m) {
        set_error("line " + std::to_string(lineno) + ": " + m);
        delete a;
        return QSIM_EINVAL;
    };
    while (std::getline(in, raw)) {
        ++lineno;
        const size_t bang = raw.find('!');
        if (bang != std::string::npos) raw.resize(bang);
        for (char &c : raw)
            if (c == ',' || c == '=' || c == '\t' || c == '\r') c = ' ';
        std::istringstream ls(raw);
        std::vector<std::string> tk;
        for (std::string t; ls >> t;) tk.push_back(t);
        if (tk.empty()) continue;
        const std::string op = upper(tk[0]);
        const size_t na = tk.size() - 1;
        auto qubit = [&](size_t i, int &q) -> bool {
            int64_t v;
            if (i >= tk.size() || !to_int(tk[i], v) || v < 0 || v >= a->n) return false;
            q = (int)v;
            return true;
        };
        if (op == "QUBITS") {
            int64_t v;
            if (a->n) return fail("QUBITS may appear only once, as the first instruction");
            if (na != 1 || !to_int(tk[1], v) || v < 2 || v > 63) return fail("QUBITS N needs 1 < N < 64");
            a->n = (int)v;
            continue;
        }
        if (!a->n) return fail("QUBITS N must be the first instruction (PAPER.md:1421)");
        qsim_asm_op o{};
        o.line = lineno;
        qsim_gate &g = o.gate;
        g.kind = QSIM_GATE_U;
        g.target2 = -1;
        g.controls[0] = g.controls[1] = -1;
        const double r2 = 1.0 / std::sqrt(2.0);
        if (op == "BIT" && na >= 1 && upper(tk[1]) == "ASSIGNMENT") {
            if (seen_gate) return fail("BIT ASSIGNMENT must come before the first gate");
            if ((int)na - 1 != a->n) return fail("BIT ASSIGNMENT needs N integers");
            std::vector<int> p(a->n), seen(a->n, 0);
            for (int j = 0; j < a->n; ++j) {
                int q;
                if (!qubit(2 + j, q) || seen[q]) return fail("BIT ASSIGNMENT must be a permutation of 0..N-1");
                seen[q] = 1;
                p[j] = q;
            }
            a->perm = p;
            continue;
        }
        if (op == "DEPOLARIZING" && na >= 1 && upper(tk[1]) == "CHANNEL") {
            if (seen_gate) return fail("DEPOLARIZING CHANNEL must come before the first gate");
            for (size_t i = 2; i + 1 < tk.size(); i += 2) {
                const std::string key = upper(tk[i]);
                double v;
                if (!to_double(tk[i + 1], v)) return fail("bad value for " + key);
                if (key == "P_X") a->depol[0] = v;
                else if (key == "P_Y") a->depol[1] = v;
                else if (key == "P_Z") a->depol[2] = v;
                else if (key == "SEED") a->depol[3] = v;
                else return fail("unknown DEPOLARIZING CHANNEL argument " + key);
            }
            if ((tk.size() - 2) % 2) return fail("DEPOLARIZING CHANNEL arguments are KEY = value pairs");
            const double px = a->depol[0], py = a->depol[1], pz = a->depol[2];
            if (px < 0 || py < 0 || pz < 0 || px > 1 || py > 1 || pz > 1 || px + py + pz > 1)
                return fail("need 0 <= p_x, p_y, p_z <= 1 and p_x + p_y + p_z <= 1 (PAPER.md:1503)");
            continue;
        }
        if (op == "BEGIN" && na == 1 && upper(tk[1]) == "MEASUREMENT") {
            o.type = QSIM_ASM_MEASURE_ALL;
            a->ops.push_back(o);
            continue;
        }
        if (op == "GENERATE" && na == 3 && upper(tk[1]) == "EVENTS") {
            if (!to_int(tk[2], o.args[0]) || o.args[0] < 1 || !to_int(tk[3], o.args[1]))
                return fail("GENERATE EVENTS events seed: events > 0, seed an integer");
            o.type = QSIM_ASM_EVENTS;
            a->ops.push_back(o);
            continue;
        }
        if (op == "EXIT") {
            if (na) return fail("EXIT takes no arguments");
            o.type = QSIM_ASM_EXIT;
            a->ops.push_back(o);
            continue;
        }
        if (op == "M" || op == "CLEAR" || op == "SET") {
            int q;
            if (na != 1 || !qubit(1, q)) return fail(op + " n: n in 0..N-1");
            o.type = op == "M" ? QSIM_ASM_M : op == "CLEAR" ? QSIM_ASM_CLEAR : QSIM_ASM_SET;
            o.args[0] = q;
            a->ops.push_back(o);
            continue;
        }
        if (op == "SHORBOX") {
            if (na != 3 || !to_int(tk[1], o.args[0]) || !to_int(tk[2], o.args[1]) || !to_int(tk[3], o.args[2]) ||
                o.args[0] < 1 || o.args[0] >= a->n || o.args[1] < 2 || o.args[2] < 1 || o.args[2] >= o.args[1])
                return fail("SHORBOX nx G y: 0 < nx < N, G >= 2, 1 <= y < G");
            o.type = QSIM_ASM_SHORBOX;
            a->ops.push_back(o);
            continue;
        }
        // ---- gates ----
        o.type = QSIM_ASM_GATE;
        int q = 0;
        if (op == "CNOT" || op == "U") {
            int c, t;
            if (!qubit(1, c) || !qubit(2, t) || c == t) return fail(op + ": control != target in 0..N-1");
            if (op == "CNOT") {
                if (na != 2) return fail("CNOT control target");
                set_u(g, 0, 0, 1, 0, 1, 0, 0, 0);
            } else {
                int64_t k;
                if (na != 3 || !to_int(tk[3], k)) return fail("U control target k: k an integer");
                set_phase(g, (k >= 0 ? 2.0 : -2.0) * M_PI / std::ldexp(1.0, (int)std::llabs(k)));
            }
            g.target = t;
            g.ncontrols = 1;
            g.controls[0] = c;
        } else if (op == "TOFFOLI") {
            int c1, c2, t;
            if (na != 3 || !qubit(1, c1) || !qubit(2, c2) || !qubit(3, t) || c1 == c2 || c1 == t || c2 == t)
                return fail("TOFFOLI control1 control2 target: distinct, in 0..N-1");
            set_u(g, 0, 0, 1, 0, 1, 0, 0, 0);
            g.target = t;
            g.ncontrols = 2;
            g.controls[0] = c1;
            g.controls[1] = c2;
        } else {
            static const char *one[] = {"I", "H", "X", "Y", "Z", "S", "S+", "T", "T+", "+X", "-X", "+Y", "-Y"};
            bool simple = false;
            for (const char *m : one) simple = simple || op == m;
            if (simple) {
                if (na != 1 || !qubit(1, q)) return fail(op + " n: n in 0..N-1");
            } else if (op == "U1" || op == "U2" || op == "U3" || op == "R") {
                const size_t want = op == "U1" ? 2 : op == "U2" ? 3 : op == "U3" ? 4 : 2;
                if (na != want || !qubit(1, q)) return fail(op + ": bad arguments");
            } else {
                return fail("unknown instruction " + tk[0]);
            }
            g.target = q;
            double th = 0, ph = 0, la = 0;
            if (op == "I") {
                seen_gate = true;  // a no-operation
                continue;
            } else if (op == "H") set_u(g, r2, 0, r2, 0, r2, 0, -r2, 0);
            else if (op == "X") set_u(g, 0, 0, 1, 0, 1, 0, 0, 0);
            else if (op == "Y") set_u(g, 0, 0, 0, -1, 0, 1, 0, 0);
            else if (op == "Z") set_u(g, 1, 0, 0, 0, 0, 0, -1, 0);
            else if (op == "S") set_u(g, 1, 0, 0, 0, 0, 0, 0, 1);
            else if (op == "S+") set_u(g, 1, 0, 0, 0, 0, 0, 0, -1);
            else if (op == "T") set_u(g, 1, 0, 0, 0, 0, 0, r2, r2);
            else if (op == "T+") set_u(g, 1, 0, 0, 0, 0, 0, r2, -r2);
            else if (op == "+X") set_u(g, r2, 0, 0, r2, 0, r2, r2, 0);
            else if (op == "-X") set_u(g, r2, 0, 0, -r2, 0, -r2, r2, 0);
            else if (op == "+Y") set_u(g, r2, 0, r2, 0, -r2, 0, r2, 0);
            else if (op == "-Y") set_u(g, r2, 0, -r2, 0, r2, 0, r2, 0);
            else if (op == "R") {
                int64_t k;
                if (!to_int(tk[2], k)) return fail("R n k: k an integer");
                set_phase(g, (k >= 0 ? 2.0 : -2.0) * M_PI / std::ldexp(1.0, (int)std::llabs(k)));
            } else {
                const size_t nang = op == "U1" ? 1 : op == "U2" ? 2 : 3;
                double v[3] = {0, 0, 0};
                for (size_t i = 0; i < nang; ++i)
                    if (!to_double(tk[2 + i], v[i])) return fail(op + ": angles are numbers (radians)");
                if (op == "U1") {
                    set_phase(g, v[0]);
                } else {
                    if (op == "U2") {
                        th = M_PI / 2;
                        ph = v[0];
                        la = v[1];
                    } else {
                        th = v[0];
                        ph = v[1];
                        la = v[2];
                    }
                    const double c = std::cos(th / 2), s = std::sin(th / 2);
                    // U3 = [[c, -e^{i la} s], [e^{i ph} s, e^{i (ph + la)} c]]  (
                    // U2 = U3(pi/2, ph, la))
                    set_u(g, c, 0, -std::cos(la) * s, -std::sin(la) * s, std::cos(ph) * s, std::sin(ph) * s,
                          std::cos(ph + la) * c, std::sin(ph + la) * c);
                }
            }
        }
        seen_gate = true;
        a->ops.push_back(o);
    }
    if (!a->n) {
        lineno = 0;
        return fail("empty program: QUBITS N missing");
    }
    *out = a;
    return QSIM_OK;
}

int qsim_asm_info(const qsim_asm *a, int *n_qubits, int64_t *nops, int *perm, double *depol) {
    if (!a) return QSIM_EINVAL;
    if (n_qubits) *n_qubits = a->n;
    if (nops) *nops = (int64_t)a->ops.size();
    if (perm)
        for (int j = 0; j < a->n; ++j) perm[j] = a->perm.empty() ? j : a->perm[j];
    if (depol) std::memcpy(depol, a->depol, sizeof(a->depol));
    return QSIM_OK;
}

int qsim_asm_get_op(const qsim_asm *a, int64_t i, qsim_asm_op *op) {
    if (!a || !op || i < 0 || i >= (int64_t)a->ops.size()) {
        set_error("qsim_asm_get_op: bad index");
        return QSIM_EINVAL;
    }
    *op = a->ops[(size_t)i];
    return QSIM_OK;
}

void qsim_asm_destroy(qsim_asm *a) { delete a; }

int qsim_asm_run(const qsim_asm *a, int encoding, int ngpus, uint64_t seed, qsim_asm_result **out) {
    if (!a || !out) {
        set_error("qsim_asm_run: null argument");
        return QSIM_EINVAL;
    }
    qsim_state *s = nullptr;
    qsim_config cfg{};  // ngpus shards on the current device (QSIM_TRANSPORT_LOCAL)
    cfg.n_qubits = a->n;
    cfg.encoding = encoding;
    cfg.nshards = ngpus;
    cfg.transport = QSIM_TRANSPORT_LOCAL;
    cfg.device = -1;
    cfg.fuse = 1;
    int rc = qsim_create_ex(&cfg, &s);
    if (rc) return rc;
    auto r = new qsim_asm_result();
    r->n = a->n;
    auto done = [&](int code) {
        if (code) {
            std::string keep = qsim_last_error();
            qsim_destroy(s);
            delete r;
            set_error(keep);
            return code;
        }
        qsim_destroy(s);
        *out = r;
        return QSIM_OK;
    };
    if (!a->perm.empty() && (rc = qsim_set_qubit_map(s, a->perm.data()))) return done(rc);
    const double px = a->depol[0], py = a->depol[1], pz = a->depol[2];
    const bool depol = px > 0 || py > 0 || pz > 0;
    const uint64_t dseed = a->depol[3] > 0 ? (uint64_t)a->depol[3] : seed;
    uint64_t gate_count = 0, meas_count = 0;
    std::vector<qsim_gate> batch;
    auto flush = [&]() -> int {
        if (batch.empty()) return QSIM_OK;
        int c = qsim_apply_circuit(s, batch.data(), batch.size());
        batch.clear();
        return c;
    };
    auto measure = [&](int qb) -> int {
        int outcome = 0;
        int c = qsim_measure(s, qb, seed + meas_count++, &outcome);
        if (c) return c;
        r->outcomes.push_back(qb);
        r->outcomes.push_back(outcome);
        return QSIM_OK;
    };
    for (const qsim_asm_op &o : a->ops) {
        if (o.type == QSIM_ASM_GATE) {
            batch.push_back(o.gate);
            if (depol) {  // reading R-B11: after every gate, one exclusive X / Y / Z draw per qubit
                for (int j = 0; j < a->n; ++j) {
                    const double u = (double)(splitmix64(dseed ^ ((gate_count << 32) + (uint64_t)j)) >> 11) *
                                     (1.0 / 9007199254740992.0);
                    qsim_gate e{};
                    e.kind = QSIM_GATE_U;
                    e.target = j;
                    e.target2 = -1;
                    e.controls[0] = e.controls[1] = -1;
                    if (u < px) set_u(e, 0, 0, 1, 0, 1, 0, 0, 0);
                    else if (u < px + py) set_u(e, 0, 0, 0, -1, 0, 1, 0, 0);
                    else if (u < px + py + pz) set_u(e, 1, 0, 0, 0, 0, 0, -1, 0);
                    else continue;
                    batch.push_back(e);
                }
            }
            ++gate_count;
            continue;
        }
        if ((rc = flush())) return done(rc);
        switch (o.type) {
            case QSIM_ASM_MEASURE_ALL: {
                const size_t at = r->tables.size();
                r->tables.resize(at + 3 * (size_t)a->n);
                if ((rc = qsim_expectations(s, r->tables.data() + at))) return done(rc);
                break;
            }
            case QSIM_ASM_EVENTS: {
                const size_t at = r->events.size();
                r->events.resize(at + (size_t)o.args[0]);
                const uint64_t es = o.args[1] > 0 ? (uint64_t)o.args[1] : seed;
                if ((rc = qsim_sample(s, (size_t)o.args[0], es, r->events.data() + at))) return done(rc);
                return done(QSIM_OK);  // "This operation destroys the state ... force QC to exit"
            }
            case QSIM_ASM_M:
                if ((rc = measure((int)o.args[0]))) return done(rc);
                break;
            case QSIM_ASM_CLEAR:
            case QSIM_ASM_SET:
                if ((rc = qsim_project(s, (int)o.args[0], o.type == QSIM_ASM_SET ? 1 : 0))) return done(rc);
                break;
            case QSIM_ASM_SHORBOX:
                if ((rc = qsim_prepare_shorbox(s, (int)o.args[0], (uint64_t)o.args[1], (uint64_t)o.args[2])))
                    return done(rc);
                break;
            case QSIM_ASM_EXIT:
                for (int j = 0; j < a->n; ++j)
                    if ((rc = measure(j))) return done(rc);
                return done(QSIM_OK);
            default:
                break;
        }
    }
    if ((rc = flush())) return done(rc);
    if ((rc = qsim_sync(s))) return done(rc);
    return done(QSIM_OK);
}

int qsim_asm_result_get(const qsim_asm_result *r, int what, void *buf, int64_t cap, int64_t *count) {
    if (!r || !count) return QSIM_EINVAL;
    const void *src = nullptr;
    size_t n = 0, sz = 0;
    if (what == QSIM_ASM_R_TABLES) {
        src = r->tables.data();
        n = r->tables.size();
        sz = 8;
    } else if (what == QSIM_ASM_R_OUTCOMES) {
        src = r->outcomes.data();
        n = r->outcomes.size();
        sz = 4;
    } else if (what == QSIM_ASM_R_EVENTS) {
        src = r->events.data();
        n = r->events.size();
        sz = 8;
    } else {
        set_error("qsim_asm_result_get: unknown item");
        return QSIM_EINVAL;
    }
    *count = (int64_t)n;
    if (buf && cap > 0) std::memcpy(buf, src, sz * (size_t)std::min<int64_t>(cap, (int64_t)n));
    return QSIM_OK;
}

void qsim_asm_result_destroy(qsim_asm_result *r) { delete r; }

}  // extern "C"
