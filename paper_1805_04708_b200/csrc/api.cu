// api.cu -- the qsim C-ABI: state lifetime, the executor that follows the
// planner's ops (fused tile passes, sweeps, swap exchanges), reductions and
// read-out.  See include/qsim.h for the contract of every entry point.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <condition_variable>
#include <deque>
#include <functional>
#include <thread>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"
#include "kernels.h"
#include "kernels_a.h"
#include "lpass.h"

namespace qsim {

static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }

#define CU(call)                                                                            \
    do {                                                                                    \
        cudaError_t _e = (call);                                                            \
        if (_e != cudaSuccess) {                                                            \
            set_error(std::string(#call) + ": " + cudaGetErrorString(_e));                  \
            return QSIM_ECUDA;                                                              \
        }                                                                                   \
    } while (0)
#define NC(call)                                                                            \
    do {                                                                                    \
        ncclResult_t _r = (call);                                                           \
        if (_r != ncclSuccess) {                                                            \
            set_error(std::string(#call) + ": " + ncclGetErrorString(_r));                  \
            return QSIM_ECOMM;                                                              \
        }                                                                                   \
    } while (0)
#define RC(call)                       \
    do {                               \
        int _rc = (call);              \
        if (_rc != QSIM_OK) return _rc; \
    } while (0)

static inline uint64_t ins0(uint64_t w, int p) { return ((w >> p) << (p + 1)) | (w & ((1ull << p) - 1ull)); }

struct Shard {
    int index = 0;            // global shard index (rank bits)
    void *amps = nullptr;     // 2^nl amplitudes
    void *amps2 = nullptr;    // A, lazy bounds: the out-of-place target of a dense gate (swapped after it)
};

}  // namespace qsim

using namespace qsim;

namespace qsim {
struct QGroup;
}
struct qsim_state {
    int n = 0, enc = 0, P = 1, nl = 0, transport = 0, rank = 0, dev = 0, fuse = 1;
    qsim::QGroup *group = nullptr;  // QSIM_TRANSPORT_DEVICES: this handle drives P member handles
    int a_policy = 0;               // QSIM_A_POLICY_*
    int32_t *d_oor = nullptr;       // lazy policy: "an output left the kept range" flag
    std::vector<PersistGate> h_pg;  // qsim_apply_circuit_persistent: gate records (physical bits)
    void *h_pc = nullptr;           // pinned staging of its phase / op records
    struct PcEntry {                // planned circuits (device records), keyed by the physical gate list
        uint64_t key = 0, stamp = 0;
        int lcs = 0, K = 0;
        void *d = nullptr;
        std::vector<std::pair<int, int>> lens;  // (phases, ops) per launch
        std::vector<PersistGate> recs;          // the records it was planned from (a hit compares them)
    };
    std::vector<PcEntry> pc_cache;
    uint64_t pc_clock = 0;
    size_t pg_cap = 0;
    int pass_r = 4;  // register qubits per pass stage (QSIM_PASS_R=5 selects 32-amplitude groups)
    int pass_k = LP_MAX_K;  // tile qubits of the relabelling pass (QSIM_LPASS_K = 9..12)
    bool pass_k_env = false;  // QSIM_LPASS_K given: no small-shard reduction
    size_t amp_bytes = 16;
    uint64_t alloc_amps = 0;  // max(2^nl, 256): small shards are padded with zero amplitudes
    Planner pl;
    std::vector<Shard> shards;
    uint64_t chunk_amps = 0;
    void *stage[2] = {nullptr, nullptr};
    cudaStream_t stream = nullptr, comm_stream = nullptr;
    cudaEvent_t ev_recv[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_start = nullptr;
    ncclComm_t comm = nullptr;
    double *d_partials = nullptr, *d_out = nullptr, *h_out = nullptr;  // reduction scratch
    qsim_stats st{};
    // A variant
    double r0 = 0.5, r1 = 0.5;
    bool r_stale = false;  // dense gates update (r0, r1) in the device tables only (read back on demand)
    double *d_acc = nullptr;  // (min, -max) of |z|^2 of a dense A gate
    ATables *atab = nullptr;
    // profiling (qsim_profile): event pairs around each launch
    struct ProfRec {
        int kind;
        double bytes, flops;
        cudaEvent_t a, b;
    };
    bool prof = false;
    bool capturing = false;      // qsim_graph_begin .. qsim_graph_end
    bool prof_saved = false;
    std::vector<int> cap_pos;    // qubit map at qsim_graph_begin
    std::vector<uint32_t> cap_gphys;
    std::vector<ProfRec> prof_recs;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<uint32_t> gphys, ginv;  // storage index -> physical global bits (phi) and inverse
    cudaEvent_t prof_a = nullptr;  // pending start event
};

namespace qsim {

// ============================================================================
// helpers
// ============================================================================
static cudaEvent_t pool_get(qsim_state *s) {
    if (!s->ev_pool.empty()) {
        cudaEvent_t e = s->ev_pool.back();
        s->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
// Bracket one launch: prof_begin before, prof_end(kind, bytes) after.
static void prof_begin(qsim_state *s) {
    if (!s->prof) return;
    s->prof_a = pool_get(s);
    cudaEventRecord(s->prof_a, s->stream);
}
static void prof_end(qsim_state *s, int kind, double bytes, double flops = 0.0) {
    if (!s->prof || !s->prof_a) return;
    cudaEvent_t b = pool_get(s);
    cudaEventRecord(b, s->stream);
    s->prof_recs.push_back({kind, bytes, flops, s->prof_a, b});
    s->prof_a = nullptr;
}
// Physical global bits held by a shard's storage: phi(index).  Permutation
// gates on global qubits (planner op QSIM_OP_RELABEL) permute phi instead of
// moving data.
static uint32_t shard_phys(const qsim_state *s, const Shard &sh) { return s->gphys[sh.index]; }
static uint64_t shard_base(const qsim_state *s, const Shard &sh) { return (uint64_t)shard_phys(s, sh) << s->nl; }

static int rank_bit(const qsim_state *s, const Shard &sh, int phys_bit) {
    return (shard_phys(s, sh) >> (phys_bit - s->nl)) & 1;
}
static void reset_labels(qsim_state *s) {
    s->gphys.resize(s->P);
    s->ginv.resize(s->P);
    for (int r = 0; r < s->P; ++r) s->gphys[r] = s->ginv[r] = (uint32_t)r;
}

// Whether all controls that sit on global bits are 1 for this shard.
static bool global_ctrls_ok(const qsim_state *s, const Shard &sh, const PlanOp &o) {
    for (int c = 0; c < o.nctrl; ++c)
        if (o.ctrl[c] >= s->nl && !rank_bit(s, sh, o.ctrl[c])) return false;
    return true;
}

static uint64_t full_cmask(const PlanOp &o) {
    uint64_t m = 0;
    for (int c = 0; c < o.nctrl; ++c) m |= 1ull << o.ctrl[c];
    return m;
}

// Algorithmic bytes of one gate on one shard had it run alone.
static double gate_bytes_alone(const qsim_state *s, const Shard &sh, const PlanOp &o, const double *u) {
    if (!global_ctrls_ok(s, sh, o)) return 0.0;
    int nlc = 0;
    for (int c = 0; c < o.nctrl; ++c)
        if (o.ctrl[c] < s->nl) ++nlc;
    double amps = std::ldexp(1.0, s->nl - nlc);
    double per = 2.0 * (double)s->amp_bytes;  // read + write
    if (o.cls == CLS_DIAG) {
        if (o.l >= s->nl) {
            int bit = rank_bit(s, sh, o.l);
            double fr = bit ? u[6] : u[0], fi = bit ? u[7] : u[1];
            return (fr == 1.0 && fi == 0.0) ? 0.0 : amps * per;
        }
        bool one0 = u[0] == 1.0 && u[1] == 0.0, one1 = u[6] == 1.0 && u[7] == 0.0;
        if (one0 || one1) return amps * 0.5 * per;
    }
    return amps * per;
}

// Algorithmic fp64 flops of one gate on one shard: a dense 2x2
// is 14 flops per amplitude it updates (4 complex multiplies + 2 complex adds
// per pair), a phase 6 per amplitude whose factor is not 1, a permutation 0.
static double gate_flops(const qsim_state *s, const Shard &sh, const PlanOp &o, const double *u) {
    if (!global_ctrls_ok(s, sh, o)) return 0.0;
    int nlc = 0;
    for (int c = 0; c < o.nctrl; ++c)
        if (o.ctrl[c] < s->nl) ++nlc;
    double amps = std::ldexp(1.0, s->nl - nlc);
    if (o.cls == CLS_DENSE) return 14.0 * amps;
    if (o.cls == CLS_ANTI) {
        bool perm = u[2] == 1.0 && u[3] == 0.0 && u[4] == 1.0 && u[5] == 0.0;
        return perm ? 0.0 : 6.0 * amps;
    }
    if (o.cls == CLS_DIAG) {
        bool one0 = u[0] == 1.0 && u[1] == 0.0, one1 = u[6] == 1.0 && u[7] == 0.0;
        if (o.l >= s->nl) {
            int bit = rank_bit(s, sh, o.l);
            return (bit ? one1 : one0) ? 0.0 : 6.0 * amps;
        }
        return 6.0 * amps * ((one0 ? 0.0 : 0.5) + (one1 ? 0.0 : 0.5));
    }
    return 0.0;
}

// ============================================================================
// E single-gate sweep on every shard
// ============================================================================
static int sweep_gate_e(qsim_state *s, const PlanOp &o, const double *u) {
    for (auto &sh : s->shards) {
        if (!global_ctrls_ok(s, sh, o)) continue;
        int locs[3], nloc = 0;
        uint64_t cm = 0;
        for (int c = 0; c < o.nctrl; ++c)
            if (o.ctrl[c] < s->nl) {
                locs[nloc++] = o.ctrl[c];
                cm |= 1ull << o.ctrl[c];
            }
        if (o.l >= s->nl) {  // diagonal gate on a global bit: uniform factor on the shard
            int bit = rank_bit(s, sh, o.l);
            ScaleParams p{};
            p.a = sh.amps;
            p.f[0] = bit ? u[6] : u[0];
            p.f[1] = bit ? u[7] : u[1];
            if (p.f[0] == 1.0 && p.f[1] == 0.0) continue;
            std::sort(locs, locs + nloc);
            for (int k = 0; k < nloc; ++k) p.ins[k] = locs[k];
            p.nins = nloc;
            p.cmask = cm;
            p.nitems = 1ull << (s->nl - nloc);
            prof_begin(s);
            launch_scale_e(p, s->stream);
            prof_end(s, QSIM_K_SWEEP, gate_bytes_alone(s, sh, o, u), gate_flops(s, sh, o, u));
        } else {
            SweepParams p{};
            p.a = sh.amps;
            locs[nloc++] = o.l;
            std::sort(locs, locs + nloc);
            for (int k = 0; k < nloc; ++k) p.ins[k] = locs[k];
            p.nins = nloc;
            p.cmask = cm;
            p.t = o.l;
            p.cls = o.cls;
            p.nitems = 1ull << (s->nl - nloc);
            std::memcpy(p.u, u, sizeof(p.u));
            bool one0 = u[0] == 1.0 && u[1] == 0.0, one1 = u[6] == 1.0 && u[7] == 0.0;
            p.touch = (o.cls == CLS_DIAG) ? (one0 ? 2 : (one1 ? 1 : 3)) : 3;
            prof_begin(s);
            launch_sweep_e(p, s->stream);
            prof_end(s, QSIM_K_SWEEP, gate_bytes_alone(s, sh, o, u), gate_flops(s, sh, o, u));
        }
        s->st.kernels++;
        s->st.sweeps++;
        s->st.hbm_bytes += gate_bytes_alone(s, sh, o, u);
    }
    CU(cudaGetLastError());
    return QSIM_OK;
}


// ---- relabelling tile pass (lpass.h) ----
static PlanOp plan_op_of(const LGate &g) {
    PlanOp o{};
    o.type = QSIM_OP_GATE;
    o.g = -1;
    o.l = g.t;
    o.cls = classify(g.u);
    o.nctrl = g.nctl;
    o.ctrl[0] = g.nctl > 0 ? g.ctl[0] : 0;
    o.ctrl[1] = g.nctl > 1 ? g.ctl[1] : 0;
    o.gate_index = -1;
    return o;
}

// lpass_run's callbacks: launch k_lpass_e on every shard / a single-gate sweep.
// Synthetic (deferred) diagonals are excluded from the algorithmic flops.
struct LaunchSink : LPassSink {
    qsim_state *s;
    const std::vector<PlanOp> *run;
    const std::vector<const double *> *us;
    int pass(const LPassParams &p, const LCompileStats &cs, const std::vector<int> &ids) override {
        int nreal = 0;
        for (int id : ids) nreal += id >= 0;
        if (getenv("QSIM_DEBUG_PASSES"))
            fprintf(stderr, "lpass: %zu gates (%d circuit), %d stages, %d ops (%d tables, %d shears, %d dense, %d flips, "
                            "%d relabels, %d swaps), %d tile-level permutations, %d events, %d coefficients, "
                            "%d carried, %d deferred\n",
                    ids.size(), nreal, cs.stages, cs.ops, cs.diagt, cs.shears, cs.dense, cs.flips, cs.relabels,
                    cs.cswaps, cs.tile_free, cs.events, p.ncoef, cs.carried, cs.deferred);
        static thread_local LPassParams q;  // large: keep off the stack; one per thread (handles on other threads)
        std::memcpy(&q, &p, sizeof(q));
        q.noio = getenv("QSIM_DEBUG_PASS_NOIO") ? 1 : 0;
        s->st.stages += p.nstages;
        for (auto &sh : s->shards) {
            q.a = sh.amps;
            q.shard_base = shard_base(s, sh);
            double fl = 0.0;
            for (int id : ids)
                if (id >= 0) fl += gate_flops(s, sh, (*run)[id], (*us)[id]);
            prof_begin(s);
            s->st.jit_passes += launch_lpass_e(q, s->stream);
            prof_end(s, QSIM_K_PASS, std::ldexp(2.0 * (double)s->amp_bytes, s->nl), fl);
            s->st.kernels++;
            s->st.passes++;
            s->st.fused_gates += nreal;
            s->st.hbm_bytes += std::ldexp(2.0 * (double)s->amp_bytes, s->nl);
        }
        CU(cudaGetLastError());
        return QSIM_OK;
    }
    int sweep(const LGate &g, int id) override {
        if (id >= 0) return sweep_gate_e(s, (*run)[id], (*us)[id]);
        return sweep_gate_e(s, plan_op_of(g), g.u);
    }
    double gate_bytes(const LGate &g) override { return gate_bytes_alone(s, s->shards[0], plan_op_of(g), g.u); }
};

// Program cache of the host pass compiler: lpass_run is deterministic in
// its gate list, its configuration and the state's shape (gate_bytes), so
// a repeated run (the same circuit applied again, e.g. config 1's repeated
// calls) replays the recorded pass programs and sweeps instead of compiling
// them again (~0.2-0.3 ms of host time for 200 gates).  QSIM_PLAN_CACHE=0
// disables it.
struct LRecord {
    bool is_pass;
    std::unique_ptr<LPassParams> p;
    LCompileStats cs;
    std::vector<int> ids;
    LGate g;
    int id;
};
struct LRecorder : LPassSink {
    LPassSink *inner;
    std::vector<LRecord> recs;
    int pass(const LPassParams &p, const LCompileStats &cs, const std::vector<int> &ids) override {
        LRecord r{};
        r.is_pass = true;
        r.p.reset(new LPassParams(p));
        r.cs = cs;
        r.ids = ids;
        recs.push_back(std::move(r));
        return inner->pass(p, cs, ids);
    }
    int sweep(const LGate &g, int id) override {
        LRecord r{};
        r.is_pass = false;
        r.g = g;
        r.id = id;
        recs.push_back(std::move(r));
        return inner->sweep(g, id);
    }
    double gate_bytes(const LGate &g) override { return inner->gate_bytes(g); }
};
struct LProgramCache {
    std::mutex mu;
    std::unordered_map<std::string, std::shared_ptr<std::vector<LRecord>>> map;
    std::deque<std::string> order;  // FIFO eviction
    size_t bytes = 0;
    static constexpr size_t kMax = 64, kMaxBytes = size_t(256) << 20;
    static size_t entry_bytes(const std::vector<LRecord> &r) {
        size_t b = 0;
        for (const LRecord &x : r) b += x.is_pass ? sizeof(LPassParams) : sizeof(LGate);
        return b;
    }
};
static LProgramCache &lprogram_cache() {
    static LProgramCache *c = new LProgramCache();  // never destroyed: no exit-order issues
    return *c;
}

static int run_gates_lpass(qsim_state *s, const std::vector<PlanOp> &run, const std::vector<const double *> &us) {
    std::vector<LGate> lg(run.size());
    for (size_t k = 0; k < run.size(); ++k) {
        const PlanOp &o = run[k];
        LGate &g = lg[k];
        g.t = o.l;
        g.nctl = o.nctrl;
        g.ctl[0] = o.nctrl > 0 ? o.ctrl[0] : 0;
        g.ctl[1] = o.nctrl > 1 ? o.ctrl[1] : 0;
        std::memcpy(g.u, us[k], sizeof(g.u));
    }
    LRunConfig cfg;
    cfg.nl = s->nl;
    // small shards: tiles of at most nl - 3 qubits (>= 8 tiles, i.e. CTAs) where that
    // keeps K >= LP_MIN_K -- a latency-bound pass of 4 tiles ran on 4 SMs (config 1,
    // N = 14: 39 -> 28.5 us per circuit with a graph at K = 11); QSIM_LPASS_K overrides
    cfg.K = std::min(s->pass_k, s->nl);
    if (!s->pass_k_env) cfg.K = std::min(cfg.K, std::max(std::min(s->nl, LP_MIN_K), s->nl - 3));
    cfg.R = s->pass_r;
    cfg.max_coef = lpass_max_coef(cfg.R);
    cfg.defer = getenv("QSIM_LPASS_NODEFER") == nullptr;
    cfg.pass_bytes = std::ldexp(2.0 * (double)s->amp_bytes, s->nl);
    LaunchSink sink;
    sink.s = s;
    sink.run = &run;
    sink.us = &us;
    static const bool use_cache = !(getenv("QSIM_PLAN_CACHE") && atoi(getenv("QSIM_PLAN_CACHE")) == 0);
    std::string key;
    if (use_cache) {
        // everything lpass_run and gate_bytes read: configuration, state shape, gate records
        const int shape[8] = {cfg.nl, cfg.K, cfg.R, cfg.max_coef, cfg.defer ? 1 : 0, s->n,
                              (int)s->shards.size(), (int)s->amp_bytes};
        // gate_bytes reads shard 0's global bits (global controls / diagonal targets)
        const uint64_t sb0 = shard_base(s, s->shards[0]);
        key.assign(reinterpret_cast<const char *>(shape), sizeof(shape));
        key.append(reinterpret_cast<const char *>(&sb0), sizeof(sb0));
        key.append(reinterpret_cast<const char *>(lg.data()), lg.size() * sizeof(LGate));
        std::shared_ptr<std::vector<LRecord>> hit;
        {
            LProgramCache &c = lprogram_cache();
            std::lock_guard<std::mutex> lk(c.mu);
            auto it = c.map.find(key);
            if (it != c.map.end()) hit = it->second;
        }
        if (hit) {
            for (const LRecord &r : *hit) RC(r.is_pass ? sink.pass(*r.p, r.cs, r.ids) : sink.sweep(r.g, r.id));
            return QSIM_OK;
        }
    }
    LRecorder rec;
    rec.inner = &sink;
    std::string err;
    const int rc = lpass_run(lg.data(), (int)lg.size(), cfg, use_cache ? (LPassSink &)rec : (LPassSink &)sink, &err);
    if (rc == -1) {
        set_error("lpass: " + err);
        return QSIM_EINVAL;
    }
    if (rc == 0 && use_cache) {
        LProgramCache &c = lprogram_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        const size_t eb = LProgramCache::entry_bytes(rec.recs);
        if (!c.map.count(key) && eb <= LProgramCache::kMaxBytes) {
            while (!c.order.empty() && (c.order.size() >= LProgramCache::kMax || c.bytes + eb > LProgramCache::kMaxBytes)) {
                auto it = c.map.find(c.order.front());
                c.bytes -= LProgramCache::entry_bytes(*it->second);
                c.map.erase(it);
                c.order.pop_front();
            }
            c.map.emplace(key, std::make_shared<std::vector<LRecord>>(std::move(rec.recs)));
            c.order.push_back(key);
            c.bytes += eb;
        }
    }
    return rc;
}

// Local gates of an E state (a3-a6): the relabelling tile pass when the shard
// holds a tile (lpass.h), single-gate sweeps otherwise (or with fusion off).
static int run_gates_e(qsim_state *s, const std::vector<PlanOp> &run, const std::vector<const double *> &us) {
    if (s->fuse && std::min(LP_MAX_K, s->nl) >= LP_MIN_K) return run_gates_lpass(s, run, us);
    for (size_t i = 0; i < run.size(); ++i) RC(sweep_gate_e(s, run[i], us[i]));
    return QSIM_OK;
}

// ============================================================================
// exchange (a7): swap physical global bit g with local bit l; optionally apply
// the triggering gate (now on bit l) to each (kept, received) pair on arrival.
// ============================================================================
static int exchange_impl(qsim_state *s, const PlanOp &x, const PlanOp *gop, const double *u) {
    const int j = x.g - s->nl;
    const int l = x.l;
    const uint64_t half = 1ull << (s->nl - 1);
    uint64_t C = std::min<uint64_t>(s->chunk_amps, half);
    C = std::min<uint64_t>(C, 1ull << l);
    const uint64_t nchunks = half / C;
    const size_t ab = s->amp_bytes;
    // bounds of every chunk the kernels and copies touch (checked, not assumed:
    // no compute-sanitizer on the GPU pool): the exchanged global bit and the
    // victim are in range, a chunk is a power of two that divides the half
    // shard and fits under bit l (so its source run ins0(c C, l) .. + C is
    // contiguous and inside the shard), and the staging buffers hold it
    if (j < 0 || (s->P > 1 && (1 << j) >= s->P) || l < 0 || l >= s->nl || C == 0 || (C & (C - 1)) ||
        half % C || C > (1ull << l) || C > s->chunk_amps) {
        set_error("exchange: internal bounds check failed (g " + std::to_string(x.g) + ", l " + std::to_string(l) +
                  ", chunk " + std::to_string(C) + ")");
        return QSIM_EINVAL;
    }
    auto fill = [&](XchgParams &p, const Shard &sh, int b, uint64_t c, const void *stg) {
        p.own = sh.amps;
        p.stage = stg;
        p.p0 = c * C;
        p.n = C;
        p.l = l;
        p.b = b;
        p.shard_base = shard_base(s, sh);
        if (gop) {
            p.mode = 1;
            p.cls = gop->cls;
            p.cmask = full_cmask(*gop);
            std::memcpy(p.u, u, sizeof(p.u));
        } else {
            p.mode = 0;
        }
    };
    auto account = [&]() {
        s->st.kernels++;
        s->st.hbm_bytes += (double)C * ab * (gop ? 4.0 : 2.0);
    };
    static const bool via_comm = getenv("QSIM_XCHG_VIA_COMM") != nullptr;
    if (s->transport == QSIM_TRANSPORT_LOCAL && !via_comm) {
        for (auto &sa : s->shards) {
            if ((shard_phys(s, sa) >> j) & 1) continue;
            Shard *sb = nullptr;
            const uint32_t want = s->ginv[shard_phys(s, sa) | (1u << j)];
            for (auto &t : s->shards)
                if ((uint32_t)t.index == want) sb = &t;
            for (uint64_t c = 0; c < nchunks; ++c) {
                // sa (b=0) sends slot(l=1), sb (b=1) sends slot(l=0)
                const char *src_a = (const char *)sa.amps + ins0(c * C, l) * ab + ((size_t)1 << l) * ab;
                const char *src_b = (const char *)sb->amps + ins0(c * C, l) * ab;
                CU(cudaMemcpyAsync(s->stage[0], src_b, C * ab, cudaMemcpyDeviceToDevice, s->stream));
                CU(cudaMemcpyAsync(s->stage[1], src_a, C * ab, cudaMemcpyDeviceToDevice, s->stream));
                XchgParams pa{}, pb{};
                fill(pa, sa, 0, c, s->stage[0]);
                fill(pb, *sb, 1, c, s->stage[1]);
                prof_begin(s);
                if (s->enc == QSIM_ENC_FP64) {
                    launch_xchg_e(pa, s->stream);
                    launch_xchg_e(pb, s->stream);
                } else {
                    launch_xchg_a(pa, s->atab, s->stream);
                    launch_xchg_a(pb, s->atab, s->stream);
                }
                prof_end(s, QSIM_K_XCHG, 2.0 * (double)C * ab * (gop ? 4.0 : 2.0));
                account();
                account();
            }
            s->st.exchange_bytes += 2.0 * (double)half * ab;
            s->st.exchanges++;
        }
        CU(cudaGetLastError());
        return QSIM_OK;
    }
    // ---- NCCL (one shard per process): the double-buffered chunk pipeline.
    // QSIM_XCHG_VIA_COMM=1 runs it with the loopback transport on one GPU --
    // every shard of this process, device copies on the comm stream standing
    // in for ncclSend / ncclRecv, per-shard receive buffers -- so its
    // schedule, events and hazards are tested without a second GPU.
    // Hazards: a sent chunk's slot is overwritten only by the kernel of that
    // chunk, which waits on the comm work that sent it; a receive buffer is
    // reused (chunk c + 2) only after the kernel that read it (ev_comp).
    const bool nccl = s->transport == QSIM_TRANSPORT_NCCL;
    const size_t ns = s->shards.size();
    std::vector<int> bbit(ns);
    std::vector<size_t> partner_of(ns);
    for (size_t i = 0; i < ns; ++i) {
        bbit[i] = (shard_phys(s, s->shards[i]) >> j) & 1;
        if (!nccl) {
            const uint32_t want = s->ginv[shard_phys(s, s->shards[i]) ^ (1u << j)];
            size_t r = 0;
            while ((uint32_t)s->shards[r].index != want) ++r;
            partner_of[i] = r;
        }
    }
    char *rbuf = nullptr;  // loopback: per shard and buffer k, one chunk
    if (!nccl) {
        if (cudaMalloc(&rbuf, 2 * ns * C * ab) != cudaSuccess) {
            cudaGetLastError();
            set_error("exchange (comm path): staging allocation failed");
            return QSIM_ENOMEM;
        }
        if (!s->comm_stream) {
            CU(cudaStreamCreateWithFlags(&s->comm_stream, cudaStreamNonBlocking));
            for (int k2 = 0; k2 < 2; ++k2) {
                CU(cudaEventCreateWithFlags(&s->ev_recv[k2], cudaEventDisableTiming));
                CU(cudaEventCreateWithFlags(&s->ev_comp[k2], cudaEventDisableTiming));
            }
            CU(cudaEventCreateWithFlags(&s->ev_start, cudaEventDisableTiming));
        }
    }
    auto recv_buf = [&](size_t i, int k) -> void * {
        return nccl ? s->stage[k] : (void *)(rbuf + ((size_t)k * ns + i) * C * ab);
    };
    auto send_src = [&](size_t i, uint64_t c) {
        return (const char *)s->shards[i].amps + ins0(c * C, l) * ab + (bbit[i] ? 0 : ((size_t)1 << l) * ab);
    };
    // one profile record for the whole pipeline (transfers included: the
    // compute stream waits on every chunk's arrival), bytes = sent per direction
    prof_begin(s);
    CU(cudaEventRecord(s->ev_start, s->stream));
    CU(cudaStreamWaitEvent(s->comm_stream, s->ev_start, 0));
    int rc = QSIM_OK;
    for (uint64_t c = 0; c < nchunks && !rc; ++c) {
        const int k = (int)(c & 1);
        if (c >= 2) CU(cudaStreamWaitEvent(s->comm_stream, s->ev_comp[k], 0));
        if (nccl) {
            const int partner = (int)s->ginv[shard_phys(s, s->shards[0]) ^ (1u << j)];
            NC(ncclGroupStart());
            NC(ncclSend(send_src(0, c), C * ab, ncclUint8, partner, s->comm, s->comm_stream));
            NC(ncclRecv(s->stage[k], C * ab, ncclUint8, partner, s->comm, s->comm_stream));
            NC(ncclGroupEnd());
        } else {
            for (size_t i = 0; i < ns; ++i)  // shard i's sent half lands in its partner's receive buffer
                CU(cudaMemcpyAsync(recv_buf(partner_of[i], k), send_src(i, c), C * ab, cudaMemcpyDeviceToDevice,
                                   s->comm_stream));
        }
        CU(cudaEventRecord(s->ev_recv[k], s->comm_stream));
        CU(cudaStreamWaitEvent(s->stream, s->ev_recv[k], 0));
        for (size_t i = 0; i < ns; ++i) {
            XchgParams p{};
            fill(p, s->shards[i], bbit[i], c, recv_buf(i, k));
            if (s->enc == QSIM_ENC_FP64)
                launch_xchg_e(p, s->stream);
            else
                launch_xchg_a(p, s->atab, s->stream);
            account();
        }
        CU(cudaEventRecord(s->ev_comp[k], s->stream));
    }
    if (!nccl) {
        cudaStreamSynchronize(s->stream);
        cudaFree(rbuf);
    }
    if (rc) return rc;
    prof_end(s, QSIM_K_XCHG, (double)ns * (double)half * ab);
    s->st.exchange_bytes += (double)ns * (double)half * ab;
    s->st.exchanges++;
    CU(cudaGetLastError());
    return QSIM_OK;
}

// All-to-all remap (planner QSIM_OP_REMAP group, remap.cu): m (global g_i,
// local l_i) pairs swapped at once.  Shard phi trades its block B(t) (l bits
// = t) with block B(phi[j]) of the shard phi with j bits := t, for every
// t != phi[j].  The qubit map was updated by the planner.
static int remap_impl(qsim_state *s, std::vector<std::pair<int, int>> pairs) {
    std::sort(pairs.begin(), pairs.end(), [](const std::pair<int, int> &x, const std::pair<int, int> &y) {
        return x.second < y.second;  // by local bit
    });
    const int m = (int)pairs.size();
    if (m < 1 || m > kRemapMaxBits) {  // RemapVals holds 2^3 - 1 partners (the planner caps groups)
        set_error("remap: " + std::to_string(m) + " bits in one group (at most " + std::to_string(kRemapMaxBits) + ")");
        return QSIM_EINVAL;
    }
    RemapBlock blk{};
    blk.m = m;
    int jb[8];
    for (int i = 0; i < m; ++i) {
        blk.pos[i] = pairs[i].second;
        jb[i] = pairs[i].first - s->nl;
    }
    const uint64_t nblock = 1ull << (s->nl - m);
    const size_t ab = s->amp_bytes;
    auto jval = [&](uint32_t phi) {  // phi's j bits as a block value
        uint32_t v = 0;
        for (int i = 0; i < m; ++i) v |= ((phi >> jb[i]) & 1u) << i;
        return v;
    };
    auto with_j = [&](uint32_t phi, uint32_t t) {
        for (int i = 0; i < m; ++i) phi = (phi & ~(1u << jb[i])) | (((t >> i) & 1u) << jb[i]);
        return phi;
    };
    const uint32_t nt = 1u << m;
    static const bool via_pack = getenv("QSIM_REMAP_VIA_PACK") != nullptr;
    if (s->transport == QSIM_TRANSPORT_LOCAL && !via_pack) {
        prof_begin(s);
        for (auto &sa : s->shards) {
            const uint32_t pa = shard_phys(s, sa), ta = jval(pa);
            for (uint32_t t = 0; t < nt; ++t) {
                if (t == ta) continue;
                const uint32_t idxb = s->ginv[with_j(pa, t)];
                if (idxb < (uint32_t)sa.index) continue;  // each pair once
                Shard *sb = nullptr;
                for (auto &x : s->shards)
                    if ((uint32_t)x.index == idxb) sb = &x;
                launch_blockswap(sa.amps, sb->amps, nblock, blk, t, ta, ab, s->stream);
                s->st.kernels++;
                s->st.hbm_bytes += 4.0 * (double)nblock * ab;
            }
            s->st.exchange_bytes += (double)(nt - 1) * (double)nblock * ab;
        }
        prof_end(s, QSIM_K_XCHG, 2.0 * (double)s->P * (double)(nt - 1) * (double)nblock * ab);
        s->st.exchanges++;
        CU(cudaGetLastError());
        return QSIM_OK;
    }
    // ---- the pack / transfer / unpack pipeline: NCCL (one shard per process)
    // and, as its one-GPU test path (QSIM_REMAP_VIA_PACK with the loopback
    // transport), every shard of this process with device copies on the comm
    // stream standing in for the grouped sends / receives -- the same schedule,
    // buffers, events and slot / peer mapping.  Every chunk round trades one
    // slice of each of the 2^m - 1 foreign blocks with their owners.
    // Double-buffered: chunk c + 2 is packed while chunk c + 1 travels; buffer
    // k = c & 1 is one half of the staging.  Hazards: pack(c + 2) is enqueued on
    // the compute stream after unpack(c), which waited on the comm work of
    // chunk c (its sends read sendb[k], its receives wrote recvb[k]); the comm
    // work of chunk c + 2 waits on the event recorded after pack(c + 2).
    const bool nccl = s->transport == QSIM_TRANSPORT_NCCL;
    const size_t ns = s->shards.size();
    uint64_t C = 1;
    while (C * 2 * (nt - 1) * 2 <= s->chunk_amps && C * 2 <= nblock) C *= 2;
    const uint64_t nch = nblock / C;
    const size_t slot_bytes = (size_t)C * ab, area = slot_bytes * (nt - 1);
    char *send_base = nullptr, *recv_base = nullptr;
    if (nccl) {
        send_base = (char *)s->stage[0];
        recv_base = (char *)s->stage[1];
    } else {
        if (cudaMalloc(&send_base, 2 * area * ns) != cudaSuccess || cudaMalloc(&recv_base, 2 * area * ns) != cudaSuccess) {
            cudaGetLastError();
            if (send_base) cudaFree(send_base);
            set_error("remap (pack path): staging allocation failed");
            return QSIM_ENOMEM;
        }
        if (!s->comm_stream) {  // the loopback test path borrows the NCCL transport's stream and events
            CU(cudaStreamCreateWithFlags(&s->comm_stream, cudaStreamNonBlocking));
            for (int k2 = 0; k2 < 2; ++k2) {
                CU(cudaEventCreateWithFlags(&s->ev_recv[k2], cudaEventDisableTiming));
                CU(cudaEventCreateWithFlags(&s->ev_comp[k2], cudaEventDisableTiming));
            }
            CU(cudaEventCreateWithFlags(&s->ev_start, cudaEventDisableTiming));
        }
    }
    auto sendb = [&](size_t i, int k) { return send_base + ((size_t)k * ns + i) * area; };
    auto recvb = [&](size_t i, int k) { return recv_base + ((size_t)k * ns + i) * area; };
    std::vector<RemapVals> vals(ns);
    for (size_t i = 0; i < ns; ++i) {
        const uint32_t ta = jval(shard_phys(s, s->shards[i]));
        vals[i] = RemapVals{};
        for (uint32_t t = 0; t < nt; ++t)
            if (t != ta) vals[i].v[vals[i].n++] = t;  // slot p <-> block vals[i].v[p]
    }
    auto slot_of = [&](size_t i, uint32_t t) {  // position of block value t among shard i's slots
        int k = 0;
        while (vals[i].v[k] != t) ++k;
        return k;
    };
    auto issue = [&](uint64_t c) -> int {
        const int k = (int)(c & 1);
        for (size_t i = 0; i < ns; ++i)
            launch_pack_multi(s->shards[i].amps, sendb(i, k), c * C, C, blk, vals[i], ab, s->stream);
        CU(cudaEventRecord(s->ev_comp[k], s->stream));
        CU(cudaStreamWaitEvent(s->comm_stream, s->ev_comp[k], 0));
        if (nccl) {
            const uint32_t pa = shard_phys(s, s->shards[0]);
            NC(ncclGroupStart());
            for (int q = 0; q < vals[0].n; ++q) {
                const int peer = (int)s->ginv[with_j(pa, vals[0].v[q])];
                NC(ncclSend(sendb(0, k) + (size_t)q * slot_bytes, slot_bytes, ncclUint8, peer, s->comm, s->comm_stream));
                NC(ncclRecv(recvb(0, k) + (size_t)q * slot_bytes, slot_bytes, ncclUint8, peer, s->comm, s->comm_stream));
            }
            NC(ncclGroupEnd());
        } else {
            // shard i's slot for block t goes to the shard with j bits t, which
            // receives it into its slot for block ta(i)
            for (size_t i = 0; i < ns; ++i) {
                const uint32_t pa = shard_phys(s, s->shards[i]), ta = jval(pa);
                for (int q = 0; q < vals[i].n; ++q) {
                    const uint32_t idx = s->ginv[with_j(pa, vals[i].v[q])];
                    size_t r = 0;
                    while ((uint32_t)s->shards[r].index != idx) ++r;
                    CU(cudaMemcpyAsync(recvb(r, k) + (size_t)slot_of(r, ta) * slot_bytes,
                                       sendb(i, k) + (size_t)q * slot_bytes, slot_bytes, cudaMemcpyDeviceToDevice,
                                       s->comm_stream));
                }
            }
        }
        CU(cudaEventRecord(s->ev_recv[k], s->comm_stream));
        return QSIM_OK;
    };
    prof_begin(s);
    CU(cudaEventRecord(s->ev_start, s->stream));
    CU(cudaStreamWaitEvent(s->comm_stream, s->ev_start, 0));
    int rc = issue(0);
    if (!rc && nch > 1) rc = issue(1);
    for (uint64_t c = 0; c < nch && !rc; ++c) {
        const int k = (int)(c & 1);
        CU(cudaStreamWaitEvent(s->stream, s->ev_recv[k], 0));
        for (size_t i = 0; i < ns; ++i)
            launch_unpack_multi(s->shards[i].amps, recvb(i, k), c * C, C, blk, vals[i], ab, s->stream);
        s->st.kernels += 2 * (int64_t)ns;
        s->st.hbm_bytes += 4.0 * (double)ns * (double)(nt - 1) * (double)C * ab;
        if (c + 2 < nch) rc = issue(c + 2);
    }
    if (!nccl) {
        cudaStreamSynchronize(s->stream);
        cudaFree(send_base);
        cudaFree(recv_base);
    }
    if (rc) return rc;
    prof_end(s, QSIM_K_XCHG, 2.0 * (double)ns * (double)(nt - 1) * (double)nblock * ab);
    s->st.exchange_bytes += (double)ns * (double)(nt - 1) * (double)nblock * ab;
    s->st.exchanges++;
    CU(cudaGetLastError());
    return QSIM_OK;
}

// A rank that fails inside the exchange pipeline leaves its partners blocked in
// their sends / receives: abort the communicator so they fail fast;
// every later collective of this handle then returns QSIM_ECOMM.
static void comm_abort(qsim_state *s) {
    if (s->transport == QSIM_TRANSPORT_NCCL && s->comm) {
        ncclCommAbort(s->comm);
        s->comm = nullptr;
    }
}
static int exchange(qsim_state *s, const PlanOp &x, const PlanOp *gop, const double *u) {
    if (s->transport == QSIM_TRANSPORT_NCCL && !s->comm) {
        set_error("the NCCL communicator was aborted after an earlier error");
        return QSIM_ECOMM;
    }
    const int rc = exchange_impl(s, x, gop, u);
    if (rc) comm_abort(s);
    return rc;
}
static int remap(qsim_state *s, std::vector<std::pair<int, int>> pairs) {
    if (s->transport == QSIM_TRANSPORT_NCCL && !s->comm) {
        set_error("the NCCL communicator was aborted after an earlier error");
        return QSIM_ECOMM;
    }
    const int rc = remap_impl(s, std::move(pairs));
    if (rc) comm_abort(s);
    return rc;
}

// ============================================================================
// executor
// ============================================================================
static int run_gates_a(qsim_state *s, const std::vector<PlanOp> &run, const std::vector<const double *> &us);

static int execute(qsim_state *s, const qsim_gate *gates, size_t ngates, const std::vector<PlanOp> &ops) {
    std::vector<PlanOp> run;
    std::vector<const double *> us;
    std::deque<std::array<double, 8>> synth;  // phase parts of relabelled anti-diagonal gates
    auto flush = [&]() -> int {
        if (run.empty()) return QSIM_OK;
        int rc = (s->enc == QSIM_ENC_FP64) ? run_gates_e(s, run, us) : run_gates_a(s, run, us);
        run.clear();
        us.clear();
        return rc;
    };
    for (size_t i = 0; i < ops.size(); ++i) {
        const PlanOp &o = ops[i];
        if (o.type == QSIM_OP_RELABEL) {
            // anti-diagonal U = X . diag(u10, u01) with target and controls on global
            // bits: the phase part is a diagonal gate (per-shard factor), the X part
            // permutes the shards' physical labels -- no data moves
            const double *u = gates[o.gate_index].u;
            if (!(u[2] == 1.0 && u[3] == 0.0 && u[4] == 1.0 && u[5] == 0.0)) {
                synth.push_back({u[4], u[5], 0.0, 0.0, 0.0, 0.0, u[2], u[3]});
                PlanOp d = o;
                d.type = QSIM_OP_GATE;
                d.cls = classify(synth.back().data());
                if (d.cls != CLS_IDENT) {
                    run.push_back(d);
                    us.push_back(synth.back().data());
                }
            }
            RC(flush());
            const uint32_t tb = 1u << (o.l - s->nl);
            for (int r = 0; r < s->P; ++r) {
                bool on = true;
                for (int c = 0; c < o.nctrl; ++c) on = on && ((s->gphys[r] >> (o.ctrl[c] - s->nl)) & 1u);
                if (on) s->gphys[r] ^= tb;
            }
            for (int r = 0; r < s->P; ++r) s->ginv[s->gphys[r]] = (uint32_t)r;
            continue;
        }
        if (o.type == QSIM_OP_REMAP) {
            RC(flush());
            std::vector<std::pair<int, int>> pairs;
            size_t k = i;
            while (k < ops.size() && ops[k].type == QSIM_OP_REMAP && ops[k].gate_index == o.gate_index) {
                pairs.push_back({ops[k].g, ops[k].l});
                ++k;
            }
            i = k - 1;
            RC(remap(s, pairs));
            continue;
        }
        if (o.type == QSIM_OP_EXCHANGE) {
            RC(flush());
            const PlanOp *g = nullptr;
            if (i + 1 < ops.size() && ops[i + 1].type == QSIM_OP_GATE && ops[i + 1].gate_index == o.gate_index &&
                ops[i + 1].l == o.l) {
                g = &ops[i + 1];
                ++i;
            }
            if (g && s->enc == QSIM_ENC_ADAPTIVE2 && g->cls == CLS_DENSE) {
                // A dense gates need exact global bounds first: exchange, then the 2-phase gate
                RC(exchange(s, o, nullptr, nullptr));
                run.push_back(*g);
                us.push_back(gates[g->gate_index].u);
                RC(flush());
                continue;
            }
            RC(exchange(s, o, g, g ? gates[g->gate_index].u : nullptr));
            continue;
        }
        run.push_back(o);
        us.push_back(gates[o.gate_index].u);
    }
    RC(flush());
    s->st.gates += (int64_t)ngates;
    for (size_t g = 0; g < ngates; ++g) {
        if (gates[g].kind == QSIM_GATE_SWAP) continue;
        // per-gate algorithmic bytes (for the "effective" GB/s figure) on shard 0's view
        PlanOp o{};
        o.cls = classify(gates[g].u);
        if (o.cls == CLS_IDENT) continue;
        o.l = 0;
        o.nctrl = gates[g].ncontrols;
        o.ctrl[0] = o.ctrl[1] = 1;  // local placeholder: controls count, position irrelevant
        double amps = std::ldexp(1.0, s->nl - o.nctrl);
        double per = 2.0 * (double)s->amp_bytes;
        double bytes = amps * per;
        if (o.cls == CLS_DIAG) {
            const double *u = gates[g].u;
            bool one0 = u[0] == 1.0 && u[1] == 0.0, one1 = u[6] == 1.0 && u[7] == 0.0;
            if (one0 || one1) bytes *= 0.5;
        }
        s->st.gate_bytes += bytes * (double)s->shards.size();
    }
    return QSIM_OK;
}

// ============================================================================
// reductions
// ============================================================================
// phys[0] = norm^2, phys[1 + b] = sum_{physical bit b = 1} |a|^2 for every physical bit b < n
static int phys_probs(qsim_state *s, std::vector<double> &phys) {
    phys.assign(1 + s->n, 0.0);
    for (auto &sh : s->shards) {
        // the reduction walks 256-amplitude segments: shards below 2^8 amplitudes
        // are zero-padded to 256 (alloc_amps), so reduce over the padded size
        const int nr = std::max(s->nl, 8);
        if (s->enc == QSIM_ENC_FP64)
            launch_probs_e(sh.amps, nr, s->d_partials, s->d_out, s->stream);
        else
            launch_probs_a(sh.amps, nr, s->atab, s->d_partials, s->d_out, s->stream);
        s->st.kernels += 2;
        CU(cudaMemcpyAsync(s->h_out, s->d_out, RED_SLOTS * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
        CU(cudaStreamSynchronize(s->stream));
        phys[0] += s->h_out[0];
        for (int b = 0; b < s->nl; ++b) phys[1 + b] += s->h_out[1 + b];
        for (int b = s->nl; b < s->n; ++b)
            if (rank_bit(s, sh, b)) phys[1 + b] += s->h_out[0];
    }
    if (s->transport == QSIM_TRANSPORT_NCCL) {
        CU(cudaMemcpyAsync(s->d_out, phys.data(), phys.size() * sizeof(double), cudaMemcpyHostToDevice, s->stream));
        NC(ncclAllReduce(s->d_out, s->d_out, phys.size(), ncclFloat64, ncclSum, s->comm, s->stream));
        CU(cudaMemcpyAsync(phys.data(), s->d_out, phys.size() * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
        CU(cudaStreamSynchronize(s->stream));
    }
    return QSIM_OK;
}

}  // namespace qsim

// ============================================================================
// C-ABI
// ============================================================================
// ============================================================================
// QSIM_TRANSPORT_DEVICES: one process drives P GPUs (SURVEY.md §8(e) process
// model).  The handle owns P member handles, member r on
// device base + r with the NCCL transport as rank r of a communicator whose
// ranks all live in this process; one host thread per device runs every call
// on its member concurrently (NCCL collectives of one communicator need all
// ranks to enter them), so the exchange, remap and read-out code is exactly
// the one-process-per-GPU path.  Results of collective read-outs are
// identical on every rank; the caller gets member 0's.
// ============================================================================
namespace qsim {
struct QGroup {
    int P = 0, base = 0;
    std::vector<qsim_state *> m;
    std::vector<std::thread> th;
    std::mutex mu;
    std::condition_variable cv, cv_done;
    const std::function<int(int, qsim_state *)> *job = nullptr;
    uint64_t gen = 0;
    int pending = 0;
    bool stop = false;
    std::vector<int> rc;
    std::vector<std::string> err;
};

static void group_worker(QGroup *g, int r) {
    cudaSetDevice(g->base + r);
    uint64_t seen = 0;
    for (;;) {
        const std::function<int(int, qsim_state *)> *job;
        {
            std::unique_lock<std::mutex> lk(g->mu);
            g->cv.wait(lk, [&] { return g->stop || g->gen != seen; });
            if (g->stop) return;
            seen = g->gen;
            job = g->job;
        }
        cudaSetDevice(g->base + r);
        const int rc = (*job)(r, g->m[r]);
        std::string e = rc ? std::string(qsim_last_error()) : std::string();
        std::lock_guard<std::mutex> lk(g->mu);
        g->rc[r] = rc;
        g->err[r] = e;
        if (--g->pending == 0) g->cv_done.notify_all();
    }
}

// run f(r, member r) on every member's thread; the first failing rank's code / message
static int group_run(QGroup *g, const std::function<int(int, qsim_state *)> &f) {
    {
        std::unique_lock<std::mutex> lk(g->mu);
        g->job = &f;
        g->pending = g->P;
        ++g->gen;
        g->cv.notify_all();
        g->cv_done.wait(lk, [&] { return g->pending == 0; });
        g->job = nullptr;
    }
    for (int r = 0; r < g->P; ++r)
        if (g->rc[r]) {
            set_error("device " + std::to_string(g->base + r) + ": " + g->err[r]);
            return g->rc[r];
        }
    return QSIM_OK;
}

static void group_stop(QGroup *g) {
    {
        std::lock_guard<std::mutex> lk(g->mu);
        g->stop = true;
        g->cv.notify_all();
    }
    for (auto &t : g->th)
        if (t.joinable()) t.join();
}
}  // namespace qsim

#define GROUP_ALL(s, expr)                                                                              \
    do {                                                                                                \
        if ((s) && (s)->group)                                                                          \
            return group_run((s)->group, [&](int r_, qsim_state *m_) -> int { (void)r_; return (expr); }); \
    } while (0)

extern "C" {

const char *qsim_last_error(void) { return g_err.c_str(); }

int qsim_nccl_unique_id(uint8_t out[128]) {
    if (!out) return QSIM_EINVAL;
    ncclUniqueId id;
    NC(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
    return QSIM_OK;
}

int qsim_destroy(qsim_state *s) {
    if (!s) return QSIM_OK;
    if (s->group) {
        QGroup *g = s->group;
        group_run(g, [&](int r, qsim_state *m) {
            const int rc = qsim_destroy(m);
            g->m[r] = nullptr;
            return rc;
        });
        group_stop(g);
        delete g;
        delete s;
        return QSIM_OK;
    }
    if (s->dev >= 0) cudaSetDevice(s->dev);
    if (s->stream) cudaStreamSynchronize(s->stream);
    if (s->comm_stream) cudaStreamSynchronize(s->comm_stream);
    if (s->comm) ncclCommDestroy(s->comm);
    for (auto &sh : s->shards) {
        if (sh.amps) cudaFree(sh.amps);
        if (sh.amps2) cudaFree(sh.amps2);
    }
    if (s->d_oor) cudaFree(s->d_oor);
    for (auto &e : s->pc_cache)
        if (e.d) cudaFree(e.d);
    if (s->h_pc) cudaFreeHost(s->h_pc);
    for (int k = 0; k < 2; ++k) {
        if (s->stage[k]) cudaFree(s->stage[k]);
        if (s->ev_recv[k]) cudaEventDestroy(s->ev_recv[k]);
        if (s->ev_comp[k]) cudaEventDestroy(s->ev_comp[k]);
    }
    if (s->ev_start) cudaEventDestroy(s->ev_start);
    for (auto &r : s->prof_recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : s->ev_pool) cudaEventDestroy(e);
    if (s->d_partials) cudaFree(s->d_partials);
    if (s->d_out) cudaFree(s->d_out);
    if (s->d_acc) cudaFree(s->d_acc);
    if (s->h_out) cudaFreeHost(s->h_out);
    if (s->atab) atables_free(s->atab);
    if (s->stream) cudaStreamDestroy(s->stream);
    if (s->comm_stream) cudaStreamDestroy(s->comm_stream);
    delete s;
    return QSIM_OK;
}

static int init_state(qsim_state *s) {
    // |0...0>: a(0) = 1 on shard 0 (E); codes (127, 0) at 0, (-128, 0) elsewhere (A)
    reset_labels(s);
    for (auto &sh : s->shards) {
        size_t bytes = s->alloc_amps * s->amp_bytes;
        if (s->enc == QSIM_ENC_FP64) {
            CU(cudaMemsetAsync(sh.amps, 0, bytes, s->stream));
            if (sh.index == 0) {
                static const double one[2] = {1.0, 0.0};
                CU(cudaMemcpyAsync(sh.amps, one, sizeof(one), cudaMemcpyHostToDevice, s->stream));
            }
        } else {
            launch_init_a(sh.amps, s->alloc_amps, sh.index == 0, s->stream);
            s->st.kernels++;
        }
    }
    s->r0 = s->r1 = 0.5;
    s->r_stale = false;
    if (s->enc == QSIM_ENC_ADAPTIVE2) RC(atables_set(s->atab, s->r0, s->r1, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    return QSIM_OK;
}

int qsim_create_ex(const qsim_config *cfg, qsim_state **out) {
    if (!cfg || !out) {
        set_error("qsim_create_ex: null argument");
        return QSIM_EINVAL;
    }
    *out = nullptr;
    const int n = cfg->n_qubits, P = cfg->nshards;
    if (n < 2 || n > 63) {
        set_error("n_qubits must be in [2, 63] (PAPER.md:1418-1419)");
        return QSIM_EINVAL;
    }
    if (P < 1 || (P & (P - 1))) {
        set_error("nshards must be a power of two");
        return QSIM_EINVAL;
    }
    if (cfg->encoding != QSIM_ENC_FP64 && cfg->encoding != QSIM_ENC_ADAPTIVE2) {
        set_error("unknown encoding");
        return QSIM_EINVAL;
    }
    int k = 0;
    while ((1 << k) < P) ++k;
    const int nl = n - k;
    if (P > 1 && nl < 10) {
        set_error("a sharded state needs at least 10 local qubits (N - log2(P) >= 10)");
        return QSIM_EINVAL;
    }
    // nshards = 1 defaults to LOCAL; an explicit NCCL request with one rank is honoured
    // (communicator + collective read-out paths, used to test NCCL on one GPU)
    const int transport =
        (P == 1 && cfg->transport != QSIM_TRANSPORT_NCCL && cfg->transport != QSIM_TRANSPORT_DEVICES)
            ? QSIM_TRANSPORT_LOCAL
            : cfg->transport;
    if (transport == QSIM_TRANSPORT_DEVICES) {
        // one process, P devices: member r = rank r of an in-process NCCL communicator on device base + r
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
            cudaGetLastError();
            ndev = 0;
        }
        const int base = cfg->device >= 0 ? cfg->device : 0;
        if (base + P > ndev) {
            set_error("QSIM_TRANSPORT_DEVICES: " + std::to_string(P) + " shards need devices " + std::to_string(base) +
                      ".." + std::to_string(base + P - 1) + ", " + std::to_string(ndev) +
                      " visible (QSIM_TRANSPORT_LOCAL keeps every shard on one device)");
            return QSIM_EINVAL;
        }
        uint8_t id[128];
        RC(qsim_nccl_unique_id(id));
        auto *g = new QGroup();
        g->P = P;
        g->base = base;
        g->m.assign(P, nullptr);
        g->rc.assign(P, 0);
        g->err.assign(P, std::string());
        for (int r = 0; r < P; ++r) g->th.emplace_back(group_worker, g, r);
        int rc = group_run(g, [&](int r, qsim_state *) {
            qsim_config c = *cfg;
            c.transport = QSIM_TRANSPORT_NCCL;
            c.rank = r;
            c.device = base + r;
            c.nccl_id = id;
            return qsim_create_ex(&c, &g->m[r]);
        });
        if (rc) {
            const std::string msg = qsim_last_error();
            group_run(g, [&](int r, qsim_state *m) {
                qsim_destroy(m);
                g->m[r] = nullptr;
                return QSIM_OK;
            });
            group_stop(g);
            delete g;
            set_error(msg);
            return rc;
        }
        auto *s = new qsim_state();
        s->n = n;
        s->enc = cfg->encoding;
        s->P = P;
        s->nl = nl;
        s->transport = QSIM_TRANSPORT_DEVICES;
        s->dev = base;
        s->fuse = cfg->fuse;
        s->group = g;
        *out = s;
        return QSIM_OK;
    }
    if (transport != QSIM_TRANSPORT_LOCAL && transport != QSIM_TRANSPORT_NCCL) {
        set_error("unknown transport");
        return QSIM_EINVAL;
    }
    if (transport == QSIM_TRANSPORT_NCCL && (cfg->rank < 0 || cfg->rank >= P || !cfg->nccl_id)) {
        set_error("NCCL transport needs 0 <= rank < nshards and a 128-byte nccl_id");
        return QSIM_EINVAL;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        set_error("no CUDA device available (the library has no CPU fallback)");
        return QSIM_ECUDA;
    }
    auto *s = new qsim_state();
    s->n = n;
    s->enc = cfg->encoding;
    s->P = P;
    s->nl = nl;
    s->transport = transport;
    s->rank = transport == QSIM_TRANSPORT_NCCL ? cfg->rank : 0;
    s->fuse = cfg->fuse;
    s->a_policy = cfg->a_policy;
    if (cfg->a_policy != QSIM_A_POLICY_EXACT && cfg->a_policy != QSIM_A_POLICY_LAZY &&
        cfg->a_policy != QSIM_A_POLICY_FP32) {
        delete s;
        set_error("unknown a_policy");
        return QSIM_EINVAL;
    }
    if (const char *pr = getenv("QSIM_PASS_R")) s->pass_r = (atoi(pr) == 4) ? 4 : 5;
    if (const char *lk = getenv("QSIM_LPASS_K")) {
        s->pass_k = std::max(LP_MIN_K, std::min(LP_MAX_K, atoi(lk)));
        s->pass_k_env = true;
    }
    s->amp_bytes = s->enc == QSIM_ENC_FP64 ? 16 : 2;
    if (cfg->device >= 0) {
        if (cudaSetDevice(cfg->device) != cudaSuccess) {
            delete s;
            set_error("cudaSetDevice failed");
            return QSIM_ECUDA;
        }
    }
    cudaGetDevice(&s->dev);
    s->pl.init(n, P, nullptr);
    s->pl.remap = getenv("QSIM_NO_REMAP") == nullptr;  // all-to-all remaps (NEXT-1 (i)); off: pairwise only
    int rc = QSIM_OK;
    auto fail = [&](int code) {
        qsim_destroy(s);
        return code;
    };
    if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess) {
        set_error("cudaStreamCreate failed");
        return fail(QSIM_ECUDA);
    }
    // shards owned by this process
    if (transport == QSIM_TRANSPORT_NCCL) {
        s->shards.resize(1);
        s->shards[0].index = cfg->rank;
    } else {
        s->shards.resize(P);
        for (int r = 0; r < P; ++r) s->shards[r].index = r;
    }
    // capacity check before any allocation (also guards 2^nl * bytes overflow)
    {
        size_t free_b = 0, total_b = 0;
        cudaMemGetInfo(&free_b, &total_b);
        const double need = std::ldexp((double)s->amp_bytes, nl) * (double)s->shards.size();
        if (nl > 40 || need > (double)total_b) {
            set_error("state needs " + std::to_string(need) + " B on this device (2^" + std::to_string(nl) + " x " +
                      std::to_string(s->amp_bytes) + " B x " + std::to_string(s->shards.size()) +
                      " shard(s)); the device has " + std::to_string((double)total_b) + " B");
            return fail(QSIM_ENOMEM);
        }
    }
    s->alloc_amps = std::max<uint64_t>(1ull << nl, 256);
    const size_t shard_bytes = s->alloc_amps * s->amp_bytes;
    for (auto &sh : s->shards) {
        if (cudaMalloc(&sh.amps, shard_bytes) != cudaSuccess) {
            cudaGetLastError();
            set_error("cudaMalloc of " + std::to_string(shard_bytes) + " B per shard (" +
                      std::to_string(s->shards.size()) + " shard(s) on this device; state needs 2^" +
                      std::to_string(n) + " x " + std::to_string(s->amp_bytes) + " B in total) failed");
            return fail(QSIM_ENOMEM);
        }
    }
    if (P > 1) {
        // communication buffers of 2^{N-3} bytes in total by default
        int64_t cb = cfg->chunk_bytes;
        if (cb <= 0) {
            double tot = std::ldexp(1.0, n - 3) / P / 2.0;
            cb = (int64_t)std::min(tot, 512.0 * 1024 * 1024);
        }
        uint64_t ca = (uint64_t)cb / s->amp_bytes;
        uint64_t p2 = 1;
        while (p2 * 2 <= ca) p2 *= 2;
        s->chunk_amps = std::max<uint64_t>(p2, 256);
        s->chunk_amps = std::min<uint64_t>(s->chunk_amps, 1ull << (nl - 1));
        for (int k2 = 0; k2 < 2; ++k2) {
            if (cudaMalloc(&s->stage[k2], s->chunk_amps * s->amp_bytes) != cudaSuccess) {
                cudaGetLastError();
                set_error("cudaMalloc of the exchange staging buffers failed");
                return fail(QSIM_ENOMEM);
            }
        }
    }
    if (cudaMalloc(&s->d_partials, (size_t)red_blocks() * RED_SLOTS * sizeof(double) * 2) != cudaSuccess ||
        cudaMalloc(&s->d_out, 4096 * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&s->d_acc, 2 * sizeof(double)) != cudaSuccess ||
        cudaMallocHost(&s->h_out, 4096 * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        set_error("reduction scratch allocation failed");
        return fail(QSIM_ENOMEM);
    }
    if (s->enc == QSIM_ENC_ADAPTIVE2) {
        rc = atables_alloc(&s->atab);
        if (rc) return fail(rc);
    }
    if (transport == QSIM_TRANSPORT_NCCL) {
        if (cudaStreamCreateWithFlags(&s->comm_stream, cudaStreamNonBlocking) != cudaSuccess) return fail(QSIM_ECUDA);
        for (int k2 = 0; k2 < 2; ++k2) {
            cudaEventCreateWithFlags(&s->ev_recv[k2], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&s->ev_comp[k2], cudaEventDisableTiming);
        }
        cudaEventCreateWithFlags(&s->ev_start, cudaEventDisableTiming);
        ncclUniqueId id;
        std::memcpy(&id, cfg->nccl_id, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&s->comm, P, id, cfg->rank);
        if (r != ncclSuccess) {
            set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
            s->comm = nullptr;
            return fail(QSIM_ECOMM);
        }
    }
    rc = init_state(s);
    if (rc) return fail(rc);
    *out = s;
    return QSIM_OK;
}

int qsim_create(int n_qubits, int encoding, int ngpus, qsim_state **out) {
    qsim_config c{};
    c.n_qubits = n_qubits;
    c.encoding = encoding;
    c.nshards = ngpus;
    c.transport = ngpus > 1 ? QSIM_TRANSPORT_DEVICES : QSIM_TRANSPORT_LOCAL;
    c.device = -1;
    c.fuse = 1;
    return qsim_create_ex(&c, out);
}

int qsim_apply_circuit(qsim_state *s, const qsim_gate *gates, size_t ngates) {
    GROUP_ALL(s, qsim_apply_circuit(m_, gates, ngates));
    if (!s || (!gates && ngates)) {
        set_error("null argument");
        return QSIM_EINVAL;
    }
    RC(validate_gates(s->n, gates, ngates, true));
    cudaSetDevice(s->dev);
    std::vector<PlanOp> ops;
    s->pl.plan(gates, ngates, ops, true);
    return execute(s, gates, ngates, ops);
}

int qsim_apply_circuit_persistent(qsim_state *s, const qsim_gate *gates, size_t ngates) {
    if (!s || (!gates && ngates)) {
        set_error("null argument");
        return QSIM_EINVAL;
    }
    if (s->group || s->P != 1 || s->enc != QSIM_ENC_FP64 || s->capturing) {
        set_error("qsim_apply_circuit_persistent: one E shard on one device, outside graph capture");
        return QSIM_EUNSUPPORTED;
    }
    if (s->n < PERSIST_MIN_N || s->n > PERSIST_MAX_N) {
        set_error("qsim_apply_circuit_persistent: N must be in [" + std::to_string(PERSIST_MIN_N) + ", " +
                  std::to_string(PERSIST_MAX_N) + "] (the state lives in one cluster's shared memory)");
        return QSIM_EINVAL;
    }
    RC(validate_gates(s->n, gates, ngates, true));
    if (!ngates) return QSIM_OK;
    cudaSetDevice(s->dev);
    // logical -> physical through the qubit map; SWAP records relabel it (0 bytes)
    s->h_pg.resize(ngates);
    int ng = 0;
    for (size_t k = 0; k < ngates; ++k) {
        const qsim_gate &g = gates[k];
        if (g.kind == QSIM_GATE_SWAP) {
            s->pl.swap_bits(s->pl.pos[g.target], s->pl.pos[g.target2]);
            continue;
        }
        PersistGate &p = s->h_pg[ng++];
        std::memcpy(p.u, g.u, sizeof(p.u));
        p.t = s->pl.pos[g.target];
        p.cmask = 0;
        for (int c = 0; c < g.ncontrols; ++c) p.cmask |= 1u << s->pl.pos[g.controls[c]];
    }
    if (!ng) return QSIM_OK;
    int lcs = std::min(persist_lcs(), s->n - 3);
    if (const char *e = getenv("QSIM_PERSIST_LCS")) lcs = std::max(1, std::min(atoi(e), std::min(4, s->n - 3)));
    int K = persist_k(s->n, lcs);
    if (const char *e = getenv("QSIM_PERSIST_K")) K = std::max(3, std::min(atoi(e), std::min(4, s->n - lcs)));
    // a circuit seen before (same physical records, size and shape) replays its
    // device records: no planning, no upload, no host synchronisation
    uint64_t key = 1469598103934665603ull;
    {
        const unsigned char *b = reinterpret_cast<const unsigned char *>(s->h_pg.data());
        for (size_t i = 0; i < (size_t)ng * sizeof(PersistGate); ++i) key = (key ^ b[i]) * 1099511628211ull;
        key ^= ((uint64_t)s->n << 48) ^ ((uint64_t)lcs << 40) ^ ((uint64_t)K << 32) ^ (uint64_t)ng;
    }
    qsim_state::PcEntry *ent = nullptr;
    for (auto &e : s->pc_cache)
        if (e.d && e.key == key && e.lcs == lcs && e.K == K && e.recs.size() == (size_t)ng &&
            std::memcmp(e.recs.data(), s->h_pg.data(), (size_t)ng * sizeof(PersistGate)) == 0)
            ent = &e;
    if (!ent) {
        // phases of gates on <= K qubits (persist.cu), one launch per PERSIST_MAX_GATES gates
        std::vector<PersistPhase> ph;
        std::vector<PersistOp> ops;
        std::vector<std::pair<int, int>> lens;
        std::vector<char> rec;
        for (int k0 = 0; k0 < ng; k0 += PERSIST_MAX_GATES) {
            const int kn = std::min(ng - k0, PERSIST_MAX_GATES);
            if (persist_plan(s->h_pg.data() + k0, kn, s->n, K, lcs, ph, ops)) {
                set_error("qsim_apply_circuit_persistent: phase planning failed");
                return QSIM_EINVAL;
            }
            const size_t o = rec.size();
            rec.resize(o + ops.size() * sizeof(PersistOp) + ph.size() * sizeof(PersistPhase));
            std::memcpy(rec.data() + o, ops.data(), ops.size() * sizeof(PersistOp));
            std::memcpy(rec.data() + o + ops.size() * sizeof(PersistOp), ph.data(), ph.size() * sizeof(PersistPhase));
            lens.emplace_back((int)ph.size(), (int)ops.size());
            if (getenv("QSIM_PERSIST_DEBUG")) {
                int rem = 0;
                for (auto &x : ph) rem += x.remote != 0;
                fprintf(stderr, "persist: n %d cluster %d K %d gates %d phases %zu remote %d\n", s->n, 1 << lcs, K,
                        kn, ph.size(), rem);
            }
        }
        // the entry to (re)use: a free slot, else the least recently used of 8
        if (s->pc_cache.size() < 8) s->pc_cache.emplace_back();
        ent = &s->pc_cache[0];
        for (auto &e : s->pc_cache)
            if (!e.d || e.stamp < ent->stamp) ent = &e;
        CU(cudaStreamSynchronize(s->stream));  // the pinned staging and an evicted entry are free
        if (ent->d) cudaFree(ent->d);
        ent->d = nullptr;
        if (rec.size() > s->pg_cap) {
            if (s->h_pc) cudaFreeHost(s->h_pc);
            s->h_pc = nullptr;
            s->pg_cap = 0;
            if (cudaMallocHost(&s->h_pc, rec.size()) != cudaSuccess) {
                cudaGetLastError();
                set_error("qsim_apply_circuit_persistent: staging allocation failed");
                return QSIM_ENOMEM;
            }
            s->pg_cap = rec.size();
        }
        if (cudaMalloc(&ent->d, rec.size()) != cudaSuccess) {
            cudaGetLastError();
            ent->d = nullptr;
            set_error("qsim_apply_circuit_persistent: record buffer allocation failed");
            return QSIM_ENOMEM;
        }
        std::memcpy(s->h_pc, rec.data(), rec.size());
        CU(cudaMemcpyAsync(ent->d, s->h_pc, rec.size(), cudaMemcpyHostToDevice, s->stream));
        ent->key = key;
        ent->lcs = lcs;
        ent->K = K;
        ent->lens = lens;
        ent->recs.assign(s->h_pg.begin(), s->h_pg.begin() + ng);
    }
    ent->stamp = ++s->pc_clock;
    size_t at = 0;
    for (size_t c = 0; c < ent->lens.size(); ++c) {
        const int nph = ent->lens[c].first, kn = ent->lens[c].second;
        const PersistOp *d_ops = reinterpret_cast<const PersistOp *>(reinterpret_cast<char *>(ent->d) + at);
        const PersistPhase *d_ph = reinterpret_cast<const PersistPhase *>(d_ops + kn);
        at += kn * sizeof(PersistOp) + nph * sizeof(PersistPhase);
        prof_begin(s);
        if (launch_persist_e(s->shards[0].amps, s->n, lcs, K, d_ph, nph, d_ops, kn, s->stream)) {
            set_error("qsim_apply_circuit_persistent: cluster launch failed");
            return QSIM_ECUDA;
        }
        prof_end(s, QSIM_K_PASS, std::ldexp(32.0 * kn, s->n), 14.0 * kn * std::ldexp(1.0, s->n));
        s->st.kernels++;
    }
    s->st.gates += (int64_t)ngates;
    return QSIM_OK;
}

int qsim_apply_gate(qsim_state *s, const double u[8], int target, const int *controls, int ncontrols) {
    GROUP_ALL(s, qsim_apply_gate(m_, u, target, controls, ncontrols));
    if (!s || !u || (ncontrols > 0 && !controls) || ncontrols < 0 || ncontrols > 2) {
        set_error("qsim_apply_gate: bad arguments (ncontrols must be 0..2)");
        return QSIM_EINVAL;
    }
    qsim_gate g{};
    g.kind = QSIM_GATE_U;
    g.target = target;
    g.ncontrols = ncontrols;
    for (int c = 0; c < ncontrols; ++c) g.controls[c] = controls[c];
    std::memcpy(g.u, u, sizeof(g.u));
    return qsim_apply_circuit(s, &g, 1);
}

int qsim_apply_matrix(qsim_state *s, const double *U, const int *qubits, int k) {
    GROUP_ALL(s, qsim_apply_matrix(m_, U, qubits, k));
    if (!s || !U || !qubits || k < 1 || k > 3) {
        set_error("qsim_apply_matrix: bad arguments (k must be 1..3)");
        return QSIM_EINVAL;
    }
    for (int b = 0; b < k; ++b) {
        if (qubits[b] < 0 || qubits[b] >= s->n) {
            set_error("qsim_apply_matrix: qubit out of range");
            return QSIM_EINVAL;
        }
        for (int c = 0; c < b; ++c)
            if (qubits[c] == qubits[b]) {
                set_error("qsim_apply_matrix: duplicate qubits");
                return QSIM_EINVAL;
            }
    }
    const int M = 1 << k;
    for (int i = 0; i < 2 * M * M; ++i)
        if (!std::isfinite(U[i])) {
            set_error("qsim_apply_matrix: non-finite matrix entry");
            return QSIM_EINVAL;
        }
    // ||U^dagger U - I||_max <= 1e-10 (the same bound as qsim_apply_gate)
    for (int r = 0; r < M; ++r)
        for (int c = 0; c < M; ++c) {
            double re = 0.0, im = 0.0;
            for (int m = 0; m < M; ++m) {
                const double ar = U[2 * (m * M + r)], ai = -U[2 * (m * M + r) + 1];  // conj(U[m][r])
                const double br = U[2 * (m * M + c)], bi = U[2 * (m * M + c) + 1];
                re += ar * br - ai * bi;
                im += ar * bi + ai * br;
            }
            if (std::fabs(re - (r == c ? 1.0 : 0.0)) > 1e-10 || std::fabs(im) > 1e-10) {
                set_error("qsim_apply_matrix: ||U^dagger U - I||_max > 1e-10");
                return QSIM_ENOTUNITARY;
            }
        }
    if (s->enc != QSIM_ENC_FP64) {
        set_error("qsim_apply_matrix: E encoding only");
        return QSIM_EUNSUPPORTED;
    }
    cudaSetDevice(s->dev);
    // bring every global qubit of the set to a local bit (half-shard swap
    // exchanges), victims outside the set
    for (int b = 0; b < k; ++b) {
        const int pb = s->pl.pos[qubits[b]];
        if (pb < s->nl) continue;
        int avoid[3];
        int na = 0;
        for (int c = 0; c < k; ++c)
            if (s->pl.pos[qubits[c]] < s->nl) avoid[na++] = s->pl.pos[qubits[c]];
        const int l = s->pl.choose_victim(nullptr, 0, 0, avoid, na, false);
        if (l < 0) {
            set_error("qsim_apply_matrix: no local bit left for the exchange");
            return QSIM_EINVAL;
        }
        PlanOp x{};
        x.type = QSIM_OP_EXCHANGE;
        x.g = pb;
        x.l = l;
        RC(exchange(s, x, nullptr, nullptr));
        s->pl.swap_bits(pb, l);
    }
    MatKParams p{};
    p.k = k;
    p.ngroups = 1ull << (s->nl - k);
    for (int b = 0; b < k; ++b) p.phys[b] = p.sorted[b] = s->pl.pos[qubits[b]];
    std::sort(p.sorted, p.sorted + k);
    std::memcpy(p.u, U, sizeof(double) * 2 * M * M);
    for (auto &sh : s->shards) {
        p.a = sh.amps;
        prof_begin(s);
        launch_matk_e(p, s->stream);
        prof_end(s, QSIM_K_SWEEP, std::ldexp(32.0, s->nl), std::ldexp(8.0 * M, s->nl));
        s->st.kernels++;
        s->st.sweeps++;
        s->st.hbm_bytes += std::ldexp(32.0, s->nl);
        s->st.gate_bytes += std::ldexp(32.0, s->nl);
    }
    s->st.gates++;
    CU(cudaGetLastError());
    return QSIM_OK;
}

int qsim_apply_swap(qsim_state *s, int q1, int q2) {
    GROUP_ALL(s, qsim_apply_swap(m_, q1, q2));
    if (!s) return QSIM_EINVAL;
    qsim_gate g{};
    g.kind = QSIM_GATE_SWAP;
    g.target = q1;
    g.target2 = q2;
    return qsim_apply_circuit(s, &g, 1);
}

int qsim_reset(qsim_state *s) {
    GROUP_ALL(s, qsim_reset(m_));
    if (s && s->capturing) {
        set_error("qsim_reset: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (!s) return QSIM_EINVAL;
    cudaSetDevice(s->dev);
    if (s->comm_stream) CU(cudaStreamSynchronize(s->comm_stream));
    s->pl.init(s->n, s->P, nullptr);
    return init_state(s);
}

int qsim_reset_basis(qsim_state *s, uint64_t x) {
    GROUP_ALL(s, qsim_reset_basis(m_, x));
    if (!s) return QSIM_EINVAL;
    if (s->n < 64 && (x >> s->n)) {
        set_error("qsim_reset_basis: x must be < 2^N");
        return QSIM_EINVAL;
    }
    RC(qsim_reset(s));  // |0...0>, identity qubit map
    if (!x) return QSIM_OK;
    // move the single 1 from physical index 0 to physical index x (the map is the identity)
    const uint64_t lmask = (1ull << s->nl) - 1ull;
    for (auto &sh : s->shards) {
        const uint64_t base = shard_base(s, sh);
        if (base == 0) {  // holds index 0: back to zero
            if (s->enc == QSIM_ENC_FP64) {
                CU(cudaMemsetAsync(sh.amps, 0, 16, s->stream));
            } else {
                static const uint16_t zero_code = 0x0080u;  // (b0, b1) = (-128, 0)
                CU(cudaMemcpyAsync(sh.amps, &zero_code, 2, cudaMemcpyHostToDevice, s->stream));
            }
        }
        if (base == (x & ~lmask)) {
            char *dst = static_cast<char *>(sh.amps) + (x & lmask) * s->amp_bytes;
            if (s->enc == QSIM_ENC_FP64) {
                static const double one[2] = {1.0, 0.0};
                CU(cudaMemcpyAsync(dst, one, 16, cudaMemcpyHostToDevice, s->stream));
            } else {
                static const uint16_t one_code = 0x007fu;  // (b0, b1) = (127, 0): r = 1 exactly
                CU(cudaMemcpyAsync(dst, &one_code, 2, cudaMemcpyHostToDevice, s->stream));
            }
        }
    }
    CU(cudaStreamSynchronize(s->stream));
    return QSIM_OK;
}

int qsim_profile(qsim_state *s, int enable) {
    GROUP_ALL(s, qsim_profile(m_, enable));
    if (!s) return QSIM_EINVAL;
    s->prof = enable != 0;
    return QSIM_OK;
}

int qsim_profile_read(qsim_state *s, qsim_kernel_profile *out, int max, int *nout) {
    GROUP_ALL(s, r_ == 0 ? qsim_profile_read(m_, out, max, nout) : QSIM_OK);  // member 0's records
    if (s && s->capturing) {
        set_error("qsim_profile_read: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (!s || (!out && max > 0)) return QSIM_EINVAL;
    CU(cudaStreamSynchronize(s->stream));
    qsim_kernel_profile agg[QSIM_K_NUM];
    std::memset(agg, 0, sizeof(agg));
    for (auto &r : s->prof_recs) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        agg[r.kind].kind = r.kind;
        agg[r.kind].launches++;
        agg[r.kind].ms += ms;
        agg[r.kind].bytes += r.bytes;
        agg[r.kind].flops += r.flops;
        s->ev_pool.push_back(r.a);
        s->ev_pool.push_back(r.b);
    }
    s->prof_recs.clear();
    int k = 0;
    for (int c = 0; c < QSIM_K_NUM && k < max; ++c)
        if (agg[c].launches) out[k++] = agg[c];
    if (nout) *nout = k;
    return QSIM_OK;
}

int qsim_jit_sync(void) {
    lpass_jit_sync();
    return QSIM_OK;
}

int qsim_jit_shutdown(void) {
    lpass_jit_shutdown();
    return QSIM_OK;
}

int qsim_sync(qsim_state *s) {
    GROUP_ALL(s, qsim_sync(m_));
    if (!s) return QSIM_EINVAL;
    if (s->capturing) {
        set_error("qsim_sync: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    CU(cudaStreamSynchronize(s->stream));
    if (s->comm_stream) CU(cudaStreamSynchronize(s->comm_stream));
    return QSIM_OK;
}

struct qsim_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    qsim_state *owner = nullptr;
};

int qsim_graph_begin(qsim_state *s) {
    if (s && s->group) {
        set_error("qsim_graph_begin: not available for the multi-device transport");
        return QSIM_EUNSUPPORTED;
    }
    if (!s) return QSIM_EINVAL;
    if (s->capturing) {
        set_error("qsim_graph_begin: a capture is already open");
        return QSIM_EINVAL;
    }
    if (s->enc != QSIM_ENC_FP64 || (s->P > 1 && s->transport != QSIM_TRANSPORT_LOCAL)) {
        set_error("qsim_graph_begin: graphs need the E encoding and the loopback transport");
        return QSIM_EUNSUPPORTED;
    }
    CU(cudaStreamSynchronize(s->stream));
    s->cap_pos = s->pl.pos;
    s->cap_gphys = s->gphys;
    s->prof_saved = s->prof;
    s->prof = false;
    CU(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
    s->capturing = true;
    return QSIM_OK;
}

int qsim_graph_end(qsim_state *s, qsim_graph **out) {
    if (!s || !out) return QSIM_EINVAL;
    *out = nullptr;
    if (!s->capturing) {
        set_error("qsim_graph_end: no capture open");
        return QSIM_EINVAL;
    }
    s->capturing = false;
    s->prof = s->prof_saved;
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(s->stream, &g);
    if (e != cudaSuccess || !g) {
        cudaGetLastError();
        set_error(std::string("qsim_graph_end: capture failed: ") + cudaGetErrorString(e));
        if (g) cudaGraphDestroy(g);
        return QSIM_ECUDA;
    }
    if (s->pl.pos != s->cap_pos || s->gphys != s->cap_gphys) {
        cudaGraphDestroy(g);
        set_error("qsim_graph_end: the captured gates change the qubit map / shard labels; a replay would see "
                  "another layout (call qsim_reset)");
        return QSIM_EUNSUPPORTED;
    }
    auto *G = new qsim_graph();
    G->graph = g;
    G->owner = s;
    if (cudaGraphInstantiate(&G->exec, g, 0) != cudaSuccess) {
        cudaGetLastError();
        cudaGraphDestroy(g);
        delete G;
        set_error("qsim_graph_end: cudaGraphInstantiate failed");
        return QSIM_ECUDA;
    }
    *out = G;
    return QSIM_OK;
}

int qsim_graph_launch(qsim_state *s, qsim_graph *g) {
    if (!s || !g || g->owner != s || s->capturing) {
        set_error("qsim_graph_launch: graph / handle mismatch or capture open");
        return QSIM_EINVAL;
    }
    CU(cudaGraphLaunch(g->exec, s->stream));
    return QSIM_OK;
}

int qsim_graph_destroy(qsim_graph *g) {
    if (!g) return QSIM_OK;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
    return QSIM_OK;
}

void *qsim_stream(qsim_state *s, int shard) {
    if (s && s->group) {  // member `shard`'s stream (its device's)
        const int r = shard >= 0 && shard < s->P ? shard : 0;
        return (void *)s->group->m[r]->stream;
    }
    return s ? (void *)s->stream : nullptr;
}

int qsim_get_stats(qsim_state *s, qsim_stats *out) {
    if (s && s->group && out) {  // summed over the members (the shards this process owns)
        std::vector<qsim_stats> v(s->P);
        RC(group_run(s->group, [&](int r, qsim_state *m) { return qsim_get_stats(m, &v[r]); }));
        qsim_stats t{};
        for (const auto &x : v) {
            t.gates = x.gates;
            t.kernels += x.kernels;
            t.sweeps += x.sweeps;
            t.passes += x.passes;
            t.fused_gates += x.fused_gates;
            t.exchanges = std::max(t.exchanges, x.exchanges);
            t.hbm_bytes += x.hbm_bytes;
            t.gate_bytes += x.gate_bytes;
            t.exchange_bytes += x.exchange_bytes;
            t.stages += x.stages;
            t.jit_passes += x.jit_passes;
            t.a_rescales = std::max(t.a_rescales, x.a_rescales);  // per gate, the same on every member
            t.a_dense = std::max(t.a_dense, x.a_dense);
        }
        *out = t;
        return QSIM_OK;
    }
    if (!s || !out) return QSIM_EINVAL;
    *out = s->st;
    return QSIM_OK;
}
int qsim_reset_stats(qsim_state *s) {
    GROUP_ALL(s, qsim_reset_stats(m_));
    if (!s) return QSIM_EINVAL;
    s->st = qsim_stats{};
    return QSIM_OK;
}

int qsim_get_qubit_map(qsim_state *s, int *pos) {
    GROUP_ALL(s, r_ == 0 ? qsim_get_qubit_map(m_, pos) : QSIM_OK);  // identical on every member
    if (!s || !pos) return QSIM_EINVAL;
    for (int q = 0; q < s->n; ++q) pos[q] = s->pl.pos[q];
    return QSIM_OK;
}

int qsim_norm(qsim_state *s, double *norm2) {
    std::vector<double> g_sc(s && s->group ? s->P : 0);
    GROUP_ALL(s, qsim_norm(m_, r_ == 0 ? norm2 : &g_sc[r_]));
    if (s && s->capturing) {
        set_error("qsim_norm: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (!s || !norm2) return QSIM_EINVAL;
    cudaSetDevice(s->dev);
    std::vector<double> phys;
    RC(phys_probs(s, phys));
    *norm2 = phys[0];
    return QSIM_OK;
}

int qsim_magnitude_range(qsim_state *s, double *min_nonzero, double *max) {
    std::vector<double> g_sc(s && s->group ? 2 * s->P : 0);
    GROUP_ALL(s, qsim_magnitude_range(m_, r_ == 0 ? min_nonzero : &g_sc[2 * r_], r_ == 0 ? max : &g_sc[2 * r_ + 1]));
    if (!s || !min_nonzero || !max) return QSIM_EINVAL;
    if (s->capturing) {
        set_error("qsim_magnitude_range: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (s->enc != QSIM_ENC_FP64) {
        set_error("qsim_magnitude_range: E encoding only (an A state's range is its bounds, qsim_get_codes)");
        return QSIM_EUNSUPPORTED;
    }
    cudaSetDevice(s->dev);
    double mn = INFINITY, mx = 0.0;
    for (auto &sh : s->shards) {
        uint64_t init[2] = {0x7ff0000000000000ull, 0ull};  // (+inf, 0) as bit patterns
        CU(cudaMemcpyAsync(s->d_out, init, sizeof(init), cudaMemcpyHostToDevice, s->stream));
        launch_absrange_e(sh.amps, 1ull << s->nl, s->d_out, s->stream);
        s->st.kernels++;
        CU(cudaMemcpyAsync(s->h_out, s->d_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
        CU(cudaStreamSynchronize(s->stream));
        mn = std::min(mn, s->h_out[0]);
        mx = std::max(mx, s->h_out[1]);
    }
    if (s->transport == QSIM_TRANSPORT_NCCL && s->P > 1) {
        double v[2] = {mn, -mx};
        CU(cudaMemcpyAsync(s->d_out, v, sizeof(v), cudaMemcpyHostToDevice, s->stream));
        NC(ncclAllReduce(s->d_out, s->d_out, 2, ncclDouble, ncclMin, s->comm, s->stream));
        CU(cudaMemcpyAsync(s->h_out, s->d_out, sizeof(v), cudaMemcpyDeviceToHost, s->stream));
        CU(cudaStreamSynchronize(s->stream));
        mn = s->h_out[0];
        mx = -s->h_out[1];
    }
    *min_nonzero = std::isinf(mn) ? 0.0 : std::sqrt(mn);
    *max = std::sqrt(mx);
    return QSIM_OK;
}

int qsim_overlap(qsim_state *a, qsim_state *b, double *out) {
    if ((a && a->group) || (b && b->group)) {
        set_error("qsim_overlap: not available for the multi-device transport");
        return QSIM_EUNSUPPORTED;
    }
    if (!a || !b || !out) return QSIM_EINVAL;
    if (a->capturing || b->capturing) {
        set_error("qsim_overlap: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (a->n != b->n || a->P != b->P || a->dev != b->dev || (a->P > 1 && (a->transport != QSIM_TRANSPORT_LOCAL ||
                                                                         b->transport != QSIM_TRANSPORT_LOCAL))) {
        set_error("qsim_overlap: the handles need the same N, shard count and device, loopback transport");
        return QSIM_EUNSUPPORTED;
    }
    if (a->pl.pos != b->pl.pos || a->gphys != b->gphys) {
        set_error("qsim_overlap: the handles have different qubit maps / shard labels");
        return QSIM_EUNSUPPORTED;
    }
    cudaSetDevice(a->dev);
    CU(cudaStreamSynchronize(b->stream));
    double sr = 0.0, si = 0.0;
    for (size_t k = 0; k < a->shards.size(); ++k) {
        launch_overlap(a->shards[k].amps, a->enc == QSIM_ENC_FP64 ? nullptr : a->atab, b->shards[k].amps,
                       b->enc == QSIM_ENC_FP64 ? nullptr : b->atab, 1ull << a->nl, a->d_partials, a->d_out, a->stream);
        a->st.kernels += 2;
        CU(cudaMemcpyAsync(a->h_out, a->d_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, a->stream));
        CU(cudaStreamSynchronize(a->stream));
        sr += a->h_out[0];
        si += a->h_out[1];
    }
    out[0] = sr;
    out[1] = si;
    return QSIM_OK;
}

int qsim_probabilities(qsim_state *s, double *p1) {
    std::vector<double> g_sc(s && s->group ? (size_t)s->P * s->n : 0);
    GROUP_ALL(s, qsim_probabilities(m_, r_ == 0 ? p1 : &g_sc[(size_t)r_ * s->n]));
    if (s && s->capturing) {
        set_error("qsim_probabilities: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (!s || !p1) return QSIM_EINVAL;
    cudaSetDevice(s->dev);
    std::vector<double> phys;
    RC(phys_probs(s, phys));
    for (int q = 0; q < s->n; ++q) p1[q] = phys[1 + s->pl.pos[q]];
    return QSIM_OK;
}

static int pair_sums_local(qsim_state *s, int b, double &sr, double &si) {
    sr = si = 0.0;
    for (auto &sh : s->shards) {
        if (s->enc == QSIM_ENC_FP64)
            launch_pairdot_e(sh.amps, s->nl, b, s->d_partials, s->d_out, s->stream);
        else
            launch_pairdot_a(sh.amps, s->nl, b, s->atab, s->d_partials, s->d_out, s->stream);
        s->st.kernels += 2;
        CU(cudaMemcpyAsync(s->h_out, s->d_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
        CU(cudaStreamSynchronize(s->stream));
        sr += s->h_out[0];
        si += s->h_out[1];
    }
    return QSIM_OK;
}

int qsim_expectations(qsim_state *s, double *q) {
    std::vector<double> g_sc(s && s->group ? (size_t)s->P * 3 * s->n : 0);
    GROUP_ALL(s, qsim_expectations(m_, r_ == 0 ? q : &g_sc[(size_t)r_ * 3 * s->n]));
    if (s && s->capturing) {
        set_error("qsim_expectations: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (!s || !q) return QSIM_EINVAL;
    cudaSetDevice(s->dev);
    std::vector<double> phys;
    RC(phys_probs(s, phys));
    std::vector<double> Sr(s->n, 0.0), Si(s->n, 0.0);
    std::vector<int> done(s->n, 0);
    // local qubits first
    for (int lq = 0; lq < s->n; ++lq) {
        int b = s->pl.pos[lq];
        if (b >= s->nl) continue;
        RC(pair_sums_local(s, b, Sr[lq], Si[lq]));
        done[lq] = 1;
    }
    for (int lq = 0; lq < s->n; ++lq) {
        if (done[lq]) continue;
        int b = s->pl.pos[lq];
        if (s->transport == QSIM_TRANSPORT_LOCAL) {
            // pairs across shards r (bit 0) and r | 2^(b-nl): dot products, no data movement
            const int j = b - s->nl;
            for (auto &sa : s->shards) {
                if ((shard_phys(s, sa) >> j) & 1) continue;
                for (auto &sb : s->shards)
                    if ((uint32_t)sb.index == s->ginv[shard_phys(s, sa) | (1u << j)]) {
                        if (s->enc == QSIM_ENC_FP64)
                            launch_dot_e(sa.amps, sb.amps, 1ull << s->nl, s->d_partials, s->d_out, s->stream);
                        else
                            launch_dot_a(sa.amps, sb.amps, 1ull << s->nl, s->atab, s->d_partials, s->d_out,
                                         s->stream);
                        s->st.kernels += 2;
                        CU(cudaMemcpyAsync(s->h_out, s->d_out, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                                           s->stream));
                        CU(cudaStreamSynchronize(s->stream));
                        Sr[lq] += s->h_out[0];
                        Si[lq] += s->h_out[1];
                    }
            }
        } else {
            // NCCL: move the qubit to a local bit with a pure swap exchange (a relabelling)
            int avoid[1] = {-1};
            int l = s->pl.choose_victim(nullptr, 0, 0, avoid, 0, false);
            PlanOp x{};
            x.type = QSIM_OP_EXCHANGE;
            x.g = b;
            x.l = l;
            RC(exchange(s, x, nullptr, nullptr));
            s->pl.swap_bits(b, l);
            RC(pair_sums_local(s, l, Sr[lq], Si[lq]));
        }
    }
    if (s->transport == QSIM_TRANSPORT_NCCL) {
        std::vector<double> v(2 * s->n);
        for (int i = 0; i < s->n; ++i) {
            v[i] = Sr[i];
            v[s->n + i] = Si[i];
        }
        CU(cudaMemcpyAsync(s->d_out, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, s->stream));
        NC(ncclAllReduce(s->d_out, s->d_out, v.size(), ncclFloat64, ncclSum, s->comm, s->stream));
        CU(cudaMemcpyAsync(v.data(), s->d_out, v.size() * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
        CU(cudaStreamSynchronize(s->stream));
        for (int i = 0; i < s->n; ++i) {
            Sr[i] = v[i];
            Si[i] = v[s->n + i];
        }
    }
    // expectation values of the normalised state (Eq. STAT1; reading R-B7)
    const double nrm = phys[0];
    for (int lq = 0; lq < s->n; ++lq) {
        q[3 * lq + 0] = (nrm - 2.0 * Sr[lq]) / (2.0 * nrm);
        q[3 * lq + 1] = (nrm - 2.0 * Si[lq]) / (2.0 * nrm);
        q[3 * lq + 2] = phys[1 + s->pl.pos[lq]] / nrm;
    }
    return QSIM_OK;
}

static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Project qubit onto `out` and renormalise (M's collapse, CLEAR / SET).
static int collapse(qsim_state *s, int b, int out, double keep) {
    if (!(keep >= 1e-14)) {
        set_error("projection onto a state with norm^2 < 1e-14 (PAPER.md:1481)");
        return QSIM_EZERONORM;
    }
    const double f = 1.0 / std::sqrt(keep);
    if (s->enc == QSIM_ENC_FP64) {
        for (auto &sh : s->shards) {
            if (b < s->nl) {
                launch_collapse_e(sh.amps, 1ull << s->nl, b, out, f, s->stream);
            } else if (rank_bit(s, sh, b) != out) {
                CU(cudaMemsetAsync(sh.amps, 0, ((size_t)1 << s->nl) * s->amp_bytes, s->stream));
            } else {
                launch_scale_all_e(sh.amps, 1ull << s->nl, f, s->stream);
            }
            s->st.kernels++;
        }
    } else {
        RC(measure_collapse_a(s, b, out, f));
    }
    CU(cudaStreamSynchronize(s->stream));
    return QSIM_OK;
}

int qsim_measure_u(qsim_state *s, int qubit, double u, int *outcome, double *p0_out) {
    std::vector<int> g_o(s && s->group ? s->P : 0);
    std::vector<double> g_p(s && s->group ? s->P : 0);
    GROUP_ALL(s, qsim_measure_u(m_, qubit, u, r_ == 0 ? outcome : &g_o[r_], r_ == 0 ? p0_out : (p0_out ? &g_p[r_] : nullptr)));
    if (s && s->capturing) {
        set_error("qsim_measure_u: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (!s || !outcome || qubit < 0 || qubit >= s->n) {
        set_error("qsim_measure: bad qubit or null outcome");
        return QSIM_EINVAL;
    }
    cudaSetDevice(s->dev);
    std::vector<double> phys;
    RC(phys_probs(s, phys));
    const int b = s->pl.pos[qubit];
    const double s1 = phys[1 + b], s0 = phys[0] - s1;
    const double p0 = s0 / phys[0];
    if (p0_out) *p0_out = p0;
    const int out = (u < p0) ? 0 : 1;
    RC(collapse(s, b, out, out ? s1 : s0));
    *outcome = out;
    return QSIM_OK;
}

int qsim_project(qsim_state *s, int qubit, int value) {
    GROUP_ALL(s, qsim_project(m_, qubit, value));
    if (s && s->capturing) {
        set_error("qsim_project: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (!s || qubit < 0 || qubit >= s->n || (value != 0 && value != 1)) {
        set_error("qsim_project: bad qubit or value (0 = CLEAR, 1 = SET)");
        return QSIM_EINVAL;
    }
    cudaSetDevice(s->dev);
    std::vector<double> phys;
    RC(phys_probs(s, phys));
    const int b = s->pl.pos[qubit];
    const double s1 = phys[1 + b], s0 = phys[0] - s1;
    return collapse(s, b, value, value ? s1 : s0);
}

int qsim_sample(qsim_state *s, size_t nsamples, uint64_t seed, uint64_t *out) {
    std::vector<uint64_t> g_sc(s && s->group ? (size_t)s->P * nsamples : 0);
    GROUP_ALL(s, qsim_sample(m_, nsamples, seed, r_ == 0 ? out : &g_sc[(size_t)r_ * nsamples]));
    if (s && s->capturing) {
        set_error("qsim_sample: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (!s || (nsamples && !out)) return QSIM_EINVAL;
    if (s->transport == QSIM_TRANSPORT_NCCL && !s->comm) {
        set_error("the NCCL communicator was aborted after an earlier error");
        return QSIM_ECOMM;
    }
    if (s->n > 34) {
        set_error("qsim_sample needs an 8 B x 2^N probability array (N <= 34)");
        return QSIM_EINVAL;
    }
    cudaSetDevice(s->dev);
    std::vector<void *> amps;
    std::vector<uint64_t> bases;
    for (auto &sh : s->shards) {
        amps.push_back(sh.amps);
        bases.push_back(shard_base(s, sh));
    }
    s->st.kernels += 4;
    return sample_logical(amps.data(), bases.data(), (int)amps.size(), s->nl, s->n, s->pl.inv.data(), s->enc, s->atab,
                          nsamples, seed, out, s->stream,
                          s->transport == QSIM_TRANSPORT_NCCL ? (void *)s->comm : nullptr);
}

int qsim_set_qubit_map(qsim_state *s, const int *pos) {
    GROUP_ALL(s, qsim_set_qubit_map(m_, pos));
    if (!s || !pos) return QSIM_EINVAL;
    std::vector<int> seen(s->n, 0);
    for (int q = 0; q < s->n; ++q) {
        if (pos[q] < 0 || pos[q] >= s->n || seen[pos[q]]) {
            set_error("qsim_set_qubit_map: not a permutation of 0..N-1");
            return QSIM_EINVAL;
        }
        seen[pos[q]] = 1;
    }
    for (int q = 0; q < s->n; ++q) {
        s->pl.pos[q] = pos[q];
        s->pl.inv[pos[q]] = q;
    }
    return QSIM_OK;
}

int qsim_aux_amplitudes(int n_qubits, const qsim_gate *gates, size_t ngates, const uint64_t *idx, size_t m,
                        double *out, double *abs_sum) {
    if ((ngates && !gates) || (m && (!idx || !out)) || n_qubits < 2 || n_qubits > 63) {
        set_error("qsim_aux_amplitudes: bad arguments");
        return QSIM_EINVAL;
    }
    RC(validate_gates(n_qubits, gates, ngates, true));
    for (size_t k = 0; k < m; ++k)
        if (idx[k] >> n_qubits) {
            set_error("qsim_aux_amplitudes: index out of range");
            return QSIM_EINVAL;
        }
    return aux_amplitudes(n_qubits, gates, ngates, idx, m, out, abs_sum, 40);
}

int qsim_prepare_shorbox(qsim_state *s, int nx, uint64_t G, uint64_t y) {
    GROUP_ALL(s, qsim_prepare_shorbox(m_, nx, G, y));
    if (!s || nx < 0 || nx >= s->n || G < 2 || y < 1 || y >= G) {
        set_error("qsim_prepare_shorbox: need 0 <= nx < N, G >= 2, 1 <= y < G");
        return QSIM_EINVAL;
    }
    if (s->n - nx < 64 && G > (1ull << (s->n - nx))) {
        set_error("qsim_prepare_shorbox: G does not fit the f-register (N - nx qubits)");
        return QSIM_EINVAL;
    }
    cudaSetDevice(s->dev);
    if (s->comm_stream) CU(cudaStreamSynchronize(s->comm_stream));
    std::vector<void *> amps;
    std::vector<uint64_t> bases;
    for (auto &sh : s->shards) {
        amps.push_back(sh.amps);
        bases.push_back(shard_base(s, sh));
    }
    RC(shorbox(amps.data(), bases.data(), (int)amps.size(), s->nl, s->n, s->pl.inv.data(), s->enc, nx, G, y, s->stream));
    s->st.kernels += (int64_t)amps.size();
    if (s->enc == QSIM_ENC_ADAPTIVE2) {
        const double r = (nx == 0) ? 0.5 : std::ldexp(1.0, -nx / 2) * ((nx & 1) ? 0.70710678118654752440 : 1.0);
        s->r0 = s->r1 = r;  // every non-zero amplitude has magnitude 2^{-nx/2} (reading R-A7/R-A8)
        s->r_stale = false;
        RC(atables_set(s->atab, s->r0, s->r1, s->stream));
    }
    return QSIM_OK;
}

int qsim_measure(qsim_state *s, int qubit, uint64_t seed, int *outcome) {
    std::vector<int> g_o(s && s->group ? s->P : 0);
    GROUP_ALL(s, qsim_measure(m_, qubit, seed, r_ == 0 ? outcome : &g_o[r_]));
    if (s && s->capturing) {
        set_error("qsim_measure: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    uint64_t x = splitmix64(seed);
    double u = (double)(x >> 11) * (1.0 / 9007199254740992.0);
    return qsim_measure_u(s, qubit, u, outcome, nullptr);
}

static uint64_t logical_to_phys(const qsim_state *s, uint64_t L) {
    uint64_t p = 0;
    for (int q = 0; q < s->n; ++q)
        if ((L >> q) & 1ull) p |= 1ull << s->pl.pos[q];
    return p;
}

int qsim_get_amplitudes(qsim_state *s, const uint64_t *idx, size_t m, double *out) {
    std::vector<double> g_sc(s && s->group ? (size_t)(s->P - 1) * 2 * m : 0);
    GROUP_ALL(s, qsim_get_amplitudes(m_, idx, m, r_ == 0 ? out : &g_sc[(size_t)(r_ - 1) * 2 * m]));
    if (s && s->capturing) {
        set_error("qsim_get_amplitudes: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (!s || (m && (!idx || !out))) return QSIM_EINVAL;
    cudaSetDevice(s->dev);
    const uint64_t dim_mask = (s->n == 64) ? ~0ull : ((1ull << s->n) - 1ull);
    for (size_t k = 0; k < m; ++k)
        if (idx[k] & ~dim_mask) {
            set_error("amplitude index out of range");
            return QSIM_EINVAL;
        }
    if (!m) return QSIM_OK;
    // device scratch: offsets + results for m entries.  A local failure must not
    // skip the NCCL all-reduce the other ranks enter: it is folded
    // into the reduction as an error count instead.
    uint64_t *d_off = nullptr;
    double *d_val = nullptr;
    std::vector<double> res(2 * m, 0.0);
    std::vector<uint64_t> off;
    std::vector<size_t> which;
    int rc = QSIM_OK;
    if (cudaMalloc(&d_off, m * sizeof(uint64_t)) != cudaSuccess || cudaMalloc(&d_val, m * 2 * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        rc = QSIM_ENOMEM;
    }
    const uint64_t lmask = (1ull << s->nl) - 1ull;
    for (auto &sh : s->shards) {
        if (rc) break;
        off.clear();
        which.clear();
        for (size_t k = 0; k < m; ++k) {
            uint64_t p = logical_to_phys(s, idx[k]);
            if ((p >> s->nl) == (uint64_t)shard_phys(s, sh)) {
                off.push_back(p & lmask);
                which.push_back(k);
            }
        }
        if (off.empty()) continue;
        if (cudaMemcpyAsync(d_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice, s->stream) != cudaSuccess) {
            rc = QSIM_ECUDA;
            break;
        }
        if (s->enc == QSIM_ENC_FP64)
            launch_gather_e(sh.amps, d_off, off.size(), d_val, s->stream);
        else
            launch_gather_a(sh.amps, d_off, off.size(), s->atab, d_val, s->stream);
        s->st.kernels++;
        std::vector<double> tmp(2 * off.size());
        cudaMemcpyAsync(tmp.data(), d_val, tmp.size() * 8, cudaMemcpyDeviceToHost, s->stream);
        if (cudaStreamSynchronize(s->stream) != cudaSuccess) {
            rc = QSIM_ECUDA;
            break;
        }
        for (size_t k = 0; k < which.size(); ++k) {
            res[2 * which[k]] = tmp[2 * k];
            res[2 * which[k] + 1] = tmp[2 * k + 1];
        }
    }
    if (s->transport == QSIM_TRANSPORT_NCCL) {
        // chunks of the pre-allocated 4096-double scratch: element 0 = error count,
        // then up to 4095 values; the same number of chunks on every rank
        const size_t per = 4095;
        const size_t nchunk = (res.size() + per - 1) / per;
        int nerr = 0;
        for (size_t c = 0; c < std::max<size_t>(nchunk, 1); ++c) {
            const size_t lo = c * per, cnt = std::min(per, res.size() - std::min(res.size(), lo));
            s->h_out[0] = rc ? 1.0 : 0.0;
            std::memcpy(s->h_out + 1, res.data() + lo, cnt * 8);
            if (!s->comm) {
                rc = QSIM_ECOMM;
                break;
            }
            cudaMemcpyAsync(s->d_out, s->h_out, (cnt + 1) * 8, cudaMemcpyHostToDevice, s->stream);
            if (ncclAllReduce(s->d_out, s->d_out, cnt + 1, ncclFloat64, ncclSum, s->comm, s->stream) != ncclSuccess)
                nerr++;
            cudaMemcpyAsync(s->h_out, s->d_out, (cnt + 1) * 8, cudaMemcpyDeviceToHost, s->stream);
            cudaStreamSynchronize(s->stream);
            if (s->h_out[0] != 0.0 && !rc) rc = QSIM_ECOMM;  // another rank failed
            std::memcpy(res.data() + lo, s->h_out + 1, cnt * 8);
        }
        if (nerr && !rc) rc = QSIM_ECOMM;
    }
    cudaFree(d_off);
    cudaFree(d_val);
    if (rc) {
        set_error("qsim_get_amplitudes failed");
        return rc;
    }
    std::memcpy(out, res.data(), res.size() * 8);
    return QSIM_OK;
}

static int upload_inv(qsim_state *s, int **d_inv) {
    CU(cudaMalloc(d_inv, s->n * sizeof(int)));
    CU(cudaMemcpyAsync(*d_inv, s->pl.inv.data(), s->n * sizeof(int), cudaMemcpyHostToDevice, s->stream));
    return QSIM_OK;
}

int qsim_get_state(qsim_state *s, double *out) {
    GROUP_ALL(s, qsim_get_state(m_, out));  // collective: every member writes the same bytes
    if (s && s->capturing) {
        set_error("qsim_get_state: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (!s || !out) return QSIM_EINVAL;
    if (s->n > 30) {
        set_error("qsim_get_state is for N <= 30");
        return QSIM_EINVAL;
    }
    cudaSetDevice(s->dev);
    const size_t dim = (size_t)1 << s->n;
    void *d_full = nullptr;
    int *d_inv = nullptr;
    CU(cudaMalloc(&d_full, dim * 16));
    RC(upload_inv(s, &d_inv));
    CU(cudaMemsetAsync(d_full, 0, dim * 16, s->stream));
    for (auto &sh : s->shards) {
        if (s->enc == QSIM_ENC_FP64)
            launch_to_logical_e(sh.amps, 1ull << s->nl, shard_base(s, sh), d_inv, s->n, d_full, s->stream);
        else
            launch_to_logical_a(sh.amps, 1ull << s->nl, shard_base(s, sh), d_inv, s->n, s->atab, d_full, s->stream);
        s->st.kernels++;
    }
    if (s->transport == QSIM_TRANSPORT_NCCL)
        NC(ncclAllReduce(d_full, d_full, 2 * dim, ncclFloat64, ncclSum, s->comm, s->stream));
    CU(cudaMemcpyAsync(out, d_full, dim * 16, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    cudaFree(d_full);
    cudaFree(d_inv);
    return QSIM_OK;
}

int qsim_set_state(qsim_state *s, const double *amps) {
    GROUP_ALL(s, qsim_set_state(m_, amps));
    if (s && s->capturing) {
        set_error("qsim_set_state: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (!s || !amps) return QSIM_EINVAL;
    if (s->enc != QSIM_ENC_FP64) {
        set_error("qsim_set_state: E only (use qsim_set_codes for A)");
        return QSIM_EUNSUPPORTED;
    }
    if (s->n > 30) {
        set_error("qsim_set_state is for N <= 30");
        return QSIM_EINVAL;
    }
    cudaSetDevice(s->dev);
    const size_t dim = (size_t)1 << s->n;
    void *d_full = nullptr;
    int *d_inv = nullptr;
    CU(cudaMalloc(&d_full, dim * 16));
    RC(upload_inv(s, &d_inv));
    CU(cudaMemcpyAsync(d_full, amps, dim * 16, cudaMemcpyHostToDevice, s->stream));
    for (auto &sh : s->shards) {
        launch_from_logical_e(sh.amps, 1ull << s->nl, shard_base(s, sh), d_inv, s->n, d_full, s->stream);
        s->st.kernels++;
    }
    CU(cudaStreamSynchronize(s->stream));
    cudaFree(d_full);
    cudaFree(d_inv);
    return QSIM_OK;
}

// (r0, r1) of the current A tables back to the host after dense gates built them on the device
static int sync_bounds(qsim_state *s) {
    if (!s->r_stale) return QSIM_OK;
    double rr[2];
    CU(cudaMemcpyAsync(rr, reinterpret_cast<const char *>(s->atab->d[s->atab->cur]) + offsetof(ATabData, r0),
                       sizeof(rr), cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    s->r0 = rr[0];
    s->r1 = rr[1];
    s->r_stale = false;
    return QSIM_OK;
}

int qsim_get_bounds(qsim_state *s, double *r0, double *r1) {
    std::vector<double> g_sc(s && s->group ? 2 * s->P : 0);
    GROUP_ALL(s, qsim_get_bounds(m_, r_ == 0 ? r0 : &g_sc[2 * r_], r_ == 0 ? r1 : &g_sc[2 * r_ + 1]));
    if (!s || !r0 || !r1) return QSIM_EINVAL;
    if (s->capturing) {
        set_error("qsim_get_bounds: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (s->enc != QSIM_ENC_ADAPTIVE2) {
        set_error("qsim_get_bounds: A only");
        return QSIM_EUNSUPPORTED;
    }
    cudaSetDevice(s->dev);
    RC(sync_bounds(s));
    *r0 = s->r0;
    *r1 = s->r1;
    return QSIM_OK;
}

int qsim_get_codes(qsim_state *s, int8_t *codes, double *r0, double *r1) {
    std::vector<double> g_sc(s && s->group ? 2 * s->P : 0);
    GROUP_ALL(s, qsim_get_codes(m_, codes, r_ == 0 ? r0 : &g_sc[2 * r_], r_ == 0 ? r1 : &g_sc[2 * r_ + 1]));
    if (s && s->capturing) {
        set_error("qsim_get_codes: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (!s || !codes) return QSIM_EINVAL;
    if (s->enc != QSIM_ENC_ADAPTIVE2) {
        set_error("qsim_get_codes: A only");
        return QSIM_EUNSUPPORTED;
    }
    if (s->n > 32) {
        set_error("qsim_get_codes is for N <= 32");
        return QSIM_EINVAL;
    }
    cudaSetDevice(s->dev);
    const size_t dim = (size_t)1 << s->n;
    void *d_full = nullptr;
    int *d_inv = nullptr;
    CU(cudaMalloc(&d_full, dim * 2));
    RC(upload_inv(s, &d_inv));
    for (auto &sh : s->shards) {
        launch_codes_to_logical_a(sh.amps, 1ull << s->nl, shard_base(s, sh), d_inv, s->n, d_full, s->stream);
        s->st.kernels++;
    }
    CU(cudaMemcpyAsync(codes, d_full, dim * 2, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    cudaFree(d_full);
    cudaFree(d_inv);
    RC(sync_bounds(s));
    if (r0) *r0 = s->r0;
    if (r1) *r1 = s->r1;
    return QSIM_OK;
}

int qsim_set_codes(qsim_state *s, const int8_t *codes, double r0, double r1) {
    GROUP_ALL(s, qsim_set_codes(m_, codes, r0, r1));
    if (s && s->capturing) {
        set_error("qsim_set_codes: not allowed while a graph capture is open");
        return QSIM_EINVAL;
    }
    if (!s || !codes) return QSIM_EINVAL;
    if (s->enc != QSIM_ENC_ADAPTIVE2) {
        set_error("qsim_set_codes: A only");
        return QSIM_EUNSUPPORTED;
    }
    if (s->n > 32 || !(r0 > 0.0) || !(r1 >= r0) || !(r1 < 1.0)) {
        set_error("qsim_set_codes: N <= 32 and 0 < r0 <= r1 < 1 required");
        return QSIM_EINVAL;
    }
    cudaSetDevice(s->dev);
    const size_t dim = (size_t)1 << s->n;
    void *d_full = nullptr;
    int *d_inv = nullptr;
    CU(cudaMalloc(&d_full, dim * 2));
    RC(upload_inv(s, &d_inv));
    CU(cudaMemcpyAsync(d_full, codes, dim * 2, cudaMemcpyHostToDevice, s->stream));
    for (auto &sh : s->shards) {
        launch_codes_from_logical_a(sh.amps, 1ull << s->nl, shard_base(s, sh), d_inv, s->n, d_full, s->stream);
        s->st.kernels++;
    }
    s->r0 = r0;
    s->r1 = r1;
    s->r_stale = false;
    RC(atables_set(s->atab, r0, r1, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    cudaFree(d_full);
    cudaFree(d_inv);
    return QSIM_OK;
}

}  // extern "C"

// ============================================================================
// A variant executor (a8, a9)
// ============================================================================
namespace qsim {

// The diagonal gates that follow a dense gate, applied as its apply kernel
// stores the codes (AEpilogue; the same integer b1 steps as diag_run_a, so
// the result is bit-identical to the separate sweep): run[i..j).
struct AEpiRun {
    const std::vector<PlanOp> *run = nullptr;
    const std::vector<const double *> *us = nullptr;
    size_t i = 0, j = 0;
};

// The epilogue of the dense gate o for shard sh; false when the run does not fit.
// A unit holds 16 codes: local bits 0..3 (target < 4) or bits 0..2 and the
// target (code index bit 3); a diagonal gate's step for a code depends on its
// target and control bits -- all inside the unit (a per-code constant), all
// outside (one value per unit) or both (a per-unit condition on a per-code pattern).
static bool build_epi(const qsim_state *s, const Shard &sh, const PlanOp &o, const AEpiRun &r, AEpilogue &e) {
    e = AEpilogue{};
    const int ib[4] = {0, 1, 2, o.l < 4 ? 3 : o.l};
    uint64_t imask = 0;
    for (int q = 0; q < 4; ++q) imask |= 1ull << ib[q];
    auto jbit = [&](int j, int bit) {
        for (int q = 0; q < 4; ++q)
            if (ib[q] == bit) return (j >> q) & 1;
        return 0;
    };
    for (size_t k = r.i; k < r.j; ++k) {
        const PlanOp &g = (*r.run)[k];
        const double *u = (*r.us)[k];
        if (!global_ctrls_ok(s, sh, g)) continue;
        uint64_t cm = 0;
        for (int c = 0; c < g.nctrl; ++c)
            if (g.ctrl[c] < s->nl) cm |= 1ull << g.ctrl[c];
        int k0 = a_phase_steps(u[0], u[1]), k1 = a_phase_steps(u[6], u[7]);
        int t = g.l;
        if (g.l >= s->nl) {
            t = -1;
            k0 = k1 = rank_bit(s, sh, g.l) ? k1 : k0;
        }
        const uint64_t ci = cm & imask, ce = cm & ~imask;
        const bool ti = t >= 0 && ((imask >> t) & 1ull);
        auto step = [&](int j, int sel) {  // the gate's step for code j (sel: an outside target bit)
            for (int q = 0; q < 4; ++q)
                if (((ci >> ib[q]) & 1ull) && !((j >> q) & 1)) return 0;
            return (ti ? jbit(j, t) : sel) ? k1 : k0;
        };
        if (!ce && (t < 0 || ti)) {
            for (int j = 0; j < 16; ++j) e.base[j] = (int8_t)(e.base[j] + step(j, 0));
        } else if (!ci && !ti) {
            if (e.nscalar == A_EPI_MAX_SCALAR) return false;
            AEpiScalar &x = e.s[e.nscalar++];
            x.cext = ce;
            x.t = (int16_t)t;
            x.k0 = (int8_t)k0;
            x.k1 = (int8_t)k1;
        } else {
            if (e.nmixed == A_EPI_MAX_MIXED) return false;
            AEpiMixed &m = e.m[e.nmixed++];
            m.cext = ce;
            m.t = (int16_t)(ti ? -1 : t);
            for (int sel = 0; sel < 2; ++sel)
                for (int j = 0; j < 16; ++j) m.pat[sel][j] = (int8_t)step(j, sel);
        }
    }
    return true;
}
static void set_epi(const qsim_state *s, const Shard &sh, const PlanOp &o, const AEpiRun &r, AGateParams &p) {
    if (r.i >= r.j) return;
    build_epi(s, sh, o, r, p.epi);  // fits: checked on every shard by run_gates_a
    p.has_epi = 1;
}

// Exact global bounds of the post-gate magnitudes (reading R-A4), then the
// decode-apply-encode sweep with those bounds.
// the exact policy's two phases (reading R-A4) from the shards' codes; aout: the
// out-of-place target (lazy policy) or in place
static int dense_gate_a_exact(qsim_state *s, const PlanOp &o, const double *u, bool out_of_place,
                              const AEpiRun &r) {
    // phase 1 on every shard: (min, -max) of the post-gate |z|^2 merged on the
    // device; across ranks one ncclAllReduce(min); the next tables are built
    // on the device from the result -- no host round trip per gate
    bool first = true;
    for (auto &sh : s->shards) {
        AGateParams p{};
        fill_agate(p, s, sh, o, u);
        prof_begin(s);
        launch_bounds_a(p, s->atab, s->d_partials, s->d_acc, first, s->stream);
        prof_end(s, QSIM_K_A_BOUNDS, std::ldexp((double)s->amp_bytes, s->nl));
        first = false;
        s->st.kernels += 2;
        s->st.hbm_bytes += std::ldexp((double)s->amp_bytes, s->nl);
    }
    if (s->transport == QSIM_TRANSPORT_NCCL)
        NC(ncclAllReduce(s->d_acc, s->d_acc, 2, ncclFloat64, ncclMin, s->comm, s->stream));
    launch_tables_next(s->d_acc, s->atab, s->stream);
    s->st.kernels++;
    if (getenv("QSIM_ABND_DEBUG")) {
        cudaStreamSynchronize(s->stream);
        a_bounds_debug_print();
    }
    for (auto &sh : s->shards) {
        AGateParams p{};
        fill_agate(p, s, sh, o, u);
        set_epi(s, sh, o, r, p);
        if (out_of_place) p.aout = sh.amps2;
        prof_begin(s);
        if (s->a_policy == QSIM_A_POLICY_FP32)
            launch_apply_a_fp32(p, s->atab, s->stream);
        else
            launch_apply_a(p, s->atab, s->stream);
        prof_end(s, QSIM_K_A_APPLY, std::ldexp(2.0 * (double)s->amp_bytes, s->nl));
        s->st.kernels++;
        s->st.hbm_bytes += std::ldexp(2.0 * (double)s->amp_bytes, s->nl);
    }
    s->r_stale = true;  // (r0, r1) now live in the device tables only
    RC(atables_commit_next(s->atab, s->stream));
    s->st.a_rescales++;
    CU(cudaGetLastError());
    return QSIM_OK;
}

// Lazy policy (reading R-A25): one out-of-place pass with the kept tables,
// which also certifies that every output stayed within one step of (r0, r1);
// if one left, the exact policy runs from the (intact) input codes.  Then the
// two code buffers swap.
static int dense_gate_a_lazy(qsim_state *s, const PlanOp &o, const double *u, const AEpiRun &r) {
    for (auto &sh : s->shards)
        if (!sh.amps2) {
            if (cudaMalloc(&sh.amps2, s->alloc_amps * s->amp_bytes) != cudaSuccess) {
                cudaGetLastError();
                set_error("lazy A policy: the second code buffer (" + std::to_string(s->alloc_amps * s->amp_bytes) +
                          " B per shard) does not fit");
                return QSIM_ENOMEM;
            }
            CU(cudaMemsetAsync(sh.amps2, 0, s->alloc_amps * s->amp_bytes, s->stream));
        }
    if (!s->d_oor) CU(cudaMalloc(&s->d_oor, sizeof(int32_t)));
    RC(sync_bounds(s));
    bool rescale = !(s->r1 > s->r0);  // degenerate kept bounds: d = 0, any other magnitude leaves them
    if (!rescale) {
        CU(cudaMemsetAsync(s->d_oor, 0, sizeof(int32_t), s->stream));
        for (auto &sh : s->shards) {
            AGateParams p{};
            fill_agate(p, s, sh, o, u);
            set_epi(s, sh, o, r, p);
            p.aout = sh.amps2;
            p.oor = s->d_oor;
            prof_begin(s);
            launch_apply_a_lazy(p, s->atab, s->stream);
            prof_end(s, QSIM_K_A_APPLY, std::ldexp(2.0 * (double)s->amp_bytes, s->nl));
            s->st.kernels++;
            s->st.hbm_bytes += std::ldexp(2.0 * (double)s->amp_bytes, s->nl);
        }
        int32_t h = 0;
        if (s->transport == QSIM_TRANSPORT_NCCL)
            NC(ncclAllReduce(s->d_oor, s->d_oor, 1, ncclInt32, ncclMax, s->comm, s->stream));
        CU(cudaMemcpyAsync(&h, s->d_oor, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
        CU(cudaStreamSynchronize(s->stream));
        rescale = h != 0;
    }
    if (rescale) RC(dense_gate_a_exact(s, o, u, true, r));
    for (auto &sh : s->shards) std::swap(sh.amps, sh.amps2);
    return QSIM_OK;
}

static int dense_gate_a(qsim_state *s, const PlanOp &o, const double *u, const AEpiRun &r = AEpiRun{}) {
    s->st.a_dense++;
    if (s->a_policy == QSIM_A_POLICY_LAZY) return dense_gate_a_lazy(s, o, u, r);
    return dense_gate_a_exact(s, o, u, false, r);
}
static int diag_run_a(qsim_state *s, const std::vector<PlanOp> &run, const std::vector<const double *> &us, size_t i,
                      size_t j) {
    for (auto &sh : s->shards) {
        ADiagRunParams p{};
        p.a = sh.amps;
        p.n = s->alloc_amps;
        double bytes = 0.0;
        for (size_t k = i; k < j; ++k) {
            const PlanOp &o = run[k];
            const double *u = us[k];
            if (!global_ctrls_ok(s, sh, o)) continue;
            ADiagRunGate g{};
            for (int c = 0; c < o.nctrl; ++c)
                if (o.ctrl[c] < s->nl) g.cmask |= 1u << o.ctrl[c];
            const int k0 = a_phase_steps(u[0], u[1]), k1 = a_phase_steps(u[6], u[7]);
            if (o.l >= s->nl) {
                g.t = -1;
                g.k0 = (int8_t)(rank_bit(s, sh, o.l) ? k1 : k0);
                g.k1 = g.k0;
            } else {
                g.t = (int16_t)o.l;
                g.k0 = (int8_t)k0;
                g.k1 = (int8_t)k1;
            }
            p.g[p.ngates++] = g;
            bytes += gate_bytes_alone(s, sh, o, u);
        }
        if (!p.ngates) continue;
        prof_begin(s);
        launch_diag_run_a(p, s->stream);
        prof_end(s, QSIM_K_A_FAST, bytes);
        s->st.kernels++;
        s->st.hbm_bytes += std::ldexp(2.0 * (double)s->amp_bytes, s->nl);
    }
    CU(cudaGetLastError());
    return QSIM_OK;
}

static int run_gates_a(qsim_state *s, const std::vector<PlanOp> &run, const std::vector<const double *> &us) {
    static const bool fuse_diag = getenv("QSIM_A_NO_DIAG_RUN") == nullptr;
    const bool epilogue = getenv("QSIM_A_NO_EPILOGUE") == nullptr;  // read per call: tests compare both
    for (size_t i = 0; i < run.size(); ++i) {
        const PlanOp &o = run[i];
        const double *u = us[i];
        if (o.cls == CLS_DENSE) {
            // the diagonal gates that follow fold into this gate's apply kernel
            AEpiRun r{&run, &us, i + 1, i + 1};
            if (epilogue) {
                AEpilogue e;
                for (;;) {
                    if (r.j >= run.size() || run[r.j].cls != CLS_DIAG) break;
                    AEpiRun t = r;
                    ++t.j;
                    bool fits = true;
                    for (auto &sh : s->shards) fits = fits && build_epi(s, sh, o, t, e);
                    if (!fits) break;
                    r = t;
                }
            }
            RC(dense_gate_a(s, o, u, r));
            i = r.j - 1;
            continue;
        }
        if (fuse_diag && o.cls == CLS_DIAG && s->nl <= 32) {
            size_t j = i;
            while (j < run.size() && run[j].cls == CLS_DIAG && (int)(j - i) < A_MAX_DIAG_RUN) ++j;
            if (j - i >= 2) {
                RC(diag_run_a(s, run, us, i, j));
                i = j - 1;
                continue;
            }
        }
        // perm (anti-diagonal) and phase (diagonal) gates move or rotate codes; bounds unchanged
        for (auto &sh : s->shards) {
            if (!global_ctrls_ok(s, sh, o)) continue;
            AGateParams p{};
            fill_agate(p, s, sh, o, u);
            prof_begin(s);
            launch_fast_a(p, s->atab, s->stream);
            prof_end(s, QSIM_K_A_FAST, gate_bytes_alone(s, sh, o, u));
            s->st.kernels++;
            s->st.hbm_bytes += gate_bytes_alone(s, sh, o, u);
        }
        CU(cudaGetLastError());
    }
    return QSIM_OK;
}

int measure_collapse_a(qsim_state *s, int b, int out, double f) {
    (void)f;
    // Collapse = a diagonal projector followed by rescaling: decode, zero the
    // other half, scale by f, re-encode with exact new bounds (two-phase).
    double mn = INFINITY, mx = -INFINITY;
    for (auto &sh : s->shards) {
        ACollapseParams p{};
        p.a = sh.amps;
        p.n = s->alloc_amps;
        p.shard_base = shard_base(s, sh);
        p.bit = b;
        p.keep = out;
        p.f = f;
        launch_collapse_bounds_a(p, s->atab, s->d_partials, s->d_out, s->stream);
        CU(cudaMemcpyAsync(s->h_out, s->d_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
        CU(cudaStreamSynchronize(s->stream));
        mn = std::min(mn, s->h_out[0]);
        mx = std::max(mx, -s->h_out[1]);
    }
    if (s->transport == QSIM_TRANSPORT_NCCL) {
        s->h_out[0] = mn;
        s->h_out[1] = -mx;
        CU(cudaMemcpyAsync(s->d_out, s->h_out, 2 * sizeof(double), cudaMemcpyHostToDevice, s->stream));
        NC(ncclAllReduce(s->d_out, s->d_out, 2, ncclFloat64, ncclMin, s->comm, s->stream));
        CU(cudaMemcpyAsync(s->h_out, s->d_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
        CU(cudaStreamSynchronize(s->stream));
        mn = s->h_out[0];
        mx = -s->h_out[1];
    }
    double r0n = 0.5, r1n = 0.5;
    if (mn <= mx) {
        r0n = std::sqrt(mn);
        r1n = std::sqrt(mx);
    }
    RC(atables_set_next(s->atab, r0n, r1n, s->stream));
    for (auto &sh : s->shards) {
        ACollapseParams p{};
        p.a = sh.amps;
        p.n = s->alloc_amps;
        p.shard_base = shard_base(s, sh);
        p.bit = b;
        p.keep = out;
        p.f = f;
        launch_collapse_apply_a(p, s->atab, s->stream);
    }
    s->r0 = r0n;
    s->r1 = r1n;
    s->r_stale = false;
    RC(atables_commit_next(s->atab, s->stream));
    return QSIM_OK;
}

void fill_agate(AGateParams &p, const qsim_state *s, const Shard &sh, const PlanOp &o, const double *u) {
    p.a = sh.amps;
    p.nl = s->nl;
    p.shard_base = shard_base(s, sh);
    p.t = o.l;
    p.cls = o.cls;
    p.cmask = full_cmask(o);
    std::memcpy(p.u, u, sizeof(p.u));
}

}  // namespace qsim
