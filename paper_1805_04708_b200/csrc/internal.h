// internal.h -- shared declarations of the qsim library (not part of the C-ABI).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/qsim.h"

namespace qsim {

// ---- error handling --------------------------------------------------------
void set_error(const std::string &msg);
struct Error {
    int code;
    std::string msg;
};

// ---- gate classes: the kernels specialise on these ---------
enum GateClass : int32_t { CLS_DENSE = 0, CLS_DIAG = 1, CLS_ANTI = 2, CLS_IDENT = 3 };
int32_t classify(const double u[8]);

// ---- planner (a2, a7) --------------------------------------------------------
struct PlanOp {
    int32_t type;  // QSIM_OP_EXCHANGE / QSIM_OP_GATE
    int32_t g, l, cls, nctrl;
    int32_t ctrl[2];
    int32_t gate_index;
};

// An all-to-all remap swaps at most this many global bits at once: each shard
// then trades 2^m - 1 blocks (RemapVals holds 7 partners); more global bits
// than this are remapped in several groups.
constexpr int kRemapMaxBits = 3;

struct Planner {
    int n = 0, nl = 0;
    std::vector<int> pos, inv;  // logical -> physical bit, physical -> logical
    bool relabel_global = true; // permutation gates on global bits only -> QSIM_OP_RELABEL
    bool remap = true;          // several global targets ahead -> one all-to-all (QSIM_OP_REMAP)
    void init(int n_, int nshards, const int *initial_map);
    // Appends the ops for gates[0..ngates) to `ops` and updates the map.
    // `lookahead` enables Belady victim selection over the remaining gates.
    void plan(const qsim_gate *gates, size_t ngates, std::vector<PlanOp> &ops, bool lookahead);
    int choose_victim(const qsim_gate *gates, size_t ngates, size_t cur, const int *avoid, int navoid, bool lookahead,
                      bool wide = false);
    void swap_bits(int a, int b);  // exchange the logical qubits at physical bits a and b
};

int validate_gates(int n, const qsim_gate *gates, size_t ngates, bool check_unitary);

// ---- auxiliary-variable evaluator (aux.cu) ----
int aux_num_vars(int n, const qsim_gate *gates, size_t ngates, int *P);
int aux_amplitudes(int n, const qsim_gate *gates, size_t ngates, const uint64_t *idx, size_t m, double *out,
                   double *abs_sum, int max_vars);

}  // namespace qsim

struct qsim_plan {
    qsim::Planner pl;
    std::vector<qsim::PlanOp> ops;
};
