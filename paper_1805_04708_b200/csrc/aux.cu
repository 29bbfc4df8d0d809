// aux.cu -- auxiliary-variable amplitude evaluator (SURVEY.md §8(f) NEXT-3,
// PAPER.md §4.2).
//
// <y|psi> = 2^{-P} sum_{s in {+-1}^P} prod_j <y_j| W_j(s) |0>_j      (Eq. appa7)
//
// Host: every CNOT_{ct} becomes H_t U_{ct}(pi) H_t; each
// controlled phase U_{ct}(a) (Eq. appa4) gets an auxiliary variable s_p and
// contributes diag(e^{i(x s - a/4)}, e^{-i(x s - a/4)}) to qubits c and t,
// cos 2x = e^{ia/2} (Eqs. appa5-appa6).  For every qubit j the 2-vectors
// W_j(s)|0> depend only on the variables S_j that touch j, so the host
// tabulates them for all 2^|S_j| values (a qubit with S_j empty is a constant
// factor).  Device: one thread per term s (grid-stride), the product over the
// qubits with variables for a tile of amplitudes, a fixed-order two-level sum
// (deterministic), and alongside it 2^{-P} sum_s |term| (the scale of the
// terms that cancel -- the sum's rounding error is relative to it).
// Controlled diagonal / anti-diagonal gates follow reading R-B9; two controls
// or a controlled dense 2x2 are outside the method (QSIM_EUNSUPPORTED).
#include <cuda_runtime.h>

#include <cmath>
#include <complex>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

namespace qsim {

using cplx = std::complex<double>;

namespace {

struct AuxOp {
    int kind;  // 0: 2x2 on qubit q; 1: auxiliary variable p on qubit q
    int q, p;
    cplx m[4];
};

struct AuxPlan {
    int n = 0, P = 0;
    std::vector<double> a, xr, xi;       // per variable: a_p, x_p
    std::vector<std::vector<AuxOp>> chain;  // per qubit, circuit order
    std::vector<std::vector<int>> S;        // per qubit: variables, in order of appearance
};

void add_u(AuxPlan &pl, int q, cplx u00, cplx u01, cplx u10, cplx u11) {
    AuxOp o{0, q, -1, {u00, u01, u10, u11}};
    pl.chain[q].push_back(o);
}
void add_cp(AuxPlan &pl, int c, int t, double a) {
    const int p = pl.P++;
    const cplx x = std::acos(std::exp(cplx(0.0, 0.5 * a))) / 2.0;  // cos 2x = e^{ia/2}
    pl.a.push_back(a);
    pl.xr.push_back(x.real());
    pl.xi.push_back(x.imag());
    for (int q : {c, t}) {
        AuxOp o{1, q, p, {}};
        pl.chain[q].push_back(o);
        pl.S[q].push_back(p);
    }
}

int build_plan(int n, const qsim_gate *gates, size_t ngates, AuxPlan &pl) {
    pl.n = n;
    pl.chain.assign(n, {});
    pl.S.assign(n, {});
    const double r2 = 1.0 / std::sqrt(2.0);
    for (size_t g = 0; g < ngates; ++g) {
        const qsim_gate &x = gates[g];
        if (x.kind != QSIM_GATE_U) {
            set_error("aux: SWAP records are outside the auxiliary-variable method");
            return QSIM_EUNSUPPORTED;
        }
        const cplx u00(x.u[0], x.u[1]), u01(x.u[2], x.u[3]), u10(x.u[4], x.u[5]), u11(x.u[6], x.u[7]);
        if (x.ncontrols == 0) {
            add_u(pl, x.target, u00, u01, u10, u11);
            continue;
        }
        if (x.ncontrols > 1) {
            set_error("aux: gates with two controls are outside the method (PAPER.md:470-472)");
            return QSIM_EUNSUPPORTED;
        }
        const int c = x.controls[0], t = x.target;
        const bool diag = u01 == 0.0 && u10 == 0.0, anti = u00 == 0.0 && u11 == 0.0;
        if (!diag && !anti) {
            set_error("aux: a controlled dense 2x2 is outside the method (PAPER.md:470-472)");
            return QSIM_EUNSUPPORTED;
        }
        // controlled diag(d0, d1) = diag(1, d0) on c, then U_ct(arg(d1 / d0))   (reading R-B9)
        const cplx d0 = diag ? u00 : u10, d1 = diag ? u11 : u01;
        add_u(pl, c, 1.0, 0.0, 0.0, d0);
        if (d1 != d0) add_cp(pl, c, t, std::arg(d1 / d0));  // U_ct(0) = I: no variable (one per CNOT)
        if (anti) {  // U = X diag(u10, u01): then CNOT_ct = H_t U_ct(pi) H_t
            add_u(pl, t, r2, r2, r2, -r2);
            add_cp(pl, c, t, M_PI);
            add_u(pl, t, r2, r2, r2, -r2);
        }
    }
    return QSIM_OK;
}

constexpr int AUX_MT = 4;         // amplitudes per block tile
constexpr int AUX_THREADS = 256;
constexpr int AUX_MAX_ACT = 128;  // qubits with variables (<= 2P)
constexpr int AUX_MAX_BITS = 1024;

struct AuxDev {
    int P, nact, m, nblocks;
    uint64_t nterms;
    int act_q[AUX_MAX_ACT];
    int act_nb[AUX_MAX_ACT];
    int act_boff[AUX_MAX_ACT];
    int64_t act_toff[AUX_MAX_ACT];
    int16_t bits[AUX_MAX_BITS];
};

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

__global__ void __launch_bounds__(AUX_THREADS) k_aux_terms(const __grid_constant__ AuxDev d,
                                                           const double2 *__restrict__ tab,
                                                           const uint64_t *__restrict__ yy, double *partial) {
    const int m0 = blockIdx.y * AUX_MT;
    uint64_t y[AUX_MT];
#pragma unroll
    for (int k = 0; k < AUX_MT; ++k) y[k] = (m0 + k < d.m) ? yy[m0 + k] : 0ull;
    double sr[AUX_MT], si[AUX_MT], sa[AUX_MT];
#pragma unroll
    for (int k = 0; k < AUX_MT; ++k) sr[k] = si[k] = sa[k] = 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * AUX_THREADS;
    for (uint64_t t = (uint64_t)blockIdx.x * AUX_THREADS + threadIdx.x; t < d.nterms; t += stride) {
        double2 pr[AUX_MT];
#pragma unroll
        for (int k = 0; k < AUX_MT; ++k) pr[k] = make_double2(1.0, 0.0);
        for (int a = 0; a < d.nact; ++a) {
            uint32_t idx = 0;
            const int nb = d.act_nb[a], bo = d.act_boff[a];
            for (int b = 0; b < nb; ++b) idx |= (uint32_t)((t >> d.bits[bo + b]) & 1ull) << b;
            const double2 *T = tab + d.act_toff[a] + 2 * (int64_t)idx;
            const int q = d.act_q[a];
#pragma unroll
            for (int k = 0; k < AUX_MT; ++k) pr[k] = zmul(pr[k], __ldg(T + ((y[k] >> q) & 1ull)));
        }
#pragma unroll
        for (int k = 0; k < AUX_MT; ++k) {
            sr[k] += pr[k].x;
            si[k] += pr[k].y;
            sa[k] += hypot(pr[k].x, pr[k].y);
        }
    }
    // fixed-order block reduction: warp shuffles, then warp 0
    __shared__ double sm[AUX_THREADS / 32][3 * AUX_MT];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < AUX_MT; ++k)
        for (int o = 16; o > 0; o >>= 1) {
            sr[k] += __shfl_xor_sync(0xffffffffu, sr[k], o);
            si[k] += __shfl_xor_sync(0xffffffffu, si[k], o);
            sa[k] += __shfl_xor_sync(0xffffffffu, sa[k], o);
        }
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < AUX_MT; ++k) {
            sm[w][3 * k] = sr[k];
            sm[w][3 * k + 1] = si[k];
            sm[w][3 * k + 2] = sa[k];
        }
    __syncthreads();
    if (threadIdx.x < 3 * AUX_MT) {
        double acc = 0.0;
        for (int ww = 0; ww < AUX_THREADS / 32; ++ww) acc += sm[ww][threadIdx.x];
        // partial[(m * 3 + c) * nblocks + block]
        const int k = threadIdx.x / 3, c = threadIdx.x % 3;
        if (m0 + k < d.m) partial[((int64_t)(m0 + k) * 3 + c) * d.nblocks + blockIdx.x] = acc;
    }
}

__global__ void k_aux_final(const double *partial, int nblocks, int m, double *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // (amplitude, component)
    if (i >= 3 * m) return;
    double acc = 0.0;
    for (int b = 0; b < nblocks; ++b) acc += partial[(int64_t)i * nblocks + b];
    out[i] = acc;
}

}  // namespace

int aux_num_vars(int n, const qsim_gate *gates, size_t ngates, int *P) {
    AuxPlan pl;
    const int rc = build_plan(n, gates, ngates, pl);
    if (rc) return rc;
    *P = pl.P;
    return QSIM_OK;
}

int aux_amplitudes(int n, const qsim_gate *gates, size_t ngates, const uint64_t *idx, size_t m, double *out,
                   double *abs_sum, int max_vars) {
    AuxPlan pl;
    int rc = build_plan(n, gates, ngates, pl);
    if (rc) return rc;
    if (pl.P > max_vars) {
        set_error("aux: " + std::to_string(pl.P) + " auxiliary variables (2^P terms) exceed the limit " +
                  std::to_string(max_vars));
        return QSIM_EUNSUPPORTED;
    }
    // per-qubit tables W_j(s)|0> for every value of the variables in S_j
    std::vector<double2> tab;
    AuxDev d{};
    d.P = pl.P;
    d.m = (int)m;
    d.nterms = 1ull << pl.P;
    std::vector<cplx> cst(2 * (size_t)n, cplx(1.0, 0.0));  // W_j|0> of qubits without variables
    int nbits = 0;
    for (int j = 0; j < n; ++j) {
        const int nb = (int)pl.S[j].size();
        if (nb > 20) {
            set_error("aux: qubit " + std::to_string(j) + " carries " + std::to_string(nb) +
                      " auxiliary variables (table 2^nb > 2^20)");
            return QSIM_EUNSUPPORTED;
        }
        if (nb > 0 && (d.nact >= AUX_MAX_ACT || nbits + nb > AUX_MAX_BITS)) {
            set_error("aux: too many qubits with auxiliary variables");
            return QSIM_EUNSUPPORTED;
        }
        const size_t nval = (size_t)1 << nb;
        const size_t off = tab.size() / 2;
        for (size_t v = 0; v < nval; ++v) {
            cplx a0 = 1.0, a1 = 0.0;
            int k = 0;
            for (const AuxOp &o : pl.chain[j]) {
                if (o.kind == 0) {
                    const cplx b0 = o.m[0] * a0 + o.m[1] * a1, b1 = o.m[2] * a0 + o.m[3] * a1;
                    a0 = b0;
                    a1 = b1;
                } else {
                    const double s = ((v >> k) & 1) ? -1.0 : 1.0;  // s_p = +1 for bit 0
                    const cplx th = cplx(pl.xr[o.p], pl.xi[o.p]) * s - pl.a[o.p] / 4.0;
                    a0 *= std::exp(cplx(0.0, 1.0) * th);
                    a1 *= std::exp(cplx(0.0, -1.0) * th);
                    ++k;
                }
            }
            if (nb == 0) {
                cst[2 * j] = a0;
                cst[2 * j + 1] = a1;
            } else {
                tab.push_back(make_double2(a0.real(), a0.imag()));
                tab.push_back(make_double2(a1.real(), a1.imag()));
            }
        }
        if (nb == 0) continue;
        d.act_q[d.nact] = j;
        d.act_nb[d.nact] = nb;
        d.act_boff[d.nact] = nbits;
        d.act_toff[d.nact] = (int64_t)off * 2;
        // variable index of table bit k: bit (p) of the term counter
        for (int k = 0; k < nb; ++k) d.bits[nbits + k] = (int16_t)pl.S[j][k];
        nbits += nb;
        d.nact++;
    }
    if (tab.empty()) tab.push_back(make_double2(0.0, 0.0));
    // device run
    int dev = 0, nsm = 148;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) {
        set_error("aux: no usable CUDA device");
        return QSIM_ECUDA;
    }
    const uint64_t want = (d.nterms + AUX_THREADS - 1) / AUX_THREADS;
    d.nblocks = (int)(want < (uint64_t)nsm * 8 ? want : (uint64_t)nsm * 8);
    const int mtiles = (int)((m + AUX_MT - 1) / AUX_MT);
    double2 *d_tab = nullptr;
    uint64_t *d_y = nullptr;
    double *d_part = nullptr, *d_out = nullptr;
    auto fail = [&](const char *what) {
        set_error(std::string("aux: ") + what + ": " + cudaGetErrorString(cudaGetLastError()));
        cudaFree(d_tab);
        cudaFree(d_y);
        cudaFree(d_part);
        cudaFree(d_out);
        return QSIM_ECUDA;
    };
    if (m == 0) return QSIM_OK;
    if (cudaMalloc(&d_tab, tab.size() * sizeof(double2)) || cudaMalloc(&d_y, m * 8) ||
        cudaMalloc(&d_part, (size_t)m * 3 * d.nblocks * 8) || cudaMalloc(&d_out, (size_t)m * 3 * 8))
        return fail("cudaMalloc");
    if (cudaMemcpy(d_tab, tab.data(), tab.size() * sizeof(double2), cudaMemcpyHostToDevice) ||
        cudaMemcpy(d_y, idx, m * 8, cudaMemcpyHostToDevice))
        return fail("cudaMemcpy");
    k_aux_terms<<<dim3(d.nblocks, mtiles), AUX_THREADS>>>(d, d_tab, d_y, d_part);
    k_aux_final<<<(int)((3 * m + 255) / 256), 256>>>(d_part, d.nblocks, (int)m, d_out);
    std::vector<double> h(3 * m);
    if (cudaMemcpy(h.data(), d_out, 3 * m * 8, cudaMemcpyDeviceToHost)) return fail("kernel");
    cudaFree(d_tab);
    cudaFree(d_y);
    cudaFree(d_part);
    cudaFree(d_out);
    const double scale = std::ldexp(1.0, -pl.P);
    for (size_t k = 0; k < m; ++k) {
        cplx c(1.0, 0.0);
        for (int j = 0; j < n; ++j)
            if (pl.S[j].empty()) c *= cst[2 * j + ((idx[k] >> j) & 1)];
        const cplx v = c * cplx(h[3 * k], h[3 * k + 1]) * scale;
        out[2 * k] = v.real();
        out[2 * k + 1] = v.imag();
        if (abs_sum) abs_sum[k] = std::abs(c) * h[3 * k + 2] * scale;
    }
    return QSIM_OK;
}

}  // namespace qsim
