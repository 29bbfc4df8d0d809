"""Auxiliary-variable amplitude evaluator on the GPU (qsim_aux_amplitudes,
PAPER.md §4.2, Eq. appa7) vs the oracle (oracle/aux_hs.py, same method step
by step), vs the state-vector oracle, and at full size (N = 36) vs the oracle
on sampled amplitudes.  Tolerance: the HS terms are not bounded by 1 (complex
x), so both sums carry rounding errors relative to 2^-P sum_s |term_s|, which
both sides report."""
import math

import numpy as np
import pytest

import oracle
import paper_1805_04708_b200 as q
import qsim_inputs as C
from oracle import aux_hs

pytestmark = pytest.mark.gpu
EPS = 2.0 ** -52


def _tol(ab, P):
    return 64 * EPS * (P + 8) * ab + 1e-15


def _hs_circuit(n, ngates, seed, kinds=8):
    rng = np.random.default_rng(seed)
    c = C.Circuit(n)
    for _ in range(ngates):
        qq = [int(v) for v in rng.permutation(n)[:2]]
        k = int(rng.integers(0, kinds))
        th = float(rng.uniform(0, 2 * math.pi))
        if k == 0:
            c.add("H", C.mat_H(), qq[0])
        elif k == 1:
            c.add("Rx", C.mat_Rx(th), qq[0])
        elif k == 2:
            c.add("Haar", C.mat_haar(rng), qq[0])
        elif k == 3:
            c.add("T", C.mat_T(), qq[0])
        elif k == 4:
            c.add("CNOT", C.mat_X(), qq[1], [qq[0]])
        elif k == 5:
            c.add("CPHASE", C.mat_U1(th), qq[1], [qq[0]])
        elif k == 6:
            c.add("CZ", C.mat_Z(), qq[1], [qq[0]])
        else:
            c.add("CY", C.mat_Y(), qq[1], [qq[0]])
    return c


@pytest.mark.parametrize("seed", range(5))
def test_gpu_hs_matches_oracles(seed):
    n = 8
    c = _hs_circuit(n, 18, seed)
    P = aux_hs.num_aux(c)
    assert q.qsim_aux_num_vars(n, c) == P
    idx = np.arange(1 << n)
    got, ab = q.qsim_aux_amplitudes(n, c, idx, return_abs_sum=True)
    ref, rab = aux_hs.amplitudes(n, c, idx, return_abs_sum=True)
    assert np.allclose(ab, rab, rtol=1e-12, atol=1e-15)
    assert np.all(np.abs(got - ref) <= _tol(ab, P))
    sv = oracle.e_simulate(n, c)
    assert np.all(np.abs(got - sv) <= _tol(ab, P))


def test_gpu_hs_qft_closed_form():
    n, x = 6, 0b100111
    c = C.Circuit(n)
    for qq in range(n):
        if (x >> qq) & 1:
            c.add("X", C.mat_X(), qq)
    c.extend(C.qft_register(n, n, swaps=False))
    got, ab = q.qsim_aux_amplitudes(n, c, np.arange(1 << n), return_abs_sum=True)
    P = n * (n - 1) // 2
    for y in range(1 << n):
        ry = int(format(y, f"0{n}b")[::-1], 2)
        ref = 2.0 ** (-n / 2) * np.exp(2j * math.pi * ((x * y) % (1 << n)) / (1 << n))
        assert abs(got[ry] - ref) <= _tol(ab[ry], P)


def test_full_size_n36_sampled_vs_oracle():
    """Config-3 structure at N = 36 (H wall, layers of U(2) on every qubit) with
    16 entangling gates kept (P = 16..24): the 2^36-amplitude state is never
    formed; 64 sampled amplitudes vs the oracle."""
    n = 36
    rng = np.random.default_rng(36)
    c = C.h_wall(n)
    for layer in range(3):
        for qq in range(n):
            c.add("U", C.mat_haar(rng), qq)
        for _ in range(5 if layer < 2 else 6):
            a, b = [int(v) for v in rng.permutation(n)[:2]]
            if rng.integers(0, 2):
                c.add("CNOT", C.mat_X(), b, [a])
            else:
                c.add("CPHASE", C.mat_U1(float(rng.uniform(0, 2 * math.pi))), b, [a])
    P = aux_hs.num_aux(c)
    assert 16 <= P <= 24
    idx = rng.integers(0, 1 << n, size=64, dtype=np.uint64)
    got, ab = q.qsim_aux_amplitudes(n, c, idx, return_abs_sum=True)
    ref, rab = aux_hs.amplitudes(n, c, idx.astype(np.int64), return_abs_sum=True)
    assert np.all(np.abs(got - ref) <= _tol(ab, P))
    # |amplitude|^2 of a random 36-qubit state is ~2^-36: the check is not vacuous
    assert np.max(np.abs(ref)) > 2.0 ** -20


def test_product_state_p0_and_edge_cases():
    n = 20
    c = C.layered(n, 2, seed=8, entangle=False)
    assert q.qsim_aux_num_vars(n, c) == 0
    idx = np.array([0, 1, (1 << n) - 1, 12345], dtype=np.uint64)
    v = [np.array([1, 0], dtype=np.complex128) for _ in range(n)]
    for g in range(len(c)):
        _, _, t, _, _, u = c.gate(g)
        v[t] = u @ v[t]
    ref = np.array([np.prod([v[j][(int(y) >> j) & 1] for j in range(n)]) for y in idx])  # Eq. appa2
    assert np.max(np.abs(q.qsim_aux_amplitudes(n, c, idx) - ref)) <= 1e-14
    assert len(q.qsim_aux_amplitudes(n, c, np.array([], dtype=np.uint64))) == 0
    with pytest.raises(q.QsimError) as e:
        q.qsim_aux_amplitudes(n, c, np.array([1 << n], dtype=np.uint64))
    assert e.value.code == q.QSIM_EINVAL
    t = C.Circuit(3)
    t.add("TOF", C.mat_X(), 2, [0, 1])
    with pytest.raises(q.QsimError) as e:
        q.qsim_aux_amplitudes(3, t, [0])
    assert e.value.code == q.QSIM_EUNSUPPORTED
