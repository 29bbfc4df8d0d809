"""Pins of the auxiliary-variable (Hubbard-Stratonovich) oracle, oracle/aux_hs.py
(§4.2, Eqs. appa4-appa7).  None of these re-types the oracle's sum:
they compare it with the textbook 4x4 controlled phase (Eq. appa4), with the
state-vector oracle (itself pinned to Kronecker products), and with the QFT
closed form.  Tolerances scale with the size of the cancelling HS terms,
2^-P sum_s |prod_j ...|, returned by the oracle (the sum is not a convex
combination: |e^{i x s}| != 1 for complex x)."""
import math

import numpy as np
import pytest

import oracle
import qsim_inputs as C
from oracle import aux_hs

EPS = 2.0 ** -52


def _tol(absum, P):
    return 64 * EPS * (P + 8) * absum + 1e-15


def test_single_controlled_phase_is_eq_appa4():
    """HS sum of one U_01(a) on H|0>H|0> equals the 4x4 matrix of Eq. appa4."""
    for a in (0.3, math.pi, -2.0 * math.pi / 8, 2.5):
        c = C.Circuit(2)
        c.add("H", C.mat_H(), 0).add("H", C.mat_H(), 1).add("CP", C.mat_U1(a), 1, [0])
        got, ab = aux_hs.amplitudes(2, c, range(4), return_abs_sum=True)
        ref = np.array([1, 1, 1, np.exp(1j * a)]) / 2.0  # Eq. appa4 applied to |++>
        assert np.max(np.abs(got - ref)) <= 1e-14


def _hs_circuit(n, ngates, seed):
    rng = np.random.default_rng(seed)
    c = C.Circuit(n)
    for _ in range(ngates):
        q = [int(v) for v in rng.permutation(n)[:2]]
        k = int(rng.integers(0, 8))
        th = float(rng.uniform(0, 2 * math.pi))
        if k == 0:
            c.add("H", C.mat_H(), q[0])
        elif k == 1:
            c.add("Rx", C.mat_Rx(th), q[0])
        elif k == 2:
            c.add("Haar", C.mat_haar(rng), q[0])
        elif k == 3:
            c.add("T", C.mat_T(), q[0])
        elif k == 4:
            c.add("CNOT", C.mat_X(), q[1], [q[0]])
        elif k == 5:
            c.add("CPHASE", C.mat_U1(th), q[1], [q[0]])
        elif k == 6:
            c.add("CZ", C.mat_Z(), q[1], [q[0]])
        else:
            c.add("CY", C.mat_Y(), q[1], [q[0]])  # controlled anti-diagonal with phases
    return c


@pytest.mark.parametrize("seed", range(6))
def test_hs_sum_equals_state_vector_oracle(seed):
    n = 7
    c = _hs_circuit(n, 22, seed)
    P = aux_hs.num_aux(c)
    assert 1 <= P <= 20
    ref = oracle.e_simulate(n, c)
    got, ab = aux_hs.amplitudes(n, c, range(1 << n), return_abs_sum=True)
    assert np.all(np.abs(got - ref) <= _tol(ab, P))


def test_qft_without_swaps_closed_form():
    """QFT (reading A15) without the final swaps: a(rev(y)) = 2^{-N/2} e^{2 pi i x y / 2^N}."""
    n, x = 6, 0b101101
    c = C.Circuit(n)
    for q in range(n):
        if (x >> q) & 1:
            c.add("X", C.mat_X(), q)
    c.extend(C.qft_register(n, n, swaps=False))
    got, ab = aux_hs.amplitudes(n, c, range(1 << n), return_abs_sum=True)
    P = aux_hs.num_aux(c)
    assert P == n * (n - 1) // 2
    for y in range(1 << n):
        ry = int(format(y, f"0{n}b")[::-1], 2)
        ref = 2.0 ** (-n / 2) * np.exp(2j * math.pi * ((x * y) % (1 << n)) / (1 << n))
        assert abs(got[ry] - ref) <= _tol(ab[ry], P)


def test_no_entangling_gate_is_the_product_state():
    """P = 0: Eq. appa7 reduces to Eq. appa2, checked against the state-vector oracle."""
    n = 8
    c = C.layered(n, 2, seed=3, entangle=False)
    assert aux_hs.num_aux(c) == 0
    assert np.max(np.abs(aux_hs.amplitudes(n, c, range(1 << n)) - oracle.e_simulate(n, c))) <= 1e-14


def test_outside_the_method_is_rejected():
    c = C.Circuit(3)
    c.add("TOF", C.mat_X(), 2, [0, 1])
    with pytest.raises(ValueError):
        aux_hs.amplitudes(3, c, [0])
    c = C.Circuit(2)
    c.add("CH", C.mat_H(), 1, [0])
    with pytest.raises(ValueError):
        aux_hs.amplitudes(2, c, [0])


def test_library_counts_the_same_auxiliary_variables():
    """Host-only C-ABI planner (no GPU): P of qsim_aux_num_vars = the oracle's."""
    import paper_1805_04708_b200 as q

    for seed in range(4):
        c = _hs_circuit(9, 40, seed)
        assert q.qsim_aux_num_vars(9, c) == aux_hs.num_aux(c)
