"""The seeded input generator: its gate matrices against App. B as printed, and
the workload recipes of SURVEY.md §8(d) (gate counts, determinism)."""
import math

import numpy as np
import pytest

import qsim_inputs as C

s = 1 / math.sqrt(2)


def test_app_b_matrices_as_printed():
    """PAPER.md:1131-1294, each compared with the printed matrix."""
    assert np.allclose(C.mat_H(), [[s, s], [s, -s]], atol=0)
    assert np.array_equal(C.mat_X(), [[0, 1], [1, 0]])
    assert np.array_equal(C.mat_Y(), [[0, -1j], [1j, 0]])
    assert np.array_equal(C.mat_Z(), [[1, 0], [0, -1]])
    assert np.array_equal(C.mat_S(), [[1, 0], [0, 1j]])
    assert np.array_equal(C.mat_S(True), [[1, 0], [0, -1j]])
    assert np.allclose(C.mat_T(), [[1, 0], [0, (1 + 1j) * s]], atol=1e-16)
    assert np.allclose(C.mat_pX(+1), [[s, 1j * s], [1j * s, s]], atol=1e-16)
    assert np.allclose(C.mat_pY(-1), [[s, -s], [s, s]], atol=1e-16)
    assert np.allclose(C.mat_R(3), [[1, 0], [0, np.exp(2j * math.pi / 8)]], atol=1e-16)
    assert np.allclose(C.mat_R(-3), [[1, 0], [0, np.exp(-2j * math.pi / 8)]], atol=1e-16)
    assert np.allclose(C.mat_R(0), np.eye(2))  # reading A16
    # U3(theta, phi, lam) generalises U2 and U1
    assert np.allclose(C.mat_U3(math.pi / 2, 0.3, 0.7), C.mat_U2(0.3, 0.7), atol=1e-15)
    assert np.allclose(C.mat_U3(0, 0, 0.4), C.mat_U1(0.4), atol=1e-15)
    # reading A13: +X = Rx(-pi/2); Rz(t) = e^{-it/2} U1(t)
    assert np.allclose(C.mat_Rx(-math.pi / 2), C.mat_pX(+1), atol=1e-15)
    assert np.allclose(C.mat_Rz(0.9), np.exp(-0.45j) * C.mat_U1(0.9), atol=1e-15)


def test_haar_unitary_and_seeded():
    rng = np.random.default_rng(0)
    for _ in range(100):
        u = C.mat_haar(rng)
        assert np.allclose(u.conj().T @ u, np.eye(2), atol=1e-14)
    a = C.layered(10, 2, seed=3)
    b = C.layered(10, 2, seed=3)
    assert np.array_equal(a.u, b.u) and np.array_equal(a.target, b.target)


def test_config_gate_counts():
    """cfg2 930 gates (630 dense incl. 30 H, 300 CNOT), cfg3
    N + 10 (N + floor(N/2)), cfg4 39 + 10*(39+19) = 619, cfg5 35 H + 595
    CPHASE + 17 SWAP (+ X preparation)."""
    c2 = C.config(1)
    assert len(c2) == 930 and sum(c2.nctrl == 1) == 300
    for n in (33, 34, 35, 36):
        assert len(C.layered(n, 10, 3)) == n + 10 * (n + n // 2)
    c4 = C.config(3)
    assert len(c4) == 619
    c5, x = C.qft(35, seed=5)
    names = c5.names
    assert names.count("H") == 35 and names.count("CPHASE") == 595 and names.count("SWAP") == 17
    assert names.count("X") == bin(x).count("1")


@pytest.mark.parametrize("seed", range(3))
def test_cfg1_qubits_distinct(seed):
    c = C.config(0, seed=seed)
    for g in range(len(c)):
        _, kind, t, _, ctl, u = c.gate(g)
        assert t not in ctl and len(set(ctl)) == len(ctl)
        assert np.allclose(u.conj().T @ u, np.eye(2), atol=1e-14)
