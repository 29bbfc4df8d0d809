"""Pins for the E (exact fp64) oracle against what the paper and mathematics fix.

None of these re-derive the oracle's own loops: the dense check builds the
2^N x 2^N operator with numpy Kronecker products, the closed forms come from
the paper (H wall, GHZ, product state Eq. appa2, QFT), and the expectation
values are checked against a dense <psi|(1 - sigma)|psi>/2.
"""
import math
import os

import numpy as np
import pytest

import oracle
import qsim_inputs as C

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

I2 = np.eye(2, dtype=np.complex128)
P1 = np.array([[0, 0], [0, 1]], dtype=np.complex128)
SX = np.array([[0, 1], [1, 0]], dtype=np.complex128)
SY = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
SZ = np.array([[1, 0], [0, -1]], dtype=np.complex128)


def kron_ops(n, ops):
    """ops: dict qubit -> 2x2; qubit n-1 is the leftmost Kronecker factor
    (qubit 0 = rightmost bit)."""
    m = np.array([[1.0 + 0j]])
    for q in range(n - 1, -1, -1):
        m = np.kron(m, ops.get(q, I2))
    return m


def dense_gate(n, u, t, ctl):
    """I + P1(c1) x P1(c2) x (U - I)(t): the controlled-U operator."""
    ops = {t: np.asarray(u) - I2}
    for c in ctl:
        ops[c] = P1
    return np.eye(1 << n, dtype=np.complex128) + kron_ops(n, ops)


def dense_swap(n, q1, q2):
    m = np.zeros((1 << n, 1 << n), dtype=np.complex128)
    for i in range(1 << n):
        b1, b2 = (i >> q1) & 1, (i >> q2) & 1
        j = i & ~((1 << q1) | (1 << q2)) | (b1 << q2) | (b2 << q1)
        m[j, i] = 1
    return m


def dense_run(circ):
    n = circ.n
    v = np.zeros(1 << n, dtype=np.complex128)
    v[0] = 1
    for g in range(len(circ)):
        name, kind, t, t2, ctl, u = circ.gate(g)
        v = (dense_swap(n, t, t2) if kind == 1 else dense_gate(n, u, t, ctl)) @ v
    return v


@pytest.mark.parametrize("n,seed", [(2, 0), (3, 1), (5, 2), (6, 3), (8, 4)])
def test_dense_kronecker_random(n, seed):
    """BASELINE north_star / SPEC S:259: dense 2^N x 2^N products for N <= 8."""
    kinds = C.CFG1_KINDS if n >= 3 else tuple(k for k in C.CFG1_KINDS if k != "TOFFOLI")
    circ = C.random_circuit(n, 60, seed, kinds=kinds)
    circ.swap(0, n - 1)
    ref = dense_run(circ)
    got = oracle.e_simulate(n, circ)
    assert np.max(np.abs(got - ref)) <= 1e-12


@pytest.mark.parametrize("n", [4, 8])
def test_dense_kronecker_qft(n):
    circ, _ = C.qft(n, x=(0b1011 % (1 << n)))
    assert np.max(np.abs(oracle.e_simulate(n, circ) - dense_run(circ))) <= 1e-12


def test_gate_on_each_qubit_vs_kron():
    """Eq. NUM2 on every target j, with controls above and below j."""
    n = 5
    rng = np.random.default_rng(7)
    v0 = rng.standard_normal(32) + 1j * rng.standard_normal(32)
    for t in range(n):
        for ctl in [(), ((t + 1) % n,), ((t + 2) % n, (t + 4) % n)]:
            u = C.mat_haar(rng)
            got = oracle.e_apply(v0.copy(), n, u, t, ctl)
            assert np.max(np.abs(got - dense_gate(n, u, t, ctl) @ v0)) <= 1e-13


def _golden(name):
    rows = [l.split() for l in open(os.path.join(GOLDEN, name)) if l.strip() and not l.startswith("#")]
    return np.array(rows[0], dtype=float)


@pytest.mark.parametrize("n", [1, 5, 12, 16])
def test_h_wall_closed_form(n):
    """PAPER.md §5.1 (653-657): uniform amplitude 2^{-N/2}; Table 2 expectations."""
    a = oracle.e_simulate(n, C.h_wall(n))
    assert np.max(np.abs(a - 2.0 ** (-n / 2))) <= 1e-14
    q = oracle.e_expectations(a, n)
    t2 = _golden("table2_hwall.txt")[3:]
    assert np.all(np.abs(q - t2[None, :]) <= 5e-4)  # printed to 3 decimals
    assert np.all(np.abs(q - np.array([0.0, 0.5, 0.5])) <= 1e-13)


@pytest.mark.parametrize("n", [2, 7, 15])
def test_ghz_closed_form(n):
    """PAPER.md §5.2 (743-745): (|0..0> + |1..1>)/sqrt2; Table 3 expectations."""
    a = oracle.e_simulate(n, C.ghz_chain(n))
    ref = np.zeros(1 << n, dtype=np.complex128)
    ref[0] = ref[-1] = 1 / math.sqrt(2)
    assert np.max(np.abs(a - ref)) <= 1e-15
    q = oracle.e_expectations(a, n)
    assert np.all(np.abs(q - _golden("table3_ghz.txt")[3:][None, :]) <= 5e-4)
    assert np.all(np.abs(q - 0.5) <= 1e-15)


@pytest.mark.parametrize("n,x", [(6, 37), (11, 1234), (14, 9999)])
def test_qft_closed_form(n, x):
    """a(y) = 2^{-N/2} exp(2 pi i x y / 2^N) (BASELINE config 5; reading A15),
    phase from x*y mod 2^N in integer arithmetic."""
    circ, _ = C.qft(n, x=x)
    a = oracle.e_simulate(n, circ)
    y = np.arange(1 << n, dtype=np.uint64)
    ph = ((np.uint64(x) * y) % np.uint64(1 << n)).astype(np.float64) * (2 * math.pi / (1 << n))
    ref = 2.0 ** (-n / 2) * np.exp(1j * ph)
    assert np.max(np.abs(a - ref)) <= 1e-12
    assert np.all(np.abs(oracle.e_probabilities(a, n) - 0.5) <= 1e-12)


def test_product_state_closed_form():
    """Eq. appa2: single-qubit-only circuit -> prod_j V_j|0>."""
    n = 12
    circ = C.layered(n, 3, seed=11, entangle=False)
    a = oracle.e_simulate(n, circ)
    v = [np.array([1, 0], dtype=np.complex128) for _ in range(n)]
    for g in range(len(circ)):
        _, _, t, _, _, u = circ.gate(g)
        v[t] = u @ v[t]
    ref = np.array([1.0 + 0j])
    for q in range(n - 1, -1, -1):
        ref = np.kron(ref, v[q])
    assert np.max(np.abs(a - ref)) <= 1e-13


def test_norm_and_involutions():
    """Eq. STAT1 norm preservation; X^2 = H^2 = Toffoli^2 = SWAP^2 = I;
    H_1 U_01(pi) H_1 = CNOT_01."""
    n = 9
    circ = C.random_circuit(n, 150, seed=3)
    a = oracle.e_simulate(n, circ)
    assert abs(oracle.e_norm2(a, n) - 1.0) <= 1e-12
    b = a.copy()
    for u, t, ctl in [(C.mat_X(), 3, ()), (C.mat_H(), 5, ()), (C.mat_X(), 1, (0, 7))]:
        oracle.e_apply(b, n, u, t, ctl)
        oracle.e_apply(b, n, u, t, ctl)
        assert np.max(np.abs(b - a)) <= 1e-14
    oracle.e_swap(b, n, 2, 8)
    oracle.e_swap(b, n, 8, 2)
    assert np.max(np.abs(b - a)) <= 1e-15
    c1 = a.copy()
    oracle.e_apply(c1, n, C.mat_H(), 1)
    oracle.e_apply(c1, n, C.mat_U1(math.pi), 1, (0,))
    oracle.e_apply(c1, n, C.mat_H(), 1)
    c2 = oracle.e_apply(a.copy(), n, C.mat_X(), 1, (0,))
    assert np.max(np.abs(c1 - c2)) <= 1e-14


def test_expectations_vs_dense_pauli():
    """<Q alpha(n)> = <psi|(1 - sigma^alpha_n)|psi>/2."""
    n = 6
    a = oracle.e_simulate(n, C.random_circuit(n, 80, seed=5))
    q = oracle.e_expectations(a, n)
    for k in range(n):
        for col, s in enumerate((SX, SY, SZ)):
            op = np.eye(1 << n) - kron_ops(n, {k: s})
            ref = (np.vdot(a, op @ a) / 2).real
            assert abs(q[k, col] - ref) <= 1e-13
    p = oracle.e_probabilities(a, n)
    assert np.max(np.abs(p - q[:, 2])) <= 1e-14


def test_single_qubit_textbook_expectations():
    """|+>: Qx=0; |->: Qx=1; S|+> = |+i>: Qy=0; |1>: Qz=1."""
    n = 1
    a = oracle.e_apply(oracle.e_init(1), n, C.mat_H(), 0)
    assert np.allclose(oracle.e_expectations(a, n), [[0, 0.5, 0.5]], atol=1e-15)
    b = oracle.e_apply(oracle.e_apply(oracle.e_init(1), n, C.mat_X(), 0), n, C.mat_H(), 0)
    assert np.allclose(oracle.e_expectations(b, n), [[1, 0.5, 0.5]], atol=1e-15)
    c = oracle.e_apply(a.copy(), n, C.mat_S(), 0)
    assert np.allclose(oracle.e_expectations(c, n), [[0.5, 0, 0.5]], atol=1e-15)
    d = oracle.e_apply(oracle.e_init(1), n, C.mat_X(), 0)
    assert np.allclose(oracle.e_expectations(d, n), [[0.5, 0.5, 1]], atol=1e-15)


def test_measure_projects_and_renormalises():
    """M: outcome 0 iff u < p0; kept half scaled by 1/sqrt(p)."""
    n = 7
    a = oracle.e_simulate(n, C.ghz_chain(n))
    b = a.copy()
    out, p0 = oracle.e_measure(b, n, 3, 0.25)
    assert out == 0 and abs(p0 - 0.5) <= 1e-15
    ref = np.zeros(1 << n, dtype=np.complex128)
    ref[0] = 1
    assert np.max(np.abs(b - ref)) <= 1e-15
    c = a.copy()
    out, _ = oracle.e_measure(c, n, 6, 0.75)
    ref = np.zeros(1 << n, dtype=np.complex128)
    ref[-1] = 1
    assert out == 1 and np.max(np.abs(c - ref)) <= 1e-15
    # random state: projected state equals P|psi>/|P psi|
    s = oracle.e_simulate(n, C.random_circuit(n, 50, seed=9))
    p1 = oracle.e_probabilities(s, n)[2]
    t = s.copy()
    out, p0 = oracle.e_measure(t, n, 2, 0.999999)
    assert out == 1 and abs(p0 - (1 - p1)) <= 1e-14
    proj = s * (((np.arange(1 << n) >> 2) & 1) == 1)
    assert np.max(np.abs(t - proj / np.linalg.norm(proj))) <= 1e-14
    # zero-norm projection fails
    z = oracle.e_init(n)
    assert oracle.e_measure(z, n, 0, 1.0)[0] == -5  # u = 1 forces outcome 1, p1 = 0


def test_clear_set_vs_dense_projector():
    """CLEAR / SET: (|v><v|_n x I) psi / ||...||; failure on zero norm."""
    n = 6
    a = oracle.e_simulate(n, C.layered(n, 2, seed=12))  # every qubit in superposition
    for qubit in (0, 3, 5):
        for value in (0, 1):
            P = np.diag([1.0 - value, float(value)]).astype(np.complex128)
            ref = kron_ops(n, {qubit: P}) @ a
            ref /= np.linalg.norm(ref)
            b = a.copy()
            assert oracle.e_project(b, n, qubit, value) == 0
            assert np.max(np.abs(b - ref)) <= 1e-14
    z = oracle.e_init(n)
    assert oracle.e_project(z, n, 2, 1) == -5 and z[0] == 1


def test_generate_events_inverse_cdf():
    """GENERATE EVENTS: inverse CDF in index order, checked
    against numpy cumsum + searchsorted, and GHZ events are only |0..0> / |1..1>."""
    n = 9
    a = oracle.e_simulate(n, C.layered(n, 2, seed=4))
    u = C.splitmix_uniform(77, 3000)
    got = oracle.e_sample(a, n, u)
    cum = np.cumsum(np.abs(a) ** 2)
    ref = np.searchsorted(cum, u * cum[-1], side="right")
    close = np.abs(cum[np.minimum(ref, (1 << n) - 1)] - u * cum[-1]) < 1e-12
    assert np.all((got == ref) | close)
    g = oracle.e_simulate(n, C.ghz_chain(n))
    ev = oracle.e_sample(g, n, u)
    assert set(np.unique(ev).tolist()) == {0, (1 << n) - 1}
    frac1 = np.mean(ev == (1 << n) - 1)
    assert abs(frac1 - 0.5) < 0.05


def test_shorbox_closed_form_and_period():
    """SHORBOX: amplitude 2^{-nx/2} exactly at x + 2^nx (y^x mod G);
    after the QFT on the x-register the x-distribution sits on multiples of 2^nx / r
    (G = 15, y = 7: period r = 4 divides 2^nx, so the peaks are exact)."""
    n, nx, G, y = 8, 4, 15, 7
    a = oracle.e_shorbox(n, nx, G, y)
    nz = np.flatnonzero(np.abs(a) > 0)
    want = sorted(x + (pow(y, x, G) << nx) for x in range(1 << nx))
    assert nz.tolist() == want
    assert np.allclose(a[nz], 2.0 ** (-nx / 2), atol=0) and abs(oracle.e_norm2(a, n) - 1) <= 1e-15
    oracle.e_run(a, n, C.qft_register(n, nx))
    px = (np.abs(a.reshape(1 << (n - nx), 1 << nx)) ** 2).sum(axis=0)
    assert np.all(px[[0, 4, 8, 12]] > 0.2) and px[[k for k in range(16) if k % 4]].max() <= 1e-15
