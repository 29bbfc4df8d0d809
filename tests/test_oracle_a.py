"""Pins for the A (adaptive 2-byte encoding) oracle, §4.1 (446-460).

Worked examples and invariants fixed by the paper's definition (specials,
the linear magnitude map, theta = pi b1/128), the quantisation half-step
round-trip bound, encode/decode idempotence, and the paper's statement that
the H-wall and GHZ results are exact in A (Tables 2-3 captions).
"""
import math

import numpy as np
import pytest

import oracle
import qsim_inputs as C


def test_worked_examples():
    """r=0 <-> b0=-128, r=1 <-> b0=127."""
    r0, r1 = 0.1, 0.6
    assert oracle.a_encode(0j, r0, r1)[0] == -128
    assert oracle.a_encode(1 + 0j, r0, r1) == (127, 0)
    assert oracle.a_encode(r0 * 1j, r0, r1) == (-127, 64)  # lower endpoint, theta = pi/2
    assert oracle.a_encode(r1 * np.exp(-0.25j * math.pi), r0, r1) == (126, -32)  # upper endpoint
    assert oracle.a_decode(-128, 77, r0, r1) == 0
    z = oracle.a_decode(127, -128, r0, r1)
    assert abs(z - (-1)) <= 1e-15  # e^{-i pi}
    # decode map of PAPER.md:453 at its end points and midpoint
    assert abs(abs(oracle.a_decode(-127, 0, r0, r1)) - r0) <= 1e-15
    assert abs(abs(oracle.a_decode(126, 0, r0, r1)) - r1) <= 1e-15
    assert abs(abs(oracle.a_decode(0, 0, r0, r1)) - (127 * (r1 - r0) / 253 + r0)) <= 1e-15
    # angle grid theta = pi b1 / 128
    for b1 in (-128, -64, -1, 0, 1, 32, 127):
        z = oracle.a_decode(127, b1, r0, r1)
        assert abs(z - np.exp(1j * math.pi * b1 / 128)) <= 1e-15
    # theta = +pi wraps to b1 = -128 (reading R-A6)
    assert oracle.a_encode(-0.3 + 0j, r0, r1)[1] == -128


def test_round_trip_half_step_bound_and_idempotence():
    """|decode(encode(z)) - z| <= pi/256 * |z| + (r1-r0)/506 (+1e-12) for z in the
    annulus (half a step in angle and magnitude); encode(decode(c)) = c."""
    rng = np.random.default_rng(1)
    r0, r1 = 0.013, 0.47
    m = rng.uniform(r0, r1, 20000)
    th = rng.uniform(-math.pi, math.pi, 20000)
    for mm, tt in zip(m[:3000], th[:3000]):
        z = mm * np.exp(1j * tt)
        b0, b1 = oracle.a_encode(z, r0, r1)
        zz = oracle.a_decode(b0, b1, r0, r1)
        assert abs(abs(zz) - mm) <= (r1 - r0) / 506 + 1e-12
        dth = (math.atan2(zz.imag, zz.real) - tt + math.pi) % (2 * math.pi) - math.pi
        assert abs(dth) <= math.pi / 256 + 1e-12
        assert abs(zz - z) <= mm * math.pi / 256 + (r1 - r0) / 506 + 1e-12
    for b0 in range(-128, 128):
        for b1 in (-128, -77, 0, 5, 127):
            c = (b0, b1)
            z = oracle.a_decode(b0, b1, r0, r1)
            e = oracle.a_encode(z, r0, r1)
            if b0 == -128:
                assert e[0] == -128
            else:
                assert e == c


def test_degenerate_bounds():
    """r0 == r1 (reading R-A7): any b0 in [-127,126] decodes to r0; encode emits 0."""
    r = 0.25
    for b0 in (-127, 0, 126):
        assert abs(abs(oracle.a_decode(b0, 3, r, r)) - r) <= 1e-15
    assert oracle.a_encode(r * 1j, r, r) == (0, 64)


def test_bounds_definition():
    """min/max of |z| over 0<|z|<1; sentinel when none (R-A8)."""
    z = np.array([0, 1, 0.3j, -0.5, 0.2 + 0.2j, -1j], dtype=np.complex128)
    r0, r1 = oracle.a_bounds(z)
    assert r0 == pytest.approx(math.hypot(0.2, 0.2), abs=1e-16) and r1 == 0.5
    assert oracle.a_bounds(np.array([0, 1, -1j, 0], dtype=np.complex128)) == (0.5, 0.5)


@pytest.mark.parametrize("n", [1, 6, 13])
def test_h_wall_exact_in_a(n):
    """Table 2 caption: A gives the same exact results as E;
    bounds become r0 = r1 = 2^{-N/2}."""
    s = oracle.AState(n).run(C.h_wall(n))
    z = s.decoded()
    assert np.max(np.abs(z - 2.0 ** (-n / 2))) <= 1e-14
    q = oracle.e_expectations(z, n)
    assert np.all(np.abs(q - np.array([0.0, 0.5, 0.5])) <= 1e-13)
    if n > 1:
        assert s.r0 == pytest.approx(2.0 ** (-n / 2), rel=1e-14) and s.r1 == pytest.approx(2.0 ** (-n / 2), rel=1e-14)
    # a T gate after the wall leaves the bounds unchanged
    r0, r1 = s.r0, s.r1
    s.apply(C.mat_T(), 0)
    assert (s.r0, s.r1) == pytest.approx((r0, r1), rel=1e-14)


@pytest.mark.parametrize("n", [2, 9])
def test_ghz_exact_in_a(n):
    """Table 3 caption: GHZ is exact in A."""
    z = oracle.AState(n).run(C.ghz_chain(n)).decoded()
    ref = np.zeros(1 << n, dtype=np.complex128)
    ref[0] = ref[-1] = 1 / math.sqrt(2)
    assert np.max(np.abs(z - ref)) <= 1e-15
    assert np.all(np.abs(oracle.e_expectations(z, n) - 0.5) <= 1e-15)


def test_permutation_circuits_bit_exact():
    """X / CNOT only swap amplitudes -> codes move untouched
    (SPEC S:334): on basis states A == E bit-exactly."""
    n = 8
    rng = np.random.default_rng(4)
    circ = C.Circuit(n)
    for _ in range(60):
        q = [int(v) for v in rng.choice(n, 3, replace=False)]
        k = rng.integers(4)
        if k == 0:
            circ.add("X", C.mat_X(), q[0])
        elif k == 1:
            circ.add("CNOT", C.mat_X(), q[1], [q[0]])
        elif k == 2:
            circ.add("TOFFOLI", C.mat_X(), q[2], q[:2])
        else:
            circ.swap(q[0], q[1])
    s = oracle.AState(n).run(circ)
    e = oracle.e_simulate(n, circ)
    assert np.array_equal(s.decoded(), e)
    # phase gates whose angle is a multiple of pi/128 are exact b1 additions
    s2 = oracle.AState(n).run(circ)
    k = int(np.flatnonzero(np.abs(e) > 0.5)[0])
    for g, shift in [(C.mat_Z(), 128), (C.mat_S(), 64), (C.mat_T(), 32), (C.mat_R(8), 1)]:
        before = s2.codes[2 * k + 1]
        s2.apply(g, 0)
        bit = (k >> 0) & 1
        exp = ((int(before) + shift * bit + 128) % 256) - 128
        assert s2.codes[2 * k + 1] == exp and s2.codes[2 * k] == 127


def test_a_accuracy_vs_e():
    """PAPER.md:131-132 ("about 3 digits"), Table 4 worst deviation 0.011:
    expectation values of A track E on a small random circuit."""
    n = 10
    circ = C.rz_rx_cphase(n, 4, seed=4)
    e = oracle.e_simulate(n, circ)
    s = oracle.AState(n).run(circ)
    z = s.decoded()
    qe, qa = oracle.e_expectations(e, n), oracle.e_expectations(z, n)
    assert np.max(np.abs(qe - qa)) <= 0.011 * 2
    f = abs(np.vdot(e, z)) ** 2 / (np.vdot(z, z).real * np.vdot(e, e).real)
    assert f >= 0.95
