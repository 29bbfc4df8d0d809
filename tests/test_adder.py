"""The QFT adder (section 5.3, Table 4; NEXT-2 of
SURVEY §8(f)): the generator (qsim_inputs.draper_adder) and the oracle
pinned to the closed form -- the circuit maps the basis state |b>|a> to
|a + b mod 2^k>|a> -- and the register layout pinned to the printed E
columns of Table 4 (reading R-B12: the a-register in reversed bit order)."""
import os

import numpy as np
import pytest

import oracle
import qsim_inputs as C


def adder_index(k, a, b):
    """Closed form: the output basis index of draper_adder(k, a, b)."""
    idx = (a + b) % (1 << k)
    for j in range(k):
        if (a >> j) & 1:
            idx |= 1 << (2 * k - 1 - j)
    return idx


def closed_form_expectations(n, idx):
    """<Qx>, <Qy>, <Qz> of a basis state: 1/2, 1/2, bit."""
    return np.array([[0.5, 0.5, float((idx >> q) & 1)] for q in range(n)])


def test_adder_closed_form_on_the_oracle():
    rng = np.random.default_rng(11)
    for k in (3, 5, 7, 8):
        for _ in range(3):
            a, b = (int(v) for v in rng.integers(0, 1 << k, 2))
            psi = oracle.e_simulate(2 * k, C.draper_adder(k, a, b))
            ref = np.zeros_like(psi)
            ref[adder_index(k, a, b)] = 1.0
            assert np.max(np.abs(psi - ref)) <= 1e-12


def test_adder_gate_count():
    k, a, b = 15, 13410, 19357
    c = C.draper_adder(k, a, b)
    assert len(c) == bin(a).count("1") + bin(b).count("1") + 3 * k * (k + 1) // 2


def test_table4_layout_matches_the_printed_exact_columns():
    """Table 4's E columns are the closed form of the paper's instance
    (k = 19, 210018 + 314269 = 2^19 - 1) with this register layout."""
    rows = np.loadtxt(os.path.join(os.path.dirname(__file__), "golden", "table4_adder.txt"))
    k, a, b = 19, 210018, 314269
    q = closed_form_expectations(2 * k, adder_index(k, a, b))
    assert np.array_equal(rows[:, 0], np.arange(2 * k))
    assert np.max(np.abs(rows[:, 4:7] - q)) <= 5e-4
    # the paper's A columns deviate from exact by at most 0.011 (the A accuracy bar)
    assert np.max(np.abs(rows[:, 1:4] - rows[:, 4:7])) == pytest.approx(0.011, abs=1e-9)
