"""Pins of the oracle's lazy-bounds A policy (NEXT-4 of SURVEY §8(f);
reading R-A25: (r0, r1) are kept while every output magnitude stays within
one step of them, recomputed exactly -- the exact policy's step -- when one
leaves).  Each pin checks the policy against something
other than itself: closed forms of the paper's workloads, the exact policy
(pinned in test_oracle_a.py) on the gates where both recompute, the pinned
encode / decode primitives where it keeps the bounds, and the paper's
accuracy level."""
import math

import numpy as np

import oracle
import qsim_inputs as C


def test_h_wall_rescales_every_gate_and_is_exact():
    """Tables 2 caption: the H wall is exact in A.  From
    the sentinel bounds every H leaves the (degenerate) range: N rescales."""
    n = 10
    a = oracle.AState(n)
    rs = a.run_lazy(C.h_wall(n))
    assert rs == n
    assert np.max(np.abs(a.decoded() - 2.0 ** (-n / 2))) <= 1e-15


def test_ghz_is_exact_and_cnots_keep_the_bounds():
    """Table 3 caption: GHZ exact in A; the CNOT chain
    only moves amplitudes: no rescale after the H."""
    n = 9
    a = oracle.AState(n)
    rs = a.run_lazy(C.ghz_chain(n))
    z = a.decoded()
    ref = np.zeros(1 << n)
    ref[0] = ref[-1] = 1 / math.sqrt(2)
    assert rs == 1 and np.max(np.abs(z - ref)) <= 1e-15


def test_equals_the_exact_policy_on_permutations_and_phases():
    """X / CNOT / Toffoli / SWAP and diagonal gates leave the set of
    magnitudes unchanged, so the exact policy's recomputed bounds equal the
    kept ones: identical codes from any start."""
    n = 10
    codes, r0, r1 = C.random_codes(n, seed=3)
    codes[2], codes[4] = -127, 126  # the extreme codes present: (r0, r1) are exact
    rng = np.random.default_rng(4)
    circ = C.Circuit(n)
    for _ in range(40):
        a, b, c = (int(v) for v in rng.choice(n, 3, replace=False))
        k = rng.integers(6)
        if k == 0:
            circ.add("X", C.mat_X(), a)
        elif k == 1:
            circ.add("CNOT", C.mat_X(), b, [a])
        elif k == 2:
            circ.add("TOF", C.mat_X(), c, [a, b])
        elif k == 3:
            circ.swap(a, b)
        elif k == 4:
            circ.add("Rz", C.mat_Rz(rng.uniform(0, 6.3)), a)
        else:
            circ.add("CPHASE", C.mat_U1(rng.uniform(0, 6.3)), b, [a])
    lazy = oracle.AState(n, codes, r0, r1)
    exact = oracle.AState(n, codes, r0, r1)
    assert lazy.run_lazy(circ) == 0
    exact.run(circ)
    # the exact policy recomputes |e^{i phi} z| (rounding: 1e-16 relative); the lazy one keeps (r0, r1)
    assert np.array_equal(lazy.codes, exact.codes)
    assert (lazy.r0, lazy.r1) == (r0, r1)
    assert abs(exact.r0 / r0 - 1) <= 1e-12 and abs(exact.r1 / r1 - 1) <= 1e-12


def test_keep_step_is_the_pinned_encode_and_rescale_step_is_the_exact_policy():
    """One dense gate from identical codes: if the output stays in range the
    codes are oracle_a_encode (pinned) of the fp64 gate output with the old
    bounds; if not, the exact policy's result."""
    n = 9
    kept = rescaled = 0
    for seed in range(12):
        codes, r0, r1 = C.random_codes(n, seed=seed)
        codes[2], codes[4] = -127, 126
        u = C.mat_haar(np.random.default_rng(seed)) if seed % 3 else C.mat_Rx(0.05 * seed)
        t = seed % n
        lazy = oracle.AState(n, codes, r0, r1)
        did = lazy.apply_lazy(u, t)
        if did:
            exact = oracle.AState(n, codes, r0, r1)
            exact.apply(u, t)
            assert np.array_equal(lazy.codes, exact.codes) and (lazy.r0, lazy.r1) == (exact.r0, exact.r1)
            rescaled += 1
        else:
            z = oracle.e_run(oracle.AState(n, codes, r0, r1).decoded(), n, C.Circuit(n).add("U", u, t))
            ref = oracle.AState(n)
            for i, zi in enumerate(z):
                b0, b1 = oracle.a_encode(zi, r0, r1)
                ref.codes[2 * i], ref.codes[2 * i + 1] = b0, b1
            assert np.array_equal(lazy.codes, ref.codes) and (lazy.r0, lazy.r1) == (r0, r1)
            kept += 1
    assert kept and rescaled  # both branches exercised


def test_paper_accuracy_on_the_config4_recipe():
    """About 3 digits: expectation values within the
    paper's A-vs-exact level (0.011, Table 4) of E, and fidelity >= 0.95, on
    the config-4 recipe at N = 12 -- as for the exact policy."""
    n = 12
    circ = C.rz_rx_cphase(n, 6, seed=4)
    a = oracle.AState(n)
    rs = a.run_lazy(circ)
    z = a.decoded()
    e = oracle.e_simulate(n, circ)
    f = abs(np.vdot(z, e)) ** 2 / (np.vdot(z, z).real * np.vdot(e, e).real)
    assert f >= 0.95
    assert np.max(np.abs(oracle.e_expectations(z, n) - oracle.e_expectations(e, n))) <= 0.011
    assert 0 < rs < len(circ)  # lazy: fewer rescales than gates
