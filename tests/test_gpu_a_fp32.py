"""The fp32-arithmetic A variant (QSIM_A_POLICY_FP32, reading R-A26; SURVEY
8(f) NEXT-4 "fp32 decode/apply"): exact bounds as the default policy, the
decode / apply / encode in fp32 without the certified fp64 fallback.  Per
gate from identical codes against the oracle-A (§4.1,
the fp64 step-by-step decode-apply-encode): bounds equal, every magnitude
code within one step, every angle code within one step where fp32 resolves
the angle (an output's fp32 error is ~1e-6 (|a0| + |a1|), so its angle is
within a step once |z| >= 2e-4 r1; a near-cancelled output's angle is not
determined in fp32, and its decoded value is still within one magnitude step
+ 2|z| of the reference), almost all codes identical; whole circuits against
E: fidelity close to the certified policy's."""
import numpy as np
import pytest

import oracle
import qsim_inputs as C

pytestmark = pytest.mark.gpu
q = pytest.importorskip("paper_1805_04708_b200")


def code_diff(cg, co):
    b0 = np.abs(cg[0::2].astype(int) - co[0::2].astype(int))
    d1 = np.abs(cg[1::2].astype(int) - co[1::2].astype(int)) % 256
    b1 = np.minimum(d1, 256 - d1)
    zero = (cg[0::2] == -128) & (co[0::2] == -128)
    return np.where(zero, 0, b0), np.where(zero, 0, b1)


CASES = [("H", C.mat_H), ("Rx", lambda: C.mat_Rx(1.1)), ("Haar", lambda: C.mat_haar(np.random.default_rng(9)))]


@pytest.mark.parametrize("name,mk", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("t,ctl", [(0, ()), (3, ()), (7, ()), (5, (11,)), (12, (2, 9))])
def test_per_gate_vs_oracle_a(name, mk, t, ctl):
    n = 16
    codes, r0, r1 = C.random_codes(n, seed=31 + t)
    codes[2], codes[4] = -127, 126
    u = mk()
    ref = oracle.AState(n, codes, r0, r1)
    ref.apply(u, t, ctl)
    with q.State(n, q.ENC_ADAPTIVE2, 1, a_policy=q.A_POLICY_FP32) as s:
        s.set_codes(codes, r0, r1)
        s.apply_gate(u, t, ctl)
        cg, g0, g1 = s.get_codes()
        zg = s.get_state()
    assert g0 == pytest.approx(ref.r0, rel=1e-12, abs=1e-15 * ref.r1) and g1 == pytest.approx(ref.r1, rel=1e-12)
    db0, db1 = code_diff(cg, ref.codes)
    zr = ref.decoded()
    resolved = np.abs(zr) >= 2e-4 * r1
    assert db0.max() <= 1 and db1[resolved].max() <= 1
    step = (ref.r1 - ref.r0) / 253.0
    assert np.all(np.abs(zg - zr) <= step + 2 * np.abs(zr) + 1e-12)
    # uncertified: a code differs where the fp32 error straddles a rounding
    # boundary (the certified policy sends those to fp64) -- ~1e-3 of them here
    assert np.mean((db0 == 0) & (db1 == 0)) >= 0.995


def test_special_codes_and_whole_circuit():
    """The specials: a basis state (|z| = 1 exactly, the special one) through
    X / phase gates and H, zero amplitudes kept; and the config-4 recipe at
    N = 18 against E, fidelity within 2e-3 of the certified policy's."""
    n = 12
    circ = C.Circuit(n)
    for b in (0, 5, 11):
        circ.add("X", C.mat_X(), b)
    circ.add("S", C.mat_S(), 5)
    circ.add("H", C.mat_H(), 3)
    with q.State(n, q.ENC_ADAPTIVE2, 1, a_policy=q.A_POLICY_FP32) as s:
        s.apply_circuit(circ)
        z = s.get_state()
    e = oracle.e_simulate(n, circ)
    assert np.max(np.abs(z - e)) <= 1e-12
    n = 18
    circ = C.rz_rx_cphase(n, 6, seed=4)
    e = oracle.e_simulate(n, circ)
    f = {}
    for pol in (q.A_POLICY_EXACT, q.A_POLICY_FP32):
        with q.State(n, q.ENC_ADAPTIVE2, 1, a_policy=pol) as s:
            s.apply_circuit(circ)
            z = s.get_state()
        f[pol] = abs(np.vdot(z, e)) ** 2 / (np.vdot(z, z).real * np.vdot(e, e).real)
    assert abs(f[q.A_POLICY_FP32] - f[q.A_POLICY_EXACT]) <= 2e-3, f


def test_shard_count_independent():
    """As for the certified policy, the fp32 variant's codes do not depend on
    the sharding: the bounds are the exact global extremes and each pair's
    fp32 arithmetic is the same wherever it runs (1 vs 4 loopback shards,
    dense gates on global qubits through the exchange path)."""
    n = 14
    circ = C.rz_rx_cphase(n, 3, seed=8)
    out = []
    for P in (1, 4):
        with q.State(n, q.ENC_ADAPTIVE2, P, a_policy=q.A_POLICY_FP32) as s:
            s.apply_circuit(circ)
            out.append(s.get_codes())
    assert out[0][1:] == out[1][1:]
    assert np.array_equal(out[0][0], out[1][0])
