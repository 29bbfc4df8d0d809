"""The diagonal-run epilogue of the dense A apply kernel: the diagonal gates
that follow a dense gate are applied as its apply kernel stores the codes
(integer b1 steps, PAPER.md:442-444 -- a phase gate on the A encoding moves
b1 only).  The codes must be bit-identical to the separate diagonal sweeps
(QSIM_A_NO_EPILOGUE=1), for every placement of the diagonal gates' target and
controls relative to the dense gate's 16-code unit (inside, outside, both,
global), in both bounds policies, on one shard and on loopback shards (global
qubits), including runs longer than the epilogue holds; and fewer kernels
launch.  Parity of the whole path against the oracle-A is covered by
test_gpu_a_size.py (the config-4 recipe interleaves Rz runs with Rx gates)."""
import os

import numpy as np
import pytest

import qsim_inputs as C

pytestmark = pytest.mark.gpu
q = pytest.importorskip("paper_1805_04708_b200")


def epilogue_circuit(n, seed, ndense=24):
    rng = np.random.default_rng(seed)
    c = C.Circuit(n)
    for q0 in range(n):
        c.add("H", C.mat_H(), q0)
    dense = [C.mat_H(), C.mat_Rx(0.7), C.mat_haar(rng), C.mat_U3(0.3, 0.2, 0.1)]
    diag = [C.mat_Rz(0.9), C.mat_S(), C.mat_T(), C.mat_Z(), C.mat_R(5), C.mat_U1(-2.1), C.mat_T(True)]
    for _ in range(ndense):
        t = int(rng.integers(0, n))
        nc = int(rng.integers(0, 2))
        ctl = tuple(int(x) for x in rng.choice([b for b in range(n) if b != t], nc, replace=False))
        c.add("D", dense[int(rng.integers(0, len(dense)))], t, ctl)
        # a run of diagonal gates: lengths past the epilogue's capacity, targets and
        # controls on the unit's own bits (0..3 and the dense target), on others, on both
        run = int(rng.choice([0, 1, 3, 8, 30, 70]))
        near = sorted({0, 1, 2, 3, t} & set(range(n)))
        for _ in range(run):
            pool = near if rng.random() < 0.5 else list(range(n))
            tt = int(rng.choice(pool))
            k = int(rng.integers(0, 3))
            cands = [b for b in range(n) if b != tt]
            cc = tuple(int(x) for x in rng.choice(cands, min(k, len(cands)), replace=False))
            c.add("P", diag[int(rng.integers(0, len(diag)))], tt, cc)
    return c


def run_codes(n, circ, P, policy, epilogue):
    old = os.environ.pop("QSIM_A_NO_EPILOGUE", None)
    if not epilogue:
        os.environ["QSIM_A_NO_EPILOGUE"] = "1"
    try:
        with q.State(n, q.ENC_ADAPTIVE2, P, a_policy=policy) as s:
            s.apply_circuit(circ)
            st = s.stats()
            codes, r0, r1 = s.get_codes()
    finally:
        os.environ.pop("QSIM_A_NO_EPILOGUE", None)
        if old is not None:
            os.environ["QSIM_A_NO_EPILOGUE"] = old
    return codes, r0, r1, st


@pytest.mark.parametrize("policy", ["exact", "lazy"])
@pytest.mark.parametrize("n,P", [(14, 1), (12, 4), (16, 2), (18, 4), (21, 1)])
def test_epilogue_bit_identical(n, P, policy):
    pol = q.A_POLICY_LAZY if policy == "lazy" else q.A_POLICY_EXACT
    circ = epilogue_circuit(n, seed=n * 10 + P)
    c1, a0, a1, st1 = run_codes(n, circ, P, pol, True)
    c0, b0, b1, st0 = run_codes(n, circ, P, pol, False)
    assert (a0, a1) == (b0, b1)
    assert np.array_equal(c1, c0)
    assert st1["a_dense"] == st0["a_dense"] and st1["a_rescales"] == st0["a_rescales"]
    assert st1["kernels"] < st0["kernels"], (st1["kernels"], st0["kernels"])


def test_epilogue_config4_recipe():
    """The config-4 recipe (coin-flip Rz / Rx layers + CPHASE) at N = 20: the
    Rz runs fold into the Rx gates' apply kernels, codes unchanged."""
    n = 20
    circ = C.rz_rx_cphase(n, 6, seed=4)
    c1, a0, a1, st1 = run_codes(n, circ, 1, q.A_POLICY_EXACT, True)
    c0, b0, b1, st0 = run_codes(n, circ, 1, q.A_POLICY_EXACT, False)
    assert (a0, a1) == (b0, b1) and np.array_equal(c1, c0)
    assert st1["kernels"] < st0["kernels"]
