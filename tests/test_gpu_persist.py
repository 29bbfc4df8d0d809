"""The single-persistent-kernel mode of SURVEY §8(d) config 1
(qsim_apply_circuit_persistent: the whole circuit in one cluster launch, the
state in distributed shared memory): parity with the oracle (E, 1e-12,
Eq. NUM2 with controls) on the config-1 recipe, on targets
and controls among the cluster-select bits, with SWAP relabels, and mixed
with the ordinary path."""
import numpy as np
import pytest

import oracle
import qsim_inputs as C

pytestmark = pytest.mark.gpu
q = pytest.importorskip("paper_1805_04708_b200")
TOL = 1e-12


@pytest.mark.parametrize("seed", range(5))
def test_config1_persistent_vs_oracle(seed):
    n = 14
    circ = C.config(0, seed=seed)
    with q.State(n) as s:
        s.apply_circuit_persistent(circ)
        st = s.stats()
        z = s.get_state()
    assert np.max(np.abs(z - oracle.e_simulate(n, circ))) <= TOL
    assert st["kernels"] == 1  # one launch for 200 gates


@pytest.mark.parametrize("n", [4, 9, 16])
def test_sizes_cluster_bits_controls_and_swaps(n):
    rng = np.random.default_rng(n)
    circ = C.random_circuit(n, 150, seed=n)
    for _ in range(10):  # gates on the top (cluster-select) bits, with controls there and below
        t = int(rng.integers(n - 3, n))
        c = int(rng.integers(0, n))
        while c == t:
            c = int(rng.integers(0, n))
        circ.add("Haar", C.mat_haar(rng), t, [c])
        a, b = (int(v) for v in rng.choice(n, 2, replace=False))
        circ.swap(a, b)
    with q.State(n) as s:
        s.apply_circuit_persistent(circ)
        z = s.get_state()
    assert np.max(np.abs(z - oracle.e_simulate(n, circ))) <= TOL


def test_mixed_with_the_ordinary_path_and_errors():
    n = 14
    c1 = C.config(0, seed=7)
    c2 = C.layered(n, 2, seed=7)
    with q.State(n) as s:
        s.apply_circuit(c1)
        s.apply_circuit_persistent(c2)
        s.apply_circuit(c1)
        z = s.get_state()
    ref = oracle.e_simulate(n, c1)
    ref = oracle.e_run(oracle.e_run(ref, n, c2), n, c1)
    assert np.max(np.abs(z - ref)) <= TOL
    with q.State(17) as s, pytest.raises(q.QsimError) as err:
        s.apply_circuit_persistent(C.h_wall(17))
    assert err.value.code == -1
    with q.State(12, q.ENC_ADAPTIVE2) as s, pytest.raises(q.QsimError) as err:
        s.apply_circuit_persistent(C.h_wall(12))
    assert err.value.code == -7


@pytest.mark.parametrize("lcs,K", [(3, 3), (3, 4), (4, 3), (4, 4)])
def test_cluster_sizes_and_phase_widths(lcs, K, monkeypatch):
    """Every cluster size (8 / 16 CTAs) and phase width (K = 3 / 4 qubits per
    register group) the kernel can run, against the oracle: phases on local
    bits, phases holding cluster-select bits (DSMEM), controls inside and
    outside a phase's qubits."""
    monkeypatch.setenv("QSIM_PERSIST_LCS", str(lcs))
    monkeypatch.setenv("QSIM_PERSIST_K", str(K))
    for n in (12, 15):
        circ = C.config(0, n=n, seed=n + K)
        with q.State(n) as s:
            s.apply_circuit_persistent(circ)
            z = s.get_state()
        assert np.max(np.abs(z - oracle.e_simulate(n, circ))) <= TOL


def test_planned_circuit_cache():
    """A gate list seen before replays its device records (no planning, no
    upload): the same circuit twice, another in between, more circuits than
    the cache holds, and a relabel (SWAP) changing the physical records."""
    n = 13
    cs = [C.config(0, n=n, seed=20 + i) for i in range(10)]
    order = [0, 0, 1, 0, 2, 3, 4, 5, 6, 7, 8, 9, 0, 1]
    ref = oracle.e_init(n)
    with q.State(n) as s:
        for i in order:
            s.apply_circuit_persistent(cs[i])
            ref = oracle.e_run(ref, n, cs[i])
        sw = C.Circuit(n).swap(0, n - 1)
        s.apply_circuit_persistent(sw)
        s.apply_circuit_persistent(cs[0])
        ref = oracle.e_run(oracle.e_run(ref, n, sw), n, cs[0])
        z = s.get_state()
    assert np.max(np.abs(z - ref)) <= TOL
