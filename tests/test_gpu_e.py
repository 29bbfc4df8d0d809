"""GPU parity for the E (complex fp64) path through the C-ABI, against the
oracle on the same seeded inputs.  Bar (BASELINE.json north_star): max
|delta amplitude| <= 1e-12 after each circuit; norms <= 1e-10;
expectation values <= 1e-12."""
import math

import numpy as np
import pytest

import oracle
import qsim_inputs as C

pytestmark = pytest.mark.gpu

q = pytest.importorskip("paper_1805_04708_b200")

TOL = 1e-12


def gpu_run(n, circ, ngpus=1, **ex):
    s = q.State(n, q.ENC_FP64, ngpus, **ex) if ex else q.State(n, q.ENC_FP64, ngpus)
    s.apply_circuit(circ)
    return s


@pytest.mark.parametrize("seed", range(10))
def test_config1_random_circuits(seed):
    """BASELINE config 1: N=14, 200 gates from {H,X,Y,Z,S,T,Rz,Rx,Haar,CNOT,CPHASE,Toffoli}."""
    circ = C.config(0, seed=seed)
    ref = oracle.e_simulate(14, circ)
    with gpu_run(14, circ) as s:
        got = s.get_state()
        assert np.max(np.abs(got - ref)) <= TOL
        assert abs(s.norm() - 1.0) <= 1e-10
        st = s.stats()
        assert st["kernels"] > 0 and st["gates"] == 200


@pytest.mark.parametrize("fuse", [0, 1])
@pytest.mark.parametrize("n", [2, 3, 5, 8, 9, 12, 13, 17])
def test_small_and_ragged_sizes(n, fuse):
    """Tiny states (below one tile: padded shards), one tile, several tiles."""
    kinds = C.CFG1_KINDS if n >= 3 else tuple(k for k in C.CFG1_KINDS if k != "TOFFOLI")
    circ = C.random_circuit(n, 120, seed=n, kinds=kinds)
    ref = oracle.e_simulate(n, circ)
    s = q.State(n, q.ENC_FP64, 1, fuse=fuse)
    s.apply_circuit(circ)
    assert np.max(np.abs(s.get_state() - ref)) <= TOL
    s.close()


def test_every_target_and_class():
    """a3/a4/a5: dense, diagonal (both halves, |1>-only, |0>-only), anti-diagonal,
    with 0/1/2 controls below and above the target, on every target bit."""
    n = 14
    rng = np.random.default_rng(3)
    mats = [C.mat_haar(rng), C.mat_Z(), C.mat_T(), np.diag([np.exp(0.3j), 1.0]), C.mat_Y(), C.mat_X(),
            C.mat_Rz(1.1), C.mat_U1(0.7)]
    circ = C.h_wall(n)
    circ.extend(C.layered(n, 1, seed=9, h_first=False))
    for t in range(n):
        for m in mats:
            ctl = [] if t % 3 == 0 else ([(t + 5) % n] if t % 3 == 1 else [(t + 1) % n, (t + 7) % n])
            circ.add("M", m, t, ctl)
    ref = oracle.e_simulate(n, circ)
    for fuse in (0, 1):
        s = q.State(n, q.ENC_FP64, 1, fuse=fuse)
        s.apply_circuit(circ)
        assert np.max(np.abs(s.get_state() - ref)) <= TOL
        s.close()


def test_apply_gate_one_by_one_equals_circuit():
    n = 13
    circ = C.config(0, n=n, seed=4)
    ref = oracle.e_simulate(n, circ)
    with q.State(n) as s:
        for g in range(len(circ)):
            name, kind, t, t2, ctl, u = circ.gate(g)
            s.apply_gate(u, t, ctl)
        assert np.max(np.abs(s.get_state() - ref)) <= TOL


def test_fused_layers_config2_shape():
    """Config 2 recipe (H wall + layers of Haar on every qubit + CNOT matching) at
    N = 20, fused vs unfused vs oracle."""
    n = 20
    circ = C.layered(n, 3, seed=1)
    ref = oracle.e_simulate(n, circ)
    for fuse in (1, 0):
        s = q.State(n, q.ENC_FP64, 1, fuse=fuse)
        s.apply_circuit(circ)
        assert np.max(np.abs(s.get_state() - ref)) <= TOL
        st = s.stats()
        if fuse:
            assert st["passes"] > 0 and st["fused_gates"] > len(circ) // 2
        else:
            assert st["passes"] == 0
        s.close()


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_loopback_transparency(P):
    """PAPER.md §3.2 / SPEC S:475: results independent of the shard count and
    swap schedule (<= 1e-12); global-qubit gates go through the exchange."""
    n = 14
    circ = C.config(0, n=n, seed=P)
    circ.extend(C.layered(n, 2, seed=P, h_first=False))
    ref = oracle.e_simulate(n, circ)
    s = q.State(n, q.ENC_FP64, P)
    s.apply_circuit(circ)
    got = s.get_state()
    assert np.max(np.abs(got - ref)) <= TOL
    st = s.stats()
    assert st["exchanges"] > 0
    # exchange volume: a pairwise exchange moves half a shard per direction per
    # shard; an m-bit all-to-all remap moves 1 - 2^-m of every shard
    nl = n - int(math.log2(P))
    ops, _ = q.qsim_plan(n, P, circ)
    npair = sum(o["type"] == q.OP_EXCHANGE for o in ops)
    groups = {}
    for o in ops:
        if o["type"] == q.OP_REMAP:
            groups[o["gate_index"]] = groups.get(o["gate_index"], 0) + 1
    want = npair * P * (1 << (nl - 1)) * 16
    want += sum(P * ((1 << m) - 1) * (1 << (nl - m)) * 16 for m in groups.values())
    assert st["exchange_bytes"] == pytest.approx(want)
    pe = s.expectations()
    qe = oracle.e_expectations(ref, n)
    assert np.max(np.abs(pe - qe)) <= TOL
    assert np.max(np.abs(s.probabilities() - oracle.e_probabilities(ref, n))) <= TOL
    s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4, 8])
def test_global_permutation_gates_relabel_shards(P):
    """X / Y / CNOT / Toffoli whose target and controls are
    all global bits relabel the shards (which shard holds which global bits)
    instead of exchanging half-shards; the result, the expectations and the
    logical read-out are unchanged."""
    n = 14
    k = int(math.log2(P))
    perm_only = C.global_permutations(n, P, seed=P)
    nrelabel = sum(1 for o in q.qsim_plan(n, P, perm_only)[0] if o["type"] == q.OP_RELABEL)
    assert nrelabel > 0
    circ = C.global_permutations(n, P, seed=P)
    circ.extend(C.config(0, n=n, seed=P))
    circ.extend(C.layered(n, 1, seed=P, h_first=False))
    circ.extend(C.global_permutations(n, P, seed=P + 10))
    ref = oracle.e_simulate(n, circ)
    with q.State(n, q.ENC_FP64, P) as s:
        s.apply_circuit(perm_only)
        assert s.stats()["exchanges"] == 0  # permutations among global bits move no data
        s.reset()
        s.apply_circuit(circ)
        got = s.get_state()
        assert np.max(np.abs(got - ref)) <= TOL
        idx = np.array([0, 1, (1 << n) - 1, 12345, 1 << (n - 1), (1 << (n - k)) + 7], dtype=np.uint64)
        assert np.max(np.abs(s.get_amplitudes(idx) - ref[idx.astype(np.int64)])) <= TOL
        assert np.max(np.abs(s.expectations() - oracle.e_expectations(ref, n))) <= TOL
        assert abs(s.norm() - 1.0) <= 1e-10


@pytest.mark.gpu
def test_sharded_small_chunks_and_unfused():
    n = 13
    circ = C.layered(n, 2, seed=7)
    ref = oracle.e_simulate(n, circ)
    s = q.State(n, q.ENC_FP64, 4, chunk_bytes=4096, fuse=0)
    s.apply_circuit(circ)
    assert np.max(np.abs(s.get_state() - ref)) <= TOL
    s.close()


def test_local_gates_move_no_bytes_between_shards():
    """gates on local qubits (and diagonal gates anywhere) never exchange."""
    n = 14
    s = q.State(n, q.ENC_FP64, 4)
    c = C.Circuit(n)
    for t in range(12):
        c.add("H", C.mat_H(), t)
    c.add("Z", C.mat_Z(), 13)
    c.add("CP", C.mat_U1(0.4), 12, [13])
    c.add("CNOT", C.mat_X(), 3, [13])  # global control, local target
    s.apply_circuit(c)
    assert s.stats()["exchanges"] == 0
    assert np.max(np.abs(s.get_state() - oracle.e_simulate(n, c))) <= TOL
    s.close()


def test_expectations_probabilities_norm():
    n = 12
    circ = C.config(0, n=n, seed=11)
    ref = oracle.e_simulate(n, circ)
    with gpu_run(n, circ) as s:
        assert np.max(np.abs(s.expectations() - oracle.e_expectations(ref, n))) <= TOL
        assert np.max(np.abs(s.probabilities() - oracle.e_probabilities(ref, n))) <= TOL
        assert abs(s.norm() - oracle.e_norm2(ref, n)) <= 1e-12


def test_tables_2_3_on_gpu():
    """Tables 2-3 on the GPU path."""
    for circ, expect in [(C.h_wall(16), (0.0, 0.5, 0.5)), (C.ghz_chain(16), (0.5, 0.5, 0.5))]:
        with gpu_run(16, circ, ngpus=2) as s:
            assert np.max(np.abs(s.expectations() - np.array(expect)[None, :])) <= 1e-12


@pytest.mark.parametrize("P", [1, 4])
def test_measure(P):
    n = 12
    circ = C.config(0, n=n, seed=21)
    ref = oracle.e_simulate(n, circ)
    s = gpu_run(n, circ, ngpus=P)
    for qubit, u in [(0, 0.3), (11, 0.9), (5, 0.5)]:
        out, p0 = s.measure_u(qubit, u)
        ro, rp0 = oracle.e_measure(ref, n, qubit, u)
        assert out == ro and abs(p0 - rp0) <= 1e-12
        assert np.max(np.abs(s.get_state() - ref)) <= TOL
    # seeded variant: splitmix64 -> u = (x >> 11) 2^-53 (include/qsim.h)
    out = s.measure(3, seed=12345)
    assert out in (0, 1)
    s.close()
    z = q.State(4)
    with pytest.raises(q.QsimError) as e:
        z.measure_u(2, 1.0)
    assert e.value.code == q.QSIM_EZERONORM


def test_get_amplitudes_logical_indices():
    n, P = 14, 4
    circ = C.layered(n, 2, seed=2)
    ref = oracle.e_simulate(n, circ)
    with gpu_run(n, circ, ngpus=P) as s:
        idx = np.random.default_rng(0).integers(0, 1 << n, 3000, dtype=np.uint64)
        got = s.get_amplitudes(idx)
        assert np.max(np.abs(got - ref[idx.astype(np.int64)])) <= TOL
        assert s.qubit_map() != list(range(n))  # swaps were deferred, readout is logical


def test_swap_is_relabel_and_set_state():
    n = 11
    rng = np.random.default_rng(5)
    v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    v /= np.linalg.norm(v)
    with q.State(n) as s:
        s.set_state(v)
        s.apply_swap(0, 10)
        s.apply_gate(C.mat_H(), 10)
        ref = oracle.e_apply(oracle.e_swap(v.copy(), n, 0, 10), n, C.mat_H(), 10)
        assert np.max(np.abs(s.get_state() - ref)) <= TOL
        assert s.stats()["kernels"] >= 1


def test_errors():
    with pytest.raises(q.QsimError) as e:
        q.State(1)
    assert e.value.code == q.QSIM_EINVAL
    with pytest.raises(q.QsimError):
        q.State(12, q.ENC_FP64, 3)
    with pytest.raises(q.QsimError):
        q.State(12, q.ENC_FP64, 8)  # only 9 local qubits
    with q.State(5) as s:
        for bad in [lambda: s.apply_gate(C.mat_H(), 5), lambda: s.apply_gate(C.mat_H(), 1, [1]),
                    lambda: s.apply_gate(C.mat_X(), 0, [1, 1])]:
            with pytest.raises(q.QsimError) as e:
                bad()
            assert e.value.code == q.QSIM_EINVAL
        with pytest.raises(q.QsimError) as e:
            s.apply_gate(np.array([[1, 1], [0, 1]]), 0)
        assert e.value.code == q.QSIM_ENOTUNITARY
        assert np.max(np.abs(s.get_state() - oracle.e_init(5))) == 0  # failed calls changed nothing


# ----------------------------------------------------------------------------- full size (BASELINE configs)


@pytest.mark.slow
def test_full_size_h_wall_and_qft_n30():
    """N=30 (config 2 size): H wall and QFT closed forms on sampled amplitudes."""
    n = 30
    with q.State(n) as s:
        s.apply_circuit(C.h_wall(n))
        idx = np.random.default_rng(1).integers(0, 1 << n, 100000, dtype=np.uint64)
        assert np.max(np.abs(s.get_amplitudes(idx) - 2.0 ** (-n / 2))) <= 1e-15
        assert abs(s.norm() - 1) <= 1e-10
    circ, x = C.qft(n, seed=5)
    with q.State(n) as s:
        s.apply_circuit(circ)
        y = np.random.default_rng(2).integers(0, 1 << n, 100000, dtype=np.uint64)
        ph = ((np.uint64(x) * y) % np.uint64(1 << n)).astype(np.float64) * (2 * math.pi / (1 << n))
        assert np.max(np.abs(s.get_amplitudes(y) - 2.0 ** (-n / 2) * np.exp(1j * ph))) <= TOL
        assert np.max(np.abs(s.probabilities() - 0.5)) <= 1e-12


@pytest.mark.slow
def test_full_size_config2_product_state_pin():
    """Config 2 circuit at N=30 with the CNOTs removed (same U(2) draws): the
    product-state closed form Eq. appa2 on 10^5 sampled amplitudes, in the
    launch configuration bench.py times (fused passes)."""
    n = 30
    circ = C.layered(n, 20, seed=1, entangle=False)
    v = [np.array([1, 0], dtype=np.complex128) for _ in range(n)]
    for g in range(len(circ)):
        _, _, t, _, _, u = circ.gate(g)
        v[t] = u @ v[t]
    V = np.array(v)  # (n, 2)
    idx = np.random.default_rng(3).integers(0, 1 << n, 100000, dtype=np.uint64)
    bits = ((idx[:, None] >> np.arange(n, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(np.int64)
    ref = np.prod(V[np.arange(n)[None, :], bits], axis=1)
    with q.State(n) as s:
        s.apply_circuit(circ)
        assert np.max(np.abs(s.get_amplitudes(idx) - ref)) <= TOL
        assert abs(s.norm() - 1) <= 1e-10
        assert s.stats()["passes"] > 0


@pytest.mark.slow
def test_full_size_config2_vs_oracle_sampled():
    """Config 2 recipe at its full size N=30 (CNOTs kept, 2 of the 20 layers so
    the host oracle finishes in about a minute): GPU vs the oracle's full
    16 GiB state on 10^6 sampled amplitudes and the norm."""
    n = 30
    circ = C.layered(n, 2, seed=1)
    idx = np.random.default_rng(4).integers(0, 1 << n, 1000000, dtype=np.uint64)
    with q.State(n) as s:
        s.apply_circuit(circ)
        got = s.get_amplitudes(idx)
        nrm = s.norm()
    ref = oracle.e_simulate(n, circ)
    assert np.max(np.abs(got - ref[idx.astype(np.int64)])) <= TOL
    assert abs(nrm - 1) <= 1e-10


def _inverse(circ):
    """The inverse circuit: gates in reverse order, each U replaced by U^dagger
    (controls kept; SWAP is its own inverse)."""
    inv = C.Circuit(circ.n)
    for i in reversed(range(len(circ))):
        name, kind, t, t2, ctl, u = circ.gate(i)
        if kind == 1:
            inv.swap(t, t2)
        else:
            inv.add(name + "^dag", u.conj().T, t, ctl)
    return inv


@pytest.mark.slow
def test_full_size_config2_mirror_returns_to_zero():
    """The whole bench circuit (config 2: N=30, H wall + 20 layers, CNOTs
    kept, 930 gates, seed 1) in bench.py's launch configuration, then its
    inverse: U^dagger U = 1 returns the state to |0...0> at any size -- every
    fused pass of the timed step checked at full size (the oracle cannot run
    it): amplitude 0 and 10^5 sampled others, and the norm after each half."""
    n = 30
    circ = C.layered(n, 20, seed=1)
    assert len(circ) == 930
    with q.State(n) as s:
        s.apply_circuit(circ)
        assert abs(s.norm() - 1) <= 1e-10
        s.apply_circuit(_inverse(circ))
        idx = np.random.default_rng(8).integers(1, 1 << n, 100000, dtype=np.uint64)
        a0 = s.get_amplitudes(np.array([0], dtype=np.uint64))[0]
        assert abs(a0 - 1) <= 1e-10
        assert np.max(np.abs(s.get_amplitudes(idx))) <= 1e-12
        assert abs(s.norm() - 1) <= 1e-10
        assert s.stats()["passes"] > 0


@pytest.mark.slow
def test_max_size_config3_n33_product_pin_and_qft():
    """BASELINE config 3's per-GPU size (2^33 amplitudes = 128 GiB of HBM): the
    config-3 recipe (H wall + 10 layers of Haar U(2), CNOTs removed) against the
    product-state closed form (Eq. appa2) on 10^5 sampled amplitudes, then the
    QFT closed form at the same size (the largest E state one B200 holds)."""
    n = 33
    circ = C.layered(n, 10, seed=3, entangle=False)
    v = [np.array([1, 0], dtype=np.complex128) for _ in range(n)]
    for g in range(len(circ)):
        _, _, t, _, _, u = circ.gate(g)
        v[t] = u @ v[t]
    V = np.array(v)
    idx = np.random.default_rng(5).integers(0, 1 << n, 100000, dtype=np.uint64)
    bits = ((idx[:, None] >> np.arange(n, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(np.int64)
    ref = np.prod(V[np.arange(n)[None, :], bits], axis=1)
    with q.State(n) as s:
        s.apply_circuit(circ)
        assert np.max(np.abs(s.get_amplitudes(idx) - ref)) <= TOL
        assert abs(s.norm() - 1) <= 1e-10
        s.reset()
        qc, x = C.qft(n, seed=5)
        s.apply_circuit(qc)
        y = np.random.default_rng(6).integers(0, 1 << n, 100000, dtype=np.uint64)
        ph = ((np.uint64(x) * y) % np.uint64(1 << n)).astype(np.float64) * (2 * math.pi / (1 << n))
        assert np.max(np.abs(s.get_amplitudes(y) - 2.0 ** (-n / 2) * np.exp(1j * ph))) <= TOL
        assert np.max(np.abs(s.probabilities() - 0.5)) <= 1e-12


def test_nccl_transport_single_rank():
    """The NCCL transport with one rank on one GPU: communicator creation from a
    qsim_nccl_unique_id, and every collective read-out path (probabilities,
    expectations, amplitudes, state, measure; A bounds all-reduce)."""
    uid = q.qsim_nccl_unique_id()
    assert len(uid) == 128
    n = 14
    circ = C.config(0, seed=3)
    ref = oracle.e_simulate(n, circ)
    s = q.State(n, q.ENC_FP64, 1, transport=q.TRANSPORT_NCCL, rank=0, nccl_id=uid)
    s.apply_circuit(circ)
    assert np.max(np.abs(s.get_state() - ref)) <= TOL
    assert np.max(np.abs(s.probabilities() - oracle.e_probabilities(ref, n))) <= TOL
    assert np.max(np.abs(s.expectations() - oracle.e_expectations(ref, n))) <= TOL
    idx = np.arange(0, 1 << n, 7, dtype=np.uint64)
    assert np.max(np.abs(s.get_amplitudes(idx) - ref[idx.astype(np.int64)])) <= TOL
    with q.State(n) as loc:  # GENERATE EVENTS through the NCCL path: the same events as one shard
        loc.apply_circuit(circ)
        assert np.array_equal(s.sample(500, 9), loc.sample(500, 9))
    out, p0 = s.measure_u(2, 0.4)
    ro, rp0 = oracle.e_measure(ref, n, 2, 0.4)
    assert out == ro and abs(p0 - rp0) <= 1e-12
    s.close()
    a = q.State(12, q.ENC_ADAPTIVE2, 1, transport=q.TRANSPORT_NCCL, rank=0, nccl_id=q.qsim_nccl_unique_id())
    ca = C.rz_rx_cphase(12, 2, seed=4)
    a.apply_circuit(ca)
    codes, r0, r1 = a.get_codes()
    ra = oracle.AState(12).run(ca)
    assert r0 == pytest.approx(ra.r0, rel=1e-12) and r1 == pytest.approx(ra.r1, rel=1e-12)
    a.close()


@pytest.mark.parametrize("P", [1, 4])
def test_clear_set(P):
    """CLEAR / SET through qsim_project (incl. a global qubit when sharded)."""
    n = 12
    circ = C.config(0, n=n, seed=31)
    ref = oracle.e_simulate(n, circ)
    with gpu_run(n, circ, ngpus=P) as s:
        for qubit, value in [(0, 1), (11, 0), (6, 1)]:
            s.project(qubit, value)
            assert oracle.e_project(ref, n, qubit, value) == 0
            assert np.max(np.abs(s.get_state() - ref)) <= TOL
        with pytest.raises(q.QsimError) as e:
            s.project(0, 0)  # qubit 0 is already |1>
        assert e.value.code == q.QSIM_EZERONORM
        assert np.max(np.abs(s.get_state() - ref)) <= TOL


def test_too_large_state_is_enomem():
    with pytest.raises(q.QsimError) as e:
        q.State(40)  # 16 TiB
    assert e.value.code == q.QSIM_ENOMEM


@pytest.mark.parametrize("P", [1, 4])
def test_generate_events(P):
    """GENERATE EVENTS on the GPU == the oracle's inverse CDF for the same
    counter-based draws (up to draws within 1e-12 of a CDF boundary), in
    logical order even after deferred swaps."""
    n = 13
    circ = C.layered(n, 2, seed=8)
    circ.swap(0, 12)
    ref = oracle.e_simulate(n, circ)
    with gpu_run(n, circ, ngpus=P) as s:
        got = s.sample(20000, seed=99)
        assert s.qubit_map() != list(range(n))
        st = s.get_state()
    assert np.max(np.abs(st - ref)) <= TOL  # sampling leaves the state unchanged
    u = C.splitmix_uniform(99, 20000)
    want = oracle.e_sample(ref, n, u)
    cum = np.cumsum(np.abs(ref) ** 2)
    near = np.abs(cum[want.astype(np.int64)] - u * cum[-1]) < 1e-12
    assert np.all((got == want) | near)


@pytest.mark.parametrize("P", [1, 4])
def test_shorbox_vs_oracle(P):
    n, nx, G, y = 12, 7, 21, 2
    ref = oracle.e_shorbox(n, nx, G, y)
    with q.State(n, q.ENC_FP64, P) as s:
        s.apply_circuit(C.layered(n, 1, seed=1))  # any prior state is replaced
        s.prepare_shorbox(nx, G, y)
        assert np.max(np.abs(s.get_state() - ref)) == 0
        s.apply_circuit(C.qft_register(n, nx))
        assert np.max(np.abs(s.get_state() - oracle.e_run(ref, n, C.qft_register(n, nx)))) <= TOL


def _table5():
    import os
    rows = [l.split() for l in open(os.path.join(os.path.dirname(__file__), "golden", "table5_shor.txt"))
            if l.strip() and not l.startswith("#")]
    return np.array(rows, dtype=float)


@pytest.mark.slow
def test_table5_shor_n30_exact_columns():
    """PAPER.md Table 5 (lines 939-979): Shor, N=30, G=1007, y=529, 20-qubit
    x-register: SHORBOX + QFT, per-qubit expectations equal the printed exact
    closed-form columns (3 decimals); the E results are numerically exact
    ("The expectation values produced by E are numerically exact")."""
    t = _table5()
    with q.State(30) as s:
        s.prepare_shorbox(20, 1007, 529)
        s.apply_circuit(C.qft_register(30, 20))
        e = s.expectations()[:20]
    # <Qz>: the printed exact column to its 3 printed decimals
    assert np.max(np.abs(e[:, 2] - t[:, 6])) <= 5e-4 + 1e-12
    # <Qx>, <Qy>: printed as 0.500; the full state gives up to 0.5058 (qubit 5),
    # between the printed exact and A columns (reading R-B6) -- bounded by the
    # paper's own A-vs-exact level 0.011
    assert np.max(np.abs(e[:, :2] - t[:, 4:6])) <= 0.011


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3, 5, 7])
def test_small_states_below_256_amplitudes(n):
    """N < 8: shards are zero-padded to 256 amplitudes; every read-out still
    covers exactly the 2^N logical amplitudes."""
    circ = C.config(0, n=n, seed=n, layers=None) if n >= 3 else C.h_wall(n)
    ref = oracle.e_simulate(n, circ)
    with q.State(n) as s:
        s.apply_circuit(circ)
        assert np.max(np.abs(s.get_state() - ref)) <= TOL
        assert abs(s.norm() - 1.0) <= 1e-10
        assert np.max(np.abs(s.probabilities() - oracle.e_probabilities(ref, n))) <= TOL
        assert np.max(np.abs(s.expectations() - oracle.e_expectations(ref, n))) <= TOL



@pytest.mark.parametrize("fuse", [0, 1])
@pytest.mark.parametrize("P", [1, 2])
def test_graph_replay_applies_the_captured_circuit(fuse, P):
    """qsim_graph_*: capturing a config-1 circuit runs nothing; each replay
    applies the circuit again to the current state (oracle: the circuit
    applied once, then three times).  P = 2 (loopback shards): the circuit
    avoids the global qubit, so the capture leaves the map unchanged."""
    n = 14
    if P == 1:
        circ = C.config(0, seed=3)
    else:
        circ, sub = C.Circuit(n), C.random_circuit(n - 1, 200, seed=3)
        for i in range(len(sub)):
            name, kind, t, t2, ctl, u = sub.gate(i)
            circ.add(name, u, t, ctl)
    s = q.State(n, q.ENC_FP64, P, fuse=fuse)
    g = s.capture(lambda st: st.apply_circuit(circ))
    assert np.array_equal(s.get_state(), oracle.e_init(n))  # capturing ran nothing
    g.launch()
    ref = oracle.e_simulate(n, circ)
    assert np.max(np.abs(s.get_state() - ref)) <= TOL
    g.launch()
    g.launch()
    for _ in range(2):
        ref = oracle.e_run(ref.copy(), n, circ)
    assert np.max(np.abs(s.get_state() - ref)) <= TOL
    g.close()
    s.close()


def test_graph_capture_rejects_layout_changes_and_readouts():
    """A capture whose gates move a qubit across the shard boundary (an
    exchange changes the qubit map) cannot be replayed: EUNSUPPORTED; read-out
    calls inside a capture: EINVAL; A encoding: EUNSUPPORTED."""
    n = 12
    s = q.State(n, q.ENC_FP64, 2)
    with pytest.raises(q.QsimError) as e:
        s.capture(lambda st: st.apply_gate(C.mat_H(), n - 1))
    assert e.value.code == -7
    s.reset()
    with pytest.raises(q.QsimError) as e:
        s.capture(lambda st: st.norm())
    assert e.value.code == -1
    s.reset()
    assert abs(s.norm() - 1.0) <= 1e-15  # the handle is usable after a failed capture
    s.close()
    a = q.State(n, q.ENC_ADAPTIVE2, 1)
    with pytest.raises(q.QsimError) as e:
        a.capture(lambda st: st.apply_gate(C.mat_H(), 0))
    assert e.value.code == -7
    a.close()


@pytest.mark.parametrize("P", [4, 8])
def test_all_to_all_remap_loopback(P, monkeypatch):
    """NEXT-1 (i): a config-3 shaped circuit (every layer hits all global
    qubits with dense gates) on P loopback shards: the plan holds all-to-all
    remaps; the state equals the oracle's, and the remaps move fewer bytes
    than the pairwise exchanges of the same circuit (QSIM_NO_REMAP=1)."""
    n = 14
    circ = C.layered(n, 3, seed=3)
    ref = oracle.e_simulate(n, circ)
    with q.State(n, q.ENC_FP64, P) as s:
        s.apply_circuit(circ)
        assert np.max(np.abs(s.get_state() - ref)) <= TOL
        st = s.stats()
    monkeypatch.setenv("QSIM_NO_REMAP", "1")
    with q.State(n, q.ENC_FP64, P) as s:
        s.apply_circuit(circ)
        assert np.max(np.abs(s.get_state() - ref)) <= TOL
        st0 = s.stats()
    assert st["exchanges"] < st0["exchanges"]
    assert st["exchange_bytes"] < st0["exchange_bytes"]


def _run_n22(mode, tmp_path, recipe="C.layered(n, 3, seed=1)", n=22, extra_env=None):
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / f"state_{mode}_{abs(hash(str(extra_env)))}.npy")
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1805_04708_b200 as q, qsim_inputs as C; "
            "n = %d; s = q.State(n, q.ENC_FP64, 1); s.apply_circuit(%s); st = s.stats(); "
            "np.save(%r, s.get_state()); print(st['jit_passes'], st['passes'])" % (root, n, recipe, out))
    env = dict(os.environ, QSIM_LPASS_JIT=str(mode), **(extra_env or {}))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    jit, passes = (int(x) for x in r.stdout.split()[-2:])
    return np.load(out), jit, passes


def test_specialised_pass_kernels_match_the_interpreter_and_the_oracle(tmp_path):
    """The run-time specialised pass kernels (NVRTC, QSIM_LPASS_JIT=2: compiled
    before their first launch) run every pass of a config-2 shaped circuit at
    N = 22 (1024 tiles); the state equals the interpreter's (QSIM_LPASS_JIT=0)
    and the oracle's."""
    a, jit, passes = _run_n22(2, tmp_path)
    b, jit0, passes0 = _run_n22(0, tmp_path)
    assert passes > 0 and jit == passes and jit0 == 0 and passes0 == passes
    assert np.max(np.abs(a - b)) <= 1e-14
    ref = oracle.e_simulate(22, C.layered(22, 3, seed=1))
    assert np.max(np.abs(a - ref)) <= TOL


@pytest.mark.parametrize("recipe,n", [("C.qft(n, seed=5)[0]", 20), ("C.random_circuit(n, 400, seed=11)", 16),
                                      ("C.config(3, n=n)", 18)])
def test_specialised_kernels_with_phase_ops_match_the_oracle(tmp_path, recipe, n):
    """Specialised pass kernels compiled before their first launch
    (QSIM_LPASS_JIT=2) on programs with DIAG1 / PHASES ops (QFT ladders,
    controlled phases with outside controls, random gate mixes, the config-4
    recipe in E): the state equals the interpreter's and the oracle's."""
    circ = eval(recipe, {"C": C, "n": n})
    ref = oracle.e_simulate(n, circ)
    for hoist in ("1", "0"):  # per-tile hoisting forced on (auto: off below 1024 tiles) and off
        a, jit, passes = _run_n22(2, tmp_path, recipe, n, {"LPASS_HOIST": hoist})
        b, jit0, _ = _run_n22(0, tmp_path, recipe, n, {"LPASS_HOIST": hoist})
        assert passes > 0 and jit == passes and jit0 == 0
        assert np.max(np.abs(a - b)) <= 1e-14
        assert np.max(np.abs(a - ref)) <= TOL


@pytest.mark.parametrize("knob", [{"QSIM_LPASS_G": "2"}, {"QSIM_LPASS_NT": "256"}, {"QSIM_LPASS_PREFETCH": "1"},
                                  {"QSIM_LPASS_STAGE_ASM": "0"}, {"QSIM_LPASS_MINB": "2"}])
def test_specialised_kernel_variants_match_the_oracle(tmp_path, knob):
    """The measured-and-rejected build variants of the specialised pass kernel
    (two register groups per thread, 256 threads per CTA, L2 prefetch of the
    next tile, plain C++ stage accesses, 2 CTAs per SM -- DESIGN.md §7, the
    environment knobs) still compute the same states: config-3 recipe and the
    QFT at N = 20, every pass specialised, vs the oracle."""
    for recipe in ("C.config(2, n=n)", "C.qft(n, seed=5)[0]"):
        a, jit, passes = _run_n22(2, tmp_path, recipe, 20, knob)
        assert passes > 0 and jit == passes
        circ = eval(recipe, {"C": C, "n": 20})
        assert np.max(np.abs(a - oracle.e_simulate(20, circ))) <= TOL


@pytest.mark.parametrize("hoist", ["1", "0"])
@pytest.mark.parametrize("recipe,n,P", [("C.config(0, n=n, seed=3)", 14, 1), ("C.config(2, n=n)", 20, 1),
                                        ("C.qft(n, seed=5)[0]", 20, 1), ("C.random_circuit(n, 400, seed=11)", 16, 1),
                                        ("C.config(3, n=n)", 18, 4), ("C.config(2, n=n)", 19, 2)])
def test_bounds_checked_pass_kernels(tmp_path, recipe, n, P, hoist):
    """compute-sanitizer is closed on the GPU pool, so the specialised pass
    kernels have a checked build of their own (QSIM_LPASS_CHECK=1, LP_CHECK in
    lpass_dev.cuh): every shared-memory slot, table and coefficient-pool read
    and every HBM run of a tile is asserted in range (a violation traps and
    the process fails).  Small shards, the config-3/4 recipes, QFT ladders
    (hoisted terms, tile scalars -- forced on with LPASS_HOIST=1 at these sizes,
    and off), random gate mixes, and sharded loopback states (shard bits in
    the full index); results vs the oracle."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "state.npy")
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1805_04708_b200 as q, qsim_inputs as C; "
            "n = %d; s = q.State(n, q.ENC_FP64, %d); s.apply_circuit(%s); q.qsim_jit_sync(); st = s.stats(); "
            "np.save(%r, s.get_state()); print(st['jit_passes'], st['passes'])" % (root, n, P, recipe, out))
    env = dict(os.environ, QSIM_LPASS_JIT="2", QSIM_LPASS_CHECK="1", QSIM_JIT_DISK_CACHE="0", LPASS_HOIST=hoist)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "lpass check failed" not in r.stdout + r.stderr, r.stdout + r.stderr
    jit, passes = (int(x) for x in r.stdout.split()[-2:])
    assert passes > 0 and jit == passes
    circ = eval(recipe, {"C": C, "n": n})
    assert np.max(np.abs(np.load(out) - oracle.e_simulate(n, circ))) <= TOL


@pytest.mark.parametrize("P", [1, 4])
def test_reset_basis_is_the_x_prepared_state(P):
    """qsim_reset_basis(x): the basis state X on the set bits of x makes from
    |0...0> (config 5's input |x>); the QFT from it equals the oracle's QFT of
    the X-prepared state, and the closed form 2^{-N/2} e^{2 pi i x y / 2^N}."""
    n = 16
    circ, x = C.qft(n, seed=7)
    core = C.qft_register(n, n)
    assert len(circ) == len(core) + bin(x).count("1")
    ref = oracle.e_simulate(n, circ)
    with q.State(n, q.ENC_FP64, P) as s:
        s.reset_basis(x)
        basis = s.get_state()
        assert basis[x] == 1.0 and np.count_nonzero(basis) == 1
        s.apply_circuit(core)
        got = s.get_state()
        assert np.max(np.abs(got - ref)) <= TOL
        y = np.arange(1 << n)
        closed = np.exp(2j * np.pi * ((x * y) % (1 << n)) / (1 << n)) / 2 ** (n / 2)
        assert np.max(np.abs(got - closed)) <= TOL
        s.reset_basis(0)
        z = s.get_state()
        assert z[0] == 1.0 and np.count_nonzero(z) == 1
        with pytest.raises(q.QsimError):
            s.reset_basis(1 << n)
    # A: the same codes as the X-prepared state (X moves codes)
    xs = C.Circuit(n)
    for b in range(n):
        if (x >> b) & 1:
            xs.add("X", C.mat_X(), b)
    with q.State(n, q.ENC_ADAPTIVE2, P) as a, q.State(n, q.ENC_ADAPTIVE2, P) as b:
        a.reset_basis(x)
        b.apply_circuit(xs)
        assert np.array_equal(a.get_codes()[0], b.get_codes()[0])


@pytest.mark.parametrize("enc", ["E", "A"])
@pytest.mark.parametrize("P", [1, 4])
def test_empty_inputs_and_smallest_states(enc, P):
    """Degenerate inputs: an empty circuit leaves |0...0> (and the stats at
    zero gates), an empty index list reads nothing, zero samples draw nothing;
    the smallest states (N = 2, and the smallest sharded N = 10 + log2 P) run
    a circuit equal to the oracle's."""
    e = q.ENC_FP64 if enc == "E" else q.ENC_ADAPTIVE2
    n = 10 + int(math.log2(P)) if P > 1 else 2
    with q.State(n, e, P) as s:
        s.apply_circuit(C.Circuit(n))
        z = s.get_state()
        assert z[0] == 1.0 and np.count_nonzero(z) == 1
        assert s.stats()["gates"] == 0
        assert s.get_amplitudes(np.array([], dtype=np.uint64)).size == 0
        assert s.sample(0, 1).size == 0
        if enc == "E":
            kinds = tuple(k for k in C.CFG1_KINDS if k != "TOFFOLI") if n < 3 else C.CFG1_KINDS
            circ = C.random_circuit(n, 60, seed=n + P, kinds=kinds)
        else:  # H wall, a CNOT, phases, X: codes equal to the oracle-A's
            circ = C.h_wall(n)
            circ.add("CNOT", C.mat_X(), n - 1, [0])
            circ.add("T", C.mat_T(), 1)
            circ.add("Z", C.mat_Z(), n - 1)
            circ.add("X", C.mat_X(), 0)
        s.apply_circuit(circ)
        got = s.get_state()
        codes = s.get_codes()[0] if enc == "A" else None
    if enc == "E":
        assert np.max(np.abs(got - oracle.e_simulate(n, circ))) <= TOL
    else:  # decoded amplitudes equal the oracle-A's within one step (the codes themselves
        # may differ where every magnitude ties: degenerate bounds r0 = r1 decided by an ulp)
        ra = oracle.AState(n).run(circ)
        zr = ra.decoded()
        step = (ra.r1 - ra.r0) / 253.0
        assert codes.size == 2 << n
        assert np.max(np.abs(np.abs(got) - np.abs(zr))) <= step + 1e-12
        both = (np.abs(got) > 0) & (np.abs(zr) > 0)
        assert np.all(np.abs(np.angle(got[both] * np.conj(zr[both]))) <= math.pi / 128 + 1e-12)


@pytest.mark.parametrize("enc,P", [("E", 1), ("E", 4), ("A", 1), ("A", 2)])
def test_repeated_runs_are_bit_identical(enc, P):
    """A race detector by determinism (compute-sanitizer's racecheck is closed
    on the pool): every kernel's arithmetic and every reduction here has a
    fixed order (the A bounds are exact extremes, order-free), so the same
    circuit run again from |0...0> must give the same bits -- a shared-memory
    race in the tile pass, the exchange or the A kernels' warp queues would
    show up as run-to-run differences.  Four runs, states / codes and
    probabilities compared bit for bit."""
    n = 22 if enc == "E" else 18
    e = q.ENC_FP64 if enc == "E" else q.ENC_ADAPTIVE2
    circ = C.config(2, n=n) if enc == "E" else C.config(3, n=n)
    gates = q.pack_gates(circ)
    outs = []
    with q.State(n, e, P) as s:
        s.apply_circuit(gates)  # warm-up: the pass specialisations it queues are ready below
        s.sync()
        q.qsim_jit_sync()
        for _ in range(4):
            s.reset()
            s.apply_circuit(gates)
            st = s.get_codes()[0] if enc == "A" else s.get_state()
            outs.append((st, s.probabilities()))
    for st, pr in outs[1:]:
        assert np.array_equal(st, outs[0][0]) and np.array_equal(pr, outs[0][1])


def _apply_matrix_ref(psi, n, U, qubits):
    """Test-side reference: U (2^k x 2^k, qubits[0] the most significant index)
    on a logical state vector (numpy; bit j of the index = qubit j)."""
    k = len(qubits)
    t = psi.reshape((2,) * n)  # axis a <-> qubit n-1-a
    axes = [n - 1 - q for q in qubits]
    Ut = U.reshape((2,) * (2 * k))
    out = np.tensordot(Ut, t, axes=(list(range(k, 2 * k)), axes))
    # tensordot puts the k output axes first, in qubits order; move them back
    out = np.moveaxis(out, list(range(k)), axes)
    return out.reshape(-1)


def test_apply_matrix_pins_and_random_unitaries():
    """qsim_apply_matrix (SPEC apply_two / apply_three): kron(A, B) on
    (q1, q0) equals A on q1 then B on q0; the 8x8 Toffoli matrix equals the
    Toffoli gate; Haar 4x4 / 8x8 on a random state equal the test-side
    tensor contraction; P = 2 loopback with a qubit on the global bit."""
    n = 9
    rng = np.random.default_rng(21)
    A, B = C.mat_haar(rng), C.mat_haar(rng)
    circ = C.Circuit(n)
    circ.add("Haar", A, 5)
    circ.add("Haar", B, 2)
    with q.State(n, q.ENC_FP64, 1) as s:
        s.apply_matrix(np.kron(A, B), [5, 2])
        assert np.max(np.abs(s.get_state() - oracle.e_simulate(n, circ))) <= TOL
    tof = np.eye(8, dtype=complex)
    tof[[6, 7]] = tof[[7, 6]]
    with q.State(n, q.ENC_FP64, 1) as s:
        s.apply_circuit(C.h_wall(n))
        s.apply_gate(C.mat_Rz(0.3), 7)
        s.apply_matrix(tof, [7, 3, 1])  # controls 7, 3 (matrix MSBs), target 1
        ref = oracle.e_run(oracle.e_simulate(n, C.h_wall(n)).copy(), n, _one(n, "Rz", C.mat_Rz(0.3), 7))
        ref = oracle.e_run(ref, n, _one(n, "TOFFOLI", C.mat_X(), 1, [7, 3]))
        assert np.max(np.abs(s.get_state() - ref)) <= TOL
    n = 11  # sharded states need >= 10 local qubits; qubit 10 is global at P = 2
    psi = rng.normal(size=2 ** n) + 1j * rng.normal(size=2 ** n)
    psi /= np.linalg.norm(psi)
    for k, qs in ((2, [3, 10]), (3, [0, 10, 4]), (1, [10]), (3, [9, 2, 6])):
        z = rng.normal(size=(2 ** k, 2 ** k)) + 1j * rng.normal(size=(2 ** k, 2 ** k))
        U, _ = np.linalg.qr(z)
        for P in (1, 2):
            with q.State(n, q.ENC_FP64, P) as s:
                s.set_state(psi)
                s.apply_matrix(U, qs)
                assert np.max(np.abs(s.get_state() - _apply_matrix_ref(psi, n, U, qs))) <= TOL


def _one(n, name, u, t, ctl=()):
    c = C.Circuit(n)
    c.add(name, u, t, list(ctl))
    return c


def test_apply_matrix_errors():
    with q.State(6, q.ENC_FP64, 1) as s:
        with pytest.raises(q.QsimError) as e:
            s.apply_matrix(np.eye(16), [0, 1, 2, 3])
        assert e.value.code == -1
        with pytest.raises(q.QsimError) as e:
            s.apply_matrix(np.eye(4), [1, 1])
        assert e.value.code == -1
        with pytest.raises(q.QsimError) as e:
            s.apply_matrix(np.ones((4, 4)), [0, 1])
        assert e.value.code == q.QSIM_ENOTUNITARY
    with q.State(6, q.ENC_ADAPTIVE2, 1) as a:
        with pytest.raises(q.QsimError) as e:
            a.apply_matrix(np.eye(4), [0, 1])
        assert e.value.code == -7


@pytest.mark.parametrize("enc", ["E", "A"])
@pytest.mark.parametrize("n,P", [(13, 8), (14, 16)])
def test_remap_pack_unpack_path(tmp_path, enc, n, P):
    """The NCCL remap's data flow on one GPU (QSIM_REMAP_VIA_PACK=1: chunked
    multi-partner pack -> device copies standing in for ncclSend / ncclRecv
    -> multi-partner unpack, small chunks so every block takes several
    rounds): E equals the oracle, A equals the single-shard run bit for bit;
    P = 16 (4 global qubits) exercises remaps split into groups of <= 3 bits."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / f"r_{enc}_{P}.npy")
    getter = "s.get_state()" if enc == "E" else "s.get_codes()[0]"
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1805_04708_b200 as q, qsim_inputs as C; "
            "s = q.State(%d, q.ENC_%s, %d, chunk_bytes=2048); c = C.layered(%d, 2, seed=7); "
            "c.extend(C.rz_rx_cphase(%d, 1, seed=7)); s.apply_circuit(c); st = s.stats(); np.save(%r, %s); "
            "print(st['exchanges'])" % (root, n, "FP64" if enc == "E" else "ADAPTIVE2", P, n, n, out, getter))
    env = dict(os.environ, QSIM_REMAP_VIA_PACK="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert int(r.stdout.split()[-1]) > 0
    got = np.load(out)
    circ = C.layered(n, 2, seed=7)
    circ.extend(C.rz_rx_cphase(n, 1, seed=7))
    ops, _ = q.qsim_plan(n, P, circ)
    assert sum(o["type"] == q.OP_REMAP for o in ops) > 0
    if enc == "E":
        assert np.max(np.abs(got - oracle.e_simulate(n, circ))) <= TOL
    else:
        with q.State(n, q.ENC_ADAPTIVE2, 1) as s1:
            s1.apply_circuit(circ)
            assert np.array_equal(got, s1.get_codes()[0])


def test_program_cache_replay_is_identical():
    """A circuit applied again replays the host compiler's recorded pass
    programs (api.cu program cache): same state bit for bit, equal to the
    oracle; sharded states (the key includes shard 0's global bits) too."""
    n = 14
    c = C.config(0, seed=9)
    ref = oracle.e_simulate(n, c)
    for P in (1, 4):
        with q.State(n, q.ENC_FP64, P) as s:
            s.apply_circuit(c)
            a = s.get_state()
            s.reset()
            s.apply_circuit(c)
            b = s.get_state()
        assert np.array_equal(a, b), P
        assert np.max(np.abs(a - ref)) <= TOL, P
    # more distinct gate lists than the cache holds (64): the first is
    # evicted and compiled again, the last still replays
    circs = [C.random_circuit(n, 30, seed=1000 + k) for k in range(70)]
    with q.State(n) as s:
        for cc in circs:
            s.reset()
            s.apply_circuit(cc)
        for cc in (circs[0], circs[-1]):
            s.reset()
            s.apply_circuit(cc)
            assert np.max(np.abs(s.get_state() - oracle.e_simulate(n, cc))) <= TOL


def test_jit_shutdown_then_interpreter(tmp_path):
    """qsim_jit_shutdown stops the compile threads; later passes run in the
    interpreter with the same results, and the process exits cleanly."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "s.npy")
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1805_04708_b200 as q, qsim_inputs as C; "
            "n = 14; c = C.config(0, seed=4); s = q.State(n, q.ENC_FP64, 1); s.apply_circuit(c); s.sync(); "
            "q.qsim_jit_sync(); s.reset(); s.reset_stats(); s.apply_circuit(c); s.sync(); "
            "j1 = s.stats()['jit_passes']; "
            "q.qsim_jit_shutdown(); s.reset(); s.reset_stats(); s.apply_circuit(c); np.save(%r, s.get_state()); "
            "print(j1, s.stats()['jit_passes'])" % (root, out))
    ref = oracle.e_simulate(14, C.config(0, seed=4))
    for mode in ("1", "2"):  # compile in the background / before the first launch
        env = dict(os.environ, QSIM_LPASS_JIT=mode)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env)
        assert r.returncode == 0, r.stderr
        j1, j2 = (int(x) for x in r.stdout.split()[-2:])
        assert j1 > 0 and j2 == 0, (mode, j1, j2)  # specialised before the shutdown, interpreted after
        assert np.max(np.abs(np.load(out) - ref)) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("enc", ["E", "A"])
def test_exchange_comm_pipeline_path(tmp_path, enc):
    """The NCCL pairwise exchange's pipeline on one GPU (QSIM_XCHG_VIA_COMM=1:
    comm stream, double-buffered receive buffers, events; device copies stand
    in for ncclSend / ncclRecv; QSIM_NO_REMAP=1 so every global gate takes a
    pairwise exchange; small chunks so each exchange takes many rounds): E
    equals the oracle, A equals the single-shard run bit for bit."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    n = 13
    for P in (2, 4):
        out = str(tmp_path / f"x_{enc}_{P}.npy")
        getter = "s.get_state()" if enc == "E" else "s.get_codes()[0]"
        code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1805_04708_b200 as q, qsim_inputs as C; "
                "s = q.State(%d, q.ENC_%s, %d, chunk_bytes=2048); c = C.layered(%d, 2, seed=8); "
                "c.extend(C.rz_rx_cphase(%d, 1, seed=8)); s.apply_circuit(c); st = s.stats(); np.save(%r, %s); "
                "print(st['exchanges'])" % (root, n, "FP64" if enc == "E" else "ADAPTIVE2", P, n, n, out, getter))
        env = dict(os.environ, QSIM_XCHG_VIA_COMM="1", QSIM_NO_REMAP="1")
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        assert int(r.stdout.split()[-1]) > 0
        got = np.load(out)
        circ = C.layered(n, 2, seed=8)
        circ.extend(C.rz_rx_cphase(n, 1, seed=8))
        if enc == "E":
            assert np.max(np.abs(got - oracle.e_simulate(n, circ))) <= TOL
        else:
            with q.State(n, q.ENC_ADAPTIVE2, 1) as s1:
                s1.apply_circuit(circ)
                assert np.array_equal(got, s1.get_codes()[0])
