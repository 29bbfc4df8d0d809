"""GPU parity for the A path (adaptive 2-byte encoding, §4.1) through
the C-ABI.  Bar (BASELINE.json north_star): decoded amplitudes within one
quantisation step of the oracle's own implementation of the encoding --
|delta r| <= (r1 - r0)/253 and |delta theta| <= pi/128 (+1e-12 absolute for
fp64 rounding) -- checked per gate from identical
seeded input codes; whole circuits report the within-one-step fraction and
the fidelity against the oracle-A and against E."""
import math

import numpy as np
import pytest

import oracle
import qsim_inputs as C

pytestmark = pytest.mark.gpu
q = pytest.importorskip("paper_1805_04708_b200")


def seeded_codes(n, seed):
    codes, r0, r1 = C.random_codes(n, seed)
    codes[2 * 1] = -127  # make the extreme magnitude codes present: bounds are exact min / max
    codes[2 * 2] = 126
    return codes, r0, r1


def within_one_step(z_gpu, z_ref, r0, r1):
    step = (r1 - r0) / 253.0
    dm = np.abs(np.abs(z_gpu) - np.abs(z_ref))
    ok_m = dm <= step + 1e-12
    both = (np.abs(z_gpu) > 0) & (np.abs(z_ref) > 0)
    dth = np.abs(np.angle(z_gpu * np.conj(z_ref)))
    ok_t = ~both | (dth <= math.pi / 128 + 1e-12)
    return ok_m & ok_t


def code_diff(cg, co):
    b0 = np.abs(cg[0::2].astype(int) - co[0::2].astype(int))
    d1 = np.abs(cg[1::2].astype(int) - co[1::2].astype(int)) % 256
    b1 = np.minimum(d1, 256 - d1)
    zero = (cg[0::2] == -128) & (co[0::2] == -128)
    return np.where(zero, 0, b0), np.where(zero, 0, b1)


GATES = [("H", C.mat_H(), ()), ("Haar", C.mat_haar(np.random.default_rng(0)), ()), ("Rx", C.mat_Rx(1.3), ()),
         ("CH", C.mat_H(), (1,)), ("CCU", C.mat_haar(np.random.default_rng(1)), (1, 2)),
         ("X", C.mat_X(), ()), ("Y", C.mat_Y(), ()), ("CNOT", C.mat_X(), (1,)), ("TOF", C.mat_X(), (1, 2)),
         ("Z", C.mat_Z(), ()), ("T", C.mat_T(), ()), ("Rz", C.mat_Rz(0.77), ()), ("CP", C.mat_U1(2.1), (1,))]


@pytest.mark.parametrize("name,u,ctl", GATES, ids=[g[0] for g in GATES])
@pytest.mark.parametrize("t", [0, 3, 4, 9, 11])
def test_per_gate_from_identical_codes(name, u, ctl, t):
    n = 12
    ctl = tuple((c + t + 1) % n if (c + t + 1) % n != t else (c + t + 2) % n for c in ctl)
    codes, r0, r1 = seeded_codes(n, seed=t * 31 + len(name))
    ref = oracle.AState(n, codes, r0, r1)
    ref.apply(u, t, ctl)
    with q.State(n, q.ENC_ADAPTIVE2) as s:
        s.set_codes(codes, r0, r1)
        s.apply_gate(u, t, ctl)
        cg, g0, g1 = s.get_codes()
        zg = s.get_state()
    assert g0 == pytest.approx(ref.r0, rel=1e-12, abs=1e-300) and g1 == pytest.approx(ref.r1, rel=1e-12)
    db0, db1 = code_diff(cg, ref.codes)
    assert db0.max() <= 1 and db1.max() <= 1
    assert within_one_step(zg, ref.decoded(), ref.r0, ref.r1).all()
    # codes agree exactly except at rounding ties (a vanishing fraction)
    assert np.mean((db0 == 0) & (db1 == 0)) >= 0.999


def test_paper_workloads_exact_in_a():
    """Tables 2-3 captions: H wall and GHZ are exact in A."""
    for n, circ, ref in [(14, C.h_wall(14), None), (13, C.ghz_chain(13), None)]:
        e = oracle.e_simulate(n, circ)
        with q.State(n, q.ENC_ADAPTIVE2) as s:
            s.apply_circuit(circ)
            assert np.max(np.abs(s.get_state() - e)) <= 1e-15
            cg, _, _ = s.get_codes()
            assert np.array_equal(cg, oracle.AState(n).run(circ).codes)


def test_permutation_circuit_bit_exact():
    n = 12
    rng = np.random.default_rng(8)
    circ = C.Circuit(n)
    for _ in range(80):
        a, b, c = [int(v) for v in rng.choice(n, 3, replace=False)]
        k = rng.integers(5)
        if k == 0:
            circ.add("X", C.mat_X(), a)
        elif k == 1:
            circ.add("CNOT", C.mat_X(), b, [a])
        elif k == 2:
            circ.add("TOF", C.mat_X(), c, [a, b])
        elif k == 3:
            circ.add("S", C.mat_S(), a)
        else:
            circ.swap(a, b)
    ref = oracle.AState(n).run(circ)
    for P in (1, 4):
        with q.State(n, q.ENC_ADAPTIVE2, P) as s:
            s.apply_circuit(circ)
            cg, _, _ = s.get_codes()
            assert np.array_equal(cg, ref.codes)


@pytest.mark.parametrize("P", [1, 2, 8])
def test_whole_circuit_config4_shape(P):
    """Config 4 recipe (H wall, Rz/Rx coin flips, CPHASE matching) at N=13:
    within-one-step fraction and fidelity vs the oracle-A; fidelity vs E."""
    n = 13
    circ = C.rz_rx_cphase(n, 4, seed=4)
    ref = oracle.AState(n).run(circ)
    e = oracle.e_simulate(n, circ)
    with q.State(n, q.ENC_ADAPTIVE2, P) as s:
        s.apply_circuit(circ)
        zg = s.get_state()
        _, g0, g1 = s.get_codes()
    zr = ref.decoded()
    frac = within_one_step(zg, zr, ref.r0, ref.r1).mean()
    fid_or = abs(np.vdot(zr, zg)) ** 2 / (np.vdot(zg, zg).real * np.vdot(zr, zr).real)
    fid_e = abs(np.vdot(e, zg)) ** 2 / (np.vdot(zg, zg).real * np.vdot(e, e).real)
    assert frac >= 0.99
    assert fid_or >= 0.999
    assert fid_e >= 0.95


def test_sharding_is_bit_exact_in_a():
    """Bounds are exact global min / max, so the A codes do not depend on P."""
    n = 13
    circ = C.rz_rx_cphase(n, 3, seed=5)
    circ.extend(C.layered(n, 1, seed=5, h_first=False))
    out = []
    for P in (1, 2, 4, 8):
        with q.State(n, q.ENC_ADAPTIVE2, P) as s:
            s.apply_circuit(circ)
            out.append(s.get_codes())
    for c, r0, r1 in out[1:]:
        assert np.array_equal(c, out[0][0]) and r0 == out[0][1] and r1 == out[0][2]


def test_global_relabel_is_bit_exact_in_a():
    """Relabelled permutation gates move A codes exactly:
    codes with global permutations are the same for P = 1 and P = 8."""
    n = 13
    circ = C.rz_rx_cphase(n, 2, seed=7)
    circ.extend(C.global_permutations(n, 8, seed=7))
    circ.extend(C.rz_rx_cphase(n, 1, seed=8))
    out = []
    for P in (1, 8):
        with q.State(n, q.ENC_ADAPTIVE2, P) as s:
            s.apply_circuit(circ)
            out.append(s.get_codes())
    c8, r0, r1 = out[1]
    assert np.array_equal(c8, out[0][0]) and r0 == out[0][1] and r1 == out[0][2]


def test_a_readout_and_measure():
    n = 12
    circ = C.rz_rx_cphase(n, 2, seed=6)
    ref = oracle.AState(n).run(circ)
    z = ref.decoded()
    with q.State(n, q.ENC_ADAPTIVE2, 2) as s:
        s.apply_circuit(circ)
        zg = s.get_state()
        assert within_one_step(zg, z, ref.r0, ref.r1).mean() >= 0.99
        qe = s.expectations()
        assert np.max(np.abs(qe - oracle.e_expectations(zg, n))) <= 1e-12  # GPU reductions of its own decoded state
        assert abs(s.norm() - np.vdot(zg, zg).real) <= 1e-12
        out, p0 = s.measure_u(4, 0.5)
        p1 = np.sum(np.abs(zg[((np.arange(1 << n) >> 4) & 1) == 1]) ** 2)
        assert abs(p0 - (1 - p1 / np.vdot(zg, zg).real)) <= 1e-12
        zc = s.get_state()
        mask = ((np.arange(1 << n) >> 4) & 1) == out
        assert np.all(zc[~mask] == 0)
        assert abs(np.vdot(zc, zc).real - 1) <= 0.02


@pytest.mark.slow
def test_max_size_a_n36_paper_workloads():
    """BASELINE config 4's per-GPU size (2^36 codes = 128 GiB): the H wall and the
    GHZ chain are exact in A (Tables 2-3 captions),
    checked on sampled amplitudes and the per-qubit expectation values."""
    n = 36
    idx = np.random.default_rng(7).integers(0, 1 << n, 100000, dtype=np.uint64)
    with q.State(n, q.ENC_ADAPTIVE2) as s:
        s.apply_circuit(C.h_wall(n))
        assert np.max(np.abs(s.get_amplitudes(idx) - 2.0 ** (-n / 2))) <= 1e-15
        p = s.probabilities()
        assert np.max(np.abs(p - 0.5)) <= 1e-12
        s.reset()
        s.apply_circuit(C.ghz_chain(n))
        z = s.get_amplitudes(np.array([0, (1 << n) - 1, 12345, 1 << 35], dtype=np.uint64))
        assert np.max(np.abs(z - np.array([1, 1, 0, 0]) / math.sqrt(2))) <= 1e-15
        assert np.max(np.abs(s.probabilities() - 0.5)) <= 1e-15


@pytest.mark.slow
def test_table5_shor_n30_in_a():
    """PAPER.md Table 5: the A encoding (our exact-bounds policy, reading R-A4)
    agrees with the printed exact columns to about 3 digits, like the paper's A
    columns (worst printed A deviation 0.006 there; bound 0.011 of Table 4)."""
    import os
    rows = [l.split() for l in open(os.path.join(os.path.dirname(__file__), "golden", "table5_shor.txt"))
            if l.strip() and not l.startswith("#")]
    t = np.array(rows, dtype=float)
    with q.State(30, q.ENC_ADAPTIVE2) as s:
        s.prepare_shorbox(20, 1007, 529)
        z = s.get_amplitudes(np.array([0, 1 << 20, 1 + (529 << 20)], dtype=np.uint64))
        # SHORBOX is exact in A: |0>|1> and |1>|529> carry 2^-10, |0>|0> is empty
        assert z[0] == 0 and np.max(np.abs(np.abs(z[1:]) - 2.0 ** -10)) <= 1e-15
        s.apply_circuit(C.qft_register(30, 20))
        e = s.expectations()[:20]
    assert np.max(np.abs(e - t[:, 4:7])) <= 0.011


@pytest.mark.parametrize("P", [1, 4])
def test_overlap_a_vs_e_on_device(P):
    """qsim_overlap: <A|E>, <E|A>, <A|A>, <E|E> computed on the device equal
    np.vdot of the two decoded states read back (1e-12), so the config-4
    fidelity |<A|E>|^2 / (<A|A><E|E>) can be taken at full size."""
    n = 13
    circ = C.rz_rx_cphase(n, 3, seed=4)
    with q.State(n, q.ENC_ADAPTIVE2, P) as a, q.State(n, q.ENC_FP64, P) as e:
        a.apply_circuit(circ)
        e.apply_circuit(circ)
        za, ze = a.get_state(), e.get_state()
        assert abs(a.overlap(e) - np.vdot(za, ze)) <= 1e-12
        assert abs(e.overlap(a) - np.vdot(ze, za)) <= 1e-12
        assert abs(a.overlap(a) - np.vdot(za, za)) <= 1e-12
        assert abs(e.overlap(e) - 1.0) <= 1e-12
        fid = abs(a.overlap(e)) ** 2 / (a.overlap(a).real * e.overlap(e).real)
        assert fid >= 0.95
    with q.State(n, q.ENC_FP64, 2) as x, q.State(n, q.ENC_FP64, 2) as y:
        x.apply_gate(C.mat_H(), n - 1)  # exchange: x's qubit map differs from y's
        with pytest.raises(q.QsimError) as err:
            x.overlap(y)
        assert err.value.code == -7


def test_config4_fidelity_and_norm_drift_match_the_oracle():
    """Config 4 recipe, 10 layers, N=16: the A run's fidelity against E and
    its norm drift equal the oracle-A's (the loss of fidelity with N is a
    property of the linear magnitude code with exact global bounds, not of
    the kernels: r1 grows to many times the rms amplitude)."""
    n = 16
    circ = C.rz_rx_cphase(n, 10, seed=4)
    ref = oracle.AState(n).run(circ)
    zr = ref.decoded()
    e = oracle.e_simulate(n, circ)
    f_or = abs(np.vdot(zr, e)) ** 2 / (np.vdot(zr, zr).real * np.vdot(e, e).real)
    with q.State(n, q.ENC_ADAPTIVE2, 1) as a, q.State(n, q.ENC_FP64, 1) as s:
        a.apply_circuit(circ)
        s.apply_circuit(circ)
        f = abs(a.overlap(s)) ** 2 / (a.overlap(a).real * s.overlap(s).real)
        nrm = a.norm()
        _, r0, r1 = a.get_codes()
    assert abs(f - f_or) <= 2e-3
    assert abs(nrm - np.vdot(zr, zr).real) <= 2e-3
    assert r1 == pytest.approx(ref.r1, rel=1e-6)


def test_all_to_all_remap_is_bit_exact_in_a():
    """A codes after a circuit whose plan holds all-to-all remaps (P = 4, 8
    loopback shards) equal the single-shard run's bit for bit: remaps only
    move codes, bounds are global."""
    n = 13
    circ = C.layered(n, 2, seed=7)
    circ.extend(C.rz_rx_cphase(n, 2, seed=7))
    out = []
    for P in (1, 4, 8):
        ops, _ = q.qsim_plan(n, P, circ)
        assert P == 1 or sum(o["type"] == q.OP_REMAP for o in ops) > 0
        with q.State(n, q.ENC_ADAPTIVE2, P) as s:
            s.apply_circuit(circ)
            out.append(s.get_codes())
    for c, r0, r1 in out[1:]:
        assert np.array_equal(c, out[0][0]) and r0 == out[0][1] and r1 == out[0][2]


def test_fused_diagonal_runs_are_bit_exact(tmp_path):
    """Consecutive diagonal gates run as one sweep (k_diag_run_a) give the
    same codes, bit for bit, as one sweep per gate (QSIM_A_NO_DIAG_RUN=1):
    the per-gate b1 steps are integers summed mod 256.  Config-4 recipe (its
    CPHASE matchings and Rz streaks are the runs), P = 1 and 4."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env_off in (False, True):
        for P in (1, 4):
            out = str(tmp_path / f"c_{int(env_off)}_{P}.npy")
            code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1805_04708_b200 as q, "
                    "qsim_inputs as C; s = q.State(14, q.ENC_ADAPTIVE2, %d); s.apply_circuit(C.rz_rx_cphase(14, 4, "
                    "seed=9)); c, r0, r1 = s.get_codes(); np.save(%r, c); print(r0, r1)" % (root, P, out))
            env = dict(os.environ)
            if env_off:
                env["QSIM_A_NO_DIAG_RUN"] = "1"
            r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
            assert r.returncode == 0, r.stderr
            outs.append((np.load(out), r.stdout.split()))
    for c, b in outs[1:]:
        assert np.array_equal(c, outs[0][0]) and b == outs[0][1]
