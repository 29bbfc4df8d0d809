"""A-encoding parity at the sizes where the config-4 fidelity falls (VERDICT r1
"What's weak" #1): the GPU A path against the oracle's own step-by-step A
implementation (§4.1, reading R-A4: exact global bounds
per gate) on the config-4 recipe at N = 24, per-gate from identical codes on
full-grid shards (N = 22, every kernel's grid-stride path), and the Table-5
workload (SHORBOX + QFT) against the oracle.  Tolerance (BASELINE north_star,
DESIGN.md R-B2): decoded amplitudes within one quantisation step of the
oracle-A, |dr| <= (r1 - r0)/253, |dtheta| <= pi/128 (+1e-12)."""
import math

import numpy as np
import pytest

import oracle
import qsim_inputs as C

pytestmark = pytest.mark.gpu
q = pytest.importorskip("paper_1805_04708_b200")


def within_one_step(z_gpu, z_ref, r0, r1):
    step = (r1 - r0) / 253.0
    ok_m = np.abs(np.abs(z_gpu) - np.abs(z_ref)) <= step + 1e-12
    both = (np.abs(z_gpu) > 0) & (np.abs(z_ref) > 0)
    ok_t = ~both | (np.abs(np.angle(z_gpu * np.conj(z_ref))) <= math.pi / 128 + 1e-12)
    return ok_m & ok_t


def code_diff(cg, co):
    b0 = np.abs(cg[0::2].astype(int) - co[0::2].astype(int))
    d1 = np.abs(cg[1::2].astype(int) - co[1::2].astype(int)) % 256
    b1 = np.minimum(d1, 256 - d1)
    zero = (cg[0::2] == -128) & (co[0::2] == -128)
    return np.where(zero, 0, b0), np.where(zero, 0, b1)


def fidelity(x, y):
    return abs(np.vdot(x, y)) ** 2 / (np.vdot(x, x).real * np.vdot(y, y).real)


@pytest.mark.parametrize("n", [24, 26])
def test_config4_whole_circuit_vs_oracle_a(n):
    """Config 4 recipe (H wall, 10 layers of coin-flip Rz/Rx + CPHASE on a
    random matching, seed 4) at N = 24 (384 gates) and 26 (416 gates): within-one-step fraction
    >= 0.99, fidelity against E and norm equal to the oracle-A's within 2e-3,
    r1 equal to 1e-6 relative; and the exact E state's own maximum magnitude
    equals r1 to a few per cent, i.e. the heavy tail that sets the A step
     is a property of the exact state, not of the encoder."""
    circ = C.rz_rx_cphase(n, 10, seed=4)
    ref = oracle.AState(n).run(circ)
    zr = ref.decoded()
    e = oracle.e_simulate(n, circ)
    with q.State(n, q.ENC_ADAPTIVE2) as a, q.State(n, q.ENC_FP64) as s:
        a.apply_circuit(circ)
        s.apply_circuit(circ)
        zg = a.get_state()
        _, g0, g1 = a.get_codes()
        nrm = a.norm()
        f_dev = abs(a.overlap(s)) ** 2 / (a.overlap(a).real * s.overlap(s).real)
        lo, hi = s.magnitude_range()
        ze = s.get_state()
    assert np.max(np.abs(ze - e)) <= 1e-12
    frac = within_one_step(zg, zr, ref.r0, ref.r1).mean()
    f_or = fidelity(zr, e)
    assert frac >= 0.99, frac
    assert abs(f_dev - f_or) <= 2e-3, (f_dev, f_or)
    assert abs(fidelity(zg, e) - f_dev) <= 1e-9
    assert abs(nrm - np.vdot(zr, zr).real) <= 2e-3
    assert g1 == pytest.approx(ref.r1, rel=1e-6)
    assert hi == pytest.approx(np.abs(e).max(), rel=1e-12)
    assert lo == pytest.approx(np.abs(e[np.abs(e) > 0]).min(), rel=1e-12)
    assert abs(hi / ref.r1 - 1) <= 0.05, (hi, ref.r1)


DENSE = [("H", C.mat_H()), ("Haar", C.mat_haar(np.random.default_rng(22))), ("Rx", C.mat_Rx(2.2))]


@pytest.mark.parametrize("name,u", DENSE, ids=[d[0] for d in DENSE])
@pytest.mark.parametrize("t", [0, 3, 4, 12, 21])
def test_per_gate_full_grid_n22(name, u, t):
    """Per gate from identical seeded codes at N = 22 (4 Mi amplitudes: the
    bounds and apply kernels run their grid-stride loops over a full grid, the
    target classes bit 0..3 inside a 16-code unit and a runtime bit >= 4)."""
    n = 22
    codes, r0, r1 = C.random_codes(n, seed=100 + t)
    codes[2] = -127  # extreme magnitude codes present: the input bounds are exact
    codes[4] = 126
    ref = oracle.AState(n, codes, r0, r1)
    ref.apply(u, t)
    with q.State(n, q.ENC_ADAPTIVE2) as s:
        s.set_codes(codes, r0, r1)
        s.apply_gate(u, t)
        cg, g0, g1 = s.get_codes()
        zg = s.get_state()
    # r0 is the smallest output magnitude: a near-cancellation u00 a0 + u01 a1
    # whose fp64 rounding (FMA on the GPU, separate products in the oracle)
    # differs by a few ulps of the INPUT magnitudes, ~eps * r1 absolute
    assert g0 == pytest.approx(ref.r0, rel=1e-12, abs=1e-15 * ref.r1) and g1 == pytest.approx(ref.r1, rel=1e-12)
    db0, db1 = code_diff(cg, ref.codes)
    assert db0.max() <= 1 and db1.max() <= 1
    assert within_one_step(zg, ref.decoded(), ref.r0, ref.r1).all()
    assert np.mean((db0 == 0) & (db1 == 0)) >= 0.999


@pytest.mark.parametrize("ctl", [(5,), (5, 17)])
def test_per_gate_full_grid_controlled_n22(ctl):
    """Controlled dense A gates on a full grid (N = 22), target above and below
    the controls."""
    n = 22
    for t in (0, 20):
        codes, r0, r1 = C.random_codes(n, seed=7 + t + len(ctl))
        codes[2] = -127
        codes[4] = 126
        u = C.mat_haar(np.random.default_rng(t))
        ref = oracle.AState(n, codes, r0, r1)
        ref.apply(u, t, ctl)
        with q.State(n, q.ENC_ADAPTIVE2) as s:
            s.set_codes(codes, r0, r1)
            s.apply_gate(u, t, ctl)
            cg, _, _ = s.get_codes()
        db0, db1 = code_diff(cg, ref.codes)
        assert db0.max() <= 1 and db1.max() <= 1
        assert np.mean((db0 == 0) & (db1 == 0)) >= 0.999


def test_table5_recipe_in_a_vs_oracle_a_n24():
    """The Table-5 workload (SHORBOX + QFT on the x-register)
    at the largest size the oracle-A runs gate by gate in a test (N = 24:
    G = 247, y = 2, 16-qubit x-register; the paper's N = 30 instance is
    checked in E below).  SHORBOX codes equal the oracle's; then EVERY gate of
    the QFT is checked from identical input codes (the GPU's codes before the
    gate, fed to the oracle-A): decoded amplitudes within one step.  Over the
    whole circuit the two runs drift apart at rounding ties -- the CPHASE
    R_9 phase is exactly half a b1 step (SURVEY §8(c) "A on QFT"), which the
    GPU's phase path rounds away from zero while the oracle's fp64
    decode-rotate-encode lands on either side of the tie -- so the whole
    circuit is bounded by the paper's accuracy level instead: expectations
    within 0.011 of E (Table 4) and fidelity >= 0.99 against
    the oracle-A."""
    n, nx, G, y = 24, 16, 247, 2
    ze0 = oracle.e_shorbox(n, nx, G, y)
    ref = oracle.AState(n)
    ref.encode_from(ze0)
    circ = C.qft_register(n, nx)
    with q.State(n, q.ENC_ADAPTIVE2) as s:
        s.prepare_shorbox(nx, G, y)
        c0, _, _ = s.get_codes()
        assert np.array_equal(c0, ref.codes)
        for i in range(len(circ)):
            c, r0, r1 = s.get_codes()
            one = oracle.AState(n, c, r0, r1)
            g = circ.slice(i, i + 1)
            one.run(g)
            s.apply_circuit(g)
            zg = s.get_state()
            ok = within_one_step(zg, one.decoded(), one.r0, one.r1)
            assert ok.all(), (i, 1 - ok.mean())
        zg = s.get_state()
        ex = s.expectations()
    ref.run(circ)
    zr = ref.decoded()
    f = fidelity(zg, zr)
    assert f >= 0.99, f
    ee = oracle.e_expectations(oracle.e_run(ze0, n, circ), n)
    assert np.max(np.abs(ex - oracle.e_expectations(zg, n))) <= 1e-12
    assert np.max(np.abs(ex - ee)) <= 0.011


@pytest.mark.slow
def test_table5_shor_n30_e_vs_oracle():
    """Table 5 (Shor, N = 30, G = 1007, y = 529): the GPU's E expectations and
    amplitudes equal the oracle's (1e-12) -- the printed columns are checked
    separately (test_gpu_e.py::test_table5_shor_n30_exact_columns)."""
    n, nx = 30, 20
    circ = C.qft_register(n, nx)
    ref = oracle.e_run(oracle.e_shorbox(n, nx, 1007, 529), n, circ)
    idx = np.random.default_rng(30).integers(0, 1 << n, 1 << 20, dtype=np.uint64)
    with q.State(n) as s:
        s.prepare_shorbox(nx, 1007, 529)
        s.apply_circuit(circ)
        ex = s.expectations()
        z = s.get_amplitudes(idx)
    assert np.max(np.abs(z - ref[idx.astype(np.int64)])) <= 1e-12
    assert np.max(np.abs(ex - oracle.e_expectations(ref, n))) <= 1e-12
