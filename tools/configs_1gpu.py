"""The BASELINE configs that are not the bench line, at their per-GPU size on
one B200 (SURVEY.md §8(d) "Configs as concrete synthetic inputs" and the
supplementary paper-workload rows S1/S2).  Each row: the circuit from
qsim_inputs (seeded), the device time from the library's CUDA events on its
stream (qsim_profile), gates/s, effective GB/s (algorithmic bytes), and the
check the config names, computed here on the GPU results:

  cfg3_n33   E, N=33 (the P=1 point of the weak-scaling series: 2^33 amplitudes
             = 128 GiB), H wall + 10 layers; norm.
  cfg4_n33   A, N=33 (config 4's per-GPU code count at P=64 ... here the
             fidelity run of config 4): A and E runs of the same circuit on
             one device; fidelity |<A|E>|^2/(<A|A><E|E>) by qsim_overlap, norm
             drift of A.
  cfg5_n32   E QFT, N=32 (config 5's 2^32 amplitudes per GPU) of a seeded basis
             state; closed form 2^{-N/2} e^{2 pi i x y / 2^N} on 2^20 sampled y,
             marginals = 1/2.
  cfg5_n32_basis  the same with |x> from qsim_reset_basis and the 544-gate QFT
             circuit alone timed.
  s1_hwall   H wall, E N=32 and A N=35 (64 GiB each); closed form.
  s2_ghz     CNOT chain (H + CNOT(i -> i+1)), E N=32 and A N=35; closed form.

Usage: python tools/configs_1gpu.py [row ...] > configs.json (default: all)
"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402


def run(s, circ, warm=True):
    """Apply circ with per-kernel events; returns (device ms, wall s, profile, stats).
    warm: apply it once first, wait for the fused-pass specialisations it
    queued (qsim_jit_sync), reset to |0...0>, then time the second application."""
    gates = q.pack_gates(circ)
    if warm:
        s.apply_circuit(gates)
        s.sync()
        q.qsim_jit_sync()
        s.reset()
    s.sync()
    s.reset_stats()
    s.profile(True)
    s.profile_read()
    t0 = time.perf_counter()
    s.apply_circuit(gates)
    s.sync()
    wall = time.perf_counter() - t0
    prof = s.profile_read()
    s.profile(False)
    st = s.stats()
    dev = sum(v["ms"] for v in prof.values())
    return dev, wall, prof, st


def summary(name, circ, dev, wall, prof, st, **extra):
    row = {"row": name, "n": circ.n, "gates": len(circ), "device_ms": dev, "wall_ms": wall * 1e3,
           "gates_per_s": len(circ) / (dev / 1e3), "effective_GBps": st["gate_bytes"] / (dev / 1e3) / 1e9,
           "hbm_GBps": st["hbm_bytes"] / (dev / 1e3) / 1e9,
           "kernels": {k: {"launches": v["launches"], "ms": v["ms"]} for k, v in prof.items()},
           "stats": {k: st[k] for k in ("kernels", "sweeps", "passes", "fused_gates", "exchanges")}}
    row.update(extra)
    print("%-10s N=%d %4d gates  %9.1f ms  %10.0f gates/s  eff %7.0f GB/s  %s" % (
        name, circ.n, len(circ), dev, row["gates_per_s"], row["effective_GBps"],
        " ".join("%s=%s" % (k, v) for k, v in extra.items())), file=sys.stderr)
    return row


def cfg3_n33():
    n = 33
    circ = C.config(2, n=n)
    with q.State(n, q.ENC_FP64, 1) as s:
        dev, wall, prof, st = run(s, circ)
        nrm = s.norm()
    return summary("cfg3_n33", circ, dev, wall, prof, st, norm_err=abs(nrm - 1.0))


def cfg4_n33():
    n = 33
    circ = C.config(3, n=n)
    with q.State(n, q.ENC_ADAPTIVE2, 1) as a:
        dev, wall, prof, st = run(a, circ, warm=False)
        with q.State(n, q.ENC_FP64, 1) as e:
            dev_e, _, _, _ = run(e, circ)
            ae = a.overlap(e)
            aa = a.overlap(a).real
            ee = e.overlap(e).real
    fid = abs(ae) ** 2 / (aa * ee)
    return summary("cfg4_n33", circ, dev, wall, prof, st, fidelity_vs_E=fid, norm_A=aa, norm_E=ee,
                   E_device_ms=dev_e)


def cfg5_n32():
    n = 32
    circ, x = C.qft(n, seed=5)
    rng = np.random.default_rng(55)
    ys = rng.integers(0, 2 ** n, size=2 ** 20, dtype=np.uint64)
    with q.State(n, q.ENC_FP64, 1) as s:
        dev, wall, prof, st = run(s, circ)
        z = s.get_amplitudes(ys)
        p1 = s.probabilities()
    ph = (int(x) * ys.astype(object)) % (2 ** n)
    ref = 2.0 ** (-n / 2) * np.exp(2j * math.pi * np.array([float(v) for v in ph]) / 2.0 ** n)
    return summary("cfg5_n32", circ, dev, wall, prof, st, x=int(x), max_err_sampled=float(np.max(np.abs(z - ref))),
                   max_marginal_err=float(np.max(np.abs(p1 - 0.5))))


def cfg5_n32_basis():
    """Config 5 with the input |x> prepared by qsim_reset_basis (outside the
    timed region, like the reset of every row) and the standard QFT circuit
    timed: 544 gates at N = 32 (no X gates, so no relabel-only pass)."""
    n = 32
    _, x = C.qft(n, seed=5)
    circ = C.qft_register(n, n)
    rng = np.random.default_rng(55)
    ys = rng.integers(0, 2 ** n, size=2 ** 20, dtype=np.uint64)
    gates = q.pack_gates(circ)
    with q.State(n, q.ENC_FP64, 1) as s:
        s.reset_basis(x)
        s.apply_circuit(gates)
        s.sync()
        q.qsim_jit_sync()
        s.reset_basis(x)
        s.sync()
        s.reset_stats()
        s.profile(True)
        s.profile_read()
        t0 = time.perf_counter()
        s.apply_circuit(gates)
        s.sync()
        wall = time.perf_counter() - t0
        prof = s.profile_read()
        s.profile(False)
        st = s.stats()
        dev = sum(v["ms"] for v in prof.values())
        z = s.get_amplitudes(ys)
        p1 = s.probabilities()
    ph = (int(x) * ys.astype(object)) % (2 ** n)
    ref = 2.0 ** (-n / 2) * np.exp(2j * math.pi * np.array([float(v) for v in ph]) / 2.0 ** n)
    return summary("cfg5_basis", circ, dev, wall, prof, st, x=int(x), max_err_sampled=float(np.max(np.abs(z - ref))),
                   max_marginal_err=float(np.max(np.abs(p1 - 0.5))))


def s1_hwall():
    rows = []
    for n, enc in ((32, q.ENC_FP64), (35, q.ENC_ADAPTIVE2)):
        circ = C.h_wall(n)
        with q.State(n, enc, 1) as s:
            dev, wall, prof, st = run(s, circ, warm=enc == q.ENC_FP64)
            idx = np.random.default_rng(1).integers(0, 2 ** n, size=2 ** 16, dtype=np.uint64)
            err = float(np.max(np.abs(s.get_amplitudes(idx) - 2.0 ** (-n / 2))))
        rows.append(summary("s1_hwall_" + ("E" if enc == q.ENC_FP64 else "A"), circ, dev, wall, prof, st,
                            max_err_sampled=err))
    return rows


def s2_ghz():
    rows = []
    for n, enc in ((32, q.ENC_FP64), (35, q.ENC_ADAPTIVE2)):
        circ = C.ghz_chain(n)
        with q.State(n, enc, 1) as s:
            dev, wall, prof, st = run(s, circ, warm=enc == q.ENC_FP64)
            z = s.get_amplitudes(np.array([0, 2 ** n - 1, 1, 2 ** (n - 1)], dtype=np.uint64))
        err = float(np.max(np.abs(z - np.array([1, 1, 0, 0]) / math.sqrt(2))))
        rows.append(summary("s2_ghz_" + ("E" if enc == q.ENC_FP64 else "A"), circ, dev, wall, prof, st,
                            max_err_sampled=err))
    return rows


def table4_adder():
    """NEXT-2: the scaled Table-4 QFT adder, a = 210018 mod 2^k,
    b = 2^k - 1 - a: E at N = 30 (k = 15) and A at N = 30 and N = 34 (k = 17);
    max deviation of the expectation values from the closed form."""
    rows = []
    for k, enc in ((15, q.ENC_FP64), (15, q.ENC_ADAPTIVE2), (17, q.ENC_ADAPTIVE2)):
        a = 210018 % (1 << k)
        b = (1 << k) - 1 - a
        n = 2 * k
        circ = C.draper_adder(k, a, b)
        idx = (a + b) % (1 << k)
        for j in range(k):
            if (a >> j) & 1:
                idx |= 1 << (n - 1 - j)
        ref = np.array([[0.5, 0.5, float((idx >> qq) & 1)] for qq in range(n)])
        with q.State(n, enc, 1) as s:
            dev, wall, prof, st = run(s, circ, warm=enc == q.ENC_FP64)
            ex = s.expectations()
        rows.append(summary("table4_adder_" + ("E" if enc == q.ENC_FP64 else "A"), circ, dev, wall, prof, st,
                            k=k, max_dev_vs_closed_form=float(np.max(np.abs(ex - ref))),
                            min_sum_bit_Qz=float(np.min(ex[:k, 2]))))
    return rows


def cfg4_lazy():
    """NEXT-4: config 4 at N = 33 under the lazy-bounds A policy (reading R-A25)
    and the fp32-arithmetic variant (reading R-A26) vs the exact policy:
    device time, dense gates that rescaled, fidelity against E (same circuit,
    E run on the same GPU)."""
    n = 33
    circ = C.config(3, n=n)
    rows = []
    with q.State(n, q.ENC_FP64, 1) as e:
        e.apply_circuit(circ)
        e.sync()
        for pol in (q.A_POLICY_EXACT, q.A_POLICY_LAZY, q.A_POLICY_FP32):
            with q.State(n, q.ENC_ADAPTIVE2, 1, a_policy=pol) as a:
                dev, wall, prof, st = run(a, circ, warm=False)
                ae = a.overlap(e)
                aa = a.overlap(a).real
                ee = e.overlap(e).real
            rows.append(summary("cfg4_" + {0: "exact", 1: "lazy", 2: "fp32"}[pol], circ, dev, wall, prof, st,
                                fidelity_vs_E=abs(ae) ** 2 / (aa * ee), norm_A=aa,
                                dense=st["a_dense"], rescaled=st["a_rescales"]))
    return rows


def cfg4_trend():
    """Config-4 fidelity and norm drift of A against E as N grows (10 layers)."""
    rows = []
    for n in (16, 20, 24, 28, 30):
        circ = C.config(3, n=n)
        with q.State(n, q.ENC_ADAPTIVE2, 1) as a, q.State(n, q.ENC_FP64, 1) as e:
            dev, wall, prof, st = run(a, circ, warm=False)
            e.apply_circuit(circ)
            ae, aa, ee = a.overlap(e), a.overlap(a).real, e.overlap(e).real
            _, r0, r1 = a.get_codes() if n <= 32 else (None, float("nan"), float("nan"))
        rows.append(summary("cfg4_trend", circ, dev, wall, prof, st, fidelity_vs_E=abs(ae) ** 2 / (aa * ee),
                            norm_A=aa, r1_over_rms=r1 * 2 ** (n / 2)))
    return rows


ROWS = {"cfg4_lazy": cfg4_lazy, "table4_adder": table4_adder, "cfg4_trend": cfg4_trend, "cfg3_n33": cfg3_n33, "cfg4_n33": cfg4_n33, "cfg5_n32": cfg5_n32, "cfg5_n32_basis": cfg5_n32_basis, "s1_hwall": s1_hwall, "s2_ghz": s2_ghz}
want = sys.argv[1:] or list(ROWS)
out = []
for name in want:
    try:
        r = ROWS[name]()
        out.extend(r if isinstance(r, list) else [r])
    except Exception as ex:  # report and continue with the other rows
        out.append({"row": name, "error": repr(ex)})
        print(name, "ERROR", repr(ex), file=sys.stderr)
print(json.dumps(out))
