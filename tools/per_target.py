"""Per-gate time by target qubit index ("report
per-gate time by target index 0..29 (unfused)").

Unfused single-gate sweeps (fuse=0) on a resident state at N qubits; for each
target t, W warm-up then R timed repetitions of the same gate, timed with the
library's own per-launch CUDA events (qsim_profile, on its stream); median and
min per launch.  E: dense Haar U(2) (k_sweep_e), CNOT with control (t+1) mod N,
T (diagonal, half the amplitudes).  A: dense gate = k_bounds_a + k_apply_a
(two phases, reading R-A4), Rz (k_diag_a).  The state content does not change
the E timing; for A it is a config-4 style state (H wall + one Rz/Rx/CPHASE
layer) so that the bounds are non-degenerate.

Usage: python tools/per_target.py {E|A} N [REPS] > per_target_{E|A}.json
(A_POLICY=lazy|fp32 selects the A policy; default exact.)
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

enc_name = sys.argv[1] if len(sys.argv) > 1 else "E"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
warm = 3
enc = q.ENC_ADAPTIVE2 if enc_name == "A" else q.ENC_FP64
pol = {"exact": q.A_POLICY_EXACT, "lazy": q.A_POLICY_LAZY, "fp32": q.A_POLICY_FP32}[os.environ.get("A_POLICY", "exact")]
s = q.State(n, enc, 1, fuse=0, a_policy=pol)
if enc == q.ENC_ADAPTIVE2:
    s.apply_circuit(C.rz_rx_cphase(n, 1, seed=4))
else:
    s.apply_circuit(C.h_wall(n))
s.sync()
rng = np.random.default_rng(7)
U = C.mat_haar(rng)
amp_bytes = 2 if enc == q.ENC_ADAPTIVE2 else 16
shard_bytes = float(2 ** n) * amp_bytes
kinds = [("dense", U, lambda t: ()), ("cnot", C.mat_X(), lambda t: ((t + 1) % n,)), ("T", C.mat_T(), lambda t: ())]
if enc == q.ENC_ADAPTIVE2:
    kinds = [("dense", U, lambda t: ()), ("Rx", C.mat_Rx(0.7), lambda t: ()), ("H", C.mat_H(), lambda t: ()),
             ("Rz", C.mat_Rz(0.7), lambda t: ())]

out = {"enc": enc_name, "a_policy": os.environ.get("A_POLICY", "exact"), "n": n, "reps": reps, "warmup": warm, "unit": "ms per gate (CUDA events, library stream)",
       "rows": []}
targets = [int(x) for x in os.environ["TARGETS"].split(",")] if os.environ.get("TARGETS") else list(range(n))
for name, u, ctl in kinds:
    for t in targets:
        s.profile(False)
        for _ in range(warm):
            s.apply_gate(u, t, ctl(t))
        s.sync()
        per = []
        s.profile(True)
        s.profile_read()
        for _ in range(reps):
            s.apply_gate(u, t, ctl(t))
            prof = s.profile_read()  # synchronises; one gate's launches
            per.append(sum(v["ms"] for v in prof.values()))
            last = prof
        s.profile(False)
        byts = sum(v["bytes"] for v in last.values())  # algorithmic bytes of the gate (sum over its phases)
        med = statistics.median(per)
        out["rows"].append({"gate": name, "target": t, "ms_median": med, "ms_min": min(per),
                            "kernels": {k: v["ms"] for k, v in last.items()},
                            "alg_bytes": byts, "GBps_median": byts / med / 1e6})
for r in out["rows"]:
    print("%-6s t=%2d  median %.3f ms  min %.3f ms  %7.0f GB/s  %s" % (
        r["gate"], r["target"], r["ms_median"], r["ms_min"], r["GBps_median"],
        " ".join("%s=%.3f" % kv for kv in r["kernels"].items())), file=sys.stderr)
print(json.dumps(out))
