"""Per-pass timing of the config-5 QFT at N qubits (E, fused passes, every
pass specialised before its first launch when QSIM_LPASS_JIT=2): the HBM
fraction of each light pass.  argv: n [reps]."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
circ, x = C.qft(n, seed=5)
s = q.State(n, q.ENC_FP64, 1)
gates = q.pack_gates(circ)
s.apply_circuit(gates)
s.sync()
q.qsim_jit_sync()
for _ in range(2):
    s.reset()
    s.apply_circuit(gates)
s.sync()
s.profile(True)
s.profile_read()
for _ in range(reps):
    s.reset()
    s.apply_circuit(gates)
s.sync()
prof = s.profile_read()
st = s.stats()
pk = prof.get("pass_e", {})
out = {"n": n, "gates": len(circ), "reps": reps, "profile": prof,
       "passes_per_circuit": pk.get("launches", 0) / reps,
       "ms_per_circuit_passes": pk.get("ms", 0.0) / reps,
       "hbm_GBps_passes": pk.get("bytes", 0.0) / max(pk.get("ms", 1e-9), 1e-9) / 1e6,
       "pass_GB": (1 << n) * 32 / 1e9,
       "stats": st}
print(json.dumps(out))
