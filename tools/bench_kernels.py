"""Per-kernel-class timing of a workload (CUDA events from the library's own
qsim_profile records); prints one JSON line.  Usage:
  python tools/bench_kernels.py {E|A} N LAYERS [fuse] [recipe: layered|rzrx|qft|hwall]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

def pairs(n, layers):
    """Synthetic: layers x (Haar on qubits 0..11, CNOT 2i -> 2i+1): pure pair blocks."""
    import numpy as np
    rng = np.random.default_rng(0)
    c = C.Circuit(n)
    for _ in range(layers):
        for i in range(6):
            c.add("Haar", C.mat_haar(rng), 2 * i)
            c.add("Haar", C.mat_haar(rng), 2 * i + 1)
            c.add("CNOT", C.mat_X(), 2 * i + 1, [2 * i])
    return c


def singles(n, layers):
    """Synthetic: layers x Haar on qubits 0..11 (no entanglers)."""
    import numpy as np
    rng = np.random.default_rng(0)
    c = C.Circuit(n)
    for _ in range(layers):
        for i in range(12):
            c.add("Haar", C.mat_haar(rng), i)
    return c


enc = q.ENC_ADAPTIVE2 if sys.argv[1] == "A" else q.ENC_FP64
n, layers = int(sys.argv[2]), int(sys.argv[3])
fuse = int(sys.argv[4]) if len(sys.argv) > 4 else 1
recipe = sys.argv[5] if len(sys.argv) > 5 else ("rzrx" if enc == q.ENC_ADAPTIVE2 else "layered")
circ = {"layered": lambda: C.layered(n, layers, seed=1), "rzrx": lambda: C.rz_rx_cphase(n, layers, seed=4),
        "qft": lambda: C.qft(n, seed=5)[0], "hwall": lambda: C.h_wall(n), "ghz": lambda: C.ghz_chain(n),
        "cfg1": lambda: C.random_circuit(n, 200 * layers, seed=0), "pairs": lambda: pairs(n, layers),
        "single": lambda: singles(n, layers)}[recipe]()
s = q.State(n, enc, 1, fuse=fuse)
gates = q.pack_gates(circ)
s.apply_circuit(gates)  # warm-up (also: the state is non-trivial for the timed run)
s.sync()
s.reset_stats()
s.profile(True)
s.profile_read()
reps = int(os.environ.get("REPS", "1"))
t0 = time.perf_counter()
for _ in range(reps):
    s.apply_circuit(gates)
s.sync()
wall = (time.perf_counter() - t0) / reps
prof = s.profile_read()
st = s.stats()
out = {"enc": sys.argv[1], "n": n, "recipe": recipe, "gates": len(circ), "wall_s": wall, "reps": reps,
       "gates_per_s": len(circ) / wall, "stats": st,
       "kernels": {k: dict(v, avg_ms=v["ms"] / v["launches"], GBps=v["bytes"] / v["ms"] / 1e6,
                           TFLOPs=v["flops"] / v["ms"] / 1e9) for k, v in prof.items()}}
print(json.dumps(out))
