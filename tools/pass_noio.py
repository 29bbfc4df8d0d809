"""How much of a specialised pass is tile I/O: the config-3 recipe (layered,
seed 3) at N qubits, per-pass device time with the tile loads / stores
(normal) and without them (QSIM_DEBUG_PASS_NOIO=1: the stages only, on
whatever the shared-memory tile holds -- timing only).  Usage:
python tools/pass_noio.py [N]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
circ = C.layered(n, 10, seed=3)
out = {}
with q.State(n) as s:
    for mode in ("io", "noio", "io"):
        if mode == "noio":
            os.environ["QSIM_DEBUG_PASS_NOIO"] = "1"
        else:
            os.environ.pop("QSIM_DEBUG_PASS_NOIO", None)
        for rep in range(3):
            s.reset()
            s.profile(True)
            s.apply_circuit(circ)
            s.sync()
            recs = s.profile_read()
            s.profile(False)
        k = max(recs, key=lambda kk: recs[kk]["ms"])  # the pass kernel class
        out[mode] = {"kernel": k, "passes": recs[k]["launches"], "ms_total": recs[k]["ms"],
                     "ms_per_pass": recs[k]["ms"] / max(1, recs[k]["launches"])}
        print(mode, out[mode], flush=True)
print(json.dumps({"n": n, "workload": "config-3 recipe (layered, 10 layers, seed 3)", "modes": out}))
