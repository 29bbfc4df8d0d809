"""Config-1 persistent-kernel variants (cluster size 2^c, phase width K) on one
GPU: device time per circuit (CUDA events on the state's stream) for N = 14
and 16.  Usage: python tools/persist_sweep.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

rows = []
for n in (14, 16):
    circ = C.config(0, n=n, seed=0)
    for lcs in (3, 4):
        for K in (3, 4):
            os.environ["QSIM_PERSIST_LCS"] = str(lcs)
            os.environ["QSIM_PERSIST_K"] = str(K)
            with q.State(n) as s:
                st = torch.cuda.ExternalStream(s.stream())
                for _ in range(5):
                    s.apply_circuit_persistent(circ)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 100
                e0.record(st)
                for _ in range(reps):
                    s.apply_circuit_persistent(circ)
                e1.record(st)
                e1.synchronize()
                rows.append({"n": n, "cluster": 1 << lcs, "K": K, "us_per_circuit": e0.elapsed_time(e1) * 1e3 / reps})
                print(rows[-1], flush=True)
os.environ["QSIM_PERSIST_DEBUG"] = "1"
for n in (14, 16):
    with q.State(n) as s:
        s.apply_circuit_persistent(C.config(0, n=n, seed=0))
        s.sync()
print(json.dumps(rows))
