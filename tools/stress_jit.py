"""Stress check of the fused pass on the GPU: long random circuits of every
gate kind (config-1 mix), several seeds and sizes, each run with the
specialised kernels (QSIM_LPASS_JIT=2: compiled before first launch, so
every pass runs specialised code), compared with the oracle (max |delta
amplitude|); run with QSIM_LPASS_JIT=0 for the interpreter.  Test infrastructure: it
imports oracle/.  Usage: QSIM_LPASS_JIT=2 python tools/stress_jit.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

rows = []
worst = 0.0
for n, ng, seeds in ((18, 1500, range(4)), (21, 1000, range(3)), (23, 800, range(2))):
    for sd in seeds:
        circ = C.random_circuit(n, ng, seed=100 + sd)
        ref = oracle.e_simulate(n, circ)
        for P in (1, 4):
            with q.State(n, q.ENC_FP64, P) as s:
                s.apply_circuit(circ)
                err = float(np.max(np.abs(s.get_state() - ref)))
                st = s.stats()
            worst = max(worst, err)
            rows.append({"n": n, "gates": ng, "seed": 100 + sd, "P": P, "max_err": err, "passes": st["passes"],
                         "jit_passes": st["jit_passes"]})
            print(rows[-1], file=sys.stderr)
print(json.dumps({"worst": worst, "rows": rows}))
