"""Throughput of the auxiliary-variable evaluator (qsim_aux_amplitudes, PAPER.md
§4.2) on one GPU: config-3 structure at N=36 with P entangling gates kept,
M sampled amplitudes.  Prints terms/s (2^P x M per call) and the fp64 rate of
the term products (6 flops per complex multiply, one per qubit with variables
per term per amplitude).  The call is synchronous: wall time includes the host
tables, H2D, both kernels and D2H."""
import json
import math
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 36
ncp = int(sys.argv[2]) if len(sys.argv) > 2 else 24
M = int(sys.argv[3]) if len(sys.argv) > 3 else 64
rng = np.random.default_rng(7)
c = C.h_wall(n)
for qq in range(n):
    c.add("U", C.mat_haar(rng), qq)
for _ in range(ncp):
    a, b = [int(v) for v in rng.permutation(n)[:2]]
    c.add("CPHASE", C.mat_U1(float(rng.uniform(0, 2 * math.pi))), b, [a])
    c.add("U", C.mat_haar(rng), b)
P = q.qsim_aux_num_vars(n, c)
idx = rng.integers(0, 1 << n, size=M, dtype=np.uint64)
q.qsim_aux_amplitudes(n, c, idx)  # warm-up
reps = 3
t0 = time.perf_counter()
for _ in range(reps):
    q.qsim_aux_amplitudes(n, c, idx)
dt = (time.perf_counter() - t0) / reps
nact = len({t for g in range(len(c)) for t in ([c.gate(g)[2]] + list(c.gate(g)[4])) if len(c.gate(g)[4])})
terms = (1 << P) * M
print(json.dumps({"n": n, "P": P, "M": M, "qubits_with_variables": nact, "s_per_call": dt,
                  "terms_per_s": terms / dt, "fp64_TFLOPs": terms * nact * 6 / dt / 1e12}))
