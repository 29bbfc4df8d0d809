"""Drive a few dense A gates for ncu (one launch of each kernel class):
N qubits (default 28), a config-4 style state (H wall + one Rz/Rx/CPHASE
layer) -- here seeded random codes (qsim_set_codes) -- then Haar on t=10, Rx on t=2, H on t=20, and a CNOT (k_anti_a) and
CPHASE (k_diag_a).  Usage: python tools/a_gate_prof.py [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
s = q.State(n, q.ENC_ADAPTIVE2, 1, fuse=0)
codes, r0, r1 = C.random_codes(n, seed=1)  # seeded random codes: no kernels of the profiled kinds before
codes[2], codes[4] = -127, 126
s.set_codes(codes, r0, r1)
s.sync()
s.apply_gate(C.mat_haar(np.random.default_rng(3)), 10)
s.apply_gate(C.mat_Rx(0.7), 2)
s.apply_gate(C.mat_H(), 20)
s.apply_gate(C.mat_X(), 5, (17,))
s.apply_gate(C.mat_U1(0.9), 6, (21,))
s.sync()
print("done", s.bounds())
