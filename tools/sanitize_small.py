"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck):
N = 14 config-1 circuit through the fused relabelling pass with the
specialised kernels compiled first (QSIM_LPASS_JIT=2), the same circuit over
4 loopback shards (k_xchg_e exchanges, remaps), and a few A gates.
Usage: compute-sanitizer --tool racecheck python tools/sanitize_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

n = 14
circ = C.config(0, seed=0)
with q.State(n) as s:
    s.apply_circuit(circ)
    s.sync()
    z1 = s.get_state()
with q.State(n, q.ENC_FP64, 4, chunk_bytes=4096) as s:
    s.apply_circuit(circ)
    s.sync()
    z4 = s.get_state()
print("E 1 vs 4 shards", float(np.max(np.abs(z1 - z4))))
with q.State(12, q.ENC_ADAPTIVE2, 2) as s:
    s.apply_circuit(C.rz_rx_cphase(12, 2, seed=4))
    s.sync()
    print("A norm", s.norm())
print("done")
