"""Config-4 recipe (A, seed 4, 10 layers) at N qubits, for ncu: profile the
dense-gate kernels late in the circuit (heavy-tailed structured state), e.g.
  ncu -k regex:k_bounds_a --launch-skip 120 -c 2 python tools/a_cfg4_prof.py 28"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
with q.State(n, q.ENC_ADAPTIVE2) as s:
    s.apply_circuit(C.rz_rx_cphase(n, 10, seed=4))
    s.sync()
    print("done", s.bounds())
