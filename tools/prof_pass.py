"""Small driver for ncu: a few fused passes (and sweeps) at N qubits."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 1
fuse = int(sys.argv[3]) if len(sys.argv) > 3 else 1
enc = q.ENC_ADAPTIVE2 if (len(sys.argv) > 4 and sys.argv[4] == "A") else q.ENC_FP64
s = q.State(n, enc, 1, fuse=fuse)
circ = C.layered(n, layers, seed=1) if enc == q.ENC_FP64 else C.rz_rx_cphase(n, layers, seed=4)
s.apply_circuit(circ)
s.sync()
print("ok", s.stats())
