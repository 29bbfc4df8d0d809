"""Probe: Table 5 (Shor, N=30, G=1007, y=529) expectation values on the GPU, E and A."""
import sys

sys.path.insert(0, '.')
import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

for enc in (q.ENC_FP64, q.ENC_ADAPTIVE2):
    with q.State(30, enc) as s:
        s.prepare_shorbox(20, 1007, 529)
        s.apply_circuit(C.qft_register(30, 20))
        e = s.expectations()[:20]
        nrm = s.norm()
    print("enc", enc, "norm", nrm)
    for i in range(20):
        print(i, " ".join(f"{v:.5f}" for v in e[i]))
