import sys, numpy as np
sys.path.insert(0, '.')
import paper_1805_04708_b200 as q, qsim_inputs as C, oracle
n = 14
circ = C.config(0, seed=3)
def frac(z, ra):
    ref = ra.decoded(); step = (ra.r1 - ra.r0) / 253.0
    return np.mean(np.abs(np.abs(z) - np.abs(ref)) <= step + 1e-12)
for kw in [dict(), dict(transport=q.TRANSPORT_DEVICES, device=0)]:
    with q.State(n, 1, 1, **kw) as s:
        s.apply_circuit(circ)
        z = s.get_state()
    print(kw, 'whole', frac(z, oracle.AState(n).run(circ)))
# per gate from identical codes, local transport
with q.State(n, 1, 1) as s:
    worst = []
    for i in range(len(circ)):
        c, r0, r1 = s.get_codes()
        one = oracle.AState(n, c, r0, r1); g = circ.slice(i, i + 1); one.run(g)
        s.apply_circuit(g)
        z = s.get_state()
        f = frac(z, one)
        if f < 1: worst.append((i, circ.names[i], circ.gate(i)[2], circ.gate(i)[4], f, r0, r1, one.r0, one.r1))
    print('per-gate failures', len(worst)); [print(w) for w in worst[:10]]
