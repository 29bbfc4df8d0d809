"""Config-4 magnitude tail vs the A bounds (VERDICT r1 "Next round" #1): for
N = 16 ... 33, run the config-4 recipe (H wall + 10 layers of coin-flip Rz/Rx
and CPHASE on a random matching, seed 4) in E and in A on one B200 and report

  maxE_rms  = max_x |psi_E(x)| * 2^{N/2}   (the exact state's own tail,
              qsim_magnitude_range)
  r1_rms    = r1 * 2^{N/2}                  (the A state's upper bound)
  F         = |<A|E>|^2 / (<A|A><E|E>)      (qsim_overlap)
  norm_A    = <A|A>

If maxE_rms tracks r1_rms, the coarse magnitude step (r1 - r0)/253 that limits
F is set by the exact state, not by an encoder bug.

Usage: python tools/a_magnitudes.py [N ...] > profiles/round2_a_magnitudes.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

ns = [int(a) for a in sys.argv[1:]] or [16, 20, 24, 28, 30, 32, 33]
rows = []
for n in ns:
    circ = C.rz_rx_cphase(n, 10, seed=4)
    g = q.pack_gates(circ)
    with q.State(n, q.ENC_FP64) as e, q.State(n, q.ENC_ADAPTIVE2) as a:
        t0 = time.perf_counter()
        e.apply_circuit(g)
        e.sync()
        te = time.perf_counter() - t0
        t0 = time.perf_counter()
        a.apply_circuit(g)
        a.sync()
        ta = time.perf_counter() - t0
        lo, hi = e.magnitude_range()
        r0, r1 = a.bounds()
        ov = a.overlap(e)
        fid = abs(ov) ** 2 / (a.overlap(a).real * e.overlap(e).real)
        row = {"n": n, "gates": len(circ), "maxE_rms": hi * 2 ** (n / 2), "r1_rms": r1 * 2 ** (n / 2),
               "r0_rms": r0 * 2 ** (n / 2), "minE_rms": lo * 2 ** (n / 2), "F": fid, "norm_A": a.norm(),
               "wall_s_E": te, "wall_s_A": ta}
    rows.append(row)
    print("N=%2d maxE*2^(N/2)=%6.2f r1*2^(N/2)=%6.2f F=%.4f norm_A=%.4f (E %.2fs, A %.2fs)" % (
        n, row["maxE_rms"], row["r1_rms"], fid, row["norm_A"], te, ta), file=sys.stderr)
print(json.dumps({"what": "config-4 recipe (seed 4, 10 layers): exact-state magnitude tail vs A bounds", "rows": rows},
                 indent=1))
