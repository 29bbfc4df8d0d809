"""Config 5's full check: the QFT of a seeded basis state
|x> against the closed form 2^{-N/2} e^{2 pi i x y / 2^N} on EVERY amplitude
y, at N = 30 on one GPU (the state read back in logical order with
qsim_get_state, 16 GiB; the closed form evaluated on the host in chunks,
phase from the exact integer x*y mod 2^N).  Prints one JSON line.
Usage: python tools/qft_full_check.py [N]
"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
circ, x = C.qft(n, seed=5)
t0 = time.perf_counter()
with q.State(n, q.ENC_FP64, 1) as s:
    s.apply_circuit(circ)
    s.sync()
    t_gpu = time.perf_counter() - t0
    z = s.get_state()
mask = (1 << n) - 1
amp = 2.0 ** (-n / 2)
worst = 0.0
chunk = 1 << 24
for lo in range(0, 1 << n, chunk):
    y = np.arange(lo, lo + chunk, dtype=np.uint64)
    ph = (np.uint64(x) * y) & np.uint64(mask)  # x*y mod 2^N, exact in uint64 (x, y < 2^32)
    ref = amp * np.exp(2j * math.pi * ph.astype(np.float64) / float(1 << n))
    worst = max(worst, float(np.max(np.abs(z[lo:lo + chunk] - ref))))
out = {"row": "cfg5_full_check", "n": n, "x": int(x), "amplitudes_checked": 1 << n, "max_abs_err": worst,
       "gpu_circuit_s": t_gpu, "check_s": time.perf_counter() - t0}
print(json.dumps(out))
