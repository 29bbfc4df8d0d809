"""Device-side cost of the global-qubit paths on ONE GPU (loopback transport:
all shards on this device, the partner's half-shard arrives by a device copy
instead of NVLink) -- SURVEY.md §8(a) a7 / NEXT-1 (i).  This is not the
NVLink figure (one GPU per gpurun call here); it is what the exchange costs
on the device side: copy into staging + the on-arrival gate kernel, and the
all-to-all block swaps.

Rows (E, 2^30 amplitudes per shard):
  pairwise  P = 2, N = 31: a dense gate on the qubit that sits on the global
            bit -> half-shard swap exchange fused with the gate, repeated.
  remap     P = 4 / 8, N = 32 / 33: dense gates on all global qubits back to
            back -> one all-to-all remap (1 - 2^-m of every shard).
Usage: python tools/xchg_loopback.py > xchg.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

out = []


def timed(s, fn, reps):
    fn()
    s.sync()
    s.reset_stats()
    s.profile(True)
    s.profile_read()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    s.sync()
    wall = (time.perf_counter() - t0) / reps
    prof = s.profile_read()
    s.profile(False)
    return wall, prof, s.stats()


# pairwise: P = 2
n, P = 31, 2
with q.State(n, q.ENC_FP64, P) as s:
    U = C.mat_haar(np.random.default_rng(3))
    nl = n - 1

    def one():
        pos = s.qubit_map()
        lq = pos.index(nl)  # the logical qubit on the global bit
        s.apply_gate(U, lq)

    wall, prof, st = timed(s, one, 5)
    xk = prof.get("xchg", {"ms": 0.0, "launches": 0})
    per = st["exchange_bytes"] / 5  # bytes sent per direction summed over shards, per gate
    out.append({"row": "pairwise", "n": n, "P": P, "wall_ms_per_gate": wall * 1e3,
                "xchg_kernel_ms_per_gate": xk["ms"] / 5, "exchanges_per_gate": st["exchanges"] / 5,
                "bytes_per_direction_per_gate": per, "device_GBps": per / (wall) / 1e9})
# remap: P = 4, 8
for n, P in ((32, 4), (33, 8)):
    k = int(np.log2(P))
    with q.State(n, q.ENC_FP64, P) as s:
        U = C.mat_haar(np.random.default_rng(4))
        nl = n - k

        def layer():
            pos = s.qubit_map()
            glob = [pos.index(nl + j) for j in range(k)]  # logical qubits on the global bits
            c = C.Circuit(n)
            for lq in glob:
                c.add("Haar", U, lq)
            s.apply_circuit(c)

        wall, prof, st = timed(s, layer, 3)
        per = st["exchange_bytes"] / 3
        out.append({"row": "remap", "n": n, "P": P, "m": k, "wall_ms_per_layer": wall * 1e3,
                    "exchanges_per_layer": st["exchanges"] / 3, "bytes_moved_per_layer": per,
                    "device_GBps": per / wall / 1e9,
                    "kernels": {kk: v["ms"] / 3 for kk, v in prof.items()}})
for r in out:
    print(r, file=sys.stderr)
print(json.dumps(out))
