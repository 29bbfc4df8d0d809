"""BASELINE config 1 (N=14, 200 gates, 256 KiB state: latency-bound, SURVEY.md
§8(d)): gates/s with one launch per gate, with the fused relabelling pass,
with each replayed from a CUDA graph (qsim_graph_*), and with the single
persistent cluster kernel (qsim_apply_circuit_persistent).

Timing: wall clock over REPS back-to-back circuits on the library stream,
synchronised once at each end (so host planning / compilation overlaps the
device where the mode allows it); the graph modes replay without any host
planning.  Device time per circuit from the library's CUDA events as well
(non-graph modes).  Usage: python tools/latency_cfg1.py [REPS] > latency.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04708_b200 as q  # noqa: E402
import qsim_inputs as C  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
n = 14
circ = C.config(0)
gates = q.pack_gates(circ)
out = {"workload": "config 1: N=14 E, 200 gates, seed 0", "reps": reps, "modes": {}}


def timed(fn, s, reps):
    for _ in range(5):
        fn()
    s.sync()
    q.qsim_jit_sync()  # specialised fused-pass kernels (if enabled for this size) are ready
    for _ in range(3):
        fn()
    s.sync()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    s.sync()
    return (time.perf_counter() - t0) / reps


for fuse in (0, 1):
    s = q.State(n, q.ENC_FP64, 1, fuse=fuse)
    label = "fused_pass" if fuse else "per_gate_launch"
    wall = timed(lambda: s.apply_circuit(gates), s, reps)
    s.reset_stats()
    s.profile(True)
    s.profile_read()
    s.apply_circuit(gates)
    prof = s.profile_read()
    s.profile(False)
    st = s.stats()
    dev_ms = sum(v["ms"] for v in prof.values())
    out["modes"][label] = {"us_per_circuit": wall * 1e6, "gates_per_s": 200 / wall, "kernels_per_circuit": st["kernels"],
                           "device_us_per_circuit": dev_ms * 1e3}
    g = s.capture(lambda st_: st_.apply_circuit(gates))
    wall_g = timed(g.launch, s, reps)
    out["modes"][label + "+cuda_graph"] = {"us_per_circuit": wall_g * 1e6, "gates_per_s": 200 / wall_g,
                                          "kernels_per_circuit": st["kernels"]}
    g.close()
    s.close()
# the whole circuit in one persistent cluster kernel (qsim_apply_circuit_persistent)
s = q.State(n, q.ENC_FP64, 1)
wall = timed(lambda: s.apply_circuit_persistent(gates), s, reps)
s.reset_stats()
s.profile(True)
s.profile_read()
s.apply_circuit_persistent(gates)
prof = s.profile_read()
s.profile(False)
out["modes"]["persistent_kernel"] = {"us_per_circuit": wall * 1e6, "gates_per_s": 200 / wall, "kernels_per_circuit": 1,
                                     "device_us_per_circuit": sum(v["ms"] for v in prof.values()) * 1e3}
s.close()
# one host call per gate (qsim_apply_gate), unfused
s = q.State(n, q.ENC_FP64, 1, fuse=0)
idx = list(range(len(circ)))


def per_call():
    for i in idx:
        _, _, t, _, ctl, u = circ.gate(i)
        s.apply_gate(u, t, ctl)


wall = timed(per_call, s, max(reps // 10, 5))
out["modes"]["apply_gate_per_call"] = {"us_per_circuit": wall * 1e6, "gates_per_s": 200 / wall}
s.close()
for k, v in out["modes"].items():
    print("%-28s %9.1f us/circuit  %12.0f gates/s" % (k, v["us_per_circuit"], v["gates_per_s"]), file=sys.stderr)
print(json.dumps(out))
