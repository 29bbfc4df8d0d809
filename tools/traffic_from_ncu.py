"""Turn an `ncu --page raw --csv` export of one k_lpass_e launch into the
profiles/traffic.json entry bench.py reads (DRAM bytes / algorithmic bytes).
Usage: python tools/traffic_from_ncu.py raw.csv N_qubits capture_note"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw, n, note = sys.argv[1], int(sys.argv[2]), sys.argv[3]
rows = list(csv.reader(open(raw)))
hdr = rows[0]
units = rows[1]
vals = rows[2]
m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(key):
    v, u = m[key]
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return x * scale


alg = 32.0 * 2 ** n
rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
keep = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.per_cycle_active"]
entry = {"capture": note, "dram_read_GB": rd / 1e9, "dram_write_GB": wr / 1e9, "algorithmic_GB": alg / 1e9,
         "dram_over_algorithmic": (rd + wr) / alg,
         "metrics": {k: f"{m[k][0]} {m[k][1]}".strip() for k in keep if k in m}}
stalls = []
for h in hdr:
    if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
        try:
            stalls.append((float(m[h][0].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
entry["top_stalls"] = sorted(stalls, reverse=True)[:8]
path = os.path.join(ROOT, "profiles", "traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d["pass_e"] = entry
json.dump(d, open(path, "w"), indent=1)
print(json.dumps(entry, indent=1))
