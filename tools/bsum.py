"""Print the key fields of the last JSON line of a bench log."""
import json
import sys

for path in sys.argv[1:]:
    lines = [l for l in open(path).read().strip().splitlines() if l.startswith("{")]
    if not lines:
        print(path, "no JSON line")
        continue
    d = json.loads(lines[-1])
    r = d.get("roofline") or {}
    print(path, f"value={d['value']:.1f} {d['unit']} gates/s={d.get('gates_per_s', 0):.1f} ms/step={d['ms_per_step']:.1f}",
          f"bound={r.get('bound')} frac={r.get('frac', 0):.3f} avg_launch_ms={r.get('avg_launch_ms', 0):.2f}",
          f"lib={d.get('library')}")
