"""One-line digest of a bench JSON line (for gpurun logs)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        line = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:   # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    r = line.get("roofline") or {}
    p = line.get("parity") or {}
    e = line.get("e2e") or {}
    c = line.get("cpu_baseline") or {}
    print(f"{f}: ms {line.get('ms_per_step')} kern {line.get('kernel_ms_per_step')} value {line.get('value')} "
          f"e2e_ms {e.get('ms_per_step')} frac {r.get('frac')} parity {p.get('all_equal')} "
          f"cpu {c.get('value')} counts {line.get('counts')} clocks {line.get('clocks')}")
