"""Print ms_per_step and the isolated phases of bench.py JSON lines read from stdin."""
import json
import sys

for line in sys.stdin:
    if line.startswith("{"):
        d = json.loads(line)
        ph = d.get("phases_ms", {})
        print(f"ms_per_step {d['ms_per_step']:.1f}  " +
              " ".join(f"{k} {v:.1f}" for k, v in ph.items() if isinstance(v, float)))
