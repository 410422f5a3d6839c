"""Summarise bench JSON lines: workload, value, ms, march frac, traffic/sample, e2e."""
import json
import sys

for path in sys.argv[1:]:
    for ln in open(path):
        ln = ln.strip()
        if not ln.startswith("{"):
            continue
        d = json.loads(ln)
        if "unavailable" in d:
            print(path, d)
            continue
        r = d.get("roofline") or {}
        e = d.get("e2e") or {}
        print(f"{d.get('lib', ''):<8} {d['config']['workload']:<40} {d['value']/1e9:7.3f} G/s  {d['ms_per_step']:8.3f} ms  "
              f"march {r.get('kernel_ms', 0):7.3f} ms frac {r.get('frac', 0):.3f}  "
              f"traffic/sample {r.get('traffic_per_sample') or 0:6.1f}  e2e {e.get('value', 0)/1e9:7.3f} G/s  "
              f"flags {d.get('detail', {}).get('flags', '')}")
