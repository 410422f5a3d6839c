"""Per-kernel mean duration from an ncu --metrics gpu__time_duration.sum CSV log."""
import collections, csv, sys
lines = open(sys.argv[1]).read().splitlines()
i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[i:]))
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[1:]:
    v = float(r[vi]) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
    agg[r[ki].split("(")[0].replace("<unnamed>::", "")[-48:]].append(v)
for k, v in agg.items():
    print(f"{k:50s} n={len(v):3d} mean={sum(v)/len(v):9.1f} us")
