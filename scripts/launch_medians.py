"""Median duration per kernel name in an ncu --csv launch list (last N launches each)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki][:48]].append(float(r[vi].replace(",", "")))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
for k, v in d.items():
    v = sorted(v[-n:])
    print(f"  {k:48s} n={len(v):3d} median {v[len(v) // 2] / 1e3:8.1f} us")
