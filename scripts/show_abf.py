"""Summarise gpurun_out/abf_TAG.jsonl: scene mode flags -> frame ms, march ms, rest."""
import json, sys, collections
d = collections.defaultdict(list)
for l in open(sys.argv[1]):
    try:
        j = json.loads(l)
    except ValueError:
        continue
    r = j["roofline"]
    d[(j["config"]["scene"], j["config"]["mode"], j["config"]["flags"])].append((r["frame_kernels_ms"], r["kernel_ms"]))
for k, v in sorted(d.items()):
    f = min(x[0] for x in v); m = min(x[1] for x in v)
    print(f"{k[0]:10s} {k[1]:14s} {k[2]:>9s} frame {f:7.3f} march {m:7.3f} rest {f - m:7.3f}")
