"""Per-rank device time of a pixel-sharded frame, every rank of N emulated
one after another on one GPU (the kernels of a rank do not depend on the
others; the gather is not included).  Reports, per N, the slowest rank's
frame and N x that against the one-GPU frame (the strong-scaling ceiling
before the merge).  Usage: python scripts/shard_timing.py [scene [mode]]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cases as C  # noqa: E402
import paper_1908_01906_b200 as B  # noqa: E402
from paper_1908_01906_b200 import distributed as D  # noqa: E402
from paper_1908_01906_b200.device import device_scene_for  # noqa: E402

scene = sys.argv[1] if len(sys.argv) > 1 else "radial272"
mode = sys.argv[2] if len(sys.argv) > 2 else "skip-adaptive"
flags = int(sys.argv[3], 0) if len(sys.argv) > 3 else 0   # e.g. 0x300: 8 lanes per ray
sc = C.build_scene(B, scene)
cam, par = C.camera(B, scene), C.params(B, scene)
dev = device_scene_for(sc)
mid = {"reference": 0, "skip": 1, "skip-adaptive": 2}[mode]
stream = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
base = None
for n in (1, 2, 4, 8):
    per_rank, march = [], []
    for r in range(n):
        f = D.ShardedFrame(dev, sc, cam, mid, par, track=mid != 0, rank=r, world=n, compact=False,
                           flags=flags)
        for _ in range(3):
            f.run(stream)
        ms, mm = [], []
        for _ in range(10):
            flush.fill_(1)
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            me = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            f.run(stream, kernel_events=ev, march_events=me)
            torch.cuda.synchronize()
            ms.append(ev[0].elapsed_time(ev[1]))
            mm.append(me[0].elapsed_time(me[1]))
        per_rank.append(float(np.median(ms)))
        march.append(float(np.median(mm)))
    worst = max(per_rank)
    if n == 1:
        base = worst
    print(json.dumps({"scene": scene, "mode": mode, "n": n, "rank_ms": [round(x, 4) for x in per_rank],
                      "slowest_ms": round(worst, 4),
                      "march_ms": [round(x, 4) for x in march], "flags": hex(flags), "speedup_ceiling": round(base / worst, 3),
                      "efficiency_ceiling": round(base / worst / n, 3)}), flush=True)
