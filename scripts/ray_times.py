"""March timeline per ray (diagnostics library built with -DTR_RAY_TIMES=1:
each ray's start / end globaltimer in rgba.r / .g):
TETRAY_B200_LIB=build/ab/times/libtetray_b200.so python scripts/ray_times.py [scene [N]]
Prints the march span, when the last ray started, the samples of the rays
that finish last, and the per-round time of the longest rays."""
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

scene = sys.argv[1] if len(sys.argv) > 1 else "grid272"
sc = C.build_scene(B, scene)
cam, par = C.camera(B, scene), C.params(B, scene)
dev = device_scene_for(sc)
stream = torch.cuda.current_stream()
for n in [int(x) for x in (sys.argv[2:] or ["1", "8"])]:
    for mode, mid in (("skip-adaptive", 2), ("reference", 0)):
        f = D.ShardedFrame(dev, sc, cam, mid, par, track=mid != 0, rank=0, world=n, compact=False)
        for _ in range(3):
            f.run(stream)
        f.rgba.zero_()   # other ranks' tiles (N > 1) stay zero: not counted
        f.run(stream)
        torch.cuda.synchronize()
        rgba = f.rgba.cpu().numpy().reshape(-1, 4)
        smp = f.samples.cpu().numpy().reshape(-1)
        marched = rgba[:, 1] > 0
        t0, t1 = rgba[marched, 0], rgba[marched, 1]
        s = smp[marched]
        base = t0.min()
        st, en = (t0 - base) / 1e3, (t1 - base) / 1e3   # us
        span = en.max()
        dur = en - st
        print(f"{scene} {mode} N={n}: rays {marched.sum()}, march span {span:.0f} us, "
              f"last start {st.max():.0f} us, mean samples {s.mean():.0f}, max {s.max()}", flush=True)
        late = en > 0.9 * span
        print(f"  rays ending in the last 10%: {late.sum()}, their samples mean {s[late].mean():.0f} "
              f"max {s[late].max()}, start mean {st[late].mean():.0f} us, duration mean "
              f"{dur[late].mean():.0f} us", flush=True)
        top = np.argsort(-s)[:20]
        print(f"  20 longest rays: samples {s[top].min()}-{s[top].max()}, start "
              f"{st[top].min():.0f}-{st[top].max():.0f} us, end {en[top].min():.0f}-{en[top].max():.0f} us, "
              f"us per 4-sample round {np.median(dur[top] / (s[top] / 4.0)):.2f}", flush=True)
        for q in (0.25, 0.5, 0.75, 0.9, 0.99):
            print(f"  {int(q * 100)}% of rays done by {np.quantile(en, q):.0f} us", flush=True)
        # active rays over time
        ts = np.linspace(0, span, 11)
        act = [int(((st <= t) & (en > t)).sum()) for t in ts]
        print("  active rays at 0,10,..100% of span:", act, flush=True)
