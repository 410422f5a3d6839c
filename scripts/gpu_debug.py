"""Per-case GPU vs oracle comparison with verbose diagnostics (debug aid)."""
import sys, traceback
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
import cases as C
import paper_1908_01906_b200 as B
from oracle.oracle import OracleScene

only = sys.argv[1:]
for cid, recipe, modes, jitter in C.FRAME_CASES + C.BIG_CASES:
    if only and cid not in only:
        continue
    try:
        sc = C.build_scene(B, recipe)
        orc = OracleScene(sc)
        cam, par = C.camera(B, recipe), C.params(B, recipe)
        for mode in modes:
            ref = orc.render(cam, mode, par, jitter=jitter)
            for flags in (0, 3, 8, 0x40, 0x80, 0x1000, 0x300):
                fb, st = B.render(sc, cam, mode, par, jitter=jitter, flags=flags)
                ds = int((fb.samples != ref[1]).sum())
                dr = int((fb.rgba != ref[0]).any(axis=2).sum())
                mx = float(np.abs(fb.rgba - ref[0]).max())
                pp = None if ref[3] is None else int((st.per_partition_samples != ref[3]).sum())
                print(f"{cid:22s} {mode:14s} flags={flags} samples_diff_px={ds} rgba_diff_px={dr} "
                      f"max_abs={mx:.3g} ppart_diff={pp} tot={st.total_samples}/{int(ref[1].sum())} "
                      f"vis={st.partitions_visited_mean}/{float(ref[2].mean())} ms={st.device_ms:.3f}",
                      flush=True)
                if ds and ds < 5:
                    idx = np.argwhere(fb.samples != ref[1])[:3]
                    for iy, ix in idx:
                        print("   px", ix, iy, fb.samples[iy, ix], ref[1][iy, ix], fb.rgba[iy, ix], ref[0][iy, ix])
    except Exception:
        traceback.print_exc()
        print(f"{cid}: EXCEPTION", flush=True)
