"""Build one scene's device-resident point structures once with the device
point build (for an ncu launch list of csrc/pbuild.cu's kernels).
Usage: python scripts/pbuild_once.py radial272"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import torch  # noqa: E402
import cases as C  # noqa: E402
import paper_1908_01906_b200 as B  # noqa: E402
from paper_1908_01906_b200.device import device_scene_for  # noqa: E402

sc = C.build_scene(B, sys.argv[1])
sc.point_build = "device"
dev = device_scene_for(sc)
torch.cuda.synchronize()
print(sys.argv[1], dev.build_phases, flush=True)
