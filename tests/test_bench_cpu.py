"""bench.py's contract pieces that run without a GPU: the reference arm
(the stock reference render() from baseline/_ref, numba) on a small scene --
one JSON line, the same `config` dict the GPU arm prints, and none of this
repository's product libraries mapped into the process."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(not (ROOT / "baseline" / "_ref" / "tetray").exists(),
                    reason="the stock reference is not installed under baseline/_ref")
def test_reference_arm_runs_stock_render_without_product_library(built_oracle, tmp_path):
    env = {"NUMBA_CACHE_DIR": str(tmp_path / "numba"), "PATH": "/usr/bin:/bin"}
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--scene", "radial16", "--scale", "0.125", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, timeout=900,
                         cwd=str(ROOT), env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "samples/s" and d["value"] > 0
    assert d["config"] == {"workload": "radial16 64x64 skip-adaptive", "scene": "radial16",
                           "mode": "skip-adaptive", "width": 64, "height": 64, "n_tets": 20480,
                           "n_partitions": d["config"]["n_partitions"],
                           "samples_per_frame": d["config"]["samples_per_frame"]}
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "reference"
    assert not any("libtetray_b200" in p for p in d["detail"]["repo_libs_mapped"])


def test_workload_config_names_grid_scenes_by_their_radial_recipe():
    sys.path.insert(0, str(ROOT))
    import bench
    args = bench.parse(["--scene", "grid272"])
    assert bench.public_name(args.scene) == "radial272"
    a = bench.workload_config(args, 100618240, 4096, 34935023)
    b = bench.workload_config(bench.parse(["--scene", "radial272"]), 100618240, 4096, 34935023)
    assert a == b and a["workload"] == "radial272 512x512 skip-adaptive"


def test_weak_scaling_grows_the_frame_side_with_sqrt_n():
    sys.path.insert(0, str(ROOT))
    import bench
    sides = {}
    for n in (1, 2, 4, 8):
        args = bench.parse(["--gpus", str(n)])
        bench.weak_scale(args, n)
        sides[n] = bench.workload_config(args, 1, 1, 1)["width"]
    assert sides == {1: 512, 2: 728, 4: 1024, 8: 1448}
    for n in (1, 2, 4, 8):   # rays per GPU within 1% of the 512^2 frame
        assert abs(sides[n] ** 2 / n / 512 ** 2 - 1.0) < 0.011
    args = bench.parse(["--gpus", "8", "--scaling", "strong"])
    bench.weak_scale(args, 8)
    assert bench.workload_config(args, 1, 1, 1)["width"] == 512
