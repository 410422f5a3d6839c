"""bench.py's N > 1 path end to end on the one GPU of this run: `--gpus 2`
re-launches itself under torch.distributed.run, both ranks render their
interleaved tiles (gloo in place of NCCL, which refuses two ranks on one
device), rank 0 gathers the frame and prints one line for 2 GPUs whose frame
has the reference's sample total (radial59 skip-adaptive,
tests/golden/reference_frames.json)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def _two_ranks(*extra):
    env = dict(os.environ, TETRAY_DIST_BACKEND="gloo", TETRAY_ONE_DEVICE="1")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--scene",
                          "radial59", "--steps", "2", "--warmup", "1", "--no-cpu", "--no-traffic",
                          *extra],
                         capture_output=True, text=True, timeout=900, cwd=str(ROOT), env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    return d


@pytest.mark.parametrize("shard", ["pixels", "records"])
def test_bench_two_ranks_on_one_device(golden, shard):
    """The 512^2 frame split over 2 ranks (strong) or over 2 KD bricks."""
    d = _two_ranks("--shard", shard, "--scaling", "strong")
    want = golden["frames"]["radial59/skip-adaptive"]["total_samples"]
    assert d["config"]["samples_per_frame"] == want and d["scaling"] == "strong"
    if shard == "pixels":
        assert d["detail"]["comm_nranks"] == 2
        assert d["e2e"]["value"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    else:
        assert d["detail"]["exact_vs_one_gpu_render"] is True


def test_bench_two_ranks_weak_scaling():
    """The default at N > 1: the frame side x sqrt(2) (728^2), ~512^2 rays per rank."""
    d = _two_ranks()
    assert d["scaling"] == "weak"
    assert d["config"]["width"] == d["config"]["height"] == 728
    assert d["config"]["workload"] == "radial59 728x728 skip-adaptive"
    assert d["e2e"]["d2h_bytes_per_step"] >= 728 * 728 * 40
