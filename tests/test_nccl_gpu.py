"""The NCCL transport of the sharded frame (distributed.py: gather of the
compact tile slots to rank 0, int64 reduce of the counters, tr_scatter_tiles)
executed on the one GPU of this run: a one-rank NCCL group through
render_sharded (compact slots forced), bit-identical to render().  The
multi-rank split itself is covered over gloo (test_sharded_dist_gpu.py,
test_bench_dist_gpu.py)."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import sys
sys.path[:0] = [{root!r}, {tests!r}]
import numpy as np, torch, torch.distributed as dist
import cases
import paper_1908_01906_b200 as B
from paper_1908_01906_b200.distributed import render_sharded
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
assert dist.get_backend() == "nccl"
for recipe, scale in (("radial16", 0.25), ("golden_radial4", 1.0), ("radial59", 0.5)):
    sc = cases.build_scene(B, recipe)
    cam, par = cases.camera(B, recipe, scale=scale), cases.params(B, recipe)
    for mode in ("reference", "skip", "skip-adaptive"):
        a, sa = render_sharded(sc, cam, mode, par)
        b, sb = B.render(sc, cam, mode, par)
        assert np.array_equal(a.rgba, b.rgba) and np.array_equal(a.samples, b.samples), (recipe, mode)
        assert sa.total_samples == sb.total_samples
        assert sa.partitions_visited_mean == sb.partitions_visited_mean
        if sb.per_partition_samples is not None:
            assert np.array_equal(sa.per_partition_samples, sb.per_partition_samples)
dist.destroy_process_group()
print("nccl ok")
"""


def test_nccl_one_rank_sharded_frame_equals_render(built_lib):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    code = SCRIPT.format(root=str(ROOT), tests=str(ROOT / "tests"))
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=600, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    assert "nccl ok" in res.stdout
