"""The multi-GPU frame path on ONE GPU: every rank's shard is
rendered with the same tr_render_frame call bench.py's ranks make (TrFrame
shard_rank / shard_count, compact slot-major outputs), the NCCL all-gather is
stood in for by concatenating the ranks' buffers in rank order (what
all_gather_into_tensor produces) and the all-reduce by summing the counters;
tr_scatter_tiles then rebuilds the image.  The result must equal the 1-GPU
frame bit for bit, so only the NCCL transport itself is left untested here
(tests/test_distributed.py covers the collective plumbing with gloo)."""

import ctypes as C

import numpy as np
import pytest

import cases
from paper_1908_01906_b200 import _lib
from paper_1908_01906_b200 import distributed as D

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("recipe,mode,world", [
    ("conftest48", "skip", 2), ("radial16", "skip-adaptive", 3), ("radial16", "reference", 8),
    ("radial59", "skip-adaptive", 8), ("a6fog", "skip", 5)])
def test_shards_reassemble_the_single_gpu_frame(B, recipe, mode, world):
    import torch
    from paper_1908_01906_b200.device import device_scene_for
    sc = cases.build_scene(B, recipe)
    cam, par = cases.camera(B, recipe), cases.params(B, recipe)
    if recipe == "conftest48":   # ragged frame: partial tiles on the right and bottom
        cam = B.Camera(position=cam.position, look_at=cam.look_at, up=cam.up,
                       fov_y_deg=cam.fov_y_deg, width=45, height=38)
    full, st = B.render(sc, cam, mode, par)
    dev = device_scene_for(sc)
    mode_id = {"reference": 0, "skip": 1, "skip-adaptive": 2}[mode]
    track = mode != "reference"
    w, h = cam.width, cam.height
    slots = D.slots_per_rank(w, h, world)
    stream = torch.cuda.current_stream()
    rgba, samples, visited, counters = [], [], [], []
    for r in range(world):
        frame = dev._frame_desc(sc, cam, mode_id, par, False, track, 0, r, world, True)
        fb = dev.frame_buffers(w, h, compact_slots=slots)
        ep = dev.epoch(sc.meta_state(), par)
        dev.launch(frame, ep, fb, stream)
        rgba.append(fb.rgba.clone())
        samples.append(fb.samples.clone())
        visited.append(fb.visited.clone())
        counters.append(fb.counters.clone())
    g_rgba, g_samples, g_visited = torch.cat(rgba), torch.cat(samples), torch.cat(visited)
    tot = torch.stack(counters).sum(dim=0)
    out_rgba = torch.empty((h * w, 4), dtype=torch.float64, device=g_rgba.device)
    out_samples = torch.empty(h * w, dtype=torch.int64, device=g_rgba.device)
    out_visited = torch.empty(h * w, dtype=torch.int32, device=g_rgba.device)
    _lib.check(_lib.lib().tr_scatter_tiles(
        w, h, world, C.c_void_p(g_rgba.data_ptr()), C.c_void_p(g_samples.data_ptr()),
        C.c_void_p(g_visited.data_ptr()), slots, C.c_void_p(out_rgba.data_ptr()),
        C.c_void_p(out_samples.data_ptr()), C.c_void_p(out_visited.data_ptr()),
        C.c_void_p(stream.cuda_stream)), "tr_scatter_tiles")
    assert np.array_equal(out_rgba.view(h, w, 4).cpu().numpy(), full.rgba)
    assert np.array_equal(out_samples.view(h, w).cpu().numpy(), full.samples)
    t = tot.cpu().numpy()
    assert int(t[0]) == st.total_samples
    assert float(np.float64(t[1]) / np.float64(w * h)) == st.partitions_visited_mean
    if track:
        assert np.array_equal(t[3:], st.per_partition_samples)
