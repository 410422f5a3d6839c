"""Metadata-epoch consistency on the device path: a frame rendered while the
transfer function is being swapped corresponds to ONE complete epoch, never a
mix of two (the reference's contract, scene.py:48-50, and its test
pkg/tests/test_viewer.py:266-300, restated through this package's render()).
The device keeps a per-epoch upload cache (DeviceScene.epoch, keyed by the
immutable MetaEpoch object), so this also checks that a cached epoch is never
reused for a different TF.  Every distinct frame must equal the oracle's
frame of its epoch."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B(built_lib):
    import paper_1908_01906_b200 as B
    return B


def _setup(B, device_meta):
    mesh = B.generate_synthetic(2, "radial", B.Centering.VERTEX)
    tfs = [B.TransferFunction((0.0, 1.8),
                              np.array([[i / 8.0, 1.0 - i / 8.0, 0.3, 0.08 * i],
                                        [1.0 - i / 8.0, i / 8.0, 0.6, 0.05 * i]]))
           for i in range(8)]
    scene = B.Scene.build(mesh, tfs[0], kd_config=B.KdBuildConfig(10))
    cam = B.Camera(position=[6.0, 4.0, 5.0], look_at=[1.0, 1.0, 1.0], up=[0.0, 1.0, 0.0],
                   fov_y_deg=40.0, width=12, height=12)
    params = B.AdaptiveParams(s1=0.1, s2=0.3, p=2.0)
    return scene, cam, params, tfs


@pytest.mark.parametrize("device_meta", [False, True])
def test_concurrent_tf_updates_yield_whole_epoch_frames(B, device_meta):
    from oracle.oracle import OracleScene
    scene, cam, params, tfs = _setup(B, device_meta)
    dev = "cuda:0" if device_meta else None
    refs = {}
    orc = OracleScene(scene)
    for i, tf in enumerate(tfs):
        scene.set_transfer_function(tf, device=dev)
        fb, st = B.render(scene, cam, "skip-adaptive", params)
        rgba, samples, _, _ = orc.render(cam, "skip-adaptive", params)
        assert np.array_equal(fb.rgba, rgba) and np.array_equal(fb.samples, samples)
        refs[fb.rgba.tobytes()] = (i, fb.samples.tobytes())
    assert len(refs) == 8   # the epochs are visually distinct

    stop = threading.Event()
    errors = []

    def churn():
        try:
            while not stop.is_set():
                for tf in tfs:
                    scene.set_transfer_function(tf, device=dev)
        except Exception as e:   # pragma: no cover - reported below
            errors.append(e)

    seen = set()

    def renderer(n):
        try:
            for _ in range(n):
                fb, _ = B.render(scene, cam, "skip-adaptive", params)
                key = fb.rgba.tobytes()
                assert key in refs, "frame mixes two metadata epochs"
                assert refs[key][1] == fb.samples.tobytes()
                seen.add(refs[key][0])
        except Exception as e:
            errors.append(e)

    worker = threading.Thread(target=churn)
    readers = [threading.Thread(target=renderer, args=(40,)) for _ in range(2)]
    worker.start()
    for r in readers:
        r.start()
    try:
        for r in readers:
            r.join(timeout=300)
    finally:
        stop.set()
        worker.join(timeout=60)
    assert not errors, errors[0]
    assert len(seen) >= 2   # frames really came from several epochs


def test_stale_epoch_reupload_renders_the_same_frame(B):
    """mark_epochs_stale (bench.py's end-to-end steps): the cached epoch's
    page-locked block is copied again in place (after the first upload: one
    kernel reading it over PCIe and recomputing the steps); frames are
    unchanged even when the device copy was wiped in between."""
    scene, cam, params, tfs = _setup(B, False)
    from paper_1908_01906_b200.device import device_scene_for
    fb0, st0 = B.render(scene, cam, "skip-adaptive", params)
    dev = device_scene_for(scene)
    ep = next(iter(dev._epochs.values()))
    for i in range(3):
        dev.mark_epochs_stale()
        assert ep.stale
        if i:   # the re-upload really rewrites the device sections and steps
            ep.buf.zero_()
        fb, st = B.render(scene, cam, "skip-adaptive", params)
        assert not ep.stale and next(iter(dev._epochs.values())) is ep
        assert np.array_equal(fb.rgba, fb0.rgba) and st.total_samples == st0.total_samples


def test_held_frames_are_not_reused(B):
    """render() hands out page-locked result blocks again only once no
    returned array views them: frames (or slices of them) a caller keeps are
    never overwritten by later frames."""
    scene, cam, params, tfs = _setup(B, False)
    kept, copies = [], []
    for i in range(7):
        scene.set_transfer_function(tfs[i])
        fb, st = B.render(scene, cam, "skip-adaptive", params)
        keep = fb.rgba if i % 2 == 0 else fb.samples[3:9]   # a whole frame, or a slice
        kept.append(keep)
        copies.append(keep.copy())
        del fb, st
    for _ in range(6):   # more frames while the kept ones are alive
        B.render(scene, cam, "skip-adaptive", params)
    for k, c in zip(kept, copies):
        assert np.array_equal(k, c)
    from paper_1908_01906_b200.device import device_scene_for
    pool = device_scene_for(scene)._results
    kept.clear()
    n = len(pool.blocks)
    for _ in range(4):   # freed blocks are reused, not multiplied
        B.render(scene, cam, "skip-adaptive", params)
    assert len(pool.blocks) <= max(n, pool.KEEP)
