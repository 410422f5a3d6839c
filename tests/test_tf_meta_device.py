"""TF partition metadata on the GPU (tr_tf_meta_device, csrc/meta.cu)
equals the host restatement (tr_tf_meta, itself bit-identical to the
reference's transfer.py:95-141 -- test_scene_build.py) bit for bit."""

import numpy as np
import pytest

import cases
from paper_1908_01906_b200 import transfer as TR

pytestmark = pytest.mark.gpu


def _random_tf(B, rng, n, lo=-1.0, hi=2.0):
    table = rng.uniform(0.0, 1.0, (n, 4))
    table[rng.uniform(size=n) < 0.3, 3] = 0.0          # transparent stretches
    return B.TransferFunction(table=table, domain=(lo, hi))


def _same(a, b):
    for k in ("max_opacity", "raw_variance", "sigma", "active"):
        assert np.array_equal(a[k], b[k]), k


def test_device_meta_equals_host_random(B):
    rng = np.random.default_rng(11)
    for n in (2, 3, 7, 8, 9, 64, 129, 256, 300, 1000):
        tf = _random_tf(B, rng, n)
        lo = rng.uniform(-1.5, 2.5, 3000)
        w = rng.exponential(0.3, 3000) * (rng.uniform(size=3000) < 0.9)   # some empty ranges
        vr = np.stack([lo, lo + w], axis=1)
        vr[:5] = [[-5.0, -4.0], [3.0, 9.0], [-1.0, 2.0], [0.5, 0.5], [-1e300, 1e300]]
        _same(TR.partition_meta_arrays_device(tf, vr), TR.partition_meta_arrays(tf, vr))


def test_device_meta_equals_host_scenes(B):
    for recipe in ("radial16", "golden_radial4", "a6fog", "sinus"):
        sc = cases.build_scene(B, recipe)
        vr = np.array([p.value_range for p in sc.partitions])
        _same(TR.partition_meta_arrays_device(sc.tf, vr), TR.partition_meta_arrays(sc.tf, vr))


def test_set_transfer_function_on_device(B):
    a = cases.build_scene(B, "radial16")
    b = cases.build_scene(B, "radial16")
    b.set_transfer_function(a.tf, device="cuda:0")
    for x, y in zip(a.meta_state()[:2], b.meta_state()[:2]):
        assert np.array_equal(x, y)
    cam, par = cases.camera(B, "radial16"), cases.params(B, "radial16")
    fa, _ = B.render(a, cam, "skip-adaptive", par)
    fb, _ = B.render(b, cam, "skip-adaptive", par)
    assert np.array_equal(fa.rgba, fb.rgba)


def test_device_meta_rejects_inverted_range(B):
    tf = B.TransferFunction(table=np.ones((4, 4)), domain=(0.0, 1.0))
    with pytest.raises(RuntimeError):
        TR.partition_meta_arrays_device(tf, np.array([[0.5, 0.2]]))


def _host_steps(sig, par):
    import ctypes as C
    from paper_1908_01906_b200 import _lib
    sig = np.ascontiguousarray(sig, dtype=np.float64)
    out = np.empty_like(sig)
    ratio = np.empty(2 * len(sig))
    _lib.check(_lib.lib().tr_epoch_steps(len(sig), _lib.ptr(sig, C.c_double), float(par.s1),
                                         float(par.s2), float(par.p), out.ctypes.data,
                                         ratio.ctypes.data), "tr_epoch_steps")
    return out, ratio


@pytest.mark.parametrize("recipe", ["radial16", "golden_radial4", "a6fog", "radial59"])
def test_device_epoch_steps_equal_host(B, recipe):
    """Epoch step sizes (K:20-22) and K:27 exponents made on the device with
    the restated glibc pow are the host's bit for bit."""
    from paper_1908_01906_b200 import device as DV
    sc = cases.build_scene(B, recipe)
    par = cases.params(B, recipe)
    dev = DV.device_scene_for(sc)
    rng = np.random.default_rng(5)
    active, sigma, tf = sc.meta_state()
    sigmas = [np.asarray(sigma, dtype=np.float64),
              rng.choice([0.0, 1.0, 0.5, 2.0, 1e-300, 1 - 2**-52, 1e-12, 0.999], len(sigma)),
              rng.uniform(0.0, 1.5, len(sigma))]
    for p in (float(par.p), 1.0, 2.0, 3.7):
        par2 = B.AdaptiveParams(s1=par.s1, s2=par.s2, p=p,
                                termination_opacity=par.termination_opacity)
        for sg in sigmas:
            ep = DV.Epoch(dev, (active, sg, tf), par2)
            assert ep._step_dev == DV._steps_on_device(sg, float(par2.p))
            want, want_ratio = _host_steps(sg, par2)
            assert np.array_equal(ep.step_host, want)
            ratio = ep.buf[ep.desc.step_ratio - ep.buf.data_ptr():][:16 * len(sg)]
            assert np.array_equal(ratio.cpu().numpy().view(np.float64), want_ratio)
            if ep._step_dev:
                flag = ep.buf[ep.desc.inexact - ep.buf.data_ptr():][:4]
                assert int(flag.cpu().numpy().view(np.int32)[0]) == 0
            else:
                assert not ep.desc.inexact
