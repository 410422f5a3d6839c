"""Host logic of the point-location build choice (device.point_build_mode):
the default is the device build (csrc/pbuild.cu), overridable per scene or by
$TETRAY_POINT_BUILD; bad names raise; one-leaf meshes keep the host build."""

import types

import numpy as np
import pytest

from paper_1908_01906_b200 import device as DV


def _scene(n_tets, **kw):
    return types.SimpleNamespace(mesh=types.SimpleNamespace(n_tets=n_tets), **kw)


def test_default_is_the_device_build(monkeypatch):
    monkeypatch.delenv(DV.POINT_BUILD_ENV, raising=False)
    assert DV.point_build_mode(_scene(1000)) == "device"


def test_scene_attribute_and_environment(monkeypatch):
    monkeypatch.setenv(DV.POINT_BUILD_ENV, "host")
    assert DV.point_build_mode(_scene(1000)) == "host"
    assert DV.point_build_mode(_scene(1000, point_build="device-nowalk")) == "device-nowalk"
    monkeypatch.setenv(DV.POINT_BUILD_ENV, "device-hostwalk")
    assert DV.point_build_mode(_scene(1000)) == "device-hostwalk"


def test_bad_names_raise(monkeypatch):
    monkeypatch.delenv(DV.POINT_BUILD_ENV, raising=False)
    with pytest.raises(ValueError):
        DV.point_build_mode(_scene(1000, point_build="gpu"))
    monkeypatch.setenv(DV.POINT_BUILD_ENV, "fast")
    with pytest.raises(ValueError):
        DV.point_build_mode(_scene(1000))


def test_one_leaf_meshes_use_the_host_build(monkeypatch):
    monkeypatch.delenv(DV.POINT_BUILD_ENV, raising=False)
    assert DV.point_build_mode(_scene(8)) == "host"
    assert DV.point_build_mode(_scene(5, point_build="device")) == "host"


def test_device_build_symbols_exported():
    from paper_1908_01906_b200 import _lib
    L = _lib.lib()
    for name in ("tr_pbvh_build_device", "tr_dpb_sizes", "tr_dpb_grid", "tr_dpb_walk", "tr_dpb_copy",
                 "tr_dpb_free", "tr_pack_tets_device", "tr_upload", "tr_ipc_alloc", "tr_ipc_open",
                 "tr_ipc_close", "tr_dev_free"):
        assert hasattr(L, name), name
    # argument validation happens before any CUDA call
    h = _lib.C.c_void_p()
    assert L.tr_pbvh_build_device(0, None, 0, None, 0.0, 8, 0.9, 2, 96, None, _lib.C.byref(h)) != 0
    assert b"invalid" in L.tr_last_error()
    assert L.tr_upload(None, None, -1, None) != 0
    assert L.tr_upload(None, None, 0, None) == 0
