"""The C-ABI library loads, exports every symbol include/tetray_b200.h
declares, and its record layouts match the header.  No device calls."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "tetray_b200.h"


@pytest.fixture(scope="module")
def L(built_lib):
    from paper_1908_01906_b200 import _lib
    return _lib


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tr_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported_and_bound(L):
    lib = L.lib()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(names) == sorted(L.EXPORTED_SYMBOLS)


def test_record_layouts_match_header(L):
    assert L.TET_RECORD_DTYPE.itemsize == 128
    assert L.PNODE_DTYPE.itemsize == 64
    assert L.PLEAF_DTYPE.itemsize == 64
    assert L.BNODE_DTYPE.itemsize == 112
    assert C.sizeof(L.TrFrame) % 8 == 0
    assert L.lib().tr_abi_version() == 2


def test_ctypes_structs_match_the_c_layouts(L):
    sizes = (C.c_int64 * 11)()
    assert L.lib().tr_struct_sizes(sizes, 11) == 0
    want = [C.sizeof(L.TrDeviceScene), C.sizeof(L.TrEpoch), C.sizeof(L.TrFrame),
            C.sizeof(L.TrOutputs), C.sizeof(L.TrBricks), L.RAY_STATE_BYTES,
            L.TET_RECORD_DTYPE.itemsize, L.PNODE_DTYPE.itemsize, L.PLEAF_DTYPE.itemsize,
            L.BNODE_DTYPE.itemsize, L.KNODE_DTYPE.itemsize]
    assert list(sizes) == want


def test_errors_are_reported_not_aborted(L):
    lib = L.lib()
    rc = lib.tr_render_frame(None, None, None, None, None)
    assert rc != 0
    assert b"null" in lib.tr_last_error()
    with pytest.raises(RuntimeError):
        L.check(rc, "tr_render_frame")


def test_tile_helpers_match_python(L):
    from paper_1908_01906_b200 import distributed as D
    lib = L.lib()
    for w, h, n in [(512, 512, 1), (513, 37, 3), (9, 7, 8), (1, 1, 4)]:
        assert lib.tr_num_tiles(w, h) == D.num_tiles(w, h)
        assert lib.tr_slots_per_rank(w, h, n) == D.slots_per_rank(w, h, n)


def test_host_step_size_and_opacity_match_reference(L):
    import json
    misc = json.loads((ROOT / "tests" / "golden" / "reference_misc.json").read_text())
    lib = L.lib()
    for s1, s2, p, sig, want in misc["step_size"]:
        assert lib.tr_step_size(s1, s2, p, sig) == want
    for a, s, s1, want in misc["opacity_correction"]:
        assert lib.tr_opacity_correction(a, s, s1) == want


def test_product_path_has_no_cpu_fallback(L, monkeypatch):
    """render() must fail loudly without a CUDA device."""
    import torch

    import cases as Cs
    import paper_1908_01906_b200 as B
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    sc = Cs.build_scene(B, "golden_radial4")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        B.render(sc, Cs.camera(B, "golden_radial4"), "skip", Cs.params(B, "golden_radial4"))


def test_product_package_never_imports_the_oracle():
    pkg = ROOT / "paper_1908_01906_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "oracle" not in re.sub(r'""".*?"""|#.*', "", src, flags=re.S), f
