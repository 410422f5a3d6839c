"""ctypes binding of libtetray_b200.so (the C ABI declared in include/tetray_b200.h).

There is no fallback: if the shared library is missing or fails to load,
every product entry point raises.  Build it with `__graft_entry__.build()` or
`python -m paper_1908_01906_b200._build`.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

import os

# TETRAY_B200_LIB: an alternative build of the same library (A/B tuning runs)
LIB_PATH = Path(os.environ.get("TETRAY_B200_LIB") or
                Path(__file__).resolve().parent / "libtetray_b200.so")

c_i64p = C.POINTER(C.c_int64)
c_f64p = C.POINTER(C.c_double)
c_u8p = C.POINTER(C.c_uint8)
c_u32p = C.POINTER(C.c_uint32)


class TrDeviceScene(C.Structure):
    _fields_ = [
        ("tets", C.c_void_p), ("pnodes", C.c_void_p), ("pleaves", C.c_void_p),
        ("pleaf_ids", C.c_void_p),
        ("n_tets", C.c_int64), ("n_pnodes", C.c_int64), ("n_pleaves", C.c_int64),
        ("centering", C.c_int32), ("pad0", C.c_int32),
        ("bnodes", C.c_void_p), ("part_lo", C.c_void_p), ("part_hi", C.c_void_p),
        ("n_parts", C.c_int64), ("n_bnodes", C.c_int64),
        ("mesh_lo", C.c_double * 3), ("mesh_hi", C.c_double * 3),
        ("pgrid", C.c_void_p), ("pgrid_leaf", C.c_void_p), ("gdim", C.c_int32 * 3),
        ("pad1", C.c_int32),
        ("gorg", C.c_double * 3), ("gscale", C.c_double * 3),
        ("knodes", C.c_void_p), ("kleaf_pids", C.c_void_p), ("n_knodes", C.c_int64),
        ("kroot", C.c_double * 6),
        ("cell_off", C.c_void_p), ("cell_recs", C.c_void_p), ("tbox", C.c_void_p),
        ("cdim", C.c_int32 * 3), ("cells_first", C.c_int32),
        ("corg", C.c_double * 3), ("cscale", C.c_double * 3),
        ("pgrid_pred", C.c_void_p), ("pred_classes", C.c_int32), ("pad2", C.c_int32),
        ("pred_class", C.c_float * 24),
        ("grid_n", C.c_int64), ("grid_pad", C.c_double), ("grid_brick", C.c_int32),
        ("pad3", C.c_int32), ("class_walk", C.c_void_p),
    ]


class TrEpoch(C.Structure):
    _fields_ = [
        ("active", C.c_void_p), ("bnode_active", C.c_void_p), ("step", C.c_void_p),
        ("tf_table", C.c_void_p), ("n_tf", C.c_int64), ("tf_lo", C.c_double),
        ("tf_hi", C.c_double), ("knode_active", C.c_void_p), ("step_ratio", C.c_void_p),
        ("inexact", C.c_void_p),
    ]


class TrEpochUpload(C.Structure):
    _fields_ = [
        ("n_parts", C.c_int64), ("sigma", C.c_void_p), ("active", C.c_void_p),
        ("bnode_active", C.c_void_p), ("knode_active", C.c_void_p), ("n_bnodes", C.c_int64),
        ("n_knodes", C.c_int64), ("tf_table", C.c_void_p), ("n_tf", C.c_int64),
        ("tf_lo", C.c_double), ("tf_hi", C.c_double), ("s1", C.c_double), ("s2", C.c_double),
        ("p", C.c_double), ("steps_on_device", C.c_int32), ("packed", C.c_int32),
        ("host_buf", C.c_void_p), ("dev_buf", C.c_void_p), ("buf_bytes", C.c_int64),
    ]


class TrFrame(C.Structure):
    _fields_ = [
        ("cam_pos", C.c_double * 3), ("cam_right", C.c_double * 3),
        ("cam_up", C.c_double * 3), ("cam_fwd", C.c_double * 3),
        ("tan_half", C.c_double), ("aspect", C.c_double),
        ("width", C.c_int64), ("height", C.c_int64),
        ("jitter", C.c_int32), ("mode", C.c_int32),
        ("s1", C.c_double), ("term", C.c_double), ("eps", C.c_double),
        ("bg", C.c_double * 4),
        ("track_ppart", C.c_int32), ("shard_rank", C.c_int32), ("shard_count", C.c_int32),
        ("compact", C.c_int32), ("flags", C.c_int32), ("pad0", C.c_int32),
    ]


class TrOutputs(C.Structure):
    _fields_ = [
        ("rgba", C.c_void_p), ("samples", C.c_void_p), ("visited", C.c_void_p),
        ("ppart", C.c_void_p), ("totals", C.c_void_p), ("work", C.c_void_p),
        ("scratch", C.c_void_p), ("scratch_bytes", C.c_int64),
        ("ev_march_begin", C.c_void_p), ("ev_march_end", C.c_void_p),
    ]


class TrBricks(C.Structure):
    _fields_ = [
        ("rank", C.c_int32), ("n_bricks", C.c_int32),
        ("owner", C.c_void_p), ("brick_lo", C.c_void_p), ("brick_hi", C.c_void_p),
        ("state", C.c_void_p), ("queue", C.c_void_p), ("counters", C.c_void_p),
        ("zero_foreign", C.c_int32), ("write_background", C.c_int32),
        ("exchange_tag", C.c_uint32), ("n_peers", C.c_int32),
        ("peer_inbox", C.c_void_p), ("inbox", C.c_void_p),
    ]


RAY_STATE_BYTES = 64   # TrRayState

# numpy views of the device record layouts (sizes pinned by tests against the header)
TET_RECORD_DTYPE = np.dtype([("inv", "<f8", 9), ("orig", "<f8", 3), ("f", "<f8", 4)])
PNODE_DTYPE = np.dtype([("lo0", "<f4", 3), ("hi0", "<f4", 3), ("lo1", "<f4", 3),
                        ("hi1", "<f4", 3), ("child", "<i4", 2), ("minid", "<u4", 2)])
PLEAF_DTYPE = np.dtype([("ex_lo", "<f4", 3), ("ex_hi", "<f4", 3), ("start", "<u4"),
                        ("count", "<u4"), ("walk", "<u4", 8)])
BNODE_DTYPE = np.dtype([("box", "<f8", (2, 6)), ("child", "<i4", 2), ("pad", "<i4", 2)])
KNODE_DTYPE = np.dtype([("split", "<f8"), ("info", "<i4"), ("aux", "<i4")])

TR_FLAG_NO_GRID = 2
TR_FLAG_STATS = 4
TR_FLAG_NO_BSP = 8
STAT_NAMES = ["rounds", "partial_rounds", "lane_samples", "found", "grid_hits", "descents",
              "inline_intervals", "pow_calls", "trace_intervals", "trace_rays", "bsp_overflow",
              "bsp_cells", "trace_max_intervals", "bsp_nodes", "trace_max_nodes", "max_ray_samples",
              "tile_cycles", "tile_max_cycles", "march_t0", "march_tq", "march_t1"]
CHILD_NONE = -2**31

# (name, restype, argtypes) for every symbol include/tetray_b200.h declares
_SIGNATURES = [
    ("tr_kd_build", C.c_int, [C.c_int64, c_f64p, C.c_int64, c_i64p, c_f64p, C.c_int32, c_f64p,
                              c_f64p, C.c_int64, C.c_int64, C.POINTER(C.c_void_p)]),
    ("tr_kd_build_grid", C.c_int, [C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_int32,
                                   C.POINTER(C.c_void_p)]),
    ("tr_kd_sizes", C.c_int, [C.c_void_p, c_i64p]),
    ("tr_kd_copy", C.c_int, [C.c_void_p, c_i64p, c_i64p, c_f64p, c_f64p, c_f64p, c_f64p, c_f64p]),
    ("tr_pbvh_build", C.c_int, [C.c_int64, c_f64p, c_f64p, C.c_int32, C.POINTER(C.c_void_p)]),
    ("tr_pbvh_sizes", C.c_int, [C.c_void_p, c_i64p]),
    ("tr_pbvh_copy", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("tr_leaf_walk", C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p]),
    ("tr_grid_walk_pred", C.c_int, [C.c_double, C.c_void_p, C.c_void_p]),
    ("tr_pbvh_grid", C.c_int, [C.c_void_p, C.c_void_p, c_f64p, c_f64p, C.c_void_p]),
    ("tr_pbvh_coverage", C.c_double, [C.c_void_p]),
    ("tr_cells_build", C.c_int, [C.c_void_p, c_f64p, c_f64p, C.c_int32, C.c_int32,
                                 C.POINTER(C.c_void_p)]),
    ("tr_cells_sizes", C.c_int, [C.c_void_p, c_i64p]),
    ("tr_cells_copy", C.c_int, [C.c_void_p, C.c_void_p, c_f64p, c_f64p, C.c_void_p, C.c_void_p,
                                C.c_void_p]),
    ("tr_bbvh_build", C.c_int, [C.c_int64, c_f64p, c_f64p, C.POINTER(C.c_void_p)]),
    ("tr_bbvh_sizes", C.c_int, [C.c_void_p, c_i64p]),
    ("tr_bbvh_copy", C.c_int, [C.c_void_p, C.c_void_p]),
    ("tr_bbvh_activity", C.c_int, [C.c_void_p, c_u8p, c_u8p]),
    ("tr_bnodes_activity", C.c_int, [C.c_int64, C.c_void_p, c_u8p, c_u8p]),
    ("tr_kbsp_build", C.c_int, [C.c_int64, c_f64p, c_f64p, C.POINTER(C.c_void_p)]),
    ("tr_kbsp_sizes", C.c_int, [C.c_void_p, c_i64p]),
    ("tr_kbsp_copy", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, c_f64p]),
    ("tr_knodes_activity", C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, c_u8p, c_u8p]),
    ("tr_host_free", None, [C.c_void_p]),
    ("tr_pack_tets", C.c_int, [C.c_int64, c_i64p, c_f64p, c_f64p, c_f64p, C.c_int32, C.c_void_p,
                               C.c_void_p]),
    ("tr_tet_boxes", C.c_int, [C.c_int64, c_f64p, c_i64p, C.c_double, c_f64p, c_f64p]),
    ("tr_tf_meta", C.c_int, [C.c_int64, c_f64p, c_f64p, C.c_int64, C.c_double, C.c_double,
                             c_f64p, c_f64p, c_f64p, c_u8p]),
    ("tr_tf_meta_device", C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_double,
                                    C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p]),
    ("tr_epoch_steps_device", C.c_int, [C.c_int64, C.c_void_p, C.c_double, C.c_double, C.c_double,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("tr_epoch_bytes", C.c_int64, [C.c_int64, C.c_int64, C.c_int64, C.c_int64]),
    ("tr_epoch_upload", C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                  C.c_int64, C.c_void_p, C.c_int64, C.c_double, C.c_double, C.c_double,
                                  C.c_double, C.c_double, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64,
                                  C.POINTER(TrEpoch), C.POINTER(C.c_int64), C.c_void_p]),
    ("tr_epoch_steps", C.c_int, [C.c_int64, c_f64p, C.c_double, C.c_double, C.c_double, C.c_void_p,
                                 C.c_void_p]),
    ("tr_step_sizes", C.c_int, [C.c_int64, c_f64p, C.c_double, C.c_double, C.c_double, c_f64p]),
    ("tr_step_size", C.c_double, [C.c_double, C.c_double, C.c_double, C.c_double]),
    ("tr_opacity_correction", C.c_double, [C.c_double, C.c_double, C.c_double]),
    ("tr_host_device_pointer", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tr_host_register", C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_void_p)]),
    ("tr_host_unregister", C.c_int, [C.c_void_p]),
    ("tr_memset_async", C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p]),
    ("tr_copy_async", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    ("tr_pow_glibc_available", C.c_int, []),
    ("tr_pow_glibc_host", C.c_double, [C.c_double, C.c_double, C.POINTER(C.c_int32)]),
    ("tr_pow_glibc_batch", C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("tr_render_sync", C.c_int, [C.POINTER(TrDeviceScene), C.POINTER(TrEpoch), C.POINTER(TrFrame),
                                 C.POINTER(TrOutputs), C.c_int64, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.POINTER(C.c_float), C.c_void_p]),
    ("tr_epoch_upload_s", C.c_int, [C.POINTER(TrEpochUpload), C.POINTER(TrEpoch),
                                    C.POINTER(C.c_int64), C.c_void_p]),
    ("tr_render_frame", C.c_int, [C.POINTER(TrDeviceScene), C.POINTER(TrEpoch),
                                  C.POINTER(TrFrame), C.POINTER(TrOutputs), C.c_void_p]),
    ("tr_brick_trace", C.c_int, [C.POINTER(TrDeviceScene), C.POINTER(TrEpoch), C.POINTER(TrFrame),
                                 C.POINTER(TrBricks), C.POINTER(TrOutputs), C.c_void_p]),
    ("tr_brick_round", C.c_int, [C.POINTER(TrDeviceScene), C.POINTER(TrEpoch), C.POINTER(TrFrame),
                                 C.POINTER(TrBricks), C.POINTER(TrOutputs), C.c_void_p]),
    ("tr_grid_scene_sizes", C.c_int, [C.c_int64, c_i64p, c_i64p, c_i64p]),
    ("tr_grid_scene_build", C.c_int, [C.c_int64, C.c_int32, C.c_double, c_f64p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("tr_pbvh_build_device", C.c_int, [C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_double,
                                       C.c_int32, C.c_double, C.c_int32, C.c_int32, C.c_void_p,
                                       C.POINTER(C.c_void_p)]),
    ("tr_dpb_sizes", C.c_int, [C.c_void_p, c_i64p]),
    ("tr_dpb_grid", C.c_int, [C.c_void_p, C.c_void_p, c_f64p, c_f64p, c_f64p, C.c_void_p, c_f64p,
                              c_f64p]),
    ("tr_dpb_walk", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("tr_dpb_copy", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p]),
    ("tr_dpb_free", None, [C.c_void_p]),
    ("tr_pack_tets_device", C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("tr_ipc_alloc", C.c_int, [C.c_int64, C.POINTER(C.c_void_p), C.c_void_p]),
    ("tr_ipc_open", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tr_ipc_close", C.c_int, [C.c_void_p]),
    ("tr_dev_free", C.c_int, [C.c_void_p]),
    ("tr_upload", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    ("tr_quantize_rgb", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    ("tr_heatmap_rgb", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p]),
    ("tr_ssim_rgb", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_void_p,
                              C.c_void_p, C.c_double, C.c_double, C.c_void_p, C.c_void_p]),
    ("tr_field_at_many", C.c_int, [C.POINTER(TrDeviceScene), C.c_int64, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p]),
    ("tr_scatter_tiles", C.c_int, [C.c_int64, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p]),
    ("tr_num_tiles", C.c_int64, [C.c_int64, C.c_int64]),
    ("tr_scratch_bytes", C.c_int64, [C.c_int64]),
    ("tr_slots_per_rank", C.c_int64, [C.c_int64, C.c_int64, C.c_int32]),
    ("tr_last_launch", C.c_int, [c_i64p]),
    ("tr_kernel_stats", C.c_int, [c_i64p, C.c_int32, C.c_int32]),
    ("tr_last_error", C.c_char_p, []),
    ("tr_abi_version", C.c_int, []),
    ("tr_struct_sizes", C.c_int, [C.POINTER(C.c_int64), C.c_int32]),
]

EXPORTED_SYMBOLS = [name for name, _, _ in _SIGNATURES]

_lib = None


def lib():
    """The loaded library (loaded once).  Raises if it is missing."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH.name} is not built; run __graft_entry__.build() "
                "(there is no CPU fallback for the render path)")
        L = C.CDLL(str(LIB_PATH))
        for name, res, args in _SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().tr_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed (code {rc}): {msg}")


def ptr(a: np.ndarray, ctype):
    """ctypes pointer to a C-contiguous numpy array (caller keeps `a` alive)."""
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


def vptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return C.c_void_p(a.ctypes.data)
