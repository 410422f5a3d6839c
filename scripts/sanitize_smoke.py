"""Small frames through every kernel path, for compute-sanitizer runs:
the point-location builds (device / device-nowalk / host), candidate raster / BSP walk / BVH, all modes, jitter, ragged frame, shards,
bricks, direct host framebuffer and staged outputs, chunked frames."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
import cases as C
import paper_1908_01906_b200 as B
from paper_1908_01906_b200 import bricks as BR, device as DV

for recipe in ("golden_radial4", "conftest48", "inside", "axis", "a6fog", "jitter8"):
    sc = C.build_scene(B, recipe)
    cam, par = C.camera(B, recipe), C.params(B, recipe)
    if recipe == "conftest48":
        cam = B.Camera(position=cam.position, look_at=cam.look_at, up=cam.up,
                       fov_y_deg=cam.fov_y_deg, width=45, height=38)
    for mode in ("reference", "skip", "skip-adaptive"):
        ref = None
        for flags in (0, 0x800000, 0x800008, 0x80, 0x400, 0x1000000, 0x2000000, 0x4000000):
            for jitter in (False, True):
                fb, st = B.render(sc, cam, mode, par, flags=flags, jitter=jitter)
                if not jitter:
                    if ref is None:
                        ref = fb.rgba.copy()
                    assert np.array_equal(ref, fb.rgba), (recipe, mode, flags)
    DV.DIRECT_HOST_OUTPUTS = False
    B.render(sc, cam, "skip-adaptive", par)
    DV.DIRECT_HOST_OUTPUTS = True
    DV.MAX_CHUNK_RAYS = 256
    DV.device_scene_for(sc)._frames.clear()
    B.render(sc, cam, "skip", par)
    DV.MAX_CHUNK_RAYS = 1 << 20
    DV.device_scene_for(sc)._frames.clear()
    br = BR.BrickRenderer(sc, 3, max(par.s1, par.s2))
    for mode in ("reference", "skip-adaptive"):
        a = B.render(sc, cam, mode, par)
        b = br.render(cam, mode, par)
        assert np.array_equal(a[0].rgba, b[0].rgba), (recipe, mode, "bricks")
    print(recipe, "ok", flush=True)
# the point-location builds (default: device LBVH + host walk tables): the
# device build alone (cell lists on the unstructured mesh) and the host build
for recipe in ("golden_radial4", "jitter8"):
    cam, par = C.camera(B, recipe), C.params(B, recipe)
    ref = {m: B.render(C.build_scene(B, recipe), cam, m, par)[0].rgba for m in ("reference", "skip-adaptive")}
    for build in ("device-nowalk", "host"):
        sc = C.build_scene(B, recipe)
        sc.point_build = build
        for mode in ("reference", "skip-adaptive"):
            assert np.array_equal(ref[mode], B.render(sc, cam, mode, par)[0].rgba), (recipe, build, mode)
    print(recipe, "point builds ok", flush=True)
# an HBM-generated grid: analytic cube leaves (default) and leaf headers
sc = C.build_scene(B, "grid12")
cam, par = C.camera(B, "radial16", scale=0.125), C.params(B, "radial16")
for mode in ("reference", "skip", "skip-adaptive"):
    a = B.render(sc, cam, mode, par)[0].rgba
    for flags in (0x8000000, 0x4000000, 0x2000000):
        assert np.array_equal(a, B.render(sc, cam, mode, par, flags=flags)[0].rgba), (mode, flags)
print("grid12 ok", flush=True)
print("sanitize smoke ok")
