"""Small frames through every frame-pipeline variant, for compute-sanitizer:

  compute-sanitizer --tool memcheck python tools/sanitize_frames.py
  compute-sanitizer --tool racecheck python tools/sanitize_frames.py

Renders golden model 'smoke' (and its iso variant) at 96x64 under each
xb_tuning variant of the parity matrix, plus the cell-location path, the ray
batch API and the builders."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402

from paper_2009_03076_b200 import _native as N  # noqa: E402
from paper_2009_03076_b200.accel import TransferFunction  # noqa: E402
from paper_2009_03076_b200.bricks import BrickBuildParams, build_bricks  # noqa: E402
from paper_2009_03076_b200.model import CellList  # noqa: E402
from paper_2009_03076_b200.orbit import orbit_cameras  # noqa: E402
from paper_2009_03076_b200.regions import build_regions  # noqa: E402
from paper_2009_03076_b200.render import Camera, MarchParams, build_scene, integrate_ray, render_frame_float  # noqa: E402
from tests_util import golden_cells  # noqa: E402

VARIANTS = {"warp": {}, "warp_cap1": {"leaf_cap": 1}, "warp_nowalk": {"walk_lists": 0}, "warp_short": {"short_rays": 1},
            "warp_kshort": {"short_rays": 1, "fuse_short": 0}, "warp_2pass": {"walk_cap1": 2, "walk2_min": 0},
            "warp_wide_short": {"short_rays": 1, "short_leaves": 16, "short_samples": 4096},
            "warp_grab8": {"grab_fixed": 8}, "tile": {"kernel": 1}, "lbvh": {"traversal": 1}}

i, j, k, lev, vals = golden_cells("smoke")
model, tree = build_bricks(CellList(i, j, k, lev, vals), BrickBuildParams(keep_split_tree=True))
regions = build_regions(model)
lo, hi = model.value_range(0)
tf = TransferFunction.grayscale((lo, hi), max_alpha=0.5)
cam = orbit_cameras(regions.bounds, 4, 96, 64)[1]
params = MarchParams(seed=3, gradient_mode="analytic")
b = regions.bounds
inside = Camera(0.5 * (np.asarray(b.lo) + np.asarray(b.hi)), (-0.6, -0.5, 0.62), (0.0, 0.0, 1.0), 70.0, 48, 40)
for iso, cam in ((None, cam), (0.5 * (lo + hi), cam), (None, inside), (0.45 * (lo + hi), inside)):
    scene = build_scene(model, regions, tf, iso_value=iso, tree=tree)
    ref = None
    for name, fields in VARIANTS.items():
        with N.tuning(**fields):
            u8, f64, cnt, st = render_frame_float(scene, cam, tf, params)
        if ref is None:
            ref = cnt
        assert np.array_equal(cnt, ref), name
        print(f"iso={iso is not None} {name}: samples {int(st[1])}", flush=True)
    u8, f64, cnt, st = render_frame_float(scene, cam, tf, params, use_celllocation=True)
    assert np.array_equal(cnt, ref), "celllocation"
    print(f"iso={iso is not None} celllocation: samples {int(st[1])}", flush=True)
for gm in ("central", "clampedCentral", "none"):
    u8, f64, cnt, st = render_frame_float(build_scene(model, regions, tf), cam, tf,
                                          MarchParams(seed=3, gradient_mode=gm))
    print(f"gradient {gm}: samples {int(st[1])}", flush=True)
o, d = cam.ray(40, 30)
print("integrate_ray", integrate_ray(o, d, build_scene(model, regions, tf), tf, params, pixel=30 * 96 + 40)[1])
# TF edits: active sets rebuilt from the stream-ordered pool and released
from paper_2009_03076_b200.accel import build_iso_bvh, build_volume_bvh  # noqa: E402

keep = []
for q in range(6):
    b = build_volume_bvh(regions, TransferFunction.grayscale((lo, hi), max_alpha=0.2 + 0.1 * q), 0, model=model)
    c = build_iso_bvh(regions, lo + (q + 1) * (hi - lo) / 8, 0, model=model)
    if q % 2:
        keep.append(b)
    del c
print("active sets:", [len(b.prims) for b in keep])
print("sanitize frames done")
