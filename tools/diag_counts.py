"""Diagnostics: frame-stat repeatability and kernel agreement on a config."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2009_03076_b200.bricks import build_bricks  # noqa: E402
from paper_2009_03076_b200.regions import build_regions  # noqa: E402
from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame, render_frame_float  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
cells = bench.make_cells(cfg)
model, _ = build_bricks(cells)
regions = build_regions(model)
tf = bench.tf_for(model.value_range(0), cfg)
scene = build_scene(model, regions, tf)
cam = bench.cameras_for(regions.bounds, cfg, 8)[0]
params = MarchParams(seed=0, gradient_mode=cfg["gradient"])
for i in range(3):
    fr = render_frame(scene, cam, tf, params)
    print("render_frame", i, fr.stats)
u8, f64, cnt, st = render_frame_float(scene, cam, tf, params, count_bytes=True)
print("count variant", st, cnt[..., 1].sum(), cnt[..., 0].sum())
u8b, f64b, cntb, stb = render_frame_float(scene, cam, tf, params)
print("float variant", stb, cntb[..., 1].sum())
from paper_2009_03076_b200 import _native as N  # noqa: E402

with N.tuning(kernel=1):
    u8t, f64t, cntt, stt = render_frame_float(scene, cam, tf, params)
print("tile kernel", stt, cntt[..., 1].sum())
d = np.abs(f64 - f64t).max()
print("max |f64 frame - tile|", d, "count mismatches", int((cnt != cntt).any(-1).sum()))
bad = np.argwhere((cnt != cntt).any(-1))
print("first mismatching pixels", bad[:10].tolist())
for y, x in bad[:5]:
    print(y, x, cnt[y, x], cntt[y, x], f64[y, x], f64t[y, x])
