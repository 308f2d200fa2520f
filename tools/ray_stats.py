"""Per-ray work distribution of a frame (regions / samples per pixel):
python tools/ray_stats.py CONFIG"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2009_03076_b200 import render as R  # noqa: E402
from paper_2009_03076_b200.bricks import build_bricks  # noqa: E402
from paper_2009_03076_b200.regions import build_regions  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
cells = bench.make_cells(cfg)
model, _ = build_bricks(cells)
regions = build_regions(model)
del cells
tf = bench.tf_for(model.value_range(0), cfg)
scene = R.build_scene(model, regions, tf, iso_value=cfg.get("iso"))
cam = bench.cameras_for(regions.bounds, cfg, 8)[0]
params = R.MarchParams(seed=0, gradient_mode=cfg["gradient"])
_, _, cnt, st = R.render_frame_float(scene, cam, tf, params)
reg, smp = cnt[..., 0].ravel().astype(np.int64), cnt[..., 1].ravel().astype(np.int64)
hit = reg > 0
print("pixels", reg.size, "with regions", int(hit.sum()), "regions", int(reg.sum()), "samples", int(smp.sum()))
for name, v in (("regions", reg[hit]), ("samples", smp[hit])):
    q = np.percentile(v, [50, 90, 99, 99.9, 99.99])
    top = np.sort(v)[-8:][::-1]
    print(f"{name}: p50/90/99/99.9/99.99 {q.round(1).tolist()} max {top.tolist()}")
s = np.sort(smp[hit])[::-1]
cs = np.cumsum(s)
for k in (10, 100, 1000, 10000):
    if k <= len(s):
        print(f"top {k} rays hold {100 * cs[k - 1] / cs[-1]:.1f} % of samples")
