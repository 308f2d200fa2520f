"""Render a few frames of a bench config with given xb_tuning fields (for ncu launch lists):
python tools/frames.py CONFIG [k:field=v+field=v] [n_frames] [view]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2009_03076_b200 import _native as N  # noqa: E402
from paper_2009_03076_b200.bricks import build_bricks  # noqa: E402
from paper_2009_03076_b200.regions import build_regions  # noqa: E402
from paper_2009_03076_b200.render import MarchParams, build_scene, render_native  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1]]
fields = {}
if len(sys.argv) > 2 and sys.argv[2].startswith("k:"):
    fields = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in sys.argv[2][2:].split("+")}
n = int(sys.argv[3]) if len(sys.argv) > 3 else 3
view = int(sys.argv[4]) if len(sys.argv) > 4 else 0
cells = bench.make_cells(cfg)
model, _ = build_bricks(cells)
regions = build_regions(model)
tf = bench.tf_for(model.value_range(0), cfg)
scene = build_scene(model, regions, tf, iso_value=cfg.get("iso"))
cam = bench.cameras_for(regions.bounds, cfg, 8)[view]
params = MarchParams(seed=0, gradient_mode=cfg["gradient"])
W, H = cfg["res"]
out = torch.empty((H, W, 4), dtype=torch.uint8, device="cuda")
with N.tuning(**fields):
    for _ in range(n):
        st = render_native(scene, cam, tf, params, out.data_ptr())
print("stats", st)
