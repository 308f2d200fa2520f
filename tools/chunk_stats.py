"""k_warp work statistics (XB_DEBUG_CHUNKS; needs a library built with `make DEBUG_CHUNKS=1`):
python tools/chunk_stats.py CONFIG"""
import os
import sys

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
os.environ["XB_DEBUG_CHUNKS"] = "1"
fr = R.render_frame(scene, cam, tf, params)
print("frame: regions", fr.stats.regions, "samples", fr.stats.samples, flush=True)
