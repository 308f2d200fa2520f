"""Diagnose e2e outliers: bench-like sequence with gc / allocator event logging."""
import gc
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2009_03076_b200 import render as R  # noqa: E402
from paper_2009_03076_b200.bricks import build_bricks  # noqa: E402
from paper_2009_03076_b200.parallel import TiledRenderer  # noqa: E402
from paper_2009_03076_b200.regions import build_regions  # noqa: E402

cfg = bench.CONFIGS["c3"]
cells = bench.make_cells(cfg)
model, _ = build_bricks(cells)
regions = build_regions(model)
del cells
tf = bench.tf_for(model.value_range(0), cfg)
scene = R.build_scene(model, regions, tf)
cam = bench.cameras_for(regions.bounds, cfg, 8)[0]
params = R.MarchParams(seed=0, gradient_mode=cfg["gradient"])
W, H = cfg["res"]
rend = TiledRenderer(scene, W, H, torch.device("cuda:0"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    rend.render(cam, tf, params)
for _ in range(10):
    flush.zero_()
    rend.render(cam, tf, params)
torch.cuda.synchronize()
ev = []
gc.callbacks.append(lambda phase, info: ev.append((time.perf_counter(), phase, info.get("generation"))))
for trial in range(3):
    for _ in range(3):
        R.render_frame(scene, cam, tf, params)
    torch.cuda.synchronize()
    ts = []
    t00 = time.perf_counter()
    for _ in range(10):
        tq = time.perf_counter()
        fr = R.render_frame(scene, cam, tf, params)
        ts.append((time.perf_counter() - tq) * 1e3)
    print("trial", trial, np.round(ts, 2).tolist(), flush=True)
    print("   gc events:", [(round((t - t00) * 1e3, 2), p, g) for t, p, g in ev if t >= t00], flush=True)
    if trial == 1:
        gc.disable()
