"""Pixels of configs[3] view 0 that show the iso-surface (differ from the
DVR-only frame), for a few iso values: python tools/iso_check.py"""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2009_03076_b200.bricks import build_bricks
from paper_2009_03076_b200.regions import build_regions
from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame_float
cfg = bench.CONFIGS['c4']
cells = bench.make_cells(cfg)
model, _ = build_bricks(cells); regions = build_regions(model); del cells
lo, hi = model.value_range(0); print('value range', lo, hi)
tf = bench.tf_for((lo, hi), cfg)
cams = bench.cameras_for(regions.bounds, cfg, 8)
params = MarchParams(seed=0, gradient_mode='analytic')
for iso in (None, 0.5, 0.25, 0.1, 0.05):
    sc = build_scene(model, regions, tf, iso_value=iso)
    u8, f, cnt, st = render_frame_float(sc, cams[0], tf, params)
    if iso is None: base = f.copy(); print('dvr samples', st[1]); continue
    d = np.abs(f - base).max(-1)
    print(f'iso {iso}: samples {st[1]}, pixels differing from DVR-only {int((d > 1e-9).sum())}, alpha==1 px {int((f[...,3] >= 1.0).sum())}')
