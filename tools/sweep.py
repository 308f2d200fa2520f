"""Kernel-variant sweep on a bench config: CUDA-event frame times (L2 flushed
between frames) for XB_KSTEPS x XB_MINB, plus the default and tile kernels."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2009_03076_b200.bricks import build_bricks  # noqa: E402
from paper_2009_03076_b200.regions import build_regions  # noqa: E402
from paper_2009_03076_b200.render import MarchParams, build_scene, render_native  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["default", "tile"] + [
    f"{k}x{b}" for k in (1, 2, 3) for b in (4, 5, 6)]
cells = bench.make_cells(cfg)
model, _ = build_bricks(cells)
regions = build_regions(model)
tf = bench.tf_for(model.value_range(0), cfg)
scene = build_scene(model, regions, tf)
cam = bench.camera_for(regions.bounds, cfg, 0)
params = MarchParams(seed=0, gradient_mode=cfg["gradient"])
W, H = cfg["res"]
out = torch.empty((H, W, 4), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()
res = {}
for v in variants:
    for k in ("XB_KERNEL", "XB_KSTEPS", "XB_MINB"):
        os.environ.pop(k, None)
    if v in ("tile", "frame"):
        os.environ["XB_KERNEL"] = v
    elif v != "default":
        ks, mb = v.split("x")
        os.environ["XB_KERNEL"] = "frame"
        os.environ["XB_KSTEPS"], os.environ["XB_MINB"] = ks, mb
    for _ in range(3):
        render_native(scene, cam, tf, params, out.data_ptr(), stream=stream.cuda_stream)
    ts = []
    for _ in range(8):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        render_native(scene, cam, tf, params, out.data_ptr(), stream=stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    st = render_native(scene, cam, tf, params, out.data_ptr(), stream=stream.cuda_stream)
    res[v] = {"ms": sorted(ts)[len(ts) // 2], "min_ms": min(ts), "samples": int(st[1])}
    print(v, res[v], flush=True)
print(json.dumps(res))
