"""Where the e2e frame time goes (host output through the public API):
python tools/e2e_probe.py CONFIG [reps]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2009_03076_b200 import render as R  # noqa: E402
from paper_2009_03076_b200.bricks import build_bricks  # noqa: E402
from paper_2009_03076_b200.regions import build_regions  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cells = bench.make_cells(cfg)
model, _ = build_bricks(cells)
regions = build_regions(model)
del cells
tf = bench.tf_for(model.value_range(0), cfg)
scene = R.build_scene(model, regions, tf, iso_value=cfg.get("iso"))
cam = bench.cameras_for(regions.bounds, cfg, 8)[0]
params = R.MarchParams(seed=0, gradient_mode=cfg["gradient"])
W, H = cfg["res"]
dev = torch.empty((H, W, 4), dtype=torch.uint8, device="cuda")
pinned = torch.empty((H, W, 4), dtype=torch.uint8, pin_memory=True)
pn = pinned.numpy()


def timeit(name, fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t) * 1e3)
    print(f"{name:34s} median {np.median(ts):7.3f} ms  mean {np.mean(ts):7.3f}  min {np.min(ts):7.3f}  max "
          f"{np.max(ts):7.3f}", flush=True)
    if os.environ.get("ALL"):
        print("   ", np.round(ts, 2).tolist())


timeit("python structs", lambda: (R.camera_struct(cam), R.march_struct(tf, params)))
timeit("_host_image", lambda: R._host_image(H, W))
timeit("D2H 4WH pinned", lambda: (pinned.copy_(dev), torch.cuda.synchronize()))
def enqueue_only():
    torch.cuda.synchronize()
    t = time.perf_counter()
    R.render_native(scene, cam, tf, params, dev.data_ptr(), sync=False)
    dt = time.perf_counter() - t
    torch.cuda.synchronize()
    return dt


enq = [enqueue_only() for _ in range(reps)]
print(f"{'host enqueue (xb_render, no sync)':34s} median {np.median(enq) * 1e3:7.3f} ms", flush=True)
timeit("render device out, no stats", lambda: (R.render_native(scene, cam, tf, params, dev.data_ptr(), sync=False),
                                               torch.cuda.synchronize()))
timeit("render device out + stats", lambda: R.render_native(scene, cam, tf, params, dev.data_ptr()))
timeit("render pinned out + stats", lambda: R.render_native(scene, cam, tf, params, pn))
timeit("render_frame", lambda: R.render_frame(scene, cam, tf, params))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    timeit("render_native on a side stream", lambda: R.render_native(scene, cam, tf, params, pn, stream=s.cuda_stream))
