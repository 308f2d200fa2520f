"""A/B frame timing of march-kernel variants (XB_KERNEL values), interleaved:
python tools/ab.py CONFIG warp,frame [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2009_03076_b200.bricks import build_bricks  # noqa: E402
from paper_2009_03076_b200.regions import build_regions  # noqa: E402
from paper_2009_03076_b200.render import MarchParams, build_scene, render_native  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
variants = (sys.argv[2] if len(sys.argv) > 2 else "warp,frame").split(",")
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
cells = bench.make_cells(cfg)
model, _ = build_bricks(cells)
regions = build_regions(model)
tf = bench.tf_for(model.value_range(0), cfg)
scene = build_scene(model, regions, tf, iso_value=cfg.get("iso"))
cam = bench.camera_for(regions.bounds, cfg, 0)
params = MarchParams(seed=0, gradient_mode=cfg["gradient"])
W, H = cfg["res"]
out = torch.empty((H, W, 4), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()


def setv(v):
    for k in [k for k in os.environ if k.startswith("XB_") and k != "XB_LIB"]:
        os.environ.pop(k)
    """warp | frame | tile | warpN (k_warp with __launch_bounds__ min blocks N) | gD (guided grab divisor D)"""
    for k in ("XB_KERNEL", "XB_WMINB", "XB_GRAB_DIV", "XB_GRAB_FIXED", "XB_WALK", "XB_LEAF_CAP", "XB_WALK_NOTAU",
              "XB_TRAVERSAL", "XB_SHORT", "XB_SHORT_LEAVES", "XB_SHORT_SAMPLES"):
        os.environ.pop(k, None)
    for k in ("XB_WALK_CAP1", "XB_WALK2_MIN", "XB_WALK_CAP2", "XB_CUT_TAU"):
        os.environ.pop(k, None)
    if v.startswith("e:"):  # e:K=V+K2=V2: arbitrary XB_* settings
        for kv in v[2:].split("+"):
            k, val = kv.split("=")
            os.environ[k] = val
        return
    if v.startswith("w2_"):  # w2_X_Y: pass-1 cap X, pass-2 cap Y
        os.environ["XB_WALK_CAP1"], os.environ["XB_WALK_CAP2"] = v[3:].split("_")
        return
    if v.startswith("c1_") :  # c1_X_Y: pass-1 cap X, pass-2 minimum Y
        os.environ["XB_WALK_CAP1"], os.environ["XB_WALK2_MIN"] = v[3:].split("_")
        return
    if v.startswith("sl") and "_" in v:  # slL_S: short-ray thresholds
        os.environ["XB_SHORT_LEAVES"], os.environ["XB_SHORT_SAMPLES"] = v[2:].split("_")
        return
    if v == "cutnotau":
        os.environ["XB_CUT_TAU"] = "0"
        return
    if v == "short":
        os.environ["XB_SHORT"] = "1"
    elif v == "noshort":
        os.environ["XB_SHORT"] = "0"
    elif v == "lbvh":
        os.environ["XB_TRAVERSAL"] = "lbvh"
    elif v == "notau":
        os.environ["XB_WALK_NOTAU"] = "1"
    elif v == "nowalk":
        os.environ["XB_WALK"] = "0"
    elif v.startswith("cap") and v[3:].isdigit():
        os.environ["XB_LEAF_CAP"] = v[3:]
    elif v.startswith("f") and v[1:].isdigit():
        os.environ["XB_GRAB_FIXED"] = v[1:]
    elif v.startswith("g") and v[1:].isdigit():  # guided grabs with divisor D
        os.environ["XB_GRAB_DIV"] = v[1:]
        os.environ["XB_GRAB_FIXED"] = "0"
    elif v.startswith("warp") and len(v) > 4:
        os.environ["XB_WMINB"] = v[4:]
    elif v != "warp":
        os.environ["XB_KERNEL"] = v


times = {v: [] for v in variants}
for v in variants:
    setv(v)
    for _ in range(3):
        render_native(scene, cam, tf, params, out.data_ptr(), stream=stream.cuda_stream)
torch.cuda.synchronize()
# enqueue everything first (no host sync inside the loop): the GPU queue stays
# ahead of the host, so host-side stalls never land between two events
evs = []
for it in range(reps):
    for v in variants:
        setv(v)
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        render_native(scene, cam, tf, params, out.data_ptr(), stream=stream.cuda_stream, sync=False)
        b.record(stream)
        evs.append((v, a, b))
torch.cuda.synchronize()
for v, a, b in evs:
    times[v].append(a.elapsed_time(b))
for v in variants:
    t = np.array(times[v])
    print(f"{v:8s} median {np.median(t):8.3f} ms  min {t.min():8.3f}  max {t.max():8.3f}  all {np.round(t, 2).tolist()}")
