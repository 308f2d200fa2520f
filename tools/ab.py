"""A/B frame timing of frame-pipeline variants (xb_tuning fields), interleaved:
python tools/ab.py CONFIG warp,tile,lbvh,k:leaf_cap=48+short_rays=0 [reps]

warp = the defaults; tile = one thread per pixel; lbvh = per-visit LBVH
queries (the reference's traversal); k:F=V+F2=V2 sets xb_tuning fields.
Every repetition renders each variant over the 8-view orbit (AB_VIEWS=1: view 0
only); L2 is flushed before every frame.  The printed times are per orbit-mean
frame.  Other libraries: XB_LIB=path/to/libexabricks.so (tools/ab_libs.sh)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2009_03076_b200 import _native as N  # noqa: E402
from paper_2009_03076_b200.bricks import build_bricks  # noqa: E402
from paper_2009_03076_b200.regions import build_regions  # noqa: E402
from paper_2009_03076_b200.render import MarchParams, build_scene, render_native  # noqa: E402

NAMED = {"warp": {}, "tile": {"kernel": 1}, "lbvh": {"traversal": 1}, "nowalk": {"walk_lists": 0},
         "short": {"short_rays": 1}, "noshort": {"short_rays": 0}, "kshort": {"short_rays": 1, "fuse_short": 0}}


def fields_of(v):
    if v.startswith("k:"):
        return {kv.split("=")[0]: int(kv.split("=")[1]) for kv in v[2:].split("+")}
    return NAMED[v]


def setv(v):
    if not hasattr(N.lib(), "xb_tuning_set"):  # round-1 build: its defaults only
        return
    t = N.XbTuning()
    N.lib().xb_tuning_defaults(C.byref(t))
    for k, val in fields_of(v).items():
        setattr(t, k, val)
    N.check(N.lib().xb_tuning_set(C.byref(t)))


def main():
    cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    variants = (sys.argv[2] if len(sys.argv) > 2 else "warp").split(",")
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    cells = bench.make_cells(cfg)
    model, _ = build_bricks(cells)
    regions = build_regions(model)
    del cells
    tf = bench.tf_for(model.value_range(0), cfg)
    scene = build_scene(model, regions, tf, iso_value=cfg.get("iso"))
    n_views = int(os.environ.get("AB_VIEWS", "8"))
    cams = bench.cameras_for(regions.bounds, cfg, 8)[:n_views]
    params = MarchParams(seed=0, gradient_mode=cfg["gradient"])
    W, H = cfg["res"]
    out = torch.empty((H, W, 4), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    for v in variants:
        setv(v)
        for cam in cams:
            render_native(scene, cam, tf, params, out.data_ptr(), stream=stream.cuda_stream)
    torch.cuda.synchronize()
    # enqueue everything first (no host sync inside the loop): the GPU queue stays
    # ahead of the host, so host-side stalls never land between two events
    evs = []
    for it in range(reps):
        for v in variants:
            setv(v)
            for cam in cams:
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                render_native(scene, cam, tf, params, out.data_ptr(), stream=stream.cuda_stream, sync=False)
                b.record(stream)
                evs.append((v, it, a, b))
    torch.cuda.synchronize()
    times = {v: np.zeros(reps) for v in variants}
    for v, it, a, b in evs:
        times[v][it] += a.elapsed_time(b) / len(cams)
    for v in variants:
        t = times[v]
        print(f"{v:10s} orbit-mean frame: median {np.median(t):8.4f} ms  min {t.min():8.4f}  max {t.max():8.4f}")


if __name__ == "__main__":
    main()
