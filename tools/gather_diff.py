"""Frame differences between two library builds (e.g. the FP32 and the exact
FP64 gather in k_warp): per build, `python tools/gather_diff.py dump TAG CONFIG
[views]` (XB_LIB selects the library) writes /tmp/gd_TAG_CONFIG_VIEW.npz with
the float RGBA frame and the per-pixel counters; `python tools/gather_diff.py
cmp TAG_A TAG_B CONFIG [views]` prints max |dRGBA|, the pixels whose counters
differ and, for builds that export xb_fixup_stats (the FP32-gather experiment,
3a9dfc7), the k_fixup counts."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def views_of(a):
    return [int(v) for v in a.split(",")] if a else [0]


def dump(tag, cfg_name, views):
    import torch
    import bench
    from paper_2009_03076_b200 import _native as N
    from paper_2009_03076_b200.bricks import build_bricks
    from paper_2009_03076_b200.regions import build_regions
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_native
    cfg = bench.CONFIGS[cfg_name]
    cells = bench.make_cells(cfg)
    model, _ = build_bricks(cells)
    regions = build_regions(model)
    del cells
    tf = bench.tf_for(model.value_range(0), cfg)
    scene = build_scene(model, regions, tf, iso_value=cfg.get("iso"))
    cams = bench.cameras_for(regions.bounds, cfg, 8)
    params = MarchParams(seed=0, gradient_mode=cfg["gradient"])
    W, H = cfg["res"]
    for v in views:
        out8 = np.zeros((H, W, 4), np.uint8)
        outf = np.zeros((H, W, 4), np.float64)
        cnt = np.zeros((H, W, 2), np.int32)
        has_fix = hasattr(N.lib(), "xb_fixup_stats")
        if has_fix:
            N.check(N.lib().xb_fixup_stats(0, (C.c_int64 * 3)()))
        render_native(scene, cams[v], tf, params, out8, outf, cnt)
        fx = (C.c_int64 * 3)()
        if has_fix:
            N.check(N.lib().xb_fixup_stats(0, fx))
        np.savez(f"/tmp/gd_{tag}_{cfg_name}_{v}.npz", f=outf, c=cnt, fix=np.array(list(fx)))
        torch.cuda.synchronize()


def cmp(ta, tb, cfg_name, views):
    for v in views:
        a = np.load(f"/tmp/gd_{ta}_{cfg_name}_{v}.npz")
        b = np.load(f"/tmp/gd_{tb}_{cfg_name}_{v}.npz")
        d = np.abs(a["f"] - b["f"])
        dc = np.any(a["c"] != b["c"], axis=-1)
        ds = np.abs(a["c"][..., 1].astype(np.int64) - b["c"][..., 1])
        print(f"{cfg_name} view {v}: max|dRGBA| {np.nanmax(d):.3e} (alpha {np.nanmax(d[..., 3]):.3e}), "
              f"pixels > 1e-6: {int((d.max(-1) > 1e-6).sum())}, counter-differing pixels {int(dc.sum())} "
              f"(max |d samples| {int(ds.max())}), non-finite {int((~np.isfinite(a['f'])).sum())}/"
              f"{int((~np.isfinite(b['f'])).sum())}, k_fixup {a['fix'].tolist()}/{b['fix'].tolist()}")


if __name__ == "__main__":
    if sys.argv[1] == "dump":
        dump(sys.argv[2], sys.argv[3], views_of(sys.argv[4] if len(sys.argv) > 4 else ""))
    else:
        cmp(sys.argv[2], sys.argv[3], sys.argv[4], views_of(sys.argv[5] if len(sys.argv) > 5 else ""))
