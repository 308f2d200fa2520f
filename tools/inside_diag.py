"""Diagnose a golden frame's mismatches per pipeline variant: python tools/inside_diag.py KEY"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from conftest import frame_meta, golden_frames  # noqa: E402
import test_gpu_parity as T  # noqa: E402
from paper_2009_03076_b200 import _native as N  # noqa: E402
from paper_2009_03076_b200.accel import TransferFunction  # noqa: E402
from paper_2009_03076_b200.render import build_scene, render_frame_float  # noqa: E402

key = sys.argv[1]
fr = golden_frames()
meta = frame_meta(fr, key)
model, _, regions = T._build(T.FRAME_MODEL[key.split("_")[0]])
tf = TransferFunction(meta["tf_domain"], fr[f"{key}_tf_rgba"])
scene = build_scene(model, regions, tf, iso_value=meta["iso"])
cam = T._camera(meta)
want = fr[f"{key}_rgba_f64"]
pr, ps = fr[f"{key}_px_regions"], fr[f"{key}_px_samples"]
for name, var in sorted(T.KERNEL_VARIANTS.items()):
    with N.tuning(**var):
        u8, f64, cnt, st = render_frame_float(scene, cam, tf, T._params(meta))
    d = np.abs(f64 - want).max(axis=2).ravel()
    bad = np.nonzero((d > 1e-3) | (cnt[..., 0].ravel() != pr) | (cnt[..., 1].ravel() != ps))[0]
    print(f"{name:16s} max {d.max():.3g}  bad px {len(bad)}")
    for p in bad[:6]:
        y, x = divmod(int(p), meta["width"])
        print(f"   px ({x},{y}) got {f64[y, x].round(5)} cnt {cnt[y, x]}  want {want[y, x].round(5)} cnt {pr[p]},{ps[p]}")
