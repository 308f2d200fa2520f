"""Golden frames with the eye INSIDE the volume (fly-through views), made by
the reference itself — none of make_golden.py's frames puts the camera inside
the model, where every ray starts in the middle of an active region (the
reference's first query starts at t = 0 inside a region box,
R/accel.py:285-352, and the lattice's first sample is cut at t = 0,
R/render.py:404-418).  The reference service accepts any camera
(R/service.py:101-114).

Runs ONLY in the build container (imports the reference read-only):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_inside.py

-> tests/golden/frames_inside.npz, same keys / layout as frames.npz
(conftest.golden_frames() merges both files, so the oracle's bit-exact frame
test and the GPU frame-parity matrix pick them up).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as G  # noqa: E402  (imports the reference)

R = G.R


def views(regions):
    b = regions.bounds
    lo, hi = np.asarray(b.lo, float), np.asarray(b.hi, float)
    c = 0.5 * (lo + hi)
    return [
        ("inside_centre", c, (1.0, 0.0, 0.0), (0.0, 1.0, 0.0)),
        ("inside_oblique", c + 0.13 * (hi - lo), (-0.6, -0.5, 0.62), (0.0, 0.0, 1.0)),
        ("inside_corner", lo + 0.07 * (hi - lo), (1.0, 1.0, 1.0), (0.0, 1.0, 0.0)),
        ("inside_axis", c, (0.0, 0.0, -1.0), (0.0, 1.0, 0.0)),  # axis-parallel central ray
    ]


def main():
    out = {}
    for name, (w, h), max_alpha in (("smoke", (48, 40), 1.0), ("c1", (64, 48), 0.5)):
        cells = G.avio.generate_synthetic(G.SPECS[name])
        model, _, regions = G.build_case(name, cells, 32)
        lo, hi = model.value_range(0)
        tf = G.TransferFunction.grayscale((lo, hi), max_alpha=max_alpha)
        scene = R.build_scene(model, regions, tf)
        for tag, pos, fwd, up in views(regions):
            cam = R.Camera(pos, fwd, up, 70.0, w, h)
            key = f"{name}_{tag}"
            G.store_frame(out, key, scene, cam, tf, R.MarchParams(seed=3, gradient_mode="analytic"))
            print(key, int(out[f"{key}_px_samples"].sum()), "samples")
        if name == "smoke":  # iso surface + volume (make_golden's smoke_iso) seen from inside
            iso_v = float(lo + 0.45 * (hi - lo))
            g05 = G.TransferFunction.grayscale((lo, hi), max_alpha=0.5)
            si = R.build_scene(model, regions, g05, iso_value=iso_v)
            for tag, pos, fwd, up in views(regions)[:3]:
                key = f"{name}_{tag}_iso"
                G.store_frame(out, key, si, R.Camera(pos, fwd, up, 70.0, w, h), g05,
                              R.MarchParams(seed=1, early_term_threshold=0.9), iso=iso_v)
                print(key, int(out[f"{key}_px_samples"].sum()), "samples")
    # ---- edge cases of the march arguments (also none in make_golden.py)
    cells = G.avio.generate_synthetic(G.SPECS["c1"])
    model, _, regions = G.build_case("c1", cells, 32)
    lo, hi = model.value_range(0)
    b = regions.bounds
    blo, bhi = np.asarray(b.lo, float), np.asarray(b.hi, float)
    c = np.floor(0.5 * (blo + bhi))  # integer coordinates: on cell / region faces
    g = G.TransferFunction.grayscale((lo, hi), max_alpha=0.7)
    scene = R.build_scene(model, regions, g)
    edge = [
        # odd size: the centre ray is exactly (0, 0, 1) through region faces (zero-direction slab rule)
        ("edge_axis_out", R.Camera([c[0], c[1], blo[2] - 9.0], [0.0, 0.0, 1.0], [0.0, 1.0, 0.0], 30.0, 33, 31),
         R.MarchParams(seed=5, gradient_mode="analytic")),
        ("edge_axis_in", R.Camera(c, [0.0, 1.0, 0.0], [1.0, 0.0, 0.0], 50.0, 31, 33),
         R.MarchParams(seed=5, gradient_mode="central")),
        # coarse steps, no early termination, the largest seed, non-square frame
        ("edge_coarse", R.Camera(c + [0.3, -0.2, 0.1], [0.3, 0.2, 1.0], [0.0, 1.0, 0.0], 60.0, 40, 17),
         R.MarchParams(samples_per_cell=1.0, rate_scale=0.3, early_term_threshold=1.0, seed=2**64 - 1,
                       gradient_mode="analytic")),
        # fine steps, eye inside behind two clip planes, clamped central gradients
        ("edge_clip_in", R.Camera(c + [1.5, 0.5, -0.5], [-1.0, 0.1, 0.4], [0.0, 1.0, 0.0], 80.0, 24, 24),
         R.MarchParams(samples_per_cell=3.0, rate_scale=1.9, seed=77, gradient_mode="clampedCentral",
                       clip_planes=[((1.0, 0.0, 0.0), float(c[0]) - 3.0), ((0.2, -1.0, 0.3), -float(c[1]) - 4.0)])),
        # a one-pixel-wide frame
        ("edge_column", R.Camera(c + [0.5, 0.5, 0.5], [0.0, 0.0, -1.0], [0.0, 1.0, 0.0], 90.0, 1, 9),
         R.MarchParams(seed=11, gradient_mode="none")),
    ]
    for tag, cam, params in edge:
        key = f"c1_{tag}"
        G.store_frame(out, key, scene, cam, g, params)
        print(key, int(out[f"{key}_px_samples"].sum()), "samples")
    # ---- edge cases of the transfer function / iso value, from an orbit view
    cam = G.orbit_cameras(regions.bounds, 8, 40, 36)[3]
    zero = np.tile(np.linspace(0.0, 1.0, 256)[:, None], (1, 4))
    zero[:, 3] = 0.0  # nothing active: every ray misses
    top = np.tile(np.linspace(0.0, 1.0, 256)[:, None], (1, 4))
    top[:, 3] = 0.2
    top[255, 3] = 1.0  # opaque only at the top: alpha exactly 1 behind short last steps
    tfs = [
        ("tf_empty", G.TransferFunction((lo, hi), zero), None, "analytic"),
        ("tf_top_opaque", G.TransferFunction((lo, hi), top), None, "analytic"),
        # domain below most values: samples clamp to the last (opaque) entry
        ("tf_narrow", G.TransferFunction.grayscale((lo, lo + 0.3 * (hi - lo)), max_alpha=1.0), None, "central"),
        ("iso_above_range", g, float(hi + 1.0), "analytic"),  # no iso candidates at all
        ("iso_at_max", g, float(hi), "none"),
    ]
    for tag, tf, iso, mode in tfs:
        sc = R.build_scene(model, regions, tf, iso_value=iso)
        key = f"c1_edge_{tag}"
        G.store_frame(out, key, sc, cam, tf, R.MarchParams(seed=9, gradient_mode=mode), iso=iso)
        print(key, int(out[f"{key}_px_samples"].sum()), "samples")
    np.savez_compressed(G.OUT / "frames_inside.npz", **out)


if __name__ == "__main__":
    sys.setrecursionlimit(100000)
    main()
