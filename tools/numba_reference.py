"""Time the reference's own CPU renderer (amrvol.render_frame, numba prange on all
host cores, R/render.py:654-691) at a bench config, on the box, and check it
against our GPU frame of the same view.

  python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \\
      --target baseline/_ref <copy of /root/reference/pkg> --no-deps      # once, here
  python tools/numba_reference.py c2 [view] > profiles/rNN_numba_reference_c2.json   # on the GPU box

The model/regions given to the reference are the oracle's C builds (pinned
bit-exact to the reference's builders; its own Python builders need ~5 min at
C2); the reference builds its volume BVH itself (build_scene).  Reported:
build_scene time, one warm frame's time, samples/regions (FrameStats), the numba
thread count and CPU model, and the comparison with the GPU frame (RGBA8 max
difference, equal stats)."""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
sys.path.insert(0, str(ROOT))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count()))

import numba  # noqa: E402
import numpy as np  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    view = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    import amrvol
    from amrvol.accel import TransferFunction as RTF
    from amrvol.model import AmrModel as RModel
    from amrvol.regions import RegionSet as RRegions
    from amrvol.render import Camera as RCam
    from amrvol.render import MarchParams as RParams
    from amrvol.render import build_scene as r_build_scene
    from amrvol.render import render_frame as r_render_frame

    cfg = bench.CONFIGS[name]
    cells = bench.make_cells(dict(cfg, gpu_gen=False))
    m = oracle.build_bricks(cells.i, cells.j, cells.k, cells.level, cells.values)
    r = oracle.build_regions(*(m[k] for k in bench.MODEL_KEYS))
    model = RModel(("value",), m["brick_lower"], m["brick_level"], m["brick_dims"], m["scalars"])
    regions = RRegions(r["lo"], r["hi"], r["brick_off"], r["brick_ids"], r["value_range"], r["finest_width"],
                       ("value",))
    vr = (float(m["scalars"][0].min()), float(m["scalars"][0].max()))
    tf_ours = bench.tf_for(vr, cfg)
    tf = RTF(tf_ours.domain, tf_ours.rgba)
    t0 = time.perf_counter()
    scene = r_build_scene(model, regions, tf, iso_value=cfg.get("iso"))
    t_scene = time.perf_counter() - t0
    from paper_2009_03076_b200.model import Box3

    cams = bench.cameras_for(Box3(r["lo"].min(axis=0), r["hi"].max(axis=0)), cfg, 8)
    c = cams[view]
    cam = RCam(c.position, c.forward, c.up, c.fov_y, c.width, c.height)
    params = RParams(seed=0, gradient_mode=cfg["gradient"])
    small = RCam(c.position, c.forward, c.up, c.fov_y, 32, 32)
    t0 = time.perf_counter()
    r_render_frame(scene, small, tf, params)  # JIT compile + point index
    t_jit = time.perf_counter() - t0
    t0 = time.perf_counter()
    fr = r_render_frame(scene, cam, tf, params)
    t_frame = time.perf_counter() - t0
    out = {"config": name, "view": view, "reference": f"amrvol {amrvol.__version__ if hasattr(amrvol, '__version__') else ''}"
           " render_frame (numba prange), baseline/_ref", "numba": numba.__version__,
           "numba_threads": numba.get_num_threads(), **bench.host_info(),
           "width": c.width, "height": c.height, "frame_s": t_frame, "fps": 1.0 / t_frame,
           "samples": fr.stats.samples, "regions": fr.stats.regions,
           "msamples_per_s": fr.stats.samples / t_frame / 1e6, "build_scene_s": t_scene, "jit_and_warmup_s": t_jit}
    try:  # the GPU frame of the same view
        from paper_2009_03076_b200.bricks import build_bricks
        from paper_2009_03076_b200.regions import build_regions
        from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame

        gm, _ = build_bricks(cells)
        gr = build_regions(gm)
        gs = build_scene(gm, gr, tf_ours, iso_value=cfg.get("iso"))
        gf = render_frame(gs, c, tf_ours, MarchParams(seed=0, gradient_mode=cfg["gradient"]))
        out["gpu_vs_reference"] = {
            "rgba8_max_abs_diff": int(np.abs(gf.rgba.astype(int) - fr.rgba.astype(int)).max()),
            "rgba8_pixels_differing": int(np.count_nonzero((gf.rgba != fr.rgba).any(-1))),
            "samples_equal": gf.stats.samples == fr.stats.samples, "regions_equal": gf.stats.regions == fr.stats.regions}
    except Exception as e:  # no GPU here
        out["gpu_vs_reference"] = f"not run: {e}"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
