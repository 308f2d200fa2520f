"""Where the reference's numba frame and ours differ (C3 view 0): saves both RGBA8
frames, our float frame and per-pixel counters, and for the differing pixels the
oracle's float RGBA and counters and the reference's integrate_ray RGBA.
python tools/numba_diff_probe.py c3 0 -> gpurun_out/numba_diff_c3.npz"""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
sys.path.insert(0, str(ROOT))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")

import numpy as np  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    view = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    from amrvol.accel import TransferFunction as RTF
    from amrvol.model import AmrModel as RModel
    from amrvol.regions import RegionSet as RRegions
    from amrvol.render import Camera as RCam
    from amrvol.render import MarchParams as RParams
    from amrvol.render import build_scene as r_build_scene
    from amrvol.render import render_frame as r_render_frame

    from paper_2009_03076_b200.bricks import build_bricks
    from paper_2009_03076_b200.model import Box3
    from paper_2009_03076_b200.regions import build_regions
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame_float

    cfg = bench.CONFIGS[name]
    cells = bench.make_cells(dict(cfg, gpu_gen=False))
    m = oracle.build_bricks(cells.i, cells.j, cells.k, cells.level, cells.values)
    r = oracle.build_regions(*(m[k] for k in bench.MODEL_KEYS))
    vr = (float(m["scalars"][0].min()), float(m["scalars"][0].max()))
    tf = bench.tf_for(vr, cfg)
    cams = bench.cameras_for(Box3(r["lo"].min(axis=0), r["hi"].max(axis=0)), cfg, 8)
    c = cams[view]
    gm, _ = build_bricks(cells)
    gr = build_regions(gm)
    gs = build_scene(gm, gr, tf)
    params = MarchParams(seed=0, gradient_mode=cfg["gradient"])
    g8, gf, gcnt, gst = render_frame_float(gs, c, tf, params)
    print("gpu done", gst, flush=True)
    model = RModel(("value",), m["brick_lower"], m["brick_level"], m["brick_dims"], m["scalars"])
    regions = RRegions(r["lo"], r["hi"], r["brick_off"], r["brick_ids"], r["value_range"], r["finest_width"],
                       ("value",))
    rtf = RTF(tf.domain, tf.rgba)
    scene = r_build_scene(model, regions, rtf)
    cam = RCam(c.position, c.forward, c.up, c.fov_y, c.width, c.height)
    rparams = RParams(seed=0, gradient_mode=cfg["gradient"])
    fr = r_render_frame(scene, cam, rtf, rparams)
    print("ref done", fr.stats, flush=True)
    diff = np.argwhere((fr.rgba != g8).any(-1))
    print("differing pixels", len(diff), "max", int(np.abs(fr.rgba.astype(int) - g8.astype(int)).max()), flush=True)
    W = c.width
    pix = diff[:, 0] * W + diff[:, 1]
    osc = oracle.OracleScene(m, r)
    osc.set_tf(tf.domain, tf.rgba)
    ocam = bench.oracle_camera(c)
    of = np.zeros((len(pix), 4))
    ocnt = np.zeros((len(pix), 2), np.int64)
    for q, p in enumerate(pix[:400]):
        f_, _, pr, ps = osc.render(ocam, tf.domain, tf.rgba, pix_range=(int(p), int(p) + 1), seed=0,
                                   gradient_mode=cfg["gradient"])
        of[q] = f_[0]
        ocnt[q] = (pr[0], ps[0])
    from amrvol.render import integrate_ray

    rf = np.zeros((min(len(pix), 400), 4))
    for q, (y, x) in enumerate(diff[:400]):
        o, d = cam.ray(int(x), int(y))
        rf[q] = integrate_ray(o, d, scene, rtf, rparams, pixel=int(y * W + x))[0]
    out = ROOT / "gpurun_out" / f"numba_diff_{name}.npz"
    out.parent.mkdir(exist_ok=True)
    np.savez_compressed(out, ref8=fr.rgba, gpu8=g8, diff=diff, gpuf=gf.reshape(-1, 4)[pix],
                        gpucnt=gcnt.reshape(-1, 2)[pix], oraclef=of, oraclecnt=ocnt, refray=rf)
    print("saved", out, flush=True)


if __name__ == "__main__":
    main()
