"""Calibrate the large synthetic configs on the GPU: cell counts per level and
build times.  python tools/calib.py c3|c5 [build]"""
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2009_03076_b200 import io as xio  # noqa: E402


def gear(rh, rr):
    c = 6144.0
    return xio.SyntheticSpec(field="gaussian", extent=(16384, 8192, 8192), max_level=12, threshold=0.05, seed=0,
                             holes=((c, c, c, rh),), refine_spheres=((c, c, c, rr),),
                             field_params={"center": (c, c, c), "sigma": 600.0})


def jet(thr, rh, rr, step=80, sigma=400.0):
    X, Y, Z = 2048, 1024, 1024
    xs = np.arange(0.2 * X, 0.8 * X + 1e-9, step)
    holes = tuple((float(x), Y / 2, Z / 2, float(rh)) for x in xs)
    refine = tuple((float(x), Y / 2, Z / 2, float(rr)) for x in xs)
    return xio.SyntheticSpec(field="gaussian", extent=(X, Y, Z), max_level=3, threshold=thr, seed=0, holes=holes,
                             refine_spheres=refine, field_params={"center": (X / 2, Y / 2, Z / 2), "sigma": sigma})


def run(spec, build=False):
    t = time.perf_counter()
    dc = xio.generate_synthetic_device(spec)
    tg = time.perf_counter() - t
    cl = None
    out = {"cells": len(dc), "gen_s": round(tg, 2)}
    if build:
        from paper_2009_03076_b200.bricks import build_bricks
        from paper_2009_03076_b200.regions import build_regions

        t = time.perf_counter()
        m, _ = build_bricks(dc)
        out["bricks"] = m.n_bricks
        out["bricks_s"] = round(time.perf_counter() - t, 2)
        t = time.perf_counter()
        r = build_regions(m)
        out["regions"] = len(r)
        out["regions_s"] = round(time.perf_counter() - t, 2)
    return out


if __name__ == "__main__":
    which = sys.argv[1]
    build = len(sys.argv) > 2
    if which == "c3":
        for rh, rr in ((200, 412), (200, 420)):
            print("gear", rh, rr, run(gear(rh, rr), build), flush=True)
    else:
        for thr, rh, rr in ((0.0029, 80, 240), (0.0028, 80, 240), (0.003, 80, 290), (0.003, 80, 300)):
            print("jet", thr, rh, rr, run(jet(thr, rh, rr), False), flush=True)
