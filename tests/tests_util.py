"""Helpers shared by the parity tests (CPU side)."""
import hashlib
from functools import lru_cache

import numpy as np

from conftest import golden_digests, golden_model

MODEL_KEYS = ("brick_lower", "brick_level", "brick_dims", "brick_offset", "scalars")
REGION_KEYS = ("lo", "hi", "brick_off", "brick_ids", "value_range", "finest_width")


def sha(a) -> str:
    """Same digest as tests/golden/make_golden.py:sha."""
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def canonical_cells(model):
    """Cells in AmrModel.cell_list() order: ascending brick, x-fastest (R/model.py:311-332)."""
    lo, lev, dims, off = model["brick_lower"], model["brick_level"], model["brick_dims"], model["brick_offset"]
    n = int(off[-1])
    ci, cj, ck, cl = (np.empty(n, np.int32) for _ in range(4))
    for b in range(len(lev)):
        s, e = int(off[b]), int(off[b + 1])
        w = 1 << int(lev[b])
        nx, ny, nz = (int(d) for d in dims[b])
        gz, gy, gx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        ci[s:e] = lo[b, 0] + gx.ravel() * w
        cj[s:e] = lo[b, 1] + gy.ravel() * w
        ck[s:e] = lo[b, 2] + gz.ravel() * w
        cl[s:e] = lev[b]
    return ci, cj, ck, cl, model["scalars"].T.copy()


def spec_from_digest(d):
    from paper_2009_03076_b200.io import SyntheticSpec

    s = d["spec"]
    fp = {k: (tuple(v) if isinstance(v, list) else v) for k, v in s["field_params"].items()}
    return SyntheticSpec(
        field=s["field"], extent=tuple(s["extent"]), max_level=s["max_level"],
        threshold=(np.inf if s["threshold_inf"] else s["threshold"]), seed=s["seed"],
        holes=tuple(tuple(h) for h in s["holes"]), refine_spheres=tuple(tuple(h) for h in s["refine_spheres"]),
        field_params=fp,
    )


@lru_cache(maxsize=None)
def golden_cells(name):
    """Cell arrays of a golden case: stored arrays, or regenerated + digest-checked."""
    d = golden_digests()["models"][name]
    src = d.get("cells_from", name)
    g = golden_model(src)
    if "cells_i" in g:
        return tuple(g[f"cells_{a}"] for a in ("i", "j", "k", "level", "values"))
    from paper_2009_03076_b200 import io as xio

    cl = xio.generate_synthetic(spec_from_digest(golden_digests()["models"][src]))
    for a in ("i", "j", "k", "level", "values"):
        assert sha(getattr(cl, a)) == d[f"cells.{a}"], f"synthetic generator drifted on {name}.{a}"
    return cl.i, cl.j, cl.k, cl.level, cl.values


@lru_cache(maxsize=None)
def scene_arrays(name):
    """(model, regions) array dicts for a golden case, digest-checked."""
    g = golden_model(name)
    d = golden_digests()["models"][name]
    if "model_scalars" in g:
        model = {k: g[f"model_{k}"] for k in MODEL_KEYS}
        regions = {k: g[f"regions_{k}"] for k in REGION_KEYS}
        return model, regions
    import oracle

    i, j, k, lev, vals = golden_cells(name)
    model = oracle.build_bricks(i, j, k, lev, vals, d["max_brick_width"])
    regions = oracle.build_regions(*(model[k] for k in MODEL_KEYS))
    for k in MODEL_KEYS:
        assert sha(model[k]) == d[f"model.{k}"], k
    for k in REGION_KEYS:
        assert sha(regions[k]) == d[f"regions.{k}"], k
    return model, regions
