"""Pin the CPU oracle (`oracle/`) to the reference's own outputs.

The golden fixtures were produced by importing the reference package in the
build container (tests/golden/make_golden.py).  Every comparison here is exact:
builders array-equal, samples / gradients / traversal intervals / float RGBA
frames bit-identical.  CPU only.
"""
import ctypes as C
import json

import numpy as np
import pytest

import oracle
from conftest import frame_meta, golden_digests, golden_frames, golden_model

MODEL_KEYS = ("brick_lower", "brick_level", "brick_dims", "brick_offset", "scalars")
REGION_KEYS = ("lo", "hi", "brick_off", "brick_ids", "value_range", "finest_width")
TREE_KEYS = ("axis", "pos", "left", "right", "brick_start", "brick_count", "box_lo", "box_hi", "max_half")

DIG = golden_digests()["models"]
FULL = sorted(n for n, d in DIG.items() if d["full"] and "cells_from" not in d)
VARIANTS = sorted(n for n, d in DIG.items() if "cells_from" in d)


def cells_of(name):
    d = DIG[name]
    src = d.get("cells_from", name)
    g = golden_model(src)
    return g["cells_i"], g["cells_j"], g["cells_k"], g["cells_level"], g["cells_values"], d["max_brick_width"]


@pytest.mark.parametrize("name", FULL + VARIANTS)
def test_oracle_builders_match_reference(name):
    i, j, k, lev, vals, width = cells_of(name)
    m = oracle.build_bricks(i, j, k, lev, vals, width, keep_split_tree=True)
    g = golden_model(name) if name not in VARIANTS else None
    if g is not None:
        for key in MODEL_KEYS:
            assert np.array_equal(m[key], g[f"model_{key}"]), key
        for key in TREE_KEYS:
            assert np.array_equal(m["tree"][key], g[f"tree_{key}"]), key
    r = oracle.build_regions(m["brick_lower"], m["brick_level"], m["brick_dims"], m["brick_offset"], m["scalars"])
    from tests_util import sha
    for key in MODEL_KEYS:
        assert sha(m[key]) == DIG[name][f"model.{key}"], key
    for key in TREE_KEYS:
        assert sha(m["tree"][key]) == DIG[name][f"tree.{key}"], key
    for key in REGION_KEYS:
        assert sha(r[key]) == DIG[name][f"regions.{key}"], key


def _scene(name):
    g = golden_model(name)
    model = {k: g[f"model_{k}"] for k in MODEL_KEYS}
    regions = {k: g[f"regions_{k}"] for k in REGION_KEYS}
    return g, oracle.OracleScene(model, regions)


SAMPLED = [n for n in FULL if "pts" in golden_model(n)]


@pytest.mark.parametrize("name", SAMPLED)
def test_oracle_samples_and_gradients_bit_exact(name):
    g, sc = _scene(name)
    from tests_util import canonical_cells
    ci, cj, ck, cl, cv = canonical_cells(sc.model)
    for t, p in enumerate(g["pts"]):
        rid = int(g["pts_region"][t])
        assert sc.point_query(p) == (None if rid < 0 else rid)
        if rid >= 0:
            num, den = sc.sample_region(rid, p)
        else:
            num, den = oracle.sample_cells(ci, cj, ck, cl, cv[:, 0], p)
        valid = den > 1e-12
        assert valid == bool(g["pts_valid"][t])
        assert den == g["pts_wsum"][t]
        assert (num / den if valid else 0.0) == g["pts_value"][t]
        if rid >= 0:
            a = sc.gradient_region(rid, p)
            gv = a[1] > 1e-12
            assert gv == bool(g["grad_analytic_valid"][t])
            if gv:
                vec = (a[2:5] * a[1] - a[0] * a[5:8]) / (a[1] * a[1])
                assert np.array_equal(vec, g["grad_analytic"][t])


@pytest.mark.parametrize("name", ["smoke", "gauss_aniso"])
def test_oracle_traversal_matches_reference(name):
    g, sc = _scene(name)
    for tag in ("all", "pruned"):
        if tag == "pruned":
            sc.set_tf(g["rays_pruned_domain"], g["rays_pruned_tf"])
            bvh = sc.vol_bvh
        else:
            bvh = sc.all_bvh
        off = g[f"rays_{tag}_off"]
        for q in range(len(off) - 1):
            got = sc.iterate_intervals(bvh, g[f"rays_{tag}_o"][q], g[f"rays_{tag}_d"][q], 0.0, 1e9)
            s, e = off[q], off[q + 1]
            want = list(zip(g[f"rays_{tag}_tin"][s:e], g[f"rays_{tag}_tout"][s:e], g[f"rays_{tag}_region"][s:e]))
            assert len(got) == len(want)
            for a, b in zip(got, want):
                assert a[0] == b[0] and a[1] == b[1] and a[2] == b[2]


FRAME_MODEL = {"smoke": "smoke", "ramp": "ramp", "c1": "c1", "aniso": "gauss_aniso"}


def frame_keys():
    fr = golden_frames()
    return sorted({k[: -len("_rgba_f64")] for k in fr if k.endswith("_rgba_f64")})


def oracle_scene_for(key):
    from tests_util import scene_arrays
    model, regions = scene_arrays(FRAME_MODEL[key.split("_")[0]])
    return oracle.OracleScene(model, regions)


@pytest.mark.parametrize("key", frame_keys())
def test_oracle_frames_bit_exact(key, frames):
    meta = frame_meta(frames, key)
    sc = oracle_scene_for(key)
    dom, rgba = meta["tf_domain"], frames[f"{key}_tf_rgba"]
    sc.set_tf(dom, rgba)
    sc.set_iso(meta["iso"])
    r, u, f = meta["basis"]
    cam = oracle.camera_struct(meta["width"], meta["height"], meta["position"], r, u, f, meta["tan_half"],
                               meta["width"] / meta["height"])
    out_f, out_u8, pr, ps = sc.render(cam, dom, rgba, spc=meta["spc"], rate=meta["rate"], early=meta["early"],
                                      seed=meta["seed"], gradient_mode=meta["gradient_mode"], clip_planes=meta["clip_planes"])
    assert np.array_equal(pr, frames[f"{key}_px_regions"])
    assert np.array_equal(ps, frames[f"{key}_px_samples"])
    assert np.array_equal(out_u8, frames[f"{key}_rgba_u8"])
    assert np.array_equal(out_f, frames[f"{key}_rgba_f64"])


def test_oracle_max_opacity_and_rho():
    g = dict(np.load(__import__("conftest").GOLDEN / "tf_rho.npz"))
    for t in range(len(g["tf_rgba"])):
        dom = g[f"tf{t}_domain"]
        got = [oracle.max_opacity(dom, g["tf_rgba"][t], a, b) for a, b in g["tf_ranges"][t]]
        assert np.array_equal(np.array(got), g["tf_max_opacity"][t])
    for si, s in enumerate(g["rho_seeds"]):
        got = [oracle.pixel_rho(int(p), int(s)) for p in g["rho_pixels"]]
        assert np.array_equal(np.array(got), g["rho_values"][si])


def test_oracle_two_cell_rays():
    g = dict(np.load(__import__("conftest").GOLDEN / "rays.npz"))["two_cell_rays"]
    for width, rate, r, gg, b, a, nreg, nsmp in g:
        m = oracle.build_bricks([0, 1], [0, 0], [0, 0], [0, 0], [4.0, 4.0], int(width))
        reg = oracle.build_regions(m["brick_lower"], m["brick_level"], m["brick_dims"], m["brick_offset"], m["scalars"])
        sc = oracle.OracleScene(m, reg)
        rgba = np.ones((256, 4))
        rgba[:, 3] = 0.3
        sc.set_tf((3.0, 5.0), rgba)
        out, st = sc.integrate_ray((-3.0, 0.5, 0.5), (1.0, 0.0, 0.0), (3.0, 5.0), rgba, rate=rate, gradient_mode="none", early=1.0)
        assert np.array_equal(out, [r, gg, b, a])
        assert st == {"regions": int(nreg), "samples": int(nsmp)}
