"""GPU parity at the benchmarked scales (BASELINE.json configs[0]-[2]).

* configs[1] (C2, 9.53M cells): GPU builders np.array_equal to the C oracle's
  (run live), and frame bands of two orbit views within max |dRGBA| <= 1e-3
  with per-pixel region and sample counters equal.
* configs[2] (C3, 266M cells): GPU builders against the oracle's sha256
  digests (tests/golden/scale_digests.json, tools/make_scale_digests.py —
  the oracle needs ~3 min for it).
* configs[0] (C1) at its stated 256x256, whole frame.
* Active sets (T/test_accel.py:111-137): the volume set equals the regions
  with max_opacity(tf, value_range) > 0 and the iso set the regions with
  lo <= iso <= hi, for every golden frame's TF, step TFs at value quantiles,
  and C2.
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle
from conftest import frame_meta
from tests_util import sha

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
RGBA_TOL = 1e-3
MODEL_KEYS = ("brick_lower", "brick_level", "brick_dims", "brick_offset", "scalars")
REGION_KEYS = ("lo", "hi", "brick_off", "brick_ids", "value_range", "finest_width")


def _bench():
    import sys

    sys.path.insert(0, str(ROOT))
    import bench

    return bench


def _build(cells):
    from paper_2009_03076_b200.bricks import build_bricks
    from paper_2009_03076_b200.regions import build_regions

    model, _ = build_bricks(cells)
    return model, build_regions(model)


@pytest.fixture(scope="module")
def c2():
    bench = _bench()
    cfg = bench.CONFIGS["c2"]
    cells = bench.make_cells(cfg)
    model, regions = _build(cells)
    return cfg, cells, model, regions


def _oracle_scene(model, regions):
    return oracle.OracleScene({k: getattr(model, k) for k in MODEL_KEYS}, {k: getattr(regions, k) for k in REGION_KEYS})


def _ocam(cam):
    r, u, f = cam.basis()
    return oracle.camera_struct(cam.width, cam.height, cam.position, r, u, f, math.tan(math.radians(cam.fov_y) * 0.5),
                                cam.width / cam.height)


def test_c2_builders_equal_oracle(c2):
    cfg, cells, model, regions = c2
    assert len(cells) == 9_534_568
    om = oracle.build_bricks(cells.i, cells.j, cells.k, cells.level, cells.values)
    for k in MODEL_KEYS:
        assert np.array_equal(getattr(model, k), om[k]), k
    orr = oracle.build_regions(*(om[k] for k in MODEL_KEYS))
    for k in REGION_KEYS:
        assert np.array_equal(getattr(regions, k), orr[k]), k


@pytest.mark.parametrize("view", [0, 3])
def test_c2_frame_bands_match_oracle(c2, view):
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame_float

    bench = _bench()
    cfg, cells, model, regions = c2
    tf = bench.tf_for(model.value_range(0), cfg)
    scene = build_scene(model, regions, tf)
    cam = bench.cameras_for(regions.bounds, cfg, 8)[view]
    params = MarchParams(seed=0, gradient_mode="analytic")
    u8, f64, cnt, stats = render_frame_float(scene, cam, tf, params)
    osc = _oracle_scene(model, regions)
    osc.set_tf(tf.domain, tf.rgba)
    W = cam.width
    f, c = f64.reshape(-1, 4), cnt.reshape(-1, 2)
    for y0 in (300, 500, 700):  # three 8-row bands through the volume
        b, e = y0 * W, (y0 + 8) * W
        of, ou, pr, ps = osc.render(_ocam(cam), tf.domain, tf.rgba, pix_range=(b, e), seed=0,
                                    gradient_mode="analytic")
        assert ps.sum() > 0
        assert np.abs(f[b:e] - of).max() <= RGBA_TOL, y0
        assert np.array_equal(c[b:e, 0], pr), y0
        assert np.array_equal(c[b:e, 1], ps), y0
        assert np.abs(u8.reshape(-1, 4)[b:e].astype(int) - ou.astype(int)).max() <= 1


def test_c2_active_sets_match_enumeration(c2):
    """T/test_accel.py:111-137 at configs[1] scale."""
    from paper_2009_03076_b200.accel import TransferFunction, build_iso_bvh, build_volume_bvh

    cfg, cells, model, regions = c2
    osc = _oracle_scene(model, regions)
    vr = regions.value_range[:, 0]
    lo, hi = float(vr.min()), float(vr.max())
    tfs = [_bench().tf_for((lo, hi), cfg)]
    for q in (0.3, 0.6, 0.9):  # step TFs opaque above a value quantile (the reference test's construction)
        cut = float(np.quantile(vr[:, 1], q))
        a = np.zeros(256)
        a[int(np.ceil((cut - lo) / (hi - lo) * 255)) + 1:] = 1.0
        tfs.append(TransferFunction((lo, hi), np.c_[np.ones((256, 3)), a]))
    for tf in tfs:
        got = build_volume_bvh(regions, tf, 0, model=model).prims
        want = osc.active_volume(tf.domain, tf.rgba)
        assert np.array_equal(np.sort(got), want)
    for q in (0.1, 0.5, 0.9):
        iso = float(np.quantile(vr[:, 1], q))
        got = build_iso_bvh(regions, iso, 0, model=model).prims
        assert np.array_equal(np.sort(got), osc.active_iso(iso))


def test_golden_frame_tfs_active_sets(frames):
    """Every golden frame's TF (and a mid-range iso value) on its model."""
    from conftest import golden_digests
    from paper_2009_03076_b200.accel import TransferFunction, build_iso_bvh, build_volume_bvh
    from paper_2009_03076_b200.bricks import BrickBuildParams, build_bricks
    from paper_2009_03076_b200.model import CellList
    from paper_2009_03076_b200.regions import build_regions
    from tests_util import golden_cells

    dig = golden_digests()["models"]
    model_of = {"smoke": "smoke", "ramp": "ramp", "c1": "c1", "aniso": "gauss_aniso"}
    keys = sorted({k[: -len("_tf_rgba")] for k in frames if k.endswith("_tf_rgba")})
    assert len(keys) >= 12
    built = {}
    for key in keys:
        name = model_of[key.split("_")[0]]
        if name not in built:
            i, j, k, lev, vals = golden_cells(name)
            m, _ = build_bricks(CellList(i, j, k, lev, vals),
                                BrickBuildParams(max_brick_width=dig[name]["max_brick_width"]))
            built[name] = (m, build_regions(m))
        model, regions = built[name]
        meta = frame_meta(frames, key)
        tf = TransferFunction(meta["tf_domain"], frames[f"{key}_tf_rgba"])
        osc = _oracle_scene(model, regions)
        got = build_volume_bvh(regions, tf, 0, model=model).prims
        assert np.array_equal(np.sort(got), osc.active_volume(tf.domain, tf.rgba)), key
        vr = regions.value_range[:, 0]
        iso = float(0.5 * (vr.min() + vr.max()))
        got = build_iso_bvh(regions, iso, 0, model=model).prims
        assert np.array_equal(np.sort(got), osc.active_iso(iso)), key


def test_c1_full_frame_256_matches_oracle():
    """configs[0] at its stated 256x256: the whole frame."""
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame_float

    bench = _bench()
    cfg = bench.CONFIGS["c1"]
    cells = bench.make_cells(cfg)
    assert len(cells) == 97_840
    model, regions = _build(cells)
    tf = bench.tf_for(model.value_range(0), cfg)
    scene = build_scene(model, regions, tf)
    osc = _oracle_scene(model, regions)
    osc.set_tf(tf.domain, tf.rgba)
    for view in (0, 5):
        cam = bench.cameras_for(regions.bounds, cfg, 8)[view]
        assert (cam.width, cam.height) == (256, 256)
        params = MarchParams(seed=0, gradient_mode="analytic")
        u8, f64, cnt, stats = render_frame_float(scene, cam, tf, params)
        of, ou, pr, ps = osc.render(_ocam(cam), tf.domain, tf.rgba, seed=0, gradient_mode="analytic")
        assert np.abs(f64 - of).max() <= RGBA_TOL
        assert np.array_equal(cnt[..., 0].ravel(), pr) and np.array_equal(cnt[..., 1].ravel(), ps)
        assert int(stats[1]) == int(ps.sum()) and int(stats[0]) == int(pr.sum())


def test_c3_builders_match_oracle_digests():
    """configs[2] (266M cells): every GPU builder array has the oracle's sha256."""
    bench = _bench()
    gold = json.loads((ROOT / "tests" / "golden" / "scale_digests.json").read_text())["c3"]
    cells = bench.make_cells(bench.CONFIGS["c3"])
    assert len(cells) == gold["n_cells"]
    for a in ("i", "j", "k", "level", "values"):
        assert sha(getattr(cells, a)) == gold["cells"][a], a
    model, regions = _build(cells)
    del cells
    for k in MODEL_KEYS:
        assert sha(getattr(model, k)) == gold["model"][k], k
    for k in REGION_KEYS:
        assert sha(getattr(regions, k)) == gold["regions"][k], k


def test_far_field_subnormal_values_shade_exactly():
    """A narrow gaussian whose tail values are FP32 subnormals: the FP32 shading
    gradient of those samples underflows (it produced NaN colours before round 2's
    fix, found against the reference's own renderer at configs[2]).  Under the
    data-range TF their opacity is negligible and they shade 0.2; under a TF
    whose domain is the subnormal range itself they are opaque and the frame
    kernel defers them to the exact FP64 re-render (k_fixup).  Either way: no
    NaN, the oracle's frame within 1e-3, counters equal."""
    from paper_2009_03076_b200 import io as xio
    from paper_2009_03076_b200.orbit import orbit_cameras
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame, render_frame_float

    bench = _bench()
    spec = xio.SyntheticSpec(field="gaussian", extent=(64, 64, 64), max_level=2, threshold=0.01, seed=0,
                             field_params={"center": (32.0, 32.0, 32.0), "sigma": 2.5})
    cells = xio.generate_synthetic(spec)
    v = cells.values[:, 0]
    assert np.count_nonzero((v > 0) & (v < np.finfo(np.float32).tiny)) > 0  # subnormal tail present
    model, regions = _build(cells)
    from paper_2009_03076_b200.accel import TransferFunction

    for tf in (bench.tf_for(model.value_range(0), dict(max_alpha=0.5)),
               TransferFunction.grayscale((0.0, 2e-38), max_alpha=0.5)):
        _subnormal_frames(model, regions, tf)


def _subnormal_frames(model, regions, tf):
    from paper_2009_03076_b200.orbit import orbit_cameras
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame, render_frame_float

    scene = build_scene(model, regions, tf)
    osc = _oracle_scene(model, regions)
    osc.set_tf(tf.domain, tf.rgba)
    params = MarchParams(seed=1, gradient_mode="analytic")
    for cam in orbit_cameras(regions.bounds, 3, 160, 120):
        u8, f64, cnt, st = render_frame_float(scene, cam, tf, params)
        assert np.isfinite(f64).all()
        of, ou, pr, ps = osc.render(_ocam(cam), tf.domain, tf.rgba, seed=1, gradient_mode="analytic")
        assert np.abs(f64 - of).max() <= RGBA_TOL
        assert np.array_equal(cnt[..., 0].ravel(), pr) and np.array_equal(cnt[..., 1].ravel(), ps)
        fr = render_frame(scene, cam, tf, params)
        assert np.abs(fr.rgba.astype(int) - ou.astype(int)).max() <= 1


def test_reference_renderer_pixel_identical_c1():
    """The installed reference itself (baseline/_ref: amrvol, numba) against the
    GPU path at configs[0]: the reference's own builders give the same arrays,
    and its render_frame the same RGBA8 frame and stats (two orbit views, one
    with the iso-surface).  Skipped where the reference is not installed."""
    import os
    import sys

    ref = ROOT / "baseline" / "_ref"
    if not (ref / "amrvol").exists():
        pytest.skip("reference not installed in baseline/_ref")
    try:
        import numba  # noqa: F401
    except ImportError:
        pytest.skip("numba missing")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
    sys.path.insert(0, str(ref))
    from amrvol.accel import TransferFunction as RTF
    from amrvol.bricks import build_bricks as r_build_bricks
    from amrvol.model import CellList as RCells
    from amrvol.regions import build_regions as r_build_regions
    from amrvol.render import Camera as RCam
    from amrvol.render import MarchParams as RParams
    from amrvol.render import build_scene as r_build_scene
    from amrvol.render import render_frame as r_render_frame

    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame

    bench = _bench()
    cfg = bench.CONFIGS["c1"]
    cells = bench.make_cells(cfg)
    model, regions = _build(cells)
    rm, _ = r_build_bricks(RCells(cells.i, cells.j, cells.k, cells.level, cells.values, cells.field_names))
    rr = r_build_regions(rm)
    for k in MODEL_KEYS:
        assert np.array_equal(getattr(model, k), getattr(rm, k)), k
    for k in REGION_KEYS:
        assert np.array_equal(getattr(regions, k), getattr(rr, k)), k
    tf = bench.tf_for(model.value_range(0), cfg)
    rtf = RTF(tf.domain, tf.rgba)
    lo, hi = model.value_range(0)
    for view, iso in ((0, None), (3, 0.5 * (lo + hi))):
        cam = bench.cameras_for(regions.bounds, cfg, 8)[view]
        ours = render_frame(build_scene(model, regions, tf, iso_value=iso), cam, tf,
                            MarchParams(seed=0, gradient_mode="analytic"))
        rcam = RCam(cam.position, cam.forward, cam.up, cam.fov_y, cam.width, cam.height)
        theirs = r_render_frame(r_build_scene(rm, rr, rtf, iso_value=iso), rcam, rtf,
                                RParams(seed=0, gradient_mode="analytic"))
        assert (ours.stats.regions, ours.stats.samples) == (theirs.stats.regions, theirs.stats.samples)
        assert np.abs(ours.rgba.astype(int) - theirs.rgba.astype(int)).max() <= 1
        assert np.count_nonzero(ours.rgba != theirs.rgba) <= ours.rgba.size // 10000



def test_integrate_ray_from_inside_matches_oracle():
    """integrate_ray (R/render.py:613-632) for rays that start inside the volume
    (random eyes and directions, t_range from 0 and from mid-ray) on
    configs[0]'s model, with an opaque-topped TF: GPU ray-batch kernel against
    the oracle (pinned to the reference's frames incl. the inside-eye goldens)."""
    from paper_2009_03076_b200.accel import TransferFunction
    from paper_2009_03076_b200.render import MarchParams, build_scene, integrate_ray

    bench = _bench()
    cfg = bench.CONFIGS["c1"]
    model, regions = _build(bench.make_cells(cfg))
    lo, hi = model.value_range(0)
    rgba = np.tile(np.linspace(0.0, 1.0, 256)[:, None], (1, 4))
    rgba[:, 3] = np.linspace(0.0, 0.4, 256)
    rgba[255, 3] = 1.0
    tf = TransferFunction((lo, hi), rgba)
    scene = build_scene(model, regions, tf)
    osc = _oracle_scene(model, regions)
    osc.set_tf(tf.domain, tf.rgba)
    b = regions.bounds
    blo, bhi = np.asarray(b.lo, float), np.asarray(b.hi, float)
    rng = np.random.default_rng(17)
    params = MarchParams(seed=4, gradient_mode="analytic")
    samples = 0
    for q in range(60):
        o = blo + rng.random(3) * (bhi - blo)
        d = rng.normal(size=3)
        if q % 10 == 0:
            d = np.eye(3)[q % 3] * (1 if q % 20 else -1)  # axis-parallel
        t_range = (0.0, 1e30) if q % 2 == 0 else (float(rng.random() * 5.0), float(5.0 + rng.random() * 40.0))
        got, gs = integrate_ray(o, d, scene, tf, params, pixel=q, t_range=t_range)
        want, ws = osc.integrate_ray(o, d, tf.domain, tf.rgba, pixel=q, t_range=t_range, seed=4,
                                     gradient_mode="analytic")
        assert np.abs(got - want).max() <= RGBA_TOL, q
        assert gs == ws, q
        samples += ws["samples"]
    assert samples > 0


def test_iso_intersect_from_inside_matches_oracle():
    """iso_intersect (R/render.py:635-651) for rays starting inside the volume:
    hit / miss, t_hit and the gradient at the hit equal the oracle's."""
    from paper_2009_03076_b200.accel import TransferFunction, build_iso_bvh
    from paper_2009_03076_b200.render import MarchParams, build_scene, iso_intersect

    bench = _bench()
    cfg = bench.CONFIGS["c1"]
    model, regions = _build(bench.make_cells(cfg))
    lo, hi = model.value_range(0)
    iso = float(lo + 0.4 * (hi - lo))
    scene = build_scene(model, regions, TransferFunction.grayscale((lo, hi)), iso_value=iso)
    bvh = build_iso_bvh(regions, iso, 0, model=model)
    osc = _oracle_scene(model, regions)
    b = regions.bounds
    blo, bhi = np.asarray(b.lo, float), np.asarray(b.hi, float)
    rng = np.random.default_rng(23)
    hits = 0
    for q in range(80):
        o = blo + rng.random(3) * (bhi - blo)
        d = rng.normal(size=3) if q % 8 else np.eye(3)[q % 3]
        got = iso_intersect(o, d, bvh, scene, iso, params=MarchParams(seed=6), pixel=q)
        want = osc.iso_intersect(o, d, iso, seed=6, pixel=q)
        assert (got is None) == (want is None), q
        if want is not None:
            hits += 1
            assert got[0] == want[0], q
            assert np.array_equal(got[1], want[1]), q
    assert hits > 0
