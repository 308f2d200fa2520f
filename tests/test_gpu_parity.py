"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
fixtures and the CPU oracle.

Bars: builders bit-exact (np.array_equal / sha256 of every
AmrModel, SplitTree and RegionSet array); point samples, gradients and
traversal intervals bit-exact; frames max |dRGBA| <= 1e-3 before
quantisation, RGBA8 within 1 LSB, per-pixel region/sample counters equal.
"""
import math

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, frame_meta, golden_digests, golden_frames, golden_model
from tests_util import canonical_cells, golden_cells, scene_arrays, sha

pytestmark = pytest.mark.gpu

DIG = golden_digests()["models"]
RGBA_TOL = 1e-3  # images within max |dRGBA| <= 1e-3

MODEL_KEYS = ("brick_lower", "brick_level", "brick_dims", "brick_offset", "scalars")
REGION_KEYS = ("lo", "hi", "brick_off", "brick_ids", "value_range", "finest_width")
TREE_KEYS = ("axis", "pos", "left", "right", "brick_start", "brick_count", "box_lo", "box_hi", "max_half")


@pytest.fixture(scope="module")
def xb():
    import paper_2009_03076_b200 as pkg
    from paper_2009_03076_b200 import accel, bricks, io, model, orbit, regions, render, sampling

    return pkg


def _cells(name):
    from paper_2009_03076_b200.model import CellList

    i, j, k, lev, vals = golden_cells(name)
    return CellList(i, j, k, lev, vals)


def _build(name, keep_tree=False):
    from paper_2009_03076_b200.bricks import BrickBuildParams, build_bricks
    from paper_2009_03076_b200.regions import build_regions

    model, tree = build_bricks(_cells(name), BrickBuildParams(max_brick_width=DIG[name]["max_brick_width"],
                                                              keep_split_tree=keep_tree))
    return model, tree, build_regions(model)


# ---------------------------------------------------------------- builders


@pytest.mark.parametrize("name", sorted(DIG))
def test_builders_bit_exact(xb, name):
    model, tree, regions = _build(name, keep_tree=True)
    d = DIG[name]
    for k in MODEL_KEYS:
        assert sha(getattr(model, k)) == d[f"model.{k}"], f"{name}: model.{k}"
    for k in TREE_KEYS:
        assert sha(getattr(tree, k)) == d[f"tree.{k}"], f"{name}: tree.{k}"
    for k in REGION_KEYS:
        assert sha(getattr(regions, k)) == d[f"regions.{k}"], f"{name}: regions.{k}"


@pytest.mark.parametrize("name", ["gauss16", "smoke"])
def test_builders_permutation_invariant(xb, name):
    from paper_2009_03076_b200.bricks import BrickBuildParams, build_bricks
    from paper_2009_03076_b200.regions import build_regions

    base, btree, breg = _build(name, keep_tree=True)
    cl = _cells(name)
    for seed in (101, 202):
        m2, t2 = build_bricks(cl.permuted(np.random.default_rng(seed).permutation(len(cl))),
                              BrickBuildParams(keep_split_tree=True))
        r2 = build_regions(m2)
        for k in MODEL_KEYS:
            assert np.array_equal(getattr(m2, k), getattr(base, k))
        for k in TREE_KEYS:
            assert np.array_equal(getattr(t2, k), getattr(btree, k))
        for k in REGION_KEYS:
            assert np.array_equal(getattr(r2, k), getattr(breg, k))


def test_invalid_and_empty_inputs(xb):
    from paper_2009_03076_b200.bricks import BrickBuildParams, InvalidCellsError, build_bricks
    from paper_2009_03076_b200.model import CellList
    from paper_2009_03076_b200.regions import build_regions

    dup = CellList([0, 0], [0, 0], [0, 0], [0, 0], [1.0, 1.0])
    with pytest.raises(InvalidCellsError) as e:
        build_bricks(dup)
    assert e.value.report.duplicates == [(0, 1)]
    over = CellList([0, 0], [0, 0], [0, 0], [0, 1], [1.0, 2.0])  # level-0 cell inside a level-1 cell
    with pytest.raises(InvalidCellsError):
        build_bricks(over)
    mis = CellList([1], [0], [0], [1], [1.0])
    with pytest.raises(InvalidCellsError):
        build_bricks(mis)
    empty = CellList([], [], [], [], [])
    m, t = build_bricks(empty, BrickBuildParams(keep_split_tree=True))
    assert m.n_bricks == 0 and m.n_cells == 0 and t.n_nodes == 0
    assert len(build_regions(m)) == 0


# ---------------------------------------------------------------- sampling


SAMPLED = [n for n in sorted(DIG) if "pts" in golden_model(n)]


@pytest.mark.parametrize("name", SAMPLED)
def test_samples_and_gradients_bit_exact(xb, name):
    from paper_2009_03076_b200.sampling import (gradient_central, gradient_central_clamped, gradient_points,
                                                sample_points)

    model, _, regions = _build(name)
    g = golden_model(name)
    pts = g["pts"]
    val, den, valid, rid = sample_points(model, regions, pts)
    assert np.array_equal(rid, g["pts_region"])
    inside = rid >= 0
    assert np.array_equal(val[inside], g["pts_value"][inside])
    assert np.array_equal(den[inside], g["pts_wsum"][inside])
    assert np.array_equal(valid[inside], g["pts_valid"][inside])
    grad, gvalid, _ = gradient_points(model, regions, pts[inside], rid[inside])
    assert np.array_equal(gvalid, g["grad_analytic_valid"][inside])
    assert np.array_equal(grad, g["grad_analytic"][inside])
    for t in range(0, len(pts), 7):
        gc = gradient_central(pts[t], regions, model)
        assert gc.valid == bool(g["grad_central_valid"][t])
        assert np.array_equal(gc.vec, g["grad_central"][t])
        if rid[t] >= 0:
            gcc = gradient_central_clamped(pts[t], regions[int(rid[t])], model)
            assert gcc.valid == bool(g["grad_clamped_valid"][t])
            assert np.array_equal(gcc.vec, g["grad_clamped"][t])


@pytest.mark.parametrize("name", ["gauss16", "two_cell", "mixed_levels"])
def test_oracle_scan_matches_golden_outside(xb, name):
    from paper_2009_03076_b200.sampling import basis_sample_oracle

    model, _, regions = _build(name)
    g = golden_model(name)
    cl = model.cell_list()
    for t in np.nonzero(g["pts_region"] < 0)[0][:40]:
        s = basis_sample_oracle(g["pts"][t], cl)
        assert (s.value, s.weight_sum, s.valid) == (g["pts_value"][t], g["pts_wsum"][t], bool(g["pts_valid"][t]))
    for t in np.nonzero(g["pts_region"] >= 0)[0][:40]:
        s = basis_sample_oracle(g["pts"][t], cl)
        assert (s.value, s.weight_sum, s.valid) == (g["pts_value"][t], g["pts_wsum"][t], bool(g["pts_valid"][t]))


def _scan_cells_py(cells, p):
    """_accumulate_cells (R/sampling.py:106-120) in plain Python floats (IEEE double, no FMA)."""
    w = np.exp2(cells.level.astype(np.float64))
    hx = 1.0 - np.abs((cells.i + 0.5 * w) - p[0]) / w
    hy = 1.0 - np.abs((cells.j + 0.5 * w) - p[1]) / w
    hz = 1.0 - np.abs((cells.k + 0.5 * w) - p[2]) / w
    num = den = 0.0
    for t in np.nonzero((hx > 0) & (hy > 0) & (hz > 0))[0]:  # list order
        h = float(hx[t]) * float(hy[t]) * float(hz[t])
        num += h * float(cells.values[t, 0])
        den += h
    return num, den


@pytest.mark.parametrize("name", ["gauss16", "mixed_levels"])
def test_oracle_scan_of_plain_cell_lists(xb, name):
    """basis_sample_oracle on a CellList that is not a model's canonical list (generator
    order, and shuffled): scanned in its own order like the reference (R/sampling.py:291-298)."""
    from paper_2009_03076_b200.model import CellList
    from paper_2009_03076_b200.sampling import EPS_WEIGHT, basis_sample_oracle

    g = golden_model(name)
    c0 = _cells(name)
    perm = np.random.default_rng(3).permutation(len(c0))
    c1 = CellList(c0.i[perm], c0.j[perm], c0.k[perm], c0.level[perm], c0.values[perm])
    for cl in (c0, c1):
        for t in range(0, len(g["pts"]), max(1, len(g["pts"]) // 25)):
            p = g["pts"][t]
            num, den = _scan_cells_py(cl, p)
            s = basis_sample_oracle(p, cl)
            assert s.weight_sum == den
            assert s.valid == (den > EPS_WEIGHT)
            if s.valid:
                assert s.value == num / den


# ---------------------------------------------------------------- traversal


@pytest.mark.parametrize("name", ["smoke", "gauss_aniso", "c1"])
@pytest.mark.parametrize("traversal", ["kd", "lbvh"])
def test_traversal_intervals_bit_exact(xb, name, traversal):
    """iterate_intervals (R/accel.py:414-424): the ordered k-d walk and the LBVH
    per-visit closest-hit queries both reproduce the reference's intervals."""
    from paper_2009_03076_b200.accel import TransferFunction, build_all_regions_bvh, build_volume_bvh, trace_rays

    model, _, regions = _build(name)
    g = golden_model(name)
    for tag in ("all", "pruned"):
        if tag == "all":
            bvh = build_all_regions_bvh(regions)
        else:
            bvh = build_volume_bvh(regions, TransferFunction(g["rays_pruned_domain"], g["rays_pruned_tf"]))
        got = trace_rays(bvh, g[f"rays_{tag}_o"], g[f"rays_{tag}_d"], 0.0, 1e9, traversal=traversal)
        off = g[f"rays_{tag}_off"]
        for q in range(len(off) - 1):
            s, e = off[q], off[q + 1]
            want = list(zip(g[f"rays_{tag}_tin"][s:e].tolist(), g[f"rays_{tag}_tout"][s:e].tolist(),
                            g[f"rays_{tag}_region"][s:e].tolist()))
            assert got[q] == want, f"{name}/{tag} ray {q}"


@pytest.mark.parametrize("name", ["smoke", "gauss_aniso", "c1", "two_cell", "single", "hole_pair"])
def test_lbvh_structure_and_point_queries(xb, name):
    """LBVH (Morton + Karras + refit): a full binary tree over exactly the active
    regions, every internal box the exact union of its children; point queries
    equal the reference's region of each golden sample point (R/accel.py:355-388)."""
    from paper_2009_03076_b200.accel import TransferFunction, build_all_regions_bvh, build_volume_bvh, point_query_batch

    model, _, regions = _build(name)
    vr = regions.value_range[:, 0] if len(regions) else np.zeros((0, 2))
    sets = [build_all_regions_bvh(regions)]
    if len(regions):
        lo, hi = float(vr[:, 0].min()), float(vr[:, 1].max())
        if hi > lo:  # a band TF leaves a strict subset active
            rgba = np.zeros((256, 4))
            rgba[100:160, 3] = 0.5
            sets.append(build_volume_bvh(regions, TransferFunction((lo, hi), rgba)))
    for bvh in sets:
        lo_, hi_, left, right, start, count, prims = bvh._lbvh()
        n = bvh.n_active
        assert np.array_equal(np.sort(prims), bvh.prims)
        if n == 0:
            assert len(left) == 1 and count[0] == 0
            continue
        assert len(left) == 2 * n - 1
        leaf = left < 0
        assert leaf.sum() == n and np.all(count[leaf] == 1) and np.all(right[leaf] == -1)
        assert np.array_equal(np.sort(start[leaf]), np.arange(n))
        seen = np.zeros(2 * n - 1, int)
        for i in np.nonzero(~leaf)[0]:
            for c in (left[i], right[i]):
                seen[c] += 1
            assert np.array_equal(lo_[i], np.minimum(lo_[left[i]], lo_[right[i]]))
            assert np.array_equal(hi_[i], np.maximum(hi_[left[i]], hi_[right[i]]))
        assert seen[0] == 0 and np.all(seen[1:] == 1)  # a tree rooted at node 0
        for k in np.nonzero(leaf)[0]:
            r = prims[start[k]]
            assert np.array_equal(lo_[k], regions.lo[r]) and np.array_equal(hi_[k], regions.hi[r])
    g = golden_model(name)
    if "pts" in g and len(regions):
        got = point_query_batch(sets[0], g["pts"])
        assert np.array_equal(got, g["pts_region"].astype(np.int32)), name


# ---------------------------------------------------------------- frames


FRAME_MODEL = {"smoke": "smoke", "ramp": "ramp", "c1": "c1", "aniso": "gauss_aniso"}


def _frame_keys():
    fr = golden_frames()
    return sorted({k[: -len("_rgba_f64")] for k in fr if k.endswith("_rgba_f64")})


def _camera(meta):
    from paper_2009_03076_b200.render import Camera

    return Camera(meta["position"], meta["forward"], meta["up"], meta["fov_y"], meta["width"], meta["height"])


def _params(meta):
    from paper_2009_03076_b200.render import MarchParams

    planes = [(p[:3], p[3]) for p in meta["clip_planes"]]
    return MarchParams(samples_per_cell=meta["spc"], rate_scale=meta["rate"], early_term_threshold=meta["early"],
                       seed=meta["seed"], gradient_mode=meta["gradient_mode"], clip_planes=planes)


KERNEL_VARIANTS = {  # xb_tuning fields (include/exabricks.h) of each frame-pipeline variant
    "warp": {},                                  # default: k_classify + k_walk leaf lists + k_warp
    "warp_cap1": {"leaf_cap": 1},                # every long ray falls back to the warp frontier
    "warp_nowalk": {"walk_lists": 0},            # k_warp's frontier only
    "warp_short": {"short_rays": 1},             # short rays one per lane (k_warp's second phase) even when few
    "warp_kshort": {"short_rays": 1, "fuse_short": 0},  # ... through the separate k_short launch
    "warp_2pass": {"walk_cap1": 2, "walk2_min": 0},     # k_walk2 continues (nearly) every walk
    "warp_grab8": {"grab_fixed": 8},             # fixed 8-ray grabs instead of the guided schedule
    "warp_wide_short": {"short_rays": 1, "short_leaves": 16, "short_samples": 4096},  # every complete list lane-per-ray
    "tile": {"kernel": 1},                       # one thread per pixel
    "lbvh": {"traversal": 1},                    # per-visit LBVH closest-hit queries (the reference's traversal)
}


@pytest.fixture
def kernel_env(request):
    """Select the frame-pipeline variant (xb_tuning_set) for the test."""
    from paper_2009_03076_b200 import _native as N

    with N.tuning(**KERNEL_VARIANTS[request.param]):
        yield request.param


@pytest.mark.parametrize("kernel_env", sorted(KERNEL_VARIANTS), indirect=True)
@pytest.mark.parametrize("key", _frame_keys())
def test_frames_match_reference(xb, key, frames, kernel_env):
    from paper_2009_03076_b200.accel import TransferFunction
    from paper_2009_03076_b200.render import build_scene, render_frame, render_frame_float

    meta = frame_meta(frames, key)
    model, _, regions = _build(FRAME_MODEL[key.split("_")[0]])
    tf = TransferFunction(meta["tf_domain"], frames[f"{key}_tf_rgba"])
    scene = build_scene(model, regions, tf, iso_value=meta["iso"])
    cam = _camera(meta)
    assert np.allclose(np.array(cam.basis()), np.array(meta["basis"]), rtol=0, atol=0)
    u8, f64, cnt, stats = render_frame_float(scene, cam, tf, _params(meta))
    want_f = frames[f"{key}_rgba_f64"]
    err = np.abs(f64 - want_f).max()
    assert err <= RGBA_TOL, f"{key}: max |dRGBA| = {err}"
    assert np.abs(u8.astype(int) - frames[f"{key}_rgba_u8"].astype(int)).max() <= 1
    assert np.array_equal(cnt[..., 0].ravel(), frames[f"{key}_px_regions"])
    assert np.array_equal(cnt[..., 1].ravel(), frames[f"{key}_px_samples"])
    fr = render_frame(scene, cam, tf, _params(meta))
    assert np.array_equal(fr.rgba, u8)
    assert fr.stats.samples == int(frames[f"{key}_px_samples"].sum())
    assert fr.stats.regions == int(frames[f"{key}_px_regions"].sum())


@pytest.mark.parametrize("key", _frame_keys())
def test_cell_location_frames_match_reference(xb, key, frames):
    """use_celllocation=True: per-sample split-tree brick collection (the paper's
    cell-location baseline, R/render.py:423-425) gives the reference's frames."""
    from paper_2009_03076_b200.accel import TransferFunction
    from paper_2009_03076_b200.render import build_scene, render_frame_float

    meta = frame_meta(frames, key)
    model, tree, regions = _build(FRAME_MODEL[key.split("_")[0]], keep_tree=True)
    tf = TransferFunction(meta["tf_domain"], frames[f"{key}_tf_rgba"])
    scene = build_scene(model, regions, tf, iso_value=meta["iso"], tree=tree)
    u8, f64, cnt, stats = render_frame_float(scene, _camera(meta), tf, _params(meta), use_celllocation=True)
    assert np.abs(f64 - frames[f"{key}_rgba_f64"]).max() <= RGBA_TOL
    assert np.array_equal(cnt[..., 0].ravel(), frames[f"{key}_px_regions"])
    assert np.array_equal(cnt[..., 1].ravel(), frames[f"{key}_px_samples"])


def test_cell_location_uploaded_tree(xb):
    """A model uploaded from arrays gets the scene's SplitTree attached on demand."""
    from paper_2009_03076_b200.accel import TransferFunction
    from paper_2009_03076_b200.model import AmrModel
    from paper_2009_03076_b200.orbit import orbit_cameras
    from paper_2009_03076_b200.regions import build_regions
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame, render_frame_float

    model, tree, _ = _build("smoke", keep_tree=True)
    m2 = AmrModel(model.field_names, model.brick_lower, model.brick_level, model.brick_dims, model.scalars)
    regions = build_regions(m2)
    lo, hi = m2.value_range(0)
    tf = TransferFunction.grayscale((lo, hi), max_alpha=0.5)
    scene = build_scene(m2, regions, tf, tree=tree)
    cam = orbit_cameras(regions.bounds, 1, 64, 48)[0]
    p = MarchParams(seed=3, gradient_mode="analytic")
    a = render_frame_float(scene, cam, tf, p)
    b = render_frame_float(scene, cam, tf, p, use_celllocation=True)
    assert np.array_equal(a[2], b[2]) and np.abs(a[1] - b[1]).max() <= RGBA_TOL
    assert np.array_equal(render_frame(scene, cam, tf, p).rgba, render_frame(scene, cam, tf, p, True).rgba)


# ---------------------------------------------------------------- acceptance properties (T/test_acceptance.py)


def test_two_cell_rays_opacity_law(xb):
    from paper_2009_03076_b200.accel import TransferFunction
    from paper_2009_03076_b200.bricks import BrickBuildParams, build_bricks
    from paper_2009_03076_b200.model import CellList
    from paper_2009_03076_b200.regions import build_regions
    from paper_2009_03076_b200.render import MarchParams, build_scene, integrate_ray

    g = dict(np.load(GOLDEN / "rays.npz"))["two_cell_rays"]
    cl = CellList([0, 1], [0, 0], [0, 0], [0, 0], [4.0, 4.0])
    for width, rate, r, gg, b, a, nreg, nsmp in g:
        m, _ = build_bricks(cl, BrickBuildParams(max_brick_width=int(width)))
        tf = TransferFunction.constant_alpha((3.0, 5.0), 0.3)
        sc = build_scene(m, build_regions(m), tf)
        out, st = integrate_ray((-3.0, 0.5, 0.5), (1.0, 0.0, 0.0), sc, tf,
                                MarchParams(rate_scale=rate, gradient_mode="none", early_term_threshold=1.0))
        assert np.abs(out - [r, gg, b, a]).max() <= 1e-12
        assert st == {"regions": int(nreg), "samples": int(nsmp)}
        assert out[3] == pytest.approx(1.0 - (1.0 - 0.3) ** (3.0 / 0.5), abs=1e-4)


def test_space_skipping_neutral_and_transparent(xb):
    from paper_2009_03076_b200.accel import TransferFunction, build_all_regions_bvh
    from paper_2009_03076_b200.orbit import orbit_cameras
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame
    import dataclasses

    model, _, regions = _build("smoke")
    vmin, vmax = regions.value_range[:, 0, 0].min(), regions.value_range[:, 0, 1].max()
    rgba = np.tile(np.linspace(0.0, 1.0, 256)[:, None], (1, 4))
    rgba[:128, 3] = 0.0
    tf = TransferFunction((vmin, vmax), rgba)
    scene = build_scene(model, regions, tf)
    unpruned = dataclasses.replace(scene, volume_bvh=build_all_regions_bvh(regions))
    assert scene.volume_bvh.n_active < unpruned.volume_bvh.n_active
    cam = orbit_cameras(regions.bounds, 1, 96, 72)[0]
    a = render_frame(scene, cam, tf, MarchParams(seed=9))
    b = render_frame(unpruned, cam, tf, MarchParams(seed=9))
    assert np.array_equal(a.rgba, b.rgba) and a.rgba.any()
    assert 0 < a.stats.samples <= b.stats.samples
    clear = TransferFunction.constant_alpha((vmin, vmax), 0.0)
    blank = render_frame(build_scene(model, regions, clear), cam, clear, MarchParams(seed=9))
    assert blank.stats.samples == 0 and not blank.rgba.any()


def test_iso_hits_analytic_plane(xb):
    from paper_2009_03076_b200.accel import TransferFunction, build_iso_bvh
    from paper_2009_03076_b200.render import build_scene, iso_intersect

    model, _, regions = _build("ramp")
    tf = TransferFunction.constant_alpha((0.0, 16.0), 0.0)
    scene = build_scene(model, regions, tf)
    bvh = build_iso_bvh(regions, 7.25)
    rng = np.random.default_rng(21)
    for _ in range(200):
        o = np.array([-4.0, rng.uniform(2.0, 14.0), rng.uniform(2.0, 14.0)])
        d = np.array([1.0, rng.uniform(-0.05, 0.05), rng.uniform(-0.05, 0.05)])
        d /= np.linalg.norm(d)
        hit = iso_intersect(o, d, bvh, scene, 7.25)
        assert hit is not None
        t, grad = hit
        assert abs((o + t * d)[0] - 7.25) <= 1e-4
        assert np.allclose(grad / np.linalg.norm(grad), [1, 0, 0], atol=1e-6)
    empty = build_iso_bvh(regions, 99.0)
    assert empty.is_empty
    assert iso_intersect([-4.0, 8.0, 8.0], [1.0, 0.0, 0.0], empty, scene, 99.0) is None


def test_opaque_tf_one_sample_per_region(xb):
    from paper_2009_03076_b200.accel import TransferFunction
    from paper_2009_03076_b200.orbit import orbit_cameras
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame

    model, _, regions = _build("smoke")
    lo, hi = model.value_range(0)
    tf = TransferFunction((lo, hi), np.ones((256, 4)))
    f = render_frame(build_scene(model, regions, tf), orbit_cameras(regions.bounds, 1, 48, 36)[0], tf,
                     MarchParams(gradient_mode="none"))
    assert f.stats.samples == f.stats.regions
    assert np.array_equal(np.unique(f.rgba[:, :, 3]), [0, 255])


# ---------------------------------------------------------------- larger inputs vs the oracle


def _oracle_frame(model, regions, tf, cam, params, pix_range=None):
    osc = oracle.OracleScene({k: getattr(model, k) for k in MODEL_KEYS}, {k: getattr(regions, k) for k in REGION_KEYS})
    osc.set_tf(tf.domain, tf.rgba)
    r, u, f = cam.basis()
    ocam = oracle.camera_struct(cam.width, cam.height, cam.position, r, u, f, math.tan(math.radians(cam.fov_y) * 0.5),
                                cam.width / cam.height)
    return osc.render(ocam, tf.domain, tf.rgba, pix_range=pix_range, seed=params.seed,
                      gradient_mode=params.gradient_mode, early=params.early_term_threshold)


def test_acceptance_million_cells_vs_oracle(xb):
    """The reference's 1.59M-cell benchmark spec (T/test_acceptance.py:376-397): builders
    bit-exact vs the oracle, a 512x512 analytic frame within tolerance."""
    from paper_2009_03076_b200 import io as xio
    from paper_2009_03076_b200.accel import TransferFunction
    from paper_2009_03076_b200.bricks import build_bricks
    from paper_2009_03076_b200.orbit import orbit_cameras
    from paper_2009_03076_b200.regions import build_regions
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame_float

    spec = xio.SyntheticSpec(field="gaussian", extent=(128, 128, 128), max_level=3, threshold=0.0035, seed=11,
                             holes=((40, 88, 40, 10.0),), refine_spheres=((96, 32, 96, 12.0),))
    cells = xio.generate_synthetic(spec)
    assert len(cells) >= 1_000_000
    model, _ = build_bricks(cells)
    regions = build_regions(model)
    om = oracle.build_bricks(cells.i, cells.j, cells.k, cells.level, cells.values)
    for k in MODEL_KEYS:
        assert np.array_equal(getattr(model, k), om[k]), k
    orr = oracle.build_regions(*(om[k] for k in MODEL_KEYS))
    for k in REGION_KEYS:
        assert np.array_equal(getattr(regions, k), orr[k]), k
    vmin, vmax = regions.value_range[:, 0, 0].min(), regions.value_range[:, 0, 1].max()
    tf = TransferFunction.grayscale((vmin, vmax))
    scene = build_scene(model, regions, tf)
    cam = orbit_cameras(regions.bounds, 2, 512, 512)[1]
    params = MarchParams(gradient_mode="analytic", seed=5)
    u8, f64, cnt, stats = render_frame_float(scene, cam, tf, params)
    rows = slice(160 * 512, 224 * 512)  # a 64-row band through the volume keeps the oracle fast
    of, ou, pr, ps = _oracle_frame(model, regions, tf, cam, params, (rows.start, rows.stop))
    assert np.abs(f64.reshape(-1, 4)[rows] - of).max() <= RGBA_TOL
    assert np.array_equal(cnt.reshape(-1, 2)[rows, 0], pr)
    assert np.array_equal(cnt.reshape(-1, 2)[rows, 1], ps)
    # whole frame: the warp-per-ray kernel (default) must equal the per-lane
    # persistent kernel and the one-thread-per-pixel kernel everywhere, on every
    # repetition
    from paper_2009_03076_b200 import _native as N

    for kern in ("tile", "warp_cap1", "warp_nowalk", "warp_short", "warp_kshort", "warp_2pass", "lbvh"):
        with N.tuning(**KERNEL_VARIANTS[kern]):
            u8t, f64t, cntt, stt = render_frame_float(scene, cam, tf, params)
        assert np.array_equal(cnt, cntt), kern
        assert np.abs(f64 - f64t).max() <= RGBA_TOL, kern
    for _ in range(3):
        u8r, f64r, cntr, str_ = render_frame_float(scene, cam, tf, params)
        assert np.array_equal(cntr, cnt) and np.array_equal(u8r, u8)
        assert tuple(str_[:2]) == tuple(stats[:2])


# ---------------------------------------------------------------- screen tiles (multi-GPU layout on one GPU)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_tiled_ranks_reassemble_the_frame(xb, world):
    """Each rank's packed tiles (global pixel index in the jitter hash), rendered
    here one rank after another, unpack (device `xb_unpack_tiles` and the host
    mirror) to exactly the single-GPU frame; counters add up."""
    import torch

    from paper_2009_03076_b200 import _native as N
    from paper_2009_03076_b200.accel import TransferFunction
    from paper_2009_03076_b200.orbit import orbit_cameras
    from paper_2009_03076_b200.parallel import TILE_PX, tiles_of_rank, tiles_per_rank, unpack_host
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame, render_native

    model, _, regions = _build("gauss_aniso")
    lo, hi = model.value_range(0)
    tf = TransferFunction.grayscale((lo, hi), max_alpha=0.6)
    scene = build_scene(model, regions, tf)
    W, H = 100, 52  # partial tiles on both edges
    cam = orbit_cameras(regions.bounds, 3, W, H)[1]
    p = MarchParams(seed=9, gradient_mode="analytic")
    full = render_frame(scene, cam, tf, p)
    slots = tiles_per_rank(W, H, world)
    gathered = torch.zeros((world * slots * TILE_PX, 4), dtype=torch.uint8, device="cuda")
    bufs, tot = [], np.zeros(2, np.int64)
    for r in range(world):
        part = gathered[r * slots * TILE_PX:(r + 1) * slots * TILE_PX]
        if tiles_of_rank(W, H, r, world):
            st = render_native(scene, cam, tf, p, part.data_ptr(), tile_rank=r, tile_world=world)
            tot += st[:2]
        bufs.append(part.cpu().numpy())
    assert np.array_equal(unpack_host(bufs, W, H, world), full.rgba)
    img = torch.empty((H, W, 4), dtype=torch.uint8, device="cuda")
    N.check(N.lib().xb_unpack_tiles(N.ptr(gathered.data_ptr()), slots, world, W, H, N.ptr(img.data_ptr()), None))
    torch.cuda.synchronize()
    assert np.array_equal(img.cpu().numpy(), full.rgba)
    assert tuple(tot) == (full.stats.regions, full.stats.samples)


def test_large_frames_render_in_bands(xb):
    """Frames above 4M pixels run as interleaved tile bands (bounded walk scratch):
    pixel-identical to the single-pass float path, same counters."""
    from paper_2009_03076_b200.accel import TransferFunction
    from paper_2009_03076_b200.orbit import orbit_cameras
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame, render_frame_float

    model, _, regions = _build("smoke")
    lo, hi = model.value_range(0)
    tf = TransferFunction.grayscale((lo, hi), max_alpha=0.5)
    scene = build_scene(model, regions, tf)
    cam = orbit_cameras(regions.bounds, 3, 2304, 2048)[1]  # 4.7M px -> 2 bands
    params = MarchParams(seed=2, gradient_mode="analytic")
    fr = render_frame(scene, cam, tf, params)
    u8, f64, cnt, st = render_frame_float(scene, cam, tf, params)
    assert np.array_equal(fr.rgba, u8)
    assert (fr.stats.regions, fr.stats.samples) == (int(st[0]), int(st[1])) == (int(cnt[..., 0].sum()),
                                                                               int(cnt[..., 1].sum()))
    assert fr.stats.samples > 0


def test_render_frames_pipeline_equals_render_frame(xb):
    """render_frames (march of frame k+1 overlapping the copy of frame k) returns the
    same frames, in order, as one render_frame call per camera."""
    from paper_2009_03076_b200.accel import TransferFunction
    from paper_2009_03076_b200.orbit import orbit_cameras, run_bench
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame, render_frames

    model, _, regions = _build("smoke")
    lo, hi = model.value_range(0)
    tf = TransferFunction.grayscale((lo, hi), max_alpha=0.5)
    scene = build_scene(model, regions, tf)
    cams = orbit_cameras(regions.bounds, 5, 120, 80) + orbit_cameras(regions.bounds, 3, 64, 48)
    params = MarchParams(seed=4, gradient_mode="analytic")
    got = list(render_frames(scene, cams, tf, params))
    assert len(got) == len(cams)
    for cam, fr in zip(cams, got):
        ref = render_frame(scene, cam, tf, params)
        assert fr.rgba.shape == ref.rgba.shape and np.array_equal(fr.rgba, ref.rgba)
        assert (fr.stats.regions, fr.stats.samples) == (ref.stats.regions, ref.stats.samples)
        assert fr.stats.ms > 0
    rows, _ = run_bench(scene, tf, params, 4, 96, 64, pipelined=True)
    rows2, _ = run_bench(scene, tf, params, 4, 96, 64)
    assert [(r.regions, r.samples) for r in rows] == [(r.regions, r.samples) for r in rows2]
