"""Generate the golden fixtures that pin the CPU oracle and the CUDA path.

Runs ONLY in the build container, where the reference package (`amrvol`,
Python + numba) can be imported read-only:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Everything the reference computes here goes into `tests/golden/*.npz`; the GPU
box never sees the reference, only these files.  Per case we store:

* the synthetic cell list (or a sha256 of it for the larger specs),
* the reference `build_bricks` / `build_regions` output arrays (full arrays for
  small models, sha256 digests for all),
* point samples (`basis_sample_region` / `basis_sample_oracle`) and gradients
  (analytic, central, clamped central),
* ray traversals (`iterate_intervals`) on the all-regions and a pruned BVH,
* frames: float64 RGBA *before* RGBA8 quantisation, the uint8 frame the
  reference `render_frame` returns, and the per-pixel region / sample counters.

The float frame comes from a harness loop that repeats the per-pixel body of
`amrvol.render._render_kernel` (render.py:521-578) while calling the
reference's own numba device functions (`_rho_hash`, `_clip_ray`, `_iso_ray`,
`_volume_ray`, `_shade_factor`) so the arithmetic is the reference's.
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time
import zlib
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent

from numba import njit, prange  # noqa: E402

from amrvol import io as avio  # noqa: E402
from amrvol import render as R  # noqa: E402
from amrvol.accel import (  # noqa: E402
    TransferFunction,
    build_all_regions_bvh,
    build_iso_bvh,
    build_volume_bvh,
    iterate_intervals,
    max_opacity,
)
from amrvol.bench import orbit_cameras  # noqa: E402
from amrvol.bricks import BrickBuildParams, build_bricks  # noqa: E402
from amrvol.model import CellList  # noqa: E402
from amrvol.regions import build_regions, point_to_region  # noqa: E402
from amrvol.sampling import (  # noqa: E402
    basis_sample_oracle,
    basis_sample_region,
    gradient_analytic,
    gradient_central,
    gradient_central_clamped,
)


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def cells_of(i, j, k, lev, vals):
    v = np.asarray(vals, np.float32)
    if v.ndim == 1:
        v = v[:, None]
    return CellList(np.asarray(i), np.asarray(j), np.asarray(k), np.asarray(lev), v, ("value",))


# ---------------------------------------------------------------------------
# model cases

SPECS = {
    "gauss16": avio.SyntheticSpec(
        field="gaussian", extent=(16, 16, 16), max_level=3, threshold=0.05, seed=5,
        holes=((12, 4, 12, 2.5),), refine_spheres=((4, 12, 4, 2.5),),
    ),
    "gauss24": avio.SyntheticSpec(
        field="gaussian", extent=(24, 24, 24), max_level=3, threshold=0.08, seed=17,
        holes=((6, 18, 6, 3.0),), refine_spheres=((18, 6, 18, 3.5),),
    ),
    "smoke": avio.SyntheticSpec(
        field="gaussian", extent=(32, 32, 32), max_level=3, threshold=0.04, seed=3,
        holes=((10, 10, 10, 4.0),), refine_spheres=((24, 24, 24, 5.0),),
    ),
    "octaves32": avio.SyntheticSpec(
        field="octaves", extent=(32, 32, 32), max_level=3, threshold=0.35, seed=7,
        holes=((22, 22, 8, 3.0),), refine_spheres=((8, 24, 24, 3.5),),
    ),
    "gauss48": avio.SyntheticSpec(
        field="gaussian", extent=(48, 48, 48), max_level=3, threshold=0.02, seed=13,
        holes=((20, 36, 20, 4.0),), refine_spheres=((36, 12, 36, 5.0),),
    ),
    "ramp": avio.SyntheticSpec(
        field="ramp", extent=(16, 16, 16), max_level=2, threshold=0.0, seed=0,
        field_params={"direction": (1.0, 0.0, 0.0)},
    ),
    "constant": avio.SyntheticSpec(
        field="constant", extent=(16, 16, 16), max_level=2, threshold=np.inf,
        seed=0, refine_spheres=((4, 4, 4, 3.0),), field_params={"c": 7.5},
    ),
    "c1": avio.SyntheticSpec(field="gaussian", extent=(64, 64, 64), max_level=1, threshold=0.04, seed=0),
    "oct8_s1": avio.SyntheticSpec(field="octaves", extent=(8, 8, 8), max_level=2, threshold=0.05, seed=1, holes=((4, 4, 4, 1.5),)),
    "oct8_s2": avio.SyntheticSpec(field="octaves", extent=(8, 8, 8), max_level=2, threshold=0.05, seed=2, holes=((4, 4, 4, 1.5),)),
    # asymmetric extent + negative-free multi-level with strong jumps
    "gauss_aniso": avio.SyntheticSpec(
        field="gaussian", extent=(64, 32, 16), max_level=3, threshold=0.03, seed=4,
        holes=((40, 16, 8, 3.0),), refine_spheres=((16, 16, 8, 4.0),),
        field_params={"center": (20.0, 15.0, 9.0), "sigma": 9.0},
    ),
}

HAND = {
    "two_cell": (cells_of([0, 1], [0, 0], [0, 0], [0, 0], [0.0, 10.0]), 32),
    "two_cell_w1": (cells_of([0, 1], [0, 0], [0, 0], [0, 0], [1.0, 5.0]), 1),
    "hole_pair": (cells_of([0, 2], [0, 0], [0, 0], [0, 0], [1.0, 2.0]), 32),
    "mixed_levels": (cells_of([0, 1, 2], [0, 0, 0], [0, 0, 0], [0, 0, 1], [1.0, 2.0, 3.0]), 32),
    "negative": (cells_of([-8, -4], [-4, -4], [0, 0], [2, 2], [1.0, 2.0]), 32),
    "single": (cells_of([4], [4], [4], [2], [3.5]), 32),
    "flat4": None,  # filled below: dense 4^3 level-0 grid with a linear field
}

# brick-width variants of smoke / oct8 (builder edge cases)
WIDTH_VARIANTS = {"smoke_w4": ("smoke", 4), "oct8_s1_w1": ("oct8_s1", 1), "oct8_s2_w3": ("oct8_s2", 3), "gauss24_w7": ("gauss24", 7)}

FULL_ARRAYS_MAX_REGIONS = 40_000


def flat_grid(n):
    ax = np.arange(n)
    i, j, k = np.meshgrid(ax, ax, ax, indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    v = 2 * (i + 0.5) + 3 * (j + 0.5) - (k + 0.5) + 1
    return cells_of(i, j, k, np.zeros_like(i), v)


HAND["flat4"] = (flat_grid(4), 32)

MODEL_ATTRS = ("brick_lower", "brick_level", "brick_dims", "brick_offset", "scalars")
REGION_ATTRS = ("lo", "hi", "brick_off", "brick_ids", "value_range", "finest_width")
TREE_ATTRS = ("axis", "pos", "left", "right", "brick_start", "brick_count", "box_lo", "box_hi", "max_half")


def build_case(name, cells, width):
    model, tree = build_bricks(cells, BrickBuildParams(max_brick_width=width, keep_split_tree=True))
    regions = build_regions(model)
    return model, tree, regions


def store_model(out, prefix, cells, model, tree, regions, full):
    digests = {}
    for a in ("i", "j", "k", "level", "values"):
        digests[f"cells.{a}"] = sha(getattr(cells, a))
    for a in MODEL_ATTRS:
        digests[f"model.{a}"] = sha(getattr(model, a))
    for a in REGION_ATTRS:
        digests[f"regions.{a}"] = sha(getattr(regions, a))
    for a in TREE_ATTRS:
        digests[f"tree.{a}"] = sha(getattr(tree, a))
    if full:
        for a in ("i", "j", "k", "level", "values"):
            out[f"{prefix}cells_{a}"] = getattr(cells, a)
        for a in MODEL_ATTRS:
            out[f"{prefix}model_{a}"] = getattr(model, a)
        for a in REGION_ATTRS:
            out[f"{prefix}regions_{a}"] = getattr(regions, a)
        for a in TREE_ATTRS:
            out[f"{prefix}tree_{a}"] = getattr(tree, a)
    return digests


def sample_block(out, prefix, model, regions, rng, n):
    """Point samples: half strictly interior to random regions, half uniform."""
    b = regions.bounds
    idx = rng.integers(0, len(regions), n // 2)
    u = rng.uniform(0.05, 0.95, (n // 2, 3))
    p_in = regions.lo[idx] + u * (regions.hi[idx] - regions.lo[idx])
    p_any = rng.uniform(b.lo - 0.5, b.hi + 0.5, (n - n // 2, 3))
    pts = np.concatenate([p_in, p_any])
    # include a few lattice-aligned points (exact centres / faces) where sign rules matter
    lat = np.floor(pts[:64] * 2.0) / 2.0
    pts = np.concatenate([pts, lat])
    canon = model.cell_list()
    rid = np.full(len(pts), -1, np.int64)
    val = np.zeros(len(pts))
    wsum = np.zeros(len(pts))
    ok = np.zeros(len(pts), bool)
    ga = np.zeros((len(pts), 3))
    ga_ok = np.zeros(len(pts), bool)
    gc = np.zeros((len(pts), 3))
    gc_ok = np.zeros(len(pts), bool)
    gcc = np.zeros((len(pts), 3))
    gcc_ok = np.zeros(len(pts), bool)
    for t, p in enumerate(pts):
        r = point_to_region(regions, p)
        if r is None:
            s = basis_sample_oracle(p, canon)
        else:
            rid[t] = r
            s = basis_sample_region(p, regions[r], model)
            g = gradient_analytic(p, regions[r], model)
            ga[t], ga_ok[t] = g.vec, g.valid
            g = gradient_central_clamped(p, regions[r], model)
            gcc[t], gcc_ok[t] = g.vec, g.valid
        val[t], wsum[t], ok[t] = s.value, s.weight_sum, s.valid
        g = gradient_central(p, regions, model)
        gc[t], gc_ok[t] = g.vec, g.valid
    out[f"{prefix}pts"] = pts
    out[f"{prefix}pts_region"] = rid
    out[f"{prefix}pts_value"] = val
    out[f"{prefix}pts_wsum"] = wsum
    out[f"{prefix}pts_valid"] = ok
    out[f"{prefix}grad_analytic"] = ga
    out[f"{prefix}grad_analytic_valid"] = ga_ok
    out[f"{prefix}grad_central"] = gc
    out[f"{prefix}grad_central_valid"] = gc_ok
    out[f"{prefix}grad_clamped"] = gcc
    out[f"{prefix}grad_clamped_valid"] = gcc_ok


def rays_block(out, prefix, regions, bvh, rng, n, tag):
    b = regions.bounds
    origins, dirs, flat = [], [], []
    offs = [0]
    for _ in range(n):
        o = rng.uniform(b.lo - 10, b.hi + 10)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        if rng.uniform() < 0.15:  # axis-parallel rays exercise the half-open rule
            d = np.zeros(3)
            d[rng.integers(0, 3)] = rng.choice([-1.0, 1.0])
            o = rng.uniform(b.lo, b.hi)
        got = list(iterate_intervals(bvh, o, d, 0.0, 1e9))
        origins.append(o)
        dirs.append(d)
        for g in got:
            flat.append((g.t_in, g.t_out, g.region))
        offs.append(len(flat))
    out[f"{prefix}rays_{tag}_o"] = np.array(origins)
    out[f"{prefix}rays_{tag}_d"] = np.array(dirs)
    arr = np.array(flat, dtype=np.float64).reshape(-1, 3)
    out[f"{prefix}rays_{tag}_tin"] = arr[:, 0]
    out[f"{prefix}rays_{tag}_tout"] = arr[:, 1]
    out[f"{prefix}rays_{tag}_region"] = arr[:, 2].astype(np.int64)
    out[f"{prefix}rays_{tag}_off"] = np.array(offs, np.int64)


# ---------------------------------------------------------------------------
# float frame harness: the per-pixel body of render.py:521-578, float output


@njit(cache=True, parallel=True)
def _frame_float(out_f, px_regions, px_samples, width, height, cpos, cright, cup, cfwd, tan_half, aspect, planes,
                 vb, ib, ab, reg_lo, reg_hi, roff, rids, reg_finest, blo, blev, bdims, boff, vals,
                 tf_lo, tf_hi, tf_rgba, spc, rate, early, seed, grad_mode, iso_on, iso_value, iso_rgb):
    vnlo, vnhi, vnl, vnr, vns, vnc, vprims = vb
    inlo, inhi, inl, inr, ins, inc, iprims = ib
    anlo, anhi, anl, anr, ans, anc, aprims = ab
    dummy_f = np.zeros((1, 3))
    dummy_i = np.zeros(1, np.int32)
    dummy_h = np.zeros(1)
    for pix in prange(width * height):
        buf = np.empty(1, np.int32)
        x = pix % width
        y = pix // width
        sx = (2.0 * (x + 0.5) / width - 1.0) * tan_half * aspect
        sy = (1.0 - 2.0 * (y + 0.5) / height) * tan_half
        dx = cfwd[0] + sx * cright[0] + sy * cup[0]
        dy = cfwd[1] + sx * cright[1] + sy * cup[1]
        dz = cfwd[2] + sx * cright[2] + sy * cup[2]
        inv = 1.0 / math.sqrt(dx * dx + dy * dy + dz * dz)
        dx *= inv
        dy *= inv
        dz *= inv
        ox, oy, oz = cpos[0], cpos[1], cpos[2]
        rho = R._rho_hash(pix, seed)
        tmin, tmax = R._clip_ray(planes, ox, oy, oz, dx, dy, dz, 0.0, 1.0e30)
        if tmin >= tmax:
            for c in range(4):
                out_f[y, x, c] = 0.0
            px_regions[pix] = 0
            px_samples[pix] = 0
            continue
        t_end = tmax
        hit = False
        hx = hy = hz = 0.0
        if iso_on:
            hit, t_hit, hx, hy, hz = R._iso_ray(
                inlo, inhi, inl, inr, ins, inc, iprims, reg_lo, reg_hi, roff, rids, reg_finest,
                blo, blev, bdims, boff, vals, ox, oy, oz, dx, dy, dz, tmin, tmax, rho, spc, rate, iso_value,
            )
            if hit:
                t_end = t_hit
        r, g, b, a, nreg, nsmp = R._volume_ray(
            vnlo, vnhi, vnl, vnr, vns, vnc, vprims, anlo, anhi, anl, anr, ans, anc, aprims,
            reg_lo, reg_hi, roff, rids, reg_finest, blo, blev, bdims, boff, vals, tf_lo, tf_hi, tf_rgba,
            ox, oy, oz, dx, dy, dz, tmin, t_end, rho, spc, rate, early, grad_mode,
            False, dummy_i, dummy_i, dummy_i, dummy_i, dummy_i, dummy_f, dummy_f, dummy_h, buf,
        )
        if hit:
            f = R._shade_factor(hx, hy, hz, dx, dy, dz)
            w = 1.0 - a
            r += w * iso_rgb[0] * f
            g += w * iso_rgb[1] * f
            b += w * iso_rgb[2] * f
            a = 1.0
        out_f[y, x, 0] = r
        out_f[y, x, 1] = g
        out_f[y, x, 2] = b
        out_f[y, x, 3] = a
        px_regions[pix] = nreg
        px_samples[pix] = nsmp


def render_both(scene, cam, tf, params):
    """(float64 RGBA, uint8 RGBA from render_frame, px_regions, px_samples)."""
    w, h = cam.width, cam.height
    right, up, fwd = cam.basis()
    ab = scene.regions.point_index
    vb = R._bvh_args(scene.volume_bvh, ab)
    iso_on = scene.iso_bvh is not None and scene.iso_value is not None
    ib = R._bvh_args(scene.iso_bvh, ab)
    reg = scene.regions
    out_f = np.zeros((h, w, 4))
    pr = np.zeros(w * h, np.int64)
    ps = np.zeros(w * h, np.int64)
    _frame_float(
        out_f, pr, ps, w, h, cam.position, right, up, fwd,
        math.tan(math.radians(cam.fov_y) * 0.5), w / h, params.plane_array(),
        vb, ib, ab.kernel_args()[:7],
        np.ascontiguousarray(reg.lo), np.ascontiguousarray(reg.hi), reg.brick_off, reg.brick_ids, reg.finest_width,
        scene.model.brick_lower, scene.model.brick_level, scene.model.brick_dims, scene.model.brick_offset,
        scene.field_values, tf.domain[0], tf.domain[1], tf.rgba,
        params.samples_per_cell, params.rate_scale, params.early_term_threshold,
        np.uint64(params.seed & ((1 << 64) - 1)), R.GRADIENT_MODES[params.gradient_mode],
        iso_on, float(scene.iso_value) if iso_on else 0.0, np.array(R.ISO_COLOR),
    )
    fr = R.render_frame(scene, cam, tf, params)
    assert fr.stats.regions == int(pr.sum()) and fr.stats.samples == int(ps.sum())
    q = np.clip(out_f, 0.0, 1.0) * 255.0 + 0.5
    assert np.array_equal(q.astype(np.uint8), fr.rgba), "float harness disagrees with render_frame"
    return out_f, fr.rgba, pr, ps


def store_frame(out, key, scene, cam, tf, params, iso=None):
    f, u8, pr, ps = render_both(scene, cam, tf, params)
    right, up, fwd = cam.basis()
    out[f"{key}_rgba_f64"] = f
    out[f"{key}_rgba_u8"] = u8
    out[f"{key}_px_regions"] = pr.astype(np.int32)
    out[f"{key}_px_samples"] = ps.astype(np.int32)
    meta = {
        "width": cam.width, "height": cam.height, "fov_y": cam.fov_y,
        "position": cam.position.tolist(), "forward": cam.forward.tolist(), "up": cam.up.tolist(),
        "basis": [right.tolist(), up.tolist(), fwd.tolist()],
        "tan_half": math.tan(math.radians(cam.fov_y) * 0.5),
        "tf_domain": list(tf.domain), "spc": params.samples_per_cell, "rate": params.rate_scale,
        "early": params.early_term_threshold, "seed": params.seed, "gradient_mode": params.gradient_mode,
        "clip_planes": params.plane_array().tolist(), "iso": iso,
    }
    out[f"{key}_tf_rgba"] = tf.rgba
    out[f"{key}_meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    return meta


def main():
    t0 = time.time()
    digests = {}
    rng_master = np.random.default_rng(20240917)

    # ---- builder + sampling fixtures -------------------------------------------------
    built = {}
    for name in list(HAND) + list(SPECS) + list(WIDTH_VARIANTS):
        if name in HAND:
            cells, width = HAND[name]
        elif name in SPECS:
            cells, width = avio.generate_synthetic(SPECS[name]), 32
        else:
            base, width = WIDTH_VARIANTS[name]
            cells = built[base][0]
        model, tree, regions = build_case(name, cells, width)
        built[name] = (cells, model, tree, regions, width)
        full = len(regions) <= FULL_ARRAYS_MAX_REGIONS
        out = {}
        digests[name] = store_model(out, "", cells, model, tree, regions, full)
        digests[name]["max_brick_width"] = width
        digests[name]["n_cells"] = len(cells)
        digests[name]["n_bricks"] = model.n_bricks
        digests[name]["n_regions"] = len(regions)
        digests[name]["full"] = full
        if name in SPECS:
            s = SPECS[name]
            digests[name]["spec"] = {
                "field": s.field, "extent": list(s.extent), "max_level": s.max_level,
                "threshold": (None if not np.isfinite(s.threshold) else s.threshold),
                "threshold_inf": bool(not np.isfinite(s.threshold)), "seed": s.seed,
                "holes": [list(h) for h in s.holes], "refine_spheres": [list(h) for h in s.refine_spheres],
                "field_params": {k: (list(v) if isinstance(v, tuple) else v) for k, v in s.field_params.items()},
            }
        if name in WIDTH_VARIANTS:
            digests[name]["cells_from"] = WIDTH_VARIANTS[name][0]
        if len(regions) and name not in WIDTH_VARIANTS:
            n_pts = 600 if name in ("c1", "gauss48") else 1000
            sample_block(out, "", model, regions, np.random.default_rng(zlib.crc32(name.encode())), n_pts)
        if name in ("smoke", "gauss_aniso", "c1"):
            rng = np.random.default_rng(21)
            rays_block(out, "", regions, build_all_regions_bvh(regions), rng, 40 if name != "c1" else 16, "all")
            vr = regions.value_range[:, 0]
            lo, hi = vr.min(), vr.max()
            alpha = np.zeros(256)
            alpha[150:] = 1.0
            tf = TransferFunction((lo, hi), np.stack([np.ones(256)] * 3 + [alpha], 1))
            rays_block(out, "", regions, build_volume_bvh(regions, tf), rng, 30, "pruned")
            out["rays_pruned_tf"] = tf.rgba
            out["rays_pruned_domain"] = np.array([lo, hi])
        np.savez_compressed(OUT / f"model_{name}.npz", **out)
        print(f"{name}: cells={len(cells)} bricks={model.n_bricks} regions={len(regions)} t={time.time()-t0:.1f}s", flush=True)

    # ---- transfer-function fixtures ------------------------------------------------
    out = {}
    rng = np.random.default_rng(5)
    tfs, ranges, mo = [], [], []
    for t in range(12):
        alpha = rng.uniform(0.0, 1.0, 256)
        if t % 3 == 0:
            alpha[rng.integers(0, 256, 100)] = 0.0
        if t % 4 == 1:
            alpha[:200] = 0.0
        rgba = np.stack([rng.uniform(0, 1, 256) for _ in range(3)] + [alpha], 1)
        dom = (float(rng.uniform(-2, 0)), float(rng.uniform(0.5, 3)))
        tf = TransferFunction(dom, rgba)
        rr = np.sort(rng.uniform(dom[0] - 1, dom[1] + 1, (200, 2)), axis=1)
        rr[:20, 1] = rr[:20, 0]  # degenerate ranges
        vals = [max_opacity(tf, r) for r in rr]
        tfs.append(rgba)
        ranges.append(rr)
        mo.append(vals)
        out[f"tf{t}_domain"] = np.array(dom)
    out["tf_rgba"] = np.array(tfs)
    out["tf_ranges"] = np.array(ranges)
    out["tf_max_opacity"] = np.array(mo)
    # TransferFunction.sample and pixel_rho known answers
    samp_tf = TransferFunction((out["tf0_domain"][0], out["tf0_domain"][1]), tfs[0])
    sv = rng.uniform(-3, 4, 300)
    out["tf_sample_values"] = sv
    out["tf_sample_out"] = np.array([samp_tf.sample(v) for v in sv])
    pix = np.concatenate([np.arange(64), rng.integers(0, 2**31, 64), np.array([2**40 + 3, 2**63 - 1])]).astype(np.uint64)
    seeds = [0, 9, 42, 2**63 + 5]
    out["rho_pixels"] = pix
    out["rho_seeds"] = np.array(seeds, np.uint64)
    out["rho_values"] = np.array([[R.pixel_rho(int(p), int(s)) for p in pix] for s in seeds])
    np.savez_compressed(OUT / "tf_rho.npz", **out)

    # ---- frame fixtures ------------------------------------------------------------
    out = {}
    frames_meta = {}
    cells, model, tree, regions, _ = built["smoke"]
    lo, hi = model.value_range(0)
    gray = TransferFunction.grayscale((lo, hi))
    scene = R.build_scene(model, regions, gray)
    cam = orbit_cameras(regions.bounds, 1, 96, 72)[0]
    for mode in ("none", "analytic", "central", "clampedCentral"):
        frames_meta[f"smoke_{mode}"] = store_frame(out, f"smoke_{mode}", scene, cam, gray, R.MarchParams(seed=9, gradient_mode=mode))
    # dead band (space-skipping test TF)
    vmin, vmax = regions.value_range[:, 0, 0].min(), regions.value_range[:, 0, 1].max()
    rgba = np.tile(np.linspace(0.0, 1.0, 256)[:, None], (1, 4))
    rgba[:128, 3] = 0.0
    band = TransferFunction((vmin, vmax), rgba)
    sb = R.build_scene(model, regions, band)
    frames_meta["smoke_band"] = store_frame(out, "smoke_band", sb, cam, band, R.MarchParams(seed=9))
    # clip planes + other orbit view + rate
    cam2 = orbit_cameras(regions.bounds, 5, 80, 60)[2]
    frames_meta["smoke_clip"] = store_frame(
        out, "smoke_clip", scene, cam2, gray,
        R.MarchParams(seed=3, rate_scale=1.7, gradient_mode="analytic", clip_planes=[((1.0, 0.2, 0.0), 20.0), ((0.0, -1.0, 0.0), -3.0)]),
    )
    # opaque TF
    opaque = TransferFunction((lo, hi), np.ones((256, 4)))
    so = R.build_scene(model, regions, opaque)
    frames_meta["smoke_opaque"] = store_frame(out, "smoke_opaque", so, cam, opaque, R.MarchParams(gradient_mode="none"))
    # iso + volume on smoke (iso 0.5 of range), analytic shading, low early threshold
    iso_v = float(lo + 0.45 * (hi - lo))
    gray05 = TransferFunction.grayscale((lo, hi), max_alpha=0.5)
    si = R.build_scene(model, regions, gray05, iso_value=iso_v)
    frames_meta["smoke_iso"] = store_frame(out, "smoke_iso", si, cam, gray05, R.MarchParams(seed=1, early_term_threshold=0.9), iso=iso_v)

    # ramp: surface-only iso and volume-in-front-of-iso
    cells, model, tree, regions, _ = built["ramp"]
    lo, hi = model.value_range(0)
    white0 = np.ones((256, 4))
    white0[:, 3] = 0.0
    surf = TransferFunction((lo, hi), white0)
    sr = R.build_scene(model, regions, surf, iso_value=7.25)
    camr = R.Camera([-10.0, 8.0, 8.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], 40.0, 32, 32)
    frames_meta["ramp_iso"] = store_frame(out, "ramp_iso", sr, camr, surf, R.MarchParams(), iso=7.25)
    w12 = np.ones((256, 4))
    w12[:, 3] = 0.12
    vol = TransferFunction((lo, hi), w12)
    sv_ = R.build_scene(model, regions, vol, iso_value=7.25)
    camr2 = R.Camera([-10.0, 8.0, 8.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], 40.0, 16, 16)
    frames_meta["ramp_voliso"] = store_frame(out, "ramp_voliso", sv_, camr2, vol, R.MarchParams(), iso=7.25)

    # c1 at 128x128 (grayscale, analytic and none) — BASELINE configs[0] shape
    cells, model, tree, regions, _ = built["c1"]
    lo, hi = model.value_range(0)
    g1 = TransferFunction.grayscale((lo, hi))
    s1 = R.build_scene(model, regions, g1)
    cam1 = orbit_cameras(regions.bounds, 1, 128, 128)[0]
    frames_meta["c1_analytic"] = store_frame(out, "c1_analytic", s1, cam1, g1, R.MarchParams(seed=0, gradient_mode="analytic"))
    frames_meta["c1_none"] = store_frame(out, "c1_none", s1, cam1, g1, R.MarchParams(seed=0, gradient_mode="none"))
    # gauss_aniso half-alpha analytic, 2nd orbit view
    cells, model, tree, regions, _ = built["gauss_aniso"]
    lo, hi = model.value_range(0)
    ga = TransferFunction.grayscale((lo, hi), max_alpha=0.5)
    sa = R.build_scene(model, regions, ga)
    cama = orbit_cameras(regions.bounds, 3, 72, 40)[1]
    frames_meta["aniso_analytic"] = store_frame(out, "aniso_analytic", sa, cama, ga, R.MarchParams(seed=123456789, gradient_mode="analytic"))
    np.savez_compressed(OUT / "frames.npz", **out)

    # ---- single-ray integration (two-cell scene) -------------------------------------
    out = {}
    cl = cells_of([0, 1], [0, 0], [0, 0], [0, 0], [4.0, 4.0])
    ray_cases = []
    for width in (32, 1):
        m, _ = build_bricks(cl, BrickBuildParams(max_brick_width=width))
        rg = build_regions(m)
        a03 = np.ones((256, 4))
        a03[:, 3] = 0.3
        tf = TransferFunction((3.0, 5.0), a03)
        sc = R.build_scene(m, rg, tf)
        for rate in (0.5, 1.0, 2.7):
            params = R.MarchParams(rate_scale=rate, gradient_mode="none", early_term_threshold=1.0)
            rgba, st = R.integrate_ray((-3.0, 0.5, 0.5), (1.0, 0.0, 0.0), sc, tf, params)
            ray_cases.append((width, rate, *rgba, st["regions"], st["samples"]))
    out["two_cell_rays"] = np.array(ray_cases)
    np.savez_compressed(OUT / "rays.npz", **out)

    with open(OUT / "digests.json", "w") as fh:
        json.dump({"models": digests, "frames": frames_meta}, fh, indent=1, sort_keys=True)
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    sys.setrecursionlimit(100000)
    main()
