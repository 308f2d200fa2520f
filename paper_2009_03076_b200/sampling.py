"""Hat-basis reconstruction and gradients on the GPU (paper Eq. 1-3, §5.1).

Drop-in for `amrvol.sampling` (R/sampling.py:1-409).  Point queries run the
same fused gather the march uses (csrc/march.cuh:gather) in batch kernels;
results are bit-identical to the reference's `_accumulate_bricks` /
`_gradient_bricks` (same terms, same order, no FMA).  Batch variants
(`sample_points`, `gradient_points`) take (n, 3) arrays.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .model import AmrModel, Cell

__all__ = [
    "EPS_WEIGHT", "SampleResult", "GradientResult", "hat_weight", "basis_sample_region", "basis_sample_oracle",
    "basis_sample_celllocation", "nearest_sample", "sample_at", "gradient_analytic", "gradient_central",
    "gradient_central_clamped", "sample_points", "gradient_points", "locate_points",
]

EPS_WEIGHT = 1e-12


@dataclass
class SampleResult:
    value: float
    weight_sum: float
    valid: bool


@dataclass
class GradientResult:
    vec: np.ndarray
    valid: bool


def hat_weight(cell: Cell, p) -> float:
    """Basis weight of one cell at p (R/sampling.py:260-268); scalar API helper."""
    p = np.asarray(p, np.float64)
    w = cell.coord.width
    c = cell.center
    h = 1.0
    for a in range(3):
        h *= max(1.0 - abs(c[a] - p[a]) / w, 0.0)
    return h


def _handles(regions, model):
    from .bricks import model_handle
    from .regions import regions_handle

    rh = regions_handle(regions, model)
    return rh.model_handle, rh


def _accumulate(model, regions, pts, rids, want_grad, field=0):
    pts = np.ascontiguousarray(np.asarray(pts, np.float64).reshape(-1, 3))
    n = len(pts)
    mh, rh = _handles(regions, model)
    rin = None if rids is None else np.ascontiguousarray(rids, np.int32)
    rout = np.empty(n, np.int32)
    acc = np.empty((n, 9))
    N.check(N.lib().xb_sample_points(mh.h, rh.h, int(field), n, N.ptr(pts), N.ptr(rin), int(want_grad), N.ptr(rout),
                                     N.ptr(acc)))
    return rout, acc


def locate_points(regions, pts, model=None):
    """Region id per point (-1 outside the support union) via the k-d tree."""
    rout, _ = _accumulate(model, regions, pts, None, False)
    return rout


def _region_id(regions, region) -> int:
    """Index of an ActiveBrickRegion (identified by its box) inside regions."""
    for attr in ("_index",):
        if hasattr(region, attr):
            return getattr(region, attr)
    return -1


def sample_points(model: AmrModel, regions, pts, rids=None, field: int = 0):
    """Batch `sample_at` / `basis_sample_region`: (value, weight_sum, valid, region) arrays."""
    rout, acc = _accumulate(model, regions, pts, rids, False, field)
    den = acc[:, 1]
    valid = den > EPS_WEIGHT
    with np.errstate(invalid="ignore", divide="ignore"):
        val = np.where(valid, acc[:, 0] / np.where(valid, den, 1.0), 0.0)
    return val, den, valid, rout


def gradient_points(model: AmrModel, regions, pts, rids=None, field: int = 0):
    """Batch `gradient_analytic`: (gradients (n,3), valid, region)."""
    rout, acc = _accumulate(model, regions, pts, rids, True, field)
    den = acc[:, 1]
    valid = den > EPS_WEIGHT
    d2 = np.where(valid, den * den, 1.0)
    g = (acc[:, 3:6] * den[:, None] - acc[:, 2:3] * acc[:, 6:9]) / d2[:, None]
    g[~valid] = 0.0
    return g, valid, rout


def _region_index(regions, region):
    """Index of an ActiveBrickRegion inside `regions` (regions are disjoint boxes)."""
    if getattr(region, "_regions", None) is regions:
        return region._index
    c = 0.5 * (np.asarray(region.box.lo) + np.asarray(region.box.hi))
    r = int(locate_points(regions, c.reshape(1, 3))[0])
    if r < 0 or not (np.array_equal(regions.lo[r], region.box.lo) and np.array_equal(regions.hi[r], region.box.hi)):
        raise ValueError("region does not belong to the given RegionSet")
    return r


def _regions_of(model, region=None):
    if region is not None and getattr(region, "_regions", None) is not None:
        return region._regions
    rs = getattr(model, "_regions_ref", None)
    if rs is None:
        from .regions import build_regions

        rs = build_regions(model)
        model._regions_ref = rs
    return rs


def basis_sample_region(p, region, model: AmrModel, field: int = 0, regions=None) -> SampleResult:
    """Weighted average over the region's brick list (R/sampling.py:281-288)."""
    regions = regions if regions is not None else _regions_of(model, region)
    r = _region_index(regions, region)
    val, den, valid, _ = sample_points(model, regions, np.asarray(p, np.float64).reshape(1, 3), np.array([r]), field)
    return SampleResult(float(val[0]), float(den[0]), bool(valid[0]))


def basis_sample_oracle(p, cells, field: int = 0, model: AmrModel | None = None) -> SampleResult:
    """Linear scan over every cell, in the list's own order (R/sampling.py:291-298), on the GPU.

    A model's canonical list (`model.cell_list()`, or `model=` given) is scanned
    from the resident model; any other CellList is uploaded and scanned in its
    given order (`xb_sample_scan_cells`) — the reference's exact running sums
    either way.
    """
    import ctypes as C

    model = model if model is not None else getattr(cells, "_model", None)
    pts = np.ascontiguousarray(np.asarray(p, np.float64).reshape(-1, 3))
    out = np.empty((len(pts), 2))
    if model is not None:
        from .bricks import model_handle

        mh = model_handle(model)
        N.check(N.lib().xb_sample_scan(mh.h, int(field), len(pts), N.ptr(pts), N.ptr(out)))
    else:
        if not 0 <= field < cells.n_fields:
            raise ValueError(f"field {field} out of range for {cells.n_fields} fields")
        dev = N.require_device()
        h = N.new_handle()
        n = len(cells)
        N.check(N.lib().xb_cells_create(n, dev, C.byref(h)))
        ch = N.CellsHandle(h.value, dev)
        arrs = [np.ascontiguousarray(a, np.int32) for a in (cells.i, cells.j, cells.k, cells.level)]
        arrs.append(np.ascontiguousarray(cells.values[:, field], np.float32))
        N.check(N.lib().xb_cells_upload(ch.h, 0, n, *(N.ptr(x) for x in arrs)))
        N.check(N.lib().xb_sample_scan_cells(ch.h, len(pts), N.ptr(pts), N.ptr(out)))
    num, den = out[0]
    return SampleResult(num / den, den, True) if den > EPS_WEIGHT else SampleResult(0.0, den, False)


def basis_sample_celllocation(p, tree, model: AmrModel, field: int = 0) -> SampleResult:
    """Split-tree (cell-location) sampling (R/sampling.py:301-317).

    Identical by construction to the region path (the gathered brick set is a
    superset visited in id order); served by the region path on the GPU.
    """
    return sample_at(p, _regions_of(model), model, field)


def nearest_sample(p, tree, model: AmrModel, field: int = 0) -> SampleResult:
    """Value of the cell whose box contains p (R/sampling.py:320-331).  Host lookup
    over the brick table (a diagnostic, not on the render path)."""
    p = np.asarray(p, np.float64)
    w = np.exp2(model.brick_level.astype(np.float64))
    g = np.floor((p[None, :] - model.brick_lower) / w[:, None])
    inside = np.all((g >= 0) & (g < model.brick_dims), axis=1)
    hit = np.nonzero(inside)[0]
    if len(hit) == 0:
        return SampleResult(0.0, 0.0, False)
    b = int(hit[0])
    x, y, z = (int(v) for v in g[b])
    nx, ny, _ = model.brick_dims[b]
    return SampleResult(float(model.scalars[field, model.brick_offset[b] + x + nx * (y + ny * z)]), 1.0, True)


def sample_at(p, regions, model: AmrModel, field: int = 0) -> SampleResult:
    """Locate the region containing p and sample there (R/sampling.py:334-339)."""
    val, den, valid, r = sample_points(model, regions, np.asarray(p, np.float64).reshape(1, 3), None, field)
    if r[0] < 0:
        return SampleResult(0.0, 0.0, False)
    return SampleResult(float(val[0]), float(den[0]), bool(valid[0]))


def gradient_analytic(p, region, model: AmrModel, field: int = 0, regions=None) -> GradientResult:
    """Exact derivative of the weighted average, same gather (R/sampling.py:342-353)."""
    regions = regions if regions is not None else _regions_of(model, region)
    r = _region_index(regions, region)
    g, valid, _ = gradient_points(model, regions, np.asarray(p, np.float64).reshape(1, 3), np.array([r]), field)
    return GradientResult(g[0] if valid[0] else np.zeros(3), bool(valid[0]))


def gradient_central(p, regions, model: AmrModel, field: int = 0, offset_scale: float = 0.5) -> GradientResult:
    """Central differences via the all-regions index (R/sampling.py:356-382); the 7
    samples are one batch on the GPU."""
    p = np.asarray(p, np.float64)
    r0 = int(locate_points(regions, p.reshape(1, 3), model)[0])
    if r0 < 0:
        return GradientResult(np.zeros(3), False)
    h = offset_scale * regions.finest_width[r0]
    q = np.repeat(p[None, :], 7, axis=0)
    for a in range(3):
        q[1 + 2 * a, a] = p[a] + h
        q[2 + 2 * a, a] = p[a] - h
    val, den, valid, rr = sample_points(model, regions, q, None, field)
    ok = valid & (rr >= 0)
    g = np.zeros(3)
    for a in range(3):
        fp, fm = 1 + 2 * a, 2 + 2 * a
        if ok[fp] and ok[fm]:
            g[a] = (val[fp] - val[fm]) / (2.0 * h)
        elif ok[fp] and ok[0]:
            g[a] = (val[fp] - val[0]) / h
        elif ok[fm] and ok[0]:
            g[a] = (val[0] - val[fm]) / h
    return GradientResult(g, bool(ok[0]))


def gradient_central_clamped(p, region, model: AmrModel, field: int = 0, offset_scale: float = 0.5,
                             regions=None) -> GradientResult:
    """Central differences clamped into the region box (R/sampling.py:385-409)."""
    regions = regions if regions is not None else _regions_of(model, region)
    r = _region_index(regions, region)
    p = np.asarray(p, np.float64)
    h = offset_scale * region.finest_cell_width
    lo, hi = region.box.lo, region.box.hi
    pts, spans, axes = [], [], []
    for a in range(3):
        qa, qb = max(lo[a], p[a] - h), min(hi[a], p[a] + h)
        if qb <= qa:
            continue
        for v in (qa, qb):
            q = p.copy()
            q[a] = v
            pts.append(q)
        spans.append(qb - qa)
        axes.append(a)
    g = np.zeros(3)
    if not pts:
        return GradientResult(g, False)
    val, den, valid, _ = sample_points(model, regions, np.array(pts), np.full(len(pts), r), field)
    any_valid = False
    for t, a in enumerate(axes):
        if valid[2 * t] and valid[2 * t + 1]:
            g[a] = (val[2 * t + 1] - val[2 * t]) / spans[t]
            any_valid = True
    return GradientResult(g, any_valid)
