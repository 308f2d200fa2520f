"""Active Brick Regions built on the GPU (paper §3.2).

Drop-in for `amrvol.regions` (R/regions.py:1-244).  `build_regions` runs the
level-synchronous ABR k-d split + metadata kernels of
`csrc/build_regions.cu`; the returned RegionSet holds exactly the reference
arrays (lo/hi f64, brick_off i64, brick_ids i32, value_range (R,F,2) f64,
finest_width f64) and keeps the device copy — region records, brick-id lists
and the k-d tree the march walks — attached.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .model import AmrModel, Box3

__all__ = ["ActiveBrickRegion", "RegionSet", "build_regions", "point_to_region", "RegionStats", "region_stats"]


@dataclass
class ActiveBrickRegion:
    """R/regions.py:27-32."""

    box: Box3
    brick_ids: np.ndarray
    value_range: np.ndarray
    finest_cell_width: float


class RegionSet:
    """Columnar regions; behaves like a sequence of ActiveBrickRegion (R/regions.py:35-79)."""

    def __init__(self, lo, hi, brick_off, brick_ids, value_range, finest_width, field_names):
        self.lo = np.ascontiguousarray(lo, np.float64).reshape(-1, 3)
        self.hi = np.ascontiguousarray(hi, np.float64).reshape(-1, 3)
        self.brick_off = np.ascontiguousarray(brick_off, np.int64)
        self.brick_ids = np.ascontiguousarray(brick_ids, np.int32)
        self.value_range = np.ascontiguousarray(value_range, np.float64)
        self.finest_width = np.ascontiguousarray(finest_width, np.float64)
        self.field_names = tuple(field_names)
        self._native = {}        # device -> RegionsHandle
        self._point_index = None

    def __len__(self) -> int:
        return len(self.finest_width)

    def __getitem__(self, r: int) -> ActiveBrickRegion:
        s, e = self.brick_off[r], self.brick_off[r + 1]
        reg = ActiveBrickRegion(Box3(self.lo[r], self.hi[r]), self.brick_ids[s:e], self.value_range[r],
                                float(self.finest_width[r]))
        reg._index, reg._regions = int(r), self  # device lookups address the region by id
        return reg

    def region_bricks(self, r: int) -> np.ndarray:
        return self.brick_ids[self.brick_off[r]:self.brick_off[r + 1]]

    def volumes(self) -> np.ndarray:
        return np.prod(self.hi - self.lo, axis=1)

    @property
    def bounds(self) -> Box3:
        if len(self) == 0:
            return Box3.empty()
        return Box3(self.lo.min(axis=0), self.hi.max(axis=0))

    @property
    def point_index(self):
        """All-regions index for point lookup (R/regions.py:72-79).

        On the GPU this is the k-d tree of the region build itself; the
        object returned is the all-regions active set over it.
        """
        if self._point_index is None:
            from .accel import build_all_regions_bvh

            self._point_index = build_all_regions_bvh(self)
        return self._point_index


def build_regions(model: AmrModel) -> RegionSet:
    """Recursive top-down partition of the brick-support union (R/regions.py:90-171), on the GPU."""
    from .bricks import model_handle

    mh = model_handle(model)
    h = N.new_handle()
    N.check(N.lib().xb_build_regions(mh.h, C.byref(h)))
    rh = N.RegionsHandle(h.value, mh.device, mh)
    regions = regions_from_handle(rh, model.field_names)
    regions._model_ref = model
    return regions


def regions_from_handle(rh, names) -> RegionSet:
    L = N.lib()
    nr, ni, nk, dep = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
    N.check(L.xb_regions_info(rh.h, C.byref(nr), C.byref(ni), C.byref(nk), C.byref(dep)))
    R, I, F = nr.value, ni.value, len(names)
    lo, hi = np.empty((R, 3)), np.empty((R, 3))
    off = np.empty(R + 1, np.int64)
    ids = np.empty(I, np.int32)
    vr = np.empty((R, F, 2))
    fw = np.empty(R)
    N.check(L.xb_regions_download(rh.h, N.ptr(lo), N.ptr(hi), N.ptr(off), N.ptr(ids), N.ptr(vr), N.ptr(fw)))
    rs = RegionSet(lo, hi, off, ids, vr, fw, names)
    rs._native[rh.device] = rh
    return rs


_ARRAYS = ("lo", "hi", "brick_off", "brick_ids", "value_range", "finest_width")


def regions_handle(regions: RegionSet, model: AmrModel | None = None, dev=None):
    """Device copy (with k-d tree) of a RegionSet.

    A RegionSet that did not come from `build_regions` (e.g. `load_artifact`)
    is re-derived on the GPU from its model — the build is deterministic and
    bit-exact — and accepted only if every array matches.
    """
    dev = N.require_device(dev)
    rh = regions._native.get(dev)
    if rh is not None:
        return rh
    model = model if model is not None else getattr(regions, "_model_ref", None)
    if model is None:
        raise N.NativeError(N.XB_ERR_NO_TREE, "RegionSet has no device copy; pass the AmrModel it was built from")
    from .bricks import model_handle

    mh = model_handle(model, dev)
    h = N.new_handle()
    N.check(N.lib().xb_build_regions(mh.h, C.byref(h)))
    rh = N.RegionsHandle(h.value, dev, mh)
    again = regions_from_handle(rh, regions.field_names)
    for a in _ARRAYS:
        if not np.array_equal(getattr(again, a), getattr(regions, a)):
            raise N.NativeError(N.XB_ERR_NO_TREE, f"RegionSet.{a} differs from build_regions(model); "
                                                  "only build_regions output can be rendered on the GPU")
    regions._native[dev] = rh
    regions._model_ref = model
    return rh


def point_to_region(regions: RegionSet, p):
    """Region whose half-open box [lo, hi) contains p, else None (R/regions.py:216-220)."""
    from .accel import point_query

    return point_query(regions.point_index, p)


@dataclass
class RegionStats:
    n_regions: int
    bricks_per_region_by_count: float
    bricks_per_region_by_volume: float
    max_bricks_per_region: int
    total_volume: float


def region_stats(regions: RegionSet) -> RegionStats:
    """R/regions.py:232-244."""
    n = len(regions)
    if n == 0:
        return RegionStats(0, 0.0, 0.0, 0, 0.0)
    counts = np.diff(regions.brick_off)
    vols = regions.volumes()
    return RegionStats(n_regions=n, bricks_per_region_by_count=float(counts.mean()),
                       bricks_per_region_by_volume=float((counts * vols).sum() / vols.sum()),
                       max_bricks_per_region=int(counts.max()), total_volume=float(vols.sum()))
