"""Transfer functions and region space skipping (paper §3.3, §4.1, §5.2).

Drop-in for `amrvol.accel` (R/accel.py:1-424).  The reference keeps two
median-split BVHs over the *active* regions and restarts a closest-hit query
from the root for every region a ray enters.  On the B200 the active set is a
per-region flag computed by one kernel (exact FP64 `max_opacity`), folded
bottom-up into the k-d tree of the region build; the march walks that tree
front to back (csrc/march.cuh).  `RegionBvh` is the handle of such an active
set; `next_region` / `iterate_intervals` / `point_query` answer exactly what
the reference's BVH queries answer (tests/test_gpu_parity.py).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N

__all__ = [
    "TransferFunction", "RegionBvh", "RayInterval", "max_opacity", "build_volume_bvh", "build_iso_bvh",
    "build_all_regions_bvh", "next_region", "point_query", "iterate_intervals", "restart_epsilon", "RAMP_SIZE",
]

RAMP_SIZE = 256


class TransferFunction:
    """256-entry piecewise-linear RGBA ramp over a value domain (R/accel.py:38-88)."""

    def __init__(self, domain, rgba):
        lo, hi = float(domain[0]), float(domain[1])
        if not lo < hi:
            raise ValueError(f"transfer function domain must satisfy lo < hi, got {domain}")
        rgba = np.asarray(rgba, np.float64)
        if rgba.shape != (RAMP_SIZE, 4):
            raise ValueError(f"ramp must have shape (256, 4), got {rgba.shape}")
        if rgba.min() < 0.0 or rgba.max() > 1.0:
            raise ValueError("ramp channels must lie in [0, 1]")
        self.domain = (lo, hi)
        self.rgba = np.ascontiguousarray(rgba)

    def sample(self, value: float) -> np.ndarray:
        lo, hi = self.domain
        t = min(max((float(value) - lo) / (hi - lo), 0.0), 1.0)
        x = t * (RAMP_SIZE - 1)
        i = int(x)
        if i >= RAMP_SIZE - 1:
            return self.rgba[RAMP_SIZE - 1].copy()
        f = x - i
        return (1.0 - f) * self.rgba[i] + f * self.rgba[i + 1]

    def max_opacity(self, vmin: float, vmax: float) -> float:
        return max_opacity(self, (vmin, vmax))

    @staticmethod
    def grayscale(domain, max_alpha: float = 1.0) -> "TransferFunction":
        ramp = np.linspace(0.0, 1.0, RAMP_SIZE)
        return TransferFunction(domain, np.stack([ramp, ramp, ramp, max_alpha * ramp], axis=1))

    @staticmethod
    def constant_alpha(domain, alpha: float, color=(1.0, 1.0, 1.0)) -> "TransferFunction":
        rgba = np.empty((RAMP_SIZE, 4))
        rgba[:, 0], rgba[:, 1], rgba[:, 2] = color
        rgba[:, 3] = alpha
        return TransferFunction(domain, rgba)

    def to_dict(self) -> dict:
        return {"domain": list(self.domain), "rgba": self.rgba.tolist()}

    @staticmethod
    def from_dict(d: dict) -> "TransferFunction":
        return TransferFunction(d["domain"], d["rgba"])


def max_opacity(tf: TransferFunction, value_range) -> float:
    """Exact max alpha of the ramp over [vmin, vmax] (R/accel.py:91-115).

    Scalar helper of the public API; the per-region bulk evaluation used for
    space skipping runs on the GPU (csrc/accel.cu:max_opacity_dev) with the
    identical FP64 expression.
    """
    vmin, vmax = float(value_range[0]), float(value_range[1])
    if vmin > vmax:
        raise ValueError("value range must satisfy min <= max")
    lo, hi = tf.domain
    scale = (RAMP_SIZE - 1) / (hi - lo)
    x0 = min(max((vmin - lo) * scale, 0.0), RAMP_SIZE - 1.0)
    x1 = min(max((vmax - lo) * scale, 0.0), RAMP_SIZE - 1.0)
    alpha = tf.rgba[:, 3]

    def at(x):
        i = int(x)
        if i >= RAMP_SIZE - 1:
            return float(alpha[RAMP_SIZE - 1])
        f = x - i
        return float((1.0 - f) * alpha[i] + f * alpha[i + 1])

    m = max(at(x0), at(x1))
    k0, k1 = int(np.ceil(x0)), int(np.floor(x1))
    if k0 <= k1:
        m = max(m, float(alpha[k0:k1 + 1].max()))
    return m


@dataclass
class RayInterval:
    t_in: float
    t_out: float
    region: int


class RegionBvh:
    """Active region set on the GPU — the B200 form of the reference's RegionBvh
    (R/accel.py:125-155): a per-region active flag + per-k-d-node subtree flags
    for the frame kernel, and an LBVH (Morton sort + Karras build, csrc/lbvh.cu)
    whose node arrays carry the reference's names (`node_lo`, `node_hi`,
    `node_left`, `node_right`, `node_start`, `node_count`, `leaf_prims`,
    `kernel_args()`); topology differs from the reference's median split, which
    the queries' results do not depend on.

    `prims` lists the active region ids (ascending); `build_ms` is the device
    build time (reported as `bvhRebuildMs` on edits, R/render.py:119-132).
    """

    def __init__(self, regions, handle, kind):
        self.regions = regions
        self._h = handle
        self.kind = kind
        L = N.lib()
        na, ms = C.c_int64(), C.c_double()
        N.check(L.xb_active_info(handle.h, C.byref(na), C.byref(ms)))
        self._n_active = na.value
        self.build_ms = ms.value
        self._prims = None
        self._mask = None

    @property
    def handle(self):
        return self._h

    @property
    def n_active(self) -> int:
        return self._n_active

    @property
    def is_empty(self) -> bool:
        return self._n_active == 0

    @property
    def prims(self) -> np.ndarray:
        if self._prims is None:
            p = np.empty(self._n_active, np.int32)
            N.check(N.lib().xb_active_prims(self._h.h, N.ptr(p)))
            self._prims = p
        return self._prims

    def _lbvh(self):
        if getattr(self, "_nodes", None) is None:
            L = N.lib()
            nn, depth, ms = C.c_int64(), C.c_int32(), C.c_double()
            N.check(L.xb_active_lbvh_info(self._h.h, C.byref(nn), C.byref(depth), C.byref(ms)))
            n = nn.value
            lo, hi = np.empty((n, 3)), np.empty((n, 3))
            left, right = np.empty(n, np.int32), np.empty(n, np.int32)
            start, count = np.empty(n, np.int64), np.empty(n, np.int32)
            prims = np.empty(max(self._n_active, 1), np.int32)
            N.check(L.xb_active_lbvh_download(self._h.h, N.ptr(lo), N.ptr(hi), N.ptr(left), N.ptr(right),
                                              N.ptr(start), N.ptr(count), N.ptr(prims)))
            self._nodes = (lo, hi, left, right, start, count, prims[: self._n_active])
            self.lbvh_depth = depth.value
            self.lbvh_build_ms = ms.value
        return self._nodes

    node_lo = property(lambda self: self._lbvh()[0])
    node_hi = property(lambda self: self._lbvh()[1])
    node_left = property(lambda self: self._lbvh()[2])
    node_right = property(lambda self: self._lbvh()[3])
    node_start = property(lambda self: self._lbvh()[4])
    node_count = property(lambda self: self._lbvh()[5])
    leaf_prims = property(lambda self: self._lbvh()[6])

    def kernel_args(self):
        """The reference's argument tuple (R/accel.py:150-155), LBVH leaf order."""
        lo, hi, left, right, start, count, prims = self._lbvh()
        return lo, hi, left, right, start, count, prims, self.regions.lo, self.regions.hi

    @property
    def active_mask(self) -> np.ndarray:
        if self._mask is None:
            m = np.zeros(len(self.regions), bool)
            m[self.prims] = True
            self._mask = m
        return self._mask


def _rh(regions, model=None):
    from .regions import regions_handle

    return regions_handle(regions, model)


def _make(regions, fn, kind, *args, model=None):
    rh = _rh(regions, model)
    h = N.new_handle()
    t0 = time.perf_counter()
    N.check(fn(rh.h, *args, C.byref(h)))
    bvh = RegionBvh(regions, N.ActiveHandle(h.value, rh.device, rh), kind)
    bvh.build_ms = (time.perf_counter() - t0) * 1000.0
    return bvh


def build_volume_bvh(regions, tf: TransferFunction, field: int = 0, model=None) -> RegionBvh:
    """Regions with strictly positive max opacity under tf (R/accel.py:227-234)."""
    rgba = np.ascontiguousarray(tf.rgba, np.float64)
    return _make(regions, N.lib().xb_active_volume, "volume", int(field), tf.domain[0], tf.domain[1], N.ptr(rgba),
                 model=model)


def build_iso_bvh(regions, iso_value: float, field: int = 0, model=None) -> RegionBvh:
    """Regions whose value range brackets the iso value (R/accel.py:237-241)."""
    return _make(regions, N.lib().xb_active_iso, "iso", int(field), float(iso_value), model=model)


def build_all_regions_bvh(regions, model=None) -> RegionBvh:
    """Every region: the point-lookup index / unpruned structure (R/accel.py:244-247)."""
    return _make(regions, N.lib().xb_active_all, "all", model=model)


def restart_epsilon(t_out: float) -> float:
    """R/accel.py:391-393."""
    return max(1e-7, 1e-7 * t_out)


def trace_rays(bvh: RegionBvh, origins, directions, t_start: float, t_max: float, cap: int = 256,
               traversal: str = "kd"):
    """Batch `iterate_intervals` on the GPU: list of [(t_in, t_out, region), ...] per ray.

    traversal "kd": the ordered k-d walk (one walk per ray); "lbvh": one LBVH
    closest-hit query per region visit, the reference's own scheme."""
    if traversal not in ("kd", "lbvh"):
        raise ValueError(f"unknown traversal {traversal!r}")
    o = np.ascontiguousarray(np.asarray(origins, np.float64).reshape(-1, 3))
    d = np.ascontiguousarray(np.asarray(directions, np.float64).reshape(-1, 3))
    n = len(o)
    rh = bvh.handle.regions_handle
    L = N.lib()
    while True:
        tin, tout = np.empty((n, cap)), np.empty((n, cap))
        reg = np.empty((n, cap), np.int32)
        cnt = np.empty(n, np.int32)
        fn = L.xb_trace_intervals if traversal == "kd" else L.xb_trace_intervals_lbvh
        N.check(fn(rh.model_handle.h, rh.h, bvh.handle.h, n, N.ptr(o), N.ptr(d), float(t_start), float(t_max), cap,
                   N.ptr(tin), N.ptr(tout), N.ptr(reg), N.ptr(cnt)))
        if n == 0 or cnt.max() <= cap:
            break
        cap = int(cnt.max())
    return [[(float(tin[q, k]), float(tout[q, k]), int(reg[q, k])) for k in range(cnt[q])] for q in range(n)]


def next_region(bvh: RegionBvh, origin, direction, t_start: float, t_max: float) -> Optional[RayInterval]:
    """Closest active region with entry >= t_start, clipped to [t_start, t_max] (R/accel.py:396-405):
    one LBVH closest-hit query."""
    got = trace_rays(bvh, origin, direction, t_start, t_max, cap=1, traversal="lbvh")[0]
    if not got:
        return None
    return RayInterval(*got[0])


def point_query(bvh: RegionBvh, p) -> Optional[int]:
    """Active region whose half-open box contains p (R/accel.py:408-411): LBVH point query."""
    r = int(point_query_batch(bvh, np.asarray(p, np.float64).reshape(1, 3))[0])
    return None if r < 0 else r


def point_query_batch(bvh: RegionBvh, points) -> np.ndarray:
    """`point_query` for (n, 3) points on the GPU; -1 where no active region holds the point."""
    p = np.ascontiguousarray(np.asarray(points, np.float64).reshape(-1, 3))
    out = np.empty(len(p), np.int32)
    rh = bvh.handle.regions_handle
    N.check(N.lib().xb_point_query_lbvh(rh.model_handle.h, rh.h, bvh.handle.h, len(p), N.ptr(p), N.ptr(out)))
    return out


def iterate_intervals(bvh: RegionBvh, origin, direction, t_start: float, t_max: float):
    """Successive disjoint ascending RayIntervals along the ray (R/accel.py:414-424)."""
    for t_in, t_out, r in trace_rays(bvh, origin, direction, t_start, t_max)[0]:
        yield RayInterval(t_in, t_out, r)
