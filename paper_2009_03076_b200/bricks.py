"""Cell list -> same-level bricks on the GPU (paper §3.1.2).

Drop-in for `amrvol.bricks` (R/bricks.py:1-254).  `build_bricks` runs the
level-synchronous k-d split of `csrc/build_bricks.cu` and returns the exact
arrays of the reference builder (np.array_equal on every AmrModel / SplitTree
array).  The device copy of the model stays attached to the returned
AmrModel, so `build_regions` and rendering never re-upload it.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .model import AmrModel, CellList, CellValidationReport, _as_cell_list, validate_cells

__all__ = ["BrickBuildParams", "SplitTree", "InvalidCellsError", "build_bricks", "BrickStats", "brick_stats"]


@dataclass
class BrickBuildParams:
    """R/bricks.py:27-34."""

    max_brick_width: int = 32
    keep_split_tree: bool = False

    def __post_init__(self):
        if self.max_brick_width < 1:
            raise ValueError("max_brick_width must be >= 1")


class InvalidCellsError(ValueError):
    """Build input fails validation; carries the full report (R/bricks.py:37-42)."""

    def __init__(self, report: CellValidationReport):
        super().__init__(report.summary())
        self.report = report


@dataclass
class SplitTree:
    """Flattened k-d split tree of the brick build, preorder (R/bricks.py:45-68)."""

    axis: np.ndarray
    pos: np.ndarray
    left: np.ndarray
    right: np.ndarray
    brick_start: np.ndarray
    brick_count: np.ndarray
    box_lo: np.ndarray
    box_hi: np.ndarray
    max_half: np.ndarray

    @property
    def n_nodes(self) -> int:
        return len(self.axis)


def _empty_tree() -> SplitTree:
    z32, zf = np.zeros(0, np.int32), np.zeros(0, np.float64)
    return SplitTree(z32, zf, z32, z32, z32, z32, zf, zf, zf)  # _TreeBuilder().done() shapes


def build_bricks(cells, params: BrickBuildParams | None = None):
    """Partition validated cells into bricks on the GPU.

    Returns (AmrModel, SplitTree or None), deterministic for any input
    permutation (cells are canonically ordered by (level, k, j, i) first).
    """
    params = params or BrickBuildParams()
    from .io import DeviceCells

    if isinstance(cells, DeviceCells):  # GPU-resident cells (generate_synthetic_device)
        L = N.lib()
        h = N.new_handle()
        N.check(L.xb_build_bricks_cells(cells.handle.h, int(min(params.max_brick_width, 2**31 - 1)),
                                        int(params.keep_split_tree), C.byref(h)))
        mh = N.ModelHandle(h.value, cells.handle.device)
        model = model_from_handle(mh, cells.field_names)
        tree = None
        if params.keep_split_tree:
            tree = tree_from_handle(mh) if len(cells) else _empty_tree()
        return model, tree
    cl = _as_cell_list(cells)
    names = cl.field_names
    dev = N.require_device()
    L = N.lib()
    h = N.new_handle()
    n = len(cl)
    vals = np.ascontiguousarray(cl.values, np.float32)
    rc = L.xb_build_bricks(N.ptr(cl.i), N.ptr(cl.j), N.ptr(cl.k), N.ptr(cl.level), N.ptr(vals), n, cl.n_fields,
                           int(min(params.max_brick_width, 2**31 - 1)), int(params.keep_split_tree), dev, C.byref(h))
    if rc == N.XB_ERR_INVALID_CELLS:
        report = validate_cells(cl)
        if report.ok:  # the device check is stricter only in range limits
            raise N.NativeError(rc, "cells rejected by the device validator")
        raise InvalidCellsError(report)
    N.check(rc)
    mh = N.ModelHandle(h.value, dev)
    model = model_from_handle(mh, names)
    tree = None
    if params.keep_split_tree:
        tree = tree_from_handle(mh) if n else _empty_tree()
    return model, tree


def model_from_handle(mh, names) -> AmrModel:
    L = N.lib()
    nb, nc, nf, nt = C.c_int64(), C.c_int64(), C.c_int32(), C.c_int64()
    N.check(L.xb_model_info(mh.h, C.byref(nb), C.byref(nc), C.byref(nf), C.byref(nt)))
    B, NC, F = nb.value, nc.value, nf.value
    lower = np.empty((B, 3), np.int32)
    level = np.empty(B, np.int32)
    dims = np.empty((B, 3), np.int32)
    off = np.empty(B + 1, np.int64)
    sc = np.empty((F, NC), np.float32)
    N.check(L.xb_model_download(mh.h, N.ptr(lower), N.ptr(level), N.ptr(dims), N.ptr(off), N.ptr(sc)))
    model = AmrModel(names, lower, level, dims, sc)
    model._device[mh.device] = mh
    return model


def tree_from_handle(mh) -> SplitTree:
    L = N.lib()
    nt = C.c_int64()
    N.check(L.xb_model_info(mh.h, None, None, None, C.byref(nt)))
    T = nt.value
    a = {k: np.empty(T, np.int32) for k in ("axis", "left", "right", "brick_start", "brick_count")}
    pos, mh_ = np.empty(T), np.empty(T)
    lo, hi = np.empty((T, 3)), np.empty((T, 3))
    N.check(L.xb_model_download_tree(mh.h, N.ptr(a["axis"]), N.ptr(pos), N.ptr(a["left"]), N.ptr(a["right"]),
                                     N.ptr(a["brick_start"]), N.ptr(a["brick_count"]), N.ptr(lo), N.ptr(hi), N.ptr(mh_)))
    return SplitTree(a["axis"], pos, a["left"], a["right"], a["brick_start"], a["brick_count"], lo, hi, mh_)


def model_handle(model: AmrModel, dev=None):
    """Device copy of an AmrModel (uploaded once per device, then cached)."""
    dev = N.require_device(dev)
    mh = model._device.get(dev)
    if mh is None:
        h = N.new_handle()
        N.check(N.lib().xb_model_upload(N.ptr(model.brick_lower), N.ptr(model.brick_level), N.ptr(model.brick_dims),
                                        N.ptr(model.scalars), model.n_bricks, model.n_cells, model.n_fields, dev,
                                        C.byref(h)))
        mh = N.ModelHandle(h.value, dev)
        model._device[dev] = mh
    return mh


@dataclass
class BrickStats:
    n_cells: int
    n_bricks: int
    cells_per_level: dict = field(default_factory=dict)
    bricks_per_level: dict = field(default_factory=dict)
    min_dim: int = 0
    max_dim: int = 0
    mean_dim: float = 0.0


def brick_stats(model: AmrModel) -> BrickStats:
    """R/bricks.py:242-254."""
    st = BrickStats(n_cells=model.n_cells, n_bricks=model.n_bricks)
    if model.n_bricks == 0:
        return st
    counts = model.brick_dims.prod(axis=1, dtype=np.int64)
    for lev in np.unique(model.brick_level):
        m = model.brick_level == lev
        st.bricks_per_level[int(lev)] = int(m.sum())
        st.cells_per_level[int(lev)] = int(counts[m].sum())
    st.min_dim = int(model.brick_dims.min())
    st.max_dim = int(model.brick_dims.max())
    st.mean_dim = float(model.brick_dims.mean())
    return st
