"""ctypes binding of libexabricks.so (include/exabricks.h).

The product path: every compute call of the package goes through here into
the sm_100a kernels.  There is no CPU fallback — a missing library or CUDA
device raises `NativeUnavailable`.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["XB_LIB"]) if os.environ.get("XB_LIB") else _PKG / "libexabricks.so"  # XB_LIB: A/B builds

XB_OK = 0
XB_ERR_INVALID_CELLS = -3
XB_ERR_NO_TREE = -5

P = C.c_void_p
i32, i64, f64, u64 = C.c_int32, C.c_int64, C.c_double, C.c_uint64


class NativeUnavailable(RuntimeError):
    """libexabricks.so or a CUDA device is missing (no CPU fallback exists)."""


class NativeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libexabricks error {code}: {msg}")
        self.code = code


class XbCamera(C.Structure):
    _fields_ = [("width", i32), ("height", i32), ("position", f64 * 3), ("right", f64 * 3), ("up", f64 * 3),
                ("forward", f64 * 3), ("tan_half", f64), ("aspect", f64)]


class XbMarch(C.Structure):
    _fields_ = [("samples_per_cell", f64), ("rate_scale", f64), ("early_term_threshold", f64), ("seed", u64),
                ("gradient_mode", i32), ("n_planes", i32), ("planes", (f64 * 4) * 6), ("iso_on", i32),
                ("iso_value", f64), ("iso_rgb", f64 * 3), ("tf_lo", f64), ("tf_hi", f64), ("tf_rgba", f64 * 1024),
                ("use_tree", i32)]


class XbSynthSpec(C.Structure):
    _fields_ = [("field", i32), ("max_level", i32), ("extent", i64 * 3), ("threshold", f64), ("n_holes", i32),
                ("n_refine", i32), ("holes", (f64 * 4) * 32), ("refine", (f64 * 4) * 32), ("center", f64 * 3),
                ("sigma", f64), ("amp", f64), ("direction", f64 * 3), ("offset", f64), ("constant", f64),
                ("n_waves", i32), ("waves", (f64 * 5) * 8)]


class XbTuning(C.Structure):
    """xb_tuning (include/exabricks.h): frame-pipeline variants for A/B runs and the parity matrix."""

    _fields_ = [("kernel", i32), ("traversal", i32), ("walk_lists", i32), ("leaf_cap", i32), ("walk_cap1", i32),
                ("short_rays", i32), ("walk2_min", i64), ("fuse_short", i32), ("time_march", i32),
                ("short_leaves", i32), ("short_samples", i32), ("grab_div", i32), ("grab_fixed", i32)]


# exported symbol -> (restype, argtypes); tests check every declared symbol
SIGNATURES = {
    "xb_last_error": (C.c_char_p, []),
    "xb_abi_version": (C.c_int, []),
    "xb_device_count": (C.c_int, [P]),
    "xb_generate_synthetic": (C.c_int, [P, i32, P]),
    "xb_cells_info": (C.c_int, [P, P]),
    "xb_cells_download": (C.c_int, [P, P, P, P, P, P]),
    "xb_cells_free": (None, [P]),
    "xb_cells_create": (C.c_int, [i64, i32, P]),
    "xb_cells_upload": (C.c_int, [P, i64, i64, P, P, P, P, P]),
    "xb_build_bricks_cells": (C.c_int, [P, i32, i32, P]),
    "xb_build_bricks": (C.c_int, [P, P, P, P, P, i64, i32, i32, i32, i32, P]),
    "xb_model_upload": (C.c_int, [P, P, P, P, i64, i64, i32, i32, P]),
    "xb_model_info": (C.c_int, [P, P, P, P, P]),
    "xb_model_download": (C.c_int, [P, P, P, P, P, P]),
    "xb_model_download_tree": (C.c_int, [P, P, P, P, P, P, P, P, P, P]),
    "xb_model_upload_tree": (C.c_int, [P, i64, P, P, P, P, P, P, P, P, P]),
    "xb_model_free": (None, [P]),
    "xb_build_regions": (C.c_int, [P, P]),
    "xb_regions_info": (C.c_int, [P, P, P, P, P]),
    "xb_regions_download": (C.c_int, [P, P, P, P, P, P, P]),
    "xb_regions_free": (None, [P]),
    "xb_active_volume": (C.c_int, [P, i32, f64, f64, P, P]),
    "xb_active_iso": (C.c_int, [P, i32, f64, P]),
    "xb_active_all": (C.c_int, [P, P]),
    "xb_active_info": (C.c_int, [P, P, P]),
    "xb_active_prims": (C.c_int, [P, P]),
    "xb_active_free": (None, [P]),
    "xb_render": (C.c_int, [P, P, i32, P, P, P, P, i32, i32, P, P, P, P, i32, P]),
    "xb_tuning_defaults": (None, [P]),
    "xb_tuning_get": (C.c_int, [P]),
    "xb_tuning_set": (C.c_int, [P]),
    "xb_march_times": (C.c_int, [P, i32, P]),
    "xb_tile_count": (C.c_int, [i32, i32, i32, i32, P, P]),
    "xb_unpack_tiles": (C.c_int, [P, i64, i32, i32, i32, P, P]),
    "xb_integrate_rays": (C.c_int, [P, P, i32, P, P, i64, P, P, P, P, P, P, P]),
    "xb_iso_rays": (C.c_int, [P, P, i32, P, P, i64, P, P, P, P, P, P, P]),
    "xb_sample_points": (C.c_int, [P, P, i32, i64, P, P, i32, P, P]),
    "xb_sample_scan": (C.c_int, [P, i32, i64, P, P]),
    "xb_sample_scan_cells": (C.c_int, [P, i64, P, P]),
    "xb_trace_intervals": (C.c_int, [P, P, P, i64, P, P, f64, f64, i32, P, P, P, P]),
    "xb_active_lbvh_info": (C.c_int, [P, P, P, P]),
    "xb_active_lbvh_download": (C.c_int, [P, P, P, P, P, P, P, P]),
    "xb_trace_intervals_lbvh": (C.c_int, [P, P, P, i64, P, P, f64, f64, i32, P, P, P, P]),
    "xb_point_query_lbvh": (C.c_int, [P, P, P, i64, P, P]),
}

_lock = threading.Lock()
_lib = None


def load_library(path=None):
    """dlopen libexabricks.so (no CUDA context is created by loading)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise NativeUnavailable(f"{p} not built; run __graft_entry__.build() (nvcc, sm_100a)")
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("XB_LIB") and not hasattr(lib, name):
                continue  # an older A/B build (tools/ab.py): bind what it has
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def lib():
    return load_library()


def check(rc):
    if rc != XB_OK:
        msg = lib().xb_last_error()
        raise NativeError(rc, msg.decode() if msg else "")


class tuning:
    """Context manager selecting frame-pipeline variants (xb_tuning_set), e.g.
    `with tuning(kernel=1): ...`; restores the previous setting on exit.  The
    setting is process-wide: the library's defaults are the production path."""

    def __init__(self, **fields):
        self.fields = fields
        self.prev = None

    def __enter__(self):
        self.prev = XbTuning()
        check(lib().xb_tuning_get(C.byref(self.prev)))
        t = XbTuning()
        lib().xb_tuning_defaults(C.byref(t))
        for k, v in self.fields.items():
            if not hasattr(t, k):
                raise ValueError(f"unknown tuning field {k!r}")
            setattr(t, k, int(v))
        check(lib().xb_tuning_set(C.byref(t)))
        return t

    def __exit__(self, *exc):
        check(lib().xb_tuning_set(C.byref(self.prev)))


_dev_ok = {}


def device_index():
    """CUDA device for new native objects: LOCAL_RANK under torchrun, else
    torch's current device if torch is already imported, else 0."""
    import sys

    if "torch" in sys.modules:
        torch = sys.modules["torch"]
        try:
            if torch.cuda.is_available():
                return torch.cuda.current_device()
        except Exception:
            pass
    return int(os.environ.get("XB_DEVICE", "0"))


def require_device(dev=None):
    dev = device_index() if dev is None else dev
    if dev not in _dev_ok:
        n = C.c_int32(0)
        rc = lib().xb_device_count(C.byref(n))
        if rc != XB_OK or n.value <= dev:
            raise NativeUnavailable(f"no CUDA device {dev} for libexabricks (found {n.value}); no CPU fallback exists")
        _dev_ok[dev] = True
    return dev


def ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(P)
    return C.c_void_p(int(a))


class Handle:
    """Owns one native object; freed with the matching xb_*_free."""

    _free = None

    def __init__(self, h, device):
        self.h = h
        self.device = device

    def __del__(self):
        h = getattr(self, "h", None)
        if h and self._free and _lib is not None:
            getattr(_lib, self._free)(h)
            self.h = None


class CellsHandle(Handle):
    _free = "xb_cells_free"


class ModelHandle(Handle):
    _free = "xb_model_free"


class RegionsHandle(Handle):
    _free = "xb_regions_free"

    def __init__(self, h, device, model_handle):
        super().__init__(h, device)
        self.model_handle = model_handle  # keep the model alive while regions live


class ActiveHandle(Handle):
    _free = "xb_active_free"

    def __init__(self, h, device, regions_handle):
        super().__init__(h, device)
        self.regions_handle = regions_handle


def new_handle():
    return C.c_void_p()
