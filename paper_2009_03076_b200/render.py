"""Frame rendering on the B200 (paper §4, §5.2).

Drop-in for `amrvol.render` (R/render.py:1-691).  `render_frame` keeps the
reference signature and returns the same `Frame` (RGBA8, premultiplied) and
`FrameStats`; the per-pixel work is one fused sm_100a kernel
(csrc/render.cu:k_render) reached through `xb_render`.  Small scalar helpers
of the public API (`make_intervals`, `opacity_correct`, `shade`,
`pixel_rho`) are plain Python, as in the reference.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field as dc_field
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .accel import RegionBvh, TransferFunction, build_iso_bvh, build_volume_bvh
from .bricks import SplitTree
from .model import AmrModel
from .regions import RegionSet

__all__ = [
    "Camera", "MarchParams", "FrameStats", "Frame", "Scene", "build_scene", "make_intervals", "opacity_correct",
    "shade", "pixel_rho", "integrate_ray", "iso_intersect", "render_frame", "render_frames", "render_frame_float",
    "GRADIENT_MODES",
    "ISO_COLOR",
]

GRADIENT_MODES = {"none": 0, "analytic": 1, "central": 2, "clampedCentral": 3}
ISO_COLOR = (0.83, 0.83, 0.86)
_T_FAR = 1.0e30
_MASK64 = (1 << 64) - 1


@dataclass
class Camera:
    """Pinhole camera (R/render.py:52-89)."""

    position: np.ndarray
    forward: np.ndarray
    up: np.ndarray
    fov_y: float = 40.0
    width: int = 512
    height: int = 512

    def __post_init__(self):
        self.position = np.asarray(self.position, np.float64)
        self.forward = np.asarray(self.forward, np.float64)
        self.up = np.asarray(self.up, np.float64)
        if not 0.0 < self.fov_y < 180.0:
            raise ValueError(f"vertical fov must be in (0, 180), got {self.fov_y}")
        f = self.forward / np.linalg.norm(self.forward)
        if np.linalg.norm(np.cross(f, self.up)) < 1e-12:
            raise ValueError("forward and up are parallel")

    def basis(self):
        """Orthonormal (right, true-up, forward) frame."""
        f = self.forward / np.linalg.norm(self.forward)
        r = np.cross(f, self.up)
        r /= np.linalg.norm(r)
        u = np.cross(r, f)
        return r, u, f

    def ray(self, x: int, y: int):
        r, u, f = self.basis()
        th = math.tan(math.radians(self.fov_y) * 0.5)
        aspect = self.width / self.height
        sx = (2.0 * (x + 0.5) / self.width - 1.0) * th * aspect
        sy = (1.0 - 2.0 * (y + 0.5) / self.height) * th
        d = f + sx * r + sy * u
        return self.position.copy(), d / np.linalg.norm(d)


@dataclass
class MarchParams:
    """R/render.py:92-116."""

    samples_per_cell: float = 2.0
    rate_scale: float = 1.0
    early_term_threshold: float = 0.98
    seed: int = 0
    gradient_mode: str = "analytic"
    clip_planes: Sequence = ()

    def __post_init__(self):
        if self.samples_per_cell <= 0:
            raise ValueError("samples_per_cell must be positive")
        if not 0.0 < self.early_term_threshold <= 1.0:
            raise ValueError("early_term_threshold must be in (0, 1]")
        if self.gradient_mode not in GRADIENT_MODES:
            raise ValueError(f"unknown gradient mode {self.gradient_mode!r}")
        if len(self.clip_planes) > 6:
            raise ValueError("at most 6 clip planes are supported")

    def plane_array(self) -> np.ndarray:
        out = np.zeros((len(self.clip_planes), 4))
        for i, (n, c) in enumerate(self.clip_planes):
            out[i, :3] = np.asarray(n, np.float64)
            out[i, 3] = float(c)
        return out


@dataclass
class FrameStats:
    ms: float
    regions: int
    samples: int
    bvh_rebuild_ms: float = 0.0

    def to_dict(self) -> dict:
        return {"ms": self.ms, "regions": self.regions, "samples": self.samples, "bvhRebuildMs": self.bvh_rebuild_ms}


@dataclass
class Frame:
    width: int
    height: int
    rgba: np.ndarray  # (height, width, 4) uint8, premultiplied
    stats: FrameStats


@dataclass
class Scene:
    """Immutable render inputs (R/render.py:143-157); device copies hang off model/regions."""

    model: AmrModel
    regions: RegionSet
    volume_bvh: RegionBvh
    field: int = 0
    iso_bvh: Optional[RegionBvh] = None
    iso_value: Optional[float] = None
    tree: Optional[SplitTree] = None
    field_values: np.ndarray = dc_field(init=False)

    def __post_init__(self):
        self.field_values = np.ascontiguousarray(self.model.scalars[self.field])


def build_scene(model: AmrModel, regions: RegionSet, tf: TransferFunction, field: int = 0,
                iso_value: Optional[float] = None, tree: Optional[SplitTree] = None) -> Scene:
    """R/render.py:160-163 — active sets built on the GPU."""
    vb = build_volume_bvh(regions, tf, field, model=model)
    ib = build_iso_bvh(regions, iso_value, field, model=model) if iso_value is not None else None
    return Scene(model, regions, vb, field, ib, iso_value, tree)


# ---------------------------------------------------------------------------
# scalar helpers of the public API (R/render.py:170-219)


def make_intervals(t_in: float, t_out: float, dt: float, rho: float):
    if not t_in < t_out:
        raise ValueError("require t_in < t_out")
    if dt <= 0.0:
        raise ValueError("require dt > 0")
    out = []
    prev = t_in
    k = math.floor(t_in / dt - rho) + 1
    while True:
        tk = dt * (k + rho)
        if tk >= t_out:
            break
        if tk > prev:
            out.append((prev, tk))
            prev = tk
        k += 1
    out.append((prev, t_out))
    return out


def opacity_correct(alpha: float, s: float, s1: float) -> float:
    return 1.0 - (1.0 - alpha) ** (s / s1)


def shade(color, gradient, ray_dir):
    color = np.asarray(color, np.float64)
    g = np.asarray(gradient, np.float64)
    d = np.asarray(ray_dir, np.float64)
    n = np.linalg.norm(g)
    if n == 0.0:
        return 0.2 * color
    d = d / np.linalg.norm(d)
    return color * (0.2 + 0.8 * abs(float(g @ d)) / n)


def pixel_rho(pixel: int, seed: int) -> float:
    """splitmix64 lattice offset in [0, 1) (R/render.py:212-219; device: march.cuh:rho_hash)."""
    z = (pixel ^ seed) & _MASK64
    z = (z + 0x9E3779B97F4A7C15) & _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    z = z ^ (z >> 31)
    return (z >> 11) * (1.0 / 9007199254740992.0)


# ---------------------------------------------------------------------------
# native argument blocks


_CAM_CACHE: dict = {}


def camera_struct(camera: Camera) -> N.XbCamera:
    """XbCamera of `camera`; cached on its fields (the numpy basis costs 30-70 us
    per frame, more than the host side of the rest of the call)."""
    key = (camera.position.tobytes(), camera.forward.tobytes(), camera.up.tobytes(), float(camera.fov_y),
           int(camera.width), int(camera.height))
    c = _CAM_CACHE.get(key)
    if c is None:
        if len(_CAM_CACHE) > 256:
            _CAM_CACHE.clear()
        c = _CAM_CACHE[key] = _camera_struct(camera)
    return c


def _camera_struct(camera: Camera) -> N.XbCamera:
    r, u, f = camera.basis()
    c = N.XbCamera()
    c.width, c.height = int(camera.width), int(camera.height)
    for a in range(3):
        c.position[a] = float(camera.position[a])
        c.right[a], c.up[a], c.forward[a] = float(r[a]), float(u[a]), float(f[a])
    c.tan_half = math.tan(math.radians(camera.fov_y) * 0.5)
    c.aspect = camera.width / camera.height
    return c


def march_struct(tf: TransferFunction, params: MarchParams, iso_value=None, use_tree=False) -> N.XbMarch:
    m = N.XbMarch()
    m.use_tree = int(bool(use_tree))
    m.samples_per_cell = float(params.samples_per_cell)
    m.rate_scale = float(params.rate_scale)
    m.early_term_threshold = float(params.early_term_threshold)
    m.seed = int(params.seed) & _MASK64
    m.gradient_mode = GRADIENT_MODES[params.gradient_mode]
    planes = params.plane_array()
    m.n_planes = len(planes)
    for i in range(len(planes)):
        for c in range(4):
            m.planes[i][c] = float(planes[i, c])
    m.iso_on = int(iso_value is not None)
    m.iso_value = float(iso_value) if iso_value is not None else 0.0
    for c in range(3):
        m.iso_rgb[c] = ISO_COLOR[c]
    m.tf_lo, m.tf_hi = float(tf.domain[0]), float(tf.domain[1])
    C.memmove(C.addressof(m.tf_rgba), np.ascontiguousarray(tf.rgba, np.float64).ctypes.data, 1024 * 8)
    return m


def _scene_handles(scene: Scene):
    from .regions import regions_handle

    rh = regions_handle(scene.regions, scene.model)
    vb = scene.volume_bvh
    if vb.handle.regions_handle is not rh:
        raise ValueError("scene.volume_bvh was built for a different RegionSet")
    iso_on = scene.iso_bvh is not None and scene.iso_value is not None
    ib = scene.iso_bvh.handle if iso_on else None
    return rh.model_handle, rh, vb.handle, ib, iso_on


def _ensure_device_tree(scene: Scene, mh) -> None:
    """The model handle carries the split tree for the cell-location gather;
    attach the scene's SplitTree when the handle was built without one."""
    nb, nc, nf, nt = C.c_int64(), C.c_int64(), C.c_int32(), C.c_int64()
    N.check(N.lib().xb_model_info(mh.h, C.byref(nb), C.byref(nc), C.byref(nf), C.byref(nt)))
    if nt.value > 0:
        return
    t = scene.tree
    arr = lambda a, dt: np.ascontiguousarray(a, dt)  # noqa: E731
    keep = [arr(t.axis, np.int32), arr(t.pos, np.float64), arr(t.left, np.int32), arr(t.right, np.int32),
            arr(t.brick_start, np.int32), arr(t.brick_count, np.int32), arr(t.box_lo, np.float64),
            arr(t.box_hi, np.float64), arr(t.max_half, np.float64)]
    N.check(N.lib().xb_model_upload_tree(mh.h, len(keep[0]), *(N.ptr(a) for a in keep)))


def render_native(scene: Scene, camera: Camera, tf: TransferFunction, params: MarchParams, out8, outf=None,
                  counts=None, tile_rank=0, tile_world=1, count_bytes=False, stream=None, sync=True,
                  use_celllocation=False, dev_stats=None):
    """One `xb_render` call; outputs may be numpy arrays or device pointers (ints).

    Returns [regions, samples, algorithmic bytes].  With sync=False and device
    outputs the call only enqueues work on `stream` (no host synchronisation)
    and returns None; `dev_stats` (device pointer to 3 int64) then receives the
    counters on the stream."""
    if camera.width < 1 or camera.height < 1:
        raise ValueError("image must be at least 1x1 pixel")
    mh, rh, vh, ih, iso_on = _scene_handles(scene)
    if use_celllocation:
        if scene.tree is None:
            raise ValueError("cell-location sampling requires a scene built with the split tree")
        _ensure_device_tree(scene, mh)
    cam = camera_struct(camera)
    m = march_struct(tf, params, scene.iso_value if iso_on else None, use_tree=use_celllocation)
    stats = np.zeros(3, np.int64) if (sync or count_bytes) and dev_stats is None else None
    N.check(N.lib().xb_render(mh.h, rh.h, int(scene.field), vh.h, ih.h if ih else None, C.byref(cam), C.byref(m),
                              int(tile_rank), int(tile_world), N.ptr(out8), N.ptr(outf), N.ptr(counts),
                              N.ptr(stats) if dev_stats is None else C.c_void_p(int(dev_stats)),
                              int(bool(count_bytes)), C.c_void_p(stream) if stream else None))
    return stats


def _host_image(height: int, width: int) -> np.ndarray:
    """Frame output array.  With torch present it is page-locked memory from
    torch's caching host allocator (the D2H copy runs at full link speed and the
    block returns to the cache when the array is freed); plain numpy otherwise."""
    try:
        import torch

        if torch.cuda.is_available():
            return torch.empty((height, width, 4), dtype=torch.uint8, pin_memory=True).numpy()
    except Exception:  # pragma: no cover - torch missing or without CUDA
        pass
    return np.empty((height, width, 4), np.uint8)


def render_frame(scene: Scene, camera: Camera, tf: TransferFunction, params: MarchParams,
                 use_celllocation: bool = False) -> Frame:
    """Render a full frame on the GPU (R/render.py:654-691).

    `use_celllocation` selects the reference's per-sample split-tree lookup
    (R/render.py:423-425, `_collect_bricks` R/sampling.py:184-224) — the paper's
    cell-location baseline, run by the one-thread-per-pixel kernel; its frames
    are pixel-identical to the region path by construction (R/render.py:657-659).
    """
    if camera.width < 1 or camera.height < 1:
        raise ValueError("image must be at least 1x1 pixel")
    if use_celllocation and scene.tree is None:
        raise ValueError("cell-location sampling requires a scene built with the split tree")
    t0 = time.perf_counter()
    out = _host_image(camera.height, camera.width)
    stats = render_native(scene, camera, tf, params, out, use_celllocation=use_celllocation)
    ms = (time.perf_counter() - t0) * 1000.0
    return Frame(camera.width, camera.height, out, FrameStats(ms, int(stats[0]), int(stats[1])))


def render_frames(scene: Scene, cameras, tf: TransferFunction, params: MarchParams):
    """Render a sequence of frames (an orbit, an animation) with the host copy
    of frame k overlapping the march of frame k+1; yields one `Frame` per camera,
    in order, each with its host RGBA8 (page-locked) and `FrameStats` (`ms` =
    the frame's GPU time from CUDA events; the frames are pixel-identical to
    `render_frame`).  Two device images alternate: the march runs on one
    stream, the device-to-host copies on another, joined by events."""
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    s_march, s_copy = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    slots = []  # (device image, device stats, copy-done event)
    pending = []  # frames in flight: (camera, host image, host stats, march start/end events, copy event)
    k = 0
    for cam in cameras:
        if cam.width < 1 or cam.height < 1:
            raise ValueError("image must be at least 1x1 pixel")
        if len(slots) < 2:
            slots.append([torch.empty((cam.height, cam.width, 4), dtype=torch.uint8, device=dev),
                          torch.zeros(3, dtype=torch.int64, device=dev), None])
        img, st, done = slots[k % 2]
        if img.shape != (cam.height, cam.width, 4):
            img = slots[k % 2][0] = torch.empty((cam.height, cam.width, 4), dtype=torch.uint8, device=dev)
        if done is not None:
            s_march.wait_event(done)  # this slot's previous copy has left the device
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s_march)
        render_native(scene, cam, tf, params, img.data_ptr(), stream=s_march.cuda_stream, sync=False,
                      dev_stats=st.data_ptr())
        b.record(s_march)
        host = torch.empty((cam.height, cam.width, 4), dtype=torch.uint8, pin_memory=True)
        hst = torch.empty(3, dtype=torch.int64, pin_memory=True)
        s_copy.wait_event(b)
        with torch.cuda.stream(s_copy):
            host.copy_(img, non_blocking=True)
            hst.copy_(st, non_blocking=True)
        c = torch.cuda.Event()
        c.record(s_copy)
        slots[k % 2][2] = c
        pending.append((cam, host, hst, a, b, c))
        k += 1
        if len(pending) == 2:  # frame k-1 is ready once its copy is
            yield _finish_pending(pending.pop(0))
    while pending:
        yield _finish_pending(pending.pop(0))


def _finish_pending(p):
    cam, host, hst, a, b, c = p
    c.synchronize()
    st = hst.numpy()
    return Frame(cam.width, cam.height, host.numpy(), FrameStats(a.elapsed_time(b), int(st[0]), int(st[1])))


def render_frame_float(scene: Scene, camera: Camera, tf: TransferFunction, params: MarchParams, count_bytes=False,
                       use_celllocation=False):
    """Parity variant: (RGBA8, float64 RGBA before quantisation, per-pixel (regions, samples), stats)."""
    H, W = camera.height, camera.width
    out = np.empty((H, W, 4), np.uint8)
    outf = np.empty((H, W, 4), np.float64)
    cnt = np.empty((H, W, 2), np.int32)
    stats = render_native(scene, camera, tf, params, out, outf, cnt, count_bytes=count_bytes,
                          use_celllocation=use_celllocation)
    return out, outf, cnt, stats


def _ray_batch(scene, fn, bvh_handle, tf, params, origins, directions, t0, t1, rhos, iso_value=None):
    from .regions import regions_handle

    rh = regions_handle(scene.regions, scene.model)
    o = np.ascontiguousarray(np.asarray(origins, np.float64).reshape(-1, 3))
    d = np.ascontiguousarray(np.asarray(directions, np.float64).reshape(-1, 3))
    n = len(o)
    t0 = np.ascontiguousarray(np.broadcast_to(np.asarray(t0, np.float64), (n,)))
    t1 = np.ascontiguousarray(np.broadcast_to(np.asarray(t1, np.float64), (n,)))
    rho = np.ascontiguousarray(np.broadcast_to(np.asarray(rhos, np.float64), (n,)))
    m = march_struct(tf, params, iso_value)
    out = np.empty((n, 4))
    return rh, o, d, t0, t1, rho, m, out, n


def integrate_ray(origin, direction, scene: Scene, tf: TransferFunction, params: MarchParams, pixel: int = 0,
                  t_range=(0.0, _T_FAR)):
    """Volume-integrate one ray on the GPU; (rgba float64[4], stats) (R/render.py:613-632)."""
    dn = np.asarray(direction, np.float64)
    dn = dn / np.linalg.norm(dn)
    rh, o, d, t0, t1, rho, m, out, n = _ray_batch(scene, None, None, tf, params, origin, dn, t_range[0], t_range[1],
                                                  pixel_rho(pixel, params.seed))
    counts = np.empty((n, 2), np.int64)
    N.check(N.lib().xb_integrate_rays(rh.model_handle.h, rh.h, int(scene.field), scene.volume_bvh.handle.h,
                                      C.byref(m), n, N.ptr(o), N.ptr(d), N.ptr(t0), N.ptr(t1), N.ptr(rho), N.ptr(out),
                                      N.ptr(counts)))
    return out[0].copy(), {"regions": int(counts[0, 0]), "samples": int(counts[0, 1])}


def iso_intersect(origin, direction, iso_bvh: RegionBvh, scene: Scene, iso_value: float, t_range=(0.0, _T_FAR),
                  params: Optional[MarchParams] = None, pixel: int = 0):
    """First iso crossing along the ray on the GPU, or None (R/render.py:635-651)."""
    params = params or MarchParams()
    dn = np.asarray(direction, np.float64)
    dn = dn / np.linalg.norm(dn)
    tf = TransferFunction((0.0, 1.0), np.zeros((256, 4)))
    rh, o, d, t0, t1, rho, m, out, n = _ray_batch(scene, None, None, tf, params, origin, dn, t_range[0], t_range[1],
                                                  pixel_rho(pixel, params.seed), iso_value)
    hit = np.empty(n, np.int32)
    N.check(N.lib().xb_iso_rays(rh.model_handle.h, rh.h, int(scene.field), iso_bvh.handle.h, C.byref(m), n, N.ptr(o),
                                N.ptr(d), N.ptr(t0), N.ptr(t1), N.ptr(rho), N.ptr(out), N.ptr(hit)))
    if not hit[0]:
        return None
    return float(out[0, 0]), out[0, 1:4].copy()
