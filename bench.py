#!/usr/bin/env python
"""bench.py — ExaBricks render hot path on B200 (one JSON line on rank 0).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c3]
                  [--secondary c2] [--extra c4,c5] [--views 8]

Workload (N=1): BASELINE.json configs[2], the configuration the metric ("at
1920x1080") is quoted on — a synthetic Landing-Gear-shaped AMR volume (13
levels, 4096:1, 266M cells, SURVEY.md §8(d) "C3"), DVR + analytic-gradient
shading, grayscale TF (max alpha 0.5), 1920x1080, seed 0, over the reference
bench's 8-view orbit (R/bench.py:30-62: step k renders view k mod 8, the value
is the orbit mean).  Cells come from the numpy generator (bit-exact
restatement of the reference's generate_synthetic, R/io.py:247-295) on all
host cores.  A step is one frame: ray march of every pixel through the
resident scene (+ the NCCL tile gather and counter all-reduce for N>1).
Inputs are resident in HBM; L2 (126 MB) is flushed by a 256 MB write between
timed frames.  Metric: frames/s (whole job) with Msamples/s beside it
(`FrameStats.samples` / s, R/render.py:419).  configs[1] (C2) is timed in the
same run ("secondary"), configs[3] (C4: iso + TF-edit refresh) and configs[4]
(C5, Exajet-shaped, 647M cells) under "extra"; "ablations" times the
reference's traversal (per-visit LBVH queries) and the cell-location baseline
(paper Table 3) against the default path at C2.

Parity is checked in the same run: the GPU builders' arrays against the C
oracle's sha256 digests at this scale (tests/golden/scale_digests.json, made
by tools/make_scale_digests.py), and the GPU float frame against the oracle's
render of the CPU-baseline row bands (max |dRGBA| <= 1e-3, per-pixel region
and sample counters equal).  A violation prints the line and exits 1.

`--impl reference` runs the reference algorithm on the host only (no GPU, no
libexabricks): numpy generator, the C oracle's builders (oracle/xb_oracle.c,
a restatement of R/bricks.py + R/regions.py pinned to the reference's golden
arrays) and the oracle renderer (R/render.py restated, OpenMP on every host
thread) on full frames of the same orbit.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frames/sec and Msamples/sec at 1920×1080 (1/2/4/8 B200), % HBM roofline"
RGBA_TOL = 1e-3  # north_star: images within max |dRGBA| <= 1e-3

CONFIGS = {
    # SURVEY.md §8(d) C1 / C2 (BASELINE.json configs[0] / configs[1])
    "c1": dict(spec=dict(field="gaussian", extent=(64, 64, 64), max_level=1, threshold=0.04, seed=0),
               res=(256, 256), max_alpha=1.0, gradient="analytic",
               workload="configs[0]: synthetic 2-level gaussian AMR, 97,840 cells, 256x256 DVR + analytic shading"),
    "c2": dict(spec=dict(field="gaussian", extent=(256, 256, 256), max_level=3, threshold=0.004, seed=0),
               res=(1024, 1024), max_alpha=0.5, gradient="analytic",
               workload="configs[1]: synthetic 4-level gaussian AMR (2x ratio), 9,534,568 cells, "
                        "1024x1024 DVR + analytic gradient shading, 1 GPU"),
    # Landing-Gear-shaped, 12 refinement steps (4096:1), hole + level-0 shell,
    # 266,139,607 cells (R_h 200, R_r 420)
    "c3": dict(spec=dict(field="gaussian", extent=(16384, 8192, 8192), max_level=12, threshold=0.05, seed=0,
                         holes=((6144.0, 6144.0, 6144.0, 200.0),), refine_spheres=((6144.0, 6144.0, 6144.0, 420.0),),
                         field_params={"center": (6144.0, 6144.0, 6144.0), "sigma": 600.0}),
               res=(1920, 1080), max_alpha=0.5, gradient="analytic",
               workload="configs[2]: synthetic Landing-Gear-shaped AMR (13 levels, 4096:1 cell ratio, 266M cells), "
                        "1920x1080 DVR + analytic gradient shading"),
    # C4: C3 + implicit iso-surface (0.5) + DVR, and a timed TF-edit majorant refresh
    "c4": dict(spec="c3", res=(1920, 1080), max_alpha=0.5, gradient="analytic", iso=0.5,
               workload="configs[3]: Landing-Gear-shaped AMR (266M cells), implicit iso-surface 0.5 + DVR, "
                        "1920x1080, with a TF-edit active-set/majorant refresh"),
    # C5: Exajet-shaped, 4 levels, hole/refine chain along x (SURVEY.md §8(d) template), 647M cells
    "c5": dict(spec="jet", res=(1920, 1080), max_alpha=0.5, gradient="analytic",
               workload="configs[4]: synthetic Exajet-shaped AMR (4 levels, 647M cells), 1920x1080 DVR + analytic shading"),
}
JET = dict(thr=0.003, rh=80.0, rr=300.0, step=80.0, sigma=400.0)  # 647,115,612 cells (tools/calib.py)
MODEL_KEYS = ("brick_lower", "brick_level", "brick_dims", "brick_offset", "scalars")
REGION_KEYS = ("lo", "hi", "brick_off", "brick_ids", "value_range", "finest_width")


def spec_for(cfg):
    from paper_2009_03076_b200 import io as xio

    sp = cfg["spec"]
    if sp == "c3":
        sp = CONFIGS["c3"]["spec"]
    if sp == "jet":
        X, Y, Z = 2048, 1024, 1024
        xs = np.arange(0.2 * X, 0.8 * X + 1e-9, JET["step"])
        return xio.SyntheticSpec(field="gaussian", extent=(X, Y, Z), max_level=3, threshold=JET["thr"], seed=0,
                                 holes=tuple((float(x), Y / 2, Z / 2, JET["rh"]) for x in xs),
                                 refine_spheres=tuple((float(x), Y / 2, Z / 2, JET["rr"]) for x in xs),
                                 field_params={"center": (X / 2, Y / 2, Z / 2), "sigma": JET["sigma"]})
    return xio.SyntheticSpec(**sp)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--secondary", default="c2", help="second config timed in the same run ('' = none)")
    ap.add_argument("--extra", default="c4,c5", help="further configs timed in the same run ('' = none)")
    ap.add_argument("--views", type=int, default=8, help="orbit views (R/bench.py:30-44); step k renders view k mod V")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU-baseline sample duration")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ablations", action="store_true")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: no clocks, cpu baseline, e2e, extras or ablations")
    return ap.parse_args(argv)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def sha(a) -> str:
    """sha256 of dtype, shape and bytes (tests/tests_util.py:sha)."""
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def scale_digests(name):
    p = ROOT / "tests" / "golden" / "scale_digests.json"
    if not p.exists():
        return None
    return json.loads(p.read_text()).get(name)


def host_info():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "host_threads": os.cpu_count()}


# ---------------------------------------------------------------------------
# workload


def make_cells(cfg, host=False):
    """Synthetic cells of a config: the numpy generator (C1-C4: a bit-exact
    restatement of the reference's generate_synthetic, R/io.py:247-295, run on
    all host cores; every bench config) or the GPU generator (`gpu_gen`, cells
    left on the device unless `host`)."""
    from paper_2009_03076_b200 import io as xio

    spec = spec_for(cfg)
    if cfg.get("gpu_gen"):
        dc = xio.generate_synthetic_device(spec)
        return dc.to_host() if host else dc
    cache = os.environ.get("XB_CELL_CACHE")  # tools/ab.py: reuse one generation across A/B processes
    if cache:
        from paper_2009_03076_b200.model import CellList

        key = Path(cache) / (hashlib.sha256(repr(spec).encode()).hexdigest()[:16] + ".npz")
        if key.exists():
            z = np.load(key)
            return CellList(z["i"], z["j"], z["k"], z["level"], z["values"], (spec.field_name,))
        cl = xio.generate_synthetic(spec, workers=os.cpu_count() or 1)
        key.parent.mkdir(parents=True, exist_ok=True)
        np.savez(key, i=cl.i, j=cl.j, k=cl.k, level=cl.level, values=cl.values)
        return cl
    return xio.generate_synthetic(spec, workers=os.cpu_count() or 1)


def coll(fn, t, **kw):
    """A torch.distributed collective on tensor `t` in place: NCCL moves device
    memory directly; gloo (the shared-GPU check of the N > 1 path) goes through
    the host."""
    import torch.distributed as dist

    if t.is_cuda and dist.get_backend() == "gloo":
        c = t.cpu()
        fn(c, **kw)
        t.copy_(c)
    else:
        fn(t, **kw)


def make_cells_ranks(cfg, rank, world, dev):
    """The config's cells on every rank: generated once on rank 0 (the numpy
    generator, bit-exact to the reference's) and broadcast over NCCL into
    device-resident cells on each rank (8 host-side generations would need
    8 x 21 GB of host memory at C3)."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2009_03076_b200 import _native as N
    from paper_2009_03076_b200 import io as xio

    if world == 1:
        return make_cells(cfg)
    cl = make_cells(cfg) if rank == 0 else None
    n_t = torch.tensor([len(cl) if cl is not None else 0], dtype=torch.int64, device=dev)
    coll(dist.broadcast, n_t, src=0)
    n = int(n_t.item())
    cols = []
    for name, dt in (("i", torch.int32), ("j", torch.int32), ("k", torch.int32), ("level", torch.int32),
                     ("values", torch.float32)):
        t = torch.empty(n, dtype=dt, device=dev)
        if rank == 0:
            a = getattr(cl, name)
            t.copy_(torch.from_numpy(np.ascontiguousarray(a[:, 0] if name == "values" else a)))
        coll(dist.broadcast, t, src=0)
        cols.append(t)
    torch.cuda.synchronize()
    h = N.new_handle()
    N.check(N.lib().xb_cells_create(n, dev.index, C.byref(h)))
    ch = N.CellsHandle(h.value, dev.index)
    N.check(N.lib().xb_cells_upload(ch.h, 0, n, *(N.ptr(t.data_ptr()) for t in cols)))
    return xio.DeviceCells(ch, n, spec_for(cfg).field_name)


def cameras_for(bounds, cfg, n_views):
    from paper_2009_03076_b200.orbit import orbit_cameras

    w, h = cfg["res"]
    return orbit_cameras(bounds, n_views, w, h)


def tf_for(vr, cfg, max_alpha=None):
    from paper_2009_03076_b200.accel import TransferFunction

    return TransferFunction.grayscale((float(vr[0]), float(vr[1])),
                                      max_alpha=cfg["max_alpha"] if max_alpha is None else max_alpha)


def workload_config(cfg, n_views, n_cells, n_bricks, n_regions):
    """The workload-defining keys, identical in both arms."""
    W, H = cfg["res"]
    return {"workload": cfg["workload"], "width": W, "height": H, "views": n_views, "cells": int(n_cells),
            "bricks": int(n_bricks), "regions": int(n_regions), "gradient_mode": cfg["gradient"],
            "tf": f"grayscale max_alpha={cfg['max_alpha']}", "iso_value": cfg.get("iso"), "seed": 0,
            "cells_source": "GPU generator (csrc/synth.cu)" if cfg.get("gpu_gen") else
            "numpy generator (R/io.py:247-295 restated)"}


# ---------------------------------------------------------------------------
# clocks sampled during the timed region


class ClockSampler:
    """SM clock + throttle reasons polled every ~2 ms through NVML (the
    nvidia-smi fields clocks.sm / clocks_event_reasons.*) while the timed frames
    run."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))

    def __init__(self, device):
        self.device = device
        self.samples = []  # (sm_mhz, reason bits)
        self.max_mhz = None
        self.stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            p = torch.cuda.get_device_properties(self.device)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        rs = int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
                        self.samples.append((sm, rs))
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
        except Exception:
            pass
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0, "source": "nvml"}
        sm = [x for x, _ in self.samples]
        reasons = sorted({n for _, bits in self.samples for n, b in self.REASONS if bits & b})
        loaded = [x for x in sm if x > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "source": "nvml 2 ms poll"}


# ---------------------------------------------------------------------------
# CPU side: the oracle (C restatement of the reference) on host cores


def oracle_camera(cam):
    import oracle

    r, u, f = cam.basis()
    return oracle.camera_struct(cam.width, cam.height, cam.position, r, u, f,
                                math.tan(math.radians(cam.fov_y) * 0.5), cam.width / cam.height)


def oracle_march_kw(params):
    return dict(seed=params.seed, gradient_mode=params.gradient_mode, early=params.early_term_threshold,
                spc=params.samples_per_cell, rate=params.rate_scale)


def cpu_bands(osc, cam, tf, params, target_s, threads, iso=None):
    """The oracle renders row bands spread over the frame, sized to ~target_s of
    CPU work.  Returns (Msamples/s, frames/s equivalent, description, bands)
    with bands = [(pix_begin, pix_end, rgba_f64, regions, samples)] for the
    parity comparison."""
    W, H = cam.width, cam.height
    ocam = oracle_camera(cam)
    osc.set_tf(tf.domain, tf.rgba)
    osc.set_iso(iso)
    kw = oracle_march_kw(params)
    n_bands = 8
    centers = [int((b + 0.5) * H / n_bands) for b in range(n_bands)]

    def run(rows_per_band):
        samples, px, bands, t0 = 0, 0, [], time.perf_counter()
        for c in centers:
            y0 = max(0, min(H - rows_per_band, c - rows_per_band // 2))
            b, e = y0 * W, (y0 + rows_per_band) * W
            of, _, pr, ps = osc.render(ocam, tf.domain, tf.rgba, pix_range=(b, e), threads=threads, **kw)
            samples += int(ps.sum())
            px += e - b
            bands.append((b, e, of, pr, ps))
        return samples, px, time.perf_counter() - t0, bands

    s, px, dt, _ = run(1)
    rows = max(1, min(H // n_bands, int(target_s / max(dt, 1e-3))))
    s, px, dt, bands = run(rows)
    return (s / dt / 1e6, (px / (W * H)) / dt, f"{n_bands} bands x {rows} rows ({px} of {W * H} px) of orbit view 0",
            bands)


# ---------------------------------------------------------------------------
# reference arm


def bench_reference(args, cfg):
    """`--impl reference`: the reference algorithm on the host only (rank 0)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    import oracle
    from paper_2009_03076_b200.model import Box3
    from paper_2009_03076_b200.render import MarchParams

    t0 = time.perf_counter()
    cells = make_cells(dict(cfg, gpu_gen=False))
    t1 = time.perf_counter()
    m = oracle.build_bricks(cells.i, cells.j, cells.k, cells.level, cells.values)
    t2 = time.perf_counter()
    r = oracle.build_regions(*(m[k] for k in MODEL_KEYS))
    t3 = time.perf_counter()
    gold = scale_digests(args.config)
    digests = {"model": {k: sha(m[k]) for k in MODEL_KEYS}, "regions": {k: sha(r[k]) for k in REGION_KEYS}}
    golden_equal = None if gold is None else (digests["model"] == gold["model"] and
                                              digests["regions"] == gold["regions"])
    bounds = Box3(r["lo"].min(axis=0), r["hi"].max(axis=0))
    cams = cameras_for(bounds, cfg, args.views)
    tf = tf_for((m["scalars"][0].min(), m["scalars"][0].max()), cfg)
    params = MarchParams(seed=0, gradient_mode=cfg["gradient"])
    osc = oracle.OracleScene(m, r)
    osc.set_tf(tf.domain, tf.rgba)
    osc.set_iso(cfg.get("iso"))
    threads = os.cpu_count() or 1
    kw = oracle_march_kw(params)
    ocams = [oracle_camera(c) for c in cams]

    def frame(v):
        ta = time.perf_counter()
        _, _, _, ps = osc.render(ocams[v], tf.domain, tf.rgba, threads=threads, **kw)
        return time.perf_counter() - ta, int(ps.sum())

    for k in range(min(args.warmup, 2)):
        frame(k % args.views)
    dts, smp = [], []
    for k in range(args.steps):
        dt, s = frame(k % args.views)
        dts.append(dt)
        smp.append(s)
    v = len(dts) / sum(dts)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": min(args.warmup, 2), "ms_per_step": 1000.0 * sum(dts) / len(dts),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg, args.views, len(cells), len(m["brick_level"]), len(r["finest_width"])),
        "msamples_per_s": sum(smp) / sum(dts) / 1e6,
        "cpu_baseline": {"value": v, "unit": "frames/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} full {cfg['res'][0]}x{cfg['res'][1]} frames over the "
                                   f"{args.views}-view orbit; oracle/xb_oracle.c (C restatement of "
                                   "R/render.py:521-578), OpenMP", **host_info()},
        "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "build_s": {"generate": round(t1 - t0, 2), "oracle_bricks": round(t2 - t1, 2),
                    "oracle_regions": round(t3 - t2, 2)},
        "builders": {"digests": digests, "equal_to_golden": golden_equal},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm


class Scene:
    """A built config on this rank: model, regions, active sets, cameras."""

    def __init__(self, cfg, name, n_views, build_reps=3, cells=None, model=None, regions=None, dist_ctx=None):
        import torch

        from paper_2009_03076_b200.bricks import build_bricks
        from paper_2009_03076_b200.regions import build_regions
        from paper_2009_03076_b200.render import MarchParams, build_scene

        self.cfg, self.name = cfg, name
        if model is None:
            if cells is None:
                cells = make_cells_ranks(cfg, *dist_ctx) if dist_ctx else make_cells(cfg)
            self.n_cells = len(cells)
            # build timings: one untimed warm-up build (device pool, page-locked staging), then the
            # median of `build_reps` builds
            times = {"bricks": [], "regions": [], "tf_active_sets": []}
            for rep in range(build_reps + 1):
                torch.cuda.synchronize()
                ta = time.perf_counter()
                model, _ = build_bricks(cells)
                tb = time.perf_counter()
                regions = build_regions(model)
                tc = time.perf_counter()
                tf = tf_for(model.value_range(0), cfg)
                scene = build_scene(model, regions, tf, iso_value=cfg.get("iso"))
                td = time.perf_counter()
                if rep > 0:
                    times["bricks"].append((tb - ta) * 1e3)
                    times["regions"].append((tc - tb) * 1e3)
                    times["tf_active_sets"].append((td - tc) * 1e3)
                if rep < build_reps:
                    del scene, regions, model
            self.build_ms = {k: round(float(np.median(v)), 1) for k, v in times.items()}
            self.build_ms["reps"] = build_reps
            del cells
        else:
            self.n_cells = cells
            tf = tf_for(model.value_range(0), cfg)
            scene = build_scene(model, regions, tf, iso_value=cfg.get("iso"))
            self.build_ms = None
        self.model, self.regions, self.scene, self.tf = model, regions, scene, tf
        self.cams = cameras_for(regions.bounds, cfg, n_views)
        self.params = MarchParams(seed=0, gradient_mode=cfg["gradient"])

    def builder_parity(self):
        """GPU builder arrays vs the oracle's digests at this scale (None when absent)."""
        gold = scale_digests(self.name)
        if gold is None or gold.get("n_cells") != self.n_cells:
            return None
        bad = [f"model.{k}" for k in MODEL_KEYS if sha(getattr(self.model, k)) != gold["model"][k]]
        bad += [f"regions.{k}" for k in REGION_KEYS if sha(getattr(self.regions, k)) != gold["regions"][k]]
        return {"equal": not bad, "mismatched": bad, "reference": "oracle digests, tests/golden/scale_digests.json"}


def march_times(n):
    import ctypes as C

    from paper_2009_03076_b200 import _native as N

    buf = np.zeros(max(n, 1))
    got = C.c_int32()
    N.check(N.lib().xb_march_times(N.ptr(buf), int(n), C.byref(got)))
    return buf[:got.value]


def time_frames(S, args, steps, warmup, world, rank, dev, with_clocks=False):
    """Timed orbit frames of scene S: returns (frame_ms[steps], march_ms[steps], clocks)."""
    import torch
    import torch.distributed as dist

    from paper_2009_03076_b200 import _native as N
    from paper_2009_03076_b200.parallel import TiledRenderer

    W, H = S.cfg["res"]
    rend = TiledRenderer(S.scene, W, H, dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    V = len(S.cams)
    for k in range(warmup):
        rend.render(S.cams[k % V], S.tf, S.params, stats=world > 1)
    torch.cuda.synchronize()
    march_times(10 ** 6)  # drop stale records
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    sampler = ClockSampler(dev.index) if with_clocks else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.__enter__()
    with N.tuning(time_march=1):
        for k in range(steps):
            flush.zero_()  # L2 flush between frames (outside the per-frame events)
            a, b = ev[k]
            a.record(stream)
            rend.render(S.cams[k % V], S.tf, S.params, stats=world > 1)
            b.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if sampler:
        sampler.__exit__(None, None, None)
    frame_ms = np.array([a.elapsed_time(b) for a, b in ev])
    mt = march_times(steps)
    march_ms = mt if len(mt) == steps else np.full(steps, np.nan)
    if world > 1:  # max over ranks, per step
        t = torch.tensor(np.stack([frame_ms, march_ms]), dtype=torch.float64, device=dev)
        coll(dist.all_reduce, t, op=dist.ReduceOp.MAX)
        frame_ms, march_ms = t.cpu().numpy()
    return frame_ms, march_ms, (sampler.summary() if sampler else None), rend


def count_views(S, world, rank, dev):
    """Per-view [regions, samples, algorithmic bytes] of the whole frame (one
    untimed byte-counting launch per view on each rank, summed over ranks)."""
    import torch
    import torch.distributed as dist

    from paper_2009_03076_b200.parallel import TiledRenderer, tiles_per_rank, TILE_PX
    from paper_2009_03076_b200.render import render_native

    W, H = S.cfg["res"]
    out = torch.empty((tiles_per_rank(W, H, world) * TILE_PX, 4) if world > 1 else (H, W, 4), dtype=torch.uint8,
                      device=dev)
    rows = []
    for cam in S.cams:
        st = render_native(S.scene, cam, S.tf, S.params, out.data_ptr(), tile_rank=rank, tile_world=world,
                           count_bytes=True, stream=torch.cuda.current_stream().cuda_stream)
        rows.append([int(x) for x in st])
    torch.cuda.synchronize()
    t = torch.tensor(rows, dtype=torch.int64, device=dev)
    if world > 1:
        coll(dist.all_reduce, t)
    return t.cpu().numpy()


def roofline(bytes_total, march_ms_total, frame_ms_total, peaks):
    peak = float(peaks.get("hbm_gbs", 6650.0))
    ach = bytes_total / (march_ms_total * 1e-3) / 1e9
    ach_frame = bytes_total / (frame_ms_total * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "kernel": "k_warp (csrc/render.cu), the frame's dominant kernel: algorithmic bytes of the frame "
                      "(SURVEY §8(d), counted per view by the COUNT launch) / k_warp's CUDA-event time",
            "frame_achieved": ach_frame, "frame_frac": ach_frame / peak,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if peaks else "fallback 6.65 TB/s"}


def run_config(args, S, world, rank, dev, peaks, steps, warmup, with_clocks=False):
    """Orbit timing of a built scene: the per-config part of the JSON line."""
    fms, mms, clocks, rend = time_frames(S, args, steps, warmup, world, rank, dev, with_clocks)
    counts = count_views(S, world, rank, dev)  # (V, 3)
    V = len(S.cams)
    per_step = counts[np.arange(steps) % V]
    out = {
        "value": 1000.0 * steps / float(fms.sum()), "unit": "frames/s", "ms_per_step": float(fms.mean()),
        "msamples_per_s": float(per_step[:, 1].sum()) / (float(fms.sum()) * 1e-3) / 1e6,
        "kernel_ms": float(mms.mean()),
        "frame": {"samples": int(per_step[:, 1].sum() // steps), "region_visits": int(per_step[:, 0].sum() // steps),
                  "alg_bytes": int(per_step[:, 2].sum() // steps),
                  "alg_bytes_per_sample": float(per_step[:, 2].sum() / max(per_step[:, 1].sum(), 1))},
        "views": [{"view": v, "ms": float(np.mean(fms[v::V])) if v < steps else None,
                   "k_warp_ms": float(np.mean(mms[v::V])) if v < steps else None,
                   "samples": int(counts[v, 1]), "region_visits": int(counts[v, 0]), "alg_bytes": int(counts[v, 2])}
                  for v in range(V)],
        "roofline": roofline(float(per_step[:, 2].sum()), float(mms.sum()), float(fms.sum()), peaks),
    }
    return out, clocks, rend


def frame_parity(S, bands):
    """GPU float frame of orbit view 0 vs the oracle's bands (same pixels)."""
    from paper_2009_03076_b200.render import render_frame_float

    u8, f64, cnt, st = render_frame_float(S.scene, S.cams[0], S.tf, S.params)
    f = f64.reshape(-1, 4)
    c = cnt.reshape(-1, 2)
    d, bad_r, bad_s, px = 0.0, 0, 0, 0
    for b, e, of, pr, ps in bands:
        dd = np.abs(f[b:e] - of)
        d = max(d, float(dd.max()) if np.isfinite(dd).all() else float("inf"))  # NaN / inf fail
        bad_r += int(np.count_nonzero(c[b:e, 0] != pr))
        bad_s += int(np.count_nonzero(c[b:e, 1] != ps))
        px += e - b
    return {"view": 0, "pixels": px, "max_abs_drgba": d, "tolerance": RGBA_TOL,
            "px_region_counter_mismatches": bad_r, "px_sample_counter_mismatches": bad_s,
            "ok": d <= RGBA_TOL and bad_r == 0 and bad_s == 0}


def oracle_parity(S, seconds, view=0, osc=None):
    """Oracle row bands (~`seconds` of host work) of an orbit view against the GPU
    float frame: the in-run frame parity of the secondary / extra configs (`osc`:
    an oracle scene of the same model to reuse)."""
    import oracle

    if osc is None:
        osc = oracle.OracleScene({k: getattr(S.model, k) for k in MODEL_KEYS},
                                 {k: getattr(S.regions, k) for k in REGION_KEYS})
    cam = S.cams[view]
    _, _, _, bands = cpu_bands(osc, cam, S.tf, S.params, seconds, os.cpu_count() or 1, iso=S.cfg.get("iso"))
    from paper_2009_03076_b200.render import render_frame_float

    u8, f64, cnt, st = render_frame_float(S.scene, cam, S.tf, S.params)
    f, c = f64.reshape(-1, 4), cnt.reshape(-1, 2)
    d, bad_r, bad_s, px = 0.0, 0, 0, 0
    for b, e, of, pr, ps in bands:
        dd = np.abs(f[b:e] - of)
        d = max(d, float(dd.max()) if np.isfinite(dd).all() else float("inf"))  # NaN / inf fail
        bad_r += int(np.count_nonzero(c[b:e, 0] != pr))
        bad_s += int(np.count_nonzero(c[b:e, 1] != ps))
        px += e - b
    return {"view": view, "pixels": px, "max_abs_drgba": d, "tolerance": RGBA_TOL,
            "px_region_counter_mismatches": bad_r, "px_sample_counter_mismatches": bad_s,
            "ok": d <= RGBA_TOL and bad_r == 0 and bad_s == 0}


def e2e_orbit(S, steps):
    """The public API with host output, cycling the orbit: `render_frames` (the
    host copy of frame k overlaps the march of frame k+1; wall time over the K
    frames) and `render_frame` (one synchronous call per frame)."""
    import torch

    from paper_2009_03076_b200.render import render_frame, render_frames

    V = len(S.cams)
    cams = [S.cams[k % V] for k in range(steps)]
    for _ in range(2):  # warm: the page-locked host blocks of a pipelined run come from torch's caching allocator
        for fr in render_frames(S.scene, cams[:max(V, 8)], S.tf, S.params):
            pass
    torch.cuda.synchronize()
    ta = time.perf_counter()
    n = 0
    for fr in render_frames(S.scene, cams, S.tf, S.params):
        n += fr.stats.samples > 0
    pipelined_ms = (time.perf_counter() - ta) * 1e3 / steps
    for k in range(3):
        render_frame(S.scene, S.cams[k % V], S.tf, S.params)
    torch.cuda.synchronize()
    ts = []
    for k in range(steps):
        ta = time.perf_counter()
        render_frame(S.scene, S.cams[k % V], S.tf, S.params)
        ts.append((time.perf_counter() - ta) * 1e3)
    return pipelined_ms, ts


def ablations(S, dev):
    """Paper Table 3 (cell location vs ABR regions) and the
    reference's traversal (per-visit LBVH queries) vs the k-d walk, on view 0."""
    import torch

    from paper_2009_03076_b200 import _native as N
    from paper_2009_03076_b200.render import render_native

    W, H = S.cfg["res"]
    out = torch.empty((H, W, 4), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    cam = S.cams[0]

    def t(reps=3, **kw):
        render_native(S.scene, cam, S.tf, S.params, out.data_ptr(), stream=stream.cuda_stream, sync=False, **kw)
        ms = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            render_native(S.scene, cam, S.tf, S.params, out.data_ptr(), stream=stream.cuda_stream, sync=False, **kw)
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        return float(np.median(ms))

    res = {"config": S.name, "view": 0}
    res["region_walk_ms"] = t()
    with N.tuning(traversal=1):
        res["lbvh_per_visit_ms"] = t()
    with N.tuning(kernel=1):
        res["one_thread_per_pixel_ms"] = t()
    if S.scene.tree is not None:
        res["cell_location_ms"] = t(reps=1, use_celllocation=True)
        res["celllocation_over_region"] = res["cell_location_ms"] / res["region_walk_ms"]
        res["celllocation_over_region_same_kernel"] = res["cell_location_ms"] / res["one_thread_per_pixel_ms"]
    res["lbvh_over_kdwalk"] = res["lbvh_per_visit_ms"] / res["region_walk_ms"]
    return res


def bench_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # XB_BENCH_SHARE_GPU=1 (tests only): every rank on cuda:0 over gloo, to run the
    # N > 1 code path on a one-GPU box (NCCL refuses two ranks on one device)
    shared = os.environ.get("XB_BENCH_SHARE_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl = None
    if world > 1 and shared:
        dist.init_process_group("gloo")
    elif world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if world > 1:
        x = torch.ones(1, device=dev)
        coll(dist.all_reduce, x)  # communicator up; its size must equal the world
        nccl = {"backend": dist.get_backend(), "world": dist.get_world_size(), "allreduce_ones": int(x.item()),
                "version": ".".join(map(str, torch.cuda.nccl.version()))}
        if nccl["allreduce_ones"] != world:
            raise RuntimeError(f"NCCL communicator has {nccl['allreduce_ones']} ranks, expected {world}")
        log(f"[rank {rank}] NCCL communicator: {nccl}")
    from paper_2009_03076_b200 import _native as N

    N.require_device(local)
    peaks = {}
    pk = ROOT / "MEASURED_PEAKS.json"
    if pk.exists():
        peaks = json.loads(pk.read_text())
    cfg = CONFIGS[args.config]
    full = not args.profile
    dctx = (rank, world, dev) if world > 1 else None
    S = Scene(cfg, args.config, args.views, build_reps=3 if full else 0, dist_ctx=dctx)
    res, clocks, rend = run_config(args, S, world, rank, dev, peaks, args.steps, args.warmup, with_clocks=full)
    line = None
    ok = True
    if rank == 0:
        W, H = cfg["res"]
        line = {"metric": METRIC, "value": res["value"], "unit": "frames/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "dtype_note": "FP64 sample positions, hat weights, value sums, TF and compositing (the reference's "
                              "arithmetic); the analytic gradient that only feeds the headlight factor is FP32",
                "config": workload_config(cfg, args.views, S.n_cells, S.model.n_bricks, len(S.regions))}
        line.update({k: res[k] for k in ("msamples_per_s", "kernel_ms", "frame", "roofline", "views")})
        line["method"] = {"l2": "flushed between frames (256 MB write)", "parallelism": f"screen tiles 16x8 x{world}",
                          "orbit": f"step k renders orbit view k mod {args.views} (R/bench.py:30-62)",
                          "timing": "CUDA events per frame on the render stream, max over ranks"}
        line["build_ms"] = S.build_ms
        tp = ROOT / "profiles" / f"traffic_{args.config}.json"
        if tp.exists():
            tj = json.loads(tp.read_text())
            line["roofline"]["traffic"] = tj.get("dram_bytes_per_launch")
            line["roofline"]["traffic_source"] = tj.get("source")
        else:
            line["roofline"]["traffic"] = None
        # own kernels per frame: k_classify, k_walk, k_route, k_walk2, k_warp (+ CUB's two select
        # kernels, library code); the iso phase adds k_classify, k_walk, k_route, k_iso_warp; rank 0
        # of a tiled run adds k_unpack_tiles
        line["gpu_launches"] = args.steps * (5 + 4 * (cfg.get("iso") is not None) + (world > 1))
        if nccl:
            line["nccl"] = nccl
    if full:
        if world == 1:
            pipe_ms, e2e = e2e_orbit(S, args.steps)
            import ctypes

            line["e2e"] = {"value": 1000.0 / pipe_ms, "unit": "frames/s",
                           "h2d_bytes_per_step": ctypes.sizeof(N.XbMarch) + ctypes.sizeof(N.XbCamera),
                           "d2h_bytes_per_step": cfg["res"][0] * cfg["res"][1] * 4 + 24,
                           "ms_per_step": pipe_ms,
                           "api": "render_frames(scene, orbit cameras, tf, params) -> numpy Frames (RGBA8 + "
                                  "FrameStats; each frame's D2H overlaps the next frame's march)",
                           "sync": {"value": 1000.0 * len(e2e) / sum(e2e), "ms_per_step": float(np.mean(e2e)),
                                    "ms_steps": [round(x, 3) for x in e2e],
                                    "api": "render_frame() per frame (synchronous)"}}
        else:
            e2e_ms = e2e_tiled(S, rend, args.steps, world, rank, dev)
            if rank == 0:
                W, H = cfg["res"]
                line["e2e"] = {"value": 1000.0 / e2e_ms, "unit": "frames/s", "h2d_bytes_per_step": 0,
                               "d2h_bytes_per_step": W * H * 4 + 16, "ms_per_step": e2e_ms,
                               "api": "TiledRenderer.render(stats=True) + D2H of the image and counters"}
        if rank == 0:
            line["clocks"] = clocks
            line["parity"] = {"builders": S.builder_parity()}
            if world == 1 and not args.no_cpu_baseline:
                import oracle

                osc = oracle.OracleScene({k: getattr(S.model, k) for k in MODEL_KEYS},
                                         {k: getattr(S.regions, k) for k in REGION_KEYS})
                threads = os.cpu_count() or 1
                ms_, fs_, desc, bands = cpu_bands(osc, S.cams[0], S.tf, S.params, args.cpu_seconds, threads,
                                                  iso=cfg.get("iso"))
                line["cpu_baseline"] = {"value": fs_, "unit": "frames/s", "cores": threads, "kind": "port",
                                        "sample": desc + " (oracle/xb_oracle.c, OpenMP, on the GPU-built arrays, "
                                                         "equal to the oracle's own by the builder parity)",
                                        "msamples_per_s": ms_, **host_info()}
                line["parity"]["frame"] = frame_parity(S, bands)
                S.osc = osc  # reused by C4's frame parity (same model)
            else:
                line["cpu_baseline"] = None
            pb = line["parity"]["builders"]
            ok = (pb is None or pb["equal"]) and line["parity"].get("frame", {}).get("ok", True)
            line["parity"]["ok"] = ok
    # secondary and extra configs
    if args.secondary and args.secondary != args.config:
        S2 = Scene(CONFIGS[args.secondary], args.secondary, args.views, build_reps=1 if full else 0, dist_ctx=dctx)
        r2, _, _ = run_config(args, S2, world, rank, dev, peaks, 8, 4)
        if rank == 0:
            line["secondary"] = dict(r2, config=workload_config(S2.cfg, args.views, S2.n_cells, S2.model.n_bricks,
                                                                len(S2.regions)), build_ms=S2.build_ms)
            if full:
                line["secondary"]["parity"] = {"builders": S2.builder_parity()}
                ok = ok and (line["secondary"]["parity"]["builders"] or {"equal": True})["equal"]
                if world == 1 and not args.no_cpu_baseline:
                    fp = oracle_parity(S2, 3.0)
                    line["secondary"]["parity"]["frame"] = fp
                    ok = ok and fp["ok"]
        if full and not args.no_ablations and world == 1:
            from paper_2009_03076_b200.bricks import BrickBuildParams, build_bricks

            S2.scene.tree = build_bricks(make_cells(S2.cfg), BrickBuildParams(keep_split_tree=True))[1]
            line["ablations"] = ablations(S2, dev)
        del S2
    if full and args.extra:
        line_extra = {}
        for name in [x for x in args.extra.split(",") if x and x != args.config]:
            cfg_x = CONFIGS[name]
            if cfg_x["spec"] == "c3" and args.config == "c3":  # C4 reuses the C3 model (iso + TF refresh)
                Sx = Scene(cfg_x, name, args.views, cells=S.n_cells, model=S.model, regions=S.regions)
                Sx.build_ms = tf_refresh(Sx)
            else:
                Sx = Scene(cfg_x, name, args.views, build_reps=1, dist_ctx=dctx)
            rx, _, _ = run_config(args, Sx, world, rank, dev, peaks, 8, 4)
            if rank == 0:
                line_extra[name] = dict(rx, config=workload_config(cfg_x, args.views, Sx.n_cells, Sx.model.n_bricks,
                                                                   len(Sx.regions)), build_ms=Sx.build_ms)
                line_extra[name]["parity"] = {}
                if Sx.build_ms and "bricks" in Sx.build_ms:  # a model of its own: its builder parity
                    pb = Sx.builder_parity()
                    line_extra[name]["parity"]["builders"] = pb
                    ok = ok and (pb or {"equal": True})["equal"]
                reuse = getattr(S, "osc", None) if Sx.model is S.model else None
                if world == 1 and not args.no_cpu_baseline and (reuse is not None or Sx.n_cells < 300_000_000):
                    fp = oracle_parity(Sx, 3.0, osc=reuse)
                    line_extra[name]["parity"]["frame"] = fp
                    ok = ok and fp["ok"]
                elif world == 1:  # C5: the oracle's BVH over 50M regions takes minutes; builders by digests
                    line_extra[name]["parity"]["frame"] = "not run in the bench (oracle scene build too slow)"
            del Sx
            torch.cuda.empty_cache()
        if rank == 0:
            line["extra"] = line_extra
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if not ok:
        log("PARITY VIOLATION: see line['parity']")
        return 1
    return 0


def tf_refresh(S):
    """Config 4's interactive TF edit: rebuild the volume active set (per-region
    majorants, R/accel.py:91-115 + 227-234) for a new ramp; median of 9 after 3 warm-up rebuilds."""
    import torch

    from paper_2009_03076_b200.accel import build_volume_bvh

    import ctypes as C
    import gc

    from paper_2009_03076_b200 import _native as N

    tf2 = [tf_for(S.model.value_range(0), S.cfg, max_alpha=a) for a in (0.3, 0.4)]
    for k in range(3):  # warm: the first rebuilds grow the allocator pools
        build_volume_bvh(S.regions, tf2[k % 2], 0, model=S.model)
    wall, dev = [], []
    for k in range(9):
        gc.collect()
        torch.cuda.synchronize()
        ta = time.perf_counter()
        b = build_volume_bvh(S.regions, tf2[k % 2], 0, model=S.model)
        wall.append((time.perf_counter() - ta) * 1e3)
        na, ms = C.c_int64(), C.c_double()
        N.check(N.lib().xb_active_info(b.handle.h, C.byref(na), C.byref(ms)))
        dev.append(ms.value)
        del b
    return {"tf_refresh_ms": float(np.median(wall)), "build_active_ms": float(np.median(dev)),
            "tf_refresh_ms_all": [round(x, 2) for x in wall]}


def e2e_tiled(S, rend, steps, world, rank, dev):
    """N>1 end to end: tiles rendered, gathered and unpacked on rank 0, counters
    all-reduced, image + counters read back to the host on rank 0."""
    import torch
    import torch.distributed as dist

    W, H = S.cfg["res"]
    host = torch.empty((H, W, 4), dtype=torch.uint8, pin_memory=True)
    V = len(S.cams)
    dist.barrier()
    te = time.perf_counter()
    for k in range(steps):
        img, st = rend.render(S.cams[k % V], S.tf, S.params, stats=True)
        if rank == 0:
            host.copy_(img, non_blocking=True)
            st = st.cpu()
        torch.cuda.synchronize()
    te = time.perf_counter() - te
    tt = torch.tensor([te], dtype=torch.float64, device=dev)
    coll(dist.all_reduce, tt, op=dist.ReduceOp.MAX)
    return float(tt.item()) / steps * 1000.0


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main(argv=None):
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run on this node
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(ROOT / "bench.py")]
        cmd += sys.argv[1:] if argv is None else list(argv)
        return subprocess.call(cmd)
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        log(f"note: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}; the world size wins")
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return bench_reference(args, cfg)
    return bench_ours(args)


if __name__ == "__main__":
    sys.exit(main())
