#!/usr/bin/env python
"""bench.py — ExaBricks render hot path on B200 (one JSON line on rank 0).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c2]

Workload (N=1): BASELINE.json configs[1] — synthetic 4-level gaussian AMR
(9.53M cells, SURVEY.md §8(d) "C2"), DVR + analytic-gradient shading,
grayscale TF (max alpha 0.5), 1024x1024, orbit view 0, seed 0.  A step is one
frame: ray march of every pixel through the resident scene (+ the NCCL tile
gather for N>1).  Inputs are resident in HBM; L2 (126 MB) is flushed by a
256 MB write between timed frames.  Metric: frames/s (whole job) with
Msamples/s beside it (`FrameStats.samples` / s, R/render.py:419).

`--impl reference` times the CPU oracle port (oracle/, a C restatement of the
reference renderer, all host threads) on bounded row samples of the same frame.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frames/sec and Msamples/sec at 1920×1080 (1/2/4/8 B200), % HBM roofline"

CONFIGS = {
    # SURVEY.md §8(d) C1 / C2 (BASELINE.json configs[0] / configs[1])
    "c1": dict(spec=dict(field="gaussian", extent=(64, 64, 64), max_level=1, threshold=0.04, seed=0),
               res=(256, 256), max_alpha=1.0, gradient="analytic",
               workload="configs[0]: synthetic 2-level gaussian AMR, 97,840 cells, 256x256 DVR + analytic shading"),
    "c2": dict(spec=dict(field="gaussian", extent=(256, 256, 256), max_level=3, threshold=0.004, seed=0),
               res=(1024, 1024), max_alpha=0.5, gradient="analytic",
               workload="configs[1]: synthetic 4-level gaussian AMR (2x ratio), 9,534,568 cells, "
                        "1024x1024 DVR + analytic gradient shading, 1 GPU"),
    "c2_1080p": dict(spec=dict(field="gaussian", extent=(256, 256, 256), max_level=3, threshold=0.004, seed=0),
                     res=(1920, 1080), max_alpha=0.5, gradient="analytic",
                     workload="configs[1] model at 1920x1080, DVR + analytic gradient shading"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--view", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU-baseline sample duration")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no clocks, no cpu baseline, no e2e")
    return ap.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# workload


def make_cells(cfg):
    from paper_2009_03076_b200 import io as xio

    return xio.generate_synthetic(xio.SyntheticSpec(**cfg["spec"]))


def camera_for(bounds, cfg, view):
    from paper_2009_03076_b200.orbit import orbit_cameras

    w, h = cfg["res"]
    return orbit_cameras(bounds, 8, w, h)[view]


def tf_for(vr, cfg):
    from paper_2009_03076_b200.accel import TransferFunction

    return TransferFunction.grayscale((float(vr[0]), float(vr[1])), max_alpha=cfg["max_alpha"])


# ---------------------------------------------------------------------------
# clocks sampled during the timed region


class ClockSampler:
    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU side: the oracle port on host cores


def oracle_scene_from(model_arrays, region_arrays):
    import oracle

    return oracle.OracleScene(model_arrays, region_arrays)


def cpu_rate(osc, cam, tf, params, W, H, target_s, threads):
    """Render bounded row bands spread over the frame until ~target_s of CPU work.
    Returns (Msamples/s, frames/s-equivalent, sample description)."""
    import oracle

    r, u, f = cam.basis()
    ocam = oracle.camera_struct(W, H, cam.position, r, u, f, math.tan(math.radians(cam.fov_y) * 0.5), W / H)
    osc.set_tf(tf.domain, tf.rgba)
    kw = dict(seed=params.seed, gradient_mode=params.gradient_mode, early=params.early_term_threshold,
              spc=params.samples_per_cell, rate=params.rate_scale)
    # probe: 8 rows spread over the frame
    n_bands = 8
    centers = [int((b + 0.5) * H / n_bands) for b in range(n_bands)]

    def run(rows_per_band):
        samples, px, t0 = 0, 0, time.perf_counter()
        for c in centers:
            y0 = max(0, min(H - rows_per_band, c - rows_per_band // 2))
            _, _, _, ps = osc.render(ocam, tf.domain, tf.rgba, pix_range=(y0 * W, (y0 + rows_per_band) * W),
                                     threads=threads, **kw)
            samples += int(ps.sum())
            px += rows_per_band * W
        return samples, px, time.perf_counter() - t0

    s, px, dt = run(1)
    rows = max(1, min(H // n_bands, int(target_s / max(dt, 1e-3))))
    s, px, dt = run(rows)
    return s / dt / 1e6, (px / (W * H)) / dt, f"{n_bands} bands x {rows} rows ({px} of {W * H} px) of view frame", dt


# ---------------------------------------------------------------------------


def bench_reference(args, cfg):
    """`--impl reference`: the CPU oracle port (restated reference renderer), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_2009_03076_b200.render import MarchParams

    cells = make_cells(cfg)
    t0 = time.perf_counter()
    m = oracle.build_bricks(cells.i, cells.j, cells.k, cells.level, cells.values)
    r = oracle.build_regions(m["brick_lower"], m["brick_level"], m["brick_dims"], m["brick_offset"], m["scalars"])
    build_s = time.perf_counter() - t0
    from paper_2009_03076_b200.model import Box3

    bounds = Box3(r["lo"].min(axis=0), r["hi"].max(axis=0))
    cam = camera_for(bounds, cfg, args.view)
    tf = tf_for((m["scalars"][0].min(), m["scalars"][0].max()), cfg)
    params = MarchParams(seed=0, gradient_mode=cfg["gradient"])
    osc = oracle_scene_from(m, r)
    threads = os.cpu_count() or 1
    W, H = cfg["res"]
    per_step = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        cpu_rate(osc, cam, tf, params, W, H, per_step / 4, threads)
    rates, fps, desc, total = [], [], "", 0.0
    for _ in range(args.steps):
        ms, fs, desc, dt = cpu_rate(osc, cam, tf, params, W, H, per_step, threads)
        rates.append(ms)
        fps.append(fs)
        total += dt
    v = float(np.mean(fps))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / v, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "width": W, "height": H, "view": args.view,
                   "cells": int(len(cells)), "oracle_build_s": round(build_s, 2)},
        "msamples_per_s": float(np.mean(rates)),
        "cpu_baseline": {"value": v, "unit": "frames/s", "cores": threads, "kind": "port",
                         "sample": desc + "; oracle/xb_oracle.c (C restatement of R/render.py), OpenMP",
                         "msamples_per_s": float(np.mean(rates))},
        "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bench_ours(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    from paper_2009_03076_b200 import _native as N
    from paper_2009_03076_b200.bricks import build_bricks
    from paper_2009_03076_b200.parallel import TiledRenderer
    from paper_2009_03076_b200.regions import build_regions
    from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame, render_native

    N.require_device(local)
    cells = make_cells(cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    model, _ = build_bricks(cells)
    t1 = time.perf_counter()
    regions = build_regions(model)
    t2 = time.perf_counter()
    tf = tf_for(model.value_range(0), cfg)
    scene = build_scene(model, regions, tf)
    t3 = time.perf_counter()
    W, H = cfg["res"]
    cam = camera_for(regions.bounds, cfg, args.view)
    params = MarchParams(seed=0, gradient_mode=cfg["gradient"])
    rend = TiledRenderer(scene, W, H, dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    # algorithmic bytes + counters of this rank's share (one untimed counting launch)
    cnt_out = torch.empty((rend.slots * 128, 4) if world > 1 else (H, W, 4), dtype=torch.uint8, device=dev)
    stats = render_native(scene, cam, tf, params, cnt_out.data_ptr(), tile_rank=rank, tile_world=world,
                          count_bytes=True, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    regions_pf, samples_pf, bytes_pf = (int(x) for x in stats)
    if world > 1:
        t = torch.tensor([regions_pf, samples_pf, bytes_pf], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        tot_regions, tot_samples, tot_bytes = (int(x) for x in t.tolist())
    else:
        tot_regions, tot_samples, tot_bytes = regions_pf, samples_pf, bytes_pf

    for _ in range(args.warmup):
        rend.render(cam, tf, params)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local) if not args.profile else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.__enter__()
    wall0 = time.perf_counter()
    for k in range(args.steps):
        flush.zero_()  # L2 flush between frames (outside the per-frame events)
        a, b, c = ev[k]
        a.record(stream)
        if world > 1:
            rend.render(cam, tf, params, gather=False)
            b.record(stream)
            dist.all_gather_into_tensor(rend.gathered, rend.packed)
            if rank == 0:
                N.check(N.lib().xb_unpack_tiles(N.ptr(rend.gathered.data_ptr()), rend.slots, world, W, H,
                                                N.ptr(rend.image.data_ptr()), N.ptr(stream.cuda_stream)))
        else:
            rend.render(cam, tf, params)
            b.record(stream)
        c.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    if sampler:
        sampler.__exit__(None, None, None)
    frame_ms = np.array([a.elapsed_time(c) for a, b, c in ev])
    kern_ms = np.array([a.elapsed_time(b) for a, b, c in ev])
    t = torch.tensor([frame_ms.mean(), kern_ms.mean()], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step, ms_kernel = (float(x) for x in t.tolist())

    # ---- e2e through the public API: host output, stats read back every frame
    e2e = None
    if not args.profile:
        if world == 1:
            render_frame(scene, cam, tf, params)
            torch.cuda.synchronize()
            te = time.perf_counter()
            for _ in range(args.steps):
                fr = render_frame(scene, cam, tf, params)
            te = time.perf_counter() - te
            assert fr.stats.samples == tot_samples
            e2e_ms = te / args.steps * 1000.0
        else:
            host = torch.empty((H, W, 4), dtype=torch.uint8, pin_memory=True)
            dist.barrier()
            te = time.perf_counter()
            for _ in range(args.steps):
                img = rend.render(cam, tf, params)
                st = torch.tensor([regions_pf, samples_pf], dtype=torch.int64, device=dev)
                dist.all_reduce(st)
                if rank == 0:
                    host.copy_(img, non_blocking=True)
                    st.cpu()
                torch.cuda.synchronize()
            te = time.perf_counter() - te
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt.item()) / args.steps * 1000.0
        from paper_2009_03076_b200 import _native as NN
        import ctypes

        e2e = {"value": 1000.0 / e2e_ms, "unit": "frames/s",
               "h2d_bytes_per_step": ctypes.sizeof(NN.XbMarch) + ctypes.sizeof(NN.XbCamera),
               "d2h_bytes_per_step": W * H * 4 + 24, "ms_per_step": e2e_ms,
               "api": "render_frame() -> numpy Frame" if world == 1 else "TiledRenderer.render + D2H of the image"}

    # ---- roofline of the dominant kernel (k_render): algorithmic bytes / kernel time
    peaks = {}
    pk = ROOT / "MEASURED_PEAKS.json"
    if pk.exists():
        peaks = json.loads(pk.read_text())
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = bytes_pf / (float(kern_ms.mean()) * 1e-3) / 1e9  # this rank's launch
    traffic = None
    tp = ROOT / "profiles" / f"traffic_{args.config}.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get("dram_bytes_per_launch")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        osc = oracle_scene_from({k: getattr(model, k) for k in ("brick_lower", "brick_level", "brick_dims",
                                                                "brick_offset", "scalars")},
                                {k: getattr(regions, k) for k in ("lo", "hi", "brick_off", "brick_ids",
                                                                  "value_range", "finest_width")})
        threads = os.cpu_count() or 1
        ms_, fs_, desc, dt = cpu_rate(osc, cam, tf, params, W, H, args.cpu_seconds, threads)
        cpu = {"value": fs_, "unit": "frames/s", "cores": threads, "kind": "port",
               "sample": desc + " (oracle/xb_oracle.c, OpenMP, GPU-built bit-exact arrays)",
               "msamples_per_s": ms_}

    if rank == 0:
        fps = 1000.0 / ms_step
        line = {
            "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "width": W, "height": H, "view": args.view,
                       "cells": int(model.n_cells), "bricks": int(model.n_bricks), "regions": int(len(regions)),
                       "gradient_mode": cfg["gradient"], "tf": f"grayscale max_alpha={cfg['max_alpha']}",
                       "l2": "flushed between frames (256 MB write)", "parallelism": f"screen tiles 16x8 x{world}",
                       "build_ms": {"bricks": round((t1 - t0) * 1e3, 1), "regions": round((t2 - t1) * 1e3, 1),
                                    "tf_active_sets": round((t3 - t2) * 1e3, 1)}},
            "msamples_per_s": tot_samples / (ms_step * 1e-3) / 1e6,
            "frame": {"samples": tot_samples, "region_visits": tot_regions, "alg_bytes": tot_bytes,
                      "alg_bytes_per_sample": tot_bytes / max(tot_samples, 1)},
            "kernel_ms": ms_kernel, "wall_s_timed": wall,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k_warp<1,false,false> (csrc/render.cu)",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if peaks else "fallback 6.65 TB/s"},
            "gpu_launches": args.steps * (1 if world == 1 else 2),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if sampler:
            line["clocks"] = sampler.summary()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        bench_reference(args, cfg)
    else:
        bench_ours(args, cfg)


if __name__ == "__main__":
    main()
