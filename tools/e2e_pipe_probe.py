"""e2e variants at a bench config (host RGBA8 out): sync render_frame, render_frames,
and a ring of preallocated pinned buffers.  python tools/e2e_pipe_probe.py c3 [frames]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2009_03076_b200.bricks import build_bricks  # noqa: E402
from paper_2009_03076_b200.regions import build_regions  # noqa: E402
from paper_2009_03076_b200.render import MarchParams, build_scene, render_frame, render_frames, render_native  # noqa

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 32
cells = bench.make_cells(cfg)
model, _ = build_bricks(cells)
regions = build_regions(model)
del cells
tf = bench.tf_for(model.value_range(0), cfg)
scene = build_scene(model, regions, tf)
cams = bench.cameras_for(regions.bounds, cfg, 8)
params = MarchParams(seed=0, gradient_mode=cfg["gradient"])
seq = [cams[k % 8] for k in range(K)]
W, H = cfg["res"]


def t_sync():
    for c in seq[:3]:
        render_frame(scene, c, tf, params)
    t = time.perf_counter()
    for c in seq:
        render_frame(scene, c, tf, params)
    return (time.perf_counter() - t) / K * 1e3


def t_frames():
    for _ in render_frames(scene, seq[:3], tf, params):
        pass
    t = time.perf_counter()
    for _ in render_frames(scene, seq, tf, params):
        pass
    return (time.perf_counter() - t) / K * 1e3


def t_ring(depth=3):
    dev = torch.device("cuda", 0)
    sa, sb = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    imgs = [torch.empty((H, W, 4), dtype=torch.uint8, device=dev) for _ in range(2)]
    hosts = [torch.empty((H, W, 4), dtype=torch.uint8, pin_memory=True) for _ in range(depth)]
    done = [None, None]
    cevs = [None] * depth
    t = time.perf_counter()
    for k, c in enumerate(seq):
        i, h = k % 2, k % depth
        if done[i] is not None:
            sa.wait_event(done[i])
        if cevs[h] is not None:
            cevs[h].synchronize()  # the host buffer is being reused: its previous frame is consumed
        render_native(scene, c, tf, params, imgs[i].data_ptr(), stream=sa.cuda_stream, sync=False)
        e = torch.cuda.Event()
        e.record(sa)
        sb.wait_event(e)
        with torch.cuda.stream(sb):
            hosts[h].copy_(imgs[i], non_blocking=True)
        d = torch.cuda.Event()
        d.record(sb)
        done[i] = d
        cevs[h] = d
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / K * 1e3


def t_gpu():
    out = torch.empty((H, W, 4), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for c in seq:
        render_native(scene, c, tf, params, out.data_ptr(), stream=s.cuda_stream, sync=False)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / K * 1e3


for name, f in (("gpu only (device out, no L2 flush)", t_gpu), ("sync render_frame", t_sync),
                ("render_frames", t_frames), ("ring of 3 pinned", t_ring), ("sync render_frame", t_sync),
                ("render_frames", t_frames)):
    print(f"{name:40s} {f():7.3f} ms/frame", flush=True)
