"""World-size-2 CPU test of the screen-tile exchange (gloo stands in for NCCL).

Each rank fills its packed tile buffer with a deterministic function of the
global pixel index (what the kernel's global-pixel rho hash guarantees), the
buffers are all-gathered exactly as `TiledRenderer.render` does, and rank 0's
unpacked image must equal the single-rank frame."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pixel_value(x, y, W):
    pix = (y.astype(np.int64) * W + x).astype(np.uint64)
    v = (pix * np.uint64(2654435761)) >> np.uint64(7)
    return np.stack([(v >> np.uint64(s)) & np.uint64(255) for s in (0, 8, 16, 24)], -1).astype(np.uint8)


def _worker(rank, world, port, W, H, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2009_03076_b200.parallel import TILE_PX, packed_pixel_coords, tiles_per_rank, unpack_host

    slots = tiles_per_rank(W, H, world)
    packed = np.zeros((slots * TILE_PX, 4), np.uint8)
    x, y, valid = packed_pixel_coords(W, H, rank, world)
    packed[: len(x)][valid] = _pixel_value(x[valid], y[valid], W)
    t = torch.from_numpy(packed)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    counts = torch.tensor([int(valid.sum())], dtype=torch.int64)
    dist.all_reduce(counts)
    if rank == 0:
        img = unpack_host([p.numpy() for p in parts], W, H, world)
        out_q.put((img, int(counts.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("W,H", [(96, 40), (37, 19)])
def test_tile_gather_world2_matches_single_frame(W, H):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, W, H, q)) for r in range(2)]
    for p in procs:
        p.start()
    img, n = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    yy, xx = np.mgrid[0:H, 0:W]
    want = _pixel_value(xx.ravel(), yy.ravel(), W).reshape(H, W, 4)
    assert n == W * H
    assert np.array_equal(img, want)
