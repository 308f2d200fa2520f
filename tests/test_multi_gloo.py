"""World-size-2 CPU tests of the screen-tile exchange (gloo stands in for NCCL).

Each rank fills its TiledRenderer's packed tile buffer with a deterministic
function of the global pixel index (what the kernel's global-pixel rho hash
guarantees); `TiledRenderer.exchange()` all-gathers the buffers and
`reduce_counters()` sums the frame counters, exactly as `render()` does on the
GPU, and rank 0's unpacked image must equal the single-rank frame."""
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
    from paper_2009_03076_b200.parallel import TILE_PX, TiledRenderer, packed_pixel_coords, unpack_host

    # TiledRenderer's own exchange / counter reduction on CPU tensors; the
    # device render is stood in for by writing this rank's tiles directly
    rend = TiledRenderer(scene=None, width=W, height=H, device=torch.device("cpu"))
    x, y, valid = packed_pixel_coords(W, H, rank, world)
    packed = rend.packed.numpy()
    packed[: len(x)][valid] = _pixel_value(x[valid], y[valid], W)
    rend.counters[:] = torch.tensor([int(valid.sum()), 10 * int(valid.sum()), 0])
    g = rend.exchange()
    c = rend.reduce_counters()
    if rank == 0:
        parts = g.numpy().reshape(world, rend.slots * TILE_PX, 4)
        img = unpack_host(list(parts), W, H, world)
        out_q.put((img, int(c[0]), int(c[1])))
    dist.destroy_process_group()


def _camera_check(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2009_03076_b200.parallel import TiledRenderer

    class Cam:
        width, height = 64, 32

    rend = TiledRenderer(scene=None, width=48, height=32, device=torch.device("cpu"))
    try:
        rend.render(Cam(), None, None)
        out_q.put("no error")
    except ValueError as e:
        out_q.put(str(e))
    dist.destroy_process_group()


@pytest.mark.parametrize("W,H", [(96, 40), (37, 19)])
def test_tile_gather_world2_matches_single_frame(W, H):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, W, H, q)) for r in range(2)]
    for p in procs:
        p.start()
    img, n, n10 = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    yy, xx = np.mgrid[0:H, 0:W]
    want = _pixel_value(xx.ravel(), yy.ravel(), W).reshape(H, W, 4)
    assert n == W * H and n10 == 10 * W * H  # counters summed over the ranks
    assert np.array_equal(img, want)


def test_tiled_renderer_rejects_camera_of_another_size():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_camera_check, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all("renderer was built for 48x32" in m for m in msgs), msgs
