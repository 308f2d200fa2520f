"""Screen-tiled multi-GPU rendering (paper §5, "replicating
the data buffers on all GPUs, and assigning different GPUs to render different
regions of the image").

One process per GPU (torchrun), scene replicated on every rank (each rank runs
the deterministic GPU builders itself, so nothing is broadcast).  The frame's
16x8-pixel tiles are dealt round-robin — tile t belongs to rank t % world — so
the strongly view-dependent cost is spread evenly.  Each rank renders its
tiles into a packed buffer with the *global* pixel index feeding the jitter
hash (identical pixels to a single-GPU frame), then one NCCL all-gather (or
gather) moves the packed tiles to rank 0, which scatters them into the image
with `xb_unpack_tiles`; frame counters are summed with one all-reduce.

torch.distributed is plumbing here: NCCL over NVLink/NVSwitch on B200, gloo
for the CPU tests of the tiling logic.
"""
from __future__ import annotations

import numpy as np

from . import _native as N

TILE_W, TILE_H = 16, 8
TILE_PX = TILE_W * TILE_H


def tile_grid(width: int, height: int):
    return (width + TILE_W - 1) // TILE_W, (height + TILE_H - 1) // TILE_H


def tiles_of_rank(width: int, height: int, rank: int, world: int) -> int:
    tx, ty = tile_grid(width, height)
    total = tx * ty
    return 0 if rank >= total else (total - rank + world - 1) // world


def tiles_per_rank(width: int, height: int, world: int) -> int:
    """Gather slot size: the largest rank share (rank 0's)."""
    return tiles_of_rank(width, height, 0, world)


def packed_pixel_coords(width: int, height: int, rank: int, world: int):
    """(x, y, valid) of every slot of `rank`'s packed tile buffer — host mirror of
    the kernel's tile mapping (csrc/render.cu:k_render / k_unpack_tiles)."""
    tx, ty = tile_grid(width, height)
    n = tiles_of_rank(width, height, rank, world)
    slot = np.arange(n * TILE_PX)
    tile = rank + (slot // TILE_PX) * world
    local = slot % TILE_PX  # packed tiles are row-major 16x8 blocks
    lx, ly = local % TILE_W, local // TILE_W
    x = (tile % tx) * TILE_W + lx
    y = (tile // tx) * TILE_H + ly
    valid = (x < width) & (y < height)
    return x, y, valid


def unpack_host(packed_by_rank, width: int, height: int, world: int):
    """Host reference of `xb_unpack_tiles` for tests (packed buffers are tile-major,
    each tile row-major 16x8)."""
    img = np.zeros((height, width, 4), np.uint8)
    tx, ty = tile_grid(width, height)
    for rank, buf in enumerate(packed_by_rank):
        n = tiles_of_rank(width, height, rank, world)
        b = np.asarray(buf).reshape(-1, TILE_PX, 4)
        for t in range(n):
            tile = rank + t * world
            x0, y0 = (tile % tx) * TILE_W, (tile // tx) * TILE_H
            blk = b[t].reshape(TILE_H, TILE_W, 4)
            h, w = min(TILE_H, height - y0), min(TILE_W, width - x0)
            img[y0:y0 + h, x0:x0 + w] = blk[:h, :w]
    return img


class TiledRenderer:
    """Render one frame across all ranks of the default process group.

    Each rank renders its tiles into `packed` (global pixel index into the
    jitter hash), `exchange()` all-gathers the packed tiles (NCCL on B200,
    gloo in the CPU tests), `assemble()` scatters them into the image on rank
    0 (`xb_unpack_tiles` on the device; `unpack_host` mirrors it), and with
    `stats=True` the frame counters [regions, samples] are all-reduced — the
    multi-GPU `FrameStats` (R/render.py:684-691)."""

    def __init__(self, scene, width: int, height: int, device=None, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.group = group
        self.scene = scene
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.width, self.height = width, height
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = device
        self.slots = tiles_per_rank(width, height, self.world)
        self.n_local = tiles_of_rank(width, height, self.rank, self.world)
        self.packed = torch.zeros((self.slots * TILE_PX, 4), dtype=torch.uint8, device=self.device)
        self.gathered = torch.empty((self.world * self.slots * TILE_PX, 4), dtype=torch.uint8, device=self.device)
        self.image = torch.empty((height, width, 4), dtype=torch.uint8, device=self.device)
        self.counters = torch.zeros(3, dtype=torch.int64, device=self.device)

    def _check_camera(self, camera):
        # xb_render sizes its output from the camera: a mismatch would write past
        # (or leave holes in) the buffers allocated for width x height here
        if camera.width != self.width or camera.height != self.height:
            raise ValueError(f"camera is {camera.width}x{camera.height} but the renderer was built for "
                             f"{self.width}x{self.height}")

    def _staged(self):
        # gloo moves host memory: device buffers go through the host (CPU tests,
        # bench.py's shared-GPU check of the N > 1 path); NCCL moves them directly
        return self.packed.is_cuda and self.dist.get_backend(self.group) == "gloo"

    def exchange(self):
        """All-gather every rank's packed tiles into `gathered` (rank-major)."""
        if self.world > 1:
            if self._staged():
                out = self.torch.empty(self.gathered.shape, dtype=self.gathered.dtype)
                self.dist.all_gather_into_tensor(out, self.packed.cpu(), group=self.group)
                self.gathered.copy_(out)
            else:
                self.dist.all_gather_into_tensor(self.gathered, self.packed, group=self.group)
        return self.gathered

    def reduce_counters(self):
        """Sum [regions, samples, bytes] over the ranks (one all-reduce)."""
        if self.world > 1:
            if self._staged():
                c = self.counters.cpu()
                self.dist.all_reduce(c, group=self.group)
                self.counters.copy_(c)
            else:
                self.dist.all_reduce(self.counters, group=self.group)
        return self.counters

    def assemble(self, stream=None):
        """Rank 0: scatter the gathered tiles into `image` on the device."""
        if self.rank != 0:
            return None
        if stream is None:
            stream = self.torch.cuda.current_stream().cuda_stream
        N.check(N.lib().xb_unpack_tiles(N.ptr(self.gathered.data_ptr()), self.slots, self.world, self.width,
                                        self.height, N.ptr(self.image.data_ptr()), N.ptr(stream)))
        return self.image

    def render(self, camera, tf, params, gather=True, stats=False):
        """Render this rank's tiles; with `gather`, assemble the image on rank 0
        (device tensor on rank 0, None elsewhere).  With `stats`, returns
        (image, counters) where counters = [regions, samples, 0] summed over the
        ranks (int64 device tensor, every rank)."""
        from .render import render_native

        self._check_camera(camera)
        stream = self.torch.cuda.current_stream().cuda_stream
        dev_stats = self.counters.data_ptr() if stats else None
        if self.world == 1:
            render_native(self.scene, camera, tf, params, self.image.data_ptr(), stream=stream, sync=False,
                          dev_stats=dev_stats)
            return (self.image, self.counters) if stats else self.image
        if self.n_local:
            render_native(self.scene, camera, tf, params, self.packed.data_ptr(), tile_rank=self.rank,
                          tile_world=self.world, stream=stream, sync=False, dev_stats=dev_stats)
        elif stats:
            self.counters.zero_()
        img = None
        if gather:
            self.exchange()
            img = self.assemble(stream)
        if stats:
            self.reduce_counters()
            return img, self.counters
        return img
