"""Multi-GPU rendering: camera-batch data parallelism and spatial-block compositing.

One process per GPU over ``torch.distributed`` (NCCL on NVLink/NVSwitch; gloo
for the CPU tests).  Two ways the path shards:

1. **Camera batches** — every rank holds a full replica of the scene and
   renders its own views; no data-path collective (``camera_shard``).
   Scene replication is one ``broadcast`` at load (``broadcast_scene``).

2. **Spatial blocks** (config 5, the 50M-Gaussian city) — the scene is
   partitioned by Gaussian mean on the x-y grid with the reference's half-open
   rule (scene_manager.py:24-80; engine_api.py:182-207).  Each rank renders its
   blocks with background 0, producing premultiplied colour C_b, final
   transmittance T_b and depth D_b per pixel (5 floats).  One exchange step
   moves these images, and each pixel is composited front to back in block
   order:  C = sum_b (prod_{b'<b} T_b') C_b + (prod_b T_b) bg.
   Block order = Euclidean distance from the camera centre to the block's AABB
   centre, ties by block id (uniform grid cells are the Voronoi cells of their
   centres, so this is a valid visibility order for splats whose means lie in
   their cell).  Exchange: ``all_to_all`` by image row strips (each rank
   composites 1/N of the frame, ~1/N of the all_gather traffic), then an
   ``all_gather`` of the finished strips; ``exchange="all_gather"`` gathers
   whole block images instead (the variant the north star names).

The per-block renderer and the compositor are injectable so the exchange and
ordering logic is testable on CPU with gloo (tests/test_distributed.py); the
product path uses ``raster.render`` and the ``lmgs_composite_blocks`` kernel.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np
import torch
import torch.distributed as dist

CHANNELS = 5  # premultiplied r, g, b, transmittance, depth


# ---------------------------------------------------------------------------
# camera-batch data parallelism


def camera_shard(n_views: int, rank: int, world: int) -> range:
    """Contiguous slice of a camera batch owned by ``rank``."""
    lo = n_views * rank // world
    hi = n_views * (rank + 1) // world
    return range(lo, hi)


def broadcast_scene(tensors: Sequence[torch.Tensor], src: int = 0, group=None) -> None:
    """Replicate the scene SoA from ``src`` to every rank (one broadcast each)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    for t in tensors:
        dist.broadcast(t, src=src, group=group)


# ---------------------------------------------------------------------------
# spatial blocks


def block_of_means(means: np.ndarray, bbox: np.ndarray, grid: tuple[int, int]) -> np.ndarray:
    """Cell index iy * nx + ix of each mean, half-open bins clamped at the grid
    edge (scene_manager.py:40-46, engine_api.py:189-191)."""
    nx, ny = grid
    w = (bbox[1, 0] - bbox[0, 0]) / nx
    h = (bbox[1, 1] - bbox[0, 1]) / ny
    ix = np.clip(np.floor((means[:, 0] - bbox[0, 0]) / w).astype(np.int64), 0, nx - 1)
    iy = np.clip(np.floor((means[:, 1] - bbox[0, 1]) / h).astype(np.int64), 0, ny - 1)
    return iy * nx + ix


def block_order(camera_center: np.ndarray, block_bboxes: np.ndarray) -> list[int]:
    """Front-to-back block order: distance to each AABB centre, ties by id."""
    c = np.asarray(camera_center, dtype=np.float64).reshape(3)
    centres = 0.5 * (block_bboxes[:, 0] + block_bboxes[:, 1])
    d = np.linalg.norm(centres - c[None, :], axis=1)
    return sorted(range(len(block_bboxes)), key=lambda b: (float(d[b]), b))


def assign_blocks(n_blocks: int, world: int) -> list[list[int]]:
    """Blocks owned by each rank (round robin)."""
    return [list(range(r, n_blocks, world)) for r in range(world)]


def composite_numpy(layers: np.ndarray, order: Sequence[int], background=(0.0, 0.0, 0.0)):
    """Reference composite of (B, H, W, 5) premultiplied layers (test oracle)."""
    h, w = layers.shape[1:3]
    rgb = np.zeros((h, w, 3))
    dep = np.zeros((h, w))
    T = np.ones((h, w))
    for b in order:
        rgb += T[..., None] * layers[b, ..., :3]
        dep += T * layers[b, ..., 4]
        T = T * layers[b, ..., 3]
    rgb += T[..., None] * np.asarray(background, dtype=np.float64)
    return rgb, 1.0 - T, dep


def _composite_cuda(layers: torch.Tensor, order, background):
    from .raster import composite_blocks

    rgb = layers[..., :3].contiguous()
    trans = layers[..., 3].contiguous()
    depth = layers[..., 4].contiguous()
    return composite_blocks(rgb, trans, order, background, depth)


def render_block_layer(model, camera, tile_size=16, sh_eval_degree=3) -> torch.Tensor:
    """One block's (H, W, 5) layer: premultiplied RGB (bg 0), T_final, depth."""
    from .raster import render

    h, w = int(camera.height), int(camera.width)
    layer = torch.empty((h, w, CHANNELS), dtype=torch.float32, device=model.device)
    trans = torch.empty((h, w), dtype=torch.float32, device=model.device)
    o = render(camera, model, tile_size, (0.0, 0.0, 0.0), sh_eval_degree,
               out={"transmittance": trans})
    layer[..., :3] = o.rgb
    layer[..., 3] = trans
    layer[..., 4] = o.depth
    return layer


@dataclass
class BlockParallelRenderer:
    """Renders a block-partitioned scene across the ranks of ``group``.

    ``local_blocks``: {block_id: model} for the blocks this rank owns
    (``assign_blocks``).  ``render_fn(model, camera) -> (H, W, 5)`` and
    ``composite_fn(layers (B,H,W,5), order, background) -> (rgb, alpha, depth)``
    default to the CUDA renderer / compositor.
    """

    local_blocks: dict
    block_bboxes: np.ndarray
    n_blocks: int
    group: object = None
    exchange: str = "all_to_all"  # or "all_gather"
    render_fn: Callable | None = None
    composite_fn: Callable | None = None

    def _world(self):
        if dist.is_initialized():
            return dist.get_rank(self.group), dist.get_world_size(self.group)
        return 0, 1

    def render(self, camera, background=(0.0, 0.0, 0.0)):
        render_fn = self.render_fn or render_block_layer
        composite_fn = self.composite_fn or _composite_cuda
        rank, world = self._world()
        owned = assign_blocks(self.n_blocks, world)
        per = max(len(o) for o in owned)
        h, w = int(camera.height), int(camera.width)
        order = block_order(np.asarray(camera.center), self.block_bboxes)
        mine = owned[rank]
        layers = None
        for j, b in enumerate(mine):
            lay = render_fn(self.local_blocks[b], camera)
            if layers is None:
                layers = torch.zeros((per, h, w, CHANNELS), dtype=lay.dtype, device=lay.device)
            layers[j] = lay
        if layers is None:  # a rank without blocks contributes empty layers
            dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
                else torch.device("cpu")
            layers = torch.zeros((per, h, w, CHANNELS), dtype=torch.float32, device=dev)
            layers[..., 3] = 1.0
        for j in range(len(mine), per):  # pad slots are fully transparent
            layers[j].zero_()
            layers[j, ..., 3] = 1.0
        if world == 1:
            full = layers[: self.n_blocks]
            glob = [None] * self.n_blocks
            for j, b in enumerate(mine):
                glob[b] = j
            return composite_fn(full, [glob[b] for b in order], background)
        # slot s of rank r holds block owned[r][s]
        slot_of = {}
        for r in range(world):
            for s, b in enumerate(owned[r]):
                slot_of[b] = r * per + s
        comp_order = [slot_of[b] for b in order]
        if self.exchange == "all_gather":
            gathered = torch.empty((world * per, h, w, CHANNELS), dtype=layers.dtype,
                                   device=layers.device)
            dist.all_gather_into_tensor(gathered, layers.contiguous(), group=self.group)
            return composite_fn(gathered, comp_order, background)
        # all_to_all by row strips: rank r composites rows [r*h/world, (r+1)*h/world)
        bounds = [h * r // world for r in range(world + 1)]
        rows = bounds[1:]
        strip_h = max(rows[r] - bounds[r] for r in range(world))
        send = torch.zeros((world, per, strip_h, w, CHANNELS), dtype=layers.dtype,
                           device=layers.device)
        send[..., 3] = 1.0
        for r in range(world):
            a, b = bounds[r], bounds[r + 1]
            send[r, :, : b - a] = layers[:, a:b]
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=self.group)
        # recv[src] = src's layers for my strip -> (world*per, strip_h, w, 5)
        strip_layers = recv.reshape(world * per, strip_h, w, CHANNELS)
        s_rgb, s_alpha, s_depth = composite_fn(strip_layers, comp_order, background)
        s_rgb = torch.as_tensor(s_rgb, device=layers.device, dtype=layers.dtype)
        s_alpha = torch.as_tensor(s_alpha, device=layers.device, dtype=layers.dtype)
        s_depth = torch.as_tensor(s_depth if s_depth is not None else np.zeros(s_alpha.shape),
                                  device=layers.device, dtype=layers.dtype)
        packed = torch.cat([s_rgb, s_alpha[..., None], s_depth[..., None]], dim=-1).contiguous()
        allp = torch.empty((world * packed.shape[0],) + tuple(packed.shape[1:]),
                           dtype=packed.dtype, device=packed.device)
        dist.all_gather_into_tensor(allp, packed, group=self.group)
        allp = allp.reshape((world,) + tuple(packed.shape))
        out = torch.cat([allp[r, : bounds[r + 1] - bounds[r]] for r in range(world)], dim=0)
        return out[..., :3], out[..., 3], out[..., 4]


# ---------------------------------------------------------------------------
# spatial blocks with the exchange fused into the blend (peer memory)


def symmetric_buffers(n_floats: int, n_flags: int, group, device):
    """A symmetric-memory buffer of n_floats on every rank of ``group`` and the
    peer addresses of all ranks' buffers and signal pads (NVLink mappings)."""
    import torch.distributed._symmetric_memory as symm

    buf = symm.empty(n_floats, dtype=torch.float32, device=device)
    hdl = symm.rendezvous(buf, group)
    if hdl.signal_pad_size < 4 * n_flags:
        raise ValueError("signal pad too small for the block flags")
    symmetric_buffers.handles.append(hdl)  # keep the mappings alive
    return buf, [int(p) for p in hdl.buffer_ptrs], [int(p) for p in hdl.signal_pad_ptrs]


symmetric_buffers.handles = []


class PeerBlockRenderer:
    """Spatial-block rendering whose layer exchange happens inside the blend.

    Every rank owns a symmetric-memory receive buffer for its image strip
    (rows [r*S, (r+1)*S), S = ceil(H / world)) holding all blocks' layers:
    premultiplied RGB, T_final and depth, block-major.  A rank renders each
    of its blocks with ``lmgs_render_strips``: the blend kernel stores every
    finished pixel straight into the receive buffer of the strip's owner
    through its NVLink peer mapping, so the transfer overlaps the blend tile
    by tile and no collective moves layers.  Then it release-stores the frame
    epoch into each owner's flag for that block (``lmgs_signal_flags``).  An
    owner's stream waits for all blocks' flags (``lmgs_wait_flags``),
    composites its strip front to back (``lmgs_composite_blocks``) and
    signals "consumed" back to every producer, which waits for it before
    overwriting the buffers in the next frame.  The finished strips are
    gathered with one ``all_gather_into_tensor`` (``gather=True``).

    Signal pad words: [0, n_blocks) = block layers received, [n_blocks,
    n_blocks + world) = strip consumed by owner o.
    """

    def __init__(self, local_blocks: dict, block_bboxes: np.ndarray, n_blocks: int, width: int,
                 height: int, group=None, tile_size: int = 16, sh_eval_degree: int = 3,
                 buffers: Callable | None = None):
        """``buffers(n_floats, n_flags) -> (local buffer tensor, [peer buffer
        addresses], [peer flag-pad addresses])``; default: symmetric memory
        (``symmetric_buffers``)."""
        from .raster import context

        self.local_blocks = local_blocks
        self.block_bboxes = np.asarray(block_bboxes)
        self.n_blocks = int(n_blocks)
        self.w, self.h = int(width), int(height)
        self.group = group if group is not None else dist.group.WORLD
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        if self.world > 8:
            raise ValueError("at most 8 strips (LMGS_MAX_STRIPS)")
        self.tile_size, self.sh_eval_degree = int(tile_size), int(sh_eval_degree)
        self.strip = -(-self.h // self.world)
        self.n_strips = -(-self.h // self.strip)
        self.npix = self.strip * self.w
        self.device = torch.device("cuda", torch.cuda.current_device())
        n = self.n_blocks * self.npix * CHANNELS
        make = buffers or (lambda nf, nflag: symmetric_buffers(nf, nflag, self.group,
                                                               self.device))
        self.buf, self.peers, self.pads = make(n, self.n_blocks + self.world)
        self.epoch = 0
        self.ctx = context(self.device.index)
        dist.barrier(group=self.group)

    # byte offsets inside one receive buffer
    def _rgb_off(self, b):
        return 4 * (b * self.npix * 3)

    def _trans_off(self, b):
        return 4 * (self.n_blocks * self.npix * 3 + b * self.npix)

    def _depth_off(self, b):
        return 4 * (self.n_blocks * self.npix * 4 + b * self.npix)

    def local_layers(self):
        """(rgb (B, npix*3), trans (B, npix), depth (B, npix)) views of this
        rank's receive buffer."""
        nb, npx = self.n_blocks, self.npix
        rgb = self.buf[: nb * npx * 3].view(nb, npx * 3)
        trans = self.buf[nb * npx * 3: nb * npx * 4].view(nb, npx)
        depth = self.buf[nb * npx * 4:].view(nb, npx)
        return rgb, trans, depth

    def render(self, camera, background=(0.0, 0.0, 0.0), gather: bool = True):
        import ctypes

        from . import _lib
        from .raster import abi_camera, abi_settings, composite_blocks

        L = _lib.lib()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self.epoch += 1
        ep = self.epoch
        world, nb = self.world, self.n_blocks
        # the owners must have consumed the previous frame's layers
        _lib.check(None, L.lmgs_wait_flags(self.pads[self.rank] + 4 * nb, world,
                                           (ep - 1) & 0xFFFFFFFF, stream), "lmgs_wait_flags")
        cam = abi_camera(camera)
        st = abi_settings(self.tile_size, self.sh_eval_degree, (0.0, 0.0, 0.0))
        for b in assign_blocks(nb, world)[self.rank]:
            model = self.local_blocks[b]
            t = _lib.StripTargets()
            t.n_strips, t.strip_rows = self.n_strips, self.strip
            for o in range(self.n_strips):
                t.rgb[o] = self.peers[o] + self._rgb_off(b)
                t.trans[o] = self.peers[o] + self._trans_off(b)
                t.depth[o] = self.peers[o] + self._depth_off(b)
            g = model._abi()
            _lib.check(self.ctx.handle, L.lmgs_render_strips(
                self.ctx.handle, ctypes.byref(g), ctypes.byref(cam), ctypes.byref(st),
                ctypes.byref(t), None, stream), "lmgs_render_strips")
            flags = (ctypes.c_void_p * self.n_strips)(
                *[self.pads[o] + 4 * b for o in range(self.n_strips)])
            _lib.check(None, L.lmgs_signal_flags(flags, self.n_strips, ep, stream),
                       "lmgs_signal_flags")
        # my strip: wait for every block, composite front to back
        rgb_s, alpha_s, depth_s = None, None, None
        if self.rank < self.n_strips:
            _lib.check(None, L.lmgs_wait_flags(self.pads[self.rank], nb, ep, stream),
                       "lmgs_wait_flags")
            order = block_order(np.asarray(camera.center), self.block_bboxes)
            rgb, trans, depth = self.local_layers()
            rows = min(self.strip, self.h - self.rank * self.strip)
            c_rgb, c_alpha, c_depth = composite_blocks(
                rgb.view(nb, self.strip, self.w, 3), trans.view(nb, self.strip, self.w), order,
                background, depth.view(nb, self.strip, self.w))
            rgb_s, alpha_s, depth_s = c_rgb[:rows], c_alpha[:rows], c_depth[:rows]
        consumed = (ctypes.c_void_p * world)(*[self.pads[p] + 4 * (nb + self.rank)
                                               for p in range(world)])
        _lib.check(None, L.lmgs_signal_flags(consumed, world, ep, stream), "lmgs_signal_flags")
        if not gather:
            return rgb_s, alpha_s, depth_s
        packed = torch.zeros((self.strip, self.w, CHANNELS), dtype=torch.float32,
                             device=self.device)
        if rgb_s is not None:
            rows = rgb_s.shape[0]
            packed[:rows, :, :3] = rgb_s
            packed[:rows, :, 3] = alpha_s
            packed[:rows, :, 4] = depth_s
        allp = torch.empty((world * self.strip, self.w, CHANNELS), dtype=torch.float32,
                           device=self.device)
        dist.all_gather_into_tensor(allp, packed, group=self.group)
        out = allp[: self.h]
        return out[..., :3], out[..., 3], out[..., 4]
