"""Camera-batch renderer: many views of one device-resident scene.

The per-pose loop of the reference's render sessions (render_runtime.py:250-308,
``run_session``) batched on one device.  Each view needs one device->host read
of its instance count K; two contexts on two streams alternate views so that
while the host waits for view v's K the GPU is still sorting / blending view
v-1, keeping the device busy.  The batch joins back onto the caller's stream.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np
import torch

from . import _lib
from .raster import GaussianModel, _ptr, abi_camera, abi_settings


def tile_passes(tiles: int) -> int:
    """8-bit LSD passes of the K5 tile sort (tile ids < tiles)."""
    bits = max(int(tiles - 1).bit_length(), 1)
    return (bits + 7) // 8


def packed_tile_sort(n, tiles, tile_passes) -> bool:
    """Does the two-pass tile sort run its second pass on packed 4-byte keys
    ((tile >> 8) << id_bits | id fits 32 bits; sort.cu tile_sort)?"""
    id_bits = max(int(n - 1).bit_length(), 1)
    tile_bits = max(int(tiles - 1).bit_length(), 1)
    return tile_passes == 2 and (tile_bits - 8) + id_bits <= 32


def alg_bytes_per_view(n, s_read, group, n_vis, k, tiles, tile_passes, processed, pixels):
    """Algorithmic HBM bytes of each stage for one view (DESIGN.md §3 table).

    n Gaussians with s_read SH bytes each, inputs read once per group of views;
    n_vis visible splats; k tile instances; tile_passes 8-bit tile-sort passes;
    processed = sum over tiles of the blend's break index n_t.
    """
    return {
        # inputs 44 + S B read once per group; out 64-B record + 8-B depth bits
        # + 8-B rect + 1-B kept + 4-B touched zeroing = 85 B per Gaussian
        "preprocess": n * ((44 + s_read) / group + 85),
        # depth keys: read 8 N, write 4 N; pass 1: read 4 N keys, write 4 N keys +
        # 4 N ids (implicit payload); passes 2-3: read + write 8 N each; fix-up
        # reads the 4 N keys
        "depth_sort": n * (12 + 12 + 16 + 16 + 4),
        # ranked ids 4 B + rect gather 8 B per visible splat, 8-B key per instance
        "emit": 12 * n_vis + 8 * k,
        # each pass reads every key and writes it; the last writes the 4-B ids.
        # Two passes with packed keys (sort.cu tile_sort): 8 -> 4 B, 4 -> 4 B;
        # otherwise 8-B keys throughout; ranges 8 B per tile
        "tile_sort": (20 if packed_tile_sort(n, tiles, tile_passes) else 16 * tile_passes - 4) * k
        + 8 * tiles,
        # per processed instance a 4-B id + 64-B record; rgb, alpha, depth per
        # pixel; one range per tile; touched per Gaussian
        "blend": 68 * processed + 8 * tiles + 20 * pixels + 4 * n,
    }


class BatchRenderer:
    def __init__(self, model: GaussianModel, width: int, height: int, max_views: int,
                 tile_size: int = 16, sh_eval_degree: int = 3, background=(0.0, 0.0, 0.0),
                 with_touched: bool = True, n_streams: int = 2, group: int = 1,
                 page_mask: torch.Tensor | None = None, flags: int = 0,
                 capacity: int | None = None):
        """``capacity`` (tile instances per view) switches to the no-host-sync
        mode (LMGS_FLAG_NO_HOST_SYNC): no per-view read of K, so a batch can be
        captured in a CUDA graph (``capture``); ``overflowed()`` reports views
        whose K exceeded the capacity (their output is incomplete)."""
        self.model = model
        self.dev = model.device
        self.w, self.h, self.ts = int(width), int(height), int(tile_size)
        self.tx, self.ty = -(-self.w // self.ts), -(-self.h // self.ts)
        self.max_views = int(max_views)
        self.sh_eval_degree = int(sh_eval_degree)
        self.background = background
        self.flags = int(flags)  # extra LMGS_FLAG_*
        self.capacity = int(capacity) if capacity else 0
        if n_streams > 1:  # the streams' latency-bound sort passes share the SMs
            self.flags |= _lib.LMGS_FLAG_CONCURRENT
        if self.capacity:
            self.flags |= _lib.LMGS_FLAG_NO_HOST_SYNC
        dev = self.dev
        v = self.max_views
        self.rgb = torch.empty((v, self.h, self.w, 3), dtype=torch.float32, device=dev)
        self.alpha = torch.empty((v, self.h, self.w), dtype=torch.float32, device=dev)
        self.depth = torch.empty((v, self.h, self.w), dtype=torch.float32, device=dev)
        self.ranges = torch.empty((v, self.tx * self.ty, 2), dtype=torch.int32, device=dev)
        self.nproc = torch.empty((v, self.tx * self.ty), dtype=torch.int32, device=dev)
        n = model.count
        self.touched = torch.empty((v, n), dtype=torch.int32, device=dev) if with_touched else None
        self.kept = torch.empty((v, n), dtype=torch.uint8, device=dev)
        # group > 1: views go through lmgs_render_group `group` at a time (one
        # K1 launch reads the scene once for the whole group); n_streams sets
        # of `group` contexts/streams alternate between consecutive groups
        self.group = max(1, min(int(group), _lib.MAX_GROUP))
        nctx = n_streams * self.group
        self.ctxs = [_lib.Context(dev.index) for _ in range(nctx)]
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(nctx)]
        self.done = [torch.cuda.Event() for _ in range(n_streams)]
        self.view_done = [torch.cuda.Event() for _ in range(v)]
        self.stats = []
        self.launches_per_step = None  # liblmgs kernels per render() call (set by stage_times)
        # page_mask (device uint8 per 128-row page, as render()): rows past a
        # page's live count are culled
        self._page_mask = page_mask
        self._g = model._abi(None, page_mask, 7 if page_mask is not None else 0)

    def _frame(self, i) -> _lib.Frame:
        return _lib.Frame(_ptr(self.rgb[i]), _ptr(self.alpha[i]), _ptr(self.depth[i]), None,
                          _ptr(self.touched[i]) if self.touched is not None else None,
                          _ptr(self.kept[i]), _ptr(self.ranges[i]), _ptr(self.nproc[i]))

    def render(self, cams, stage_times: bool = False, host_rgb: torch.Tensor | None = None,
               copy_stream: torch.cuda.Stream | None = None):
        """Render len(cams) views into the batch buffers (async w.r.t. the host
        except for the per-view K read).  With ``stage_times`` the views run
        serially on one stream and per-stage CUDA-event times are summed.

        ``host_rgb`` (pinned, (V,H,W,3) fp32): each frame's D2H copy is queued on
        ``copy_stream`` right after its view is launched, so the copies overlap
        the following views' rendering instead of trailing the batch."""
        assert len(cams) <= self.max_views
        L = _lib.lib()
        caller = torch.cuda.current_stream(self.dev)
        flags = (_lib.LMGS_FLAG_STAGE_TIMES if stage_times else 0) | self.flags
        if stage_times:  # the views run serially on one stream: nothing shares the SMs
            flags &= ~_lib.LMGS_FLAG_CONCURRENT
        st = abi_settings(self.ts, self.sh_eval_degree, self.background, flags, self.capacity)
        g = self._g
        if stage_times:
            tot = {}
            inst = pairs = vis = launches = 0
            max_k = 0
            G = self.group
            for start in range(0, len(cams), G):
                idx = list(range(start, min(start + G, len(cams))))
                ctxs = self.ctxs[:len(idx)]
                self._launch(L, g, st, ctxs, [caller] * len(idx), cams, idx)
                for j, i in enumerate(idx):
                    s = ctxs[j].stats()
                    for k, v in s["stage_ms"].items():
                        tot[k] = tot.get(k, 0.0) + v
                    inst += s["n_instances"]
                    max_k = max(max_k, s["n_instances"])
                    vis += s["n_visible"]
                    launches += s["n_launches"]
                    pairs += self._pairs(i)
            self.launches_per_step = launches
            nv = len(cams)
            n = self.model.count
            s_read = int(self.model.sh.shape[1]) * 12
            k_avg = inst / nv
            v_avg = vis / nv
            pix = self.w * self.h
            t = self.tx * self.ty
            p = tile_passes(t)
            proc = self._processed_total(len(cams)) / nv
            alg = alg_bytes_per_view(n, s_read, self.group, v_avg, k_avg, t, p, proc, pix)
            return {"stage_ms": tot, "alg_bytes": alg, "launches": launches, "max_instances": max_k,
                    "per_frame": {"instances": k_avg, "visible": v_avg, "pairs": pairs / nv,
                                  "processed": proc, "tile_passes": p}}
        G = self.group
        nsets = len(self.streams) // G
        for s in self.streams:
            s.wait_stream(caller)
        for gi, start in enumerate(range(0, len(cams), G)):
            idx = list(range(start, min(start + G, len(cams))))
            base = (gi % nsets) * G
            streams = self.streams[base:base + len(idx)]
            self._launch(L, g, st, self.ctxs[base:base + len(idx)], streams, cams, idx)
            for j, i in enumerate(idx):
                self.view_done[i].record(streams[j])
                if host_rgb is not None:
                    copy_stream.wait_event(self.view_done[i])
                    with torch.cuda.stream(copy_stream):
                        host_rgb[i].copy_(self.rgb[i], non_blocking=True)
        for s in self.streams:
            caller.wait_stream(s)
        if host_rgb is not None:
            caller.wait_stream(copy_stream)
        return None

    def overflowed(self) -> bool:
        """No-sync mode: did any view since the last call exceed the instance
        capacity?  (Synchronises the device.)"""
        return any(c.stats()["overflow"] for c in self.ctxs)

    def capture(self, cams) -> torch.cuda.CUDAGraph:
        """Capture ``render(cams)`` (no-sync mode) in a CUDA graph; replay it
        with ``graph.replay()``.  One eager render first sizes every arena, so
        the captured launches never allocate or wait on the host."""
        if not self.capacity:
            raise ValueError("capture() needs the no-host-sync mode (capacity=...)")
        self.render(cams)
        torch.cuda.synchronize(self.dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self.render(cams)
        return graph

    def _launch(self, L, g, st, ctxs, streams, cams, idx):
        """Views idx on ctxs / streams: lmgs_render for one view, else one
        lmgs_render_group (shared K1 launch on streams[0])."""
        if len(idx) == 1:
            ctx, i = ctxs[0], idx[0]
            c = abi_camera(cams[i])
            fr = self._frame(i)
            _lib.check(ctx.handle, L.lmgs_render(ctx.handle, ctypes.byref(g), ctypes.byref(c),
                                                 ctypes.byref(st), ctypes.byref(fr),
                                                 streams[0].cuda_stream), "lmgs_render")
            return
        n = len(idx)
        handles = (ctypes.c_void_p * n)(*[c.handle for c in ctxs])
        cam_arr = (_lib.Camera * n)(*[abi_camera(cams[i]) for i in idx])
        frames = (_lib.Frame * n)(*[self._frame(i) for i in idx])
        sptrs = (ctypes.c_void_p * n)(*[s.cuda_stream for s in streams])
        _lib.check(ctxs[0].handle, L.lmgs_render_group(handles, n, ctypes.byref(g), cam_arr,
                                                       ctypes.byref(st), frames, sptrs),
                   "lmgs_render_group")

    def _pairs(self, i) -> float:
        """Pixel-instance pairs evaluated by the blend of view i: sum_t P_t n_t."""
        n = self.nproc[i].double()
        ts = self.ts
        # pixels per tile incl. partial edge tiles
        wx = torch.full((self.tx,), ts, dtype=torch.float64, device=self.dev)
        wx[-1] = self.w - (self.tx - 1) * ts
        wy = torch.full((self.ty,), ts, dtype=torch.float64, device=self.dev)
        wy[-1] = self.h - (self.ty - 1) * ts
        p = (wy[:, None] * wx[None, :]).reshape(-1)
        return float((n * p).sum().item())

    def _processed_total(self, nv) -> float:
        return float(self.nproc[:nv].double().sum().item())

    def bench_e2e(self, cams, steps: int, barrier=None, world: int = 1, device=None,
                  total_views: int | None = None) -> dict:
        """Frames/s through the public API with host buffers: per step the
        camera poses travel H2D (kernel parameters, from pinned host structs)
        and every RGB frame is copied D2H into pinned host memory on a copy
        stream, queued as soon as its view is launched so it overlaps the next
        views' rendering."""
        nv = len(cams)
        host = torch.empty((nv, self.h, self.w, 3), dtype=torch.float32, pin_memory=True)
        copy = torch.cuda.Stream(device=self.dev)
        caller = torch.cuda.current_stream(self.dev)

        def step():
            self.render(cams, host_rgb=host, copy_stream=copy)

        step()  # warm
        torch.cuda.synchronize()
        if barrier:
            barrier()
        t0 = time.perf_counter()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(caller)
        for _ in range(steps):
            step()
        b.record(caller)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ms = a.elapsed_time(b)
        t = torch.tensor([ms], dtype=torch.float64, device=self.dev)
        if world > 1:
            import torch.distributed as dist

            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        h2d = nv * ctypes.sizeof(_lib.Camera)
        d2h = nv * self.h * self.w * 3 * 4
        total = nv * world if total_views is None else int(total_views)
        return {"value": total * steps / (ms / 1e3), "unit": "frames/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": steps,
                "wall_s": wall,
                "path": "BatchRenderer.render (lmgs_render C-ABI) with cameras from host, "
                        "RGB frames D2H to pinned host memory each step; scene resident "
                        "(uploaded once, as the reference Engine holds its model)"}
