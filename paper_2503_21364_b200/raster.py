"""Host-side operator API: the reference's render entry points over liblmgs.

Mirrors pkg/src/landmark/gaussian_core.py:
  * ``GaussianModel``   (34-90)  — device-resident fp32 SoA, same validation;
  * ``render_image``    (582-597) — same signature and return tuple
                                    ``(image, touched[, record])``;
  * ``render``          — the north-star ``render(camera, gaussians)``
                          operator returning every output buffer (RGB, alpha,
                          depth, T_final, per-tile ranges and instance lists).

Torch is used for device memory and the current stream only; every compute
stage runs in liblmgs.so (hand-written sm_100a kernels).  There is no CPU
fallback: without a CUDA device or the library these functions raise.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .camera import Camera, camera_constants
from .errors import InvalidInputError, ShapeError

_CONTEXTS: dict = {}


def context(device: int | None = None, stream=None) -> _lib.Context:
    """The context of (device, stream): a context's arenas are stream-ordered,
    so concurrent streams never share one (lmgs.h threading rule)."""
    if device is None:
        device = torch.cuda.current_device()
    if stream is None:
        stream = torch.cuda.current_stream(device)
    key = (int(device), int(stream.cuda_stream))
    ctx = _CONTEXTS.get(key)
    if ctx is None:
        ctx = _CONTEXTS[key] = _lib.Context(device)
    return ctx


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream_handle(stream) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


# ---------------------------------------------------------------------------
# primitives


class GaussianModel:
    """Device-resident Gaussian set (fp32 SoA), validated like the reference.

    means (N,3), quats (N,4) unit (w,x,y,z), scales (N,3) > 0, opacity_logits
    (N,), sh (N,(deg+1)^2,3) — gaussian_core.py:34-61.
    """

    def __init__(self, means, quats, scales, opacity_logits, sh, sh_degree: int = 1,
                 device=None, validate: bool = True):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else \
            torch.device(device)

        def dev_f32(x):
            t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
            return t.to(device=dev, dtype=torch.float32).contiguous()

        self.means = dev_f32(means).reshape(-1, 3)
        n = self.means.shape[0]
        self.quats = dev_f32(quats).reshape(n, 4)
        self.scales = dev_f32(scales).reshape(n, 3)
        self.opacity_logits = dev_f32(opacity_logits).reshape(n)
        sh_t = dev_f32(sh)
        self.sh_degree = int(sh_degree)
        if sh_t.ndim != 3 or sh_t.shape[0] != n or sh_t.shape[2] != 3:
            raise ShapeError("sh must be (N, (deg+1)^2, 3)")
        self.sh = sh_t
        if validate:
            if n and not bool(torch.all(self.scales > 0)):
                raise InvalidInputError("scales must be positive")
            norms = self.quats.double().norm(dim=-1)
            if n and not torch.allclose(norms, torch.ones_like(norms), atol=1e-5):
                raise InvalidInputError("quaternions must be unit norm")
            if self.sh.shape[1] != (self.sh_degree + 1) ** 2:
                raise ShapeError("SH coefficient count does not match degree")

    @classmethod
    def from_host(cls, g, device=None, validate: bool = True) -> "GaussianModel":
        """From a ``scenes.HostGaussians`` or a reference ``GaussianModel``."""
        return cls(g.means, g.quats, g.scales, g.opacity_logits, g.sh, int(g.sh_degree),
                   device=device, validate=validate)

    @property
    def count(self) -> int:
        return int(self.means.shape[0])

    @property
    def device(self) -> torch.device:
        return self.means.device

    def subset(self, idx) -> "GaussianModel":
        idx = torch.as_tensor(np.asarray(idx), dtype=torch.long, device=self.device)
        return GaussianModel(self.means[idx], self.quats[idx], self.scales[idx],
                             self.opacity_logits[idx], self.sh[idx], self.sh_degree,
                             device=self.device, validate=False)

    def nbytes(self) -> int:
        return sum(t.numel() * 4 for t in (self.means, self.quats, self.scales,
                                           self.opacity_logits, self.sh))

    def _abi(self, prim_ids=None, page_mask=None, page_shift: int = 0) -> _lib.Gaussians:
        g = _lib.Gaussians()
        g.means, g.quats, g.scales = _ptr(self.means), _ptr(self.quats), _ptr(self.scales)
        g.opacity_logits, g.sh = _ptr(self.opacity_logits), _ptr(self.sh)
        g.prim_ids = _ptr(prim_ids)
        g.page_mask = _ptr(page_mask)
        g.page_shift = int(page_shift)
        g.count = self.count
        g.sh_degree = self.sh_degree
        g.sh_coeffs = int(self.sh.shape[1])
        return g


def abi_camera(cam) -> _lib.Camera:
    k = camera_constants(cam)
    c = _lib.Camera()
    c.r_wc[:] = list(k["r_wc"].reshape(9))
    c.t_wc[:] = list(k["t_wc"])
    c.center[:] = list(k["center"])
    c.fx, c.fy, c.cx, c.cy = k["fx"], k["fy"], k["cx"], k["cy"]
    c.lim_x, c.lim_y = k["lim_x"], k["lim_y"]
    c.width, c.height = k["width"], k["height"]
    return c


def abi_settings(tile_size, sh_eval_degree, background, flags=0,
                 max_instances: int = 0) -> _lib.Settings:
    s = _lib.Settings()
    s.tile_size = int(tile_size)
    s.sh_eval_degree = int(sh_eval_degree)
    bg = [float(v) for v in np.asarray(background, dtype=np.float64).reshape(3)]
    s.background[:] = bg
    s.flags = int(flags)
    s.max_instances = int(max_instances)
    return s


# ---------------------------------------------------------------------------
# outputs


@dataclass
class Splat2DBatch:
    """Screen-space splats after culling (gaussian_core.py:173-184), fp64 on
    the host, aligned arrays of length M in the reference's order: means2d
    (M,2), cov2d (M,2,2) incl. the 0.3 floor, depth (M,), radius_px (M,),
    prim_id (M,) original ids.  Values are K1's fp64 geometry, bit-equal to
    the reference's project_splats."""

    means2d: torch.Tensor
    cov2d: torch.Tensor
    depth: torch.Tensor
    radius_px: torch.Tensor
    prim_id: torch.Tensor

    def __len__(self) -> int:
        return int(self.means2d.shape[0])


@dataclass
class TileRecord:
    """Per-tile record, fields as gaussian_core.py:256-263.

    ``order`` indexes the record's splats (the reference's Splat2DBatch
    order).  With ``collect`` (``render_image(..., with_record=True)`` on
    small frames) ``sigma`` / ``t_before`` are the fp64 (K_t, P_t) blend
    tensors ``_blend`` collects (306-322, no early break) and ``t_final`` is
    fp64; otherwise ``sigma`` / ``t_before`` are ``None`` and ``t_final`` is
    the fp32 blend's transmittance.
    """

    pix_xy: torch.Tensor
    pix_idx: torch.Tensor
    order: torch.Tensor
    t_final: torch.Tensor
    sigma: torch.Tensor | None = None
    t_before: torch.Tensor | None = None


@dataclass
class RenderRecord:
    """Render bookkeeping (gaussian_core.py:266-274) on the host: the
    reference's fields (splats, colors, opacities, background, width, height,
    tiles) plus the device pipeline's own (tile ranges, instance keys,
    n_processed)."""

    width: int
    height: int
    tile_size: int
    background: torch.Tensor
    prim_id: torch.Tensor         # (M,) original id of each kept splat
    tile_ranges: torch.Tensor     # (T,2)
    inst_prim_ids: torch.Tensor   # (K,) prim id per tile instance, per-tile lists concatenated
    inst_keys: torch.Tensor       # (K,) tile << 32 | input row
    t_final: torch.Tensor         # (H,W) fp64 with collect, else the fp32 blend's
    n_processed: torch.Tensor     # (T,)
    splats: Splat2DBatch | None = None
    colors: torch.Tensor | None = None     # (M,3) fp64 view colours (clamped SH)
    opacities: torch.Tensor | None = None  # (M,) fp64 sigmoid(logit)
    _sigma: torch.Tensor | None = field(default=None, repr=False)     # flat, per tile blocks
    _t_before: torch.Tensor | None = field(default=None, repr=False)
    _offsets: np.ndarray | None = field(default=None, repr=False)     # per tile block start
    _tiles: list = field(default=None, repr=False)
    # what the render drew, so train.backward_render(image_grad, record) can
    # replay it (the reference's backward_render signature, 438)
    _model: object = field(default=None, repr=False)
    _camera: object = field(default=None, repr=False)
    _prim_ids: object = field(default=None, repr=False)
    _rows: object = field(default=None, repr=False)  # model row of each record splat
    _sh_eval_degree: int = field(default=1, repr=False)

    @property
    def tiles(self) -> list:
        if self._tiles is None:
            self._tiles = _build_tiles(self)
        return self._tiles


def _build_tiles(rec: RenderRecord) -> list:
    ts, w, h = rec.tile_size, rec.width, rec.height
    pos = {int(p): i for i, p in enumerate(rec.prim_id.tolist())}
    ranges = rec.tile_ranges.cpu().numpy()
    inst = rec.inst_prim_ids.cpu().numpy()
    tf = rec.t_final.reshape(-1)
    tiles = []
    t = 0
    for ty in range(0, h, ts):
        for tx in range(0, w, ts):
            xs = torch.arange(tx, min(tx + ts, w))
            ys = torch.arange(ty, min(ty + ts, h))
            yy, xx = torch.meshgrid(ys.double() + 0.5, xs.double() + 0.5, indexing="ij")
            pix_xy = torch.stack([xx.reshape(-1), yy.reshape(-1)], dim=-1)
            pix_idx = (ys[:, None] * w + xs[None, :]).reshape(-1)
            a, b = int(ranges[t, 0]), int(ranges[t, 1])
            order = torch.as_tensor([pos[int(p)] for p in inst[a:b]], dtype=torch.long)
            sig = tb = None
            if rec._sigma is not None:
                o, k, p = int(rec._offsets[t]), b - a, int(pix_idx.numel())
                sig = rec._sigma[o:o + k * p].reshape(k, p)
                tb = rec._t_before[o:o + k * p].reshape(k, p)
            tiles.append(TileRecord(pix_xy, pix_idx, order, tf[pix_idx].double(), sig, tb))
            t += 1
    return tiles


@dataclass
class RenderOutput:
    """Every buffer of one view (device tensors)."""

    rgb: torch.Tensor             # (H,W,3) f32
    alpha: torch.Tensor           # (H,W)   f32, 1 - T_final
    depth: torch.Tensor           # (H,W)   f32, sum w z
    transmittance: torch.Tensor | None  # (H,W) T_final
    tile_ranges: torch.Tensor     # (T,2) i32
    touched: torch.Tensor         # (N,)  i32, per input Gaussian (0 if culled)
    kept: torch.Tensor            # (N,)  u8
    n_processed: torch.Tensor     # (T,)  i32
    n_instances: int
    n_kept: int
    inst_keys: torch.Tensor | None = None      # (K,) i64 (tile << 32 | input row)
    inst_prim_ids: torch.Tensor | None = None  # (K,) i64
    stats: dict | None = None


def render(camera, gaussians: GaussianModel, tile_size: int = 16, background=(0.0, 0.0, 0.0),
           sh_eval_degree: int = 3, with_instances: bool = False, stage_times: bool = False,
           prim_ids: torch.Tensor | None = None, stream=None, ctx=None,
           out: dict | None = None, page_mask: torch.Tensor | None = None,
           page_shift: int = 7, touched_fix: bool = True,
           wide_fix_band: bool = False, fused_tile_sort: bool = False) -> RenderOutput:
    """Render one view of device-resident Gaussians (north-star operator).

    ``prim_ids`` (int64, optional) are the original ids used for depth-tie
    breaking and reported in ``inst_prim_ids`` (render_image's ``subset``).
    ``out`` may pre-supply output tensors (e.g. slices of a batch buffer)
    under the RenderOutput field names.  ``touched_fix=False`` skips the
    fp64 replay that makes ``touched`` exact (K7b); ``wide_fix_band`` replays
    every pixel within 1e-2 of TERM_EPS instead of 1e-4 (a check of the band);
    ``fused_tile_sort`` builds the tile lists with the fused emission + tile
    sort where it applies (identical lists; see LMGS_FLAG_FUSED_TILE_SORT).  ``page_mask`` (device uint8 per
    128-row page: its number of live leading rows, 0..128) restricts the
    render to those rows (the paged device pool of ``offload``).
    """
    if not isinstance(gaussians, GaussianModel):
        raise InvalidInputError("gaussians must be a GaussianModel (device SoA)")
    if int(tile_size) < 1:
        raise InvalidInputError("tile_size must be >= 1")
    dev = gaussians.device
    if ctx is None:
        ctx = context(dev.index, stream if stream is not None else torch.cuda.current_stream(dev))
    w, h = int(camera.width), int(camera.height)
    ts = int(tile_size)
    tx, ty = -(-w // ts), -(-h // ts)
    n = gaussians.count
    out = {} if out is None else out

    def buf(name, shape, dtype):
        t = out.get(name)
        if t is None:
            t = torch.empty(shape, dtype=dtype, device=dev)
        return t

    rgb = buf("rgb", (h, w, 3), torch.float32)
    alpha = buf("alpha", (h, w), torch.float32)
    depth = buf("depth", (h, w), torch.float32)
    trans = out.get("transmittance")
    ranges = buf("tile_ranges", (tx * ty, 2), torch.int32)
    touched = buf("touched", (n,), torch.int32)
    kept = buf("kept", (n,), torch.uint8)
    nproc = buf("n_processed", (tx * ty,), torch.int32)
    if prim_ids is not None:
        prim_ids = prim_ids.to(device=dev, dtype=torch.int64).contiguous()
    fr = _lib.Frame(_ptr(rgb), _ptr(alpha), _ptr(depth), _ptr(trans), _ptr(touched), _ptr(kept),
                    _ptr(ranges), _ptr(nproc))
    if page_mask is not None and (page_mask.dtype != torch.uint8 or page_mask.device != dev
                                  or page_mask.numel() < -(-n // (1 << int(page_shift)))):
        raise InvalidInputError("page_mask must be a device uint8 tensor covering every page")
    g = gaussians._abi(prim_ids, page_mask, page_shift if page_mask is not None else 0)
    cam = abi_camera(camera)
    st = abi_settings(ts, sh_eval_degree, background,
                      (_lib.LMGS_FLAG_STAGE_TIMES if stage_times else 0)
                      | (0 if touched_fix else _lib.LMGS_FLAG_NO_TOUCHED_FIX)
                      | (_lib.LMGS_FLAG_WIDE_FIX_BAND if wide_fix_band else 0)
                      | (_lib.LMGS_FLAG_FUSED_TILE_SORT if fused_tile_sort else 0))
    sh = _stream_handle(stream)
    L = _lib.lib()
    with torch.cuda.device(dev):
        _lib.check(ctx.handle, L.lmgs_render(ctx.handle, ctypes.byref(g), ctypes.byref(cam),
                                             ctypes.byref(st), ctypes.byref(fr), sh),
                   "lmgs_render")
        stats = ctx.stats() if stage_times else None
        k = stats["n_instances"] if stats else ctx.stats()["n_instances"]
        m = ctx.stats()["n_kept"] if stats is None else stats["n_kept"]
        keys = prims = None
        if with_instances:
            keys = torch.empty(k, dtype=torch.int64, device=dev)
            prims = torch.empty(k, dtype=torch.int64, device=dev)
            _lib.check(ctx.handle, L.lmgs_copy_instances(ctx.handle, _ptr(keys), _ptr(prims), sh),
                       "lmgs_copy_instances")
    return RenderOutput(rgb, alpha, depth, trans, ranges, touched, kept, nproc, int(k), int(m),
                        keys, prims, stats)


COLLECT_MAX_BYTES = 1 << 30  # sigma + t_before of a record (fp64), auto mode


def render_image(model, camera, tile_size: int = 16, background=(0.0, 0.0, 0.0),
                 with_record: bool = False, subset=None, sh_eval_degree: int = 1,
                 collect: bool | None = None):
    """Drop-in for ``landmark.gaussian_core.render_image`` (582-597).

    Returns ``(image (H,W,3), touched (M,) int64[, RenderRecord])`` with
    ``image`` an fp32 CUDA tensor.  ``model`` may be a ``GaussianModel``, a
    ``scenes.HostGaussians`` or the reference's model (uploaded each call;
    keep a ``GaussianModel`` to render one model many times).
    ``sh_eval_degree=1`` reproduces the reference's eval_sh_colors.

    The record carries the reference's fields: ``splats`` (fp64 Splat2DBatch),
    ``colors``, ``opacities``, ``background``, ``width``, ``height`` and
    ``tiles``.  ``collect`` materialises every tile's fp64 ``sigma`` /
    ``t_before`` (K_t, P_t) and fp64 ``t_final`` like the reference's
    ``rasterize(collect=True)`` (``lmgs_record_collect``); ``None`` = when
    they fit in ``COLLECT_MAX_BYTES``.
    """
    if not isinstance(model, GaussianModel):
        model = GaussianModel.from_host(model)
    cam = camera if isinstance(camera, Camera) else Camera.from_reference(camera)
    prim_ids = None
    inv = None
    src = model
    if subset is not None:
        ids = np.asarray(subset, dtype=np.int64).reshape(-1)
        order = np.argsort(ids, kind="stable")
        src = model.subset(ids[order])
        prim_ids = torch.as_tensor(ids[order], device=model.device)
        inv = torch.as_tensor(order, device=model.device)
    extra = {}
    if with_record:
        extra["transmittance"] = torch.empty((cam.height, cam.width), dtype=torch.float32,
                                             device=model.device)
    o = render(cam, src, tile_size, background, sh_eval_degree, with_instances=with_record,
               prim_ids=prim_ids, out=extra)
    touched, kept = o.touched.long(), o.kept.bool()
    if inv is not None:  # back to the caller's subset order
        t2 = torch.empty_like(touched)
        t2[inv] = touched
        k2 = torch.empty_like(kept)
        k2[inv] = kept
        touched, kept = t2, k2
        src_ids = torch.as_tensor(np.asarray(subset, dtype=np.int64), device=model.device)
    else:
        src_ids = torch.arange(model.count, device=model.device)
    touched_m = touched[kept]
    if not with_record:
        return o.rgb, touched_m
    kept_pos = torch.nonzero(kept).reshape(-1)
    rows = kept_pos if inv is None else torch.argsort(inv)[kept_pos]
    # splats: K1's fp64 geometry of the kept rows, in the reference's order
    pj = project(cam, src, sh_eval_degree=sh_eval_degree)
    c = pj["cov2d"][rows]
    cov = torch.stack([torch.stack([c[:, 0], c[:, 1]], -1), torch.stack([c[:, 1], c[:, 2]], -1)],
                      -2)
    splats = Splat2DBatch(pj["mean2d"][rows].cpu(), cov.cpu(), pj["depth"][rows].cpu(),
                          pj["radius"][rows].cpu(), src_ids[kept].cpu())
    ranges = o.tile_ranges.cpu().numpy().astype(np.int64)
    ts = int(tile_size)
    tx, ty = -(-cam.width // ts), -(-cam.height // ts)
    tw = np.minimum(ts, cam.width - np.arange(tx) * ts)
    th = np.minimum(ts, cam.height - np.arange(ty) * ts)
    pix = (th[:, None] * tw[None, :]).reshape(-1)
    blocks = (ranges[:, 1] - ranges[:, 0]) * pix
    offsets = np.concatenate([[0], np.cumsum(blocks)])
    if collect is None:
        collect = 16 * int(offsets[-1]) <= COLLECT_MAX_BYTES
    sigma = t_before = None
    colors = opac = None
    t_final = o.transmittance.double().cpu()
    if collect:
        sigma, t_before, t_final64, col64, op64 = _collect(src, cam, ts, background,
                                                           sh_eval_degree, prim_ids, offsets)
        t_final = t_final64.cpu()
        sigma, t_before = sigma.cpu(), t_before.cpu()
        colors, opac = col64[rows].cpu(), op64[rows].cpu()
    else:  # the fp32 view colours / opacities of K1
        colors, opac = pj["colors"][rows].double().cpu(), pj["opacity"][rows].double().cpu()
    rec = RenderRecord(cam.width, cam.height, ts,
                       torch.as_tensor(np.asarray(background, dtype=np.float64)),
                       src_ids[kept].cpu(), o.tile_ranges.cpu(), o.inst_prim_ids.cpu(),
                       o.inst_keys.cpu(), t_final, o.n_processed.cpu(),
                       splats=splats, colors=colors, opacities=opac, _sigma=sigma,
                       _t_before=t_before, _offsets=offsets if collect else None,
                       _model=src, _camera=cam, _prim_ids=prim_ids, _rows=rows,
                       _sh_eval_degree=int(sh_eval_degree))
    return o.rgb, touched_m, rec


def _collect(model, cam, tile_size, background, sh_eval_degree, prim_ids, offsets):
    """lmgs_record_collect for the view just rendered on the current
    context: flat fp64 sigma / t_before, fp64 t_final (H,W), per-row fp64
    colours and opacities."""
    dev = model.device
    ctx = context(dev.index, torch.cuda.current_stream(dev))
    total = int(offsets[-1])
    sigma = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
    t_before = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
    t_final = torch.empty((cam.height, cam.width), dtype=torch.float64, device=dev)
    colors = torch.empty((model.count, 3), dtype=torch.float64, device=dev)
    opac = torch.empty(model.count, dtype=torch.float64, device=dev)
    offs = torch.as_tensor(offsets[:-1], dtype=torch.int64, device=dev)
    g = model._abi(prim_ids)
    c = abi_camera(cam)
    st = abi_settings(tile_size, sh_eval_degree, background)
    with torch.cuda.device(dev):
        _lib.check(ctx.handle, _lib.lib().lmgs_record_collect(
            ctx.handle, ctypes.byref(g), ctypes.byref(c), ctypes.byref(st), _ptr(offs),
            _ptr(sigma), _ptr(t_before), _ptr(t_final), _ptr(colors), _ptr(opac),
            _stream_handle(None)), "lmgs_record_collect")
    return sigma[:total], t_before[:total], t_final, colors, opac


def project(camera, gaussians: GaussianModel, sh_eval_degree: int = 1, stream=None) -> dict:
    """Stage K1 alone (project_splats, 187-230): fp64 geometry per Gaussian."""
    dev = gaussians.device
    ctx = context(dev.index, stream if stream is not None else torch.cuda.current_stream(dev))
    n = gaussians.count
    mean2d = torch.empty((n, 2), dtype=torch.float64, device=dev)
    cov2d = torch.empty((n, 3), dtype=torch.float64, device=dev)
    depth = torch.empty(n, dtype=torch.float64, device=dev)
    radius = torch.empty(n, dtype=torch.float64, device=dev)
    colors = torch.empty((n, 3), dtype=torch.float32, device=dev)
    opac = torch.empty(n, dtype=torch.float32, device=dev)
    kept = torch.empty(n, dtype=torch.uint8, device=dev)
    g = gaussians._abi()
    cam = abi_camera(camera)
    st = abi_settings(16, sh_eval_degree, (0, 0, 0))
    with torch.cuda.device(dev):
        _lib.check(ctx.handle, _lib.lib().lmgs_project(
            ctx.handle, ctypes.byref(g), ctypes.byref(cam), ctypes.byref(st), _ptr(mean2d),
            _ptr(cov2d), _ptr(depth), _ptr(radius), _ptr(colors), _ptr(opac), _ptr(kept),
            _stream_handle(stream)), "lmgs_project")
    return dict(mean2d=mean2d, cov2d=cov2d, depth=depth, radius=radius, colors=colors,
                opacity=opac, kept=kept.bool())


def composite_blocks(rgb: torch.Tensor, trans: torch.Tensor, order, background=(0.0, 0.0, 0.0),
                     depth: torch.Tensor | None = None, stream=None):
    """Front-to-back composite of B premultiplied block renders.

    rgb (B,H,W,3), trans (B,H,W) = per-block T_final (background 0), order =
    front-to-back block indices.  Returns (rgb (H,W,3), alpha (H,W), depth or None).
    """
    b, h, w = trans.shape
    out_rgb = torch.empty((h, w, 3), dtype=torch.float32, device=rgb.device)
    out_alpha = torch.empty((h, w), dtype=torch.float32, device=rgb.device)
    out_depth = torch.empty((h, w), dtype=torch.float32, device=rgb.device) if depth is not None \
        else None
    order_np = np.ascontiguousarray(np.asarray(order, dtype=np.int32))
    bg = np.ascontiguousarray(np.asarray(background, dtype=np.float32).reshape(3))
    # contiguous copies stay bound until the kernel is enqueued on `stream`;
    # the caching allocator then orders their reuse after it
    rgb_c, trans_c = rgb.contiguous(), trans.contiguous()
    depth_c = depth.contiguous() if depth is not None else None
    st = _lib.lib().lmgs_composite_blocks(
        _ptr(rgb_c), _ptr(trans_c), _ptr(depth_c), int(b), order_np.ctypes.data,
        h * w, bg.ctypes.data, _ptr(out_rgb), _ptr(out_alpha), _ptr(out_depth),
        _stream_handle(stream))
    cur = torch.cuda.current_stream(rgb.device) if stream is None else stream
    for t in (rgb_c, trans_c, depth_c):
        if t is not None:
            t.record_stream(cur)
    _lib.check(None, st, "lmgs_composite_blocks")
    return out_rgb, out_alpha, out_depth
