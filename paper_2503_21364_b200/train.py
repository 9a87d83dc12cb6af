"""Backward of the blend and the training-loss gradients.

Mirrors the reference's training consumers of the forward path:

* ``backward_render`` — gaussian_core.py:438-486: exact reverse-mode
  gradients of the blend w.r.t. view colours and opacities, the screen-space
  positional gradient (densification statistics) and the touched counts;
* ``render_loss_and_grads`` — gaussian_core.py:600-629: mean-squared-error
  fit over cameras with the chain rule to SH coefficients
  (sh_color_grad_to_coeffs, 145-166) and opacity logits, plus the
  ``DensifyStats`` increments (488-511).

The device work runs in liblmgs (``lmgs_backward``): fp64, from per-view splat
records computed by K1's own fp64 code, over the tile lists of the forward
render of the same view.  Rows of the outputs are indexed by input Gaussian
(the reference's per-splat arrays are over its kept splats; rows of culled
Gaussians stay zero here).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from .errors import ShapeError
from .raster import GaussianModel, RenderOutput, _ptr, abi_camera, abi_settings, context, render


@dataclass
class RenderGrads:
    """gaussian_core.py:428-435, rows indexed by input Gaussian."""

    d_colors: torch.Tensor     # (N, 3) float64
    d_opacities: torch.Tensor  # (N,) float64
    d_mean2d: torch.Tensor     # (N, 2) float64
    touched: torch.Tensor      # (N,) int32


@dataclass
class DensifyStats:
    """gaussian_core.py:488-511 (device tensors)."""

    grad_norm_sum: torch.Tensor  # (N,) float64
    steps_seen: torch.Tensor     # (N,) int64

    @classmethod
    def zeros(cls, n: int, device) -> "DensifyStats":
        return cls(torch.zeros(n, dtype=torch.float64, device=device),
                   torch.zeros(n, dtype=torch.int64, device=device))

    def accumulate(self, grads: RenderGrads) -> None:
        seen = grads.touched > 0
        self.grad_norm_sum += torch.where(seen, grads.d_mean2d.norm(dim=-1),
                                          torch.zeros_like(self.grad_norm_sum))
        self.steps_seen += seen.to(torch.int64)

    def mean_grad(self) -> torch.Tensor:
        return self.grad_norm_sum / self.steps_seen.clamp_min(1).to(torch.float64)


def _backward(ctx, model: GaussianModel, camera, image_grad: torch.Tensor, tile_size: int,
              background, sh_eval_degree: int, d_sh=None, d_logits=None,
              stats: "DensifyStats | None" = None) -> RenderGrads:
    h, w = int(camera.height), int(camera.width)
    if tuple(image_grad.shape) != (h, w, 3):
        raise ShapeError("image gradient shape does not match forward record")
    n, dev = model.count, model.device
    g = image_grad.to(device=dev, dtype=torch.float32).contiguous()
    out = RenderGrads(torch.empty((n, 3), dtype=torch.float64, device=dev),
                      torch.empty((n,), dtype=torch.float64, device=dev),
                      torch.empty((n, 2), dtype=torch.float64, device=dev),
                      torch.empty((n,), dtype=torch.int32, device=dev))
    st = abi_settings(tile_size, sh_eval_degree, background, 0)
    cam = abi_camera(camera)
    ga = model._abi()
    s = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        _lib.check(ctx.handle, _lib.lib().lmgs_backward(
            ctx.handle, ctypes.byref(ga), ctypes.byref(cam), ctypes.byref(st), _ptr(g),
            _ptr(out.d_colors), _ptr(out.d_opacities), _ptr(out.d_mean2d), _ptr(out.touched),
            _ptr(d_sh) if d_sh is not None else None,
            _ptr(d_logits) if d_logits is not None else None,
            _ptr(stats.grad_norm_sum) if stats is not None else None,
            _ptr(stats.steps_seen) if stats is not None else None, s.cuda_stream),
            "lmgs_backward")
    return out


def backward_render(model, camera, image_grad=None, tile_size: int = 16,
                    background=(0.0, 0.0, 0.0), sh_eval_degree: int = 1):
    """backward_render (438-486) of ``image_grad``, two call forms:

    * ``backward_render(image_grad, record)`` — the reference's signature:
      ``record`` is the RenderRecord of ``render_image(..., with_record=True)``;
      returns RenderGrads with rows aligned with the record's splats
      (``record.prim_id``), like the reference's;
    * ``backward_render(model, camera, image_grad, tile_size, background,
      sh_eval_degree)`` — renders the view and returns ``(RenderOutput,
      RenderGrads)`` with rows indexed by input Gaussian.
    """
    from .raster import RenderRecord

    if isinstance(camera, RenderRecord):
        rec, g = camera, model
        m = rec._model
        if m is None:
            raise ShapeError("record has no render source (use render_image(..., with_record=True))")
        bg = tuple(float(v) for v in rec.background.tolist())
        ctx = context(m.device.index)
        render(rec._camera, m, rec.tile_size, bg, rec._sh_eval_degree, ctx=ctx,
               prim_ids=rec._prim_ids, touched_fix=False)
        full = _backward(ctx, m, rec._camera, torch.as_tensor(g), rec.tile_size, bg,
                         rec._sh_eval_degree)
        r = rec._rows
        return RenderGrads(full.d_colors[r], full.d_opacities[r], full.d_mean2d[r],
                           full.touched[r].long())
    ctx = context(model.device.index)
    fwd = render(camera, model, tile_size, background, sh_eval_degree, ctx=ctx)
    return fwd, _backward(ctx, model, camera, image_grad, tile_size, background, sh_eval_degree)


def render_loss_and_grads(model: GaussianModel, cameras, gt_images, tile_size: int = 16,
                          background=(0.0, 0.0, 0.0), sh_eval_degree: int = 1):
    """(loss, {"sh", "opacity_logits"}, DensifyStats) — gaussian_core.py:600-629."""
    n, dev = model.count, model.device
    ctx = context(dev.index)
    d_sh = torch.zeros((n, model.sh.shape[1], 3), dtype=torch.float64, device=dev)
    d_logit = torch.zeros((n,), dtype=torch.float64, device=dev)
    stats = DensifyStats.zeros(n, dev)
    loss_sum = torch.zeros((len(cameras) or 1,), dtype=torch.float64, device=dev)
    numels = []
    for i, (cam, gt) in enumerate(zip(cameras, gt_images)):
        # the loss needs the image only; the backward recounts touched exactly
        fwd = render(cam, model, tile_size, background, sh_eval_degree, ctx=ctx, touched_fix=False)
        gt_t = torch.as_tensor(gt, device=dev)
        if gt_t.dtype not in (torch.float32, torch.float64):
            gt_t = gt_t.to(torch.float64)
        gt_t = gt_t.contiguous()
        if tuple(gt_t.shape) != tuple(fwd.rgb.shape):
            raise ShapeError("ground-truth image shape does not match the camera")
        g_img = torch.empty_like(fwd.rgb)
        with torch.cuda.device(dev):
            _lib.check(None, _lib.lib().lmgs_mse_grad(
                _ptr(fwd.rgb), _ptr(gt_t), int(gt_t.dtype == torch.float64), fwd.rgb.numel(),
                _ptr(g_img), _ptr(loss_sum[i:]), torch.cuda.current_stream(dev).cuda_stream),
                "lmgs_mse_grad")
        numels.append(fwd.rgb.numel())
        _backward(ctx, model, cam, g_img, tile_size, background, sh_eval_degree, d_sh, d_logit,
                  stats)
    k = max(1, len(cameras))
    # total += mean(diff^2) per view (615-616): one device->host read per call
    per_view = loss_sum.cpu().tolist()
    total = sum(v / m for v, m in zip(per_view, numels))
    return total / k, {"sh": d_sh / k, "opacity_logits": d_logit / k}, stats
