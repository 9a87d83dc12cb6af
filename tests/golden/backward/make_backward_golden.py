"""Golden outputs of the reference's backward (run in the build container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/backward/make_backward_golden.py

* backward_<case>.npz — gaussian_core.backward_render (438-486) of a seeded
  random image gradient on render_image(..., with_record=True): per kept
  splat d_colors, d_opacities, d_mean2d, touched, stored per prim id;
* loss_grads.npz — gaussian_core.render_loss_and_grads (600-629) over two
  cameras with seeded random target images: loss, d_sh, d_opacity_logits and
  the DensifyStats increments.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from landmark.data_io import Camera as RefCamera  # noqa: E402
from landmark.gaussian_core import (GaussianModel, backward_render, render_image,  # noqa: E402
                                    render_loss_and_grads)

from paper_2503_21364_b200 import scenes  # noqa: E402


def ref_model(g):
    t = lambda a: torch.as_tensor(np.asarray(a, dtype=np.float64))  # noqa: E731
    return GaussianModel(means=t(g.means), quats=t(g.quats), scales=t(g.scales),
                         opacity_logits=t(g.opacity_logits), sh=t(g.sh), sh_degree=g.sh_degree)


def ref_cam(c):
    return RefCamera(fx=c.fx, fy=c.fy, cx=c.cx, cy=c.cy, width=c.width, height=c.height,
                     r_wc=c.r_wc, t_wc=c.t_wc)


def cam_arrays(c):
    return dict(cam_fx=c.fx, cam_fy=c.fy, cam_cx=c.cx, cam_cy=c.cy, cam_w=c.width,
                cam_h=c.height, cam_r=c.r_wc, cam_t=c.t_wc)


def model_arrays(g):
    return dict(means=g.means, quats=g.quats, scales=g.scales, opacity_logits=g.opacity_logits,
                sh=g.sh, sh_degree=g.sh_degree)


def backward_case(name, n, w, h, ts, bg, seed, deg=1):
    g = scenes.synthetic_gaussians(n, seed=seed, sh_degree=deg)
    cam = scenes.orbit_cameras(1, w, h, seed=seed)[0]
    m = ref_model(g)
    img, touched, rec = render_image(m, ref_cam(cam), ts, bg, with_record=True)
    rng = np.random.default_rng(seed + 100)
    gimg = rng.normal(0.0, 1.0, (h, w, 3)).astype(np.float32)  # fp32-exact values
    grads = backward_render(torch.as_tensor(gimg.astype(np.float64)), rec)
    ids = rec.splats.prim_id.numpy()
    full = lambda a, k: np.zeros((n,) + a.shape[1:], a.dtype)  # noqa: E731
    dc, do, dm, tc = (full(grads.d_colors.numpy(), 0), full(grads.d_opacities.numpy(), 0),
                      full(grads.d_mean2d.numpy(), 0), np.zeros(n, np.int64))
    dc[ids] = grads.d_colors.numpy()
    do[ids] = grads.d_opacities.numpy()
    dm[ids] = grads.d_mean2d.numpy()
    tc[ids] = grads.touched.numpy()
    np.savez_compressed(HERE / f"backward_{name}.npz", **model_arrays(g), **cam_arrays(cam),
                        tile_size=ts, background=np.asarray(bg), image_grad=gimg, image=img.numpy(),
                        d_colors=dc, d_opacities=do, d_mean2d=dm, touched=tc)


def loss_case():
    n, w, h, ts = 300, 72, 56, 16
    g = scenes.synthetic_gaussians(n, seed=31, sh_degree=1)
    cams = scenes.orbit_cameras(2, w, h, seed=31)
    rng = np.random.default_rng(131)
    gts = [rng.uniform(0, 1, (h, w, 3)) for _ in cams]
    loss, grads, stats = render_loss_and_grads(ref_model(g), [ref_cam(c) for c in cams], gts, ts)
    extra = {}
    for i, c in enumerate(cams):
        for k, v in cam_arrays(c).items():
            extra[f"{k}_{i}"] = v
    np.savez_compressed(HERE / "loss_grads.npz", **model_arrays(g), **extra, gt0=gts[0],
                        gt1=gts[1], tile_size=ts, loss=loss, d_sh=grads["sh"].numpy(),
                        d_logits=grads["opacity_logits"].numpy(),
                        grad_norm_sum=stats.grad_norm_sum.numpy(),
                        steps_seen=stats.steps_seen.numpy())


def main():
    backward_case("ts16", 400, 80, 64, 16, (0.0, 0.0, 0.0), 41)
    backward_case("ts8_bg", 300, 70, 50, 8, (0.2, 0.5, 0.1), 42)
    backward_case("ts32", 250, 96, 64, 32, (0.1, 0.1, 0.1), 43)
    loss_case()
    print("wrote", sorted(p.name for p in HERE.glob("backward_*.npz")), "loss_grads.npz")


if __name__ == "__main__":
    main()
