"""The torch custom operators ``torch.ops.lmgs.render_fwd`` / ``render_image``.

Registered by ``_lmgs_torch.so`` (csrc/torch_ops.cpp, ``TORCH_LIBRARY(lmgs)``)
over the C ABI: the op boundary SURVEY.md §8(b) names for
``render_image`` (gaussian_core.py:582-597).  Visible to the dispatcher, runs
on the current CUDA stream, outputs from the caching allocator.  ``load()``
raises when the library is missing: there is no fallback.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import torch

from .camera import camera_constants
from .errors import LmgsError

OPS_PATH = Path(__file__).resolve().parent / "_lmgs_torch.so"
_loaded = False


def load():
    """Register the lmgs operators with the dispatcher (idempotent)."""
    global _loaded
    if not _loaded:
        if not OPS_PATH.exists():
            raise LmgsError(f"{OPS_PATH} is missing; run `python -m paper_2503_21364_b200.build`")
        torch.ops.load_library(str(OPS_PATH))
        _loaded = True
    return torch.ops.lmgs


def pack_camera(camera) -> torch.Tensor:
    """Host fp64 (21,) = R (9), t (3), center (3), fx, fy, cx, cy, lim_x, lim_y,
    computed on the host exactly as the reference does."""
    k = camera_constants(camera)
    v = np.concatenate([np.asarray(k["r_wc"], np.float64).reshape(9),
                        np.asarray(k["t_wc"], np.float64).reshape(3),
                        np.asarray(k["center"], np.float64).reshape(3),
                        np.array([k["fx"], k["fy"], k["cx"], k["cy"], k["lim_x"], k["lim_y"]],
                                 np.float64)])
    return torch.from_numpy(v)


def render_fwd(camera, gaussians, tile_size: int = 16, background=(0.0, 0.0, 0.0),
               sh_eval_degree: int = 3, subset=None):
    """``torch.ops.lmgs.render_fwd`` for a Camera and a device GaussianModel:
    (rgb, alpha, depth, tile_ranges, inst_keys, inst_vals, touched, n_processed)."""
    L = load()
    sub = None if subset is None else torch.as_tensor(np.asarray(subset), dtype=torch.long)
    return L.render_fwd(gaussians.means, gaussians.quats, gaussians.scales,
                        gaussians.opacity_logits, gaussians.sh, int(gaussians.sh_degree),
                        int(sh_eval_degree), pack_camera(camera), int(camera.width),
                        int(camera.height), int(tile_size),
                        [float(b) for b in np.asarray(background, np.float64).reshape(3)], sub)
