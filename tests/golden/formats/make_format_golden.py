"""Golden files for the formats either side of the rasterizer, written by the
UNMODIFIED reference (run in the build container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/formats/make_format_golden.py

* ckpt_sh3_grid.lmgs — data_io.save_gaussian_checkpoint (256-282) of 300
  Gaussians (SH degree 3) with a 3x2 SceneGrid whose block table is permuted;
* ckpt_sh1.lmgs       — 50 Gaussians, SH degree 1, no grid;
* frame_rgb8.npz      — render_runtime.encode_frame (397-401) of a float32
  image holding values on and next to the x.5/255 rounding ties, below 0 and
  above 1, plus the JSON header (the reference's exact bytes).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import torch

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from landmark.data_io import save_gaussian_checkpoint  # noqa: E402
from landmark.gaussian_core import GaussianModel  # noqa: E402
from landmark.render_runtime import encode_frame  # noqa: E402
from landmark.scene_manager import SceneGrid  # noqa: E402

from paper_2503_21364_b200 import scenes  # noqa: E402


def ref_model(n, deg, seed):
    g = scenes.synthetic_gaussians(n, seed=seed, sh_degree=deg)
    t = lambda a: torch.as_tensor(np.asarray(a, dtype=np.float64))  # noqa: E731
    return GaussianModel(means=t(g.means), quats=t(g.quats), scales=t(g.scales),
                         opacity_logits=t(g.opacity_logits), sh=t(g.sh), sh_degree=deg)


def main():
    grid = SceneGrid(bbox=np.array([[-4.0, -4.0, -1.0], [4.0, 4.0, 1.0]]), nx=3, ny=2)
    perm = [4, 0, 5, 2, 1, 3]
    grid.block_to_submodel = {(ix, iy): perm[iy * 3 + ix] for iy in range(2) for ix in range(3)}
    save_gaussian_checkpoint(ref_model(300, 3, 21), HERE / "ckpt_sh3_grid.lmgs", grid=grid)
    save_gaussian_checkpoint(ref_model(50, 1, 22), HERE / "ckpt_sh1.lmgs")

    h, w = 6, 8
    rng = np.random.default_rng(5)
    ties = (np.arange(h * w * 3) % 256 + 0.5) / 255.0
    img = ties.astype(np.float32)
    img[::5] = np.nextafter(img[::5], np.float32(2))
    img[1::7] = np.nextafter(img[1::7], np.float32(-1))
    img[2::11] = rng.uniform(-0.5, 1.5, img[2::11].shape).astype(np.float32)
    img = img.reshape(h, w, 3)
    header = {"width": w, "height": h, "frame": 7, "latency_ms": 1.25}
    payload = encode_frame(img.astype(np.float64), header)
    np.savez_compressed(HERE / "frame_rgb8.npz", image=img, payload=np.frombuffer(payload, np.uint8),
                        header=json.dumps(header))
    print("wrote", sorted(p.name for p in HERE.glob("ckpt_*.lmgs")), "frame_rgb8.npz")


if __name__ == "__main__":
    main()
