"""Deterministic synthetic Gaussian clouds and camera sets for the benchmark configs.

The distribution extends the reference's ``generate_synthetic_scene``
(pkg/src/landmark/data_io.py:369-417) as specified in SURVEY.md §8d:

* the RNG is the reference's splittable PCG64 ``make_rng(seed, *path)``
  (pkg/src/landmark/common.py:34-42), restated here;
* means / quats / scales / logits / SH-DC are drawn in exactly the reference's
  order and dtype (f32), so for N <= 1e4 the first five arrays equal the
  reference generator's output bit for bit; the degree-1..3 SH coefficients
  are drawn afterwards (U(-0.1, 0.1)), and for N > 1e4 scales shrink by
  s(N) = (1e4 / N)^(1/3) so the tile-instance count stays ~3.5-7 per Gaussian;
* cameras follow the reference orbit (radius 2.6e, height 0.9 radius, fov 70°).

Configs (BASELINE.json ``configs``):
  c1  10k, SH3, 256x256, one view                     (the CPU reference runs it)
  c2  1M, 1920x1080, one view
  c3  6M, 1080p, 64 views (camera-batch data parallel) <- the bench workload
  c4  6M, 3840x2160, one view
  c5  50M city: 8 blocks (4x2 grid) x 6.25M, 1080p, block-parallel composite
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .camera import Camera, look_at_camera
from .errors import InvalidInputError


def make_rng(seed: int, *path: str) -> np.random.Generator:
    """PCG64 keyed by a root seed plus a string path (common.py:34-42)."""
    keys = [seed] + [int.from_bytes(p.encode(), "little") % (2**32) for p in path]
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(keys)))


@dataclass
class HostGaussians:
    """Host-side SoA Gaussian set (f32), the layout the C-ABI consumes.

    means (N,3), quats (N,4) unit (w,x,y,z), scales (N,3) > 0 (linear, not log),
    opacity_logits (N,), sh (N,(deg+1)^2,3).  Same fields as the reference's
    ``GaussianModel`` (gaussian_core.py:34-61).
    """

    means: np.ndarray
    quats: np.ndarray
    scales: np.ndarray
    opacity_logits: np.ndarray
    sh: np.ndarray
    sh_degree: int = 3

    @property
    def count(self) -> int:
        return int(self.means.shape[0])

    def subset(self, idx) -> "HostGaussians":
        idx = np.asarray(idx, dtype=np.int64)
        return HostGaussians(self.means[idx], self.quats[idx], self.scales[idx],
                             self.opacity_logits[idx], self.sh[idx], self.sh_degree)

    def nbytes(self) -> int:
        return sum(a.nbytes for a in (self.means, self.quats, self.scales, self.opacity_logits,
                                      self.sh))


def scale_factor(n: int) -> float:
    return 1.0 if n <= 10_000 else (1e4 / n) ** (1.0 / 3.0)


def _draw_gaussians(rng, n, lo, hi, extent, s, sh_degree):
    means = rng.uniform(lo, hi, (n, 3)).astype(np.float32)
    quats = rng.standard_normal((n, 4)).astype(np.float32)
    quats /= np.linalg.norm(quats, axis=1, keepdims=True).astype(np.float32)
    scales = rng.uniform(0.05, 0.25, (n, 3)).astype(np.float32) * extent / 4.0
    if s != 1.0:
        scales = (scales * np.float32(s)).astype(np.float32)
    logits = rng.uniform(-1.0, 2.0, n).astype(np.float32)
    nc = (sh_degree + 1) ** 2
    sh = np.zeros((n, nc, 3), dtype=np.float32)
    sh[:, 0, :] = rng.uniform(0.1, 3.0, (n, 3)).astype(np.float32)
    if nc > 1:
        sh[:, 1:, :] = rng.uniform(-0.1, 0.1, (n, nc - 1, 3)).astype(np.float32)
    return HostGaussians(means, quats, scales.astype(np.float32), logits, sh, sh_degree)


def synthetic_gaussians(n: int, seed: int = 0, extent: float = 4.0, sh_degree: int = 3,
                        scale_mult: float | None = None) -> HostGaussians:
    """The SURVEY §8d cloud: means in [-e,e]x[-e,e]x[-e/4,e/4]."""
    if n < 0:
        raise InvalidInputError("n must be >= 0")
    rng = make_rng(seed, "scene")
    s = scale_factor(n) if scale_mult is None else scale_mult
    return _draw_gaussians(rng, n, [-extent, -extent, -extent / 4], [extent, extent, extent / 4],
                           extent, s, sh_degree)


def orbit_cameras(n_views: int, width: int, height: int, seed: int = 0, extent: float = 4.0,
                  radius_mult: float = 2.6, fov_deg: float = 70.0) -> list[Camera]:
    """Reference orbit (data_io.py:399-408) with ``n_views`` views."""
    cam_rng = make_rng(seed, "cameras")
    radius = radius_mult * extent
    cams = []
    for i in range(n_views):
        ang = 2 * np.pi * i / n_views + cam_rng.uniform(-0.1, 0.1)
        elev = radius * 0.9 + cam_rng.uniform(-0.1, 0.1) * extent
        pos = np.array([radius * np.cos(ang), radius * np.sin(ang), elev])
        cams.append(look_at_camera(pos, (0.0, 0.0, 0.0), fov_deg=fov_deg, width=width,
                                   height=height))
    return cams


# ---------------------------------------------------------------------------
# config 5: city of 4x2 blocks


CITY_BBOX = np.array([[-16.0, -8.0, -1.0], [16.0, 8.0, 1.0]])
CITY_GRID = (4, 2)


@dataclass
class CityScene:
    """Block-partitioned city: block b = iy*nx + ix covers one grid cell.

    Block partition follows the reference's half-open grid rule
    (scene_manager.py:24-80, ``partition_scene``); each block's Gaussians are
    drawn inside its cell so a block never straddles a cell boundary by mean.
    """

    blocks: list[HostGaussians]
    block_bboxes: np.ndarray  # (B, 2, 3)
    camera: Camera
    meta: dict = field(default_factory=dict)

    @property
    def count(self) -> int:
        return sum(b.count for b in self.blocks)


def city_block_bboxes(bbox=CITY_BBOX, grid=CITY_GRID) -> np.ndarray:
    nx, ny = grid
    span = bbox[1, :2] - bbox[0, :2]
    w, h = span / np.array([nx, ny])
    out = []
    for iy in range(ny):
        for ix in range(nx):
            lo = [bbox[0, 0] + ix * w, bbox[0, 1] + iy * h, bbox[0, 2]]
            hi = [bbox[0, 0] + (ix + 1) * w, bbox[0, 1] + (iy + 1) * h, bbox[1, 2]]
            out.append([lo, hi])
    return np.asarray(out)


def city_block(b: int, per_block: int, sh_degree: int = 3, bboxes=None) -> HostGaussians:
    bboxes = city_block_bboxes() if bboxes is None else bboxes
    rng = make_rng(1000 + b, "city_block")
    s = (1e4 / per_block) ** (1.0 / 3.0) if per_block > 10_000 else 1.0
    lo, hi = bboxes[b]
    return _draw_gaussians(rng, per_block, lo, hi, 4.0, s, sh_degree)


def city_camera(width=1920, height=1080) -> Camera:
    return look_at_camera((0.0, -22.0, 16.0), (0.0, 0.0, 0.0), fov_deg=70.0, width=width,
                          height=height)


def city_scene(per_block: int = 6_250_000, width=1920, height=1080, sh_degree=3) -> CityScene:
    bbs = city_block_bboxes()
    blocks = [city_block(b, per_block, sh_degree, bbs) for b in range(len(bbs))]
    return CityScene(blocks, bbs, city_camera(width, height), {"per_block": per_block})


# ---------------------------------------------------------------------------
# named configs


CONFIGS = {
    "c1": dict(n=10_000, width=256, height=256, views=1),
    "c2": dict(n=1_000_000, width=1920, height=1080, views=1),
    "c3": dict(n=6_000_000, width=1920, height=1080, views=64),
    "c4": dict(n=6_000_000, width=3840, height=2160, views=1),
    "c5": dict(n=50_000_000, width=1920, height=1080, views=1, blocks=8),
}


def config_scene(name: str, seed: int = 0):
    """(gaussians, cameras) for c1-c4."""
    c = CONFIGS[name]
    if name == "c5":
        raise InvalidInputError("use city_scene() for c5")
    g = synthetic_gaussians(c["n"], seed=seed)
    cams = orbit_cameras(c["views"], c["width"], c["height"], seed=seed)
    return g, cams
