"""Generate golden fixtures from the UNMODIFIED reference renderer.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Each case renders a scene with ``landmark.gaussian_core.render_image(...,
with_record=True)`` (gaussian_core.py:582-597) and stores the reference's
outputs: image (H,W,3) f64, touched (M,), per-tile prim-id lists
(``splats.prim_id[tile.order]``, TileRecord 256-263) with their offsets, and
t_final (alpha = 1 - t_final).  Inputs are stored verbatim for the small cases
and as a SHA-256 of the regenerated arrays for the 10k-Gaussian config c1.
The fixtures pin the CPU oracle (oracle/oracle.c) and, on the GPU box, the
CUDA path; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np
import torch

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from landmark.common import make_rng as ref_make_rng  # noqa: E402
from landmark.data_io import Camera as RefCamera  # noqa: E402
from landmark.data_io import look_at_camera as ref_look_at  # noqa: E402
from landmark.gaussian_core import GaussianModel, render_image  # noqa: E402

from paper_2503_21364_b200 import scenes  # noqa: E402


def arrays_digest(g) -> str:
    h = hashlib.sha256()
    for a in (g.means, g.quats, g.scales, g.opacity_logits, g.sh):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def cam_fields(cam) -> dict:
    return dict(cam_fx=cam.fx, cam_fy=cam.fy, cam_cx=cam.cx, cam_cy=cam.cy,
                cam_w=cam.width, cam_h=cam.height, cam_r=np.asarray(cam.r_wc),
                cam_t=np.asarray(cam.t_wc))


def render_case(name, arrays, sh_degree, cam, tile_size=16, background=(0.0, 0.0, 0.0),
                subset=None, store_inputs=True, digest=None):
    means, quats, scales, logits, sh = arrays
    model = GaussianModel(means=means, quats=quats, scales=scales, opacity_logits=logits,
                          sh=sh, sh_degree=sh_degree)
    image, touched, rec = render_image(model, cam, tile_size, background, with_record=True,
                                       subset=subset)
    lists, offsets = [], [0]
    t_final = np.ones(cam.width * cam.height)
    for tile in rec.tiles:
        ids = rec.splats.prim_id[tile.order].numpy()
        lists.append(ids)
        offsets.append(offsets[-1] + len(ids))
        t_final[tile.pix_idx.numpy()] = tile.t_final.numpy()
    lists = np.concatenate(lists) if lists else np.zeros(0, np.int64)
    out = dict(image=image.numpy(), touched=touched.numpy().astype(np.int32),
               lists=lists.astype(np.int32), offsets=np.asarray(offsets, np.int32),
               t_final=t_final.reshape(cam.height, cam.width),
               splat_prim_id=rec.splats.prim_id.numpy().astype(np.int32),
               tile_size=np.int32(tile_size), background=np.asarray(background, np.float64),
               sh_degree=np.int32(sh_degree), **cam_fields(cam))
    if subset is not None:
        out["subset"] = np.asarray(subset, np.int64)
    if store_inputs:
        out.update(means=means, quats=quats, scales=scales, opacity_logits=logits, sh=sh)
    if digest is not None:
        out["digest"] = np.array(digest)
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(f"{name}: M={len(touched)} K={len(lists)} tiles={len(rec.tiles)}")


def f32(a):
    return np.asarray(a, dtype=np.float32)


def random_model_arrays(seed, n, extent=3.0):
    """The reference tests' random_model (tests/test_gaussian_core.py:29-43), f32."""
    rng = ref_make_rng(seed, "m")
    quats = rng.standard_normal((n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    sh = np.zeros((n, 4, 3))
    sh[:, 0] = rng.uniform(0.2, 2.5, (n, 3))
    sh[:, 1:] = rng.uniform(-0.1, 0.1, (n, 3, 3))
    means = rng.uniform(-extent, extent, (n, 3))
    scales = rng.uniform(0.05, 0.4, (n, 3))
    logits = rng.uniform(-1.5, 2.0, n)
    q = f32(quats)
    q /= np.linalg.norm(q, axis=1, keepdims=True).astype(np.float32)
    return f32(means), q, f32(scales), f32(logits), f32(sh)


def front_camera(width=32, height=32, dist=8.0, fov=60.0):
    return ref_look_at((0.0, -dist, 0.0), (0.0, 0.0, 0.0), fov_deg=fov, width=width,
                       height=height)


def main():
    # c1: the benchmark's CPU-runnable config (10k, SH3, 256x256), regenerated from seed
    g = scenes.synthetic_gaussians(10_000, seed=0)
    cam = scenes.orbit_cameras(1, 256, 256, seed=0)[0]
    render_case("c1_10k_256", (g.means, g.quats, g.scales, g.opacity_logits, g.sh), 3, cam,
                store_inputs=False, digest=arrays_digest(g))

    # reference-test-style scenes: tile sizes 8/16/32 (test_gaussian_core.py:245-251)
    for seed in range(3):
        arr = random_model_arrays(seed, 60)
        for ts in (8, 16, 32):
            render_case(f"rand{seed}_ts{ts}", arr, 1, front_camera(), tile_size=ts)

    # ragged images with partial edge tiles (SURVEY §8a row 9 note) and a background
    arr = random_model_arrays(21, 200, extent=3.0)
    render_case("ragged_100x70_ts16", arr, 1, front_camera(100, 70), tile_size=16,
                background=(0.2, 0.4, 0.6))
    render_case("ragged_130x67_ts8", arr, 1, front_camera(130, 67), tile_size=8)
    render_case("ragged_130x67_ts32", arr, 1, front_camera(130, 67), tile_size=32,
                background=(1.0, 0.0, 0.5))
    render_case("ragged_67x45_ts10", arr, 1, front_camera(67, 45), tile_size=10)

    # exact depth ties: duplicated Gaussians (densify clones, gaussian_core.py:553-556)
    m, q, s, lg, sh = random_model_arrays(5, 40)
    dup = np.array([3, 7, 7, 11, 3, 25, 30, 30, 30], dtype=np.int64)
    arr = tuple(np.concatenate([a, a[dup]]) for a in (m, q, s, lg, sh))
    render_case("ties_dup_ts16", arr, 1, front_camera(48, 40), tile_size=16)

    # subset with unsorted ids and ties (render_image remaps prim ids, 593-595)
    subset = np.array([44, 3, 40, 7, 12, 43, 45, 46, 1, 30, 47, 48, 5], dtype=np.int64)
    render_case("subset_ts16", arr, 1, front_camera(48, 40), tile_size=16, subset=subset)

    # degree-3 model through the reference (which evaluates degrees 0-1 only)
    g3 = scenes.synthetic_gaussians(500, seed=3)
    cam3 = scenes.orbit_cameras(3, 96, 64, seed=3)[1]
    render_case("sh3_500_96x64", (g3.means, g3.quats, g3.scales, g3.opacity_logits, g3.sh), 3,
                cam3, tile_size=16)

    # near-plane culling: half the scene behind the camera (gaussian_core.py:196-198)
    m, q, s, lg, sh = random_model_arrays(9, 80, extent=3.0)
    render_case("nearcull_ts16", (m, q, s, lg, sh), 1, front_camera(64, 48, dist=1.0, fov=90.0))

    # empty scene: everything culled -> pure background (233-242)
    m = np.array([[0.0, -20.0, 0.0]], np.float32)
    render_case("empty_bg", (m, f32([[1, 0, 0, 0]]), f32([[0.1, 0.1, 0.1]]), f32([0.0]),
                             np.zeros((1, 4, 3), np.float32)), 1, front_camera(24, 24),
                background=(0.2, 0.4, 0.6))

    # known answers (test_gaussian_core.py:197-230): saturated and two-splat blends
    c0 = 0.28209479177387814
    cam = RefCamera(fx=40.0, fy=40.0, cx=16.0, cy=16.0, width=32, height=32,
                    r_wc=np.eye(3), t_wc=np.zeros(3))
    two = (f32([[0.0, 0.0, 5.0], [0.0, 0.0, 6.0]]), f32([[1.0, 0.0, 0.0, 0.0]] * 2),
           f32(np.full((2, 3), 50.0)), f32([0.0, 20.0]),
           f32([[[0.9 / c0, 0, 0], [0, 0, 0], [0, 0, 0], [0, 0, 0]],
                [[0, 0.7 / c0, 0], [0, 0, 0], [0, 0, 0], [0, 0, 0]]]))
    render_case("two_splat", two, 1, cam)


if __name__ == "__main__":
    torch.set_num_threads(8)
    main()
