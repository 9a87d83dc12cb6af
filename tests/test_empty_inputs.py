"""Empty inputs through every entry point (the reference's empty-scene
behaviour, test_gaussian_core.py:233-242: background everywhere)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _empty():
    from paper_2503_21364_b200 import GaussianModel, scenes

    return GaussianModel.from_host(scenes.synthetic_gaussians(0, seed=0, sh_degree=3))


def test_project_and_instances_empty():
    from paper_2503_21364_b200 import project, render, scenes

    cam = scenes.orbit_cameras(1, 48, 32)[0]
    p = project(cam, _empty())
    assert p["kept"].numel() == 0
    out = render(cam, _empty(), 16, (0.1, 0.2, 0.3), with_instances=True)
    assert out.n_instances == 0 and out.inst_keys.numel() == 0
    assert int(out.tile_ranges.abs().sum()) == 0


def test_render_strips_empty():
    import torch

    from paper_2503_21364_b200 import _lib, scenes
    from paper_2503_21364_b200.raster import abi_camera, abi_settings, context

    cam = scenes.orbit_cameras(1, 48, 32)[0]
    rgb = torch.zeros((32, 48, 3), device="cuda")
    t = _lib.StripTargets()
    t.n_strips, t.strip_rows = 1, 32
    t.rgb[0] = rgb.data_ptr()
    ctx = context(0)
    m = _empty()
    g, c, s = m._abi(), abi_camera(cam), abi_settings(16, 3, (0.1, 0.2, 0.3))
    _lib.check(ctx.handle, _lib.lib().lmgs_render_strips(
        ctx.handle, ctypes.byref(g), ctypes.byref(c), ctypes.byref(s), ctypes.byref(t), None,
        torch.cuda.current_stream().cuda_stream), "lmgs_render_strips")
    torch.cuda.synchronize()
    np.testing.assert_allclose(rgb.cpu().numpy(), np.broadcast_to([0.1, 0.2, 0.3], (32, 48, 3)),
                               atol=1e-7)


def test_checkpoint_round_trip_empty(tmp_path):
    from paper_2503_21364_b200.checkpoint import load_gaussian_checkpoint, save_gaussian_checkpoint

    out = tmp_path / "empty.lmgs"
    save_gaussian_checkpoint(_empty(), out)
    m, grid = load_gaussian_checkpoint(out)
    assert m.count == 0 and grid is None


def test_frustum_session_sees_nothing():
    from paper_2503_21364_b200 import offload as o
    from paper_2503_21364_b200 import scenes
    from paper_2503_21364_b200.camera import look_at_camera

    g = scenes.synthetic_gaussians(2000, seed=3, sh_degree=1)
    # looking away from the scene: no voxel is visible
    cam = look_at_camera((0.0, -30.0, 0.0), (0.0, -60.0, 0.0), fov_deg=30.0, width=32,
                         height=32, near=0.01, far=5.0)
    cfg = o.SessionConfig(mode="frustum_voxel", budget_bytes=1 << 30, voxel_size=1.0)
    sess = o.FrustumSession(g, cfg)
    img, n = sess.step(cam)
    assert n == 0
    assert float(img.abs().max()) == 0.0
