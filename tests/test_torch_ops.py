"""The TORCH_LIBRARY(lmgs) operators (csrc/torch_ops.cpp): the dispatcher-
visible boundary for render_image (gaussian_core.py:582-597)."""

import numpy as np
import pytest
import torch

from conftest import GOLDEN_CASES
from paper_2503_21364_b200 import GaussianModel, ops, render, render_image, scenes


def test_ops_registered_with_schema():
    L = ops.load()
    s = str(L.render_fwd.default._schema)
    assert s.startswith("lmgs::render_fwd(Tensor means, Tensor quats, Tensor scales, "
                        "Tensor opacity_logits, Tensor sh, int sh_degree, int sh_eval_degree, "
                        "Tensor cam")
    assert "-> (Tensor rgb, Tensor alpha, Tensor depth, Tensor tile_ranges, Tensor inst_keys, " \
           "Tensor inst_vals, Tensor touched, Tensor n_processed)" in s
    assert "lmgs::render_image" in str(L.render_image.default._schema)


def test_pack_camera_matches_abi_camera():
    from paper_2503_21364_b200.raster import abi_camera

    cam = scenes.orbit_cameras(1, 640, 480, seed=3)[0]
    v = ops.pack_camera(cam).numpy()
    c = abi_camera(cam)
    assert v.dtype == np.float64 and v.shape == (21,)
    np.testing.assert_array_equal(v[:9], list(c.r_wc))
    np.testing.assert_array_equal(v[12:15], list(c.center))
    assert (v[19], v[20]) == (c.lim_x, c.lim_y)


@pytest.mark.gpu
def test_render_fwd_op_equals_render():
    g = scenes.synthetic_gaussians(20_000, seed=5)
    cam = scenes.orbit_cameras(1, 320, 240, seed=5)[0]
    m = GaussianModel.from_host(g)
    rgb, alpha, depth, ranges, keys, vals, touched, nproc = ops.render_fwd(
        cam, m, 16, (0.1, 0.2, 0.3), 3)
    o = render(cam, m, 16, (0.1, 0.2, 0.3), 3, with_instances=True)
    torch.cuda.synchronize()
    assert rgb.dtype == torch.float32 and rgb.shape == (240, 320, 3) and rgb.is_cuda
    assert torch.equal(rgb, o.rgb) and torch.equal(alpha, o.alpha) and torch.equal(depth, o.depth)
    assert torch.equal(ranges, o.tile_ranges) and torch.equal(nproc, o.n_processed)
    assert torch.equal(keys, o.inst_keys) and torch.equal(vals.long(), o.inst_prim_ids)
    assert torch.equal(touched, o.touched)


@pytest.mark.gpu
def test_render_fwd_on_side_stream():
    """The op runs on the current stream (its own context per stream)."""
    g = scenes.synthetic_gaussians(5_000, seed=6)
    cam = scenes.orbit_cameras(1, 160, 128, seed=6)[0]
    m = GaussianModel.from_host(g)
    ref = ops.render_fwd(cam, m)[0]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        out = ops.render_fwd(cam, m)[0]
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in GOLDEN_CASES if "subset" in n or "c1" in n])
def test_render_image_op_matches_golden(golden_case, name):
    c = golden_case(name)
    m = GaussianModel.from_host(c.gaussians)
    L = ops.load()
    img, touched = L.render_image(m.means, m.quats, m.scales, m.opacity_logits, m.sh,
                                  m.sh_degree, 1, ops.pack_camera(c.camera), c.camera.width,
                                  c.camera.height, c.tile_size, list(c.background),
                                  None if c.subset is None else torch.as_tensor(c.subset))
    ref_img, ref_touched = render_image(c.gaussians, c.camera, c.tile_size, c.background,
                                        subset=c.subset)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(touched.cpu().numpy(), c.touched)
    assert torch.equal(img, ref_img)
    assert np.abs(img.cpu().double().numpy() - c.image).max() <= 1e-4
