"""Backward of the blend and the training-loss chain against
the unmodified reference (tests/golden/backward/make_backward_golden.py):

* ``backward_render`` (gaussian_core.py:438-486) of a seeded random image
  gradient: d_colors, d_opacities, d_mean2d per Gaussian, touched counts;
* ``render_loss_and_grads`` (600-629): loss, d_sh, d_opacity_logits and the
  DensifyStats increments over two cameras.

Both sides compute in fp64 from the same fp64 geometry (K1's projection is
bit-exact), so the tolerance is set by summation order (per-pixel terms are
accumulated with atomics here, in tile/pixel order there) and the 1-ulp exp
differences between libdevice and the host libm: rtol 1e-9 on sums with an
absolute floor of 1e-9 x the array's largest magnitude.  The loss path feeds
the forward's fp32 image (rgb tolerance 1e-4, test_gpu_pipeline) into the
gradient, so it is checked at rtol 1e-4 of each array's scale.
"""

import numpy as np
import pytest

from conftest import GOLDEN

BW = GOLDEN / "backward"
CASES = ["ts16", "ts8_bg", "ts32"]


def _load(name):
    from paper_2503_21364_b200 import scenes
    from paper_2503_21364_b200.camera import Camera

    z = np.load(BW / name)

    def cam(sfx=""):
        return Camera(float(z["cam_fx" + sfx]), float(z["cam_fy" + sfx]), float(z["cam_cx" + sfx]),
                      float(z["cam_cy" + sfx]), int(z["cam_w" + sfx]), int(z["cam_h" + sfx]),
                      z["cam_r" + sfx], z["cam_t" + sfx])

    g = scenes.HostGaussians(z["means"], z["quats"], z["scales"], z["opacity_logits"], z["sh"],
                             int(z["sh_degree"]))
    return z, g, cam


def _close(got, ref, rtol, what):
    scale = max(float(np.abs(ref).max()), 1e-300)
    np.testing.assert_allclose(got, ref, rtol=rtol, atol=rtol * scale, err_msg=what)


def test_golden_fixtures_consistent():
    """CPU: the fixtures hold what the tests read (every kept splat touched
    something in these scenes, gradients finite)."""
    for c in CASES:
        z = np.load(BW / f"backward_{c}.npz")
        n = z["means"].shape[0]
        assert z["d_colors"].shape == (n, 3) and z["d_mean2d"].shape == (n, 2)
        assert np.isfinite(z["d_colors"]).all() and np.isfinite(z["d_opacities"]).all()
        assert (z["touched"] > 0).sum() > n // 2
    z = np.load(BW / "loss_grads.npz")
    assert z["d_sh"].shape == z["sh"].shape and 0 < float(z["loss"]) < 1


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_backward_render_matches_reference(case):
    import torch

    from paper_2503_21364_b200 import GaussianModel
    from paper_2503_21364_b200.train import backward_render

    z, g, cam = _load(f"backward_{case}.npz")
    model = GaussianModel.from_host(g)
    bg = tuple(float(v) for v in z["background"])
    fwd, gr = backward_render(model, cam(), torch.as_tensor(z["image_grad"]).cuda(),
                              int(z["tile_size"]), bg)
    np.testing.assert_allclose(fwd.rgb.cpu().numpy(), z["image"], atol=1e-4)
    tch = gr.touched.cpu().numpy().astype(np.int64)
    # touched is a count of w > 0 tests in fp64 on both sides
    assert int(np.abs(tch - z["touched"]).sum()) <= 2, case
    _close(gr.d_colors.cpu().numpy(), z["d_colors"], 1e-9, "d_colors")
    _close(gr.d_opacities.cpu().numpy(), z["d_opacities"], 1e-9, "d_opacities")
    _close(gr.d_mean2d.cpu().numpy(), z["d_mean2d"], 1e-9, "d_mean2d")


@pytest.mark.gpu
def test_backward_is_linear_in_image_grad():
    """Size-independent property: grads(a*g1 + g2) = a*grads(g1) + grads(g2)."""
    import torch

    from paper_2503_21364_b200 import GaussianModel, scenes
    from paper_2503_21364_b200.train import backward_render

    g = scenes.synthetic_gaussians(20_000, seed=5, sh_degree=1)
    model = GaussianModel.from_host(g)
    cam = scenes.orbit_cameras(1, 320, 240, seed=5)[0]
    gen = torch.Generator().manual_seed(0)
    # dyadic gradients so that 0.5*g1 + g2 is exact in the fp32 input
    g1 = torch.randint(-1024, 1025, (240, 320, 3), generator=gen).float() / 1024
    g2 = torch.randint(-1024, 1025, (240, 320, 3), generator=gen).float() / 1024
    _, a = backward_render(model, cam, g1.cuda())
    _, b = backward_render(model, cam, g2.cuda())
    _, c = backward_render(model, cam, (0.5 * g1 + g2).cuda())
    for f in ("d_colors", "d_opacities", "d_mean2d"):
        want = 0.5 * getattr(a, f) + getattr(b, f)
        _close(getattr(c, f).cpu().numpy(), want.cpu().numpy(), 1e-9, f)
    assert bool((a.touched == c.touched).all())


@pytest.mark.gpu
def test_render_loss_and_grads_matches_reference():
    from paper_2503_21364_b200 import GaussianModel
    from paper_2503_21364_b200.train import render_loss_and_grads

    z, g, cam = _load("loss_grads.npz")
    model = GaussianModel.from_host(g)
    cams = [cam("_0"), cam("_1")]
    loss, grads, stats = render_loss_and_grads(model, cams, [z["gt0"], z["gt1"]],
                                               int(z["tile_size"]))
    assert abs(loss - float(z["loss"])) <= 1e-6 * float(z["loss"])
    _close(grads["sh"].cpu().numpy(), z["d_sh"], 1e-4, "d_sh")
    _close(grads["opacity_logits"].cpu().numpy(), z["d_logits"], 1e-4, "d_logits")
    np.testing.assert_array_equal(stats.steps_seen.cpu().numpy(), z["steps_seen"])
    _close(stats.grad_norm_sum.cpu().numpy(), z["grad_norm_sum"], 1e-4, "grad_norm_sum")


@pytest.mark.gpu
def test_backward_rejects_mismatched_shapes():
    import torch

    from paper_2503_21364_b200 import GaussianModel, scenes
    from paper_2503_21364_b200.errors import ShapeError
    from paper_2503_21364_b200.train import backward_render

    g = scenes.synthetic_gaussians(100, seed=1, sh_degree=1)
    cam = scenes.orbit_cameras(1, 64, 48, seed=1)[0]
    with pytest.raises(ShapeError):
        backward_render(GaussianModel.from_host(g), cam, torch.zeros(48, 63, 3).cuda())


def _random_model(seed, n, extent=3.0):
    """test_gaussian_core.py:29-43 (random_model), drawn in f32."""
    from paper_2503_21364_b200 import scenes

    rng = np.random.default_rng(seed)
    quats = rng.standard_normal((n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    sh = np.zeros((n, 4, 3))
    sh[:, 0] = rng.uniform(0.2, 2.5, (n, 3))
    sh[:, 1:] = rng.uniform(-0.1, 0.1, (n, 3, 3))
    f = np.float32
    return scenes.HostGaussians(rng.uniform(-extent, extent, (n, 3)).astype(f), quats.astype(f),
                                rng.uniform(0.05, 0.4, (n, 3)).astype(f),
                                rng.uniform(-1.5, 2.0, n).astype(f), sh.astype(f), 1)


def _front_camera(w, h):
    from paper_2503_21364_b200.camera import look_at_camera

    return look_at_camera((0.0, -8.0, 0.0), (0.0, 0.0, 0.0), fov_deg=60.0, width=w, height=h)


@pytest.mark.gpu
def test_backward_zero_contribution_zero_gradient():
    """test_gaussian_core.py:300-307: untouched splats get exactly zero gradient."""
    import torch

    from paper_2503_21364_b200 import GaussianModel
    from paper_2503_21364_b200.train import backward_render

    g = _random_model(14, 10)
    _, gr = backward_render(GaussianModel.from_host(g), _front_camera(32, 32),
                            torch.ones(32, 32, 3).cuda())
    un = (gr.touched == 0).cpu()
    assert bool((gr.d_colors.cpu()[un] == 0).all()) and bool((gr.d_opacities.cpu()[un] == 0).all())
    assert int((~un).sum()) > 0


@pytest.mark.gpu
def test_backward_single_splat_analytic():
    """test_gaussian_core.py:310-328: one saturated splat on the pixel centre,
    dL/dc = 2 (sigma c - gt) sigma with sigma = SIGMA_MAX."""
    import torch

    from paper_2503_21364_b200 import GaussianModel, scenes
    from paper_2503_21364_b200.camera import Camera
    from paper_2503_21364_b200.train import backward_render

    c0 = 0.28209479177387814
    cam = Camera(40.0, 40.0, 0.5, 0.5, 1, 1, np.eye(3), np.zeros(3))
    sh = np.zeros((1, 4, 3), np.float32)
    sh[0, 0] = 0.8 / c0
    g = scenes.HostGaussians(np.array([[0.0, 0.0, 5.0]], np.float32),
                             np.array([[1.0, 0.0, 0.0, 0.0]], np.float32),
                             np.full((1, 3), 500.0, np.float32), np.array([200.0], np.float32), sh, 1)
    model = GaussianModel.from_host(g)
    from paper_2503_21364_b200 import render

    image = render(cam, model, 16, (0.0, 0.0, 0.0), 1).rgb
    _, gr = backward_render(model, cam, 2.0 * (image - 0.5))
    sigma = 0.9999
    expected = 2.0 * (0.8 * sigma - 0.5) * sigma
    assert torch.allclose(gr.d_colors[0].cpu(), torch.full((3,), expected, dtype=torch.float64),
                          atol=1e-4)


@pytest.mark.gpu
def test_gradients_match_finite_differences():
    """test_gaussian_core.py:331-374: analytic SH / opacity-logit gradients of
    the MSE loss against central differences of the fp64 oracle render (step
    2^-12, exact in f32), relative tolerance 1e-3, at least 30 checked."""
    import oracle

    from paper_2503_21364_b200 import GaussianModel
    from paper_2503_21364_b200.train import render_loss_and_grads

    g = _random_model(15, 10)
    cam = _front_camera(24, 24)
    gt = np.random.default_rng(1).uniform(0, 1, (24, 24, 3))
    _, grads, _ = render_loss_and_grads(GaussianModel.from_host(g), [cam], [gt])
    d_sh = grads["sh"].cpu().numpy()
    d_lg = grads["opacity_logits"].cpu().numpy()

    def loss_of(gg):
        return float(((oracle.render(gg, cam)["image"] - gt) ** 2).mean())

    h = 2.0 ** -12
    rng = np.random.default_rng(0)
    checked = 0
    for _ in range(60):
        gg = type(g)(g.means.copy(), g.quats.copy(), g.scales.copy(), g.opacity_logits.copy(),
                     g.sh.copy(), 1)
        if rng.uniform() < 0.5:
            i, k, c = int(rng.integers(10)), int(rng.integers(4)), int(rng.integers(3))
            analytic, arr, idx = float(d_sh[i, k, c]), gg.sh, (i, k, c)
        else:
            i = int(rng.integers(10))
            analytic, arr, idx = float(d_lg[i]), gg.opacity_logits, (i,)
        x = arr[idx]
        arr[idx] = x + np.float32(h)
        up = loss_of(gg)
        arr[idx] = x - np.float32(h)
        dn = loss_of(gg)
        fd = (up - dn) / (2 * h)
        if abs(fd) < 1e-8 and abs(analytic) < 1e-8:
            continue
        assert abs(analytic - fd) <= 1e-3 * max(abs(fd), abs(analytic), 1e-6), (analytic, fd)
        checked += 1
    assert checked >= 30


@pytest.mark.gpu
@pytest.mark.parametrize("ts", [1, 5, 24, 64])
def test_backward_tile_size_invariant(ts):
    """Per pixel the splats arrive in the same (depth, id) order whatever the
    tile size, so gradients equal the tile-16 ones (summation order aside) and
    touched counts are identical: exercises ragged 8x4 blocks (ts 1, 5, 24)
    and 128 blocks per tile (ts 64)."""
    import torch

    from paper_2503_21364_b200 import GaussianModel
    from paper_2503_21364_b200.train import backward_render

    z, g, cam = _load("backward_ts16.npz")
    model = GaussianModel.from_host(g)
    gi = torch.as_tensor(z["image_grad"]).cuda()
    _, ref = backward_render(model, cam(), gi, 16)
    _, got = backward_render(model, cam(), gi, ts)
    assert bool((got.touched == ref.touched).all())
    for f in ("d_colors", "d_opacities", "d_mean2d"):
        _close(getattr(got, f).cpu().numpy(), getattr(ref, f).cpu().numpy(), 1e-9, f)


@pytest.mark.gpu
@pytest.mark.parametrize("use_subset", [False, True])
def test_backward_render_reference_signature(use_subset):
    """backward_render(image_grad, record) as the reference calls it (438):
    rows aligned with the record's splats, values as the golden's."""
    import torch

    from paper_2503_21364_b200 import GaussianModel, render_image
    from paper_2503_21364_b200.train import backward_render

    z, g, cam = _load("backward_ts16.npz")
    model = GaussianModel.from_host(g)
    subset = None
    if use_subset:  # every Gaussian, shuffled: same image, record in caller order
        subset = np.random.default_rng(3).permutation(g.count)
    _, touched, rec = render_image(model, cam(), int(z["tile_size"]), (0.0, 0.0, 0.0),
                                   with_record=True, subset=subset)
    gr = backward_render(torch.as_tensor(z["image_grad"]).cuda(), rec)
    pid = rec.prim_id.numpy()
    assert gr.d_colors.shape == (len(pid), 3)
    _close(gr.d_colors.cpu().numpy(), z["d_colors"][pid], 1e-9, "d_colors")
    _close(gr.d_opacities.cpu().numpy(), z["d_opacities"][pid], 1e-9, "d_opacities")
    _close(gr.d_mean2d.cpu().numpy(), z["d_mean2d"][pid], 1e-9, "d_mean2d")
    assert int(np.abs(gr.touched.cpu().numpy() - z["touched"][pid]).sum()) <= 2
    np.testing.assert_array_equal(gr.touched.cpu().numpy(), touched.cpu().numpy())


@pytest.mark.gpu
def test_backward_empty_and_culled_scenes():
    """No splats on screen: zero gradients, zero touched, loss of the background."""
    import torch

    from paper_2503_21364_b200 import GaussianModel, scenes
    from paper_2503_21364_b200.camera import Camera
    from paper_2503_21364_b200.train import backward_render, render_loss_and_grads

    cam = Camera(40.0, 40.0, 16.0, 16.0, 32, 32, np.eye(3), np.zeros(3))
    g0 = scenes.synthetic_gaussians(0, seed=0, sh_degree=1)
    _, gr = backward_render(GaussianModel.from_host(g0), cam, torch.ones(32, 32, 3).cuda())
    assert gr.d_colors.numel() == 0
    behind = scenes.HostGaussians(np.array([[0, 0, -2.0]] * 5, np.float32),
                                  np.tile(np.array([[1, 0, 0, 0]], np.float32), (5, 1)),
                                  np.full((5, 3), 0.3, np.float32), np.zeros(5, np.float32),
                                  np.ones((5, 4, 3), np.float32), 1)
    m = GaussianModel.from_host(behind)
    _, gr = backward_render(m, cam, torch.ones(32, 32, 3).cuda(), 16, (0.2, 0.3, 0.4))
    assert float(gr.d_colors.abs().sum()) == 0.0 and int(gr.touched.sum()) == 0
    gt = np.full((32, 32, 3), 0.5)
    loss, grads, stats = render_loss_and_grads(m, [cam], [gt], 16, (0.2, 0.3, 0.4))
    assert abs(loss - float(np.mean((np.array([0.2, 0.3, 0.4]) - 0.5) ** 2))) < 1e-6
    assert float(grads["sh"].abs().sum()) == 0.0 and int(stats.steps_seen.sum()) == 0


@pytest.mark.gpu
def test_degree3_sh_gradients_match_finite_differences():
    """Our extension beyond the reference (which evaluates degrees 0-1 only):
    with sh_eval_degree=3 the chain to coefficients 4-15 (standard real SH
    basis) matches central differences of the fp64 oracle render at degree 3."""
    import oracle

    from paper_2503_21364_b200 import GaussianModel, scenes
    from paper_2503_21364_b200.train import render_loss_and_grads

    rng = np.random.default_rng(4)
    n = 12
    quats = rng.standard_normal((n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    sh = np.zeros((n, 16, 3))
    sh[:, 0] = rng.uniform(0.8, 1.6, (n, 3))  # keep the clamp gate open
    sh[:, 1:] = rng.uniform(-0.2, 0.2, (n, 15, 3))
    f = np.float32
    g = scenes.HostGaussians(rng.uniform(-2.5, 2.5, (n, 3)).astype(f), quats.astype(f),
                             rng.uniform(0.2, 0.5, (n, 3)).astype(f),
                             rng.uniform(-1.0, 1.5, n).astype(f), sh.astype(f), 3)
    cam = _front_camera(24, 24)
    gt = rng.uniform(0, 1, (24, 24, 3))
    _, grads, _ = render_loss_and_grads(GaussianModel.from_host(g), [cam], [gt], 16,
                                        sh_eval_degree=3)
    d_sh = grads["sh"].cpu().numpy()

    def loss_of(gg):
        return float(((oracle.render(gg, cam, sh_eval_degree=3)["image"] - gt) ** 2).mean())

    h = 2.0 ** -12
    checked = 0
    for i in range(n):
        for k in (4, 7, 9, 12, 15):
            c = (i + k) % 3
            gg = type(g)(g.means, g.quats, g.scales, g.opacity_logits, g.sh.copy(), 3)
            x = gg.sh[i, k, c]
            gg.sh[i, k, c] = x + np.float32(h)
            up = loss_of(gg)
            gg.sh[i, k, c] = x - np.float32(h)
            dn = loss_of(gg)
            fd = (up - dn) / (2 * h)
            an = float(d_sh[i, k, c])
            if abs(fd) < 1e-8 and abs(an) < 1e-8:
                continue
            assert abs(an - fd) <= 1e-3 * max(abs(fd), abs(an), 1e-6), (i, k, c, an, fd)
            checked += 1
    assert checked >= 30


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_reference_backward_runs_on_our_record(case):
    """The full RenderRecord (gaussian_core.py:256-274: splats, colors,
    opacities, per-tile sigma / t_before / t_final) feeds the reference's
    backward_render algorithm (restated in oracle.backward_from_record) and
    gives the reference's own gradients."""
    import oracle
    from paper_2503_21364_b200 import render_image

    z, g, cam = _load(f"backward_{case}.npz")
    bg = tuple(float(v) for v in z["background"])
    _, _, rec = render_image(g, cam(), int(z["tile_size"]), bg, with_record=True, collect=True)
    assert rec.splats is not None and rec.tiles[0].sigma is not None
    out = oracle.backward_from_record(z["image_grad"], rec)
    assert int(np.abs(out["touched"] - z["touched"]).sum()) <= 2, case
    _close(out["d_colors"], z["d_colors"], 1e-9, "d_colors")
    _close(out["d_opacities"], z["d_opacities"], 1e-9, "d_opacities")
    _close(out["d_mean2d"], z["d_mean2d"], 1e-9, "d_mean2d")
