"""Grouped views (lmgs_render_group): one K1 launch projects a staged block of
Gaussians for up to 8 views, each view then runs its own pipeline.  The bar is
bit-identity with one lmgs_render call per view for every output buffer (the
per-view math is unchanged; only the input staging is shared), plus the
oracle check of a grouped view."""

import numpy as np
import pytest
import torch

import oracle
from paper_2503_21364_b200 import GaussianModel, scenes
from paper_2503_21364_b200.batch import BatchRenderer

pytestmark = pytest.mark.gpu

FIELDS = ("rgb", "alpha", "depth", "touched", "kept", "ranges", "nproc")


def _render_all(model, cams, w, h, group, stage_times=False, page_mask=None, n_streams=2):
    r = BatchRenderer(model, w, h, len(cams), sh_eval_degree=3, n_streams=n_streams, group=group,
                      page_mask=page_mask)
    r.render(cams, stage_times=stage_times)
    torch.cuda.synchronize()
    return {f: getattr(r, f)[:len(cams)].cpu().clone() for f in FIELDS}


@pytest.fixture(scope="module")
def scene():
    # 20,000 + 37 rows: full 128-row TMA blocks plus a direct-load tail block
    g = scenes.synthetic_gaussians(20_037, seed=3)
    return g, GaussianModel.from_host(g)


@pytest.mark.parametrize("group", [2, 3, 4, 8])
def test_group_equals_per_view(scene, group):
    _, model = scene
    cams = scenes.orbit_cameras(11, 320, 200, seed=1)  # 11 views: a ragged last group
    ref = _render_all(model, cams, 320, 200, 1)
    got = _render_all(model, cams, 320, 200, group)
    for f in FIELDS:
        assert torch.equal(ref[f], got[f]), f


def test_group_stage_times_path_equal(scene):
    _, model = scene
    cams = scenes.orbit_cameras(5, 256, 256, seed=2)
    ref = _render_all(model, cams, 256, 256, 1)
    got = _render_all(model, cams, 256, 256, 4, stage_times=True)
    for f in FIELDS:
        assert torch.equal(ref[f], got[f]), f


def test_group_paged_rows_culled(scene):
    """Paged sets: pages with live count 0 and rows past a page's count are
    culled for every view of the group."""
    g, model = scene
    pages = -(-model.count // 128)
    rng = np.random.default_rng(0)
    live = rng.integers(0, 129, size=pages).astype(np.uint8)
    live[::5] = 0
    mask = torch.from_numpy(live).cuda()
    cams = scenes.orbit_cameras(6, 256, 192, seed=4)
    ref = _render_all(model, cams, 256, 192, 1, page_mask=mask)
    got = _render_all(model, cams, 256, 192, 6, page_mask=mask)
    for f in FIELDS:
        assert torch.equal(ref[f], got[f]), f
    rows = np.arange(model.count)
    dead = rows % 128 >= live[rows // 128]
    assert not got["kept"].numpy()[:, dead].any()


def test_grouped_view_matches_oracle():
    g = scenes.synthetic_gaussians(10_000, seed=0)
    model = GaussianModel.from_host(g)
    cams = scenes.orbit_cameras(4, 256, 256, seed=0)
    got = _render_all(model, cams, 256, 256, 4)
    for v in (0, 3):
        o = oracle.render(g, cams[v], 16, sh_eval_degree=3)
        kept = got["kept"][v].numpy().astype(bool)
        assert np.array_equal(got["touched"][v].numpy()[kept], o["touched"])
        err = float(np.abs(got["rgb"][v].double().numpy() - o["image"]).max())
        assert err <= 1e-4, err


def test_group_argument_errors(scene):
    """lmgs_render_group rejects empty / oversized groups and repeated contexts
    (each view needs its own arena) with the reference's InvalidInputError."""
    import ctypes

    from paper_2503_21364_b200 import _lib
    from paper_2503_21364_b200.errors import InvalidInputError
    from paper_2503_21364_b200.raster import abi_camera, abi_settings

    _, model = scene
    L = _lib.lib()
    cams = scenes.orbit_cameras(2, 64, 48, seed=0)
    r = BatchRenderer(model, 64, 48, 2, group=2)
    g = model._abi()
    st = abi_settings(16, 3, (0.0, 0.0, 0.0), 0)
    frames = (_lib.Frame * 2)(r._frame(0), r._frame(1))
    cam_arr = (_lib.Camera * 2)(*[abi_camera(c) for c in cams])
    s = torch.cuda.current_stream().cuda_stream
    sptrs = (ctypes.c_void_p * 2)(s, s)
    c0 = r.ctxs[0].handle
    for handles, n in (((c0, c0), 2), ((c0, r.ctxs[1].handle), 0), ((c0, r.ctxs[1].handle), 9)):
        arr = (ctypes.c_void_p * 2)(*handles)
        with pytest.raises(InvalidInputError):
            _lib.check(c0, L.lmgs_render_group(arr, n, ctypes.byref(g), cam_arr, ctypes.byref(st),
                                               frames, sptrs), "lmgs_render_group")


def test_group_mixed_image_sizes(scene):
    """Views of one group may differ in image size: each keeps its own
    tile grid (K1 takes every view's camera), outputs equal render()'s."""
    import ctypes

    from paper_2503_21364_b200 import _lib, render
    from paper_2503_21364_b200.raster import _ptr, abi_camera, abi_settings

    _, model = scene
    L = _lib.lib()
    specs = [(320, 200), (97, 131), (640, 360)]
    cams = [scenes.orbit_cameras(3, w, h, seed=9)[i] for i, (w, h) in enumerate(specs)]
    ctxs = [_lib.Context(0) for _ in specs]
    outs, frames = [], []
    for w, h in specs:
        o = {"rgb": torch.empty((h, w, 3), device="cuda"), "alpha": torch.empty((h, w), device="cuda"),
             "touched": torch.empty(model.count, dtype=torch.int32, device="cuda"),
             "kept": torch.empty(model.count, dtype=torch.uint8, device="cuda"),
             "ranges": torch.empty((-(-w // 16) * -(-h // 16), 2), dtype=torch.int32, device="cuda")}
        outs.append(o)
        frames.append(_lib.Frame(_ptr(o["rgb"]), _ptr(o["alpha"]), None, None, _ptr(o["touched"]),
                                 _ptr(o["kept"]), _ptr(o["ranges"]), None))
    n = len(specs)
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(ctxs[0].handle, L.lmgs_render_group(
        (ctypes.c_void_p * n)(*[c.handle for c in ctxs]), n, ctypes.byref(model._abi()),
        (_lib.Camera * n)(*[abi_camera(c) for c in cams]),
        ctypes.byref(abi_settings(16, 3, (0.1, 0.2, 0.3), 0)), (_lib.Frame * n)(*frames),
        (ctypes.c_void_p * n)(*([s] * n))), "lmgs_render_group")
    torch.cuda.synchronize()
    for cam, o in zip(cams, outs):
        ref = render(cam, model, 16, (0.1, 0.2, 0.3))
        torch.cuda.synchronize()
        assert torch.equal(o["rgb"], ref.rgb)
        assert torch.equal(o["alpha"], ref.alpha)
        assert torch.equal(o["touched"], ref.touched)
        assert torch.equal(o["kept"], ref.kept)
        assert torch.equal(o["ranges"], ref.tile_ranges)


def test_concurrent_batch_equals_lone_renders():
    """A batch over several streams (LMGS_FLAG_CONCURRENT: persistent one-CTA-
    per-SM sort grids, look-back after ranking, packed tile pass) equals one
    render() per view with the one-CTA-per-tile grids, at 1080p where every
    pass walks thousands of tiles per CTA."""
    from paper_2503_21364_b200.raster import render

    model = GaussianModel.from_host(scenes.synthetic_gaussians(200_000, seed=9), validate=False)
    cams = scenes.orbit_cameras(6, 1920, 1080, seed=9)
    got = _render_all(model, cams, 1920, 1080, 2, n_streams=4)
    for i, cam in enumerate(cams):
        o = render(cam, model, 16, sh_eval_degree=3)
        torch.cuda.synchronize()
        ref = {"rgb": o.rgb, "alpha": o.alpha, "depth": o.depth, "touched": o.touched,
               "kept": o.kept, "ranges": o.tile_ranges, "nproc": o.n_processed}
        for f in FIELDS:
            assert torch.equal(ref[f].cpu(), got[f][i]), (i, f)
