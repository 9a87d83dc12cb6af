"""Fused emission + tile sort (k_emit_ranks: rank records + per-row digit
histograms -> the onesweep pass that generates its instance keys -> the
packed second pass with the range counts) against the
separate K4 emission + two-pass K5 tile sort (the default; the fused path is
LMGS_FLAG_FUSED_TILE_SORT):
tile lists, ranges, touched, n_processed and images bit-identical, and a
fused-only tile count (1080p at 8-px tiles, 32,400 tiles) against the oracle.
"""

import numpy as np
import pytest
import torch

from paper_2503_21364_b200 import _lib, scenes
from paper_2503_21364_b200.batch import BatchRenderer
from paper_2503_21364_b200.raster import GaussianModel, render
from test_gpu_parity import IMG_TOL, _full_frame_check
from test_gpu_pipeline import _front_camera

pytestmark = pytest.mark.gpu


def _ab(g, cam, ts=16, prim_ids=None, deg=3):
    model = g if isinstance(g, GaussianModel) else GaussianModel.from_host(g, validate=False)
    outs = []
    for fused in (True, False):
        o = render(cam, model, ts, sh_eval_degree=deg, with_instances=True, prim_ids=prim_ids,
                   out={"transmittance": None}, fused_tile_sort=fused)
        torch.cuda.synchronize()
        outs.append(o)
    a, b = outs
    assert a.n_instances == b.n_instances
    for f in ("inst_keys", "inst_prim_ids", "tile_ranges", "touched", "kept", "n_processed",
              "rgb", "alpha", "depth"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f
    return a


@pytest.mark.parametrize("w,h,ts", [(1920, 1080, 16), (1920, 1080, 8), (1920, 1080, 12),
                                    (3840, 2160, 16), (272, 256, 16), (4096, 64, 16),
                                    (64, 4096, 16), (1000, 700, 5)])
def test_fused_equals_unfused(w, h, ts):
    g = scenes.synthetic_gaussians(150_000, seed=w + h + ts)
    cam = scenes.orbit_cameras(1, w, h, seed=ts)[0]
    out = _ab(g, cam, ts)
    assert out.n_instances > 0


def test_fused_giant_splats_and_subset():
    """Splats covering thousands of tiles (one rank spans many sort tiles of
    4096 slots) plus a prim-id remap (render_image's subset)."""
    g = scenes.synthetic_gaussians(20_000, seed=11)
    big = scenes.synthetic_gaussians(8, seed=12)
    big.scales[:] = 2.5
    big.means[:, :] *= 0.2
    cat = scenes.HostGaussians(np.concatenate([g.means, big.means]),
                               np.concatenate([g.quats, big.quats]),
                               np.concatenate([g.scales, big.scales]),
                               np.concatenate([g.opacity_logits, big.opacity_logits]),
                               np.concatenate([g.sh, big.sh]), g.sh_degree)
    cam = scenes.orbit_cameras(1, 1920, 1080, seed=1)[0]
    n = cat.means.shape[0]
    pid = torch.randperm(n, generator=torch.Generator().manual_seed(5)).to(torch.int64)
    out = _ab(cat, cam, 16, prim_ids=pid.cuda())
    counts = (out.tile_ranges[:, 1] - out.tile_ranges[:, 0]).cpu()
    assert int(counts.max()) > 0


def test_fused_empty_and_all_culled():
    g = scenes.synthetic_gaussians(1000, seed=2)
    g.means[:, 2] = -50.0  # behind the camera at the origin looking down +z
    cam = _front_camera(1920, 1080)
    out = _ab(g, cam, 16)
    assert out.n_instances == 0
    empty = scenes.synthetic_gaussians(0, seed=0)
    _ab(empty, cam, 16)


def test_fused_tiles_8px_1080p_vs_oracle():
    """32,400 tiles (two 8-bit digits, the largest coverage array the fused
    path takes at 1080p) against the CPU oracle."""
    g = scenes.synthetic_gaussians(60_000, seed=4)
    cam = scenes.orbit_cameras(1, 1920, 1080, seed=4)[0]
    r = _full_frame_check(g, cam, ts=8, fused_tile_sort=True)
    assert r["err"] <= IMG_TOL and r["aerr"] <= IMG_TOL
    assert r["touched_mismatch"] == 0 and r["nproc_mismatch"] == 0


def test_fused_no_host_sync_and_overflow():
    """The capacity-bounded mode: equal to the synchronised render when K fits;
    with a capacity below K the view is flagged and the ranges stay inside it."""
    g = GaussianModel.from_host(scenes.synthetic_gaussians(100_000, seed=6), validate=False)
    cams = scenes.orbit_cameras(2, 1920, 1080, seed=6)
    fl = _lib.LMGS_FLAG_FUSED_TILE_SORT
    ref = BatchRenderer(g, 1920, 1080, 2, flags=fl)
    ref.render(cams)
    torch.cuda.synchronize()
    k = max(c.stats()["n_instances"] for c in ref.ctxs if c.stats()["n_instances"] > 0)
    ok = BatchRenderer(g, 1920, 1080, 2, capacity=2 * k, flags=fl)
    ok.render(cams)
    torch.cuda.synchronize()
    assert not ok.overflowed()
    for f in ("rgb", "ranges", "nproc", "touched"):
        assert torch.equal(getattr(ok, f), getattr(ref, f)), f
    small = BatchRenderer(g, 1920, 1080, 2, capacity=k // 2, flags=fl)
    small.render(cams)
    torch.cuda.synchronize()
    assert small.overflowed()
    r = small.ranges.long()
    assert int(r.min()) >= 0 and int(r.max()) <= k // 2
    assert bool((r[..., 1] >= r[..., 0]).all())
