"""The coarse-bin tile lists (bins.cu, default) against the instance radix
sort (LMGS_FLAG_TILE_SORT) and the oracle: identical per-tile lists, ranges,
images and touched counts over bin counts of 1 to 32,400 (1 and 2 bin-sort
passes), ragged edges, big and tiny tiles."""

import numpy as np
import pytest
import torch

import oracle
from paper_2503_21364_b200 import GaussianModel, render, scenes

pytestmark = pytest.mark.gpu

CASES = [  # (n, w, h, ts, seed)
    (20_000, 320, 240, 16, 1),      # 20x15 tiles -> 3x2 bins
    (3_000, 40, 30, 16, 2),         # one bin
    (50_000, 1920, 1080, 16, 3),    # 135 bins, one pass
    (50_000, 3840, 2160, 16, 4),    # 510 bins, two passes
    (30_000, 1920, 1080, 1, 5),     # 2,073,600 tiles, 32,400 bins
    (20_000, 1000, 700, 8, 6),
    (20_000, 997, 701, 5, 7),       # ragged bins and tiles
    (20_000, 900, 600, 64, 8),
    (20_000, 900, 600, 128, 9),
]


@pytest.mark.parametrize("n,w,h,ts,seed", CASES)
def test_bins_equal_tile_sort(n, w, h, ts, seed):
    g = scenes.synthetic_gaussians(n, seed=seed)
    cam = scenes.orbit_cameras(1, w, h, seed=seed)[0]
    m = GaussianModel.from_host(g, validate=False)
    a = render(cam, m, ts, (0.1, 0.0, 0.2), 3, with_instances=True)
    b = render(cam, m, ts, (0.1, 0.0, 0.2), 3, with_instances=True, tile_sort=True)
    torch.cuda.synchronize()
    assert a.n_instances == b.n_instances
    assert torch.equal(a.tile_ranges, b.tile_ranges)
    assert torch.equal(a.inst_keys, b.inst_keys)
    assert torch.equal(a.rgb, b.rgb) and torch.equal(a.touched, b.touched)
    assert torch.equal(a.n_processed, b.n_processed)


def test_bins_vs_oracle_full_hd():
    g = scenes.synthetic_gaussians(200_000, seed=21)
    cam = scenes.orbit_cameras(3, 1920, 1080, seed=21)[2]
    out = render(cam, GaussianModel.from_host(g, validate=False), 16, sh_eval_degree=3,
                 with_instances=True)
    torch.cuda.synchronize()
    o = oracle.render(g, cam, 16, sh_eval_degree=3)
    assert out.n_instances == o["K"]
    np.testing.assert_array_equal(out.inst_prim_ids.cpu().numpy(), o["inst_prim"])
    r = out.tile_ranges.cpu().numpy().astype(np.int64)
    np.testing.assert_array_equal(r[:, 1] - r[:, 0], o["tile_counts"])
