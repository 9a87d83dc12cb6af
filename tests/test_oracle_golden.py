"""The CPU oracle against the reference's own outputs (golden fixtures).

Pins oracle/oracle.c before it is trusted as the checker for the CUDA path:
tile lists and touched counts bit-exact, image / alpha within 1e-12
(the reference blends in fp64 with MKL exp; the oracle with libm exp).
"""

import numpy as np
import pytest

import oracle
from conftest import GOLDEN_CASES


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_oracle_matches_reference(golden_case, name):
    c = golden_case(name)
    o = oracle.render(c.gaussians, c.camera, c.tile_size, c.background, sh_eval_degree=1,
                      subset=c.subset)
    assert o["K"] == len(c.lists)
    np.testing.assert_array_equal(o["offsets"], c.offsets)
    np.testing.assert_array_equal(o["inst_prim"], c.lists)
    np.testing.assert_array_equal(o["splats"]["prim_id"], c.splat_prim_id)
    np.testing.assert_array_equal(o["touched"], c.touched)
    assert np.abs(o["image"] - c.image).max() <= 1e-12
    assert np.abs(o["t_final"] - c.t_final).max() <= 1e-12


@pytest.mark.parametrize("name", ["c1_10k_256", "ragged_130x67_ts8", "ragged_67x45_ts10",
                                  "ties_dup_ts16", "nearcull_ts16"])
def test_oracle_rect_predicate_equals_brute_force(golden_case, name):
    """The per-splat tile-range restatement == the reference's per-tile mask."""
    c = golden_case(name)
    a = oracle.render(c.gaussians, c.camera, c.tile_size, c.background, subset=c.subset)
    b = oracle.render(c.gaussians, c.camera, c.tile_size, c.background, subset=c.subset,
                      brute=True)
    np.testing.assert_array_equal(a["offsets"], b["offsets"])
    np.testing.assert_array_equal(a["lists"], b["lists"])


def test_oracle_margin_certifies_c1(golden_case):
    """No bbox edge within 1e-9 px of a tile boundary: a 1-ulp radius change
    (the reference's MKL sqrt) cannot flip a tile membership."""
    c = golden_case("c1_10k_256")
    sp = oracle.project(c.gaussians, c.camera)
    assert oracle.margin(sp, 256, 256, 16) > 1e-9


def test_oracle_tile_subset_blend(golden_case):
    c = golden_case("c1_10k_256")
    full = oracle.render(c.gaussians, c.camera)
    tiles = np.array([0, 17, 100, 255])
    part = oracle.render(c.gaussians, c.camera, tiles=tiles)
    ts = 16
    for t in tiles:
        ty, tx = divmod(int(t), 256 // ts)
        sl = (slice(ty * ts, ty * ts + ts), slice(tx * ts, tx * ts + ts))
        np.testing.assert_array_equal(part["image"][sl], full["image"][sl])
    np.testing.assert_array_equal(part["n_processed"][tiles], full["n_processed"][tiles])
