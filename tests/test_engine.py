"""Engine runtime shim (engine_api.py:131-133, 291-299, 312-339)."""

import numpy as np
import pytest

from paper_2503_21364_b200.engine import Engine, EngineConfig
from paper_2503_21364_b200.errors import InvalidConfigError, InvalidInputError


def test_unknown_runtime_is_config_error():
    with pytest.raises(InvalidConfigError):
        EngineConfig(runtime="tensorrt")
    for rt in ("cuda", "optimized", "reference"):
        assert EngineConfig(runtime=rt).runtime == rt


def test_bad_tile_size_is_config_error():
    with pytest.raises(InvalidConfigError):
        EngineConfig(tile_size=0)


@pytest.mark.gpu
def test_engine_render_equals_render_image(golden_case):
    from paper_2503_21364_b200 import render_image

    c = golden_case("ragged_100x70_ts16")
    eng = Engine(c.gaussians, config=EngineConfig(runtime="optimized", tile_size=16,
                                                  background=c.background))
    img, stats = eng.render(c.camera)
    assert img.dtype == np.float64 and img.shape == (70, 100, 3)
    assert stats["latency_ms"] > 0
    ref, _ = render_image(c.gaussians, c.camera, 16, c.background)
    np.testing.assert_array_equal(img, ref.cpu().double().numpy())
    assert np.abs(img - c.image).max() <= 1e-4
    with pytest.raises(InvalidInputError):
        eng.render("not a camera")


@pytest.mark.gpu
def test_offload_engine_matches_full_model():
    """test_engine_api.py:210-218: the onload-region engine renders what the
    full model renders (here bit for bit) within its byte budget."""
    import numpy as np

    from paper_2503_21364_b200 import scenes
    from paper_2503_21364_b200.engine import EngineConfig, OffloadConfig, init_inference

    g = scenes.synthetic_gaussians(3000, seed=21, sh_degree=1)
    cams = scenes.orbit_cameras(3, 64, 48, seed=21)
    off = OffloadConfig(budget_bytes=10**9, local_plane_split=(2, 2))
    eng = init_inference(g, None, EngineConfig(offload=off))
    full = init_inference(g, None, EngineConfig())
    for cam in cams:
        a, stats = eng.render(cam)
        b, _ = full.render(cam)
        assert np.array_equal(a, b)
        assert 0 < stats["resident_bytes"] <= off.budget_bytes


@pytest.mark.gpu
def test_offload_budget_fail_fast():
    """test_engine_api.py:221-231."""
    from paper_2503_21364_b200 import scenes
    from paper_2503_21364_b200.engine import EngineConfig, OffloadConfig, init_inference
    from paper_2503_21364_b200.offload import BudgetExceededError

    g = scenes.synthetic_gaussians(3000, seed=21, sh_degree=1)
    total = g.count * 8 * (11 + 3 * 4)
    off = OffloadConfig(budget_bytes=total // 100, local_plane_split=(2, 2))
    with pytest.raises(BudgetExceededError) as exc:
        init_inference(g, None, EngineConfig(offload=off))
    assert "budget" in str(exc.value) and "onload region" in str(exc.value)
