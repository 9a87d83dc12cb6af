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
