"""B200-native 3DGS tile-based forward rasterizer (LandMarkSystem hot path).

Public API (mirrors pkg/src/landmark/gaussian_core.py):
    GaussianModel, render_image, render, project, composite_blocks
    Camera, look_at_camera                      (data_io.py:42-89)
    Engine                                      (engine_api.py runtime switch)
Compute runs in liblmgs.so (hand-written sm_100a CUDA, include/lmgs.h).
"""

from .camera import Camera, camera_constants, look_at_camera  # noqa: F401
from .errors import (FormatError, InvalidConfigError, InvalidInputError, LmgsError,  # noqa: F401
                     ShapeError)
from .raster import (GaussianModel, RenderOutput, RenderRecord, TileRecord,  # noqa: F401
                     composite_blocks, project, render, render_image)

__all__ = ["Camera", "look_at_camera", "camera_constants", "GaussianModel", "render",
           "render_image", "project", "composite_blocks", "RenderOutput", "RenderRecord",
           "TileRecord", "InvalidInputError", "ShapeError", "InvalidConfigError", "LmgsError",
           "FormatError"]
