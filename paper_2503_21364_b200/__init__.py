"""B200-native 3DGS tile-based forward rasterizer (LandMarkSystem hot path)."""
