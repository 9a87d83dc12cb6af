"""Exact-touched fix-up: queued pixels per view and K7b time at c2 / c3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_21364_b200 import GaussianModel, render, scenes  # noqa: E402
from paper_2503_21364_b200.raster import context  # noqa: E402

for n in (1_000_000, 6_000_000):
    g = scenes.synthetic_gaussians(n, seed=0)
    m = GaussianModel.from_host(g, validate=False)
    ctx = context(0)
    for cam in scenes.orbit_cameras(3, 1920, 1080, seed=0):
        o = render(cam, m, 16, (0, 0, 0), 3, ctx=ctx, stage_times=True)
        print(n, "queued", ctx.touched_fix_count(), "blend+fix ms", round(o.stats["stage_ms"]["blend"], 4))

if len(sys.argv) > 1:  # liblmgs built with -DLMGS_FIX_STATS
    import ctypes

    from paper_2503_21364_b200 import _lib

    h = (ctypes.c_uint * 8)()
    _lib.lib().lmgs_debug_fix_hist(h)
    print("rel bins <1e-7..>=1e-3:", list(h)[:6], "rounds total", h[6], "max", h[7])
