"""Backward probe for ncu: 1M Gaussians at 1080p (the bench_configs `bw`
scene), one forward + `reps` backward passes of view 0."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_21364_b200 import GaussianModel, render, scenes
from paper_2503_21364_b200.raster import context
from paper_2503_21364_b200.train import _backward

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = scenes.synthetic_gaussians(1_000_000, seed=0)
model = GaussianModel.from_host(g, validate=False)
cam = scenes.orbit_cameras(4, 1920, 1080, seed=0)[0]
ctx = context(0)
gen = torch.Generator(device="cuda").manual_seed(0)
gimg = torch.randn((1080, 1920, 3), generator=gen, device="cuda")
render(cam, model, 16, (0.0, 0.0, 0.0), 1, ctx=ctx)
for _ in range(reps):
    _backward(ctx, model, cam, gimg, 16, (0.0, 0.0, 0.0), 1)
torch.cuda.synchronize()
