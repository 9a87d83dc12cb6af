import torch
from paper_2503_21364_b200 import GaussianModel, render, scenes
g = scenes.synthetic_gaussians(6_000_000, seed=0)
m = GaussianModel.from_host(g, validate=False)
for cam in scenes.orbit_cameras(4, 1920, 1080, seed=0):
    o = render(cam, m, 16, (0,0,0), 3, stage_times=True)
    print(o.stats)
