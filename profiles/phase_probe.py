import os, sys
sys.path.insert(0, "/root/repo")
os.environ["LMGS_PHASES"] = "1"
import torch
from paper_2503_21364_b200 import GaussianModel, render, scenes
g = scenes.synthetic_gaussians(6_000_000, seed=0)
m = GaussianModel.from_host(g, validate=False)
cams = scenes.orbit_cameras(64, 1920, 1080, seed=0)
for i in range(3):
    render(cams[i], m, 16, sh_eval_degree=3)
torch.cuda.synchronize()
