"""Debug counters of the backward (liblmgs built with -DLMGS_BW_COUNT): per
pass, warp-splat evaluations, live lanes, live lanes inside the circle."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_21364_b200 import GaussianModel, _lib, render, scenes  # noqa: E402
from paper_2503_21364_b200.raster import context  # noqa: E402
from paper_2503_21364_b200.train import _backward  # noqa: E402

g = scenes.synthetic_gaussians(1_000_000, seed=0)
model = GaussianModel.from_host(g, validate=False)
cam = scenes.orbit_cameras(4, 1920, 1080, seed=0)[0]
ctx = context(0)
gimg = torch.randn((1080, 1920, 3), device="cuda")
fwd = render(cam, model, 16, (0.0, 0.0, 0.0), 1, ctx=ctx)
_backward(ctx, model, cam, gimg, 16, (0.0, 0.0, 0.0), 1)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
assert _lib.lib().lmgs_debug_bw_count(buf) == 0
for p in range(2):
    ev, lv, ins = buf[4 * p], buf[4 * p + 1], buf[4 * p + 2]
    print(f"pass {p}: warp-splat evals {ev/1e6:.2f}M, live lanes/eval {lv/ev:.1f}, "
          f"inside lanes/eval {ins/ev:.2f}")
print("instances", fwd.n_instances)
