"""Render a few c3 views (6M Gaussians, 1080p) for ncu: warm-up views first,
then the profiled ones.  usage: python profiles/view_probe.py [n_views] [width height] [group] [flags]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2503_21364_b200 import GaussianModel, scenes  # noqa: E402
from paper_2503_21364_b200.batch import BatchRenderer  # noqa: E402

nv = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w, h = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (1920, 1080)
g = scenes.synthetic_gaussians(6_000_000, seed=0)
m = GaussianModel.from_host(g, validate=False)
cams = scenes.orbit_cameras(64, w, h, seed=0)[:nv]
grp = int(sys.argv[4]) if len(sys.argv) > 4 else 1
flags = int(sys.argv[5]) if len(sys.argv) > 5 else 0  # extra LMGS_FLAG_* bits
r = BatchRenderer(m, w, h, nv, group=grp, flags=flags)
r.render(cams, stage_times=True)
torch.cuda.synchronize()
st = r.render(cams, stage_times=True)
torch.cuda.synchronize()
print({k: round(v / nv, 4) for k, v in st["stage_ms"].items()}, st["per_frame"])
