"""Marginal cost of optional stages in the overlapped c3 batch (64 views, 3
streams, pairs): frames/s with the default flags, without K7b
(LMGS_FLAG_NO_TOUCHED_FIX), and without the touched output at all.
Experiment tool, not part of the product.  usage: python stage_cost_probe.py [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2503_21364_b200 import GaussianModel, _lib, scenes  # noqa: E402
from paper_2503_21364_b200.batch import BatchRenderer  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = scenes.synthetic_gaussians(6_000_000, seed=0)
m = GaussianModel.from_host(g, validate=False)
cams = scenes.orbit_cameras(64, 1920, 1080, seed=0)
variants = [("default", 0, True), ("no K7b", _lib.LMGS_FLAG_NO_TOUCHED_FIX, True),
            ("no touched", 0, False)]
for _ in range(reps):
    for name, flags, touched in variants:
        r = BatchRenderer(m, 1920, 1080, 64, n_streams=3, group=2, flags=flags,
                          with_touched=touched)
        for _ in range(3):
            r.render(cams)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            r.render(cams)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"{name:12s} {64e3 / ms:7.1f} frames/s  {ms / 64:.4f} ms/frame", flush=True)
        del r
