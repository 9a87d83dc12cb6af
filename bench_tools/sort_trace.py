"""Phase timeline of one onesweep pass (build with -DLMGS_SORT_TRACE=<pass+1>).

usage: python bench_tools/sort_trace.py [concurrent 0|1]
Renders one c3 view (serial, one stream) and prints per-phase tile durations
(median / p90, microseconds) of the traced pass's tiles: load + early counts,
look-back, ranking, staging, write-out; plus the pass span and tiles in flight.
"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_21364_b200 import GaussianModel, _lib, scenes  # noqa: E402
from paper_2503_21364_b200.batch import BatchRenderer  # noqa: E402

conc = int(sys.argv[1]) if len(sys.argv) > 1 else 0
g = GaussianModel.from_host(scenes.synthetic_gaussians(6_000_000, seed=0), validate=False)
cams = scenes.orbit_cameras(64, 1920, 1080, seed=0)[:1]
r = BatchRenderer(g, 1920, 1080, 1, n_streams=1, group=1)
if conc:
    r.flags |= _lib.LMGS_FLAG_CONCURRENT
L = _lib.lib()
for _ in range(2):
    r.render(cams)
torch.cuda.synchronize()
L.lmgs_debug_sort_trace_reset()
r.render(cams)
torch.cuda.synchronize()
buf = np.zeros((1 << 14, 7), np.uint64)
L.lmgs_debug_sort_trace(ctypes.c_void_p(buf.ctypes.data), ctypes.c_size_t(buf.nbytes))
t = buf[buf[:, 0] > 0].astype(np.int64)
t0 = t[:, 0].min()
names = ["load+count", "look-back", "rank", "stage", "write"]
print(f"concurrent={conc} tiles={len(t)} span={(t[:, 5].max() - t0) / 1e3:.1f} us "
      f"ctas={len(np.unique(t[:, 6]))}")
for k, nm in enumerate(names):
    d = (t[:, k + 1] - t[:, k]) / 1e3
    print(f"  {nm:11s} median {np.median(d):6.2f}  p90 {np.percentile(d, 90):6.2f}  "
          f"mean {d.mean():6.2f} us")
tot = (t[:, 5] - t[:, 0]) / 1e3
print(f"  tile total  median {np.median(tot):6.2f}  p90 {np.percentile(tot, 90):6.2f}")
# tiles in flight over time
grid = np.linspace(t0, t[:, 5].max(), 50)
inflight = [int(((t[:, 0] <= x) & (t[:, 5] > x)).sum()) for x in grid]
print("  in flight:", inflight[::5])
# start-time gaps between consecutive tickets
st = np.sort(t[:, 0])
print(f"  ticket rate: {len(st) / ((st[-1] - st[0]) / 1e3):.1f} tiles/us")
