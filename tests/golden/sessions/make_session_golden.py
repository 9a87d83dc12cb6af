"""Golden outputs of the reference's streaming sessions (build container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/sessions/make_session_golden.py

run_session (render_runtime.py:250-308) over the crossing trajectory of
test_render_runtime.py:37-52 on generate_synthetic_scene(41, 80 prims), in
every mode: images and FrameStats.  Cases:
  static        static_full
  block_2x2     block_double_buffer, 2x2 grid, budget 1 GiB, instant transfers
  block_4x4_bw  block_double_buffer, 4x4 grid, 1e4 B/s (stalls)
  frustum       frustum_voxel, voxel 2.0, budget 1 GiB
  frustum_tight frustum_voxel, voxel 2.0, tightest feasible budget (evictions)
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from landmark.common import VirtualClock  # noqa: E402
from landmark.data_io import generate_synthetic_scene, look_at_camera  # noqa: E402
from landmark.memory_tiers import TransferConfig  # noqa: E402
from landmark.render_runtime import SessionConfig, run_session  # noqa: E402
from landmark.scene_manager import (frustum_visible_voxels, partition_scene,  # noqa: E402
                                    reorder_voxel_grid)


def crossing(scene, n=24, size=24):
    xs = np.linspace(scene.bbox[0, 0] + 0.3, scene.bbox[1, 0] - 0.3, n)
    cams = [look_at_camera((x, -1.0, 0.5), (x, 3.0, 0.0), fov_deg=70.0, width=size, height=size,
                           near=0.01, far=300.0) for x in xs]
    return cams, np.linspace(0.0, float(n) / 4, n)


def main():
    scene = generate_synthetic_scene(41, n_prims=80, n_cameras=2, image_size=24)
    m = scene.model
    cams, times = crossing(scene)
    index, _ = reorder_voxel_grid(m, 2.0)
    per_prim = sum(t.numel() * t.element_size() for t in (m.means, m.quats, m.scales,
                                                          m.opacity_logits, m.sh)) // m.count + 8
    tight = max(sum(int(index.ranges[v, 1] - index.ranges[v, 0]) * per_prim
                    for v in frustum_visible_voxels(index, c)) for c in cams)
    cases = {
        "static": (SessionConfig(mode="static_full"), None),
        "block_2x2": (SessionConfig(mode="block_double_buffer", budget_bytes=1 << 30),
                      partition_scene(scene.bbox, 2, 2)),
        "block_4x4_bw": (SessionConfig(mode="block_double_buffer", budget_bytes=1 << 30,
                                       transfer=TransferConfig(bandwidth_bytes_per_s=1e4)),
                         partition_scene(scene.bbox, 4, 4)),
        "frustum": (SessionConfig(mode="frustum_voxel", budget_bytes=1 << 30, voxel_size=2.0),
                    None),
        "frustum_tight": (SessionConfig(mode="frustum_voxel", budget_bytes=tight, voxel_size=2.0),
                          None),
    }
    out = dict(means=m.means.numpy(), quats=m.quats.numpy(), scales=m.scales.numpy(),
               opacity_logits=m.opacity_logits.numpy(), sh=m.sh.numpy(), sh_degree=m.sh_degree,
               bbox=scene.bbox, times=times, tight_budget=tight,
               cam_pos=np.array([c.center for c in cams]))
    meta = {}
    for name, (cfg, grid) in cases.items():
        imgs, stats = run_session(m, cams, times, cfg, grid=grid, clock=VirtualClock())
        out[f"img_{name}"] = np.stack([i.numpy() for i in imgs]).astype(np.float32)
        meta[name] = [{k: v for k, v in s.as_dict().items() if k != "latency_ms"} for s in stats]
    out["stats_json"] = json.dumps(meta)
    # host bookkeeping pins: voxel reorder, visible voxels per camera, cell groups
    out["vox_perm"] = index.permutation
    out["vox_ranges"] = index.ranges
    out["vox_keys"] = index.voxel_keys
    out["vox_max_scale"] = index.voxel_max_scale
    vis = [frustum_visible_voxels(index, c) for c in cams]
    out["vis_flat"] = np.concatenate([np.asarray(v, np.int64) for v in vis])
    out["vis_len"] = np.array([len(v) for v in vis])
    from landmark.engine_api import gaussian_cell_groups
    g44 = gaussian_cell_groups(m, partition_scene(scene.bbox, 4, 4))
    out["cells44_ids"] = np.concatenate([g44[c].tensors["ids"].numpy() for c in sorted(g44)])
    out["cells44_len"] = np.array([len(g44[c].tensors["ids"]) for c in sorted(g44)])
    np.savez_compressed(HERE / "sessions.npz", **out)
    print({k: (v[-1]["stalls"], v[-1]["peak_resident_bytes"]) for k, v in meta.items()})


if __name__ == "__main__":
    main()
