"""Config 5 across GPUs: the 50M-Gaussian city in 8 spatial blocks, rendered
block-parallel (one process per GPU) with the layer exchange fused into the
blend (PeerBlockRenderer: lmgs_render_strips into the compositing ranks'
symmetric-memory strips) or through NCCL (BlockParallelRenderer).

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \\
        --master-addr 127.0.0.1 --master-port P bench_blocks.py [--exchange peer|nccl]

Each rank generates only its own blocks (round robin).  Timing: CUDA events
on the rendering stream around K frames after W warm-up frames, barrier +
synchronize on both sides, max over ranks; rank 0 prints one JSON line.
`scaling` is "strong": the scene and frame are fixed, the blocks spread over
more GPUs.  (This image's GPU box has one GPU; the N=1 run is the measured
one here, N>1 needs an NVLink box.)
"""

from __future__ import annotations

import argparse
import json
import os

import numpy as np
import torch
import torch.distributed as dist


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--per-block", type=int, default=6_250_000)
    ap.add_argument("--exchange", choices=("peer", "nccl"), default="peer")
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29691")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)

    from paper_2503_21364_b200 import GaussianModel, scenes
    from paper_2503_21364_b200.distributed import (BlockParallelRenderer, PeerBlockRenderer,
                                                   assign_blocks)

    bboxes = scenes.city_block_bboxes()
    nb = len(bboxes)
    mine = assign_blocks(nb, world)[rank]
    models = {b: GaussianModel.from_host(scenes.city_block(b, a.per_block, 3, bboxes), device=dev,
                                         validate=False) for b in mine}
    cam = scenes.city_camera()
    if a.exchange == "peer":
        r = PeerBlockRenderer(models, bboxes, nb, cam.width, cam.height)
        frame = lambda: r.render(cam)  # noqa: E731
    else:
        r = BlockParallelRenderer(models, bboxes, nb)
        frame = lambda: r.render(cam)  # noqa: E731
    for _ in range(a.warmup):
        frame()
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.steps):
        out = frame()
    e.record()
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([s.elapsed_time(e)], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / a.steps
    if rank == 0:
        print(json.dumps({
            "metric": "c5 frames/s (50M-Gaussian city, 8 blocks, 1080p)",
            "value": 1e3 / ms, "unit": "frames/s", "n_gpus": world, "ms_per_frame": ms,
            "steps": a.steps, "warmup": a.warmup, "scaling": "strong", "exchange": a.exchange,
            "blocks_per_rank": [len(x) for x in assign_blocks(nb, world)],
            "alpha_mean": float(out[1].mean()), "data": "synthetic",
            "config": {"workload": "c5", "gaussians": a.per_block * nb, "width": cam.width,
                       "height": cam.height}}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
