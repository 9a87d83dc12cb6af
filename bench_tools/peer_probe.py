"""Probe the fused peer-store block renderer.

  python bench_tools/peer_probe.py 1        # one rank (NCCL), compare with BlockParallelRenderer
  python bench_tools/peer_probe.py 2        # two processes on the same GPU (gloo group)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def scene():
    from paper_2503_21364_b200 import GaussianModel, scenes

    city = scenes.city_scene(per_block=20_000, width=320, height=180)
    models = {b: GaussianModel.from_host(g, validate=False) for b, g in enumerate(city.blocks)}
    return city, models


def run(rank, world, backend, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    kw = {"device_id": torch.device("cuda:0")} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    from paper_2503_21364_b200.distributed import (BlockParallelRenderer, PeerBlockRenderer,
                                                   assign_blocks)

    city, models = scene()
    nb = len(city.blocks)
    mine = {b: models[b] for b in assign_blocks(nb, world)[rank]}
    cam = city.camera
    pr = PeerBlockRenderer(mine, city.block_bboxes, nb, cam.width, cam.height)
    outs = []
    for _ in range(3):  # several epochs through the same buffers
        outs.append(pr.render(cam, gather=(backend == "nccl")))
    torch.cuda.synchronize()
    if rank == 0:
        full = BlockParallelRenderer(models, city.block_bboxes, nb, group=None)
        ref = None
        if world == 1:
            ref = full.render(cam)
        else:
            from paper_2503_21364_b200.distributed import render_block_layer, _composite_cuda
            from paper_2503_21364_b200.distributed import block_order
            layers = torch.stack([render_block_layer(models[b], cam) for b in range(nb)])
            ref = _composite_cuda(layers, block_order(np.asarray(cam.center), city.block_bboxes),
                                  (0.0, 0.0, 0.0))
        rgb = outs[-1][0]
        rows = rgb.shape[0]
        d = (rgb - ref[0][:rows]).abs().max().item()
        same = all(torch.equal(o[0], outs[0][0]) for o in outs)
        q.put((rank, rows, d, same))
    else:
        q.put((rank, None, None, None))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    backend = "nccl" if world == 1 else "gloo"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=run, args=(r, world, backend, 29611 + world, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
    while not q.empty():
        print(q.get())
    print("exit codes", [p.exitcode for p in ps])
