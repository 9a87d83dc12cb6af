"""Spatial blocks with the exchange fused into the blend (PeerBlockRenderer,
lmgs_render_strips / lmgs_signal_flags / lmgs_wait_flags).

One GPU is available, so:
* one rank over NCCL with real symmetric memory: the composite equals the
  NCCL-exchange renderer (BlockParallelRenderer) bit for bit, frame after
  frame through the same buffers (epochs);
* two processes on the same GPU whose buffers and flag pads are mapped into
  each other by CUDA IPC (the stand-in for NVLink peer mappings, which torch
  symmetric memory refuses on one device): every strip equals the
  single-process composite of all blocks, over several epochs — the
  cross-process protocol (strip addressing, release/acquire flags, consumed
  handshake) is exercised for real.
"""

import os

import numpy as np
import pytest


def _city():
    from paper_2503_21364_b200 import GaussianModel, scenes

    city = scenes.city_scene(per_block=20_000, width=320, height=180)
    return city, {b: GaussianModel.from_host(g, validate=False) for b, g in enumerate(city.blocks)}


def _reference(city, models):
    import torch

    from paper_2503_21364_b200.distributed import _composite_cuda, block_order, render_block_layer

    cam = city.camera
    layers = torch.stack([render_block_layer(models[b], cam) for b in range(len(models))])
    return _composite_cuda(layers, block_order(np.asarray(cam.center), city.block_bboxes),
                           (0.0, 0.0, 0.0))


@pytest.mark.gpu
def test_peer_renderer_one_rank_matches_nccl_exchange():
    import torch
    import torch.distributed as dist

    from paper_2503_21364_b200.distributed import BlockParallelRenderer, PeerBlockRenderer

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = "29641"
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        city, models = _city()
        cam = city.camera
        nb = len(models)
        pr = PeerBlockRenderer(models, city.block_bboxes, nb, cam.width, cam.height)
        ref = BlockParallelRenderer(models, city.block_bboxes, nb).render(cam)
        for _ in range(3):
            rgb, alpha, depth = pr.render(cam)
            assert torch.equal(rgb, ref[0]) and torch.equal(alpha, ref[1])
            assert torch.equal(depth, ref[2])
    finally:
        dist.destroy_process_group()


def _ipc_worker(rank, world, port, qs, out_q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_21364_b200.distributed import PeerBlockRenderer, assign_blocks

    city, models = _city()
    nb = len(models)
    keep = []

    def ipc_buffers(n_floats, n_flags):
        buf = torch.zeros(n_floats, dtype=torch.float32, device="cuda:0")
        pad = torch.zeros(max(n_flags, 64), dtype=torch.int32, device="cuda:0")
        for r in range(world):  # hand my buffers to every peer (CUDA IPC)
            if r != rank:
                qs[r].put((rank, buf, pad))
        bufs, pads = {rank: buf}, {rank: pad}
        for _ in range(world - 1):
            r, b, p = qs[rank].get(timeout=120)
            bufs[r], pads[r] = b, p
        keep.extend(list(bufs.values()) + list(pads.values()))
        dist.barrier()
        return buf, [bufs[r].data_ptr() for r in range(world)], \
            [pads[r].data_ptr() for r in range(world)]

    mine = {b: models[b] for b in assign_blocks(nb, world)[rank]}
    cam = city.camera
    pr = PeerBlockRenderer(mine, city.block_bboxes, nb, cam.width, cam.height,
                           buffers=ipc_buffers)
    ref = _reference(city, models)
    ok = True
    for _ in range(3):
        rgb, alpha, depth = pr.render(cam, gather=False)
        torch.cuda.synchronize()
        r0 = rank * pr.strip
        ok &= bool(torch.equal(rgb, ref[0][r0:r0 + rgb.shape[0]]))
        ok &= bool(torch.equal(alpha, ref[1][r0:r0 + rgb.shape[0]]))
        dist.barrier()
    out_q.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_peer_renderer_two_processes_cuda_ipc():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    world = 2
    qs = [ctx.Queue() for _ in range(world)]
    out_q = ctx.Queue()
    ps = [ctx.Process(target=_ipc_worker, args=(r, world, 29651, qs, out_q))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [out_q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(120)
    assert sorted(res) == [(0, True), (1, True)]
    assert all(p.exitcode == 0 for p in ps)


@pytest.mark.gpu
@pytest.mark.parametrize("ts,n_strips", [(16, 3), (8, 2), (24, 5), (16, 1)])
def test_render_strips_equals_render(ts, n_strips):
    """lmgs_render_strips writes exactly the pixels lmgs_render does (C + T bg,
    T_final, depth), row y into strip y // strip_rows (ragged last strip)."""
    import ctypes

    import torch

    from paper_2503_21364_b200 import GaussianModel, _lib, render, scenes
    from paper_2503_21364_b200.raster import abi_camera, abi_settings, context

    g = scenes.synthetic_gaussians(20_000, seed=9)
    cam = scenes.orbit_cameras(1, 150, 97, seed=9)[0]
    model = GaussianModel.from_host(g)
    bg = (0.1, 0.2, 0.3)
    ref = render(cam, model, ts, bg, 3, out={"transmittance": torch.empty((97, 150),
                                                                          device="cuda")})
    rows = -(-97 // n_strips)
    rgb = [torch.zeros((rows, 150, 3), device="cuda") for _ in range(n_strips)]
    trans = [torch.zeros((rows, 150), device="cuda") for _ in range(n_strips)]
    depth = [torch.zeros((rows, 150), device="cuda") for _ in range(n_strips)]
    t = _lib.StripTargets()
    t.n_strips, t.strip_rows = n_strips, rows
    for i in range(n_strips):
        t.rgb[i], t.trans[i], t.depth[i] = rgb[i].data_ptr(), trans[i].data_ptr(), \
            depth[i].data_ptr()
    ctx = context(0)
    g_abi, c_abi, s_abi = model._abi(), abi_camera(cam), abi_settings(ts, 3, bg)
    _lib.check(ctx.handle, _lib.lib().lmgs_render_strips(
        ctx.handle, ctypes.byref(g_abi), ctypes.byref(c_abi), ctypes.byref(s_abi),
        ctypes.byref(t), None, torch.cuda.current_stream().cuda_stream), "lmgs_render_strips")
    torch.cuda.synchronize()
    got_rgb = torch.cat(rgb)[:97]
    assert torch.equal(got_rgb, ref.rgb)
    assert torch.equal(torch.cat(trans)[:97], ref.transmittance)
    assert torch.equal(torch.cat(depth)[:97], ref.depth)


@pytest.mark.gpu
@pytest.mark.slow
def test_c5_full_size_blocks_and_composite_vs_oracle():
    """Config 5 at its named size: 8 city blocks of 6.25M Gaussians (50M),
    1080p.  Every block layer (premultiplied RGB with background 0, T_final)
    against the CPU oracle's render of the same block (1e-4), block tile lists
    bit-exact for the front block, and the CUDA front-to-back composite
    against the oracle layers composited in the same block order."""
    import torch

    import oracle
    from paper_2503_21364_b200 import GaussianModel, render, scenes
    from paper_2503_21364_b200.distributed import _composite_cuda, block_order, composite_numpy

    bbs = scenes.city_block_bboxes()
    cam = scenes.city_camera()
    order = block_order(np.asarray(cam.center), bbs)
    gpu_layers, ref_layers = [], []
    for b in range(len(bbs)):
        g = scenes.city_block(b, 6_250_000, 3, bbs)
        m = GaussianModel.from_host(g, validate=False)
        trans = torch.empty((cam.height, cam.width), dtype=torch.float32, device=m.device)
        o = render(cam, m, 16, (0.0, 0.0, 0.0), 3, out={"transmittance": trans},
                   with_instances=(b == order[0]))
        torch.cuda.synchronize()
        ref = oracle.render(g, cam, 16, (0.0, 0.0, 0.0), sh_eval_degree=3)
        assert np.abs(o.rgb.cpu().double().numpy() - ref["image"]).max() <= 1e-4, b
        assert np.abs(trans.cpu().double().numpy() - ref["t_final"]).max() <= 1e-4, b
        if b == order[0]:
            assert o.n_instances == ref["K"]
            np.testing.assert_array_equal(o.inst_prim_ids.cpu().numpy(), ref["inst_prim"])
        gpu_layers.append(torch.cat([o.rgb, trans[..., None], o.depth[..., None]], -1))
        ref_layers.append(np.concatenate([ref["image"], ref["t_final"][..., None],
                                          ref["depth"][..., None]], -1))
        del m, o, trans, ref, g
    rgb, alpha, _ = _composite_cuda(torch.stack(gpu_layers), order, (0.0, 0.0, 0.0))
    want_rgb, want_alpha, _ = composite_numpy(np.stack(ref_layers), order, (0.0, 0.0, 0.0))
    assert np.abs(rgb.cpu().double().numpy() - want_rgb).max() <= 1e-4
    assert np.abs(alpha.cpu().double().numpy() - want_alpha).max() <= 1e-4
