"""bench.py's launch and multi-rank accounting (CPU; gloo for world size 2).

The driver runs ``bench.py --gpus N`` (re-executed under torchrun) or
``torchrun --nproc-per-node N bench.py --gpus N``: the job must refuse a
mismatched request, time as the max over ranks and count every rank's frames
(strong scaling over the fixed 64-view batch)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2503_21364_b200.distributed import camera_shard  # noqa: E402


def test_launch_check_decisions():
    assert bench.launch_check(1, env={}) == "run"
    assert bench.launch_check(4, env={}, visible_gpus=8) == "spawn"
    assert bench.launch_check(2, env={"WORLD_SIZE": "2"}) == "run"
    with pytest.raises(SystemExit, match="needs 2 visible GPUs, found 1"):
        bench.launch_check(2, env={}, visible_gpus=1)
    with pytest.raises(SystemExit, match="WORLD_SIZE=1"):
        bench.launch_check(2, env={"WORLD_SIZE": "1"})
    with pytest.raises(SystemExit):
        bench.launch_check(0, env={})


def test_cli_fails_fast_without_enough_gpus():
    """`python bench.py --gpus 2` on a box with fewer GPUs exits non-zero at
    once with a clear message instead of printing n_gpus: 1."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0
    assert "needs 2 visible GPUs" in r.stderr
    assert '"n_gpus"' not in r.stdout


def test_strong_scaling_shards_cover_the_batch():
    for world in (1, 2, 3, 4, 8):
        views = [i for r in range(world) for i in camera_shard(64, r, world)]
        assert views == list(range(64))
        sizes = [len(camera_shard(64, r, world)) for r in range(world)]
        assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms = [40.0, 55.0][rank]  # the slower rank sets the job time
    m = bench.max_over_ranks(ms, world)
    q.put((rank, m, bench.throughput(64, 10, m)))
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for rank, m, fps in res:
        assert m == 55.0
        # 64 views x 10 steps over the slowest rank's 55 ms
        assert fps == pytest.approx(64 * 10 / 0.055)
