"""Benchmark: 1080p frames/s at 6M Gaussians on 1-8 B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--views V] [--impl reference]

Headline workload = config c3: a batch of V = 64 camera views of the
6M-Gaussian synthetic scene (SH degree 3) at 1920x1080, data-parallel over N
GPUs.  One step renders the whole 64-view batch; each rank renders its
contiguous shard of 64 / N views (``distributed.camera_shard``), so the total
work is fixed as N grows: ``"scaling": "strong"``.  The scene is generated on
rank 0 and replicated to the other ranks with an NCCL broadcast
(``distributed.broadcast_scene``, timed as setup).  The weak-scaling variant
(64 views per rank) is reported beside it under ``weak``.  The scene (1.42 GB)
and the per-view working sets exceed the 126 MB L2, so no explicit L2 flush is
inserted between timed steps.

Config c5 (the 50M-Gaussian city in 8 spatial blocks, block-parallel over the
same N ranks with the layer exchange fused into the blend over peer memory)
is measured in the same run and reported under ``c5``.

Launch: with ``--gpus N > 1`` and no torchrun environment the script
re-executes itself under ``torch.distributed.run`` with N local ranks (and
fails at once if fewer than N GPUs are visible); under torchrun it asserts
WORLD_SIZE == N.  Timing: W untimed warm-up steps, then exactly K steps
bracketed by a barrier + cuda.synchronize on both sides, CUDA events on the
launching stream, max over ranks (all_reduce MAX).  Rank 0 prints one JSON
line.

``--impl reference`` times the reference algorithm's CPU implementation (the
fp64 C restatement in oracle/, "port": the reference is pure Python and does
not travel to the GPU box) on the host cores, one full 1080p view of the same
scene per step; under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "1080p frames/sec at 6M Gaussians, 1–8 B200; ms/frame; HBM GB/s vs peak"
UNIT = "frames/s"
N_GAUSS = 6_000_000
W, H = 1920, 1080
BATCH_VIEWS = 64  # config c3: "batch of 64 camera views data-parallel over 1/2/4/8 B200"
C5_PER_BLOCK = 6_250_000

# dram__bytes_read.sum + dram__bytes_write.sum per c3 view of each stage's
# kernels from the committed ncu launch list (stage = sum of its kernels);
# reported as `traffic` beside the algorithmic bytes.
NCU_TRAFFIC_SOURCE = "profiles/r10/ncu_launch_table.txt"
NCU_TRAFFIC = {
    "preprocess": 2784.0e6 / 2,  # one k_preprocess_tma<2> launch serves two views
    # keys, 3 passes (concurrent grids; the first stages 16-bit implicit values), fix-up
    "depth_sort": 48.1e6 + 24.5e6 + 2 * 50.2e6 + 104.9e6,
    "emit": 258.4e6,
    "tile_sort": 222.2e6 + 124.4e6,  # u64 -> packed u32 pass, u32 -> ids pass
    "blend": 159.4e6,
    "touched_fix": 110.3e6,
}


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# launch and multi-rank accounting (unit-tested with gloo: tests/test_bench_dist.py)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def launch_check(gpus: int, env=None, visible_gpus=None) -> str:
    """What to do for ``--gpus gpus``: "run" (this process is the job or one
    of its ranks) or "spawn" (re-execute under torchrun).  Raises SystemExit
    with a message when the request cannot be met."""
    env = os.environ if env is None else env
    if gpus < 1:
        raise SystemExit(f"bench.py: --gpus must be >= 1 (got {gpus})")
    if "WORLD_SIZE" in env:
        world = int(env["WORLD_SIZE"])
        if world != gpus:
            raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world}: launch one "
                             "rank per GPU (torchrun --nproc-per-node N ... --gpus N)")
        return "run"
    if gpus == 1:
        return "run"
    if visible_gpus is None:
        import torch

        visible_gpus = torch.cuda.device_count()
    if visible_gpus < gpus:
        raise SystemExit(f"bench.py: --gpus {gpus} needs {gpus} visible GPUs, found "
                         f"{visible_gpus}")
    return "spawn"


def spawn_torchrun(gpus: int, argv) -> int:
    """Re-execute this script with one rank per GPU (torchrun, 127.0.0.1)."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), str(Path(__file__).resolve()), *argv]
    return subprocess.call(cmd)


def max_over_ranks(value: float, world: int, device=None) -> float:
    """The maximum of a per-rank scalar (all_reduce MAX; identity at world 1)."""
    if world == 1:
        return float(value)
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def throughput(frames_per_step_total: int, steps: int, ms_max: float) -> float:
    """Whole-job frames/s: every rank's frames over the slowest rank's time."""
    return frames_per_step_total * steps / (ms_max / 1e3)


# ---------------------------------------------------------------------------
# reference arm: the CPU implementation of the path (oracle port), host cores


def arm_config(args, world):
    """The workload both arms report (the reference arm times a bounded sample
    of it, described in its cpu_baseline.sample)."""
    views = args.views
    my_views = views // world  # rank 0's shard (distributed.camera_shard)
    return {"workload": f"c3: 6M Gaussians (SH3), 1920x1080, batch of {views} orbit "
                        f"views per step split over {world} GPU(s), tile 16",
            "gaussians": N_GAUSS, "views_per_step": views, "views_per_gpu": my_views,
            "width": W, "height": H, "parallelism": f"camera-batch dp{world}",
            "views_per_k1_launch": args.group, "launch_mode": args.mode,
            "streams": args.streams,
            "sort_grids": "persistent, one CTA per SM (LMGS_FLAG_CONCURRENT)" if args.streams > 1
            else "one CTA per tile",
            "l2": "no flush: scene 1.42 GB and per-view buffers > 126 MB L2",
            "geometry": "fp64 (bit-exact tile lists)", "blend": "fp32",
            "scene_replication": "rank 0 generates, NCCL broadcast" if world > 1
            else "single rank"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    import numpy as np

    import oracle
    from paper_2503_21364_b200 import scenes

    threads = os.cpu_count() or 1
    oracle.set_threads(threads)
    g = scenes.synthetic_gaussians(N_GAUSS, seed=0)
    cams = scenes.orbit_cameras(BATCH_VIEWS, W, H, seed=0)
    times = []
    for step in range(args.warmup + args.steps):
        cam = cams[step % len(cams)]
        t0 = time.perf_counter()
        o = oracle.render(g, cam, 16, sh_eval_degree=3)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
        del o
    sec = float(np.mean(times))
    value = 1.0 / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": arm_config(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": "one full 1080p view of the 6M-Gaussian scene per step "
                                   "(oracle/oracle.c fp64 restatement, OpenMP)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


def cpu_baseline_sample(g, cam):
    """Oracle on the host cores, one view of the same scene (rank 0, N=1)."""
    import oracle

    threads = os.cpu_count() or 1
    oracle.set_threads(threads)
    t0 = time.perf_counter()
    oracle.render(g, cam, 16, sh_eval_degree=3)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"one full 1080p view of the 6M-Gaussian scene ({dt:.1f} s, "
                      "oracle/oracle.c fp64 restatement, OpenMP)"}


def replicate_scene(rank, world, dev):
    """Rank 0 generates the c3 scene; one NCCL broadcast per SoA tensor
    replicates it.  Returns (model, host scene or None, broadcast ms)."""
    import torch

    from paper_2503_21364_b200 import GaussianModel, scenes
    from paper_2503_21364_b200.distributed import broadcast_scene

    g_host = None
    if rank == 0:
        g_host = scenes.synthetic_gaussians(N_GAUSS, seed=0)
        model = GaussianModel.from_host(g_host, device=dev, validate=False)
    else:
        z = lambda *s: torch.empty(s, dtype=torch.float32, device=dev)  # noqa: E731
        model = GaussianModel(z(N_GAUSS, 3), z(N_GAUSS, 4), z(N_GAUSS, 3), z(N_GAUSS),
                              z(N_GAUSS, 16, 3), 3, device=dev, validate=False)
    ms = 0.0
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        broadcast_scene([model.means, model.quats, model.scales, model.opacity_logits,
                         model.sh], src=0)
        b.record()
        torch.cuda.synchronize()
        ms = max_over_ranks(a.elapsed_time(b), world, dev)
    return model, g_host, ms


def single_view_latency(model, cam, reps: int = 10) -> dict:
    """One view through the public ``render`` call (host wait for K
    included), CUDA events around each call, serial, after a warm-up."""
    import torch

    from paper_2503_21364_b200 import render

    render(cam, model, 16, sh_eval_degree=3)
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        render(cam, model, 16, sh_eval_degree=3)
        b.record()
        torch.cuda.synchronize()
        ms.append((a.elapsed_time(b), (time.perf_counter() - t0) * 1e3))
    dev_ms = sorted(m[0] for m in ms)
    wall_ms = sorted(m[1] for m in ms)
    return {"ms": statistics.median(dev_ms), "ms_min": dev_ms[0],
            "wall_ms": statistics.median(wall_ms), "reps": reps,
            "path": "paper_2503_21364_b200.render (lmgs_render) of one c3 view, serial, "
                    "CUDA events on the current stream; target <= 5 ms (north star)"}


def time_steps(step, steps, world, dev, barrier):
    import torch

    stream = torch.cuda.current_stream()
    barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(steps):
        step()
    end.record(stream)
    torch.cuda.synchronize()
    barrier()
    return max_over_ranks(start.elapsed_time(end), world, dev)


def run_c5(args, rank, world, dev, barrier):
    """Config c5: the 8-block city, block-parallel, exchange fused into the
    blend (PeerBlockRenderer).  Strong scaling (fixed scene and frame)."""
    import torch

    from paper_2503_21364_b200 import GaussianModel, render, scenes
    from paper_2503_21364_b200.distributed import (BlockParallelRenderer, PeerBlockRenderer,
                                                   assign_blocks)

    bboxes = scenes.city_block_bboxes()
    nb = len(bboxes)
    owned = assign_blocks(nb, world)
    hosts = {b: scenes.city_block(b, args.c5_per_block, 3, bboxes) for b in owned[rank]}
    models = {b: GaussianModel.from_host(h, device=dev, validate=False) for b, h in hosts.items()}
    cam = scenes.city_camera()
    exchange = ("peer stores in the blend (lmgs_render_strips into symmetric-memory strips) + "
                "strip all_gather")
    try:
        r = PeerBlockRenderer(models, bboxes, nb, cam.width, cam.height)
    except Exception as e:  # no symmetric memory on this node: the NCCL exchange instead
        r = BlockParallelRenderer(models, bboxes, nb)
        exchange = f"NCCL all_to_all of row strips (peer path unavailable: {str(e)[:120]})"
    for _ in range(max(2, args.warmup)):
        out = r.render(cam)
    torch.cuda.synchronize()
    steps = args.c5_steps
    ms = time_steps(lambda: r.render(cam), steps, world, dev, barrier)
    out = r.render(cam)
    torch.cuda.synchronize()
    res = {"metric": "c5 frames/s (50M-Gaussian city, 8 blocks, 1080p, block-parallel)",
           "value": throughput(1, steps, ms), "unit": "frames/s", "ms_per_frame": ms / steps,
           "steps": steps, "scaling": "strong", "exchange": exchange,
           "blocks_per_rank": [len(o) for o in owned], "gaussians": args.c5_per_block * nb}
    if world == 1 and not args.no_c5_monolithic:
        # deviation of the block composite from one monolithic render of the
        # whole city (reported, not gated)
        cat = lambda f: torch.cat([getattr(models[b], f) for b in range(nb)])  # noqa: E731
        mono = GaussianModel(cat("means"), cat("quats"), cat("scales"), cat("opacity_logits"),
                             cat("sh"), 3, device=dev, validate=False)
        del models, r
        o = render(cam, mono, 16, sh_eval_degree=3)
        torch.cuda.synchronize()
        d = (out[0] - o.rgb).abs()
        res["block_vs_monolithic"] = {"max_abs": float(d.max()),
                                      "frac_px_gt_1e-3": float((d.amax(-1) > 1e-3).double()
                                                               .mean()),
                                      "mean_abs": float(d.mean())}
        del mono, o
    del hosts
    return res


def run_ours(args, rank, world, local):
    import torch

    from paper_2503_21364_b200 import scenes
    from paper_2503_21364_b200.batch import BatchRenderer
    from paper_2503_21364_b200.distributed import camera_shard

    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world == 1 and "MASTER_PORT" not in os.environ:
        # a one-rank group (c5's symmetric-memory rendezvous needs one)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]),
                              RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=dev)
    assert dist.get_world_size() == args.gpus, (dist.get_world_size(), args.gpus)
    warm = torch.ones(1, device=dev)
    dist.all_reduce(warm)  # NCCL communicator warm-up
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    model, g_host, bcast_ms = replicate_scene(rank, world, dev)
    views = args.views
    all_cams = scenes.orbit_cameras(views, W, H, seed=0)
    mine = camera_shard(views, rank, world)
    cams = [all_cams[i] for i in mine]
    renderer = BatchRenderer(model, W, H, max(len(cams), 1), tile_size=16, sh_eval_degree=3,
                             n_streams=args.streams, group=args.group, flags=args.flags)

    # warm-up (also sizes every arena)
    for _ in range(args.warmup):
        renderer.render(cams)
    torch.cuda.synchronize()

    # per-stage times of one representative step (events on the launching stream)
    stage = renderer.render(cams, stage_times=True)
    torch.cuda.synchronize()

    # the timed renderer: host-synchronised views, or capacity-bounded views
    # with no host wait (K never read back), optionally replayed as one CUDA
    # graph of the whole batch; the capacity is 1.25 x the largest K of the
    # stage pass, and an overflow after the timed region fails the run
    step = lambda: renderer.render(cams)  # noqa: E731
    timed = renderer
    if args.mode != "sync":
        cap = int(1.25 * stage["max_instances"]) + 1024
        timed = BatchRenderer(model, W, H, max(len(cams), 1), tile_size=16, sh_eval_degree=3,
                              n_streams=args.streams, group=args.group, capacity=cap,
                              flags=args.flags)
        timed.render(cams)
        torch.cuda.synchronize()
        if args.mode == "graph":
            graph = timed.capture(cams)
            step = graph.replay
        else:
            step = lambda: timed.render(cams)  # noqa: E731
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    ms_max = time_steps(step, args.steps, world, dev, barrier)
    clocks = sampler.stop()
    if args.mode != "sync" and timed.overflowed():
        raise SystemExit("bench.py: a view exceeded the instance capacity; rerun --mode sync")
    ms_per_step = ms_max / args.steps
    value = throughput(views, args.steps, ms_max)

    # weak scaling beside it: every rank renders the full 64-view batch
    weak = None
    if world > 1:
        wr = BatchRenderer(model, W, H, views, tile_size=16, sh_eval_degree=3,
                           n_streams=args.streams, group=args.group, flags=args.flags)
        wr.render(all_cams)
        torch.cuda.synchronize()
        wsteps = max(1, min(args.steps, 5))
        wms = time_steps(lambda: wr.render(all_cams), wsteps, world, dev, barrier)
        weak = {"value": throughput(views * world, wsteps, wms), "unit": UNIT,
                "views_per_gpu": views, "steps": wsteps, "ms_per_step": wms / wsteps}
        del wr

    # e2e through the public API with host buffers: per step, the cameras go
    # H2D from pinned memory and every rendered frame comes back D2H.
    e2e = renderer.bench_e2e(cams, args.e2e_steps, barrier=barrier, world=world, device=dev,
                             total_views=views)
    latency = single_view_latency(model, cams[0]) if rank == 0 else None

    c5 = None
    if not args.no_c5:
        del renderer
        torch.cuda.empty_cache()
        c5 = run_c5(args, rank, world, dev, barrier)

    line = None
    if rank == 0:
        line = make_line(args, world, views, len(cams), value, ms_per_step, stage, clocks, e2e,
                         weak, latency, c5, bcast_ms, g_host, all_cams[0], args.gpu_launches)
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return line


def make_line(args, world, views, my_views, value, ms_per_step, stage, clocks, e2e, weak,
              latency, c5, bcast_ms, g_host, cam0, launches):
    pk = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    st = stage["stage_ms"]
    nv = my_views  # stage times are summed over this rank's views
    per = stage["per_frame"]
    alg = stage["alg_bytes"]  # per view
    stage_ms = {k: v / nv for k, v in st.items()}
    hbm_stages = [k for k in alg if stage_ms.get(k, 0) > 0]
    dom = max(stage_ms, key=stage_ms.get)
    stage_gbs = {k: alg[k] / (stage_ms[k] / 1e3) / 1e9 for k in hbm_stages}
    frame_ms = ms_per_step * world / views  # device time per frame on one GPU
    frame_bytes = sum(alg.values())
    roof = {"bound": "hbm", "kernel": dom, "achieved": stage_gbs.get(dom), "peak": hbm,
            "unit": "GB/s", "frac": (stage_gbs.get(dom) or 0.0) / hbm,
            "traffic": NCU_TRAFFIC.get(dom), "traffic_source": NCU_TRAFFIC_SOURCE,
            "stage_traffic": NCU_TRAFFIC,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"
            if "hbm_gbs" in pk else "fallback 6650 GB/s (B200_PROFILING.md)",
            "stage_ms_per_frame": stage_ms, "stage_alg_bytes": alg, "stage_gbs": stage_gbs,
            "stage_frac": {k: v / hbm for k, v in stage_gbs.items()},
            "frame": {"alg_bytes": frame_bytes, "ms": frame_ms,
                      "gbs": frame_bytes / (frame_ms / 1e3) / 1e9,
                      "frac": frame_bytes / (frame_ms / 1e3) / 1e9 / hbm,
                      "note": "sum of every stage's algorithmic bytes / the measured "
                              "ms per frame (overlapped streams) / peak"}}
    if dom == "blend":
        roof["note"] = ("the dominant stage (blend) is FP32/MUFU-issue bound, not HBM "
                        "bound: its HBM fraction is informational; blend_pairs is its "
                        "roofline")
    pairs = per.get("pairs", 0)
    if pairs:
        sm_clk = (clocks.get("sm_mhz") or 1965.0) * 1e6
        pair_peak = 148 * 128 * sm_clk / 17.0
        pr = pairs / (stage_ms["blend"] / 1e3)
        roof["blend_pairs"] = {"achieved": pr, "peak": pair_peak, "unit": "pairs/s",
                               "frac": pr / pair_peak,
                               "note": "k_blend16w alone (K7b is stage touched_fix); "
                                       "FP32-pipe pair roofline: 148 SM x 128 lanes x "
                                       "f_clk / 17 instr per pair"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(g_host, cam0)
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step,
        "ms_per_frame": ms_per_step / views,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": arm_config(args, world),
        "gpu_launches": launches(stage) * args.steps,
        "e2e": e2e,
        "latency_ms_single_view": latency,
        "weak": weak,
        "c5": c5,
        "setup": {"scene_broadcast_ms": bcast_ms},
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "instances_per_frame": per.get("instances"),
    }


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--views", type=int, default=BATCH_VIEWS)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-c5-monolithic", action="store_true")
    ap.add_argument("--c5-steps", type=int, default=5)
    ap.add_argument("--c5-per-block", type=int, default=C5_PER_BLOCK)
    ap.add_argument("--streams", type=int, default=4,
                    help="contexts/streams the view batch alternates over")
    ap.add_argument("--mode", default="sync", choices=["sync", "nosync", "graph"],
                    help="sync: per-view host read of K; nosync: capacity-bounded, no host "
                         "wait; graph: the nosync batch captured once as a CUDA graph")
    ap.add_argument("--group", type=int, default=2,
                    help="views per shared K1 launch (lmgs_render_group; 1 = lmgs_render)")
    ap.add_argument("--flags", type=int, default=0,
                    help="extra LMGS_FLAG_* bits (e.g. 32: the fused tile sort, an A/B)")
    args = ap.parse_args(argv)
    # liblmgs kernels per step, as the library counts them (stage_times pass)
    args.gpu_launches = lambda stage: stage["launches"]
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if launch_check(args.gpus) == "spawn":
        sys.exit(spawn_torchrun(args.gpus, argv))
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
