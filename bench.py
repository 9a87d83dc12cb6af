"""Benchmark: 1080p frames/s at 6M Gaussians (BASELINE.json metric, config c3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--views V] [--impl reference]

One step = one batch of V (default 64) camera views of the 6M-Gaussian
synthetic scene rendered at 1920x1080 on each rank (camera-batch data
parallelism, no data-path collective; "scaling": "weak").  The scene (1.42 GB)
and every per-view working set exceed the 126 MB L2, so no explicit L2 flush
is needed between timed iterations.

Timed region: W untimed warm-up steps, then exactly K steps bracketed by a
barrier + cuda.synchronize on both sides, timed with CUDA events on the
launching stream; the max over ranks is reported.  Rank 0 prints one JSON line.

``--impl reference`` times the reference algorithm's CPU implementation (the
fp64 C restatement in oracle/, "port": the reference is pure Python and does
not travel to the GPU box) on the host cores over a bounded sample (one full
1080p view of the same scene per step).
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


# dram__bytes_read.sum + dram__bytes_write.sum per launch of each stage's kernels
# on a c3 view, from the committed full ncu captures (profiles/r02/*_summary.txt;
# stage = sum of its kernels).  Reported as `traffic` beside the algorithmic bytes.
NCU_TRAFFIC = {  # profiles/r05/ncu_launch_table.txt: DRAM bytes per c3 view
    "preprocess": 2736.1e6 / 2,  # one k_preprocess_tma<2> launch serves two views
    "depth_sort": 48.1e6 + 3 * 43.1e6 + 106.7e6,
    "emit": 260.3e6,
    "tile_sort": 2 * 294.8e6,
    "blend": 171.8e6 + 114.0e6,  # k_blend16w + k_touched_fix (K7b)
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


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# reference arm: the CPU implementation of the path (oracle port), host cores


def run_reference(args, rank, world):
    if rank != 0:
        return
    import numpy as np

    import oracle
    from paper_2503_21364_b200 import scenes

    threads = os.cpu_count() or 1
    oracle.set_threads(threads)
    g = scenes.synthetic_gaussians(N_GAUSS, seed=0)
    cams = scenes.orbit_cameras(64, W, H, seed=0)
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
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": "c3: 6M Gaussians, 1920x1080, SH3, "
                                                    "one full view per step (bounded sample)"},
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


def run_ours(args, rank, world, local):
    import numpy as np
    import torch

    from paper_2503_21364_b200 import GaussianModel, scenes
    from paper_2503_21364_b200.batch import BatchRenderer

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    g_host = scenes.synthetic_gaussians(N_GAUSS, seed=0)
    model = GaussianModel.from_host(g_host, device=dev, validate=False)
    views = args.views
    all_cams = scenes.orbit_cameras(views * world, W, H, seed=0)
    cams = all_cams[rank * views:(rank + 1) * views]
    renderer = BatchRenderer(model, W, H, views, tile_size=16, sh_eval_degree=3,
                             n_streams=args.streams, group=args.group)

    # warm-up (also sizes every arena)
    for _ in range(args.warmup):
        renderer.render(cams)
    torch.cuda.synchronize()

    # per-stage times of one representative step (events on the launching stream)
    stage = renderer.render(cams, stage_times=True)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(args.steps):
        renderer.render(cams)
    end.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    ms = start.elapsed_time(end)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / args.steps
    value = views * world * args.steps / (ms_max / 1e3)

    # e2e through the public API with host buffers: per step, the cameras go
    # H2D from pinned memory and every rendered frame comes back D2H.
    e2e = renderer.bench_e2e(cams, args.e2e_steps, barrier=barrier, world=world, device=dev)

    line = None
    if rank == 0:
        pk = peaks()
        hbm = float(pk.get("hbm_gbs", 6650.0))
        st = stage["stage_ms"]
        frames = views
        dom = max(st, key=st.get)
        per = stage["per_frame"]
        # algorithmic bytes of each stage per frame
        alg = stage["alg_bytes"]
        dom_ms = st[dom] / frames
        achieved = alg[dom] / (dom_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
                "unit": "GB/s", "frac": achieved / hbm,
                "traffic": NCU_TRAFFIC.get(dom),
                "traffic_source": "profiles/r05 ncu launch list (dram bytes per c3 view)",
                "stage_traffic": NCU_TRAFFIC,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"
                if "hbm_gbs" in pk else "fallback 6650 GB/s (B200_PROFILING.md)",
                "stage_ms_per_frame": {k: v / frames for k, v in st.items()},
                "stage_gbs": {k: alg[k] / (st[k] / frames / 1e3) / 1e9 for k in st if st[k] > 0},
                "stage_alg_bytes": alg}
        roof["stage_frac"] = {k: v / hbm for k, v in roof["stage_gbs"].items()}
        if dom == "blend":
            roof["note"] = ("the dominant stage (blend) is FP32/MUFU-issue bound, not HBM "
                            "bound: its HBM fraction is informational; blend_pairs is its "
                            "roofline")
        blend_pairs = per.get("pairs", 0)
        if blend_pairs:
            sm_clk = (clocks.get("sm_mhz") or 1965.0) * 1e6
            pair_peak = 148 * 128 * sm_clk / 17.0
            pr = blend_pairs / (st["blend"] / frames / 1e3)
            roof["blend_pairs"] = {"achieved": pr, "peak": pair_peak, "unit": "pairs/s",
                                   "frac": pr / pair_peak,
                                   "note": "FP32-pipe pair roofline: 148 SM x 128 lanes x "
                                           "f_clk / 17 instr per pair"}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline_sample(g_host, cams[0])
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "ms_per_frame": ms_per_step / views,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "c3: 6M Gaussians (SH3), 1920x1080, batch of "
                                   f"{views} orbit views per GPU, tile 16",
                       "gaussians": N_GAUSS, "views_per_gpu": views, "width": W, "height": H,
                       "parallelism": f"camera-batch dp{world}",
                       "views_per_k1_launch": args.group,
                       "l2": "no flush: scene 1.42 GB and per-view buffers > 126 MB L2",
                       "geometry": "fp64 (bit-exact tile lists)", "blend": "fp32"},
            "gpu_launches": renderer.launches_per_step * args.steps,
            "e2e": e2e,
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "instances_per_frame": per.get("instances"),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--views", type=int, default=64)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=3,
                    help="contexts/streams the view batch alternates over")
    ap.add_argument("--group", type=int, default=2,
                    help="views per shared K1 launch (lmgs_render_group; 1 = lmgs_render)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
