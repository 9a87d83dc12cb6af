"""Randomised parity stress (not part of the default suite): many random
scenes x image sizes x tile sizes x backgrounds x SH degrees against the
oracle; tile lists and touched bit-exact, image within 1e-4."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2503_21364_b200 import GaussianModel, render, render_image, scenes  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
n_cases = int(sys.argv[2]) if len(sys.argv) > 2 else 200
bad = 0
for case in range(n_cases):
    n = int(rng.integers(0, 20000)) if case % 4 else int(rng.integers(0, 300000))
    w, h = int(rng.integers(8, 900)), int(rng.integers(8, 600))
    ts = int(rng.choice([1, 2, 4, 7, 8, 12, 16, 20, 32, 48, 64]))
    deg = int(rng.integers(0, 4))
    bg = tuple(float(v) for v in rng.uniform(0, 1, 3))
    seed = int(rng.integers(0, 1 << 30))
    if ts < 4 and w * h > 40000:
        ts = 8
    g = scenes.synthetic_gaussians(n, seed=seed, sh_degree=3)
    cam = scenes.orbit_cameras(1, w, h, seed=seed)[0]
    if case % 5 == 4 and n > 0:  # render_image with a shuffled subset (prim-id remap)
        sub = rng.permutation(n)[: int(rng.integers(1, n + 1))]
        img, touched = render_image(GaussianModel.from_host(g, validate=False), cam, ts, bg,
                                    subset=sub, sh_eval_degree=deg)
        o = oracle.render(g, cam, ts, bg, sh_eval_degree=deg, subset=sub)
        ok = (np.array_equal(touched.cpu().numpy(), o["touched"])
              and float(np.abs(img.cpu().double().numpy() - o["image"]).max()) <= 1e-4)
    else:
        out = render(cam, GaussianModel.from_host(g, validate=False), ts, bg, deg,
                     with_instances=True)
        o = oracle.render(g, cam, ts, bg, sh_eval_degree=deg)
        kept = out.kept.cpu().numpy().astype(bool)
        ok = (out.n_instances == o["K"]
              and np.array_equal(out.inst_prim_ids.cpu().numpy(), o["inst_prim"])
              and np.array_equal(out.touched.cpu().numpy()[kept], o["touched"])
              and float(np.abs(out.rgb.cpu().double().numpy() - o["image"]).max()) <= 1e-4)
    if not ok:
        bad += 1
        print("MISMATCH", dict(n=n, w=w, h=h, ts=ts, deg=deg, seed=seed), flush=True)
print(f"{n_cases} cases, {bad} mismatches")
