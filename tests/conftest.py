"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu`` and skipped
when no CUDA device is present; everything else runs on the CPU here."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


GOLDEN_CASES = sorted(p.stem for p in GOLDEN.glob("*.npz"))


class Case:
    """One golden fixture: inputs (or their regenerated arrays) + reference outputs."""

    def __init__(self, name: str):
        from paper_2503_21364_b200 import scenes
        from paper_2503_21364_b200.camera import Camera

        z = np.load(GOLDEN / f"{name}.npz")
        self.name = name
        self.z = z
        self.tile_size = int(z["tile_size"])
        self.background = tuple(float(v) for v in z["background"])
        self.sh_degree = int(z["sh_degree"])
        self.camera = Camera(float(z["cam_fx"]), float(z["cam_fy"]), float(z["cam_cx"]),
                             float(z["cam_cy"]), int(z["cam_w"]), int(z["cam_h"]),
                             z["cam_r"], z["cam_t"])
        self.subset = z["subset"] if "subset" in z else None
        if "means" in z:
            self.gaussians = scenes.HostGaussians(z["means"], z["quats"], z["scales"],
                                                  z["opacity_logits"], z["sh"], self.sh_degree)
        else:  # c1: regenerate from seed and check the digest
            import hashlib

            g = scenes.synthetic_gaussians(10_000, seed=0)
            h = hashlib.sha256()
            for a in (g.means, g.quats, g.scales, g.opacity_logits, g.sh):
                h.update(np.ascontiguousarray(a).tobytes())
            assert h.hexdigest() == str(z["digest"]), "synthetic generator drifted"
            self.gaussians = g
        self.image = z["image"]
        self.touched = z["touched"].astype(np.int64)
        self.lists = z["lists"].astype(np.int64)
        self.offsets = z["offsets"].astype(np.int64)
        self.t_final = z["t_final"]
        self.splat_prim_id = z["splat_prim_id"].astype(np.int64)


@pytest.fixture(scope="session")
def golden_case():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = Case(name)
        return cache[name]

    return get
