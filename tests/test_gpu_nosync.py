"""Capacity-bounded rendering with no host wait (LMGS_FLAG_NO_HOST_SYNC) and
CUDA-graph capture of a whole view batch (SURVEY §7 hard part 8)."""

import pytest
import torch

from paper_2503_21364_b200 import GaussianModel, scenes
from paper_2503_21364_b200.batch import BatchRenderer

pytestmark = pytest.mark.gpu

W, H, NV = 800, 600, 6


@pytest.fixture(scope="module")
def scene():
    g = scenes.synthetic_gaussians(300_000, seed=31)
    return GaussianModel.from_host(g, validate=False), scenes.orbit_cameras(NV, W, H, seed=31)


def _batch(model, **kw):
    return BatchRenderer(model, W, H, NV, tile_size=16, sh_eval_degree=3, n_streams=2,
                         group=2, **kw)


def _same(a, b):
    torch.cuda.synchronize()
    assert torch.equal(a.rgb, b.rgb) and torch.equal(a.alpha, b.alpha)
    assert torch.equal(a.depth, b.depth) and torch.equal(a.ranges, b.ranges)
    assert torch.equal(a.touched, b.touched) and torch.equal(a.nproc, b.nproc)


def test_nosync_equals_host_synchronised(scene):
    model, cams = scene
    ref = _batch(model)
    ref.render(cams)
    cap = 3 * 10**6
    ns = _batch(model, capacity=cap)
    ns.render(cams)
    _same(ref, ns)
    assert not ns.overflowed()
    st = ns.ctxs[0].stats()
    assert st["capacity"] == cap


def test_graph_replay_equals_eager(scene):
    model, cams = scene
    ref = _batch(model)
    ref.render(cams)
    gr = _batch(model, capacity=3 * 10**6)
    graph = gr.capture(cams)
    for t in (gr.rgb, gr.touched, gr.ranges):
        t.zero_()
    graph.replay()
    _same(ref, gr)
    graph.replay()  # replays are repeatable
    _same(ref, gr)
    assert not gr.overflowed()


def test_overflow_is_reported_not_fatal(scene):
    model, cams = scene
    small = _batch(model, capacity=10_000)
    small.render(cams)
    torch.cuda.synchronize()
    assert small.overflowed()
    assert small.ctxs[0].stats()["overflow"] is False  # reset by the previous call
