"""LMGS checkpoints (data_io.py:256-316) and RGB8 wire frames (render_runtime.py:
397-406) against files written by the unmodified reference
(tests/golden/formats/make_format_golden.py).

CPU: header parsing and the reference's FormatError cases through the C ABI
(host-only entry point), frame decoding.  GPU: rows loaded into device SoA
bit-exactly, save -> byte-identical file (the reference's round-trip test,
test_acceptance.py:592-600), GPU-encoded frame bytes identical to the
reference's encode_frame.
"""

import json
import shutil
import struct

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2503_21364_b200.checkpoint import checkpoint_info, decode_frame
from paper_2503_21364_b200.errors import FormatError

FMT = GOLDEN / "formats"
CKPT3 = FMT / "ckpt_sh3_grid.lmgs"
CKPT1 = FMT / "ckpt_sh1.lmgs"


def parse_lmgs(path):
    """Independent numpy restatement of the LMGS layout (data_io.py:3-9)."""
    data = path.read_bytes()
    magic, version, deg, n = struct.unpack_from("<4sIIQ", data, 0)
    stride = 11 + 3 * (deg + 1) ** 2
    rows = np.frombuffer(data, dtype="<f4", count=n * stride, offset=20).reshape(n, stride)
    off = 20 + 4 * n * stride
    flag = data[off]
    grid = None
    if flag:
        bbox = np.frombuffer(data, dtype="<f4", count=6, offset=off + 1).reshape(2, 3)
        nx, ny = struct.unpack_from("<II", data, off + 25)
        table = np.frombuffer(data, dtype="<u4", count=nx * ny, offset=off + 33)
        grid = (bbox, nx, ny, table)
    return dict(magic=magic, version=version, deg=deg, n=n, means=rows[:, 0:3],
                quats=rows[:, 3:7], scales=rows[:, 7:10], logits=rows[:, 10],
                sh=rows[:, 11:].reshape(n, (deg + 1) ** 2, 3), grid=grid)


def test_header_matches_reference_file():
    ref = parse_lmgs(CKPT3)
    info = checkpoint_info(CKPT3)
    assert (info.version, info.sh_degree, info.count) == (1, 3, 300)
    assert info.row_floats == 11 + 48 and info.has_grid == 1
    bbox, nx, ny, _ = ref["grid"]
    assert (info.grid_nx, info.grid_ny) == (nx, ny) == (3, 2)
    np.testing.assert_array_equal(np.asarray(info.grid_bbox, np.float32), bbox.reshape(6))
    info1 = checkpoint_info(CKPT1)
    assert (info1.sh_degree, info1.count, info1.has_grid) == (1, 50, 0)


@pytest.mark.parametrize("corrupt", ["magic", "version", "truncated_rows", "truncated_grid",
                                     "empty"])
def test_malformed_files_raise_format_error(tmp_path, corrupt):
    """data_io.py:290-294 and _Reader.take (truncation) raise FormatError."""
    data = bytearray(CKPT3.read_bytes())
    if corrupt == "magic":
        data[0:4] = b"LMGX"
    elif corrupt == "version":
        data[4:8] = struct.pack("<I", 2)
    elif corrupt == "truncated_rows":
        data = data[:20 + 4 * 59 * 100]
    elif corrupt == "truncated_grid":
        data = data[:-5]
    else:
        data = data[:3]
    p = tmp_path / "bad.lmgs"
    p.write_bytes(bytes(data))
    with pytest.raises(FormatError):
        checkpoint_info(p)


def test_missing_file_is_oserror(tmp_path):
    with pytest.raises(OSError):
        checkpoint_info(tmp_path / "nope.lmgs")


def test_decode_reference_frame():
    z = np.load(FMT / "frame_rgb8.npz")
    header, pixels = decode_frame(z["payload"].tobytes())
    assert header == json.loads(str(z["header"]))
    ref = np.round(np.clip(z["image"].astype(np.float64), 0, 1) * 255).astype(np.uint8)
    np.testing.assert_array_equal(pixels, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("path", [CKPT3, CKPT1])
def test_load_rows_bit_exact(path):
    from paper_2503_21364_b200.checkpoint import load_gaussian_checkpoint

    ref = parse_lmgs(path)
    model, grid = load_gaussian_checkpoint(path)
    for name, t in (("means", model.means), ("quats", model.quats), ("scales", model.scales),
                    ("logits", model.opacity_logits), ("sh", model.sh)):
        np.testing.assert_array_equal(t.cpu().numpy(), ref[name], err_msg=name)
    assert model.sh_degree == ref["deg"]
    if ref["grid"] is None:
        assert grid is None
    else:
        bbox, nx, ny, table = ref["grid"]
        assert (grid.nx, grid.ny) == (nx, ny)
        assert [grid.block_to_submodel[(ix, iy)] for iy in range(ny) for ix in range(nx)] == \
            table.tolist()


@pytest.mark.gpu
@pytest.mark.parametrize("path", [CKPT3, CKPT1])
def test_save_round_trip_byte_identical(tmp_path, path):
    from paper_2503_21364_b200.checkpoint import (load_gaussian_checkpoint,
                                                  save_gaussian_checkpoint)

    model, grid = load_gaussian_checkpoint(path)
    out = tmp_path / "rt.lmgs"
    save_gaussian_checkpoint(model, out, grid)
    assert out.read_bytes() == path.read_bytes()


@pytest.mark.gpu
def test_render_from_checkpoint_equals_host_upload():
    from paper_2503_21364_b200 import GaussianModel, render, scenes
    from paper_2503_21364_b200.checkpoint import load_gaussian_checkpoint

    ref = parse_lmgs(CKPT3)
    model, _ = load_gaussian_checkpoint(CKPT3)
    host = scenes.HostGaussians(ref["means"].copy(), ref["quats"].copy(), ref["scales"].copy(),
                                ref["logits"].copy(), ref["sh"].copy(), 3)
    cam = scenes.orbit_cameras(1, 96, 64, seed=1)[0]
    a = render(cam, model).rgb
    b = render(cam, GaussianModel.from_host(host)).rgb
    assert bool((a == b).all())


@pytest.mark.gpu
def test_gpu_encode_frame_matches_reference_bytes():
    import torch

    from paper_2503_21364_b200.checkpoint import encode_frame

    z = np.load(FMT / "frame_rgb8.npz")
    img = torch.as_tensor(z["image"]).cuda()
    payload = encode_frame(img, json.loads(str(z["header"])))
    assert payload == z["payload"].tobytes()


@pytest.mark.gpu
def test_large_checkpoint_streams_in_chunks(tmp_path):
    """More rows than one pinned chunk (2^17): the double-buffered path."""
    from paper_2503_21364_b200 import GaussianModel, scenes
    from paper_2503_21364_b200.checkpoint import (load_gaussian_checkpoint,
                                                  save_gaussian_checkpoint)

    g = scenes.synthetic_gaussians(300_001, seed=3)
    out = tmp_path / "big.lmgs"
    save_gaussian_checkpoint(GaussianModel.from_host(g, validate=False), out)
    ref = parse_lmgs(out)
    np.testing.assert_array_equal(ref["means"], g.means)
    np.testing.assert_array_equal(ref["sh"], g.sh)
    model, grid = load_gaussian_checkpoint(out)
    assert grid is None
    np.testing.assert_array_equal(model.sh.cpu().numpy(), g.sh)
    np.testing.assert_array_equal(model.quats.cpu().numpy(), g.quats)
    shutil.rmtree(tmp_path, ignore_errors=True)
