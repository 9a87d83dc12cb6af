"""LMGS checkpoints and wire frames, the formats either side of the rasterizer.

* ``load_gaussian_checkpoint(path)`` / ``save_gaussian_checkpoint(model, path,
  grid)`` — data_io.py:256-316 (same file format, same FormatError on a bad
  magic / version / truncation), but the rows stream straight into device
  SoA arrays through liblmgs (``lmgs_checkpoint_load``: pinned double-buffered
  chunks, async H2D, de-interleave kernel) instead of a float64 host model.
* ``encode_frame(image, header)`` — render_runtime.py:397-401: the pixel bytes
  are produced on the GPU (``lmgs_encode_rgb8``, round-half-even of
  clip(rgb, 0, 1) * 255 in fp64, exactly numpy's) and only the uint8 frame
  crosses PCIe.  ``decode_frame`` is the host-side inverse (401-406).
"""

from __future__ import annotations

import ctypes
import json
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .errors import FormatError, InvalidInputError, LmgsError
from .raster import GaussianModel, _ptr


@dataclass
class CheckpointGrid:
    """The optional scene grid block (scene_manager.SceneGrid + block table)."""

    bbox: np.ndarray            # (2, 3) float32 values
    nx: int
    ny: int
    block_to_submodel: dict     # {(ix, iy): submodel id}


def _raise(status: int, err: ctypes.Array, what: str):
    msg = err.value.decode(errors="replace")
    if status == _lib.LMGS_ERR_FORMAT:
        raise FormatError(msg)
    if status in (_lib.LMGS_ERR_INVALID, _lib.LMGS_ERR_UNSUPPORTED):
        raise InvalidInputError(f"{what}: {msg}")
    if status == _lib.LMGS_ERR_IO:
        raise OSError(msg)
    raise LmgsError(f"{what}: {msg or 'status ' + str(status)}")


def checkpoint_info(path) -> _lib.CheckpointInfo:
    info = _lib.CheckpointInfo()
    err = ctypes.create_string_buffer(512)
    st = _lib.lib().lmgs_checkpoint_info_read(str(path).encode(), ctypes.byref(info), err, 512)
    if st != _lib.LMGS_OK:
        _raise(st, err, "checkpoint_info")
    return info


def load_gaussian_checkpoint(path, device=None, stream=None):
    """(GaussianModel on the device, CheckpointGrid or None) — data_io.py:285-316."""
    info = checkpoint_info(path)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
        else torch.device(device)
    n, d = int(info.count), int(info.sh_degree)
    nc = (d + 1) ** 2
    means = torch.empty((n, 3), dtype=torch.float32, device=dev)
    quats = torch.empty((n, 4), dtype=torch.float32, device=dev)
    scales = torch.empty((n, 3), dtype=torch.float32, device=dev)
    logits = torch.empty((n,), dtype=torch.float32, device=dev)
    sh = torch.empty((n, nc, 3), dtype=torch.float32, device=dev)
    table = np.zeros(max(int(info.grid_nx) * int(info.grid_ny), 1), dtype=np.uint32) \
        if info.has_grid else None
    err = ctypes.create_string_buffer(512)
    s = torch.cuda.current_stream(dev) if stream is None else stream
    with torch.cuda.device(dev):
        st = _lib.lib().lmgs_checkpoint_load(
            str(path).encode(), _ptr(means), _ptr(quats), _ptr(scales), _ptr(logits), _ptr(sh),
            table.ctypes.data if table is not None else None, s.cuda_stream, err, 512)
    if st != _lib.LMGS_OK:
        _raise(st, err, "load_gaussian_checkpoint")
    model = GaussianModel(means, quats, scales, logits, sh, d, validate=True)
    grid = None
    if info.has_grid:
        nx, ny = int(info.grid_nx), int(info.grid_ny)
        grid = CheckpointGrid(np.asarray(info.grid_bbox, dtype=np.float32).reshape(2, 3), nx, ny,
                              {(ix, iy): int(table[iy * nx + ix])
                               for iy in range(ny) for ix in range(nx)})
    return model, grid


def save_gaussian_checkpoint(model: GaussianModel, path, grid: CheckpointGrid | None = None,
                             stream=None) -> None:
    """data_io.py:256-282 from device arrays (atomic temp-then-rename)."""
    g = model._abi()
    info = None
    table = None
    if grid is not None:
        info = _lib.CheckpointInfo()
        info.has_grid = 1
        info.grid_bbox[:] = [float(v) for v in np.asarray(grid.bbox, dtype=np.float32).reshape(6)]
        info.grid_nx, info.grid_ny = int(grid.nx), int(grid.ny)
        table = np.asarray([grid.block_to_submodel[(ix, iy)] for iy in range(grid.ny)
                            for ix in range(grid.nx)], dtype=np.uint32)
    err = ctypes.create_string_buffer(512)
    s = torch.cuda.current_stream(model.device) if stream is None else stream
    with torch.cuda.device(model.device):
        st = _lib.lib().lmgs_checkpoint_save(str(path).encode(), ctypes.byref(g),
                                             ctypes.byref(info) if info is not None else None,
                                             table.ctypes.data if table is not None else None,
                                             s.cuda_stream, err, 512)
    if st != _lib.LMGS_OK:
        _raise(st, err, "save_gaussian_checkpoint")


def encode_rgb8(image: torch.Tensor, stream=None) -> torch.Tensor:
    """(H, W, 3) fp32 CUDA image -> (H, W, 3) uint8 CUDA tensor (encode_frame's pixels)."""
    if not image.is_cuda or image.dtype != torch.float32:
        raise InvalidInputError("encode_rgb8 needs a float32 CUDA image")
    img = image.contiguous()
    out = torch.empty(img.shape, dtype=torch.uint8, device=img.device)
    s = torch.cuda.current_stream(img.device) if stream is None else stream
    st = _lib.lib().lmgs_encode_rgb8(_ptr(img), img.numel(), _ptr(out), s.cuda_stream)
    _lib.check(None, st, "lmgs_encode_rgb8")
    return out


def encode_frame(image: torch.Tensor, header: dict) -> bytes:
    """render_runtime.py:397-401 with the pixels quantised on the GPU."""
    pixels = encode_rgb8(image).cpu().numpy().tobytes()
    hdr = json.dumps(header, sort_keys=True).encode()
    return struct.pack("<I", len(hdr)) + hdr + pixels


def decode_frame(payload: bytes):
    """render_runtime.py:401-406."""
    (hlen,) = struct.unpack_from("<I", payload)
    header = json.loads(payload[4:4 + hlen].decode())
    pixels = np.frombuffer(payload[4 + hlen:], dtype=np.uint8)
    return header, pixels.reshape(header["height"], header["width"], 3)


__all__ = ["CheckpointGrid", "checkpoint_info", "load_gaussian_checkpoint",
           "save_gaussian_checkpoint", "encode_rgb8", "encode_frame", "decode_frame", "Path"]
