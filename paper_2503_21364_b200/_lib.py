"""ctypes binding of liblmgs.so (include/lmgs.h).

The product path has no fallback: if the library is missing or fails to load,
``lib()`` raises.  Build it with ``python -m paper_2503_21364_b200.build``
(``__graft_entry__.build()`` does this).
"""

from __future__ import annotations

import ctypes
from pathlib import Path

from .errors import InvalidInputError, LmgsError, ShapeError

LIB_PATH = Path(__file__).resolve().parent / "liblmgs.so"
ABI_VERSION = 5

P = ctypes.c_void_p
D = ctypes.c_double
F = ctypes.c_float
I32 = ctypes.c_int32
I64 = ctypes.c_int64
U32 = ctypes.c_uint32

(LMGS_OK, LMGS_ERR_INVALID, LMGS_ERR_CUDA, LMGS_ERR_OOM, LMGS_ERR_UNSUPPORTED, LMGS_ERR_FORMAT,
 LMGS_ERR_IO) = range(7)
LMGS_FLAG_STAGE_TIMES = 1
LMGS_FLAG_NO_TOUCHED_FIX = 2
LMGS_FLAG_NO_HOST_SYNC = 8
LMGS_FLAG_WIDE_FIX_BAND = 16
LMGS_FLAG_FUSED_TILE_SORT = 32
LMGS_FLAG_CONCURRENT = 64
MAX_STAGES = 8

# every symbol include/lmgs.h declares
EXPORTS = ("lmgs_abi_version", "lmgs_context_create", "lmgs_context_destroy", "lmgs_last_error",
           "lmgs_render", "lmgs_render_batch", "lmgs_get_stats", "lmgs_copy_instances",
           "lmgs_project", "lmgs_composite_blocks", "lmgs_checkpoint_info_read",
           "lmgs_checkpoint_load", "lmgs_checkpoint_save", "lmgs_encode_rgb8",
           "lmgs_backward", "lmgs_mse_grad", "lmgs_render_strips", "lmgs_signal_flags",
           "lmgs_wait_flags", "lmgs_touched_fix_count", "lmgs_render_group",
           "lmgs_record_collect")
MAX_GROUP = 8  # LMGS_MAX_GROUP


class Camera(ctypes.Structure):
    _fields_ = [("r_wc", D * 9), ("t_wc", D * 3), ("center", D * 3), ("fx", D), ("fy", D),
                ("cx", D), ("cy", D), ("lim_x", D), ("lim_y", D), ("width", I32),
                ("height", I32)]


class Gaussians(ctypes.Structure):
    _fields_ = [("means", P), ("quats", P), ("scales", P), ("opacity_logits", P), ("sh", P),
                ("prim_ids", P), ("count", I64), ("sh_degree", I32), ("sh_coeffs", I32),
                ("page_mask", P), ("page_shift", I32), ("reserved", I32)]


class Settings(ctypes.Structure):
    _fields_ = [("tile_size", I32), ("sh_eval_degree", I32), ("background", D * 3),
                ("flags", U32), ("max_instances", I64)]


MAX_STRIPS = 8


class StripTargets(ctypes.Structure):
    _fields_ = [("n_strips", I32), ("strip_rows", I32), ("rgb", P * MAX_STRIPS),
                ("trans", P * MAX_STRIPS), ("depth", P * MAX_STRIPS)]


class Frame(ctypes.Structure):
    _fields_ = [("rgb", P), ("alpha", P), ("depth", P), ("transmittance", P), ("touched", P),
                ("kept", P), ("tile_ranges", P), ("n_processed", P)]


class Stats(ctypes.Structure):
    _fields_ = [("n_gaussians", I64), ("n_kept", I64), ("n_instances", I64),
                ("n_visible", I64), ("n_tiles", I32), ("tiles_x", I32), ("tiles_y", I32),
                ("n_stages", I32), ("n_launches", I32),
                ("stage_ms", F * MAX_STAGES), ("stage_names", ctypes.c_char_p * MAX_STAGES),
                ("capacity", I64), ("max_instances_seen", I64), ("overflow", I32),
                ("reserved", I32)]


class CheckpointInfo(ctypes.Structure):
    _fields_ = [("version", U32), ("sh_degree", U32), ("count", I64), ("row_floats", I32),
                ("has_grid", I32), ("data_offset", I64), ("grid_bbox", F * 6),
                ("grid_nx", U32), ("grid_ny", U32), ("grid_table_offset", I64)]


_lib = None


def lib():
    """Load liblmgs.so (raises if it is absent: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise LmgsError(f"{LIB_PATH} is missing; run `python -m paper_2503_21364_b200.build`")
    L = ctypes.CDLL(str(LIB_PATH))
    L.lmgs_abi_version.restype = ctypes.c_int
    L.lmgs_context_create.argtypes = [ctypes.c_int, ctypes.POINTER(P)]
    L.lmgs_context_destroy.argtypes = [P]
    L.lmgs_context_destroy.restype = None
    L.lmgs_last_error.argtypes = [P]
    L.lmgs_last_error.restype = ctypes.c_char_p
    L.lmgs_render.argtypes = [P, ctypes.POINTER(Gaussians), ctypes.POINTER(Camera),
                              ctypes.POINTER(Settings), ctypes.POINTER(Frame), P]
    L.lmgs_render_batch.argtypes = [P, ctypes.POINTER(Gaussians), ctypes.POINTER(Camera), I32,
                                    ctypes.POINTER(Settings), ctypes.POINTER(Frame), P]
    L.lmgs_render_group.argtypes = [ctypes.POINTER(P), I32, ctypes.POINTER(Gaussians),
                                    ctypes.POINTER(Camera), ctypes.POINTER(Settings),
                                    ctypes.POINTER(Frame), ctypes.POINTER(P)]
    L.lmgs_get_stats.argtypes = [P, ctypes.POINTER(Stats)]
    L.lmgs_copy_instances.argtypes = [P, P, P, P]
    L.lmgs_project.argtypes = [P, ctypes.POINTER(Gaussians), ctypes.POINTER(Camera),
                               ctypes.POINTER(Settings), P, P, P, P, P, P, P, P]
    L.lmgs_composite_blocks.argtypes = [P, P, P, I32, P, I64, P, P, P, P, P]
    L.lmgs_checkpoint_info_read.argtypes = [ctypes.c_char_p, ctypes.POINTER(CheckpointInfo), P,
                                            ctypes.c_int]
    L.lmgs_checkpoint_load.argtypes = [ctypes.c_char_p, P, P, P, P, P, P, P, P, ctypes.c_int]
    L.lmgs_checkpoint_save.argtypes = [ctypes.c_char_p, ctypes.POINTER(Gaussians),
                                       ctypes.POINTER(CheckpointInfo), P, P, P, ctypes.c_int]
    L.lmgs_encode_rgb8.argtypes = [P, I64, P, P]
    L.lmgs_record_collect.argtypes = [P, ctypes.POINTER(Gaussians), ctypes.POINTER(Camera),
                                      ctypes.POINTER(Settings), P, P, P, P, P, P, P]
    L.lmgs_backward.argtypes = [P, ctypes.POINTER(Gaussians), ctypes.POINTER(Camera),
                                ctypes.POINTER(Settings), P, P, P, P, P, P, P, P, P, P]
    L.lmgs_mse_grad.argtypes = [P, P, ctypes.c_int, I64, P, P, P]
    L.lmgs_render_strips.argtypes = [P, ctypes.POINTER(Gaussians), ctypes.POINTER(Camera),
                                     ctypes.POINTER(Settings), ctypes.POINTER(StripTargets), P, P]
    L.lmgs_signal_flags.argtypes = [ctypes.POINTER(P), I32, U32, P]
    L.lmgs_wait_flags.argtypes = [P, I32, U32, P]
    L.lmgs_touched_fix_count.argtypes = [P, ctypes.POINTER(U32)]
    got = L.lmgs_abi_version()
    if got != ABI_VERSION:
        raise LmgsError(f"liblmgs ABI {got} != expected {ABI_VERSION}")
    _lib = L
    return L


def check(ctx, status: int, what: str) -> None:
    if status == LMGS_OK:
        return
    msg = lib().lmgs_last_error(ctx) if ctx else b""
    msg = msg.decode() if msg else ""
    text = f"{what}: {msg or 'status ' + str(status)}"
    if status == LMGS_ERR_INVALID:
        if "coefficient count" in msg:
            raise ShapeError(msg)
        raise InvalidInputError(text)
    raise LmgsError(text)


class Context:
    """Owns one lmgs_context (device arena); one per concurrently-used stream."""

    def __init__(self, device: int = 0):
        self.device = int(device)
        h = P()
        st = lib().lmgs_context_create(self.device, ctypes.byref(h))
        if st != LMGS_OK:
            raise LmgsError(f"lmgs_context_create failed with status {st}")
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            lib().lmgs_context_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    def touched_fix_count(self) -> int:
        """Pixels the last render replayed for exact touched counts (syncs)."""
        v = ctypes.c_uint32()
        check(self.handle, lib().lmgs_touched_fix_count(self.handle, ctypes.byref(v)),
              "lmgs_touched_fix_count")
        return int(v.value)

    def stats(self) -> dict:
        s = Stats()
        check(self.handle, lib().lmgs_get_stats(self.handle, ctypes.byref(s)), "lmgs_get_stats")
        names = [s.stage_names[i].decode() if s.stage_names[i] else "" for i in range(s.n_stages)]
        return dict(n_gaussians=s.n_gaussians, n_kept=s.n_kept, n_instances=s.n_instances,
                    n_visible=s.n_visible, n_launches=s.n_launches, n_tiles=s.n_tiles,
                    tiles_x=s.tiles_x, tiles_y=s.tiles_y,
                    stage_ms={names[i]: float(s.stage_ms[i]) for i in range(s.n_stages)},
                    capacity=s.capacity, max_instances_seen=s.max_instances_seen,
                    overflow=bool(s.overflow))
