"""Offload-fed rendering: a paged device tier fed by
asynchronous host->device copies, and the reference's two streaming session
modes on top of it.

Reference: render_runtime.py (SessionConfig 81-97, BlockSession 110-193,
FrustumSession 199-243, run_session 250-308, bench 311-326), memory_tiers.py
(TierStore 74-147, BufferPair 160-177, prefetch_policy 196-247) and
scene_manager.py (SceneGrid 24-73, onload_region 92-104, reorder_voxel_grid
159-187, frustum 193-253).

B200 design (not the reference's): the reference simulates the device tier
(``TierStore.load_cells`` clones tensors and a virtual clock models the
transfer) and then renders a model re-assembled by ``torch.cat`` or a
``subset`` gather every frame.  Here

* the host tier is the whole model in **pinned** memory, regrouped once so
  every group (cell or voxel) is a contiguous row range;
* the device tier is one **paged SoA pool** (pages of 128 rows, the K1 CTA
  size) sized from the byte budget; a group load is a few contiguous
  ``cudaMemcpyAsync`` per page run on a dedicated copy stream, recorded by a
  CUDA event, and the render stream waits on that event on the device (no
  host stall);
* a frame renders **straight from the pool**: ``lmgs_render`` takes the pool
  arrays plus per-page live-row counts (rows outside them are culled in K1;
  an inactive page's block returns before its TMA loads are issued) and a
  per-row prim key, so there is no gather
  and no concatenation; the key reproduces the reference's depth-tie order
  (FrustumSession: the row of the voxel-reordered model; BlockSession: the
  position in the concatenation of the front cells, i.e. (cell order, id));
* byte accounting, eviction order, prefetch decisions and stall counts follow
  the reference exactly (its virtual clock included), so the FrameStats are
  the reference's; the copies themselves are real and overlap rendering.
"""

from __future__ import annotations

import heapq
import statistics
import time
from dataclasses import asdict, dataclass, field

import numpy as np
import torch

from .camera import Camera
from .errors import InvalidConfigError, InvalidInputError
from .raster import GaussianModel, context, render

PAGE_SHIFT = 7
PAGE_ROWS = 1 << PAGE_SHIFT
RENDER_MODES = ("static_full", "block_double_buffer", "frustum_voxel")


class BudgetExceededError(RuntimeError):
    """memory_tiers.py:18."""


class NotResidentError(KeyError):
    """memory_tiers.py:22."""


class IncompleteLoadError(RuntimeError):
    """memory_tiers.py:26."""


# ---------------------------------------------------------------------------
# clock, transfer model, stats (common.py:51-60, memory_tiers.py:43-73)


@dataclass
class VirtualClock:
    now: float = 0.0

    def advance(self, dt: float) -> None:
        if dt < 0:
            raise InvalidInputError("clock cannot go backwards")
        self.now += dt


@dataclass
class TransferConfig:
    """bandwidth None means instant transfers on the virtual clock."""

    bandwidth_bytes_per_s: float | None = None
    fixed_latency_s: float = 0.0


@dataclass
class TierStats:
    loads: int = 0
    offloads: int = 0
    bytes_in: int = 0
    bytes_out: int = 0
    stalls: int = 0
    peak_resident_bytes: int = 0

    def snapshot(self) -> dict:
        return asdict(self)


@dataclass
class LoadHandle:
    cell_ids: tuple
    ready_at: float
    nbytes: int
    event: torch.cuda.Event | None = None  # the real copies' completion

    def ready(self, clock: VirtualClock) -> bool:
        return clock.now >= self.ready_at


# ---------------------------------------------------------------------------
# scene bookkeeping (scene_manager.py)


@dataclass
class SceneGrid:
    """scene_manager.py:24-73: 2D partition of the footprint on the x-y plane."""

    bbox: np.ndarray
    nx: int
    ny: int

    def __post_init__(self):
        self.bbox = np.asarray(self.bbox, dtype=np.float64)
        if self.nx < 1 or self.ny < 1:
            raise InvalidInputError("cell counts must be >= 1")
        if not np.all(self.bbox[1] > self.bbox[0]):
            raise InvalidInputError("degenerate scene bbox")

    @property
    def cell_extent(self) -> np.ndarray:
        return (self.bbox[1, :2] - self.bbox[0, :2]) / np.array([self.nx, self.ny])

    def cell_of_point(self, xy) -> tuple[int, int]:
        xy = np.asarray(xy, dtype=np.float64)[:2]
        w, h = self.cell_extent
        ix = int(np.floor((xy[0] - self.bbox[0, 0]) / w))
        iy = int(np.floor((xy[1] - self.bbox[0, 1]) / h))
        return min(max(ix, 0), self.nx - 1), min(max(iy, 0), self.ny - 1)

    def cell_bbox(self, index) -> np.ndarray:
        ix, iy = index
        w, h = self.cell_extent
        lo = np.array([self.bbox[0, 0] + ix * w, self.bbox[0, 1] + iy * h, self.bbox[0, 2]])
        hi = np.array([self.bbox[0, 0] + (ix + 1) * w, self.bbox[0, 1] + (iy + 1) * h,
                       self.bbox[1, 2]])
        return np.stack([lo, hi])

    def cells(self):
        return [(ix, iy) for iy in range(self.ny) for ix in range(self.nx)]


def partition_scene(bbox, nx: int, ny: int) -> SceneGrid:
    return SceneGrid(np.asarray(bbox, dtype=np.float64), nx, ny)


def onload_region(grid: SceneGrid, core, ring: int = 1) -> set:
    """scene_manager.py:92-104: cells within Chebyshev distance ``ring``."""
    cx, cy = core
    if not (0 <= cx < grid.nx and 0 <= cy < grid.ny):
        raise InvalidInputError(f"core cell {core} outside grid")
    if ring < 0:
        raise InvalidInputError("ring must be >= 0")
    return {(ix, iy) for ix in range(max(0, cx - ring), min(grid.nx, cx + ring + 1))
            for iy in range(max(0, cy - ring), min(grid.ny, cy + ring + 1))}


def cell_rows(means: np.ndarray, grid: SceneGrid) -> dict:
    """engine_api.py:182-207 (gaussian_cell_groups): ascending ids per cell."""
    m = np.asarray(means, dtype=np.float64)
    w, h = grid.cell_extent
    ix = np.clip(np.floor((m[:, 0] - grid.bbox[0, 0]) / w).astype(int), 0, grid.nx - 1)
    iy = np.clip(np.floor((m[:, 1] - grid.bbox[0, 1]) / h).astype(int), 0, grid.ny - 1)
    lin = iy * grid.nx + ix
    order = np.argsort(lin, kind="stable")
    bounds = np.searchsorted(lin[order], np.arange(grid.nx * grid.ny + 1))
    return {(cx, cy): order[bounds[cy * grid.nx + cx]:bounds[cy * grid.nx + cx + 1]]
            for (cx, cy) in grid.cells()}


@dataclass
class VoxelIndex:
    """scene_manager.py:129-156."""

    voxel_size: float
    origin: np.ndarray
    voxel_keys: np.ndarray
    ranges: np.ndarray
    permutation: np.ndarray
    voxel_max_scale: np.ndarray

    @property
    def n_voxels(self) -> int:
        return len(self.voxel_keys)

    def voxel_bbox(self, v: int, margin: float = 0.0) -> np.ndarray:
        lo = self.origin + self.voxel_keys[v] * self.voxel_size - margin
        hi = self.origin + (self.voxel_keys[v] + 1) * self.voxel_size + margin
        return np.stack([lo, hi])


def reorder_voxel_grid(means: np.ndarray, scales: np.ndarray, voxel_size: float) -> VoxelIndex:
    """scene_manager.py:159-187 on host arrays (f32 values, fp64 arithmetic)."""
    if voxel_size <= 0:
        raise InvalidInputError("voxel_size must be positive")
    m = np.asarray(means, dtype=np.float64)
    origin = np.floor(m.min(axis=0) / voxel_size) * voxel_size
    keys = np.floor((m - origin) / voxel_size).astype(np.int64)
    perm = np.lexsort((np.arange(len(m)), keys[:, 2], keys[:, 1], keys[:, 0]))
    sk = keys[perm]
    bnd = np.nonzero(np.any(np.diff(sk, axis=0) != 0, axis=1))[0] + 1
    starts = np.concatenate([[0], bnd]).astype(np.int64)
    ends = np.concatenate([bnd, [len(m)]]).astype(np.int64)
    max_scale = np.asarray(scales, dtype=np.float64).max(axis=-1)[perm]
    vox_scale = np.maximum.reduceat(max_scale, starts) if len(m) else np.zeros(0)
    return VoxelIndex(float(voxel_size), origin, sk[starts], np.stack([starts, ends], axis=1),
                      perm, vox_scale)


def frustum_planes(camera) -> np.ndarray:
    """scene_manager.py:193-220, same operations."""
    r, c = camera.r_wc, camera.center
    fwd = r[2]
    planes = [np.concatenate([fwd, [-(fwd @ c) - camera.near]]),
              np.concatenate([-fwd, [(fwd @ c) + camera.far]])]
    dirs = []
    for u, v in ((0.0, 0.0), (camera.width, 0.0), (camera.width, camera.height),
                 (0.0, camera.height)):
        d_cam = np.array([(u - camera.cx) / camera.fx, (v - camera.cy) / camera.fy, 1.0])
        dirs.append(r.T @ d_cam)
    for i in range(4):
        n = np.cross(dirs[i], dirs[(i + 1) % 4])
        n /= np.linalg.norm(n)
        if n @ fwd < 0:
            n = -n
        planes.append(np.concatenate([n, [-(n @ c)]]))
    return np.stack(planes)


def frustum_visible_voxels(index: VoxelIndex, camera, margin_sigma: float = 3.0) -> list[int]:
    """scene_manager.py:233-246, vectorised over voxels: a voxel is out only if
    all 8 corners of its inflated box are outside one plane."""
    if index.n_voxels == 0:
        return []
    planes = frustum_planes(camera)
    margin = margin_sigma * index.voxel_max_scale + 0.05 * index.voxel_size
    lo = index.origin + index.voxel_keys * index.voxel_size - margin[:, None]
    hi = index.origin + (index.voxel_keys + 1) * index.voxel_size + margin[:, None]
    bb = np.stack([lo, hi], axis=1)  # (V, 2, 3)
    corners = np.stack([np.stack([bb[:, i, 0], bb[:, j, 1], bb[:, k, 2]], axis=-1)
                        for i in (0, 1) for j in (0, 1) for k in (0, 1)], axis=1)  # (V, 8, 3)
    out = np.zeros(index.n_voxels, dtype=bool)
    for p in planes:
        val = corners[..., 0] * p[0] + corners[..., 1] * p[1] + corners[..., 2] * p[2] + p[3]
        out |= np.all(val < 0, axis=1)
    return np.nonzero(~out)[0].tolist()


# ---------------------------------------------------------------------------
# host tier and paged device tier


def row_bytes(sh_coeffs: int) -> int:
    """Device bytes of one Gaussian's parameters here (f32 SoA)."""
    return 4 * (3 + 4 + 3 + 1 + 3 * sh_coeffs)


def ref_row_bytes(sh_coeffs: int) -> int:
    """Bytes the reference accounts per Gaussian in a ParamGroup: its fp64
    parameters plus the int64 row id (memory_tiers.py:33-38).  Budgets and
    FrameStats use this unit so eviction, prefetch and stall decisions are the
    reference's for the same budget_bytes; the pool itself holds f32 rows and
    an int64 prim key (row_bytes + 8 per row)."""
    return 8 * (3 + 4 + 3 + 1 + 3 * sh_coeffs) + 8


class HostTier:
    """The whole model in pinned host memory, rows regrouped so every group is
    a contiguous range; ``keys`` is the per-row depth-tie key."""

    def __init__(self, g, order: np.ndarray, keys: np.ndarray, groups: dict):
        order = np.asarray(order, dtype=np.int64)

        pinned = torch.cuda.is_available()

        def pin(a, dtype=torch.float32):
            t = torch.as_tensor(np.ascontiguousarray(np.asarray(a)[order])).to(dtype)
            return t.pin_memory() if pinned else t

        self.means = pin(g.means)
        self.quats = pin(g.quats)
        self.scales = pin(g.scales)
        self.logits = pin(g.opacity_logits)
        self.sh = pin(g.sh)
        self.keys = torch.as_tensor(np.asarray(keys, dtype=np.int64))
        if pinned:
            self.keys = self.keys.pin_memory()
        self.sh_degree = int(g.sh_degree)
        self.sh_coeffs = int(self.sh.shape[1])
        self.groups = groups  # gid -> (start, end) rows of this tier
        self.group_bytes = {gid: (e - s) * ref_row_bytes(self.sh_coeffs)
                            for gid, (s, e) in groups.items()}

    @property
    def count(self) -> int:
        return int(self.means.shape[0])


class DevicePool:
    """Paged device SoA: ``n_pages`` pages of 128 rows (one K1 CTA each)."""

    def __init__(self, n_pages: int, sh_coeffs: int, sh_degree: int, device=None):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else \
            torch.device(device)
        cap = max(1, n_pages) * PAGE_ROWS
        self.n_pages = max(1, n_pages)
        z = lambda *s: torch.zeros(s, dtype=torch.float32, device=dev)  # noqa: E731
        quats = z(cap, 4)
        quats[:, 0] = 1.0
        self.model = GaussianModel(z(cap, 3), quats, torch.ones(cap, 3, device=dev), z(cap),
                                   z(cap, sh_coeffs, 3), sh_degree, device=dev, validate=False)
        self.keys = torch.zeros(cap, dtype=torch.int64, device=dev)
        self.mask = torch.zeros(self.n_pages, dtype=torch.uint8, device=dev)
        self.free = list(range(self.n_pages))
        heapq.heapify(self.free)
        self.device = dev

    def alloc(self, rows: int) -> list[int]:
        need = -(-rows // PAGE_ROWS)
        if need > len(self.free):
            raise BudgetExceededError(f"pool out of pages ({need} > {len(self.free)} free)")
        return [heapq.heappop(self.free) for _ in range(need)]

    def release(self, pages) -> None:
        for p in pages:
            heapq.heappush(self.free, p)

    def copy_in(self, host: HostTier, start: int, end: int, pages: list[int]) -> None:
        """Enqueue the H2D copies of host rows [start, end) into ``pages`` on
        the current stream (runs of consecutive pages become one copy)."""
        m = self.model
        i, r = 0, start
        while r < end:
            j = i
            while j + 1 < len(pages) and pages[j + 1] == pages[j] + 1:
                j += 1
            n = min(end - r, (j - i + 1) * PAGE_ROWS)
            d0 = pages[i] * PAGE_ROWS
            for dst, src in ((m.means, host.means), (m.quats, host.quats),
                             (m.scales, host.scales), (m.opacity_logits, host.logits),
                             (m.sh, host.sh), (self.keys, host.keys)):
                dst[d0:d0 + n].copy_(src[r:r + n], non_blocking=True)
            r += n
            i = j + 1

    def copy_out(self, host: HostTier, start: int, end: int, pages: list[int]) -> None:
        m = self.model
        r = start
        for p in pages:
            n = min(end - r, PAGE_ROWS)
            d0 = p * PAGE_ROWS
            for dst, src in ((host.means, m.means), (host.quats, m.quats),
                             (host.scales, m.scales), (host.logits, m.opacity_logits),
                             (host.sh, m.sh)):
                dst[r:r + n].copy_(src[d0:d0 + n], non_blocking=False)
            r += n

    def set_mask(self, runs) -> torch.Tensor:
        """Per-page live-row counts of a frame: ``runs`` = [(pages, rows)] of the
        groups it renders (stream-ordered device update)."""
        self.mask.zero_()
        idx, cnt = [], []
        for pages, rows in runs:
            for k, p in enumerate(pages):
                idx.append(p)
                cnt.append(min(PAGE_ROWS, rows - k * PAGE_ROWS))
        if idx:
            t = torch.tensor([idx, cnt], dtype=torch.long).to(self.device, non_blocking=False)
            self.mask.index_copy_(0, t[0], t[1].to(torch.uint8))
        return self.mask


class TierStore:
    """memory_tiers.py:74-147 with a real device tier: all-or-nothing loads
    against the byte budget, virtual-clock completion (the reference's stats),
    and asynchronous copies into the paged pool on ``copy_stream``."""

    def __init__(self, budget_bytes: int, host: HostTier, transfer: TransferConfig | None = None,
                 clock: VirtualClock | None = None, device=None):
        self.budget_bytes = int(budget_bytes)
        self.transfer = transfer or TransferConfig()
        self.clock = clock or VirtualClock()
        self.host = host
        self.device: dict = {}  # gid -> pages
        self.events: dict = {}  # gid -> cuda event of its copies
        self.resident_bytes = 0
        self.stats = TierStats()
        rb = ref_row_bytes(host.sh_coeffs)
        # budget rows plus one partial page per group that can be resident
        pages_all = sum(-(-(e - s) // PAGE_ROWS) for s, e in host.groups.values())
        n_groups = len(host.groups)
        pages = min(pages_all, self.budget_bytes // rb // PAGE_ROWS + n_groups + 1)
        self.pool = DevicePool(pages, host.sh_coeffs, host.sh_degree, device)
        self.copy_stream = torch.cuda.Stream(device=self.pool.device)
        self.render_done: torch.cuda.Event | None = None

    # -- host management
    def host_bytes(self, gid) -> int:
        return self.host.group_bytes[gid]

    def total_host_bytes(self) -> int:
        return sum(self.host.group_bytes.values())

    def _transfer_time(self, nbytes: int) -> float:
        bw = self.transfer.bandwidth_bytes_per_s
        dur = self.transfer.fixed_latency_s
        if bw is not None and bw > 0:
            dur += nbytes / bw
        return dur

    def load_cells(self, gids) -> LoadHandle:
        gids = tuple(gids)
        for g in gids:
            if g not in self.host.groups:
                raise NotResidentError(f"cell {g} not in host tier")
        new = [g for g in gids if g not in self.device]
        nbytes = sum(self.host.group_bytes[g] for g in new)
        if self.resident_bytes + nbytes > self.budget_bytes:
            raise BudgetExceededError(
                f"loading {nbytes} bytes would exceed budget "
                f"({self.resident_bytes}/{self.budget_bytes} resident)")
        ev = None
        if new:
            with torch.cuda.stream(self.copy_stream):
                if self.render_done is not None:  # pages may be reused from evicted groups
                    self.copy_stream.wait_event(self.render_done)
                for g in new:
                    s, e = self.host.groups[g]
                    pages = self.pool.alloc(e - s)
                    self.pool.copy_in(self.host, s, e, pages)
                    self.device[g] = pages
                ev = torch.cuda.Event()
                ev.record(self.copy_stream)
            for g in new:
                self.events[g] = ev
        self.resident_bytes += nbytes
        self.stats.loads += len(new)
        self.stats.bytes_in += nbytes
        self.stats.peak_resident_bytes = max(self.stats.peak_resident_bytes, self.resident_bytes)
        return LoadHandle(gids, self.clock.now + self._transfer_time(nbytes), nbytes, ev)

    def offload_cells(self, gids, write_back: bool = False) -> int:
        gids = tuple(gids)
        for g in gids:
            if g not in self.device:
                raise NotResidentError(f"cell {g} not resident on device")
        freed = 0
        for g in gids:
            pages = self.device.pop(g)
            self.events.pop(g, None)
            if write_back:
                torch.cuda.current_stream().wait_stream(self.copy_stream)
                s, e = self.host.groups[g]
                self.pool.copy_out(self.host, s, e, pages)
            self.pool.release(pages)
            freed += self.host.group_bytes[g]
        self.resident_bytes -= freed
        self.stats.offloads += len(gids)
        self.stats.bytes_out += freed
        return freed

    def is_resident(self, gid) -> bool:
        return gid in self.device

    def render_groups(self, camera, gids, cfg) -> torch.Tensor:
        """Render the union of resident groups straight from the pool: the
        render stream waits (on the device) for their copies."""
        cur = torch.cuda.current_stream(self.pool.device)
        seen = set()
        runs = []
        for g in gids:
            if g not in self.device:
                raise NotResidentError(f"cell {g} not resident on device")
            ev = self.events.get(g)
            if ev is not None and id(ev) not in seen:
                cur.wait_event(ev)
                seen.add(id(ev))
            s, e = self.host.groups[g]
            runs.append((self.device[g], e - s))
        mask = self.pool.set_mask(runs)
        out = render(camera, self.pool.model, cfg.tile_size, cfg.background, cfg.sh_eval_degree,
                     prim_ids=self.pool.keys, page_mask=mask, page_shift=PAGE_SHIFT)
        self.render_done = torch.cuda.Event()
        self.render_done.record(cur)
        return out.rgb


# ---------------------------------------------------------------------------
# double buffering and prefetch policy (memory_tiers.py:150-247)


@dataclass
class Region:
    cell_ids: frozenset
    core: tuple | None = None


@dataclass
class BufferPair:
    front: Region | None = None
    back: tuple | None = None  # (Region, LoadHandle)

    def swap(self, clock: VirtualClock) -> None:
        if self.back is None:
            raise IncompleteLoadError("no back buffer to swap in")
        region, handle = self.back
        if not handle.ready(clock):
            raise IncompleteLoadError(
                f"back buffer load completes at t={handle.ready_at:.6f}, now t={clock.now:.6f}")
        self.front, self.back = region, None


@dataclass(frozen=True)
class TriggerZones:
    inner_fraction: float = 0.5
    outer_fraction: float = 0.8

    def __post_init__(self):
        if not 0 < self.inner_fraction < self.outer_fraction <= 1:
            raise InvalidConfigError("require 0 < inner < outer <= 1")


@dataclass(frozen=True)
class PrefetchAction:
    kind: str  # none | start_load | swap | stall_then_swap
    target_core: tuple | None = None


def prefetch_policy(position, velocity, core_cell, zones: TriggerZones, pair: BufferPair,
                    grid: SceneGrid, clock: VirtualClock) -> PrefetchAction:
    """memory_tiers.py:196-247: nested trigger zones inside the core cell."""
    cb = grid.cell_bbox(core_cell)
    center = (cb[0, :2] + cb[1, :2]) / 2
    half = (cb[1, :2] - cb[0, :2]) / 2
    rel = (np.asarray(position, dtype=float)[:2] - center) / half
    frac = np.abs(rel)
    if np.all(frac < zones.inner_fraction):
        return PrefetchAction("none")
    vel = np.asarray(velocity, dtype=float)[:2]
    crossed = frac >= zones.inner_fraction
    candidates = [a for a in (0, 1) if crossed[a] and vel[a] * rel[a] > 0]
    if not candidates:
        candidates = [int(np.argmax(frac))]
    axis = max(candidates, key=lambda a: abs(vel[a]))
    step = 1 if rel[axis] > 0 else -1
    target = list(core_cell)
    target[axis] += step
    target[0] = min(max(target[0], 0), grid.nx - 1)
    target[1] = min(max(target[1], 0), grid.ny - 1)
    target = tuple(target)
    beyond_outer = bool(np.any(frac >= zones.outer_fraction))
    if beyond_outer and pair.back is not None:
        region, handle = pair.back
        if handle.ready(clock):
            return PrefetchAction("swap", target_core=region.core)
        return PrefetchAction("stall_then_swap", target_core=region.core)
    pending = pair.back is not None and pair.back[0].core == target
    front_covers = pair.front is not None and pair.front.core == target
    if pending or front_covers or target == core_cell:
        return PrefetchAction("none")
    return PrefetchAction("start_load", target_core=target)


# ---------------------------------------------------------------------------
# sessions (render_runtime.py)


@dataclass
class SessionConfig:
    """render_runtime.py:81-97 (+ sh_eval_degree: 1 = the reference's colours)."""

    mode: str = "static_full"
    budget_bytes: int | None = None
    ring: int = 1
    tile_size: int = 16
    zones: TriggerZones = field(default_factory=TriggerZones)
    transfer: TransferConfig = field(default_factory=TransferConfig)
    voxel_size: float = 1.0
    background: tuple = (0.0, 0.0, 0.0)
    sh_eval_degree: int = 1

    def __post_init__(self):
        if self.mode not in RENDER_MODES:
            raise InvalidConfigError(f"mode must be one of {RENDER_MODES}, got {self.mode!r}")
        if self.mode != "static_full" and self.budget_bytes is None:
            raise InvalidConfigError(f"mode {self.mode!r} requires budget_bytes")


@dataclass
class FrameStats:
    index: int
    t: float
    latency_ms: float
    resident_bytes: int
    peak_resident_bytes: int
    stalls: int
    core_cell: tuple | None = None
    n_primitives: int = 0

    def as_dict(self) -> dict:
        d = dict(self.__dict__)
        d["core_cell"] = list(self.core_cell) if self.core_cell else None
        return d


def _host_arrays(model):
    """(means, quats, scales, logits, sh, degree) as host numpy from a host or
    device model."""
    f = lambda t: t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)  # noqa: E731
    return (f(model.means), f(model.quats), f(model.scales), f(model.opacity_logits), f(model.sh),
            int(model.sh_degree))


class _HostModel:
    def __init__(self, arrs):
        self.means, self.quats, self.scales, self.opacity_logits, self.sh, self.sh_degree = arrs


class BlockSession:
    """render_runtime.py:110-193: the front buffer covers the camera's core
    cell region; the back buffer is filled ahead of crossings."""

    def __init__(self, model, grid: SceneGrid, cfg: SessionConfig,
                 clock: VirtualClock | None = None, device=None):
        self.grid, self.cfg = grid, cfg
        self.clock = clock or VirtualClock()
        arrs = _host_arrays(model)
        rows = cell_rows(arrs[0], grid)
        order, groups, start = [], {}, 0
        keys = []
        # prim key = (rank of the cell in sorted (ix, iy) order, original id):
        # the order of model_from_groups' concatenation over any set of cells
        for rank, cell in enumerate(sorted(grid.cells())):
            ids = rows[cell]
            order.append(ids)
            keys.append((np.int64(rank) << 32) + ids.astype(np.int64))
            groups[cell] = (start, start + len(ids))
            start += len(ids)
        host = HostTier(_HostModel(arrs), np.concatenate(order), np.concatenate(keys), groups)
        worst = max(sum(host.group_bytes[c] for c in onload_region(grid, cell, cfg.ring))
                    for cell in grid.cells())
        if 2 * worst > cfg.budget_bytes:
            raise BudgetExceededError(
                f"budget {cfg.budget_bytes} bytes cannot double-buffer the largest "
                f"onload region (2 x {worst} bytes)")
        self.store = TierStore(cfg.budget_bytes, host, cfg.transfer, self.clock, device)
        self.pair = BufferPair()
        self.stalls = 0

    def _region_cells(self, core):
        return frozenset(onload_region(self.grid, core, self.cfg.ring))

    def _load_region(self, core):
        cells = self._region_cells(core)
        handle = self.store.load_cells(sorted(cells))
        return Region(cells, core), handle

    def _drop_unreferenced(self):
        keep = set()
        if self.pair.front:
            keep |= self.pair.front.cell_ids
        if self.pair.back:
            keep |= self.pair.back[0].cell_ids
        stale = [c for c in list(self.store.device) if c not in keep]
        if stale:
            self.store.offload_cells(stale, write_back=False)

    def _force_resident(self, core):
        self.stalls += 1
        self.store.stats.stalls += 1
        region, handle = self._load_region(core)
        self.clock.advance(max(0.0, handle.ready_at - self.clock.now))
        self.pair.front, self.pair.back = region, None
        self._drop_unreferenced()

    def step(self, camera, velocity) -> tuple[torch.Tensor, int]:
        core = self.grid.cell_of_point(camera.center)
        if self.pair.front is None:
            region, handle = self._load_region(core)
            self.clock.advance(max(0.0, handle.ready_at - self.clock.now))
            self.pair.front = region
        action = prefetch_policy(camera.center, velocity, self.pair.front.core, self.cfg.zones,
                                 self.pair, self.grid, self.clock)
        if action.kind == "start_load":
            self.pair.back = self._load_region(action.target_core)
        elif action.kind == "swap":
            self.pair.swap(self.clock)
            self._drop_unreferenced()
        elif action.kind == "stall_then_swap":
            self.stalls += 1
            self.store.stats.stalls += 1
            _, handle = self.pair.back
            self.clock.advance(max(0.0, handle.ready_at - self.clock.now))
            self.pair.swap(self.clock)
            self._drop_unreferenced()
        if core not in self.pair.front.cell_ids:
            self._force_resident(core)
        cells = sorted(self.pair.front.cell_ids)
        image = self.store.render_groups(camera, cells, self.cfg)
        n = sum(e - s for s, e in (self.store.host.groups[c] for c in cells))
        return image, n


class FrustumSession:
    """render_runtime.py:199-243: least-recently-visible voxel cache bounded by
    the byte budget; each frame renders the frustum-visible voxels."""

    def __init__(self, model, cfg: SessionConfig, clock: VirtualClock | None = None,
                 device=None):
        self.cfg = cfg
        self.clock = clock or VirtualClock()
        arrs = _host_arrays(model)
        self.index = reorder_voxel_grid(arrs[0], arrs[2], cfg.voxel_size)
        perm = self.index.permutation
        groups = {v: (int(s), int(e)) for v, (s, e) in enumerate(self.index.ranges)}
        # prim key = row of the voxel-reordered model (render_image's subset ids)
        host = HostTier(_HostModel(arrs), perm, np.arange(len(perm), dtype=np.int64), groups)
        self.store = TierStore(cfg.budget_bytes, host, cfg.transfer, self.clock, device)
        self.last_visible: dict = {}
        self.frame = 0
        self.stalls = 0

    def step(self, camera) -> tuple[torch.Tensor, int]:
        self.frame += 1
        needed = frustum_visible_voxels(self.index, camera)
        store = self.store
        need_bytes = sum(store.host_bytes(v) for v in needed if not store.is_resident(v))
        if store.resident_bytes + need_bytes > store.budget_bytes:
            evictable = sorted((v for v in store.device if v not in needed),
                               key=lambda v: self.last_visible.get(v, -1))
            while evictable and store.resident_bytes + need_bytes > store.budget_bytes:
                store.offload_cells([evictable.pop(0)], write_back=False)
        handle = store.load_cells(needed)
        wait = handle.ready_at - self.clock.now
        if wait > 0:
            self.stalls += 1
            store.stats.stalls += 1
            self.clock.advance(wait)
        for v in needed:
            self.last_visible[v] = self.frame
        image = store.render_groups(camera, needed, self.cfg)
        n = int(sum(self.index.ranges[v, 1] - self.index.ranges[v, 0] for v in needed))
        return image, n


def run_session(model, cameras, timestamps, cfg: SessionConfig, grid: SceneGrid | None = None,
                clock: VirtualClock | None = None, keep_images: bool = True, device=None):
    """render_runtime.py:250-308: (images, [FrameStats]).  Frame latency is
    wall time with the frame's GPU work completed (synchronised)."""
    if len(cameras) != len(timestamps):
        raise InvalidInputError("one timestamp per camera required")
    clock = clock or VirtualClock()
    if cfg.mode == "block_double_buffer":
        if grid is None:
            raise InvalidInputError("block_double_buffer requires a scene grid")
        session = BlockSession(model, grid, cfg, clock, device)
    elif cfg.mode == "frustum_voxel":
        session = FrustumSession(model, cfg, clock, device)
    else:
        session = None
        dev_model = model if isinstance(model, GaussianModel) else \
            GaussianModel.from_host(_HostModel(_host_arrays(model)), device=device)
        # the reference's fp64 model bytes (render_runtime.py:270-273)
        model_nbytes = dev_model.count * (ref_row_bytes(int(dev_model.sh.shape[1])) - 8)
        ctx = context(dev_model.device.index)
    images, stats = [], []
    prev_pos, prev_t = None, None
    for i, (cam, t) in enumerate(zip(cameras, timestamps)):
        cam = cam if isinstance(cam, Camera) else Camera.from_reference(cam)
        if prev_t is not None and t > prev_t:
            clock.advance(t - prev_t)
        pos = cam.center
        dt = (t - prev_t) if prev_t is not None and t > prev_t else 1.0
        vel = (pos - prev_pos) / dt if prev_pos is not None else np.zeros(3)
        wall0 = time.perf_counter()
        if cfg.mode == "static_full":
            image = render(cam, dev_model, cfg.tile_size, cfg.background, cfg.sh_eval_degree,
                           ctx=ctx).rgb
            n_prims, core, resident, peak, stalls = dev_model.count, None, model_nbytes, \
                model_nbytes, 0
        elif cfg.mode == "block_double_buffer":
            image, n_prims = session.step(cam, vel)
            core = session.pair.front.core
            resident = session.store.resident_bytes
            peak = session.store.stats.peak_resident_bytes
            stalls = session.stalls
        else:
            image, n_prims = session.step(cam)
            core = None
            resident = session.store.resident_bytes
            peak = session.store.stats.peak_resident_bytes
            stalls = session.stalls
        torch.cuda.current_stream().synchronize()
        stats.append(FrameStats(i, float(t), (time.perf_counter() - wall0) * 1e3, resident, peak,
                                stalls, core, n_prims))
        if keep_images:
            images.append(image)
        prev_pos, prev_t = pos, t
    return images, stats


def bench(model, cameras, timestamps, cfg: SessionConfig, grid: SceneGrid | None = None) -> dict:
    """render_runtime.py:311-326."""
    _, stats = run_session(model, cameras, timestamps, cfg, grid=grid, keep_images=False)
    lat = [s.latency_ms for s in stats]
    total_s = sum(lat) / 1e3
    return {"frames": len(stats),
            "mean_latency_ms": statistics.fmean(lat) if lat else 0.0,
            "median_latency_ms": statistics.median(lat) if lat else 0.0,
            "fps": len(stats) / total_s if total_s > 0 else 0.0,
            "peak_resident_bytes": max((s.peak_resident_bytes for s in stats), default=0),
            "stalls": stats[-1].stalls if stats else 0}
