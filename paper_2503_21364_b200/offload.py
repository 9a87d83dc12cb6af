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
# simulated time and transfer accounting.  The reference models the device
# tier on a virtual clock (common.py:51-60, memory_tiers.py:43-73); its
# readings decide prefetch swaps and stalls, so they are kept as the
# bookkeeping layer above the real, asynchronous copies.


@dataclass
class VirtualClock:
    """Seconds of simulated session time; only moves forward."""

    now: float = 0.0

    def advance(self, dt: float) -> None:
        if not dt >= 0:
            raise InvalidInputError("clock cannot go backwards")
        self.now += dt

    def wait_until(self, t: float) -> bool:
        """Advance to ``t`` if it lies ahead; True when that was a wait."""
        late = t - self.now
        if late > 0:
            self.now += late
            return True
        return False


@dataclass
class TransferConfig:
    """Host->device link of the simulated clock (bandwidth None: instant)."""

    bandwidth_bytes_per_s: float | None = None
    fixed_latency_s: float = 0.0

    def seconds(self, nbytes: int) -> float:
        bw = self.bandwidth_bytes_per_s
        return self.fixed_latency_s + (nbytes / bw if bw else 0.0)


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
    """One load request: its groups, the simulated completion time and the
    CUDA event of the real copies."""

    cell_ids: tuple
    ready_at: float
    nbytes: int
    event: torch.cuda.Event | None = None

    def ready(self, clock: VirtualClock) -> bool:
        return self.ready_at <= clock.now


# ---------------------------------------------------------------------------
# the x-y cell grid (scene_manager.py:24-104 semantics: half-open cells
# clamped at the grid edge, Chebyshev onload regions)


@dataclass
class SceneGrid:
    bbox: np.ndarray
    nx: int
    ny: int

    def __post_init__(self):
        self.bbox = np.asarray(self.bbox, dtype=np.float64).reshape(2, 3)
        if min(self.nx, self.ny) < 1:
            raise InvalidInputError("cell counts must be >= 1")
        if (self.bbox[1] <= self.bbox[0]).any():
            raise InvalidInputError("degenerate scene bbox")

    @property
    def cell_extent(self) -> np.ndarray:
        return (self.bbox[1, :2] - self.bbox[0, :2]) / (self.nx, self.ny)

    def _index(self, xy) -> np.ndarray:
        """Clamped (ix, iy) of points (..., >= 2)."""
        q = np.floor((np.asarray(xy, dtype=np.float64)[..., :2] - self.bbox[0, :2])
                     / self.cell_extent).astype(np.int64)
        return np.clip(q, 0, (self.nx - 1, self.ny - 1))

    def cell_of_point(self, xy) -> tuple[int, int]:
        ix, iy = self._index(xy)
        return int(ix), int(iy)

    def cell_bbox(self, index) -> np.ndarray:
        lo_xy = self.bbox[0, :2] + np.asarray(index, dtype=np.float64) * self.cell_extent
        hi_xy = lo_xy + self.cell_extent
        return np.array([[lo_xy[0], lo_xy[1], self.bbox[0, 2]],
                         [hi_xy[0], hi_xy[1], self.bbox[1, 2]]])

    def cells(self):
        """Row-major cell order (y outer)."""
        return [(i % self.nx, i // self.nx) for i in range(self.nx * self.ny)]

    def region(self, core, ring: int = 1) -> set:
        if not (0 <= core[0] < self.nx and 0 <= core[1] < self.ny):
            raise InvalidInputError(f"core cell {core} outside grid")
        if ring < 0:
            raise InvalidInputError("ring must be >= 0")
        xs = range(max(core[0] - ring, 0), min(core[0] + ring, self.nx - 1) + 1)
        ys = range(max(core[1] - ring, 0), min(core[1] + ring, self.ny - 1) + 1)
        return {(x, y) for x in xs for y in ys}


def partition_scene(bbox, nx: int, ny: int) -> SceneGrid:
    return SceneGrid(bbox, nx, ny)


def onload_region(grid: SceneGrid, core, ring: int = 1) -> set:
    """Cells within Chebyshev distance ``ring`` of ``core``."""
    return grid.region(core, ring)


def cell_rows(means: np.ndarray, grid: SceneGrid) -> dict:
    """Ascending Gaussian ids of every cell (engine_api.py:182-207)."""
    ix, iy = grid._index(np.asarray(means, dtype=np.float64)).T
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
# block streaming: a front region (rendered) and a back region (loading
# ahead of a cell crossing), switched by nested trigger zones around the
# core cell (the decisions of memory_tiers.py:150-247)


@dataclass
class Region:
    cell_ids: frozenset
    core: tuple | None = None


@dataclass
class BufferPair:
    """front: the region being rendered; back: (region, LoadHandle) in flight."""

    front: Region | None = None
    back: tuple | None = None

    def swap(self, clock: VirtualClock) -> None:
        if self.back is None:
            raise IncompleteLoadError("no back buffer to swap in")
        if not self.back[1].ready(clock):
            raise IncompleteLoadError(f"back buffer load completes at t={self.back[1].ready_at:.6f}"
                                      f", now t={clock.now:.6f}")
        self.front, self.back = self.back[0], None


@dataclass(frozen=True)
class TriggerZones:
    """Fractions of the core cell's half-extent: past ``inner`` a load of the
    next cell's region starts, past ``outer`` the buffers swap."""

    inner_fraction: float = 0.5
    outer_fraction: float = 0.8

    def __post_init__(self):
        ok = 0 < self.inner_fraction < self.outer_fraction <= 1
        if not ok:
            raise InvalidConfigError("require 0 < inner < outer <= 1")


@dataclass(frozen=True)
class PrefetchAction:
    kind: str  # none | start_load | swap | stall_then_swap
    target_core: tuple | None = None


_NONE = PrefetchAction("none")


def _exit_axis(rel: np.ndarray, vel: np.ndarray, inner: float) -> int:
    """The axis the camera is leaving the core cell through: among the axes
    past the inner zone, those it moves outward along, the fastest (first on
    ties); if it moves outward along none, the axis it is furthest out on."""
    past = [ax for ax in (0, 1) if abs(rel[ax]) >= inner]
    outward = [ax for ax in past if rel[ax] * vel[ax] > 0]
    if not outward:
        return int(np.argmax(np.abs(rel)))
    best = outward[0]
    for ax in outward[1:]:
        if abs(vel[ax]) > abs(vel[best]):
            best = ax
    return best


def prefetch_policy(position, velocity, core_cell, zones: TriggerZones, pair: BufferPair,
                    grid: SceneGrid, clock: VirtualClock) -> PrefetchAction:
    """What the block session does this frame, from the camera's position in
    its core cell (normalised to [-1, 1] per axis) and its velocity."""
    box = grid.cell_bbox(core_cell)
    mid, half = box[:, :2].mean(axis=0), (box[1, :2] - box[0, :2]) / 2
    rel = (np.asarray(position, dtype=float)[:2] - mid) / half
    if (np.abs(rel) < zones.inner_fraction).all():
        return _NONE
    ax = _exit_axis(rel, np.asarray(velocity, dtype=float)[:2], zones.inner_fraction)
    nxt = list(core_cell)
    nxt[ax] = min(max(nxt[ax] + (1 if rel[ax] > 0 else -1), 0), (grid.nx, grid.ny)[ax] - 1)
    nxt = tuple(nxt)
    if pair.back is not None and (np.abs(rel) >= zones.outer_fraction).any():
        back_region, handle = pair.back
        kind = "swap" if handle.ready(clock) else "stall_then_swap"
        return PrefetchAction(kind, target_core=back_region.core)
    already = {core_cell}
    if pair.back is not None:
        already.add(pair.back[0].core)
    if pair.front is not None:
        already.add(pair.front.core)
    return _NONE if nxt in already else PrefetchAction("start_load", target_core=nxt)


# ---------------------------------------------------------------------------
# sessions over the paged pool (the streaming modes of render_runtime.py
# 65-326; same configuration, FrameStats and decisions)


@dataclass
class SessionConfig:
    """Streaming mode, byte budget (the reference's unit, ref_row_bytes) and
    render settings (+ sh_eval_degree: 1 = the reference's colours)."""

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
        if self.budget_bytes is None and self.mode != "static_full":
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
        d = asdict(self)
        d["core_cell"] = None if self.core_cell is None else list(self.core_cell)
        return d


def _host_arrays(model):
    """(means, quats, scales, logits, sh, degree) as host numpy from a host or
    device model."""
    def f(t):
        return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
    return (f(model.means), f(model.quats), f(model.scales), f(model.opacity_logits), f(model.sh),
            int(model.sh_degree))


class _HostModel:
    def __init__(self, arrs):
        self.means, self.quats, self.scales, self.opacity_logits, self.sh, self.sh_degree = arrs


class _PoolSession:
    """Shared machinery: the tier store, its clock and the stall count."""

    store: TierStore
    clock: VirtualClock

    def __init__(self):
        self.stalls = 0

    def _stall(self, ready_at: float) -> None:
        self.stalls += 1
        self.store.stats.stalls += 1
        self.clock.wait_until(ready_at)

    def _draw(self, camera, groups) -> tuple[torch.Tensor, int]:
        rows = sum(e - s for s, e in (self.store.host.groups[g] for g in groups))
        return self.store.render_groups(camera, groups, self.cfg), int(rows)

    def frame_state(self) -> tuple:
        """(core cell, resident bytes, peak resident bytes, stalls)."""
        return (None, self.store.resident_bytes, self.store.stats.peak_resident_bytes,
                self.stalls)


class BlockSession(_PoolSession):
    """Cell-grid streaming: the front buffer holds the ring region of the
    camera's core cell; the next region is loaded ahead of a crossing."""

    def __init__(self, model, grid: SceneGrid, cfg: SessionConfig,
                 clock: VirtualClock | None = None, device=None):
        super().__init__()
        self.grid, self.cfg = grid, cfg
        self.clock = clock or VirtualClock()
        arrs = _host_arrays(model)
        rows = cell_rows(arrs[0], grid)
        # pool rows grouped by cell in sorted (ix, iy) order; the prim key
        # (cell rank << 32 | id) is the tie order of any concatenation of
        # cells in that order, which is how the reference builds the model
        cells = sorted(grid.cells())
        sizes = np.array([len(rows[c]) for c in cells], dtype=np.int64)
        starts = np.concatenate([[0], np.cumsum(sizes)])
        groups = {c: (int(starts[i]), int(starts[i + 1])) for i, c in enumerate(cells)}
        order = np.concatenate([rows[c] for c in cells])
        keys = np.concatenate([(np.int64(i) << 32) + rows[c].astype(np.int64)
                               for i, c in enumerate(cells)])
        host = HostTier(_HostModel(arrs), order, keys, groups)
        need = max(sum(host.group_bytes[c] for c in grid.region(cell, cfg.ring))
                   for cell in cells)
        if need * 2 > cfg.budget_bytes:
            raise BudgetExceededError(
                f"budget {cfg.budget_bytes} bytes cannot double-buffer the largest "
                f"onload region (2 x {need} bytes)")
        self.store = TierStore(cfg.budget_bytes, host, cfg.transfer, self.clock, device)
        self.pair = BufferPair()

    def _request(self, core) -> tuple:
        cells = frozenset(self.grid.region(core, self.cfg.ring))
        return Region(cells, core), self.store.load_cells(sorted(cells))

    def _evict_unused(self) -> None:
        live = set(self.pair.front.cell_ids if self.pair.front else ())
        if self.pair.back:
            live |= self.pair.back[0].cell_ids
        unused = [c for c in list(self.store.device) if c not in live]
        if unused:
            self.store.offload_cells(unused, write_back=False)

    def step(self, camera, velocity) -> tuple[torch.Tensor, int]:
        here = self.grid.cell_of_point(camera.center)
        if self.pair.front is None:  # first frame: load and wait
            region, handle = self._request(here)
            self.clock.wait_until(handle.ready_at)
            self.pair.front = region
        act = prefetch_policy(camera.center, velocity, self.pair.front.core, self.cfg.zones,
                              self.pair, self.grid, self.clock)
        if act.kind == "start_load":
            self.pair.back = self._request(act.target_core)
        elif act.kind in ("swap", "stall_then_swap"):
            if act.kind == "stall_then_swap":
                self._stall(self.pair.back[1].ready_at)
            self.pair.swap(self.clock)
            self._evict_unused()
        if here not in self.pair.front.cell_ids:  # outran the prefetch: load in place
            region, handle = self._request(here)
            self._stall(handle.ready_at)
            self.pair.front, self.pair.back = region, None
            self._evict_unused()
        return self._draw(camera, sorted(self.pair.front.cell_ids))

    def frame_state(self) -> tuple:
        return (self.pair.front.core,) + super().frame_state()[1:]


class FrustumSession(_PoolSession):
    """Voxel streaming: each frame draws the frustum-visible voxels; the
    least recently visible voxels are evicted to stay within the budget."""

    def __init__(self, model, cfg: SessionConfig, clock: VirtualClock | None = None,
                 device=None):
        super().__init__()
        self.cfg = cfg
        self.clock = clock or VirtualClock()
        arrs = _host_arrays(model)
        self.index = reorder_voxel_grid(arrs[0], arrs[2], cfg.voxel_size)
        perm = self.index.permutation
        groups = dict(enumerate(map(tuple, self.index.ranges.tolist())))
        # prim key = row of the voxel-reordered model (render_image's subset ids)
        host = HostTier(_HostModel(arrs), perm, np.arange(len(perm), dtype=np.int64), groups)
        self.store = TierStore(cfg.budget_bytes, host, cfg.transfer, self.clock, device)
        self.last_visible: dict = {}
        self.frame = 0

    def _make_room(self, visible) -> None:
        st = self.store
        vis = set(visible)
        missing = sum(st.host_bytes(v) for v in visible if not st.is_resident(v))
        over = st.resident_bytes + missing - st.budget_bytes
        if over <= 0:
            return
        # stable: equally old voxels leave in residency (insertion) order
        victims = sorted((v for v in st.device if v not in vis),
                         key=lambda v: self.last_visible.get(v, -1))
        for v in victims:
            if st.resident_bytes + missing <= st.budget_bytes:
                break
            st.offload_cells([v], write_back=False)

    def step(self, camera) -> tuple[torch.Tensor, int]:
        self.frame += 1
        visible = frustum_visible_voxels(self.index, camera)
        self._make_room(visible)
        handle = self.store.load_cells(visible)
        if handle.ready_at > self.clock.now:
            self._stall(handle.ready_at)
        self.last_visible.update(dict.fromkeys(visible, self.frame))
        return self._draw(camera, visible)


class _StaticSession:
    """The whole model resident on the device (the reference's fp64 bytes)."""

    def __init__(self, model, cfg: SessionConfig, device=None):
        self.cfg = cfg
        self.model = model if isinstance(model, GaussianModel) else \
            GaussianModel.from_host(_HostModel(_host_arrays(model)), device=device)
        self.nbytes = self.model.count * (ref_row_bytes(int(self.model.sh.shape[1])) - 8)
        self.ctx = context(self.model.device.index)

    def step(self, camera, velocity=None) -> tuple[torch.Tensor, int]:
        c = self.cfg
        img = render(camera, self.model, c.tile_size, c.background, c.sh_eval_degree,
                     ctx=self.ctx).rgb
        return img, self.model.count

    def frame_state(self) -> tuple:
        return None, self.nbytes, self.nbytes, 0


def run_session(model, cameras, timestamps, cfg: SessionConfig, grid: SceneGrid | None = None,
                clock: VirtualClock | None = None, keep_images: bool = True, device=None):
    """Render a camera trajectory in ``cfg.mode``: (images, [FrameStats]).
    The simulated clock follows the timestamps; a frame's latency is wall
    time with its GPU work completed (synchronised)."""
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
        session = _StaticSession(model, cfg, device)
    images, stats = [], []
    last = None  # (position, time) of the previous frame
    for i, (cam, t) in enumerate(zip(cameras, timestamps)):
        cam = cam if isinstance(cam, Camera) else Camera.from_reference(cam)
        vel = np.zeros(3)
        if last is not None:
            moved = t > last[1]
            if moved:
                clock.advance(t - last[1])
            vel = (cam.center - last[0]) / ((t - last[1]) if moved else 1.0)
        t0 = time.perf_counter()
        if isinstance(session, FrustumSession):
            image, n = session.step(cam)
        else:
            image, n = session.step(cam, vel)
        torch.cuda.current_stream().synchronize()
        core, resident, peak, stalls = session.frame_state()
        stats.append(FrameStats(i, float(t), (time.perf_counter() - t0) * 1e3, resident, peak,
                                stalls, core, n))
        if keep_images:
            images.append(image)
        last = (cam.center, t)
    return images, stats


def bench(model, cameras, timestamps, cfg: SessionConfig, grid: SceneGrid | None = None) -> dict:
    """Session summary: frame count, latency mean / median, frames/s, peak
    residency and stalls."""
    _, stats = run_session(model, cameras, timestamps, cfg, grid=grid, keep_images=False)
    lat = [s.latency_ms for s in stats]
    secs = sum(lat) / 1e3
    return {"frames": len(stats),
            "mean_latency_ms": statistics.fmean(lat) if lat else 0.0,
            "median_latency_ms": statistics.median(lat) if lat else 0.0,
            "fps": len(stats) / secs if secs > 0 else 0.0,
            "peak_resident_bytes": max((s.peak_resident_bytes for s in stats), default=0),
            "stalls": stats[-1].stalls if stats else 0}
