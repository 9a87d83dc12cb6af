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
from dataclasses import asdict, dataclass, field, make_dataclass

import numpy as np
import torch

from .camera import Camera
from .errors import InvalidConfigError, InvalidInputError
from .raster import GaussianModel, context, render

PAGE_SHIFT = 7
PAGE_ROWS = 1 << PAGE_SHIFT
# session modes, named as the reference names them (render_runtime.py)
RENDER_MODES = tuple("static_full block_double_buffer frustum_voxel".split())


# error types of the reference's tier store (memory_tiers.py:18-26)
BudgetExceededError = type("BudgetExceededError", (RuntimeError,),
                           {"__doc__": "a load would exceed the device byte budget"})
NotResidentError = type("NotResidentError", (KeyError,),
                        {"__doc__": "a group is not where the call expects it"})
IncompleteLoadError = type("IncompleteLoadError", (RuntimeError,),
                           {"__doc__": "the back buffer's load has not completed"})


def _record(name: str, spec, doc: str, frozen: bool = False, **methods):
    """A dataclass from (field, type[, default]) triples."""
    cls = make_dataclass(name, spec, namespace=methods, frozen=frozen)
    cls.__doc__ = doc
    cls.__module__ = __name__
    return cls


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
        self.now += max(late, 0.0)
        return late > 0


def _link_seconds(self, nbytes: int) -> float:
    bw = self.bandwidth_bytes_per_s
    return self.fixed_latency_s + (nbytes / bw if bw is not None and bw > 0 else 0.0)


TransferConfig = _record(
    "TransferConfig", [("bandwidth_bytes_per_s", "float | None", field(default=None)),
                       ("fixed_latency_s", float, field(default=0.0))],
    "Host->device link of the simulated clock (bandwidth None: instant).",
    seconds=_link_seconds)

TierStats = _record(
    "TierStats", [(k, int, field(default=0)) for k in
                  "loads offloads bytes_in bytes_out stalls peak_resident_bytes".split()],
    "Tier store counters (the reference's names).", snapshot=lambda self: asdict(self))

LoadHandle = _record(
    "LoadHandle", [("cell_ids", tuple), ("ready_at", float), ("nbytes", int),
                   ("event", "torch.cuda.Event | None", field(default=None))],
    "One load request: its groups, the simulated completion time and the CUDA "
    "event of the real copies.", ready=lambda self, clock: self.ready_at <= clock.now)


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
            raise InvalidInputError("grid needs at least one cell per axis (cell counts must be >= 1)")
        if (self.bbox[1] <= self.bbox[0]).any():
            raise InvalidInputError("scene bbox has no volume (degenerate scene bbox)")

    @property
    def cell_extent(self) -> np.ndarray:
        return (self.bbox[1, :2] - self.bbox[0, :2]) / (self.nx, self.ny)

    def _index(self, xy) -> np.ndarray:
        """Clamped (ix, iy) of points (..., >= 2)."""
        q = np.floor((np.asarray(xy, dtype=np.float64)[..., :2] - self.bbox[0, :2])
                     / self.cell_extent).astype(np.int64)
        return np.clip(q, 0, (self.nx - 1, self.ny - 1))

    def cell_of_point(self, xy):
        ix, iy = self._index(xy)
        return int(ix), int(iy)

    def cell_bbox(self, index):
        lo_xy = self.bbox[0, :2] + np.asarray(index, dtype=np.float64) * self.cell_extent
        hi_xy = lo_xy + self.cell_extent
        return np.array([[lo_xy[0], lo_xy[1], self.bbox[0, 2]],
                         [hi_xy[0], hi_xy[1], self.bbox[1, 2]]])

    def cells(self):
        """Row-major cell order (y outer)."""
        return [(i % self.nx, i // self.nx) for i in range(self.nx * self.ny)]

    def region(self, core, ring: int = 1) -> set:
        if not (0 <= core[0] < self.nx and 0 <= core[1] < self.ny):
            raise InvalidInputError(f"core cell {core} is not a cell of the grid")
        if not ring >= 0:
            raise InvalidInputError(f"onload ring {ring} is negative")
        xs = range(max(core[0] - ring, 0), min(core[0] + ring, self.nx - 1) + 1)
        ys = range(max(core[1] - ring, 0), min(core[1] + ring, self.ny - 1) + 1)
        return {(x, y) for x in xs for y in ys}


def partition_scene(bbox, nx, ny) -> SceneGrid:
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


# ---------------------------------------------------------------------------
# voxel index and frustum visibility (scene_manager.py:129-253 semantics)


@dataclass
class VoxelIndex:
    """Voxel-sorted rows: ``permutation`` (new row -> input row), per voxel
    its integer key, row range [start, end) and largest scale."""

    voxel_size: float
    origin: np.ndarray
    voxel_keys: np.ndarray
    ranges: np.ndarray
    permutation: np.ndarray
    voxel_max_scale: np.ndarray

    @property
    def n_voxels(self) -> int:
        return int(self.voxel_keys.shape[0])

    def voxel_bbox(self, v: int, margin: float = 0.0) -> np.ndarray:
        corner = self.origin + self.voxel_size * self.voxel_keys[v]
        return np.stack([corner - margin, corner + self.voxel_size + margin])


def reorder_voxel_grid(means: np.ndarray, scales: np.ndarray, voxel_size: float) -> VoxelIndex:
    """Sort rows by voxel key (x, then y, then z; stable), fp64 arithmetic."""
    if not voxel_size > 0:
        raise InvalidInputError(f"voxel_size must be positive, got {voxel_size}")
    pts = np.asarray(means, dtype=np.float64)
    n = pts.shape[0]
    origin = voxel_size * np.floor(pts.min(axis=0) / voxel_size)
    key = np.floor((pts - origin) / voxel_size).astype(np.int64)
    perm = np.lexsort((np.arange(n), key[:, 2], key[:, 1], key[:, 0]))
    key = key[perm]
    new_voxel = np.ones(n, dtype=bool)
    new_voxel[1:] = (key[1:] != key[:-1]).any(axis=1)
    first = np.flatnonzero(new_voxel)
    last = np.append(first[1:], n)
    big = np.asarray(scales, dtype=np.float64).max(axis=-1)[perm]
    vmax = np.maximum.reduceat(big, first) if n else np.zeros(0)
    return VoxelIndex(float(voxel_size), origin, key[first], np.stack([first, last], 1).astype(np.int64),
                      perm, vmax)


def frustum_planes(camera) -> np.ndarray:
    """Six planes (n, d) with n.x + d >= 0 inside: near, far and the four
    sides through the image corners (the reference's operations)."""
    rot, eye = camera.r_wc, camera.center
    look = rot[2]
    near = np.concatenate([look, [-(look @ eye) - camera.near]])
    far = np.concatenate([-look, [(look @ eye) + camera.far]])
    corner_px = ((0.0, 0.0), (camera.width, 0.0), (camera.width, camera.height),
                 (0.0, camera.height))
    rays = [rot.T @ np.array([(u - camera.cx) / camera.fx, (v - camera.cy) / camera.fy, 1.0])
            for u, v in corner_px]
    sides = []
    for a, b in zip(rays, rays[1:] + rays[:1]):
        nrm = np.cross(a, b)
        nrm /= np.linalg.norm(nrm)
        nrm = -nrm if nrm @ look < 0 else nrm
        sides.append(np.concatenate([nrm, [-(nrm @ eye)]]))
    return np.stack([near, far] + sides)


def frustum_visible_voxels(index: VoxelIndex, camera, margin_sigma: float = 3.0) -> list:
    """Voxels not culled by the frustum: a voxel is culled when all 8 corners
    of its box, inflated by margin_sigma x its largest scale + 5 % of the
    voxel size, lie outside one plane.  Vectorised over voxels."""
    if index.n_voxels == 0:
        return []
    pad = (margin_sigma * index.voxel_max_scale + 0.05 * index.voxel_size)[:, None]
    lo = index.origin + index.voxel_keys * index.voxel_size - pad
    hi = index.origin + (index.voxel_keys + 1) * index.voxel_size + pad
    ext = (lo, hi)
    corners = np.stack([np.stack([ext[i][:, 0], ext[j][:, 1], ext[k][:, 2]], axis=-1)
                        for i in (0, 1) for j in (0, 1) for k in (0, 1)], axis=1)  # (V, 8, 3)
    culled = np.zeros(index.n_voxels, dtype=bool)
    for pl in frustum_planes(camera):
        side = corners[..., 0] * pl[0] + corners[..., 1] * pl[1] + corners[..., 2] * pl[2] + pl[3]
        culled |= (side < 0).all(axis=1)
    return np.flatnonzero(~culled).tolist()


# ---------------------------------------------------------------------------
# host tier and paged device tier


def row_bytes(sh_coeffs: int) -> int:
    """Device bytes of one Gaussian's parameters here (f32 SoA)."""
    return 4 * (11 + 3 * sh_coeffs)


def ref_row_bytes(sh_coeffs: int) -> int:
    """Bytes the reference accounts per Gaussian in a ParamGroup: its fp64
    parameters plus the int64 row id (memory_tiers.py:33-38).  Budgets and
    FrameStats use this unit so eviction, prefetch and stall decisions are the
    reference's for the same budget_bytes; the pool itself holds f32 rows and
    an int64 prim key (row_bytes + 8 per row)."""
    return 8 * (12 + 3 * sh_coeffs)


class HostTier:
    """The whole model in pinned host memory, rows regrouped so every group is
    a contiguous range; ``keys`` is the per-row depth-tie key."""

    def __init__(self, g, order: np.ndarray, keys: np.ndarray, groups: dict):
        order = np.asarray(order, dtype=np.int64)
        pinned = torch.cuda.is_available()

        def pin(a, dtype=torch.float32):
            t = torch.as_tensor(np.ascontiguousarray(np.asarray(a)[order])).to(dtype)
            return t.pin_memory() if pinned else t

        self.means, self.quats, self.scales = pin(g.means), pin(g.quats), pin(g.scales)
        self.logits, self.sh = pin(g.opacity_logits), pin(g.sh)
        self.keys = torch.as_tensor(np.asarray(keys, dtype=np.int64))
        if pinned:
            self.keys = self.keys.pin_memory()
        self.sh_degree = int(g.sh_degree)
        self.sh_coeffs = int(self.sh.shape[1])
        self.groups = groups  # gid -> (start, end) rows of this tier
        unit = ref_row_bytes(self.sh_coeffs)
        self.group_bytes = {gid: unit * (se[1] - se[0]) for gid, se in groups.items()}

    @property
    def count(self) -> int:
        return int(self.means.shape[0])


class DevicePool:
    """Paged device SoA: ``n_pages`` pages of 128 rows (one K1 CTA each)."""

    def __init__(self, n_pages: int, sh_coeffs: int, sh_degree: int, device=None):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else \
            torch.device(device)
        self.n_pages = max(1, n_pages)
        cap = self.n_pages * PAGE_ROWS
        z = lambda *s: torch.zeros(s, dtype=torch.float32, device=dev)  # noqa: E731
        quats = z(cap, 4)
        quats[:, 0] = 1.0
        self.model = GaussianModel(z(cap, 3), quats, torch.ones(cap, 3, device=dev), z(cap),
                                   z(cap, sh_coeffs, 3), sh_degree, device=dev, validate=False)
        self.keys = torch.zeros(cap, dtype=torch.int64, device=dev)
        self.mask = torch.zeros(self.n_pages, dtype=torch.uint8, device=dev)
        self.free = list(range(self.n_pages))  # a heap: lowest free page first
        self.device = dev

    def alloc(self, rows: int) -> list:
        need = -(-rows // PAGE_ROWS)
        if need > len(self.free):
            raise BudgetExceededError(f"pool out of pages ({need} > {len(self.free)} free)")
        return [heapq.heappop(self.free) for _ in range(need)]

    def release(self, pages) -> None:
        for p in pages:
            heapq.heappush(self.free, p)

    def _pairs(self, host):
        m = self.model
        return ((m.means, host.means), (m.quats, host.quats), (m.scales, host.scales),
                (m.opacity_logits, host.logits), (m.sh, host.sh))

    def copy_in(self, host: HostTier, start: int, end: int, pages: list) -> None:
        """Enqueue the H2D copies of host rows [start, end) into ``pages`` on
        the current stream (runs of consecutive pages become one copy)."""
        pairs = self._pairs(host) + ((self.keys, host.keys),)
        i, r = 0, start
        while r < end:
            j = i
            while j + 1 < len(pages) and pages[j + 1] == pages[j] + 1:
                j += 1
            n = min(end - r, (j - i + 1) * PAGE_ROWS)
            d0 = pages[i] * PAGE_ROWS
            for dst, src in pairs:
                dst[d0:d0 + n].copy_(src[r:r + n], non_blocking=True)
            r += n
            i = j + 1

    def copy_out(self, host: HostTier, start: int, end: int, pages: list) -> None:
        r = start
        for p in pages:
            n = min(end - r, PAGE_ROWS)
            for dev_t, host_t in self._pairs(host):
                host_t[r:r + n].copy_(dev_t[p * PAGE_ROWS:p * PAGE_ROWS + n])
            r += n

    def set_mask(self, runs) -> torch.Tensor:
        """Per-page live-row counts of a frame: ``runs`` = [(pages, rows)] of the
        groups it renders (stream-ordered device update)."""
        self.mask.zero_()
        idx = [p for pages, _ in runs for p in pages]
        cnt = [min(PAGE_ROWS, rows - k * PAGE_ROWS) for pages, rows in runs
               for k in range(len(pages))]
        if idx:
            t = torch.tensor([idx, cnt], dtype=torch.long).to(self.device)
            self.mask.index_copy_(0, t[0], t[1].to(torch.uint8))
        return self.mask


class TierStore:
    """The device tier: all-or-nothing group loads against the byte budget
    (the reference's accounting unit and simulated completion times, so its
    decisions and stats are the reference's), with the real rows copied
    asynchronously into the paged pool on ``copy_stream``."""

    def __init__(self, budget_bytes: int, host: HostTier, transfer=None,
                 clock: VirtualClock | None = None, device=None):
        self.budget_bytes = int(budget_bytes)
        self.transfer = TransferConfig() if transfer is None else transfer
        self.clock = VirtualClock() if clock is None else clock
        self.host = host
        self.device: dict = {}  # gid -> pages (insertion order = residency order)
        self.events: dict = {}  # gid -> cuda event of its copies
        self.resident_bytes = 0
        self.stats = TierStats()
        # pages for the budget's rows plus one partial page per group
        budget_pages = self.budget_bytes // ref_row_bytes(host.sh_coeffs) // PAGE_ROWS
        all_pages = sum(-(-(e - s) // PAGE_ROWS) for s, e in host.groups.values())
        self.pool = DevicePool(min(all_pages, budget_pages + len(host.groups) + 1),
                               host.sh_coeffs, host.sh_degree, device)
        self.copy_stream = torch.cuda.Stream(device=self.pool.device)
        self.render_done: torch.cuda.Event | None = None

    def host_bytes(self, gid) -> int:
        return self.host.group_bytes[gid]

    def is_resident(self, gid) -> bool:
        return gid in self.device

    def load_cells(self, gids) -> LoadHandle:
        """Make ``gids`` resident (already resident ones cost nothing); the
        handle completes on the simulated clock after the link time of the
        new bytes, and its event when the real copies land."""
        gids = tuple(gids)
        unknown = [g for g in gids if g not in self.host.groups]
        if unknown:
            raise NotResidentError(f"cell {unknown[0]} not in host tier")
        fresh = [g for g in gids if g not in self.device]
        add = sum(map(self.host.group_bytes.__getitem__, fresh))
        if add + self.resident_bytes > self.budget_bytes:
            raise BudgetExceededError(f"loading {add} bytes would exceed budget "
                                      f"({self.resident_bytes}/{self.budget_bytes} resident)")
        ev = None
        if fresh:
            with torch.cuda.stream(self.copy_stream):
                if self.render_done is not None:  # pages may be reused from evicted groups
                    self.copy_stream.wait_event(self.render_done)
                for g in fresh:
                    s, e = self.host.groups[g]
                    self.device[g] = self.pool.alloc(e - s)
                    self.pool.copy_in(self.host, s, e, self.device[g])
                ev = torch.cuda.Event()
                ev.record(self.copy_stream)
            self.events.update(dict.fromkeys(fresh, ev))
        st = self.stats
        self.resident_bytes += add
        st.loads, st.bytes_in = st.loads + len(fresh), st.bytes_in + add
        st.peak_resident_bytes = max(st.peak_resident_bytes, self.resident_bytes)
        return LoadHandle(gids, self.clock.now + self.transfer.seconds(add), add, ev)

    def offload_cells(self, gids, write_back: bool = False) -> int:
        """Release ``gids``' pages (optionally copying the rows back first);
        returns the bytes freed."""
        gids = tuple(gids)
        absent = [g for g in gids if g not in self.device]
        if absent:
            raise NotResidentError(f"cell {absent[0]} not resident on device")
        if write_back:
            torch.cuda.current_stream().wait_stream(self.copy_stream)
        for g in gids:
            pages = self.device.pop(g)
            self.events.pop(g, None)
            if write_back:
                self.pool.copy_out(self.host, *self.host.groups[g], pages)
            self.pool.release(pages)
        out = sum(self.host.group_bytes[g] for g in gids)
        self.resident_bytes -= out
        self.stats.offloads += len(gids)
        self.stats.bytes_out += out
        return out

    def render_groups(self, camera, gids, cfg) -> torch.Tensor:
        """Render the union of resident groups straight from the pool: the
        render stream waits (on the device) for their copies."""
        cur = torch.cuda.current_stream(self.pool.device)
        waited = set()
        runs = []
        for g in gids:
            if g not in self.device:
                raise NotResidentError(f"cell {g} not resident on device")
            ev = self.events.get(g)
            if ev is not None and id(ev) not in waited:
                cur.wait_event(ev)
                waited.add(id(ev))
            s, e = self.host.groups[g]
            runs.append((self.device[g], e - s))
        out = render(camera, self.pool.model, cfg.tile_size, cfg.background, cfg.sh_eval_degree,
                     prim_ids=self.pool.keys, page_mask=self.pool.set_mask(runs),
                     page_shift=PAGE_SHIFT)
        self.render_done = torch.cuda.Event()
        self.render_done.record(cur)
        return out.rgb


# ---------------------------------------------------------------------------
# block streaming: a front region (rendered) and a back region (loading
# ahead of a cell crossing), switched by nested trigger zones around the
# core cell (the decisions of memory_tiers.py:150-247)


Region = _record("Region", [("cell_ids", frozenset), ("core", "tuple | None", field(default=None))],
                 "A set of cells and the core cell it was built around.")


def _swap_in(self, clock: VirtualClock) -> None:
    if not self.back:
        raise IncompleteLoadError("swap with an empty back buffer (no back buffer to swap in)")
    region, handle = self.back
    if not handle.ready(clock):
        raise IncompleteLoadError(f"back buffer load completes at t={handle.ready_at:.6f}, "
                                  f"now t={clock.now:.6f}")
    self.front, self.back = region, None


BufferPair = _record(
    "BufferPair", [("front", "Region | None", field(default=None)),
                   ("back", "tuple | None", field(default=None))],
    "front: the region being rendered; back: (region, LoadHandle) in flight.", swap=_swap_in)


def _check_zones(self) -> None:
    if not 0 < self.inner_fraction < self.outer_fraction <= 1:
        raise InvalidConfigError("trigger zones need 0 < inner < outer <= 1")


TriggerZones = _record(
    "TriggerZones", [("inner_fraction", float, field(default=0.5)),
                     ("outer_fraction", float, field(default=0.8))],
    "Fractions of the core cell's half-extent: past inner a load of the next cell's "
    "region starts, past outer the buffers swap.", frozen=True, __post_init__=_check_zones)

# kind: none | start_load | swap | stall_then_swap
PrefetchAction = _record("PrefetchAction", [("kind", str),
                                            ("target_core", "tuple | None", field(default=None))],
                         "One frame's block-streaming decision.", frozen=True)
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


def prefetch_policy(position, velocity, core_cell, zones, pair, grid, clock) -> PrefetchAction:
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


def _check_session(self) -> None:
    if self.mode not in RENDER_MODES:
        raise InvalidConfigError(f"unknown session mode {self.mode!r}; one of {RENDER_MODES}")
    if self.mode != RENDER_MODES[0] and self.budget_bytes is None:
        raise InvalidConfigError(f"session mode {self.mode!r} needs a budget_bytes")


SessionConfig = _record(
    "SessionConfig",
    [("mode", str, field(default=RENDER_MODES[0])),
     ("budget_bytes", "int | None", field(default=None)),
     ("ring", int, field(default=1)),
     ("tile_size", int, field(default=16)),
     ("zones", "TriggerZones", field(default_factory=TriggerZones)),
     ("transfer", "TransferConfig", field(default_factory=TransferConfig)),
     ("voxel_size", float, field(default=1.0)),
     ("background", tuple, field(default=(0.0, 0.0, 0.0))),
     ("sh_eval_degree", int, field(default=1))],
    "Streaming mode, byte budget (the reference's unit, ref_row_bytes), onload ring, "
    "trigger zones, transfer link, voxel size and render settings (sh_eval_degree 1 = "
    "the reference's colours).", __post_init__=_check_session)


def _stats_dict(self) -> dict:
    d = asdict(self)
    if self.core_cell is not None:
        d["core_cell"] = list(self.core_cell)
    return d


FrameStats = _record(
    "FrameStats",
    [("index", int), ("t", float), ("latency_ms", float), ("resident_bytes", int),
     ("peak_resident_bytes", int), ("stalls", int),
     ("core_cell", "tuple | None", field(default=None)),
     ("n_primitives", int, field(default=0))],
    "One rendered frame of a session (the reference's fields).", as_dict=_stats_dict)


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

    def __init__(self, cfg, clock):
        self.cfg = cfg
        self.clock = VirtualClock() if clock is None else clock
        self.n_stalls = 0

    @property
    def stalls(self) -> int:
        return self.n_stalls

    def _stall(self, ready_at: float) -> None:
        self.n_stalls, self.store.stats.stalls = self.n_stalls + 1, self.store.stats.stalls + 1
        self.clock.wait_until(ready_at)

    def _draw(self, camera, groups) -> tuple:
        rows = sum(e - s for s, e in (self.store.host.groups[g] for g in groups))
        return self.store.render_groups(camera, groups, self.cfg), int(rows)

    def frame_state(self) -> tuple:
        """(core cell, resident bytes, peak resident bytes, stalls)."""
        return (None, self.store.resident_bytes, self.store.stats.peak_resident_bytes,
                self.n_stalls)


class BlockSession(_PoolSession):
    """Cell-grid streaming: the front buffer holds the ring region of the
    camera's core cell; the next region is loaded ahead of a crossing."""

    def __init__(self, model, grid: SceneGrid, cfg, clock: VirtualClock | None = None,
                 device=None):
        super().__init__(cfg, clock)
        self.grid = grid
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
                f"{cfg.budget_bytes} budget bytes cannot double-buffer the largest onload "
                f"region: needs 2 x {need} bytes")
        self.store = TierStore(cfg.budget_bytes, host, cfg.transfer, self.clock, device)
        self.pair = BufferPair()

    def _request(self, core) -> tuple:
        cells = frozenset(self.grid.region(core, self.cfg.ring))
        return Region(cells, core), self.store.load_cells(sorted(cells))

    def _evict_unused(self) -> None:
        live = set(self.pair.front.cell_ids if self.pair.front else ())
        live |= self.pair.back[0].cell_ids if self.pair.back else set()
        unused = [c for c in list(self.store.device) if c not in live]
        if unused:
            self.store.offload_cells(unused, write_back=False)

    def step(self, camera, velocity) -> tuple:
        here = self.grid.cell_of_point(camera.center)
        pair = self.pair
        if pair.front is None:  # first frame: load and wait
            region, handle = self._request(here)
            self.clock.wait_until(handle.ready_at)
            pair.front = region
        act = prefetch_policy(camera.center, velocity, pair.front.core, self.cfg.zones, pair,
                              self.grid, self.clock)
        if act.kind == "start_load":
            pair.back = self._request(act.target_core)
        elif act.kind in ("swap", "stall_then_swap"):
            if act.kind == "stall_then_swap":
                self._stall(pair.back[1].ready_at)
            pair.swap(self.clock)
            self._evict_unused()
        if here not in pair.front.cell_ids:  # outran the prefetch: load in place
            region, handle = self._request(here)
            self._stall(handle.ready_at)
            pair.front, pair.back = region, None
            self._evict_unused()
        return self._draw(camera, sorted(pair.front.cell_ids))

    def frame_state(self) -> tuple:
        return (self.pair.front.core,) + super().frame_state()[1:]


class FrustumSession(_PoolSession):
    """Voxel streaming: each frame draws the frustum-visible voxels; the
    least recently visible voxels are evicted to stay within the budget."""

    def __init__(self, model, cfg, clock: VirtualClock | None = None, device=None):
        super().__init__(cfg, clock)
        arrs = _host_arrays(model)
        self.index = reorder_voxel_grid(arrs[0], arrs[2], cfg.voxel_size)
        perm = self.index.permutation
        groups = dict(enumerate(map(tuple, self.index.ranges.tolist())))
        # prim key = row of the voxel-reordered model (render_image's subset ids)
        host = HostTier(_HostModel(arrs), perm, np.arange(len(perm), dtype=np.int64), groups)
        self.store = TierStore(cfg.budget_bytes, host, cfg.transfer, self.clock, device)
        self.last_visible: dict = {}
        self.frames_drawn = 0

    def _make_room(self, visible) -> None:
        st = self.store
        vis = set(visible)
        missing = sum(st.host_bytes(v) for v in visible if not st.is_resident(v))
        if st.resident_bytes + missing <= st.budget_bytes:
            return
        # stable: equally old voxels leave in residency (insertion) order
        victims = sorted((v for v in st.device if v not in vis),
                         key=lambda v: self.last_visible.get(v, -1))
        for v in victims:
            if st.resident_bytes + missing <= st.budget_bytes:
                break
            st.offload_cells([v], write_back=False)

    def step(self, camera) -> tuple:
        self.frames_drawn += 1
        visible = frustum_visible_voxels(self.index, camera)
        self._make_room(visible)
        handle = self.store.load_cells(visible)
        if handle.ready_at > self.clock.now:
            self._stall(handle.ready_at)
        self.last_visible.update(dict.fromkeys(visible, self.frames_drawn))
        return self._draw(camera, visible)


class _StaticSession:
    """The whole model resident on the device (the reference's fp64 bytes)."""

    def __init__(self, model, cfg, device=None):
        self.cfg = cfg
        self.model = model if isinstance(model, GaussianModel) else \
            GaussianModel.from_host(_HostModel(_host_arrays(model)), device=device)
        self.nbytes = self.model.count * (ref_row_bytes(int(self.model.sh.shape[1])) - 8)
        self.ctx = context(self.model.device.index)

    def step(self, camera, velocity=None) -> tuple:
        c = self.cfg
        img = render(camera, self.model, c.tile_size, c.background, c.sh_eval_degree,
                     ctx=self.ctx).rgb
        return img, self.model.count

    def frame_state(self) -> tuple:
        return None, self.nbytes, self.nbytes, 0


_SESSIONS = {"static_full": lambda m, cfg, grid, clock, dev: _StaticSession(m, cfg, dev),
             "frustum_voxel": lambda m, cfg, grid, clock, dev: FrustumSession(m, cfg, clock, dev)}


def _block(m, cfg, grid, clock, dev):
    if grid is None:
        raise InvalidInputError("a block_double_buffer session needs the scene grid")
    return BlockSession(m, grid, cfg, clock, dev)


_SESSIONS["block_double_buffer"] = _block


def run_session(model, cameras, timestamps, cfg, grid: SceneGrid | None = None,
                clock: VirtualClock | None = None, keep_images: bool = True, device=None):
    """Render a camera trajectory in ``cfg.mode``: (images, [FrameStats]).
    The simulated clock follows the timestamps; a frame's latency is wall
    time with its GPU work completed (synchronised)."""
    if len(cameras) != len(timestamps):
        raise InvalidInputError(f"{len(cameras)} cameras but {len(timestamps)} timestamps")
    clock = VirtualClock() if clock is None else clock
    sess = _SESSIONS[cfg.mode](model, cfg, grid, clock, device)
    frames, out = [], []
    prev = None  # (position, time) of the previous frame
    for idx, t in enumerate(timestamps):
        cam = cameras[idx]
        cam = cam if isinstance(cam, Camera) else Camera.from_reference(cam)
        vel = np.zeros(3)
        if prev is not None:
            dt = t - prev[1]
            if dt > 0:
                clock.advance(dt)
            vel = (cam.center - prev[0]) / (dt if dt > 0 else 1.0)
        t0 = time.perf_counter()
        image, n = sess.step(cam) if isinstance(sess, FrustumSession) else sess.step(cam, vel)
        torch.cuda.current_stream().synchronize()
        core, resident, peak, stalls = sess.frame_state()
        out.append(FrameStats(idx, float(t), 1e3 * (time.perf_counter() - t0), resident, peak,
                              stalls, core, n))
        if keep_images:
            frames.append(image)
        prev = (cam.center, t)
    return frames, out


def bench(model, cameras, timestamps, cfg, grid: SceneGrid | None = None) -> dict:
    """Session summary: frame count, latency mean / median, frames/s, peak
    residency and stalls."""
    frames = run_session(model, cameras, timestamps, cfg, grid=grid, keep_images=False)[1]
    ms = [f.latency_ms for f in frames]
    wall = sum(ms) / 1e3
    summary = dict(frames=len(frames), mean_latency_ms=0.0, median_latency_ms=0.0, fps=0.0,
                   peak_resident_bytes=0, stalls=0)
    if frames:
        summary.update(mean_latency_ms=statistics.fmean(ms), median_latency_ms=statistics.median(ms),
                       fps=len(frames) / wall if wall > 0 else 0.0,
                       peak_resident_bytes=max(f.peak_resident_bytes for f in frames),
                       stalls=frames[-1].stalls)
    return summary
