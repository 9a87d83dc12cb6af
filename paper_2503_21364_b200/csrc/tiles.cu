// Tile instance lists: K2b depth-order fix-up, K4 emission, K6 tile ranges,
// instance export.
//
// Reference: rasterize (gaussian_core.py:340-403) builds, for every tile, the
// list of splats whose bbox overlaps it (367-373) in _sort_order's
// (depth, prim_id) order (277-283, 392).
//
// B200 design — sort each splat once, not each (splat, tile) pair:
//   K2   one device-wide radix sort of 32-bit depth keys of all N splats
//        (K2a quantises the fp64 depth over the view's depth range; sort.cu,
//        stable, payload = id), then K2b fixes the order inside runs of equal
//        keys by the exact fp64 depth: the result is the global rank order
//        (depth, id) of the visible splats;
//   K4   walks the splats in rank order, scans their tile counts (one pass,
//        decoupled look-back) and emits one 8-byte key tile << 32 | id per
//        overlapped tile, so the instance array comes out already ordered by
//        depth rank; it also builds the tile-digit histograms of K5;
//   K5   a stable LSD radix sort of those keys on the tile bits only (sort.cu,
//        2 passes of 8 bits at 1080p) — every tile's list is then exactly the
//        reference's per-tile (depth, id) order, with no per-tile sort;
//   K6   tile ranges [start, end): the last K5 pass adds each CTA's per-tile
//        run lengths to a tile-count array, and one CTA scans it.
#include "device_util.cuh"
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

__device__ __forceinline__ void unpack_rect(uint64_t rect, int& x0, int& y0, int& x1, int& y1) {
  x0 = (int)(rect & 0xffff);
  y0 = (int)((rect >> 16) & 0xffff);
  x1 = (int)((rect >> 32) & 0xffff);
  y1 = (int)((rect >> 48) & 0xffff);
}

// ---------------------------------------------------------------------------
// K2a: 24-bit depth keys.  key = trunc((z - zmin) * (2^24 - 2) / (zmax - zmin))
// is monotone non-decreasing in z (each rounded fp64 step is), so sorting by
// it and then by the exact fp64 depth inside equal-key runs gives _sort_order's
// (depth, id) order.  24 bits = 3 radix passes; over the view's own depth
// range the runs it leaves are short (c3: 39% of splats in runs, longest 7),
// and the fix-up sorts them.  Invisible splats get kDepthKeyNone.

#ifndef LMGS_DEPTH_KEYS_U
#define LMGS_DEPTH_KEYS_U 4
#endif
#ifndef LMGS_DEPTH_KEYS_CTAS_PER_SM
#define LMGS_DEPTH_KEYS_CTAS_PER_SM 8
#endif
__global__ void __launch_bounds__(256) k_depth_keys(const uint64_t* __restrict__ key64,
                                                    const unsigned long long* zrange, int64_t n,
                                                    uint32_t* __restrict__ key32,
                                                    uint32_t* hist) {
  __shared__ uint32_t s_hist[kDepthPasses][256];
  for (int i = threadIdx.x; i < kDepthPasses * 256; i += blockDim.x) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  const double zmin = __longlong_as_double((long long)zrange[0]);
  const double zmax = __longlong_as_double((long long)zrange[1]);
  const double span = zmax - zmin;
  const double top = (double)(kDepthKeyNone - 1);
  const double scale = span > 0.0 ? top / span : 0.0;
  // LMGS_DEPTH_KEYS_U keys per thread per step (independent loads in flight)
  constexpr int U = LMGS_DEPTH_KEYS_U;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x) * U + threadIdx.x; i0 < n; i0 += stride) {
    uint64_t kb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + (int64_t)u * blockDim.x;
      kb[u] = i < n ? key64[i] : kCulledKey;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + (int64_t)u * blockDim.x;
      if (i >= n) break;
      uint32_t k = kDepthKeyNone;
      if (kb[u] != kCulledKey) {
        const double q = (__longlong_as_double((long long)kb[u]) - zmin) * scale;
        k = q >= top ? kDepthKeyNone - 1 : (uint32_t)q;
      }
      key32[i] = k;
#pragma unroll
      for (int d = 0; d < kDepthPasses; ++d) atomicAdd(&s_hist[d][(k >> (8 * d)) & 0xffu], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kDepthPasses * 256; i += blockDim.x) {
    const uint32_t v = (&s_hist[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

// ---------------------------------------------------------------------------
// K2b: exact fix-up of a run of equal keys: order by (fp64 depth bits, prim
// id).  The radix sort is stable and its payload is the input index, so a run
// is already in row order — the prim-id order unless a paged set maps rows to
// ids out of order; an in-place insertion sort is linear on the common run
// (exact duplicates) and runs are short.

__device__ __forceinline__ bool less64(uint64_t ka, int64_t ia, uint64_t kb, int64_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__device__ void fix_run(uint32_t* ids, int len, const uint64_t* __restrict__ key64,
                        const int64_t* __restrict__ pid) {
  for (int a = 1; a < len; ++a) {
    const uint32_t ki = ids[a];
    const uint64_t kd = key64[ki];
    const int64_t pi = pid ? pid[ki] : (int64_t)ki;
    int b = a - 1;
    while (b >= 0) {
      const uint32_t ib = ids[b];
      if (!less64(kd, pi, key64[ib], pid ? pid[ib] : (int64_t)ib)) break;
      ids[b + 1] = ib;
      --b;
    }
    ids[b + 1] = ki;
  }
}

// one thread per 4 consecutive keys: runs start where a key differs from
// its predecessor and continues into its successor
#ifndef LMGS_FIXUP_PER
#define LMGS_FIXUP_PER 4
#endif
constexpr int kFixupPer = LMGS_FIXUP_PER;
__global__ void k_depth_fixup(void* const* keys_slot, void* const* ids_slot, int64_t n,
                              const uint64_t* __restrict__ key64,
                              const int64_t* __restrict__ pid) {
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kFixupPer;
  if (i0 >= n) return;
  const uint32_t* __restrict__ keys = static_cast<const uint32_t*>(*keys_slot);
  uint32_t k[kFixupPer + 2];  // keys[i0 - 1 .. i0 + kFixupPer]
#pragma unroll
  for (int u = 0; u < kFixupPer + 2; ++u) {
    const int64_t i = i0 - 1 + u;
    k[u] = (i >= 0 && i < n) ? keys[i] : kDepthKeyNone + 1 + u;  // sentinels never equal
  }
#pragma unroll
  for (int u = 1; u <= kFixupPer; ++u) {
    const int64_t i = i0 - 1 + u;
    if (i >= n || k[u] == kDepthKeyNone) break;  // invisible tail
    if (k[u - 1] == k[u] || k[u + 1] != k[u]) continue;  // not the head of a run
    // keys[i + 2] is often already in registers; most runs have length 2
    int64_t len = 2;
    if (u + 2 <= kFixupPer + 1 && k[u + 2] != k[u]) {
      uint32_t* run = static_cast<uint32_t*>(*ids_slot) + i;
      const uint32_t a0 = run[0], a1 = run[1];  // independent loads
      const uint64_t d0 = key64[a0], d1 = key64[a1];
      const int64_t p0 = pid ? pid[a0] : (int64_t)a0, p1 = pid ? pid[a1] : (int64_t)a1;
      if (less64(d1, p1, d0, p0)) {
        run[0] = a1;
        run[1] = a0;
      }
      continue;
    }
    while (i + len < n && keys[i + len] == k[u]) ++len;
    fix_run(static_cast<uint32_t*>(*ids_slot) + i, (int)len, key64, pid);
  }
}

// ---------------------------------------------------------------------------
// K4: rank-ordered emission with a single-pass scan (decoupled look-back)
//
// A CTA takes the next chunk of kEmitChunk ranks (ticket order).  Warp w owns
// 256 consecutive ranks; it scans their tile counts in rank order, the CTA
// learns the chunk's global offset by look-back, and then every warp writes
// its instances with consecutive lanes on consecutive output slots (a 32-slot
// window maps slots to splats with one OR-reduction and a few shuffles).

constexpr uint64_t kLbAgg = 1ull << 62;
constexpr uint64_t kLbIncl = 2ull << 62;
constexpr uint64_t kLbMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kEmitThreads) k_emit(EmitArgs a) {
  constexpr int NW = kEmitThreads / 32;
  constexpr int PW = 32 * kEmitItems;  // ranks per warp
  __shared__ uint32_t s_end[NW][PW];   // running (inclusive) tile count within the warp
  __shared__ uint32_t s_id[NW][PW];
  __shared__ uint64_t s_rect[NW][PW];
  __shared__ uint32_t s_hist[kMaxTilePasses][256];
  __shared__ uint32_t s_wtot[NW];
  __shared__ uint32_t s_ticket;
  __shared__ unsigned long long s_excl;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kMaxTilePasses * 256; i += kEmitThreads) (&s_hist[0][0])[i] = 0;
  const int64_t n_vis = min(a.n_vis, (int64_t)*a.n_vis_dev);  // the grid covers a bound
  // chunks by ticket; a persistent grid (concurrent streams) loops over them
  for (;;) {
  if (tid == 0) s_ticket = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const int64_t chunk = s_ticket;
  if (chunk * kEmitChunk >= n_vis) break;
  const int64_t base = chunk * kEmitChunk + (int64_t)warp * PW;
  const uint32_t* __restrict__ order = static_cast<const uint32_t*>(*a.order_slot);

  // blocked layout: lane l owns ranks base + l*kEmitItems + j (item index
  // l*kEmitItems + j within the warp), so the warp's scan is one shuffle scan
  // of per-lane sums
  uint32_t id[kEmitItems];
#pragma unroll
  for (int j = 0; j < kEmitItems; ++j) {
    const int64_t r = base + lane * kEmitItems + j;
    id[j] = r < n_vis ? order[r] : 0xffffffffu;
  }
  uint64_t rect[kEmitItems];
#pragma unroll
  for (int j = 0; j < kEmitItems; ++j) rect[j] = id[j] != 0xffffffffu ? __ldg(a.rects + id[j]) : 0ull;
  uint32_t incl_local[kEmitItems];
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < kEmitItems; ++j) {
    int x0, y0, x1, y1;
    unpack_rect(rect[j], x0, y0, x1, y1);
    sum += id[j] != 0xffffffffu ? (uint32_t)(x1 - x0 + 1) * (uint32_t)(y1 - y0 + 1) : 0u;
    incl_local[j] = sum;
  }
  uint32_t scan = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, scan, o);
    if (lane >= o) scan += v;
  }
  const uint32_t lane_excl = scan - sum;
  const uint32_t run = __shfl_sync(0xffffffffu, scan, 31);
#pragma unroll
  for (int j = 0; j < kEmitItems; ++j) {
    const int k = lane * kEmitItems + j;
    s_end[warp][k] = lane_excl + incl_local[j];
    s_id[warp][k] = id[j];
    s_rect[warp][k] = rect[j];
  }
  if (lane == 0) s_wtot[warp] = run;
  __syncthreads();
  uint64_t wofs = 0, total = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t v = s_wtot[w];
    wofs += w < warp ? v : 0;
    total += v;
  }
  if (warp == 0) {
    // warp-cooperative look-back: 32 predecessors per L2 round trip
    uint64_t* lb = a.lookback;
    if (chunk == 0) {
      if (lane == 0) {
        st_relaxed_gpu(lb, kLbIncl | total);
        s_excl = 0;
      }
    } else {
      if (lane == 0) st_relaxed_gpu(lb + chunk, kLbAgg | total);
      uint64_t excl = 0;
      int64_t end = chunk;  // predecessors [end - 32, end) in this window
      while (true) {
        const int64_t idx = end - 1 - lane;
        uint64_t v = kLbIncl;  // before chunk 0: inclusive zero (never reached)
        if (idx >= 0) {
          do {
            v = ld_relaxed_gpu(lb + idx);
          } while ((v & ~kLbMask) == 0);
        }
        const uint32_t incl = __ballot_sync(0xffffffffu, (v & ~kLbMask) == kLbIncl);
        const int stop = incl ? __ffs(incl) - 1 : 31;  // nearest inclusive predecessor
        unsigned long long part = lane <= stop ? (v & kLbMask) : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        excl += part;
        if (incl) break;
        end -= 32;
      }
      if (lane == 0) {
        st_relaxed_gpu(lb + chunk, kLbIncl | (excl + total));
        s_excl = excl;
      }
    }
  }
  __syncthreads();
  const uint64_t out0 = s_excl + wofs;
  const uint32_t wtot = s_wtot[warp];
  const uint32_t* ends = s_end[warp];  // item k covers slots [ends[k-1], ends[k])
  const int passes = a.n_tile_passes;
  // Slots are written 32 at a time, lane l -> slot p0 + l.  k0 is the item
  // holding slot p0; lane j looks at item k0 + j, items starting inside the
  // window mark their offset in a 32-bit mask, and slot l's item is k0 plus
  // the number of marks at offsets <= l.
  __syncwarp();
  int k0 = 0;
  for (uint32_t p0 = 0; p0 < wtot; p0 += 32) {  // warp-uniform trip count
    const int kj = k0 + lane;
    const bool have = kj < PW;
    const uint32_t st = have ? (kj ? ends[kj - 1] : 0u) : 0xffffffffu;
    const bool mark = lane > 0 && st < p0 + 32u;
    const uint32_t smask = __reduce_or_sync(0xffffffffu, mark ? 1u << (st - p0) : 0u);
    const int idx = __popc(smask & (0xffffffffu >> (31 - lane)));
    const uint64_t my_rect = have ? s_rect[warp][kj] : 0ull;
    const uint32_t my_id = have ? s_id[warp][kj] : 0u;
    const uint32_t st_i = __shfl_sync(0xffffffffu, st, idx);
    const uint32_t r_lo = __shfl_sync(0xffffffffu, (uint32_t)my_rect, idx);
    const uint32_t r_hi = __shfl_sync(0xffffffffu, (uint32_t)(my_rect >> 32), idx);
    const uint32_t id_i = __shfl_sync(0xffffffffu, my_id, idx);
    const uint32_t p = p0 + lane;
    // instances past the capacity are dropped and not counted (no-sync overflow)
    const bool on = p < wtot && out0 + p < a.cap;
    uint32_t tile = 0;
    if (on) {
      const uint32_t q = p - st_i;
      const int x0 = (int)(r_lo & 0xffff), y0 = (int)(r_lo >> 16), x1 = (int)(r_hi & 0xffff);
      const uint32_t w = (uint32_t)(x1 - x0 + 1);
      // q / w without the integer-division sequence: q < 2^24, w < 2^16, so
      // the float quotient is within one of the truth; fix it up exactly
      uint32_t dy = (uint32_t)__fdividef((float)q, (float)w);
      if (dy * w > q) --dy;
      else if ((dy + 1) * w <= q) ++dy;
      tile = (uint32_t)(y0 + (int)dy) * (uint32_t)a.tiles_x + (uint32_t)x0 + (q - dy * w);
      a.keys[out0 + p] = ((uint64_t)tile << 32) | id_i;
      // the low digit differs across lanes (consecutive tiles of a row)
      atomicAdd(&s_hist[0][tile & 0xffu], 1u);
    }
    // higher digits are almost always warp-uniform: one aggregated add
    const uint32_t act = __ballot_sync(0xffffffffu, on);
    const int first = __ffs(act) - 1;
    for (int ps = 1; ps < passes; ++ps) {
      const uint32_t dg = (tile >> (8 * ps)) & 0xffu;
      const uint32_t d0 = __shfl_sync(0xffffffffu, dg, first);
      if (__all_sync(0xffffffffu, !on || dg == d0)) {
        if (lane == first) atomicAdd(&s_hist[ps][d0], (uint32_t)__popc(act));
      } else if (on) {
        atomicAdd(&s_hist[ps][dg], 1u);
      }
    }
    // next window starts in the item holding slot p0 + 32
    const int idx31 = __shfl_sync(0xffffffffu, idx, 31);
    k0 += idx31 + (ends[k0 + idx31] == p0 + 32u ? 1 : 0);
  }
  __syncthreads();  // s_ticket, s_end, s_id, s_rect are reused by the next chunk
  }
  const int passes = a.n_tile_passes;
  for (int i = tid; i < passes * 256; i += kEmitThreads) {
    const uint32_t v = (&s_hist[0][0])[i];
    if (v) atomicAdd(a.hist + i, v);
  }
}

// ---------------------------------------------------------------------------
// K4c: tile coverage of the fused path.  The rects are streamed in id order
// (a persistent grid, one shared array per CTA) into a 2-D difference array:
// +1 at (x0, y0) and (x1+1, y1+1), -1 at (x1+1, y0) and (x0, y1+1) — four
// shared atomics per splat, 0 net for kEmptyRect.  Its 2-D prefix sum (K4p)
// is the number of splats overlapping each tile: the tile ranges and both
// digit histograms of the fused sort without touching the instances.

constexpr int kCoverThreads = 512;
__global__ void __launch_bounds__(kCoverThreads) k_cover(const uint64_t* __restrict__ rects,
                                                         int64_t n, int tiles_x, int tiles_y,
                                                         int32_t* cover_part) {
  extern __shared__ int32_t s_cover[];
  const int tid = threadIdx.x;
  const int cw = tiles_x + 1;
  const int d = cw * (tiles_y + 1);
  for (int i = tid; i < d; i += kCoverThreads) s_cover[i] = 0;
  __syncthreads();
  constexpr int U = 4;  // rects per thread per step (two 16-B loads)
  const int64_t stride = (int64_t)gridDim.x * kCoverThreads * U;
  for (int64_t i0 = ((int64_t)blockIdx.x * kCoverThreads + tid) * U; i0 < n; i0 += stride) {
    uint64_t r[U];
    if (i0 + U <= n) {
      const uint4 v0 = __ldcs(reinterpret_cast<const uint4*>(rects + i0));
      const uint4 v1 = __ldcs(reinterpret_cast<const uint4*>(rects + i0) + 1);
      r[0] = v0.x | ((uint64_t)v0.y << 32);
      r[1] = v0.z | ((uint64_t)v0.w << 32);
      r[2] = v1.x | ((uint64_t)v1.y << 32);
      r[3] = v1.z | ((uint64_t)v1.w << 32);
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) r[u] = i0 + u < n ? rects[i0 + u] : kEmptyRect;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (r[u] == kEmptyRect) continue;
      int x0, y0, x1, y1;
      unpack_rect(r[u], x0, y0, x1, y1);
      atomicAdd(&s_cover[y0 * cw + x0], 1);
      atomicAdd(&s_cover[y0 * cw + x1 + 1], -1);
      atomicAdd(&s_cover[(y1 + 1) * cw + x0], -1);
      atomicAdd(&s_cover[(y1 + 1) * cw + x1 + 1], 1);
    }
  }
  __syncthreads();
  int32_t* part = cover_part + (int64_t)blockIdx.x * d;
  for (int i = tid; i < d; i += kCoverThreads) part[i] = s_cover[i];
}

// ---------------------------------------------------------------------------
// K4r: rank scan of the fused path (see lmgs_internal.cuh), reduce-then-scan:
// k_rank_sums adds up the tile counts of every chunk of kRankChunk ranks,
// k_rank_offsets (one CTA) scans the chunk sums, k_rank_write re-gathers the
// rects (L2-resident by then) and writes per rank {rect lo, rect hi, id,
// first slot} plus the first rank of every sort tile.  No CTA waits on
// another (a chained look-back left ~half the warps parked at a barrier).
// Thread t of a chunk owns 4 consecutive ranks (one 16-B id load).

__device__ __forceinline__ void rank_chunk_load(const RankScanArgs& a, int64_t n_vis, int64_t r0,
                                                uint32_t (&id)[kRankItems],
                                                uint64_t (&rect)[kRankItems],
                                                uint32_t (&cnt)[kRankItems]) {
  const uint32_t* __restrict__ order = static_cast<const uint32_t*>(*a.order_slot);
  if (r0 + kRankItems <= n_vis) {
    const uint4 v = *reinterpret_cast<const uint4*>(order + r0);  // 16-B aligned
    id[0] = v.x, id[1] = v.y, id[2] = v.z, id[3] = v.w;
  } else {
#pragma unroll
    for (int j = 0; j < kRankItems; ++j) id[j] = r0 + j < n_vis ? order[r0 + j] : 0xffffffffu;
  }
#pragma unroll
  for (int j = 0; j < kRankItems; ++j)
    rect[j] = id[j] != 0xffffffffu ? __ldg(a.rects + id[j]) : kEmptyRect;
#pragma unroll
  for (int j = 0; j < kRankItems; ++j) {
    int x0, y0, x1, y1;
    unpack_rect(rect[j], x0, y0, x1, y1);
    cnt[j] = (uint32_t)(x1 - x0 + 1) * (uint32_t)(y1 - y0 + 1);  // 0 for kEmptyRect
  }
}

// block-wide exclusive scan of one value per thread (kRankThreads); returns
// the exclusive prefix, *total the block sum
__device__ __forceinline__ uint32_t rank_block_scan(uint32_t v, uint32_t* total) {
  constexpr int NW = kRankThreads / 32;
  __shared__ uint32_t s_w[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  uint32_t pre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t x = s_w[w];
    pre += w < warp ? x : 0;
    tot += x;
  }
  *total = tot;
  return pre + incl - v;
}

__global__ void __launch_bounds__(kRankThreads) k_rank_sums(RankScanArgs a) {
  const int64_t n_vis = min(a.n_vis, (int64_t)*a.n_vis_dev);
  const int64_t c = blockIdx.x;
  if (c * kRankChunk >= n_vis) return;
  uint32_t id[kRankItems], cnt[kRankItems];
  uint64_t rect[kRankItems];
  rank_chunk_load(a, n_vis, c * kRankChunk + (int64_t)threadIdx.x * kRankItems, id, rect, cnt);
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < kRankItems; ++j) sum += cnt[j];
  uint32_t total;
  rank_block_scan(sum, &total);
  if (threadIdx.x == 0) a.chunk_sums[c] = total;
}

// one CTA: exclusive scan of the chunk sums in place
__global__ void __launch_bounds__(1024) k_rank_offsets(RankScanArgs a) {
  const int64_t n_vis = min(a.n_vis, (int64_t)*a.n_vis_dev);
  const int64_t chunks = (n_vis + kRankChunk - 1) / kRankChunk;
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = 0;
  for (int64_t base = 0; base < chunks; base += 1024) {
    const int64_t i = base + tid;
    const uint32_t v = i < chunks ? a.chunk_sums[i] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    __syncthreads();  // s_carry of the previous step is visible; s_w free
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    uint32_t pre = s_carry, tot = 0;
    for (int w = 0; w < 32; ++w) {
      const uint32_t x = s_w[w];
      pre += w < warp ? x : 0;
      tot += x;
    }
    if (i < chunks) a.chunk_sums[i] = pre + incl - v;
    __syncthreads();
    if (tid == 0) s_carry += tot;
  }
}

__global__ void __launch_bounds__(kRankThreads) k_rank_write(RankScanArgs a) {
  const int64_t n_vis = min(a.n_vis, (int64_t)*a.n_vis_dev);
  const int64_t c = blockIdx.x;
  if (c * kRankChunk >= n_vis) return;
  const int64_t r0 = c * kRankChunk + (int64_t)threadIdx.x * kRankItems;
  uint32_t id[kRankItems], cnt[kRankItems];
  uint64_t rect[kRankItems];
  rank_chunk_load(a, n_vis, r0, id, rect, cnt);
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < kRankItems; ++j) sum += cnt[j];
  uint32_t total;
  const uint32_t excl = rank_block_scan(sum, &total);
  uint64_t start = (uint64_t)a.chunk_sums[c] + excl;
#pragma unroll
  for (int j = 0; j < kRankItems; ++j) {
    const int64_t r = r0 + j;
    if (r >= n_vis) break;
    a.rrec[r] = make_uint4((uint32_t)rect[j], (uint32_t)(rect[j] >> 32), id[j], (uint32_t)start);
    // the sort tiles whose first slot this rank holds
    const uint64_t end = start + cnt[j];
    for (uint64_t b = (start + kSortTile - 1) / kSortTile;
         b * kSortTile < end && (int64_t)b < a.n_sort_tiles; ++b)
      a.chunk_first[b] = (uint32_t)r;
    start = end;
  }
}

__global__ void k_cover_reduce(const int32_t* __restrict__ part, int parts, int64_t d,
                               int32_t* cover) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d) return;
  const int per = (parts + gridDim.y - 1) / gridDim.y;
  const int g0 = blockIdx.y * per, g1 = min(parts, g0 + per);
  int32_t v = 0;
#pragma unroll 8
  for (int g = g0; g < g1; ++g) v += part[(int64_t)g * d + e];
  if (v) atomicAdd(cover + e, v);
}

// K4p: one CTA.  Column then row prefix sums turn the difference array into
// per-tile counts; a block scan over the tiles gives the ranges; shared
// histograms of the low / high tile digit give the fused sort's plan.
constexpr int kPlanThreads = 1024;
__global__ void __launch_bounds__(kPlanThreads) k_tile_plan(TilePlanArgs a) {
  extern __shared__ int32_t s_c[];
  __shared__ uint32_t s_lo[256], s_hi[256];
  __shared__ uint32_t s_warp[kPlanThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = a.tiles_x, ty = a.tiles_y, cw = tx + 1;
  const int d = cw * (ty + 1);
  const int tiles = tx * ty;
  for (int i0 = tid; i0 < d; i0 += 4 * kPlanThreads) {  // four loads in flight
    int32_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = i0 + u * kPlanThreads < d ? a.cover[i0 + u * kPlanThreads] : 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * kPlanThreads < d) s_c[i0 + u * kPlanThreads] = v[u];
  }
  if (tid < 256) s_lo[tid] = s_hi[tid] = 0;
  const unsigned long long k = *a.k_dev;  // == the sum of the counts (both exact)
  __syncthreads();
  // columns: warp per column, 32 rows per step (shuffle scans, not a
  // dependent walk down the rows)
  for (int x = warp; x < tx; x += kPlanThreads / 32) {
    int32_t carry = 0;
    for (int y0 = 0; y0 < ty; y0 += 32) {
      const int y = y0 + lane;
      int32_t v = y < ty ? s_c[y * cw + x] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (y < ty) s_c[y * cw + x] = v + carry;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  // rows: warp per row, 32 columns per step
  for (int y = warp; y < ty; y += kPlanThreads / 32) {
    int32_t carry = 0;
    for (int x0 = 0; x0 < tx; x0 += 32) {
      const int x = x0 + lane;
      int32_t v = x < tx ? s_c[y * cw + x] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (x < tx) s_c[y * cw + x] = v + carry;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  // tiles in row-major order: thread t owns [t * per, (t + 1) * per)
  const int per = (tiles + kPlanThreads - 1) / kPlanThreads;
  const int t0 = tid * per, t1 = min(tiles, t0 + per);
  uint32_t sum = 0;
  const int ty0 = t0 / tx, tx0 = t0 - ty0 * tx;
  for (int t = t0, y = ty0, x = tx0; t < t1; ++t) {
    const uint32_t c = (uint32_t)s_c[y * cw + x];
    sum += c;
    if (c) {
      atomicAdd(&s_lo[t & 0xff], c);
      atomicAdd(&s_hi[(t >> 8) & 0xff], c);
    }
    if (++x == tx) x = 0, ++y;
  }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint32_t run = incl - sum, total = 0;
  for (int w = 0; w < kPlanThreads / 32; ++w) {
    const uint32_t v = s_warp[w];
    run += w < warp ? v : 0;
    total += v;
  }
  const bool over = k > a.cap;
  for (int t = t0, y = ty0, x = tx0; t < t1; ++t) {
    const uint32_t c = (uint32_t)s_c[y * cw + x];
    a.ranges[t] = over ? make_int2(0, 0) : make_int2((int)run, (int)(run + c));
    if (a.tile_count) a.tile_count[t] = over ? 0u : c;
    run += c;
    if (++x == tx) x = 0, ++y;
  }
  // plan: exclusive digit starts of both passes (threads 0..255)
  __syncthreads();  // every thread has read s_warp
  if (warp < 8) {
    for (int p = 0; p < 2; ++p) {
      const uint32_t c = p ? s_hi[tid] : s_lo[tid];
      uint32_t v = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      __syncwarp();
      if (lane == 31) s_warp[warp] = v;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      uint32_t pre = 0;
      for (int w = 0; w < 8; ++w) pre += w < warp ? s_warp[w] : 0;
      a.plan->digit_start[p][tid] = pre + v - c;
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
  }
  if (tid == 0) {
    RadixPlan* pl = a.plan;
    pl->n_passes = 2;
    pl->first_active = 0;
    pl->last_active = 1;
    for (int p = 0; p < kMaxPasses; ++p) pl->active[p] = p < 2, pl->src[p] = p == 1;
    pl->result = 0;
    *a.k_eff = over ? 0ull : k;
    if (a.max_k) atomicMax(a.max_k, k);
    *a.keys_result = a.result;
  }
  (void)total;
}

// ---------------------------------------------------------------------------
// K6: tile ranges = exclusive scan of the per-tile counts (one CTA)

constexpr int kScanThreads = 1024;
constexpr int kScanPer = 8;  // counts per thread per step

__global__ void __launch_bounds__(kScanThreads) k_ranges_from_counts(const uint32_t* counts,
                                                                     int tiles, int2* ranges,
                                                                     uint32_t cap) {
  __shared__ uint32_t s_warp[kScanThreads / 32];
  __shared__ uint32_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < tiles; base += kScanThreads * kScanPer) {
    const int t0 = base + tid * kScanPer;
    uint32_t c[kScanPer];
    uint32_t sum = 0;
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
      c[j] = t0 + j < tiles ? counts[t0 + j] : 0u;
      sum += c[j];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint32_t w = s_warp[lane];
      uint32_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += v;
      }
      s_warp[lane] = wi - w;
    }
    __syncthreads();
    uint32_t run = s_carry + s_warp[warp] + (incl - sum);
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
      if (t0 + j < tiles)
        ranges[t0 + j] = make_int2((int)min(run, cap), (int)min(run + c[j], cap));
      run += c[j];
    }
    __syncthreads();
    if (tid == kScanThreads - 1) s_carry = run;
    __syncthreads();
  }
}

// instance export: keys = tile << 32 | row, prims = original id; one CTA per
// tile (the sorted ids carry no tile bits: the tile is the range's)
__global__ void k_export(InstanceExportArgs a, int tiles) {
  const uint32_t* __restrict__ ids = static_cast<const uint32_t*>(*a.keys_slot);
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int2 r = a.ranges[t];
    for (int64_t i = r.x + (int64_t)threadIdx.x; i < r.y && i < a.k; i += blockDim.x) {
      const uint32_t id = ids[i];
      if (a.keys_out) a.keys_out[i] = ((uint64_t)t << 32) | id;
      if (a.prims_out) a.prims_out[i] = a.prim_ids ? a.prim_ids[id] : (int64_t)id;
    }
  }
}

inline unsigned grid_for(int64_t n, int threads, int64_t cap = 148 * 16) {
  int64_t g = (n + threads - 1) / threads;
  if (g > cap) g = cap;
  return (unsigned)(g > 0 ? g : 1);
}

}  // namespace

int launch_depth_keys(const uint64_t* key64, const unsigned long long* zrange, int64_t n,
                      uint32_t* key32, uint32_t* hist, cudaStream_t s) {
  if (n <= 0) return 0;
  k_depth_keys<<<grid_for(n, 256, 148 * LMGS_DEPTH_KEYS_CTAS_PER_SM), 256, 0, s>>>(key64, zrange, n,
                                                                                 key32, hist);
  return 1;
}

int launch_depth_fixup(void* const* keys_slot, void* const* ids_slot, int64_t n,
                       const uint64_t* key64, const int64_t* prim_ids, cudaStream_t s) {
  if (n <= 1) return 0;
  const int64_t threads = (n + kFixupPer - 1) / kFixupPer;
  k_depth_fixup<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(keys_slot, ids_slot, n, key64,
                                                                   prim_ids);
  return 1;
}

int launch_emit(const EmitArgs& a, cudaStream_t s) {
  const int64_t chunks = emit_chunks(a.n_vis);
  if (chunks <= 0) return 0;
  int64_t grid = chunks;
  if (a.concurrent && LMGS_EMIT_PERSIST_CTAS > 0) {
    static int sms[kMaxDevices] = {};
    const int dev = current_device();
    if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
    const int64_t p = (int64_t)sms[dev] * LMGS_EMIT_PERSIST_CTAS;
    if (grid > p) grid = p;
  }
  k_emit<<<(unsigned)grid, kEmitThreads, 0, s>>>(a);
  return 1;
}

int launch_ranges_from_counts(const uint32_t* counts, int tiles, int2* ranges, int64_t cap,
                              cudaStream_t s) {
  if (tiles <= 0) return 0;
  const uint32_t c = cap < 0 || cap > 0xffffffffll ? 0xffffffffu : (uint32_t)cap;
  k_ranges_from_counts<<<1, kScanThreads, 0, s>>>(counts, tiles, ranges, c);
  return 1;
}

int cover_grid(int tiles_x, int tiles_y, int64_t n, int sms) {
  if (n <= 0) return 0;
  const size_t smem = sizeof(int32_t) * (size_t)(tiles_x + 1) * (tiles_y + 1);
  static size_t smem_set[kMaxDevices] = {};
  const int dev = current_device();
  if (smem > smem_set[dev]) {
    cudaFuncSetAttribute(k_cover, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smem_set[dev] = smem;
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cover, kCoverThreads, smem);
  if (occ < 1) occ = 1;
  const int64_t need = (n + kCoverThreads * 4 - 1) / (kCoverThreads * 4);
  return (int)(need < (int64_t)sms * occ ? need : (int64_t)sms * occ);
}

int launch_cover(const uint64_t* rects, int64_t n, int tiles_x, int tiles_y, int32_t* cover_part,
                 int grid, cudaStream_t s) {
  if (grid <= 0) return 0;
  const size_t smem = sizeof(int32_t) * (size_t)(tiles_x + 1) * (tiles_y + 1);
  k_cover<<<(unsigned)grid, kCoverThreads, smem, s>>>(rects, n, tiles_x, tiles_y, cover_part);
  return 1;
}

int launch_rank_scan(const RankScanArgs& a, cudaStream_t s) {
  const int64_t chunks = rank_chunks(a.n_vis);
  if (chunks <= 0) return 0;
  k_rank_sums<<<(unsigned)chunks, kRankThreads, 0, s>>>(a);
  k_rank_offsets<<<1, 1024, 0, s>>>(a);
  k_rank_write<<<(unsigned)chunks, kRankThreads, 0, s>>>(a);
  return 3;
}

int launch_cover_reduce(const int32_t* part, int parts, int64_t d, int32_t* cover, cudaStream_t s) {
  if (parts <= 0 || d <= 0) return 0;
  const int slices = parts < 16 ? parts : 16;
  dim3 grid((unsigned)((d + 255) / 256), (unsigned)slices);
  k_cover_reduce<<<grid, 256, 0, s>>>(part, parts, d, cover);
  return 1;
}

int launch_tile_plan(const TilePlanArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(int32_t) * (size_t)(a.tiles_x + 1) * (a.tiles_y + 1);
  static size_t smem_set[kMaxDevices] = {};
  const int dev = current_device();
  if (smem > smem_set[dev]) {
    cudaFuncSetAttribute(k_tile_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smem_set[dev] = smem;
  }
  k_tile_plan<<<1, kPlanThreads, smem, s>>>(a);
  return 1;
}

void launch_export_instances(const InstanceExportArgs& a, cudaStream_t s) {
  if (a.k <= 0 || a.tiles <= 0) return;
  k_export<<<a.tiles < 148 * 16 ? a.tiles : 148 * 16, 128, 0, s>>>(a, a.tiles);
}

}  // namespace lmgs
