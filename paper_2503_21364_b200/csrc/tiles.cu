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
#ifndef LMGS_EMIT_HIST_LANE
#define LMGS_EMIT_HIST_LANE 1  // K4's tile-digit histograms: per-lane increments for every digit
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
#ifndef LMGS_FIXUP_WARP
#define LMGS_FIXUP_WARP 1  // run heads compacted per warp (k_depth_fixup_w)
#endif
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

// Warp-compacted variant: a warp finds the run heads among its 128 keys (4 per
// lane, as above), compacts them in shared memory, and then resolves 32 heads
// at a time with every lane busy — the per-thread loop above runs each of its
// 4 head slots as a divergent path in nearly every warp (c3: ~20 % of the keys
// head a run).
__global__ void __launch_bounds__(256) k_depth_fixup_w(void* const* keys_slot, void* const* ids_slot,
                                                       int64_t n, const uint64_t* __restrict__ key64,
                                                       const int64_t* __restrict__ pid) {
  static_assert(kFixupPer == 4, "128 keys per warp: 7-bit head offsets");
  __shared__ uint8_t s_head[8][32 * kFixupPer];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbase = ((int64_t)blockIdx.x * 8 + warp) * 32 * kFixupPer;
  if (wbase >= n) return;
  const int64_t i0 = wbase + (int64_t)lane * kFixupPer;
  const uint32_t* __restrict__ keys = static_cast<const uint32_t*>(*keys_slot);
  uint32_t* __restrict__ ids = static_cast<uint32_t*>(*ids_slot);
  uint32_t k[kFixupPer + 2];  // keys[i0 - 1 .. i0 + kFixupPer]
#pragma unroll
  for (int u = 0; u < kFixupPer + 2; ++u) {
    const int64_t i = i0 - 1 + u;
    k[u] = (i >= 0 && i < n) ? keys[i] : kDepthKeyNone + 1 + u;  // sentinels never equal
  }
  uint32_t heads = 0, twos = 0;  // bit u-1: key i0 + u - 1 heads a run (of length 2)
#pragma unroll
  for (int u = 1; u <= kFixupPer; ++u) {
    const bool head = i0 - 1 + u < n && k[u] != kDepthKeyNone && k[u - 1] != k[u] &&
                      k[u + 1] == k[u];
    if (head) heads |= 1u << (u - 1);
    if (head && u + 2 <= kFixupPer + 1 && k[u + 2] != k[u]) twos |= 1u << (u - 1);
  }
  const uint32_t cnt = __popc(heads);
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  uint32_t at = incl - cnt;
#pragma unroll
  for (int u = 0; u < kFixupPer; ++u)
    if (heads >> u & 1u)
      s_head[warp][at++] = (uint8_t)(lane * kFixupPer + u) | (uint8_t)((twos >> u & 1u) << 7);
  __syncwarp();
  for (uint32_t h = lane; h < total; h += 32) {
    const uint8_t e = s_head[warp][h];
    const int64_t i = wbase + (e & 0x7f);
    uint32_t* run = ids + i;
    if (e & 0x80) {  // a run of two: two independent gathers, maybe a swap
      const uint32_t a0 = run[0], a1 = run[1];
      const uint64_t d0 = key64[a0], d1 = key64[a1];
      const int64_t p0 = pid ? pid[a0] : (int64_t)a0, p1 = pid ? pid[a1] : (int64_t)a1;
      if (less64(d1, p1, d0, p0)) {
        run[0] = a1;
        run[1] = a0;
      }
    } else {
      const uint32_t kv = keys[i];
      int64_t len = 2;
      while (i + len < n && keys[i + len] == kv) ++len;
      fix_run(run, (int)len, key64, pid);
    }
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
      atomicAdd(&s_hist[0][tile & 0xffu], 1u);
#if LMGS_EMIT_HIST_LANE
      // every digit by a per-lane increment: a window holds ~9 splats at
      // random places (depth order), so even the high digits are warp-uniform
      // in under 1% of windows (c3, ncu) and a vote-then-aggregate step costs
      // more than it saves
      for (int ps = 1; ps < passes; ++ps) atomicAdd(&s_hist[ps][(tile >> (8 * ps)) & 0xffu], 1u);
#endif
    }
#if !LMGS_EMIT_HIST_LANE
    // higher digits by one aggregated add when warp-uniform
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
#endif
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
// K4 for the fused tile sort (k_emit_ranks): the same rank-ordered scan as
// k_emit (chunks of kEmitChunk ranks by ticket, warp scans, warp-cooperative
// look-back), but instead of expanding every splat into instance keys it
// writes one 16-B record per rank {rect lo, rect hi, id, first slot} and the
// first rank of every kSortTile-slot sort tile; the tile sort's first pass
// generates its keys from them (sort.cu, kSrcEmit).  The digit histograms of
// both tile passes are computed per rect row without touching the instances:
// a row's tiles t0..t1 are consecutive ids, so their low digits are a cyclic
// range of 256 bins (a difference array: +1 / -1 at its ends, + whole cycles)
// and their high digits one or two bins.

__global__ void __launch_bounds__(kEmitThreads) k_emit_ranks(EmitArgs a) {
  constexpr int NW = kEmitThreads / 32;
  __shared__ int32_t s_dlo[257];       // low-digit difference array
  __shared__ uint32_t s_hi[256];       // high-digit counts
  __shared__ uint32_t s_wtot[NW];
  __shared__ uint32_t s_ticket;
  __shared__ uint32_t s_lo_all;        // whole 256-tile cycles (every low digit)
  __shared__ unsigned long long s_excl;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 257; i += kEmitThreads) s_dlo[i] = 0;
  for (int i = tid; i < 256; i += kEmitThreads) s_hi[i] = 0;
  if (tid == 0) s_lo_all = 0;
  const int64_t n_vis = min(a.n_vis, (int64_t)*a.n_vis_dev);  // the grid covers a bound
  const uint32_t tx = (uint32_t)a.tiles_x;
  uint32_t lo_all = 0;
  for (;;) {
  if (tid == 0) s_ticket = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const int64_t chunk = s_ticket;
  if (chunk * kEmitChunk >= n_vis) break;
  const uint32_t* __restrict__ order = static_cast<const uint32_t*>(*a.order_slot);
  // blocked layout: thread t owns ranks r0 .. r0 + kEmitItems - 1
  const int64_t r0 = chunk * kEmitChunk + (int64_t)tid * kEmitItems;
  uint32_t id[kEmitItems];
  uint64_t rect[kEmitItems];
  uint32_t cnt[kEmitItems];
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < kEmitItems; ++j) id[j] = r0 + j < n_vis ? order[r0 + j] : 0xffffffffu;
#pragma unroll
  for (int j = 0; j < kEmitItems; ++j)
    rect[j] = id[j] != 0xffffffffu ? __ldg(a.rects + id[j]) : kEmptyRect;
#pragma unroll
  for (int j = 0; j < kEmitItems; ++j) {
    int x0, y0, x1, y1;
    unpack_rect(rect[j], x0, y0, x1, y1);
    const uint32_t w = (uint32_t)(x1 - x0 + 1);
    cnt[j] = w * (uint32_t)(y1 - y0 + 1);  // 0 for kEmptyRect
    sum += cnt[j];
    // digit histograms, one rect row at a time
    for (int y = y0; y <= y1 && w; ++y) {
      const uint32_t t0 = (uint32_t)y * tx + (uint32_t)x0, t1 = t0 + w - 1;
      lo_all += w >> 8;
      const uint32_t rem = w & 255u, ds = t0 & 255u;
      if (rem) {
        atomicAdd(&s_dlo[ds], 1);
        if (ds + rem <= 256u) {
          atomicAdd(&s_dlo[ds + rem], -1);
        } else {
          atomicAdd(&s_dlo[256], -1);
          atomicAdd(&s_dlo[0], 1);
          atomicAdd(&s_dlo[ds + rem - 256u], -1);
        }
      }
      const uint32_t h0 = t0 >> 8, h1 = t1 >> 8;
      if (h0 == h1) {
        atomicAdd(&s_hi[h0 & 255u], w);
      } else {
        atomicAdd(&s_hi[h0 & 255u], 256u - (t0 & 255u));
        for (uint32_t h = h0 + 1; h < h1; ++h) atomicAdd(&s_hi[h & 255u], 256u);
        atomicAdd(&s_hi[h1 & 255u], (t1 & 255u) + 1u);
      }
    }
  }
  uint32_t scan = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, scan, o);
    if (lane >= o) scan += v;
  }
  if (lane == 31) s_wtot[warp] = scan;
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
      int64_t end = chunk;
      while (true) {
        const int64_t idx = end - 1 - lane;
        uint64_t v = kLbIncl;
        if (idx >= 0) {
          do {
            v = ld_relaxed_gpu(lb + idx);
          } while ((v & ~kLbMask) == 0);
        }
        const uint32_t incl = __ballot_sync(0xffffffffu, (v & ~kLbMask) == kLbIncl);
        const int stop = incl ? __ffs(incl) - 1 : 31;
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
  uint64_t start = s_excl + wofs + (scan - sum);
#pragma unroll
  for (int j = 0; j < kEmitItems; ++j) {
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
  }  // the loop exits right after a __syncthreads: every shared atomic has landed
  if (lo_all) atomicAdd(&s_lo_all, lo_all);
  __syncthreads();
  // no-sync overflow (K past the capacity): no histogram, so the passes place
  // the first `cap` slots inside [0, cap) and the stats report the overflow
  if (*a.k_dev > a.cap) return;
  {
    // inclusive prefix of the difference array = low-digit counts
    __shared__ uint32_t s_w[kEmitThreads / 32];
    const int d = tid;  // kEmitThreads == 256
    const int32_t v = s_dlo[d];
    int32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) s_w[warp] = (uint32_t)incl;
    __syncthreads();
    int32_t pre = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) pre += w < warp ? (int32_t)s_w[w] : 0;
    const uint32_t lo = (uint32_t)(pre + incl) + s_lo_all;
    if (lo) atomicAdd(a.hist + d, lo);
    if (s_hi[d]) atomicAdd(a.hist + 256 + d, s_hi[d]);
  }
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
  static bool once = false;
  if (!once) set_carveout(k_depth_fixup_w), set_carveout(k_depth_keys), once = true;
  if (LMGS_FIXUP_WARP)
    k_depth_fixup_w<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(keys_slot, ids_slot, n,
                                                                       key64, prim_ids);
  else
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
  static bool once = false;
  if (!once) set_carveout(k_emit), once = true;
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

int launch_emit_ranks(const EmitArgs& a, cudaStream_t s) {
  const int64_t chunks = emit_chunks(a.n_vis);
  if (chunks <= 0) return 0;
  static_assert(kEmitThreads == 256, "k_emit_ranks: one thread per digit");
  k_emit_ranks<<<(unsigned)chunks, kEmitThreads, 0, s>>>(a);
  return 1;
}

void launch_export_instances(const InstanceExportArgs& a, cudaStream_t s) {
  if (a.k <= 0 || a.tiles <= 0) return;
  k_export<<<a.tiles < 148 * 16 ? a.tiles : 148 * 16, 128, 0, s>>>(a, a.tiles);
}

}  // namespace lmgs
