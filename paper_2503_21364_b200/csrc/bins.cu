// Tile instance lists through coarse bins (K4 + K5 + K6 of the default path).
//
// Reference: rasterize (gaussian_core.py:340-403) builds, for every tile, the
// list of splats whose bbox overlaps it (367-373) in _sort_order's
// (depth, prim_id) order (277-283, 392).  After K2 the visible splats are in
// that global rank order, so a tile's list is the rank-ordered subsequence of
// splats overlapping it.
//
// The direct way — emit one 8-byte (tile, id) key per instance in rank order
// and stable-radix-sort the K keys by tile (tiles.cu k_emit + 2 onesweep
// passes at 1080p) — moves every instance through HBM five times.  Here the
// instances are written once, in place:
//
//   B1 k_bin_emit    walk the splats in rank order (chunks, decoupled look-back
//                    scan of their bin counts) and emit one entry per coarse
//                    bin (8x8 tiles) the splat's tile rect meets:
//                    id | bin << 32 | clipped local rect << 48  (E ~ 1.1 n_vis)
//   B2 onesweep      stable radix sort of the E entries on the bin bits
//                    (1 pass up to 256 bins: 1080p has 135, 4K 510 -> 2); the
//                    last pass counts each bin's entries
//   B3 k_bin_plan    bin entry ranges and the split of every bin's entry run
//                    into pieces of kPiece entries
//   B4 k_piece_count per piece: instances per tile of its bin (64 counters)
//   B5 k_bin_prefix  per (bin, tile): exclusive prefix of the pieces' counts
//                    and the tile's total; K6 scans the totals into ranges
//   B6 k_piece_write per piece: walk its entries in rank order, rank each
//                    instance stably within its tile (warp ballots per tile)
//                    and write key tile << 32 | id straight to its final slot.
//
// Every tile's list is then the reference's (depth, id) order: entries of a
// bin stay in rank order through the stable sort, pieces are consecutive, and
// inside a piece instances are ranked in entry order.
#include "device_util.cuh"
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

constexpr uint64_t kLbAgg = 1ull << 62;
constexpr uint64_t kLbIncl = 2ull << 62;
constexpr uint64_t kLbMask = (1ull << 62) - 1;

__device__ __forceinline__ void unpack_rect(uint64_t rect, int& x0, int& y0, int& x1, int& y1) {
  x0 = (int)(rect & 0xffff);
  y0 = (int)((rect >> 16) & 0xffff);
  x1 = (int)((rect >> 32) & 0xffff);
  y1 = (int)((rect >> 48) & 0xffff);
}

// local rect (lx0, ly0, lx1, ly1 in 0..7, 3 bits each) -> bit j = ly * 8 + lx
__device__ __forceinline__ uint64_t rect_mask(uint32_t lr) {
  const int lx0 = lr & 7, ly0 = (lr >> 3) & 7, lx1 = (lr >> 6) & 7, ly1 = (lr >> 9) & 7;
  const uint64_t row = ((0xffu >> (7 - (lx1 - lx0))) << lx0) & 0xffu;  // bits lx0..lx1
  uint64_t m = 0;
  for (int y = ly0; y <= ly1; ++y) m |= row << (8 * y);
  return m;
}

// ---------------------------------------------------------------------------
// B1: rank-ordered bin entries (k_emit's scan, one entry per overlapped bin)

__global__ void __launch_bounds__(kEmitThreads) k_bin_emit(BinArgs a) {
  constexpr int NW = kEmitThreads / 32;
  constexpr int PW = 32 * kEmitItems;  // ranks per warp
  __shared__ uint32_t s_end[NW][PW];
  __shared__ uint32_t s_id[NW][PW];
  __shared__ uint64_t s_rect[NW][PW];
  __shared__ uint32_t s_hist[2][256];
  __shared__ uint32_t s_wtot[NW];
  __shared__ uint32_t s_ticket;
  __shared__ unsigned long long s_excl;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_ticket = atomicAdd(a.ticket, 1u);
  for (int i = tid; i < 2 * 256; i += kEmitThreads) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  const int64_t n_vis = (int64_t)*a.n_vis;
  const int64_t chunks = (n_vis + kEmitChunk - 1) / kEmitChunk;
  const int64_t chunk = s_ticket;
  if (chunk >= chunks) return;  // grid sized for an upper bound of n_vis
  const int64_t base = chunk * kEmitChunk + (int64_t)warp * PW;
  const uint32_t* __restrict__ order = static_cast<const uint32_t*>(*a.order_slot);

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
    sum += id[j] != 0xffffffffu
               ? (uint32_t)((x1 >> 3) - (x0 >> 3) + 1) * (uint32_t)((y1 >> 3) - (y0 >> 3) + 1)
               : 0u;
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
  if (warp == 0) {  // warp-cooperative look-back, 32 predecessors per round trip
    uint64_t* lb = a.lookback;
    uint64_t excl = 0;
    if (chunk == 0) {
      if (lane == 0) st_relaxed_gpu(lb, kLbIncl | total);
    } else {
      if (lane == 0) st_relaxed_gpu(lb + chunk, kLbAgg | total);
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
      if (lane == 0) st_relaxed_gpu(lb + chunk, kLbIncl | (excl + total));
    }
    if (lane == 0) {
      s_excl = excl;
      if (chunk == chunks - 1) *a.n_entries = excl + total;  // E
    }
  }
  __syncthreads();
  const uint64_t out0 = s_excl + wofs;
  const uint32_t wtot = s_wtot[warp];
  const uint32_t* ends = s_end[warp];
  const bool two = a.n_bin_passes > 1;
  const uint64_t cap = a.entry_cap;
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
    if (p < wtot) {
      const uint32_t q = p - st_i;
      const int x0 = (int)(r_lo & 0xffff), y0 = (int)(r_lo >> 16);
      const int x1 = (int)(r_hi & 0xffff), y1 = (int)(r_hi >> 16);
      const int bx0 = x0 >> 3, by0 = y0 >> 3;
      const uint32_t wb = (uint32_t)((x1 >> 3) - bx0 + 1);
      const uint32_t dy = q / wb;  // small: a splat meets few bins
      const int bx = bx0 + (int)(q - dy * wb), by = by0 + (int)dy;
      const uint32_t bin = (uint32_t)by * (uint32_t)a.bins_x + (uint32_t)bx;
      const int ox = bx * 8, oy = by * 8;
      const uint32_t lx0 = (uint32_t)max(x0 - ox, 0), lx1 = (uint32_t)min(x1 - ox, 7);
      const uint32_t ly0 = (uint32_t)max(y0 - oy, 0), ly1 = (uint32_t)min(y1 - oy, 7);
      const uint32_t lr = lx0 | ly0 << 3 | lx1 << 6 | ly1 << 9;
      if (out0 + p < cap)
        a.entries[out0 + p] = ((uint64_t)lr << 48) | ((uint64_t)bin << 32) | id_i;
      atomicAdd(&s_hist[0][bin & 0xffu], 1u);
      if (two) atomicAdd(&s_hist[1][(bin >> 8) & 0xffu], 1u);
    }
    const int idx31 = __shfl_sync(0xffffffffu, idx, 31);
    k0 += idx31 + (ends[k0 + idx31] == p0 + 32u ? 1 : 0);
  }
  __syncthreads();
  for (int i = tid; i < a.n_bin_passes * 256; i += kEmitThreads) {
    const uint32_t v = (&s_hist[0][0])[i];
    if (v) atomicAdd(a.hist + i, v);
  }
}

// ---------------------------------------------------------------------------
// B3: bin entry ranges + pieces (one CTA)

constexpr int kPlanThreads = 1024;

__global__ void __launch_bounds__(kPlanThreads) k_bin_plan(BinArgs a) {
  __shared__ uint32_t s_w0[kPlanThreads / 32], s_w1[kPlanThreads / 32];
  __shared__ uint32_t s_c0, s_c1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    s_c0 = s_c1 = 0;
    // the sorted entries are the radix result; the instances go to the other buffer
    void* sorted = *a.entries_slot;
    *a.keys_slot = sorted == a.buf[0] ? a.buf[1] : a.buf[0];
  }
  __syncthreads();
  const int nb = a.n_bins;
  for (int b0 = 0; b0 <= nb; b0 += kPlanThreads) {
    const int b = b0 + tid;
    const uint32_t c = b < nb ? a.bin_count[b] : 0u;
    const uint32_t pc = (c + kPiece - 1) / kPiece;
    uint32_t i0 = c, i1 = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v0 = __shfl_up_sync(0xffffffffu, i0, o);
      const uint32_t v1 = __shfl_up_sync(0xffffffffu, i1, o);
      if (lane >= o) i0 += v0, i1 += v1;
    }
    if (lane == 31) s_w0[warp] = i0, s_w1[warp] = i1;
    __syncthreads();
    if (warp == 0) {
      uint32_t w0 = s_w0[lane], w1 = s_w1[lane], x0 = w0, x1 = w1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v0 = __shfl_up_sync(0xffffffffu, x0, o);
        const uint32_t v1 = __shfl_up_sync(0xffffffffu, x1, o);
        if (lane >= o) x0 += v0, x1 += v1;
      }
      s_w0[lane] = x0 - w0;
      s_w1[lane] = x1 - w1;
    }
    __syncthreads();
    const uint32_t e0 = s_c0 + s_w0[warp] + i0 - c, e1 = s_c1 + s_w1[warp] + i1 - pc;
    if (b <= nb) {
      a.bin_start[b] = e0;
      a.piece_start[b] = e1;
    }
    __syncthreads();
    if (tid == kPlanThreads - 1) s_c0 = e0 + c, s_c1 = e1 + pc;
    __syncthreads();
  }
}

// the piece handled by CTA `p`: its bin (largest b with piece_start[b] <= p)
// and entry range
__device__ __forceinline__ bool piece_of(const BinArgs& a, uint32_t p, int& bin, uint32_t& e0,
                                         uint32_t& e1) {
  if (p >= a.piece_start[a.n_bins]) return false;
  int lo = 0, hi = a.n_bins - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.piece_start[mid] <= p) lo = mid;
    else hi = mid - 1;
  }
  bin = lo;
  e0 = a.bin_start[lo] + (p - a.piece_start[lo]) * kPiece;
  e1 = min(e0 + (uint32_t)kPiece, a.bin_start[lo + 1]);
  return true;
}

// ---------------------------------------------------------------------------
// B4: instances per (piece, tile of its bin)

__global__ void __launch_bounds__(256) k_piece_count(BinArgs a) {
  __shared__ uint32_t s_cnt[64];
  int bin;
  uint32_t e0, e1;
  if (!piece_of(a, blockIdx.x, bin, e0, e1)) return;
  if (threadIdx.x < 64) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t* __restrict__ ent = static_cast<const uint64_t*>(*a.entries_slot);
  for (uint32_t e = e0 + threadIdx.x; e < e1; e += 256) {
    uint64_t m = rect_mask((uint32_t)(ent[e] >> 48));
    while (m) {
      atomicAdd(&s_cnt[__ffsll((long long)m) - 1], 1u);
      m &= m - 1;
    }
  }
  __syncthreads();
  if (threadIdx.x < 64) a.piece_counts[(size_t)blockIdx.x * 64 + threadIdx.x] = s_cnt[threadIdx.x];
}

// ---------------------------------------------------------------------------
// B5: per (bin, tile) exclusive prefix over the bin's pieces + tile totals

__global__ void k_bin_prefix(BinArgs a) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int bin = g >> 6, j = g & 63;
  if (bin >= a.n_bins) return;
  const int tx = (bin % a.bins_x) * 8 + (j & 7), ty = (bin / a.bins_x) * 8 + (j >> 3);
  const uint32_t p0 = a.piece_start[bin], p1 = a.piece_start[bin + 1];
  uint32_t run = 0;
  for (uint32_t p = p0; p < p1; ++p) {
    const uint32_t v = a.piece_counts[(size_t)p * 64 + j];
    a.piece_counts[(size_t)p * 64 + j] = run;
    run += v;
  }
  if (tx < a.tiles_x && ty < a.tiles_y) a.tile_count[ty * a.tiles_x + tx] = run;
}

// ---------------------------------------------------------------------------
// B6: stable per-tile ranking inside a piece and the final keys

__global__ void __launch_bounds__(256) k_piece_write(BinArgs a) {
  constexpr int NW = 8;
  __shared__ uint32_t s_base[64];       // next slot of each tile of the bin
  __shared__ uint32_t s_ball[NW][64];   // per warp, per tile: lanes holding it
  __shared__ uint32_t s_wofs[NW][64];   // per warp, per tile: warp's first slot
  __shared__ uint32_t s_tile[64];       // global tile id of each bin tile
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int bin;
  uint32_t e0, e1;
  if (!piece_of(a, blockIdx.x, bin, e0, e1)) return;
  if (tid < 64) {
    const int tx = (bin % a.bins_x) * 8 + (tid & 7), ty = (bin / a.bins_x) * 8 + (tid >> 3);
    const bool in = tx < a.tiles_x && ty < a.tiles_y;
    const uint32_t t = in ? (uint32_t)(ty * a.tiles_x + tx) : 0u;
    s_tile[tid] = t;
    s_base[tid] = in ? (uint32_t)a.ranges[t].x + a.piece_counts[(size_t)blockIdx.x * 64 + tid] : 0u;
  }
  __syncthreads();
  const uint64_t* __restrict__ ent = static_cast<const uint64_t*>(*a.entries_slot);
  uint64_t* __restrict__ keys = static_cast<uint64_t*>(*a.keys_slot);
  const uint32_t lt = lanemask_lt();
  for (uint32_t b = e0; b < e1; b += 256) {
    const uint32_t e = b + tid;
    uint64_t v = 0, m = 0;
    if (e < e1) {
      v = ent[e];
      m = rect_mask((uint32_t)(v >> 48));
    }
    // lane l keeps the ballots of tiles l and l + 32
    uint32_t blo = 0, bhi = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint32_t b0 = __ballot_sync(0xffffffffu, (uint32_t)(m >> j) & 1u);
      const uint32_t b1 = __ballot_sync(0xffffffffu, (uint32_t)(m >> (j + 32)) & 1u);
      if (lane == j) blo = b0, bhi = b1;
    }
    s_ball[warp][lane] = blo;
    s_ball[warp][lane + 32] = bhi;
    __syncthreads();
    if (tid < 64) {  // warps in order: each warp's first slot per tile
      uint32_t run = s_base[tid];
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        s_wofs[w][tid] = run;
        run += __popc(s_ball[w][tid]);
      }
      s_base[tid] = run;
    }
    __syncthreads();
    const uint64_t idv = v & 0xffffffffull;
    while (m) {
      const int j = __ffsll((long long)m) - 1;
      m &= m - 1;
      const uint32_t pos = s_wofs[warp][j] + __popc(s_ball[warp][j] & lt);
      keys[pos] = ((uint64_t)s_tile[j] << 32) | idv;
    }
    __syncthreads();
  }
}

}  // namespace

int launch_bin_emit(const BinArgs& a, int64_t n_vis_bound, cudaStream_t s) {
  const int64_t chunks = emit_chunks(n_vis_bound);
  if (chunks <= 0) return 0;
  k_bin_emit<<<(unsigned)chunks, kEmitThreads, 0, s>>>(a);
  return 1;
}

int launch_bin_lists(const BinArgs& a, int64_t piece_bound, cudaStream_t s) {
  int launched = 0;
  k_bin_plan<<<1, kPlanThreads, 0, s>>>(a);
  ++launched;
  if (piece_bound > 0) {
    k_piece_count<<<(unsigned)piece_bound, 256, 0, s>>>(a);
    ++launched;
  }
  const int threads = a.n_bins * 64;
  k_bin_prefix<<<(threads + 255) / 256, 256, 0, s>>>(a);
  ++launched;
  launched += launch_ranges_from_counts(a.tile_count, a.tiles_x * a.tiles_y, a.ranges, s);
  if (piece_bound > 0) {
    k_piece_write<<<(unsigned)piece_bound, 256, 0, s>>>(a);
    ++launched;
  }
  return launched;
}

}  // namespace lmgs
