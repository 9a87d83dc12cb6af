// Tile binning: K3 tile counts + scan, K4 placement, K5 per-tile sort, export.
//
// Reference: rasterize (gaussian_core.py:340-403) builds, for every tile, the
// list of splats whose bbox overlaps it (367-373) in _sort_order's
// (depth, prim_id) order (277-283, 392).
//
// B200 design — per-tile lists are built tile-locally, with no global sort
// and no hot global atomics:
//   K3a  one CTA per SM owns a contiguous slice of Gaussians and builds the
//        per-tile instance histogram of its slice in shared memory (8K-32K
//        counters), writing one row H[cta][tile];
//   K3b  a column scan turns H into per-(cta, tile) offsets and tile totals;
//   K3c  one CTA scans the tile totals: tile_ranges (an output), K, and the
//        size class of every tile;
//   K4   the same CTAs place their instances (Gaussian ids, 4 B) into the
//        tile buckets through shared-memory cursors (order inside a bucket
//        is arbitrary);
//   K5   one CTA per bucket sorts it in shared memory: one counting pass into
//        4096 bins over the bucket's fp32-key range, then per-bin insertion
//        sorts by (fp32 key, fp64 depth, id) — the exact order;
//   big  buckets above kMediumTileCap: onesweep radix on
//        (bucket index << 32 | fp32 key) + the same fix-up (sort.cu).
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ void unpack_rect(uint64_t rect, int& x0, int& y0, int& x1, int& y1) {
  x0 = (int)(rect & 0xffff);
  y0 = (int)((rect >> 16) & 0xffff);
  x1 = (int)((rect >> 32) & 0xffff);
  y1 = (int)((rect >> 48) & 0xffff);
}

// ---------------------------------------------------------------------------
// K3a: per-CTA shared-memory tile histograms

__global__ void __launch_bounds__(kBinThreads) k_bin_hist(BinArgs a) {
  extern __shared__ __align__(16) uint32_t s_cnt[];
  const int c = blockIdx.x;
  const int64_t lo = a.n * c / a.ctas, hi = a.n * (c + 1) / a.ctas;
  for (int slab = 0; slab < a.tiles; slab += kSlabTiles) {
    const int sw = min(kSlabTiles, a.tiles - slab);
    for (int t = threadIdx.x; t < sw; t += blockDim.x) s_cnt[t] = 0;
    __syncthreads();
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      if (!a.counts[i]) continue;
      int x0, y0, x1, y1;
      unpack_rect(a.rects[i], x0, y0, x1, y1);
      for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) {
          const unsigned t = (unsigned)(y * a.tiles_x + x - slab);
          if (t < (unsigned)sw) atomicAdd(s_cnt + t, 1u);
        }
    }
    __syncthreads();
    uint32_t* row = a.hist + (int64_t)c * a.tiles + slab;
    for (int t = threadIdx.x; t < sw; t += blockDim.x) row[t] = s_cnt[t];
    __syncthreads();
  }
}

// K3b: exclusive scan down each tile column of H; totals per tile.  Loads
// are batched 16 deep so the column walk is not a chain of dependent misses.
__global__ void k_bin_colscan(BinArgs a) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.tiles) return;
  uint32_t* __restrict__ col = a.hist + t;
  const int64_t stride = a.tiles;
  uint32_t run = 0;
  int c = 0;
  for (; c + 16 <= a.ctas; c += 16) {
    uint32_t v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = col[(c + j) * stride];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      col[(c + j) * stride] = run;
      run += v[j];
    }
  }
  for (; c < a.ctas; ++c) {
    const uint32_t v = col[c * stride];
    col[c * stride] = run;
    run += v;
  }
  a.tile_count[t] = run;
}

// ---------------------------------------------------------------------------
// K3c: exclusive scan of tile counts (one CTA), classification by size

constexpr int kScanTilesThreads = 1024;

__global__ void __launch_bounds__(kScanTilesThreads) k_scan_tiles(TileScanArgs a) {
  __shared__ uint32_t s_warp[kScanTilesThreads / 32];
  __shared__ unsigned long long s_carry;
  __shared__ uint32_t s_cls[3];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    s_carry = 0;
    s_cls[0] = s_cls[1] = s_cls[2] = 0;
  }
  __syncthreads();
  for (int base = 0; base < a.tiles; base += kScanTilesThreads) {
    const int t = base + tid;
    const uint32_t c = t < a.tiles ? a.tile_count[t] : 0u;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = s_warp[lane];
      uint32_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += v;
      }
      s_warp[lane] = wi - w;
    }
    __syncthreads();
    const unsigned long long excl = s_carry + s_warp[warp] + (incl - c);
    if (t < a.tiles) {
      a.ranges[t] = make_int2((int)excl, (int)(excl + c));
      if (c > 0) {
        const int cls = c <= (uint32_t)a.small_cap ? 0 : (c <= (uint32_t)a.medium_cap ? 1 : 2);
        const uint32_t slot = atomicAdd(&s_cls[cls], 1u);
        a.lists[cls][slot] = (uint32_t)t;
      }
    }
    __syncthreads();
    if (tid == kScanTilesThreads - 1) s_carry = excl + c;
    __syncthreads();
  }
  if (tid == 0) {
    *a.total = s_carry;
    a.class_counts[0] = s_cls[0];
    a.class_counts[1] = s_cls[1];
    a.class_counts[2] = s_cls[2];
  }
}

// ---------------------------------------------------------------------------
// K4: placement through shared-memory cursors (same CTA slices as K3a)

__global__ void __launch_bounds__(kBinThreads) k_bin_place(BinArgs a) {
  extern __shared__ __align__(16) uint32_t s_pos[];
  const int c = blockIdx.x;
  const int64_t lo = a.n * c / a.ctas, hi = a.n * (c + 1) / a.ctas;
  for (int slab = 0; slab < a.tiles; slab += kSlabTiles) {
    const int sw = min(kSlabTiles, a.tiles - slab);
    const uint32_t* row = a.hist + (int64_t)c * a.tiles + slab;
    for (int t = threadIdx.x; t < sw; t += blockDim.x)
      s_pos[t] = (uint32_t)a.ranges[slab + t].x + row[t];
    __syncthreads();
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      if (!a.counts[i]) continue;
      int x0, y0, x1, y1;
      unpack_rect(a.rects[i], x0, y0, x1, y1);
      for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) {
          const unsigned t = (unsigned)(y * a.tiles_x + x - slab);
          if (t < (unsigned)sw) a.bucket[atomicAdd(s_pos + t, 1u)] = (uint32_t)i;
        }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// exact fix-up of a run of equal fp32 keys: order by (fp64 depth bits, id)

__device__ __forceinline__ bool less64(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

// ids[0..len) hold one run; reorder by (key64[id], id).  Short runs are sorted
// in registers; longer ones in place (insertion sort is linear on the common
// long run — exact duplicates, already in id order).
__device__ void fix_run(uint32_t* ids, int len, const uint64_t* __restrict__ key64) {
  if (len <= kFixupRun) {
    uint64_t dk[kFixupRun];
    uint32_t id[kFixupRun];
    for (int a = 0; a < len; ++a) {
      id[a] = ids[a];
      dk[a] = key64[id[a]];
    }
    for (int a = 1; a < len; ++a) {
      const uint64_t kd = dk[a];
      const uint32_t ki = id[a];
      int b = a - 1;
      while (b >= 0 && less64(kd, ki, dk[b], id[b])) {
        dk[b + 1] = dk[b];
        id[b + 1] = id[b];
        --b;
      }
      dk[b + 1] = kd;
      id[b + 1] = ki;
    }
    for (int a = 0; a < len; ++a) ids[a] = id[a];
    return;
  }
  for (int a = 1; a < len; ++a) {
    const uint32_t ki = ids[a];
    const uint64_t kd = key64[ki];
    int b = a - 1;
    while (b >= 0) {
      const uint32_t ib = ids[b];
      if (!less64(kd, ki, key64[ib], ib)) break;
      ids[b + 1] = ib;
      --b;
    }
    ids[b + 1] = ki;
  }
}

// ---------------------------------------------------------------------------
// K5: per-tile sort in shared memory — one unstable MSD counting pass
//
// The exact order is (fp64 depth, id); the fp32 key is a monotone summary of
// the fp64 depth, so any order that is sorted by fp32 key and then by
// (fp64 depth, id) inside equal fp32 keys is exact.  Stability is therefore
// never needed: entries are scattered by shared-memory atomics into NBINS
// bins spanning the bucket's own [kmin, kmax] fp32-key range, then each bin
// (a few entries) is insertion-sorted by (fp32 key, fp64 depth, id).  Bins
// with more than kBinSortMax entries get a second counting pass over their
// own key range (CTA-wide), then the same insertion sort.
//
// smem: buf (key u32 + bucket-local index u16) x CAP, cnt/start NBINS+1 each,
// long-bin list.  Entries of the first pass are held in registers.

constexpr int kBinSortMax = 64;

__device__ __forceinline__ bool entry_less(uint32_t ka, uint32_t ia, uint32_t kb, uint32_t ib,
                                           const uint64_t* __restrict__ key64) {
  if (ka != kb) return ka < kb;
  const uint64_t da = key64[ia], db = key64[ib];
  return da < db || (da == db && ia < ib);
}

// insertion sort of buf[lo, hi) by (key, fp64 depth, id); ids resolved via the bucket
__device__ void sort_small_bin(uint32_t* key, uint16_t* idx, int lo, int hi,
                               const uint32_t* __restrict__ bucket,
                               const uint64_t* __restrict__ key64) {
  for (int a = lo + 1; a < hi; ++a) {
    const uint32_t ka = key[a];
    const uint16_t xa = idx[a];
    const uint32_t ia = (uint32_t)bucket[xa];
    int b = a - 1;
    while (b >= lo) {
      const uint32_t kb = key[b];
      if (kb < ka) break;
      if (kb == ka) {
        const uint32_t ib = (uint32_t)bucket[idx[b]];
        if (!entry_less(ka, ia, kb, ib, key64)) break;
      }
      key[b + 1] = kb;
      idx[b + 1] = idx[b];
      --b;
    }
    key[b + 1] = ka;
    idx[b + 1] = xa;
  }
}

template <int THREADS, int NBINS>
__device__ __forceinline__ void block_exclusive_scan(uint32_t* v, uint32_t* s_wsum, int count) {
  // v[0..count) -> exclusive prefix in place; v[count] = total.  count % THREADS == 0.
  constexpr int PER = NBINS / THREADS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t loc[PER];
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    loc[j] = v[tid * PER + j];
    sum += loc[j];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  uint32_t pre = 0;
  for (int w = 0; w < warp; ++w) pre += s_wsum[w];
  uint32_t run = pre + incl - sum;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    v[tid * PER + j] = run;
    run += loc[j];
  }
  if (tid == THREADS - 1) v[count] = run;
  __syncthreads();
  (void)count;
}

template <int THREADS, int CAP, int NBINS>
__global__ void __launch_bounds__(THREADS) k_tile_sort(TileSortArgs a, const uint32_t* tile_list,
                                                      const uint32_t* list_count) {
  constexpr int PER = (CAP + THREADS - 1) / THREADS;
  constexpr int NW = THREADS / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* s_key = reinterpret_cast<uint32_t*>(smem_raw);                 // [CAP]
  uint16_t* s_idx = reinterpret_cast<uint16_t*>(smem_raw + 4 * CAP);       // [CAP]
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem_raw + 6 * CAP);       // [NBINS + 1]
  uint32_t* s_start = s_cnt + (NBINS + 1);                                 // [NBINS + 1]
  uint16_t* s_long = reinterpret_cast<uint16_t*>(s_start + (NBINS + 1));   // [NBINS]
  __shared__ uint32_t s_kmin, s_kmax, s_nlong;
  __shared__ uint32_t s_wsum[NW];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t nlist = *list_count;
  for (uint32_t li = blockIdx.x; li < nlist; li += gridDim.x) {
    const int t = (int)tile_list[li];
    const int2 r = a.ranges[t];
    const int n = r.y - r.x;
    const uint32_t* __restrict__ bucket = a.bucket + r.x;
    if (tid == 0) {
      s_kmin = 0xffffffffu;
      s_kmax = 0u;
      s_nlong = 0u;
    }
    for (int i = tid; i <= NBINS; i += THREADS) s_cnt[i] = 0u;
    __syncthreads();
    // level 1: entries into registers, key range
    uint32_t rk[PER];
    uint32_t kmin = 0xffffffffu, kmax = 0u;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = tid + j * THREADS;
      rk[j] = i < n ? a.key32[bucket[i]] : 0u;
      if (i < n) {
        kmin = min(kmin, rk[j]);
        kmax = max(kmax, rk[j]);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
      kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0) {
      atomicMin(&s_kmin, kmin);
      atomicMax(&s_kmax, kmax);
    }
    __syncthreads();
    const uint32_t k0 = s_kmin;
    const uint32_t span = s_kmax - k0;
    int shift = 0;
    while ((span >> shift) >= (uint32_t)NBINS) ++shift;
    uint32_t rbin[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = tid + j * THREADS;
      rbin[j] = (rk[j] - k0) >> shift;
      if (i < n) atomicAdd(s_cnt + rbin[j], 1u);
    }
    __syncthreads();
    block_exclusive_scan<THREADS, NBINS>(s_cnt, s_wsum, NBINS);
    for (int i = tid; i <= NBINS; i += THREADS) s_start[i] = s_cnt[i];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = tid + j * THREADS;
      if (i < n) {
        const uint32_t p = atomicAdd(s_cnt + rbin[j], 1u);
        s_key[p] = rk[j];
        s_idx[p] = (uint16_t)i;
      }
    }
    __syncthreads();
    // per-bin ordering
    for (int d = tid; d < NBINS; d += THREADS) {
      const int lo = (int)s_start[d], hi = (int)s_start[d + 1];
      if (hi - lo > kBinSortMax) s_long[atomicAdd(&s_nlong, 1u)] = (uint16_t)d;
      else if (hi - lo > 1) sort_small_bin(s_key, s_idx, lo, hi, bucket, a.key64);
    }
    __syncthreads();
    // level 2 for long bins, one bin at a time, CTA-wide
    const int nlong = (int)s_nlong;
    for (int q = 0; q < nlong; ++q) {
      const int d = s_long[q];
      const int lo = (int)s_start[d], hi = (int)s_start[d + 1];
      const int len = hi - lo;
      // into registers (len <= CAP)
      uint32_t lk[PER];
      uint16_t lx[PER];
      uint32_t lmin = 0xffffffffu, lmax = 0u;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int i = tid + j * THREADS;
        if (i < len) {
          lk[j] = s_key[lo + i];
          lx[j] = s_idx[lo + i];
          lmin = min(lmin, lk[j]);
          lmax = max(lmax, lk[j]);
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
        lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
      }
      __syncthreads();
      if (tid == 0) {
        s_kmin = 0xffffffffu;
        s_kmax = 0u;
      }
      for (int i = tid; i <= NBINS; i += THREADS) s_cnt[i] = 0u;
      __syncthreads();
      if (lane == 0) {
        atomicMin(&s_kmin, lmin);
        atomicMax(&s_kmax, lmax);
      }
      __syncthreads();
      const uint32_t l0 = s_kmin, lspan = s_kmax - l0;
      if (lspan == 0) {  // all fp32 keys equal: order by (fp64 depth, id) only
        __syncthreads();
        if (tid == 0) sort_small_bin(s_key, s_idx, lo, hi, bucket, a.key64);
        __syncthreads();
        continue;
      }
      int sh = 0;
      while ((lspan >> sh) >= (uint32_t)NBINS) ++sh;
      uint32_t lb[PER];
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int i = tid + j * THREADS;
        lb[j] = (lk[j] - l0) >> sh;
        if (i < len) atomicAdd(s_cnt + lb[j], 1u);
      }
      __syncthreads();
      block_exclusive_scan<THREADS, NBINS>(s_cnt, s_wsum, NBINS);
      // s_start is still needed for the outer bins: keep the level-2 starts in
      // s_cnt (cursor) and a copy in the tail of s_long's space is not
      // available, so sub-bins are re-derived from the cursor after scatter.
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int i = tid + j * THREADS;
        if (i < len) {
          const uint32_t p = lo + atomicAdd(s_cnt + lb[j], 1u);
          s_key[p] = lk[j];
          s_idx[p] = lx[j];
        }
      }
      __syncthreads();
      // after the scatter s_cnt[b] = end of sub-bin b; sub-bin b = [end[b-1], end[b])
      for (int b = tid; b < NBINS; b += THREADS) {
        const int e = (int)s_cnt[b];
        const int st = b ? (int)s_cnt[b - 1] : 0;
        if (e - st > 1) sort_small_bin(s_key, s_idx, lo + st, lo + e, bucket, a.key64);
      }
      __syncthreads();
    }
    // write ids in order
    for (int i = tid; i < n; i += THREADS) a.sorted_ids[r.x + i] = bucket[s_idx[i]];
    __syncthreads();
  }
}

template <int THREADS, int CAP, int NBINS>
constexpr size_t tile_sort_smem() {
  return 6 * (size_t)CAP + 8 * (size_t)(NBINS + 1) + 2 * (size_t)NBINS + 16;
}

// ---------------------------------------------------------------------------
// global path for oversized buckets

__global__ void k_big_gather(TileSortArgs a, const uint32_t* big_list, int n_big,
                             const uint32_t* big_off, uint64_t* keys, uint32_t* vals) {
  for (int b = blockIdx.x; b < n_big; b += gridDim.x) {
    const int t = (int)big_list[b];
    const int2 r = a.ranges[t];
    const uint32_t o = big_off[b];
    for (int i = threadIdx.x; i < r.y - r.x; i += blockDim.x) {
      const uint32_t id = a.bucket[r.x + i];
      keys[o + i] = ((uint64_t)b << 32) | a.key32[id];
      vals[o + i] = id;
    }
  }
}

__global__ void k_big_fixup(void* const* keys_ptr, void* const* vals_ptr, int64_t n,
                            const uint64_t* __restrict__ key64) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t* keys = static_cast<const uint64_t*>(*keys_ptr);
  uint32_t* vals = static_cast<uint32_t*>(*vals_ptr);
  const uint64_t k = keys[i];
  if (i > 0 && keys[i - 1] == k) return;
  if (i + 1 >= n || keys[i + 1] != k) return;
  int64_t len = 2;
  while (i + len < n && keys[i + len] == k) ++len;
  fix_run(vals + i, (int)len, key64);
}

__global__ void k_big_scatter(TileSortArgs a, const uint32_t* big_list, int n_big,
                              const uint32_t* big_off, void* const* vals_ptr) {
  const uint32_t* vals = static_cast<const uint32_t*>(*vals_ptr);
  for (int b = blockIdx.x; b < n_big; b += gridDim.x) {
    const int t = (int)big_list[b];
    const int2 r = a.ranges[t];
    const uint32_t o = big_off[b];
    for (int i = threadIdx.x; i < r.y - r.x; i += blockDim.x) a.sorted_ids[r.x + i] = vals[o + i];
  }
}

// instance export: keys = tile << 32 | row, prims = original id
__global__ void k_export(InstanceExportArgs a) {
  const int t = blockIdx.x;
  const int2 r = a.ranges[t];
  for (int i = r.x + threadIdx.x; i < r.y; i += blockDim.x) {
    const uint32_t id = a.sorted_ids[i];
    if (a.keys_out) a.keys_out[i] = ((uint64_t)(uint32_t)t << 32) | id;
    if (a.prims_out) a.prims_out[i] = a.prim_ids ? a.prim_ids[id] : (int64_t)id;
  }
}

template <typename Kern>
void set_smem(Kern k, size_t bytes) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

size_t bin_smem_bytes(int tiles) { return sizeof(uint32_t) * (size_t)min(tiles, kSlabTiles); }

void launch_bin_hist(const BinArgs& a, cudaStream_t s) {
  const size_t smem = bin_smem_bytes(a.tiles);
  static size_t set = 0;
  if (smem > set) {
    set_smem(k_bin_hist, bin_smem_bytes(kSlabTiles));
    set_smem(k_bin_place, bin_smem_bytes(kSlabTiles));
    set = bin_smem_bytes(kSlabTiles);
  }
  k_bin_hist<<<a.ctas, kBinThreads, smem, s>>>(a);
  k_bin_colscan<<<(a.tiles + 127) / 128, 128, 0, s>>>(a);
}

void launch_scan_tiles(const TileScanArgs& a, cudaStream_t s) {
  k_scan_tiles<<<1, kScanTilesThreads, 0, s>>>(a);
}

void launch_bin_place(const BinArgs& a, cudaStream_t s) {
  k_bin_place<<<a.ctas, kBinThreads, bin_smem_bytes(a.tiles), s>>>(a);
}

void launch_tile_sort(const TileSortArgs& a, const uint32_t* tile_list,
                      const uint32_t* list_count, int n_list, int cls, cudaStream_t s) {
  if (n_list <= 0) return;
  constexpr int kST = 256, kMT = 1024, kSB = 1024, kMB = 4096;
  static bool attr = false;
  if (!attr) {
    set_smem(k_tile_sort<kST, kSmallTileCap, kSB>, tile_sort_smem<kST, kSmallTileCap, kSB>());
    set_smem(k_tile_sort<kMT, kMediumTileCap, kMB>, tile_sort_smem<kMT, kMediumTileCap, kMB>());
    attr = true;
  }
  if (cls == 0)
    k_tile_sort<kST, kSmallTileCap, kSB>
        <<<n_list, kST, tile_sort_smem<kST, kSmallTileCap, kSB>(), s>>>(a, tile_list, list_count);
  else
    k_tile_sort<kMT, kMediumTileCap, kMB>
        <<<n_list, kMT, tile_sort_smem<kMT, kMediumTileCap, kMB>(), s>>>(a, tile_list, list_count);
}

void launch_big_gather(const TileSortArgs& a, const uint32_t* big_list, int n_big,
                       const uint32_t* big_off, uint64_t* keys, uint32_t* vals, cudaStream_t s) {
  if (n_big <= 0) return;
  k_big_gather<<<n_big, 256, 0, s>>>(a, big_list, n_big, big_off, keys, vals);
}

void launch_big_fixup(void* const* keys_ptr, void* const* vals_ptr, int64_t n,
                      const uint64_t* key64, cudaStream_t s) {
  if (n <= 0) return;
  k_big_fixup<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(keys_ptr, vals_ptr, n, key64);
}

void launch_big_scatter(const TileSortArgs& a, const uint32_t* big_list, int n_big,
                        const uint32_t* big_off, void* const* vals_ptr, cudaStream_t s) {
  if (n_big <= 0) return;
  k_big_scatter<<<n_big, 256, 0, s>>>(a, big_list, n_big, big_off, vals_ptr);
}

void launch_export_instances(const InstanceExportArgs& a, int tiles, cudaStream_t s) {
  if (tiles <= 0) return;
  k_export<<<tiles, 256, 0, s>>>(a);
}

}  // namespace lmgs
