// Device-wide LSD radix sort (onesweep) and a single-pass exclusive scan.
//
// Used twice per view:
//   K2  depth_rank_sort: (fp64 depth bits, id) pairs, all 64 bits, so equal
//       depths keep ascending id order — np.lexsort((prim_id, depth)) of
//       _sort_order (gaussian_core.py:277-283) over all near-kept splats;
//   K5  tile sort: keys (tile << 32 | rank) stably by the tile bits only,
//       which turns the rank-ordered instance stream into per-tile lists in
//       (depth, id) order — the per-tile _sort_order call of rasterize (392).
//
// Structure per sort: one histogram kernel computes every digit's global
// histogram in a single read of the keys; a 1-block plan kernel scans them,
// marks digits that all keys share as trivial, and routes the ping-pong
// buffers; then one scatter kernel per digit ranks a 4096-key tile in shared
// memory (warp match + per-warp counters, stable) and finds its global
// offsets with decoupled look-back over the preceding tiles.
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagIncl = 2u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1;
constexpr int kWarps = kSortThreads / 32;

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------------------
// histogram of every digit in one pass over the keys

__global__ void __launch_bounds__(kSortThreads) k_radix_hist(const uint64_t* __restrict__ keys,
                                                             int64_t n, int begin_bit,
                                                             int n_passes, uint32_t* hist) {
  __shared__ uint32_t s_hist[kMaxPasses][kRadix];
  for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += blockDim.x) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = keys[i] >> begin_bit;
    for (int p = 0; p < n_passes; ++p) atomicAdd(&s_hist[p][(k >> (8 * p)) & 0xff], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_passes * kRadix; i += blockDim.x) {
    const uint32_t v = (&s_hist[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

// one block of kRadix threads: scan each digit histogram, detect trivial passes
__global__ void __launch_bounds__(kRadix) k_radix_plan(const uint32_t* __restrict__ hist,
                                                       int64_t n, int n_passes, RadixPlan* plan) {
  __shared__ uint32_t s_scan[kRadix];
  __shared__ int s_trivial[kMaxPasses];
  const int d = threadIdx.x;
  for (int p = 0; p < n_passes; ++p) {
    const uint32_t c = hist[p * kRadix + d];
    if (d == 0) s_trivial[p] = 0;
    __syncthreads();
    if ((int64_t)c == n) s_trivial[p] = 1;
    s_scan[d] = c;
    __syncthreads();
    for (int off = 1; off < kRadix; off <<= 1) {
      const uint32_t v = d >= off ? s_scan[d - off] : 0;
      __syncthreads();
      s_scan[d] += v;
      __syncthreads();
    }
    plan->digit_start[p][d] = s_scan[d] - c;
    __syncthreads();
  }
  if (d == 0) {
    int cur = 0;
    for (int p = 0; p < kMaxPasses; ++p) {
      const int act = p < n_passes && !s_trivial[p] && n > 1;
      plan->active[p] = act;
      plan->src[p] = cur;
      if (act) cur ^= 1;
    }
    plan->result = cur;
    plan->n_passes = n_passes;
  }
}

// one scatter pass (digit p)
__global__ void __launch_bounds__(kSortThreads) k_radix_pass(
    uint64_t* keys0, uint64_t* keys1, uint32_t* vals0, uint32_t* vals1, int64_t n, int begin_bit,
    int pass, const RadixPlan* __restrict__ plan, uint32_t* lookback, uint32_t* counter,
    int64_t lb_stride) {
  if (!plan->active[pass]) return;
  __shared__ uint32_t s_warp_cnt[kWarps][kRadix];
  __shared__ uint32_t s_base[kRadix];
  __shared__ uint32_t s_bid;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_bid = atomicAdd(counter + pass, 1u);
  for (int i = tid; i < kWarps * kRadix; i += kSortThreads) (&s_warp_cnt[0][0])[i] = 0;
  __syncthreads();
  const uint32_t bid = s_bid;
  const int64_t base = (int64_t)bid * kSortTile;
  if (base >= n) return;
  const int src = plan->src[pass];
  const uint64_t* __restrict__ kin = src ? keys1 : keys0;
  uint64_t* __restrict__ kout = src ? keys0 : keys1;
  const uint32_t* __restrict__ vin = src ? vals1 : vals0;
  uint32_t* __restrict__ vout = src ? vals0 : vals1;
  const bool has_vals = vals0 != nullptr;
  const int shift = begin_bit + 8 * pass;

  uint64_t key[kSortItems];
  uint32_t val[kSortItems];
  uint32_t rank[kSortItems];
  const int64_t wbase = base + (int64_t)warp * 32 * kSortItems;
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t idx = wbase + j * 32 + lane;
    key[j] = idx < n ? kin[idx] : ~0ull;
    if (has_vals) val[j] = idx < n ? vin[idx] : 0u;
  }
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t idx = wbase + j * 32 + lane;
    const bool valid = idx < n;
    const uint32_t d = (uint32_t)(key[j] >> shift) & 0xffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, valid ? d : 256u + lane);
    const uint32_t before = s_warp_cnt[warp][d];
    rank[j] = before + __popc(peers & lt);
    __syncwarp();
    if (valid && (peers & lt) == 0) s_warp_cnt[warp][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive prefix over warps, block total, look-back
  {
    const int d = tid;  // kSortThreads == kRadix
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = s_warp_cnt[w][d];
      s_warp_cnt[w][d] = run;
      run += c;
    }
    uint32_t* lb = lookback + ((int64_t)pass * lb_stride) * kRadix;
    uint32_t excl = 0;
    if (bid == 0) {
      st_release(lb + d, kFlagIncl | run);
    } else {
      st_release(lb + (int64_t)bid * kRadix + d, kFlagAgg | run);
      int64_t look = (int64_t)bid - 1;
      while (true) {
        uint32_t v;
        do {
          v = ld_acquire(lb + look * kRadix + d);
        } while ((v & ~kValueMask) == 0);
        excl += v & kValueMask;
        if ((v & ~kValueMask) == kFlagIncl) break;
        --look;
      }
      st_release(lb + (int64_t)bid * kRadix + d, kFlagIncl | (excl + run));
    }
    s_base[d] = plan->digit_start[pass][d] + excl;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t idx = wbase + j * 32 + lane;
    if (idx < n) {
      const uint32_t d = (uint32_t)(key[j] >> shift) & 0xffu;
      const uint32_t pos = s_base[d] + s_warp_cnt[warp][d] + rank[j];
      kout[pos] = key[j];
      if (has_vals) vout[pos] = val[j];
    }
  }
}

// ---------------------------------------------------------------------------
// exclusive scan of counts[perm[r]] (decoupled look-back, u64 status words)

constexpr unsigned long long kScanAgg = 1ull << 62;
constexpr unsigned long long kScanIncl = 2ull << 62;
constexpr unsigned long long kScanMask = (1ull << 62) - 1;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads) k_scan(const uint32_t* __restrict__ counts,
                                                       const uint32_t* perm_a,
                                                       const uint32_t* perm_b,
                                                       const RadixPlan* plan, int64_t n,
                                                       uint64_t* __restrict__ offsets,
                                                       uint64_t* total,
                                                       unsigned long long* status,
                                                       uint32_t* counter) {
  __shared__ uint32_t s_bid;
  __shared__ unsigned long long s_warp[kScanThreads / 32];
  __shared__ unsigned long long s_excl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_bid = atomicAdd(counter, 1u);
  __syncthreads();
  const uint32_t bid = s_bid;
  const int64_t base = (int64_t)bid * kScanTile + (int64_t)tid * kScanItems;
  const uint32_t* perm = perm_a ? ((plan && plan->result) ? perm_b : perm_a) : nullptr;
  uint32_t v[kScanItems];
  unsigned long long local = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t r = base + j;
    uint32_t c = 0;
    if (r < n) c = counts[perm ? perm[r] : r];
    v[j] = c;
    local += c;
  }
  // block exclusive scan of per-thread sums
  unsigned long long incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long wv = lane < kScanThreads / 32 ? s_warp[lane] : 0;
    unsigned long long wi = wv;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += o;
    }
    if (lane < kScanThreads / 32) s_warp[lane] = wi - wv;  // exclusive warp prefix
    const unsigned long long block_total = __shfl_sync(0xffffffffu, wi, kScanThreads / 32 - 1);
    if (lane == 0) {
      unsigned long long excl = 0;
      if (bid == 0) {
        st_release64(status, kScanIncl | block_total);
      } else {
        st_release64(status + bid, kScanAgg | block_total);
        int64_t look = (int64_t)bid - 1;
        while (true) {
          unsigned long long s;
          do {
            s = ld_acquire64(status + look);
          } while ((s & ~kScanMask) == 0);
          excl += s & kScanMask;
          if ((s & ~kScanMask) == kScanIncl) break;
          --look;
        }
        st_release64(status + bid, kScanIncl | (excl + block_total));
      }
      s_excl = excl;
      const int64_t nblocks = (n + kScanTile - 1) / kScanTile;
      if ((int64_t)bid == nblocks - 1) *total = excl + block_total;
    }
  }
  __syncthreads();
  unsigned long long run = s_excl + s_warp[warp] + (incl - local);
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t r = base + j;
    if (r < n) offsets[r] = run;
    run += v[j];
  }
}

}  // namespace

size_t radix_lookback_words(int64_t capacity) {
  const int64_t blocks = (capacity + kSortTile - 1) / kSortTile;
  return (size_t)kMaxPasses * (size_t)(blocks > 0 ? blocks : 1) * kRadix;
}

void radix_sort(const RadixSortBuffers& b, int64_t n, int begin_bit, int n_passes,
                cudaStream_t s) {
  if (n_passes > kMaxPasses) n_passes = kMaxPasses;
  const int64_t blocks = (n + kSortTile - 1) / kSortTile;
  cudaMemsetAsync(b.hist, 0, sizeof(uint32_t) * kMaxPasses * kRadix, s);
  cudaMemsetAsync(b.counters, 0, sizeof(uint32_t) * kMaxPasses, s);
  if (blocks > 0 && n_passes > 0)
    cudaMemsetAsync(b.lookback, 0, sizeof(uint32_t) * (size_t)n_passes * blocks * kRadix, s);
  if (n > 0) {
    int hist_blocks = (int)((n + kSortThreads * 8 - 1) / (kSortThreads * 8));
    if (hist_blocks > 148 * 8) hist_blocks = 148 * 8;
    k_radix_hist<<<hist_blocks, kSortThreads, 0, s>>>(b.keys[0], n, begin_bit, n_passes, b.hist);
  }
  k_radix_plan<<<1, kRadix, 0, s>>>(b.hist, n, n_passes, b.plan);
  if (blocks == 0) return;
  for (int p = 0; p < n_passes; ++p)
    k_radix_pass<<<(unsigned)blocks, kSortThreads, 0, s>>>(b.keys[0], b.keys[1], b.vals[0],
                                                           b.vals[1], n, begin_bit, p, b.plan,
                                                           b.lookback, b.counters, blocks);
}

size_t scan_status_words(int64_t n) {
  const int64_t blocks = (n + kScanTile - 1) / kScanTile;
  return (size_t)(blocks > 0 ? blocks : 1);
}

void scan_counts(const uint32_t* counts, const uint32_t* perm_a, const uint32_t* perm_b,
                 const RadixPlan* plan, int64_t n, uint64_t* offsets, uint64_t* total,
                 unsigned long long* status, uint32_t* counter, cudaStream_t s) {
  const int64_t blocks = (n + kScanTile - 1) / kScanTile;
  cudaMemsetAsync(counter, 0, sizeof(uint32_t), s);
  if (blocks == 0) {
    cudaMemsetAsync(total, 0, sizeof(uint64_t), s);
    return;
  }
  cudaMemsetAsync(status, 0, sizeof(unsigned long long) * blocks, s);
  k_scan<<<(unsigned)blocks, kScanThreads, 0, s>>>(counts, perm_a, perm_b, plan, n, offsets,
                                                   total, status, counter);
}

}  // namespace lmgs
