// Device-wide LSD radix sort (onesweep).
//
// Two sorts per view:
//   K2  fp32 depth keys of all Gaussians with an implicit id payload (stable,
//       so equal keys stay in id order; runs of equal fp32 keys are then fixed
//       up by the exact fp64 depth — _sort_order, gaussian_core.py:277-283);
//   K5  the instance keys tile << 32 | id, sorted on the tile bits only
//       (stable: the emitted array is already in depth-rank order).
//
// Per sort: one histogram kernel computes every digit's global histogram in a
// single read; a 1-block plan kernel scans them, marks digits all keys share
// as trivial (skipped on the device) and routes the ping-pong buffers; then
// one onesweep kernel per digit: a tile of kSortTile keys is ranked in shared
// memory (warp match + per-warp counters, stable), staged in shared memory in
// digit order, its global digit offsets found by decoupled look-back over the
// preceding tiles, and written out in coalesced per-digit runs.
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagIncl = 2u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1;
constexpr int kWarps = kSortThreads / 32;
#ifndef LMGS_LOOK_WINDOW
#define LMGS_LOOK_WINDOW 8
#endif
constexpr int kLookWindow = LMGS_LOOK_WINDOW;

// Look-back status words carry their payload (flag | value) in one atomic
// word and publish nothing else, so relaxed gpu-scope accesses suffice; an
// acquire load would invalidate L1 (CCTL.IVALL) on every poll.
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// keys and values stream through each pass once: evict-first hints keep them
// from displacing the look-back words and the other streams' working sets
#ifdef LMGS_SORT_STREAMING
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) { return __ldcs(p); }
template <typename T>
__device__ __forceinline__ void st_stream(T* p, T v) { __stcs(p, v); }
#else
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) { return *p; }
template <typename T>
__device__ __forceinline__ void st_stream(T* p, T v) { *p = v; }
#endif

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, int shift) {
  return (uint32_t)((uint64_t)key >> shift) & 0xffu;
}

__device__ __forceinline__ bool gated_off(const int* gate) { return gate && *gate == 0; }

// ---------------------------------------------------------------------------
// histogram of every digit in one pass over the keys

template <typename K>
__global__ void __launch_bounds__(kSortThreads) k_radix_hist(const K* __restrict__ keys,
                                                             int64_t n, int begin_bit,
                                                             int n_passes, uint32_t* hist,
                                                             const int* gate) {
  if (gated_off(gate)) return;
  __shared__ uint32_t s_hist[kMaxPasses][kRadix];
  for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += blockDim.x) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = (uint64_t)keys[i] >> begin_bit;
    for (int p = 0; p < n_passes; ++p) atomicAdd(&s_hist[p][(k >> (8 * p)) & 0xff], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_passes * kRadix; i += blockDim.x) {
    const uint32_t v = (&s_hist[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

// one block of kRadix threads: scan each digit histogram, detect trivial
// passes, route buffers, publish where the result will land.
__global__ void __launch_bounds__(kRadix) k_radix_plan(const uint32_t* __restrict__ hist,
                                                       int64_t n, int n_passes, RadixPlan* plan,
                                                       const int* gate, void* keys0,
                                                       void* keys1, void* vals0, void* vals1,
                                                       void** keys_result, void** vals_result,
                                                       const unsigned long long* n_dev,
                                                       unsigned long long* max_n) {
  const bool off = gated_off(gate);
  if (n_dev) {
    if (max_n && threadIdx.x == 0) atomicMax(max_n, *n_dev);
    n = min(n, (int64_t)*n_dev);
  }
  __shared__ uint32_t s_scan[kRadix];
  __shared__ int s_trivial[kMaxPasses];
  const int d = threadIdx.x;
  if (!off) {
    for (int p = 0; p < n_passes; ++p) {
      const uint32_t c = hist[p * kRadix + d];
      if (d == 0) s_trivial[p] = 0;
      __syncthreads();
      if ((int64_t)c == n) s_trivial[p] = 1;
      s_scan[d] = c;
      __syncthreads();
      for (int o = 1; o < kRadix; o <<= 1) {
        const uint32_t v = d >= o ? s_scan[d - o] : 0;
        __syncthreads();
        s_scan[d] += v;
        __syncthreads();
      }
      plan->digit_start[p][d] = s_scan[d] - c;
      __syncthreads();
    }
  }
  if (d == 0) {
    int cur = 0, first = -1, last = -1;
    for (int p = 0; p < kMaxPasses; ++p) {
      const int act = !off && p < n_passes && !s_trivial[p] && n > 1;
      plan->active[p] = act;
      plan->src[p] = cur;
      if (act) {
        cur ^= 1;
        if (first < 0) first = p;
        last = p;
      }
    }
    plan->first_active = first;
    plan->last_active = last;
    plan->result = cur;
    plan->n_passes = n_passes;
    if (!off) {
      if (keys_result) *keys_result = cur ? keys1 : keys0;
      if (vals_result) *vals_result = cur ? vals1 : vals0;
    }
  }
}

// one onesweep scatter pass (digit `pass`)
//
// 1. load kSortTile keys (warp-striped, coalesced);
// 2. early counts: the CTA's digit histogram by shared atomics, published at
//    once to the look-back array so successors never wait on our ranking;
// 3. stable rank inside each warp: lanes holding the same digit find each other
//    through a per-warp shared "match" word (atomicOr of their lane bits, read
//    back, cleared by the lowest lane) — MATCH.ANY serialises on this part;
// 4. per-digit prefix over warps, staging in shared memory in digit order;
// 5. decoupled look-back (windowed) for the global digit offsets;
// 6. coalesced write-out in per-digit runs.
template <typename K, bool VALS, bool PERSIST>
__global__ void __launch_bounds__(kSortThreads, LMGS_SORT_MIN_CTAS) k_onesweep(
    K* keys0, K* keys1, uint32_t* vals0, uint32_t* vals1, int64_t n, int begin_bit, int pass,
    const RadixPlan* __restrict__ plan, uint32_t* lookback, uint32_t* counter, int64_t lb_stride,
    bool iota_vals, uint32_t* seg_counts, int seg_shift, const unsigned long long* n_dev) {
  if (n_dev) n = min(n, (int64_t)*n_dev);  // the grid covers an upper bound
  if (!plan->active[pass]) {
    // no pass moves data (every digit trivial): the result buffers are the
    // inputs, so pass 0 materialises the implicit payload and the single
    // segment instead of separate launches
    if (pass == 0 && plan->first_active < 0) {
      if (VALS && iota_vals)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
             i += (int64_t)gridDim.x * blockDim.x)
          vals0[i] = (uint32_t)i;
      if (seg_counts && blockIdx.x == 0 && threadIdx.x == 0 && n > 0)
        seg_counts[(uint64_t)keys0[0] >> seg_shift] = (uint32_t)n;
    }
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* s_keys = reinterpret_cast<K*>(smem_raw);  // [kSortTile] staging
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(smem_raw + sizeof(K) * kSortTile);
  __shared__ uint32_t s_match[kWarps][kRadix];
  __shared__ uint32_t s_wcnt[kWarps][kRadix];
  __shared__ uint32_t s_hist[kRadix];
  __shared__ uint32_t s_local_start[kRadix];
  __shared__ uint32_t s_global[kRadix];
  __shared__ uint32_t s_bid;
  __shared__ uint32_t s_wsum[kWarps];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // tiles are taken by ticket; a CTA loops until the keys run out (with n_dev
  // the grid is a persistent one sized for the device, not for the bound)
  for (;;) {
  if (tid == 0) s_bid = atomicAdd(counter + pass, 1u);
  __syncthreads();
  const uint32_t bid = s_bid;
  const int64_t base = (int64_t)bid * kSortTile;
  if (base >= n) return;
  const int count = (int)min((int64_t)kSortTile, n - base);
  const int src = plan->src[pass];
  const K* __restrict__ kin = src ? keys1 : keys0;
  K* __restrict__ kout = src ? keys0 : keys1;
  const uint32_t* __restrict__ vin = src ? vals1 : vals0;
  uint32_t* __restrict__ vout = src ? vals0 : vals1;
  // implicit payload on the first pass that moves data: value = input index
  const bool iota = iota_vals && pass == plan->first_active;
  const int shift = begin_bit + 8 * pass;

#ifdef LMGS_SORT_RELOAD
  // only the digits stay in registers (4 per word); keys and values are
  // re-read (L2) for the scatter, which frees ~40 registers per thread
  uint32_t dg[(kSortItems + 3) / 4];
  uint32_t pos[kSortItems];
  const int wbase = warp * 32 * kSortItems;
  {
    K key[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      const int i = wbase + j * 32 + lane;
      key[j] = i < count ? ld_stream(kin + base + i) : (K)~(K)0;
    }
#pragma unroll
    for (int q = 0; q < (kSortItems + 3) / 4; ++q) dg[q] = 0;
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) dg[j >> 2] |= digit_of(key[j], shift) << (8 * (j & 3));
  }
#define LMGS_DIGIT(j) ((dg[(j) >> 2] >> (8 * ((j) & 3))) & 0xffu)
#else
  K key[kSortItems];
  uint32_t val[VALS ? kSortItems : 1];
  uint32_t pos[kSortItems];
  const int wbase = warp * 32 * kSortItems;
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int i = wbase + j * 32 + lane;
    key[j] = i < count ? ld_stream(kin + base + i) : (K)~(K)0;
    if (VALS) val[j] = iota ? (uint32_t)(base + i) : (i < count ? ld_stream(vin + base + i) : 0u);
  }
#define LMGS_DIGIT(j) digit_of(key[j], shift)
#endif
  // the loads above are in flight while the ranking state is cleared
  for (int i = tid; i < kWarps * kRadix; i += kSortThreads) {
    (&s_match[0][0])[i] = 0;
    (&s_wcnt[0][0])[i] = 0;
  }
  s_hist[tid] = 0;  // kSortThreads == kRadix
  __syncthreads();
#if defined(LMGS_DBG_COPY) && !defined(LMGS_SORT_RELOAD)
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int i = wbase + j * 32 + lane;
    if (i < count) {
      kout[base + i] = key[j];
      if (VALS) vout[base + i] = val[j];
    }
  }
  if (!PERSIST) return;
  __syncthreads();
  continue;
#endif
  // 2. early counts, published with the look-back before ranking
#pragma unroll
  for (int j = 0; j < kSortItems; ++j)
    if (wbase + j * 32 + lane < count) atomicAdd(&s_hist[LMGS_DIGIT(j)], 1u);
  __syncthreads();
  uint32_t* lb = lookback + ((int64_t)pass * lb_stride) * kRadix;
  const uint32_t total = s_hist[tid];  // thread d == digit d
  {
    const int d = tid;
    if (bid == 0) st_release(lb + d, kFlagIncl | total);
    else st_release(lb + (int64_t)bid * kRadix + d, kFlagAgg | total);
    uint32_t incl = total;  // block-wide exclusive scan over digits
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) wpre += w < warp ? s_wsum[w] : 0;
    s_local_start[d] = wpre + incl - total;
    // decoupled look-back for this tile's global digit offsets, right after
    // the early counts so the inclusive prefix is published before ranking.
    // Each digit's thread reads a window of kLookWindow predecessors with
    // independent loads (one L2 round trip per window, not per predecessor),
    // then walks it from the nearest one, re-polling only unpublished entries.
    uint32_t excl = 0;
#ifdef LMGS_DBG_NO_LOOKBACK
    if (false) {
#else
    if (bid != 0) {
#endif
      int64_t look = (int64_t)bid - 1;
      bool done = false;
      while (!done) {
        uint32_t v[kLookWindow];
#pragma unroll
        for (int w = 0; w < kLookWindow; ++w)
          v[w] = look - w >= 0 ? ld_acquire(lb + (look - w) * kRadix + d) : kFlagIncl;
#pragma unroll
        for (int w = 0; w < kLookWindow; ++w) {
          if (done) break;
          while ((v[w] & ~kValueMask) == 0) v[w] = ld_acquire(lb + (look - w) * kRadix + d);
          excl += v[w] & kValueMask;
          done = (v[w] & ~kValueMask) == kFlagIncl;
        }
        look -= kLookWindow;
      }
      st_release(lb + (int64_t)bid * kRadix + d, kFlagIncl | (excl + total));
    }
    s_global[d] = plan->digit_start[pass][d] + excl - (wpre + incl - total);
  }
  // 3. stable in-warp ranking, items in (j, lane) order
  const uint32_t lt = lanemask_lt();
  uint32_t* my_match = s_match[warp];
  uint32_t* my_cnt = s_wcnt[warp];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const bool valid = wbase + j * 32 + lane < count;
    const uint32_t d = LMGS_DIGIT(j);
    if (valid) atomicOr(my_match + d, 1u << lane);
    __syncwarp();
    const uint32_t peers = valid ? my_match[d] : (1u << lane);
    __syncwarp();
    const int leader = __ffs(peers) - 1;
    uint32_t before = 0;
    if (valid && lane == leader) {
      before = my_cnt[d];
      my_cnt[d] = before + (uint32_t)__popc(peers);
      my_match[d] = 0;
    }
    before = __shfl_sync(0xffffffffu, before, leader);
    pos[j] = before + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  // 4. per digit: exclusive prefix over warps
  {
    const int d = tid;
    uint32_t run = s_local_start[d];
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = s_wcnt[w][d];
      s_wcnt[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int i = wbase + j * 32 + lane;
    if (i < count) {
      const uint32_t p = pos[j] + my_cnt[LMGS_DIGIT(j)];
#ifdef LMGS_SORT_RELOAD
      s_keys[p] = kin[base + i];
      if (VALS) s_vals[p] = iota ? (uint32_t)(base + i) : vin[base + i];
#else
      s_keys[p] = key[j];
      if (VALS) s_vals[p] = val[j];
#endif
    }
  }
#undef LMGS_DIGIT
  __syncthreads();
  // 6. coalesced write-out: consecutive threads, consecutive staged positions
  const bool segs = seg_counts && pass == plan->last_active;
  for (int i = tid; i < count; i += kSortThreads) {
    const K k = s_keys[i];
    const uint32_t o = s_global[digit_of(k, shift)] + i;
    st_stream(kout + o, k);
    if (VALS) st_stream(vout + o, s_vals[i]);
    if (segs) {
      // the staged tile is sorted on every key bit sorted so far: runs of one
      // segment are contiguous; a run [i0, i1] adds (i1 + 1) - i0
      const uint64_t sg = (uint64_t)k >> seg_shift;
      if (i == 0 || ((uint64_t)s_keys[i - 1] >> seg_shift) != sg)
        atomicAdd(seg_counts + sg, (uint32_t)(-i));
      if (i + 1 == count || ((uint64_t)s_keys[i + 1] >> seg_shift) != sg)
        atomicAdd(seg_counts + sg, (uint32_t)(i + 1));
    }
  }
  if (!PERSIST) return;  // one tile per CTA on an exact grid
  __syncthreads();  // the staging and s_bid are reused by the next tile
  }
}

template <typename K, bool VALS>
constexpr size_t onesweep_smem() {
  return sizeof(K) * kSortTile + (VALS ? sizeof(uint32_t) * kSortTile : 0);
}

template <typename K, bool VALS, bool PERSIST>
void launch_onesweep_as(const RadixSortBuffers& b, int64_t n, int begin_bit, int p, int64_t grid,
                        int64_t blocks, cudaStream_t s) {
  constexpr size_t smem = onesweep_smem<K, VALS>();
  k_onesweep<K, VALS, PERSIST><<<(unsigned)grid, kSortThreads, smem, s>>>(
      static_cast<K*>(b.keys[0]), static_cast<K*>(b.keys[1]), b.vals[0], b.vals[1], n, begin_bit,
      p, b.plan, b.lookback, b.counters, blocks, b.iota_vals, b.seg_counts, b.seg_shift, b.n_dev);
}

template <typename K, bool VALS>
void launch_onesweep(const RadixSortBuffers& b, int64_t n, int begin_bit, int p, int64_t blocks,
                     cudaStream_t s) {
  constexpr size_t smem = onesweep_smem<K, VALS>();
  static bool attr_set[kMaxDevices] = {};
  static int occ[kMaxDevices] = {}, sms[kMaxDevices] = {};
  const int dev = current_device();
  if (!attr_set[dev]) {
    cudaFuncSetAttribute(k_onesweep<K, VALS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaFuncSetAttribute(k_onesweep<K, VALS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[dev], k_onesweep<K, VALS, true>,
                                                  kSortThreads, smem);
    if (occ[dev] < 1) occ[dev] = 1;
    attr_set[dev] = true;
  }
  if (!b.n_dev) {
    launch_onesweep_as<K, VALS, false>(b, n, begin_bit, p, blocks, blocks, s);
    return;
  }
  // the key count is on the device: a persistent grid takes tiles by ticket
  const int64_t persistent = (int64_t)sms[dev] * occ[dev];
  launch_onesweep_as<K, VALS, true>(b, n, begin_bit, p, blocks < persistent ? blocks : persistent,
                                    blocks, s);
}

template <typename K>
int radix_sort_impl(const RadixSortBuffers& b, int64_t n, int begin_bit, int n_passes,
                    cudaStream_t s) {
  int launched = 0;
  if (n_passes > kMaxPasses) n_passes = kMaxPasses;
  const int64_t blocks = (n + kSortTile - 1) / kSortTile;
  if (!b.hist_ready) cudaMemsetAsync(b.hist, 0, sizeof(uint32_t) * kMaxPasses * kRadix, s);
  cudaMemsetAsync(b.counters, 0, sizeof(uint32_t) * kMaxPasses, s);
  if (blocks > 0 && n_passes > 0)
    cudaMemsetAsync(b.lookback, 0, sizeof(uint32_t) * (size_t)n_passes * blocks * kRadix, s);
  K* k0 = static_cast<K*>(b.keys[0]);
  K* k1 = static_cast<K*>(b.keys[1]);
  if (n > 0 && n_passes > 0 && !b.hist_ready) {
    int hist_blocks = (int)((n + kSortThreads * 16 - 1) / (kSortThreads * 16));
    if (hist_blocks > 148 * 4) hist_blocks = 148 * 4;
    k_radix_hist<K><<<hist_blocks, kSortThreads, 0, s>>>(k0, n, begin_bit, n_passes, b.hist,
                                                         b.gate);
    ++launched;
  }
  k_radix_plan<<<1, kRadix, 0, s>>>(b.hist, n, n_passes, b.plan, b.gate, k0, k1, b.vals[0],
                                    b.vals[1], b.keys_result, b.vals_result, b.n_dev, b.max_n);
  ++launched;
  if (blocks == 0) return launched;
  for (int p = 0; p < n_passes; ++p) {
    if (b.vals[1]) launch_onesweep<K, true>(b, n, begin_bit, p, blocks, s);
    else launch_onesweep<K, false>(b, n, begin_bit, p, blocks, s);
  }
  return launched + n_passes;
}

}  // namespace

size_t radix_lookback_words(int64_t capacity) {
  const int64_t blocks = (capacity + kSortTile - 1) / kSortTile;
  return (size_t)kMaxPasses * (size_t)(blocks > 0 ? blocks : 1) * kRadix;
}

int radix_sort(const RadixSortBuffers& b, int64_t n, int begin_bit, int n_passes,
               cudaStream_t s) {
  if (b.key_bytes == 4) return radix_sort_impl<uint32_t>(b, n, begin_bit, n_passes, s);
  return radix_sort_impl<uint64_t>(b, n, begin_bit, n_passes, s);
}

}  // namespace lmgs
