// Device-wide LSD radix sort (onesweep).
//
// Two sorts per view:
//   K2  fp32 depth keys of all Gaussians with an implicit id payload (stable,
//       so equal keys stay in id order; runs of equal fp32 keys are then fixed
//       up by the exact fp64 depth — _sort_order, gaussian_core.py:277-283);
//   K5  the instance keys tile << 32 | id, sorted on the tile bits only
//       (stable: the emitted array is already in depth-rank order).  The last
//       pass writes the 32-bit ids alone, which is all the blend reads
//       (tile_sort below).
//
// Per sort: one histogram kernel computes every digit's global histogram in a
// single read (for K2 and K5 the producer builds it); a 1-block plan kernel
// scans them, marks digits all keys share as trivial (skipped on the device;
// not for K5, whose passes change the key format) and routes the ping-pong
// buffers; then one onesweep kernel per digit: a tile of kSortTile keys is
// ranked in shared memory (warp match + per-warp counters, stable), staged in
// shared memory in digit order, its global digit offsets found by decoupled
// look-back over the preceding tiles, and written out in coalesced per-digit
// runs.
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
#ifndef LMGS_RANK_MODE
#define LMGS_RANK_MODE 2
#endif
#ifndef LMGS_RANK_GROUP
#define LMGS_RANK_GROUP 1  // 1: 752 vs 745 frames/s at 2 (less shared memory; profiles/r07/rank_group_ab.txt)
#endif
constexpr int kMatchBufs = LMGS_RANK_MODE == 2 ? LMGS_RANK_GROUP : 1;
#ifndef LMGS_SORT_MIN_CTAS_NARROW
#define LMGS_SORT_MIN_CTAS_NARROW 4  // 32-bit keys without values: fewer registers
#endif

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
// passes (unless every pass must run), route buffers, publish where the
// result will land.
__global__ void __launch_bounds__(kRadix) k_radix_plan(const uint32_t* __restrict__ hist,
                                                       int64_t n, int n_passes, RadixPlan* plan,
                                                       const int* gate, void* keys0,
                                                       void* keys1, void* vals0, void* vals1,
                                                       void** keys_result, void** vals_result,
                                                       const unsigned long long* n_dev,
                                                       unsigned long long* max_n, bool force_all) {
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
      const int act =
          !off && p < n_passes && (force_all ? n >= 1 : (!s_trivial[p] && n > 1));
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

// Output format of a pass and how its last pass counts tile runs.
enum : int { kOutSame = 0, kOutIds = 1 };
enum : int { kSegNone = 0, kSegKey = 1 };

struct PassArgs {
  void* keys[2];  // ping-pong buffers, each large enough for n keys of the wider format
  uint32_t* vals[2];
  int64_t n;
  int shift;  // this pass's digit = (key >> shift) & 0xff
  int pass;
  const RadixPlan* plan;
  uint32_t* lookback;
  uint32_t* counter;
  int64_t lb_stride;
  bool iota_vals;
  uint32_t id_mask;  // kOutIds: out = key & id_mask
  uint32_t* seg_counts;
  int seg_shift;  // kSegKey: segment = key >> seg_shift
  const unsigned long long* n_dev;
};

template <typename KI, int OUT>
struct OutKey {
  using type = KI;
};
template <typename KI>
struct OutKey<KI, kOutIds> {
  using type = uint32_t;
};

template <typename KI, int OUT>
__device__ __forceinline__ typename OutKey<KI, OUT>::type out_key(KI k, const PassArgs& a) {
  if constexpr (OUT == kOutIds)
    return (uint32_t)k & a.id_mask;
  else
    return k;
}

template <typename KI, bool VALS>
constexpr int sort_min_ctas() {
  return (sizeof(KI) == 4 && !VALS) ? LMGS_SORT_MIN_CTAS_NARROW : LMGS_SORT_MIN_CTAS;
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
// 6. coalesced write-out in per-digit runs, in the pass's output format.
template <typename KI, int OUT, int SEG, bool VALS, bool PERSIST>
__global__ void __launch_bounds__(kSortThreads, (sort_min_ctas<KI, VALS>()))
    k_onesweep(PassArgs a) {
  using KO = typename OutKey<KI, OUT>::type;
  int64_t n = a.n;
  if (a.n_dev) n = min(n, (int64_t)*a.n_dev);  // the grid covers an upper bound
  const RadixPlan* __restrict__ plan = a.plan;
  const int pass = a.pass;
  if (!plan->active[pass]) {
    // no pass moves data (every digit trivial): the result buffers are the
    // inputs, so pass 0 materialises the implicit payload and the single
    // segment instead of separate launches (formats never change here: only
    // sorts whose passes may be skipped get here)
    if (pass == 0 && plan->first_active < 0) {
      if (VALS && a.iota_vals)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
             i += (int64_t)gridDim.x * blockDim.x)
          a.vals[0][i] = (uint32_t)i;
      if (SEG == kSegKey && a.seg_counts && blockIdx.x == 0 && threadIdx.x == 0 && n > 0)
        a.seg_counts[(uint64_t) static_cast<const KI*>(a.keys[0])[0] >> a.seg_shift] =
            (uint32_t)n;
    }
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KI* s_keys = reinterpret_cast<KI*>(smem_raw);  // [kSortTile] staging
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(smem_raw + sizeof(KI) * kSortTile);
  __shared__ uint32_t s_match[kMatchBufs][kWarps][kRadix];
  __shared__ uint32_t s_wcnt[kWarps][kRadix];
  __shared__ uint32_t s_hist[kRadix];
  __shared__ uint32_t s_local_start[kRadix];
  __shared__ uint32_t s_global[kRadix];
  __shared__ uint32_t s_bid;
  __shared__ uint32_t s_wsum[kWarps];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int src = plan->src[pass];
  // selects, not a.keys[src]: a dynamically indexed parameter goes to the stack
  const KI* __restrict__ kin = static_cast<const KI*>(src ? a.keys[1] : a.keys[0]);
  KO* __restrict__ kout = static_cast<KO*>(src ? a.keys[0] : a.keys[1]);
  const uint32_t* __restrict__ vin = src ? a.vals[1] : a.vals[0];
  uint32_t* __restrict__ vout = src ? a.vals[0] : a.vals[1];
  // implicit payload on the first pass that moves data: value = input index
  const bool iota = a.iota_vals && pass == plan->first_active;
  const int shift = a.shift;
  // tiles are taken by ticket; a CTA loops until the keys run out (with n_dev
  // the grid is a persistent one sized for the device, not for the bound)
  for (;;) {
  if (tid == 0) s_bid = atomicAdd(a.counter + pass, 1u);
  __syncthreads();
  const uint32_t bid = s_bid;
  const int64_t base = (int64_t)bid * kSortTile;
  if (base >= n) return;
  const int count = (int)min((int64_t)kSortTile, n - base);

  KI key[kSortItems];
  uint32_t val[VALS ? kSortItems : 1];
  uint32_t pos[kSortItems];
  const int wbase = warp * 32 * kSortItems;
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int i = wbase + j * 32 + lane;
    key[j] = i < count ? kin[base + i] : (KI)~(KI)0;
    if (VALS) val[j] = iota ? (uint32_t)(base + i) : (i < count ? vin[base + i] : 0u);
  }
  // the loads above are in flight while the ranking state is cleared
  for (int i = tid; i < kWarps * kRadix; i += kSortThreads) {
#pragma unroll
    for (int r = 0; r < kMatchBufs; ++r) (&s_match[r][0][0])[i] = 0;
    (&s_wcnt[0][0])[i] = 0;
  }
  s_hist[tid] = 0;  // kSortThreads == kRadix
  __syncthreads();
  // 2. early counts, published with the look-back before ranking
#pragma unroll
  for (int j = 0; j < kSortItems; ++j)
    if (wbase + j * 32 + lane < count) atomicAdd(&s_hist[digit_of(key[j], shift)], 1u);
  __syncthreads();
  uint32_t* lb = a.lookback + ((int64_t)pass * a.lb_stride) * kRadix;
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
    if (bid != 0) {
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
  uint32_t* my_cnt = s_wcnt[warp];
#if LMGS_RANK_MODE == 1
  // peers by MATCH.ANY; the leader advances the warp's digit counter
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const bool valid = wbase + j * 32 + lane < count;
    const uint32_t d = digit_of(key[j], shift);
    const uint32_t peers = __match_any_sync(0xffffffffu, valid ? d : 256u + lane);
    const int leader = __ffs(peers) - 1;
    uint32_t before = 0;
    if (valid && lane == leader) {
      before = my_cnt[d];
      my_cnt[d] = before + (uint32_t)__popc(peers);
    }
    before = __shfl_sync(0xffffffffu, before, leader);
    pos[j] = before + __popc(peers & lt);
    __syncwarp();
  }
#elif LMGS_RANK_MODE == 2
  // LMGS_RANK_GROUP items at a time, each with its own match words, so their
  // shared-memory round trips overlap; the leaders' counter updates are
  // atomics issued in item order by the one warp
#pragma unroll
  for (int j0 = 0; j0 < kSortItems; j0 += LMGS_RANK_GROUP) {
    uint32_t peers[LMGS_RANK_GROUP];
#pragma unroll
    for (int r = 0; r < LMGS_RANK_GROUP; ++r) {
      const int j = j0 + r;
      if (wbase + j * 32 + lane < count) atomicOr(&s_match[r][warp][digit_of(key[j], shift)], 1u << lane);
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < LMGS_RANK_GROUP; ++r) {
      const int j = j0 + r;
      const bool valid = wbase + j * 32 + lane < count;
      peers[r] = valid ? s_match[r][warp][digit_of(key[j], shift)] : (1u << lane);
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < LMGS_RANK_GROUP; ++r) {
      const int j = j0 + r;
      const bool valid = wbase + j * 32 + lane < count;
      const uint32_t d = digit_of(key[j], shift);
      const int leader = __ffs(peers[r]) - 1;
      uint32_t before = 0;
      if (valid && lane == leader) {
        before = atomicAdd(my_cnt + d, (uint32_t)__popc(peers[r]));
        s_match[r][warp][d] = 0;
      }
      before = __shfl_sync(0xffffffffu, before, leader);
      pos[j] = before + __popc(peers[r] & lt);
    }
    __syncwarp();
  }
#else
  uint32_t* my_match = s_match[0][warp];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const bool valid = wbase + j * 32 + lane < count;
    const uint32_t d = digit_of(key[j], shift);
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
#endif
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
      const uint32_t p = pos[j] + my_cnt[digit_of(key[j], shift)];
      s_keys[p] = key[j];
      if (VALS) s_vals[p] = val[j];
    }
  }
  __syncthreads();
  // 6. coalesced write-out: consecutive threads, consecutive staged positions
  const bool segs = SEG != kSegNone && a.seg_counts && pass == plan->last_active;
  for (int i = tid; i < count; i += kSortThreads) {
    const KI k = s_keys[i];
    const uint32_t o = s_global[digit_of(k, shift)] + i;
    kout[o] = out_key<KI, OUT>(k, a);
    if (VALS) vout[o] = s_vals[i];
    if (segs) {
      // the staged tile is sorted on every key bit sorted so far: runs of one
      // segment are contiguous; a run [i0, i1] adds (i1 + 1) - i0
      const uint64_t sg = (uint64_t)k >> a.seg_shift;
      const uint64_t sp = i > 0 ? (uint64_t)s_keys[i - 1] >> a.seg_shift : ~0ull;
      const uint64_t sn = i + 1 < count ? (uint64_t)s_keys[i + 1] >> a.seg_shift : ~0ull;
      if (sp != sg) atomicAdd(a.seg_counts + sg, (uint32_t)(-i));
      if (sn != sg) atomicAdd(a.seg_counts + sg, (uint32_t)(i + 1));
    }
  }
  if (!PERSIST) return;  // one tile per CTA on an exact grid
  __syncthreads();  // the staging and s_bid are reused by the next tile
  }
}

template <typename KI, bool VALS>
constexpr size_t onesweep_smem() {
  return sizeof(KI) * kSortTile + (VALS ? sizeof(uint32_t) * kSortTile : 0);
}

template <typename KI, int OUT, int SEG, bool VALS>
void launch_pass(const PassArgs& a, int64_t blocks, cudaStream_t s) {
  constexpr size_t smem = onesweep_smem<KI, VALS>();
  static bool attr_set[kMaxDevices] = {};
  static int occ[kMaxDevices] = {}, sms[kMaxDevices] = {};
  const int dev = current_device();
  if (!attr_set[dev]) {
    cudaFuncSetAttribute(k_onesweep<KI, OUT, SEG, VALS, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_onesweep<KI, OUT, SEG, VALS, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[dev], k_onesweep<KI, OUT, SEG, VALS, true>,
                                                  kSortThreads, smem);
    if (occ[dev] < 1) occ[dev] = 1;
    attr_set[dev] = true;
  }
  if (!a.n_dev) {
    k_onesweep<KI, OUT, SEG, VALS, false><<<(unsigned)blocks, kSortThreads, smem, s>>>(a);
    return;
  }
  // the key count is on the device: a persistent grid takes tiles by ticket
  const int64_t persistent = (int64_t)sms[dev] * occ[dev];
  k_onesweep<KI, OUT, SEG, VALS, true>
      <<<(unsigned)(blocks < persistent ? blocks : persistent), kSortThreads, smem, s>>>(a);
}

PassArgs pass_args(const RadixSortBuffers& b, int64_t n, int shift, int p, int64_t blocks) {
  PassArgs a{};
  a.keys[0] = b.keys[0];
  a.keys[1] = b.keys[1];
  a.vals[0] = b.vals[0];
  a.vals[1] = b.vals[1];
  a.n = n;
  a.shift = shift;
  a.pass = p;
  a.plan = b.plan;
  a.lookback = b.lookback;
  a.counter = b.counters;
  a.lb_stride = blocks;
  a.iota_vals = b.iota_vals;
  a.seg_counts = b.seg_counts;
  a.seg_shift = b.seg_shift;
  a.n_dev = b.n_dev;
  a.id_mask = 0xffffffffu;
  return a;
}

// memsets, the histogram (unless the producer built it) and the plan
int sort_setup(const RadixSortBuffers& b, int64_t n, int begin_bit, int n_passes, int64_t blocks,
               bool force_all, cudaStream_t s) {
  int launched = 0;
  if (!b.hist_ready) cudaMemsetAsync(b.hist, 0, sizeof(uint32_t) * kMaxPasses * kRadix, s);
  cudaMemsetAsync(b.counters, 0, sizeof(uint32_t) * kMaxPasses, s);
  if (blocks > 0 && n_passes > 0)
    cudaMemsetAsync(b.lookback, 0, sizeof(uint32_t) * (size_t)n_passes * blocks * kRadix, s);
  if (n > 0 && n_passes > 0 && !b.hist_ready) {
    int hist_blocks = (int)((n + kSortThreads * 16 - 1) / (kSortThreads * 16));
    if (hist_blocks > 148 * 4) hist_blocks = 148 * 4;
    if (b.key_bytes == 4)
      k_radix_hist<uint32_t><<<hist_blocks, kSortThreads, 0, s>>>(
          static_cast<const uint32_t*>(b.keys[0]), n, begin_bit, n_passes, b.hist, b.gate);
    else
      k_radix_hist<uint64_t><<<hist_blocks, kSortThreads, 0, s>>>(
          static_cast<const uint64_t*>(b.keys[0]), n, begin_bit, n_passes, b.hist, b.gate);
    ++launched;
  }
  k_radix_plan<<<1, kRadix, 0, s>>>(b.hist, n, n_passes, b.plan, b.gate, b.keys[0], b.keys[1],
                                    b.vals[0], b.vals[1], b.keys_result, b.vals_result, b.n_dev,
                                    b.max_n, force_all);
  return launched + 1;
}

template <typename K>
int radix_sort_impl(const RadixSortBuffers& b, int64_t n, int begin_bit, int n_passes,
                    cudaStream_t s) {
  if (n_passes > kMaxPasses) n_passes = kMaxPasses;
  const int64_t blocks = (n + kSortTile - 1) / kSortTile;
  int launched = sort_setup(b, n, begin_bit, n_passes, blocks, false, s);
  if (blocks == 0) return launched;
  for (int p = 0; p < n_passes; ++p) {
    const PassArgs a = pass_args(b, n, begin_bit + 8 * p, p, blocks);
    if (b.vals[1]) launch_pass<K, kOutSame, kSegNone, true>(a, blocks, s);
    else if (b.seg_counts) launch_pass<K, kOutSame, kSegKey, false>(a, blocks, s);
    else launch_pass<K, kOutSame, kSegNone, false>(a, blocks, s);
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

int tile_sort(const RadixSortBuffers& b, int64_t k, int tile_bits, cudaStream_t s) {
  const int n_passes = tile_bits ? (tile_bits + 7) / 8 : 1;
  const int64_t blocks = (k + kSortTile - 1) / kSortTile;
  int launched = sort_setup(b, k, 32, n_passes, blocks, true, s);
  if (blocks == 0) return launched;
  for (int p = 0; p < n_passes; ++p) {
    const PassArgs a = pass_args(b, k, 32 + 8 * p, p, blocks);
    if (p + 1 == n_passes) launch_pass<uint64_t, kOutIds, kSegKey, false>(a, blocks, s);
    else launch_pass<uint64_t, kOutSame, kSegNone, false>(a, blocks, s);
  }
  return launched + n_passes;
}

}  // namespace lmgs
