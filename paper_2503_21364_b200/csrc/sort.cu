// Device-wide LSD radix sort (onesweep).
//
// Two sorts per view:
//   K2  fp32 depth keys of all Gaussians with an implicit id payload (stable,
//       so equal keys stay in id order; runs of equal fp32 keys are then fixed
//       up by the exact fp64 depth — _sort_order, gaussian_core.py:277-283);
//   K5  the instance keys tile << 32 | id, sorted on the tile bits only
//       (stable: the emitted array is already in depth-rank order).  With two
//       passes the first writes packed 4-byte keys (tile >> 8) << id_bits | id
//       and the second the 32-bit ids alone, which is all the blend reads
//       (tile_sort below).
//
// Per sort: one histogram kernel computes every digit's global histogram in a
// single read (for K2 and K5 the producer builds it); a 1-block plan kernel
// scans them, marks digits all keys share as trivial (skipped on the device;
// not for K5, whose passes change the key format) and routes the ping-pong
// buffers; then one onesweep kernel per digit: a tile of kSortTile keys is
// ranked in shared memory ({count, match} words per warp, stable), staged in
// shared memory in digit order, its global digit offsets found by decoupled
// look-back over the preceding tiles, and written out in coalesced per-digit
// runs.
#include "device_util.cuh"
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagIncl = 2u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1;
constexpr int kWarps = kSortThreads / 32;
// the decoupled look-back after the ranking instead of before it: by then the
// predecessors have published (the look-back phase of a tile drops from ~3.4
// to ~0.7 us): depth sort 0.265 -> 0.239, tile sort 0.312 -> 0.286 ms/view,
// 775.7 -> 793.9 frames/s (profiles/r10/lookback_late_variants.txt)
// concurrent renders: the persistent grids prefetch each CTA's next tile by
// TMA (PREF).  Off: 700 vs 804 frames/s — the two 32-KB input buffers per CTA
// take the shared memory the other streams' kernels would co-reside in
// (profiles/r10/sort_prefetch_variants.txt)
#ifndef LMGS_SORT_PREFETCH
#define LMGS_SORT_PREFETCH 0
#endif
#ifndef LMGS_SORT_SMEM_PAD
#define LMGS_SORT_SMEM_PAD 0  // extra dynamic shared bytes per onesweep CTA (co-residency experiments)
#endif
#ifndef LMGS_SORT_PERSIST_CTAS_VALS
#define LMGS_SORT_PERSIST_CTAS_VALS LMGS_SORT_PERSIST_CTAS  // key-value (depth) sorts
#endif
#ifndef LMGS_SORT_IOTA16
#define LMGS_SORT_IOTA16 1  // the first pass stages implicit values as 16-bit positions
#endif
#ifndef LMGS_RANK_SPLIT
#define LMGS_RANK_SPLIT 1  // separate match / 16-bit count arrays (smaller shared footprint)
#endif
#ifndef LMGS_RANK_PAIRS
#define LMGS_RANK_PAIRS 0  // 1: two items per round with {count, matchA, matchB} words: 692 vs 815 frames/s (profiles/r10/rank_pairs_variants.txt)
#endif
#ifndef LMGS_LOOKBACK_LATE
#define LMGS_LOOKBACK_LATE 1
#endif
#ifndef LMGS_LOOK_WINDOW
#define LMGS_LOOK_WINDOW 8
#endif
constexpr int kLookWindow = LMGS_LOOK_WINDOW;
#ifndef LMGS_SORT_PERSIST_CTAS
// LMGS_FLAG_CONCURRENT: persistent onesweep grids of this many CTAs per SM
// (else one CTA per tile).  A pass is latency-bound; with one CTA per SM it
// runs slower alone (tile sort 0.32 -> 0.47 ms) but leaves the SMs' other
// slots to the other streams' kernels: 758 -> 779 frames/s at 3 streams, 783
// at 4 (profiles/r10)
#define LMGS_SORT_PERSIST_CTAS 1
#endif
#ifndef LMGS_TILE_SORT_PACKED
#define LMGS_TILE_SORT_PACKED 1  // two-pass tile sorts with a packed 4-byte second pass
#endif
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
template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, int shift) {
  return (uint32_t)((uint64_t)key >> shift) & 0xffu;
}

__device__ __forceinline__ bool gated_off(const int* gate) { return gate && *gate == 0; }

// LMGS_SORT_TRACE (experiments only): %globaltimer at the phase boundaries of
// every tile of the traced pass (pass index == LMGS_SORT_TRACE - 1; the last
// sort to run that pass wins): ticket, loaded+counted, looked back, ranked,
// staged, written — read back with lmgs_debug_sort_trace
// (bench_tools/sort_trace.py).
#ifdef LMGS_SORT_TRACE
constexpr int kTraceTiles = 1 << 14;
__device__ unsigned long long g_trace[kTraceTiles][7];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(k)                                                                     \
  if (a.pass == LMGS_SORT_TRACE - 1 && threadIdx.x == 0 && bid < kTraceTiles) {      \
    g_trace[bid][k] = gtimer();                                                      \
    if (k == 0) g_trace[bid][6] = (unsigned long long)blockIdx.x;                    \
  }
#else
#define TRACE(k)
#endif

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
//   kOutPacked: u64 tile << 32 | id in, u32 (tile >> 8) << id_bits | id out
//   (the first pass of the fused tile sort: its low tile digit is implied by
//   the bucket the key lands in, so the second pass needs 4 bytes per key)
enum : int { kOutSame = 0, kOutIds = 1, kOutPacked = 2 };
//   kSegLo: the keys are packed (tile >> 8) << id_bits | id (shift = id_bits)
//   and the low tile digit is the bucket of the previous pass (lo_pass) the
//   key's input position lies in
enum : int { kSegNone = 0, kSegKey = 1, kSegLo = 2 };
// Where a pass's keys come from: the input buffer, or generated from the rank
// records of the visible splats (fused emission, tile_sort_fused).
// kSrcIota: keys from the input, values implicit (input index) and staged as
// 16-bit tile positions (2 B, not 4, per key): the first pass of a sort with
// iota_vals, whose pass 0 is the first active one whenever it moves data
enum : int { kSrcKeys = 0, kSrcEmit = 1, kSrcIota = 2 };

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
  int lo_pass;    // kSegLo: the pass whose buckets give the low tile digit
  const unsigned long long* n_dev;
  int id_bits;  // kOutPacked
  bool concurrent;  // persistent grid sized to share the SMs (LMGS_FLAG_CONCURRENT)
  // kSrcEmit
  const uint4* rrec;             // [n_vis] {rect lo, rect hi, id, first slot}
  const uint32_t* chunk_first;   // [tiles] rank holding the tile's first slot
  const unsigned long long* n_vis_dev;
  int tiles_x;
};

template <typename KI, int OUT>
struct OutKey {
  using type = KI;
};
template <typename KI>
struct OutKey<KI, kOutIds> {
  using type = uint32_t;
};
template <typename KI>
struct OutKey<KI, kOutPacked> {
  using type = uint32_t;
};

template <typename KI, int OUT>
__device__ __forceinline__ typename OutKey<KI, OUT>::type out_key(KI k, const PassArgs& a) {
  if constexpr (OUT == kOutIds)
    return (uint32_t)k & a.id_mask;
  else if constexpr (OUT == kOutPacked)
    return ((uint32_t)((uint64_t)k >> 40) << a.id_bits) | (uint32_t)k;
  else
    return k;
}

template <typename KI, bool VALS>
constexpr int sort_min_ctas() {
  return (sizeof(KI) == 4 && !VALS) ? LMGS_SORT_MIN_CTAS_NARROW : LMGS_SORT_MIN_CTAS;
}

// Fused emission (kSrcEmit): the tile's kSortTile instance slots [base, base +
// count) are generated from the rank records instead of loaded.  Slot p
// belongs to the last rank whose first slot is <= p: every covering rank
// marks its first slot in a shared owner map (u16 offsets from the tile's
// first rank; a rank owns >= 1 slot, so at most count + 1 ranks cover the
// tile), a block max-scan fills the gaps, and each item decodes its tile from
// the owner's rectangle (row-major inside it, as K4 emits them).  Items are
// warp-striped like loaded keys, so the ranking below stays stable in slot
// (= depth rank, then row-major tile) order.  The map aliases the staging
// buffer, which is first written after the ranking.
template <typename KI>
__device__ __forceinline__ void emit_keys(const PassArgs& a, int64_t n, int64_t base, int count,
                                          unsigned char* smem, KI (&key)[kSortItems]) {
  static_assert(sizeof(KI) == 8, "emitted keys are tile << 32 | id");
  uint16_t* s_owner = reinterpret_cast<uint16_t*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b = base / kSortTile;
  const uint32_t r0 = a.chunk_first[b];
  // ranks r0 .. r_last cover the tile (r_last = the next tile's first rank,
  // which may start exactly at its first slot: the mark below skips it)
  const uint32_t n_vis = (uint32_t)*a.n_vis_dev;
  const uint32_t r_end = min(base + count < n ? a.chunk_first[b + 1] + 1 : n_vis, n_vis);
  // (clamped: a no-sync overflow leaves the records past the capacity stale)
  const int nr = max(0, min((int)(r_end - r0), count + 1));
  const uint32_t slot0 = (uint32_t)base, slot_end = (uint32_t)(base + count);
  static_assert(kSortItems % 2 == 0, "owner offsets are scanned in u16 pairs");
  for (int i = tid; i < kSortTile / 8; i += kSortThreads)
    reinterpret_cast<uint4*>(s_owner)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
#pragma unroll 4
  for (int j = tid; j < nr; j += kSortThreads) {
    const uint32_t st = __ldg(reinterpret_cast<const uint32_t*>(a.rrec + r0 + j) + 3);
    if (st < slot_end) s_owner[st > slot0 ? st - slot0 : 0u] = (uint16_t)j;
  }
  __syncthreads();
  {
    // inclusive max-scan of the marks (offsets grow with the slot): thread t
    // owns slots [kSortItems * t, kSortItems * (t + 1))
    __shared__ uint32_t s_wmax[kSortThreads / 32];
    uint32_t v[kSortItems / 2];
    const uint32_t* row = reinterpret_cast<const uint32_t*>(s_owner) + tid * (kSortItems / 2);
#pragma unroll
    for (int u = 0; u < kSortItems / 2; ++u) v[u] = row[u];
    uint32_t m = 0;
#pragma unroll
    for (int u = 0; u < kSortItems / 2; ++u) m = max(m, max(v[u] & 0xffffu, v[u] >> 16));
    uint32_t incl = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl = max(incl, x);
    }
    if (lane == 31) s_wmax[warp] = incl;
    uint32_t carry = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) carry = 0;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kSortThreads / 32; ++w) carry = w < warp ? max(carry, s_wmax[w]) : carry;
    uint32_t* wrow = reinterpret_cast<uint32_t*>(s_owner) + tid * (kSortItems / 2);
#pragma unroll
    for (int u = 0; u < kSortItems / 2; ++u) {
      const uint32_t lo = max(carry, v[u] & 0xffffu);
      const uint32_t hi = max(lo, v[u] >> 16);
      carry = hi;
      wrow[u] = lo | (hi << 16);
    }
  }
  __syncthreads();
  const int wbase = warp * 32 * kSortItems;
  // records in groups of 4 (16 registers live, not 64; mostly L1 hits: a
  // rank covers ~3.5 consecutive slots)
  constexpr int G = 4;
  static_assert(kSortItems % G == 0, "");
#pragma unroll
  for (int j0 = 0; j0 < kSortItems; j0 += G) {
    uint4 rr[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int i = wbase + (j0 + u) * 32 + lane;
      rr[u] = __ldg(a.rrec + r0 + s_owner[i < count ? i : 0]);
    }
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int i = wbase + (j0 + u) * 32 + lane;
      const uint32_t q = slot0 + (uint32_t)i - rr[u].w;
      const uint32_t x0 = rr[u].x & 0xffffu, y0 = rr[u].x >> 16, x1 = rr[u].y & 0xffffu;
      const uint32_t w = x1 - x0 + 1;
      // q / w without the integer-division sequence (q < area <= tiles < 2^16
      // on this path): the float quotient is within one of the truth; fixed up
      uint32_t dy = (uint32_t)__fdividef((float)q, (float)w);
      if (dy * w > q) --dy;
      else if ((dy + 1) * w <= q) ++dy;
      const uint32_t tile = (y0 + dy) * (uint32_t)a.tiles_x + x0 + (q - dy * w);
      key[j0 + u] = i < count ? (((uint64_t)tile << 32) | rr[u].z) : ~0ull;
    }
  }
}

// one onesweep scatter pass (digit `pass`)
//
// 1. load kSortTile keys (warp-striped, coalesced);
// 2. early counts: the CTA's digit histogram by shared atomics, published at
//    once to the look-back array so successors never wait on our ranking;
// 3. stable rank inside each warp: per warp and digit one 64-bit shared word
//    {count, match}: lanes holding the same digit OR their lane bits into the
//    match half, read the pair back with one 64-bit load (rank = count +
//    lanes below), and the lowest of them stores {count + peers, 0} — no
//    shuffle, no counter atomic (MATCH.ANY serialised; a separate match word +
//    leader atomicAdd + shuffle cost ~39 SASS per key, this ~12);
// 4. decoupled look-back (windowed) for the global digit offsets — after the
//    ranking (LMGS_LOOKBACK_LATE), when the predecessors have published;
// 5. per-digit prefix over warps, staging in shared memory in digit order;
// 6. coalesced write-out in per-digit runs, in the pass's output format (the
//    last tile pass also counts the tile runs for the ranges).
// PREF (persistent grids of concurrent renders): a CTA claims its next tile
// right after the current tile's look-back and has its keys (and values)
// copied into a second shared buffer by TMA bulk copies while it stages and
// writes the current one; full tiles only (a partial tile is loaded directly)
template <typename KI, int OUT, int SEG, bool VALS, bool PERSIST, int SRC = kSrcKeys,
          bool PREF = false>
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
  // kOutPacked stages the 4-byte output and the 1-byte digit only (5 B, not 8,
  // per key: the sort CTAs' shared footprint sets how much the co-running
  // streams' kernels keep, profiles/r10/sort_smem_pad_variants.txt)
  constexpr bool kPackedStage = OUT == kOutPacked;
  static_assert(!kPackedStage || (SEG == kSegNone && !VALS), "packed staging: keys only");
  uint32_t* s_pk = reinterpret_cast<uint32_t*>(smem_raw);
  uint8_t* s_dg8 = reinterpret_cast<uint8_t*>(smem_raw + sizeof(uint32_t) * kSortTile);
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(smem_raw + sizeof(KI) * kSortTile);
  constexpr bool kIota16 = SRC == kSrcIota;
  static_assert(!kIota16 || (VALS && kSortTile <= 65536), "16-bit implicit values");
  uint16_t* s_idx16 = reinterpret_cast<uint16_t*>(smem_raw + sizeof(KI) * kSortTile);
  // kSegLo: the staged keys' low tile digits (the vals slot: kSegLo has none)
  uint8_t* s_lo = reinterpret_cast<uint8_t*>(smem_raw + sizeof(KI) * kSortTile);
  __shared__ uint32_t s_dstart[SEG == kSegLo ? kRadix : 1];
  // digit kRadix collects the invalid items of a partial tile, so neither the
  // counts nor the ranking need a validity predicate
#if LMGS_RANK_PAIRS
  using RankWord = uint4;  // {count, match of item j, match of item j + 1, -}
#else
  using RankWord = uint2;  // {count, match}
#endif
#if LMGS_RANK_SPLIT
  // match words and 16-bit counts in separate arrays (12.3 KB, not 16.4)
#if LMGS_RANK_SPLIT == 1
  __shared__ uint32_t s_mt[kWarps][kRadix + 1];
#endif
  __shared__ uint16_t s_ct[kWarps][kRadix + 1];
#define LMGS_WCOUNT(w, d) s_ct[w][d]
#else
  __shared__ RankWord s_wm[kWarps][kRadix + 1];
#define LMGS_WCOUNT(w, d) s_wm[w][d].x
#endif
  __shared__ uint32_t s_hist[kRadix + 1];
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
  // PREF input buffers after the staging (and its vals / low digits)
  constexpr size_t kStageBytes = (kPackedStage ? 5 * (size_t)kSortTile : sizeof(KI) * kSortTile) +
                                 (VALS ? (kIota16 ? 2 : 4) * (size_t)kSortTile : 0) +
                                 (SEG == kSegLo ? kSortTile : 0);
  constexpr size_t kInBytes = sizeof(KI) * kSortTile + (VALS ? sizeof(uint32_t) * kSortTile : 0);
  __shared__ __align__(8) uint64_t s_bar[PREF ? 2 : 1];
  __shared__ uint32_t s_next;
  auto in_keys = [&](int b) {
    return reinterpret_cast<KI*>(smem_raw + ((kStageBytes + 15) & ~(size_t)15) + b * kInBytes);
  };
  auto in_vals = [&](int b) {
    return reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(in_keys(b)) +
                                       sizeof(KI) * kSortTile);
  };
  // a full tile's keys (and non-implicit values) into buffer b by TMA
  auto prefetch = [&](uint32_t t, int b) {
    if ((int64_t)(t + 1) * kSortTile > n) return;  // partial or past the end: direct loads
    const bool pv = VALS && !(a.iota_vals && pass == plan->first_active);
    mbar_expect_tx(&s_bar[b], sizeof(KI) * kSortTile + (pv ? sizeof(uint32_t) * kSortTile : 0));
    bulk_g2s(in_keys(b), kin + (int64_t)t * kSortTile, sizeof(KI) * kSortTile, &s_bar[b]);
    if (pv) bulk_g2s(in_vals(b), vin + (int64_t)t * kSortTile, sizeof(uint32_t) * kSortTile, &s_bar[b]);
  };
  uint32_t phase = 0;  // PREF: bit b = parity of buffer b's next completion
  int cur = 0;
  if constexpr (PREF) {
    if (tid == 0) {
      mbar_init(&s_bar[0], 1);
      mbar_init(&s_bar[1], 1);
      mbar_init_fence();
      s_next = atomicAdd(a.counter + pass, 1u);
      prefetch(s_next, 0);
    }
    __syncthreads();
  }
  // tiles are taken by ticket; a CTA loops until the keys run out (with n_dev
  // the grid is a persistent one sized for the device, not for the bound)
  for (;;) {
  if (PREF) {
    if (tid == 0) s_bid = s_next;
  } else {
    if (tid == 0) s_bid = atomicAdd(a.counter + pass, 1u);
  }
  __syncthreads();
  const uint32_t bid = s_bid;
  const int64_t base = (int64_t)bid * kSortTile;
  if (base >= n) return;
  const int count = (int)min((int64_t)kSortTile, n - base);
  const bool staged_in = PREF && count == kSortTile;  // this tile's keys came by TMA
  TRACE(0)

  KI key[kSortItems];
  uint32_t val[VALS && !kIota16 ? kSortItems : 1];
  uint32_t dg[kSortItems];  // digit (kRadix: invalid), then | rank in the warp << 16
  uint32_t lo_info = 0;  // kSegLo: the tile's first low digit | inner bucket starts << 16
  const int wbase = warp * 32 * kSortItems;
  if constexpr (SRC == kSrcEmit) {
    emit_keys(a, n, base, count, smem_raw, key);
  } else if (staged_in) {
    mbar_wait(&s_bar[cur], (phase >> cur) & 1u);
    phase ^= 1u << cur;
    const KI* sk = in_keys(cur);
    const uint32_t* sv = in_vals(cur);
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      const int i = wbase + j * 32 + lane;
      key[j] = sk[i];
      if (VALS && !kIota16) val[j] = iota ? (uint32_t)(base + i) : sv[i];
    }
    fence_proxy_async_smem();  // these reads before the buffer's next TMA fill
  } else {
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      const int i = wbase + j * 32 + lane;
      key[j] = i < count ? kin[base + i] : (KI)~(KI)0;
      if (VALS && !kIota16) val[j] = iota ? (uint32_t)(base + i) : (i < count ? vin[base + i] : 0u);
    }
  }
  // the loads above are in flight while the ranking state is cleared
  uint32_t my_dstart = 0;  // kSegLo: start of bucket tid of the previous pass
  if constexpr (SEG == kSegLo) my_dstart = plan->digit_start[a.lo_pass][tid];
  for (int i = tid; i < kWarps * (kRadix + 1); i += kSortThreads)
#if LMGS_RANK_SPLIT
  {
#if LMGS_RANK_SPLIT == 1
    (&s_mt[0][0])[i] = 0u;
#endif
    (&s_ct[0][0])[i] = 0;
  }
#else
    (&s_wm[0][0])[i] = RankWord{};
#endif
  s_hist[tid] = 0;  // kSortThreads == kRadix
  if (tid == 0) s_hist[kRadix] = 0;
#pragma unroll
  for (int j = 0; j < kSortItems; ++j)
    dg[j] = wbase + j * 32 + lane < count ? digit_of(key[j], shift) : (uint32_t)kRadix;
  __syncthreads();
  // 2. early counts, published with the look-back before ranking
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) atomicAdd(&s_hist[dg[j]], 1u);
  if constexpr (SEG == kSegLo) {
    // the bucket of input position p is the number of buckets starting at or
    // before p, less one (starts are non-decreasing).  The tile's first bucket
    // and the buckets starting inside the tile come from two block counts;
    // buckets average ~80K keys, so a 4096-key tile rarely holds a boundary
    const uint32_t b0 = (uint32_t)base, b1 = (uint32_t)(base + count);
    const int lo_first = __syncthreads_count(my_dstart <= b0) - 1;
    const bool inner = my_dstart > b0 && my_dstart < b1;
    const int n_inner = __syncthreads_count(inner);
    if (inner) s_dstart[tid] = my_dstart;  // read at staging (the barriers below order it)
    lo_info = (uint32_t)lo_first | (uint32_t)n_inner << 16;
  }
  __syncthreads();
  TRACE(1)
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
  }
  const uint32_t local_start = s_local_start[tid];
  // decoupled look-back for this tile's global digit offsets (thread d =
  // digit d); LMGS_LOOKBACK_LATE runs it after the ranking, when the
  // predecessors have had that long to publish
  auto look_back = [&]() {
    const int d = tid;
    // decoupled look-back for this tile's global digit offsets, right after
    // the early counts so the inclusive prefix is published before ranking.
    // Each digit's thread reads a window of kLookWindow predecessors with
    // independent loads (one L2 round trip per window, not per predecessor),
    // then walks it from the nearest one, re-polling only unpublished entries.
    uint32_t excl = 0;
    if (bid != 0) {
      // a running pointer at predecessor `look`: the window's loads use
      // immediate offsets (no 64-bit address arithmetic per load)
      int look = (int)bid - 1;
      const uint32_t* q = lb + (int64_t)look * kRadix + d;
      bool done = false;
      while (!done) {
        uint32_t v[kLookWindow];
#pragma unroll
        for (int w = 0; w < kLookWindow; ++w)
          v[w] = look - w >= 0 ? ld_acquire(q - w * kRadix) : kFlagIncl;
        bool all_pub = true;
#pragma unroll
        for (int w = 0; w < kLookWindow; ++w) all_pub &= (v[w] & ~kValueMask) != 0;
        if (all_pub) {  // the common case: a predicated walk, no polling branches
#pragma unroll
          for (int w = 0; w < kLookWindow; ++w) {
            excl += done ? 0u : (v[w] & kValueMask);
            done = done || (v[w] & ~kValueMask) == kFlagIncl;
          }
        } else {
#pragma unroll
          for (int w = 0; w < kLookWindow; ++w) {
            if (done) break;
            while ((v[w] & ~kValueMask) == 0) v[w] = ld_acquire(q - w * kRadix);
            excl += v[w] & kValueMask;
            done = (v[w] & ~kValueMask) == kFlagIncl;
          }
        }
        look -= kLookWindow;
        q -= kLookWindow * kRadix;
      }
      st_release(lb + (int64_t)bid * kRadix + d, kFlagIncl | (excl + total));
    }
    s_global[d] = plan->digit_start[pass][d] + excl - local_start;
  };
  if (!LMGS_LOOKBACK_LATE) look_back();
  // 3. stable in-warp ranking, items in (j, lane) order
#ifdef LMGS_SORT_TRACE
  __syncthreads();
  TRACE(2)
#endif
  const uint32_t lt = lanemask_lt();
#if LMGS_RANK_SPLIT
#if LMGS_RANK_SPLIT == 1
  uint32_t* my_mt = s_mt[warp];
#endif
  uint16_t* my_ct = s_ct[warp];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const uint32_t d = dg[j];
#if LMGS_RANK_SPLIT == 1
    atomicOr(&my_mt[d], 1u << lane);
    __syncwarp();
    const uint32_t peers = my_mt[d], c = my_ct[d];
#else
    // experiment: MATCH.ANY instead of the shared match words (8 KB less per CTA)
    const uint32_t peers = __match_any_sync(~0u, d), c = my_ct[d];
#endif
    __syncwarp();
    const uint32_t below = peers & lt;
    if (below == 0) {
      my_ct[d] = (uint16_t)(c + __popc(peers));
#if LMGS_RANK_SPLIT == 1
      my_mt[d] = 0u;
#endif
    }
    dg[j] |= (c + __popc(below)) << 16;
    __syncwarp();
  }
#else
  RankWord* my = s_wm[warp];
#if LMGS_RANK_PAIRS
  // two items per round, each with its own match half: item j + 1's rank
  // counts every item j of its digit first; one store per digit (the lowest
  // lane of item j holding it, else the lowest of item j + 1)
  static_assert(kSortItems % 2 == 0, "");
#pragma unroll
  for (int j = 0; j < kSortItems; j += 2) {
    const uint32_t da = dg[j], db = dg[j + 1];
    atomicOr(&my[da].y, 1u << lane);
    atomicOr(&my[db].z, 1u << lane);
    __syncwarp();
    const uint4 qa = my[da], qb = my[db];
    __syncwarp();
    const uint32_t below_a = qa.y & lt;
    if (below_a == 0) my[da] = make_uint4(qa.x + __popc(qa.y) + __popc(qa.z), 0u, 0u, 0u);
    if (qb.y == 0 && (qb.z & lt) == 0) my[db] = make_uint4(qb.x + __popc(qb.z), 0u, 0u, 0u);
    dg[j] |= (qa.x + __popc(below_a)) << 16;
    dg[j + 1] |= (qb.x + __popc(qb.y) + __popc(qb.z & lt)) << 16;
    __syncwarp();
  }
#else
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    atomicOr(&my[dg[j]].y, 1u << lane);
    __syncwarp();
    const uint2 cm = my[dg[j]];
    __syncwarp();
    const uint32_t below = cm.y & lt;
    if (below == 0) my[dg[j]] = make_uint2(cm.x + __popc(cm.y), 0u);
    dg[j] |= (cm.x + __popc(below)) << 16;
    __syncwarp();
  }
#endif
#endif
  if (LMGS_LOOKBACK_LATE == 1) look_back();
  if constexpr (PREF) {
    // the next tile, claimed once this one has published its prefix: its
    // keys stream in while this tile is staged and written
    if (tid == 0) {
      s_next = atomicAdd(a.counter + pass, 1u);
      prefetch(s_next, cur ^ 1);
    }
  }
  __syncthreads();
  TRACE(3)
  // 4. per digit: exclusive prefix over warps (the invalid items go behind
  // the tile's count, into staging slots the write-out never reads)
  {
    const int d = tid;
    uint32_t run = s_local_start[d];
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = LMGS_WCOUNT(w, d);
      LMGS_WCOUNT(w, d) = run;
      run += c;
    }
    if (tid == 0) {
      run = (uint32_t)count;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = LMGS_WCOUNT(w, kRadix);
        LMGS_WCOUNT(w, kRadix) = run;
        run += c;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const uint32_t p = (dg[j] >> 16) + LMGS_WCOUNT(warp, dg[j] & 0xffffu);
    if constexpr (kPackedStage) {
      s_pk[p] = out_key<KI, OUT>(key[j], a);
      s_dg8[p] = (uint8_t)dg[j];
    } else {
      s_keys[p] = key[j];
    }
    if constexpr (kIota16) s_idx16[p] = (uint16_t)(wbase + j * 32 + lane);
    else if (VALS) s_vals[p] = val[j];
    if constexpr (SEG == kSegLo) {
      // the key's input position's bucket: the tile's first one plus the
      // inner buckets (lo_first + 1 ..) starting at or before it
      const int lo_first = (int)(lo_info & 0xffffu), n_inner = (int)(lo_info >> 16);
      int lo = lo_first;
      for (int t = 1; t <= n_inner; ++t)
        lo += s_dstart[lo_first + t] <= (uint32_t)base + wbase + j * 32 + lane;
      s_lo[p] = (uint8_t)lo;
    }
  }
  if (LMGS_LOOKBACK_LATE == 2) look_back();  // only the write-out needs the global offsets
  __syncthreads();
  TRACE(4)
  // 6. coalesced write-out: consecutive threads, consecutive staged positions
  bool segs = SEG != kSegNone && a.seg_counts && pass == plan->last_active;
  if (SEG == kSegLo && segs && (lo_info >> 16) == 0) {
    // one low digit for the whole tile (no bucket of the previous pass starts
    // inside it): tile (d << 8 | lo) holds exactly the tile's count of digit d
    const uint32_t c = s_hist[tid];
    if (c) atomicAdd(a.seg_counts + ((uint32_t)tid << 8 | (lo_info & 0xffffu)), c);
    segs = false;
  }
  if constexpr (kPackedStage) {
    for (int i = tid; i < count; i += kSortThreads) kout[s_global[s_dg8[i]] + i] = s_pk[i];
  } else
  for (int i = tid; i < count; i += kSortThreads) {
    const KI k = s_keys[i];
    const uint32_t o = s_global[digit_of(k, shift)] + i;
    kout[o] = out_key<KI, OUT>(k, a);
    if constexpr (kIota16) vout[o] = (uint32_t)base + s_idx16[i];
    else if (VALS) vout[o] = s_vals[i];
    if (segs) {
      // the staged tile is sorted on every key bit sorted so far: runs of one
      // segment are contiguous; a run [i0, i1] adds (i1 + 1) - i0
      uint64_t sg, sp, sn;
      if constexpr (SEG == kSegLo) {
        auto seg = [&](int t) {
          return (uint64_t)(digit_of(s_keys[t], shift) << 8 | s_lo[t]);
        };
        sg = (uint64_t)(digit_of(k, shift) << 8 | s_lo[i]);
        sp = i > 0 ? seg(i - 1) : ~0ull;
        sn = i + 1 < count ? seg(i + 1) : ~0ull;
      } else {
        sg = (uint64_t)k >> a.seg_shift;
        sp = i > 0 ? (uint64_t)s_keys[i - 1] >> a.seg_shift : ~0ull;
        sn = i + 1 < count ? (uint64_t)s_keys[i + 1] >> a.seg_shift : ~0ull;
      }
      if (sp != sg) atomicAdd(a.seg_counts + sg, (uint32_t)(-i));
      if (sn != sg) atomicAdd(a.seg_counts + sg, (uint32_t)(i + 1));
    }
  }
#ifdef LMGS_SORT_TRACE
  __syncthreads();
  TRACE(5)
#endif
  if (!PERSIST) return;  // one tile per CTA on an exact grid
  if (PREF) cur ^= 1;
  __syncthreads();  // the staging and s_bid are reused by the next tile
  }
}

template <typename KI, bool VALS, int SEG = kSegNone, bool PREF = false, int OUT = kOutSame,
          int SRC = kSrcKeys>
constexpr size_t onesweep_smem() {
  return (((OUT == kOutPacked ? 5 * (size_t)kSortTile : sizeof(KI) * kSortTile) +
           (VALS ? (SRC == kSrcIota ? 2 : 4) * (size_t)kSortTile : 0) + (SEG == kSegLo ? kSortTile : 0) + 15) &
          ~(size_t)15) +
         (PREF ? 2 * (sizeof(KI) * kSortTile + (VALS ? sizeof(uint32_t) * kSortTile : 0)) : 0);
}

template <typename KI, int OUT, int SEG, bool VALS, int SRC = kSrcKeys>
void launch_pass(const PassArgs& a, int64_t blocks, cudaStream_t s) {
  constexpr size_t smem = onesweep_smem<KI, VALS, SEG, false, OUT, SRC>() + LMGS_SORT_SMEM_PAD;  // (pad: experiments)
  static_assert(SRC != kSrcEmit || smem >= 2 * kSortTile, "the owner map aliases the staging");
  static bool attr_set[kMaxDevices] = {};
  static int occ[kMaxDevices] = {}, sms[kMaxDevices] = {};
  const int dev = current_device();
  if (!attr_set[dev]) {
    cudaFuncSetAttribute(k_onesweep<KI, OUT, SEG, VALS, false, SRC>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_onesweep<KI, OUT, SEG, VALS, true, SRC>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    set_carveout(k_onesweep<KI, OUT, SEG, VALS, false, SRC>);
    set_carveout(k_onesweep<KI, OUT, SEG, VALS, true, SRC>);
    cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ[dev], k_onesweep<KI, OUT, SEG, VALS, true, SRC>, kSortThreads, smem);
    if (occ[dev] < 1) occ[dev] = 1;
    attr_set[dev] = true;
  }
  if (!a.n_dev && !a.concurrent) {
    k_onesweep<KI, OUT, SEG, VALS, false, SRC><<<(unsigned)blocks, kSortThreads, smem, s>>>(a);
    return;
  }
  // the key count is on the device: a persistent grid takes tiles by ticket
  // (concurrent streams: always, with LMGS_SORT_PERSIST_CTAS CTAs per SM,
  // leaving room for the other streams' kernels)
  constexpr int kPersist = VALS ? LMGS_SORT_PERSIST_CTAS_VALS : LMGS_SORT_PERSIST_CTAS;
  const int per_sm = a.concurrent && kPersist > 0 && kPersist < occ[dev] ? kPersist : occ[dev];
  const int64_t persistent = (int64_t)sms[dev] * per_sm;
  const unsigned grid = (unsigned)(blocks < persistent ? blocks : persistent);
  if constexpr (SRC == kSrcKeys && LMGS_SORT_PREFETCH) {
    if (a.concurrent && per_sm == 1) {
      constexpr size_t smem_pref = onesweep_smem<KI, VALS, SEG, true, OUT>();
      static bool pref_set[kMaxDevices] = {};
      if (!pref_set[dev]) {
        cudaFuncSetAttribute(k_onesweep<KI, OUT, SEG, VALS, true, SRC, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_pref);
        pref_set[dev] = true;
      }
      k_onesweep<KI, OUT, SEG, VALS, true, SRC, true><<<grid, kSortThreads, smem_pref, s>>>(a);
      return;
    }
  }
  k_onesweep<KI, OUT, SEG, VALS, true, SRC><<<grid, kSortThreads, smem, s>>>(a);
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
  a.concurrent = b.concurrent;
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
    if (b.vals[1] && b.iota_vals && p == 0 && LMGS_SORT_IOTA16)
      launch_pass<K, kOutSame, kSegNone, true, kSrcIota>(a, blocks, s);
    else if (b.vals[1]) launch_pass<K, kOutSame, kSegNone, true>(a, blocks, s);
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

int tile_sort(const RadixSortBuffers& b, int64_t k, int tile_bits, int id_bits, cudaStream_t s) {
  const int n_passes = tile_bits ? (tile_bits + 7) / 8 : 1;
  const int64_t blocks = (k + kSortTile - 1) / kSortTile;
  int launched = sort_setup(b, k, 32, n_passes, blocks, true, s);
  if (blocks == 0) return launched;
  if (n_passes == 2 && (tile_bits - 8) + id_bits <= 32 && LMGS_TILE_SORT_PACKED) {
    // the first pass writes 4-byte keys (tile >> 8) << id_bits | id (its low
    // tile digit is the bucket a key lands in); the second sorts them on the
    // high digit and writes the ids, counting tile runs with the low digit
    // recovered from the first pass's bucket bounds
    PassArgs a = pass_args(b, k, 32, 0, blocks);
    a.id_bits = id_bits;
    launch_pass<uint64_t, kOutPacked, kSegNone, false>(a, blocks, s);
    a = pass_args(b, k, id_bits, 1, blocks);
    a.id_bits = id_bits;
    a.id_mask = id_bits >= 32 ? 0xffffffffu : (1u << id_bits) - 1u;
    a.lo_pass = 0;
    launch_pass<uint32_t, kOutIds, kSegLo, false>(a, blocks, s);
    return launched + 2;
  }
  for (int p = 0; p < n_passes; ++p) {
    const PassArgs a = pass_args(b, k, 32 + 8 * p, p, blocks);
    if (p + 1 == n_passes) launch_pass<uint64_t, kOutIds, kSegKey, false>(a, blocks, s);
    else launch_pass<uint64_t, kOutSame, kSegNone, false>(a, blocks, s);
  }
  return launched + n_passes;
}

int tile_sort_fused(const RadixSortBuffers& b, int64_t k, int id_bits, const uint4* rrec,
                    const uint32_t* chunk_first, const unsigned long long* n_vis_dev, int tiles_x,
                    cudaStream_t s) {
  const int64_t blocks = (k + kSortTile - 1) / kSortTile;
  int launched = sort_setup(b, k, 32, 2, blocks, true, s);
  if (blocks == 0) return launched;
  PassArgs a = pass_args(b, k, 32, 0, blocks);
  a.id_bits = id_bits;
  a.rrec = rrec;
  a.chunk_first = chunk_first;
  a.n_vis_dev = n_vis_dev;
  a.tiles_x = tiles_x;
  // pass 0: keys generated from the rank records, low tile digit, packed out
  launch_pass<uint64_t, kOutPacked, kSegNone, false, kSrcEmit>(a, blocks, s);
  // pass 1: the high digit of the packed keys -> ids, range counts
  a = pass_args(b, k, id_bits, 1, blocks);
  a.id_bits = id_bits;
  a.id_mask = id_bits >= 32 ? 0xffffffffu : (1u << id_bits) - 1u;
  a.lo_pass = 0;
  launch_pass<uint32_t, kOutIds, kSegLo, false>(a, blocks, s);
  return launched + 2;
}

}  // namespace lmgs

#ifdef LMGS_SORT_TRACE
extern "C" int lmgs_debug_sort_trace(void* host, size_t bytes) {
  const size_t n = bytes < sizeof(lmgs::g_trace) ? bytes : sizeof(lmgs::g_trace);
  return (int)cudaMemcpyFromSymbol(host, lmgs::g_trace, n);
}
extern "C" int lmgs_debug_sort_trace_reset() {
  static unsigned long long zero[lmgs::kTraceTiles][7];
  return (int)cudaMemcpyToSymbol(lmgs::g_trace, zero, sizeof(zero));
}
#endif
