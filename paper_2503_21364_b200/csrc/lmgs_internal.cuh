// Internal declarations shared by the lmgs CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lmgs.h"

namespace lmgs {

// Reference constants, gaussian_core.py:21-27.
constexpr double kTermEps = 1e-4;     // TERM_EPS
constexpr double kSigmaMax = 0.9999;  // SIGMA_MAX
constexpr double kCov2dReg = 0.3;     // COV2D_REG
constexpr double kNearCullZ = 0.01;   // NEAR_CULL_Z
constexpr double kShC0 = 0.28209479177387814;
constexpr double kShC1 = 0.4886025119029199;
constexpr double kLog2e = 1.4426950408889634;

constexpr uint64_t kCulledKey = ~0ull;

// Per-Gaussian blend record written by K1, read by K7 once per (instance,
// tile).  64 B = two 32-B sectors.  fp64 fields feed the exact per-pixel
// circle test; the fp32 fields feed the per-pixel exponent.
struct __align__(16) BlendRec {
  double mx, my;   // mean2d (px), fp64 — rasterize lo/hi and _blend d (311)
  double r2;       // radius^2, fp64 (314)
  float qa, qb, qc;  // -0.5*log2(e)*(ca, 2cb, cc): power = qa dx^2 + qb dx dy + qc dy^2
  float log2_alpha;  // log2(sigmoid(logit))
  float cr, cg, cb;  // view colour
  float z;           // camera-space depth
};
static_assert(sizeof(BlendRec) == 64, "BlendRec must be 64 B");

// Tile rectangle, inclusive: x0 | y0 << 16 | x1 << 32 | y1 << 48 (empty -> count 0).
__host__ __device__ inline uint64_t pack_rect(uint32_t x0, uint32_t y0, uint32_t x1, uint32_t y1) {
  return (uint64_t)x0 | ((uint64_t)y0 << 16) | ((uint64_t)x1 << 32) | ((uint64_t)y1 << 48);
}

// The rect K1 writes for culled and off-screen splats: x1 + 1 == x0, so its
// area is 0 and its four coverage corners (K4c) cancel.
constexpr uint64_t kEmptyRect = 1ull;  // pack_rect(1, 0, 0, 0)

// Preferred shared-memory carveout (percent of the unified L1 / shared
// storage) for the view pipeline's kernels; -1 keeps the driver's choice.
// The streams' kernels co-reside on the SMs only when the SM's carveout fits
// them all, so one consistent carveout can matter more than each kernel's own.
#ifndef LMGS_CARVEOUT
#define LMGS_CARVEOUT -1
#endif
template <typename F>
inline void set_carveout(F* fn) {
  if (LMGS_CARVEOUT >= 0)
    cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                         cudaFuncAttributePreferredSharedMemoryCarveout, LMGS_CARVEOUT);
}

// Per-device launch caches (function attributes are per device context).
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 ? 0 : (d >= kMaxDevices ? kMaxDevices - 1 : d);
}

struct CamArgs {
  double r[9], t[3], center[3];
  double fx, fy, cx, cy, lim_x, lim_y;
  double inv_tile;  // 1 / tile_size (first guesses only; tile tests are exact)
  int32_t width, height, tile_size, tiles_x, tiles_y;
};

struct PreprocessArgs {
  const float* means;
  const float* quats;
  const float* scales;
  const float* logits;
  const float* sh;
  int64_t n;
  int32_t sh_coeffs;
  int32_t eval_degree;
  CamArgs cam;
  const uint8_t* page_mask;  // nullable: rows of pages with mask 0 are culled
  int32_t page_shift;
  // outputs
  uint64_t* depth_keys;    // [n] fp64 depth bits; kCulledKey if culled or off-screen
  uint64_t* rects;         // [n] inclusive tile rect (visible splats; count = its area)
  BlendRec* recs;          // [n]
  uint8_t* kept;           // [n] nullable
  int32_t* touched_zero;   // [n] nullable: zeroed here (the blend then adds to it)
  unsigned long long* n_kept;  // scalar (atomic): z > near
  unsigned long long* n_vis;   // scalar (atomic): tiles touched > 0
  unsigned long long* n_inst;  // scalar (atomic): sum of tile counts = K
  unsigned long long* zrange;  // [2] fp64 bits of min / max visible depth (atomic)
  // optional fp64 dump for lmgs_project
  double* dbg_mean2d;
  double* dbg_cov2d;
  double* dbg_depth;
  double* dbg_radius;
  float* dbg_colors;
  float* dbg_opacity;
};

int launch_preprocess(const PreprocessArgs& a, cudaStream_t s);  // returns kernels launched

// K1 over several views of the same Gaussians: every block stages its inputs
// once and projects them for each view (v[i] share the input arrays, n and
// page mask; outputs and counters are per view).
constexpr int kMaxPreViews = 8;
struct PreprocessMulti {
  PreprocessArgs v[kMaxPreViews];
  int32_t nv;
  int32_t persist_ctas;  // > 0: a persistent grid of this many CTAs per SM (set by the launcher's caller)
  int64_t n_blocks;      // full 128-row blocks (set by launch_preprocess_multi)
};
int launch_preprocess_multi(const PreprocessMulti& m, cudaStream_t s);

// ---------------------------------------------------------------------------
// LSD radix sort (onesweep: one histogram pass + one scatter pass per digit
// with decoupled look-back), 8-bit digits, u32/u64 keys, optional u32 values.
// The plan kernel detects trivial digits (all keys share it) and skips those
// passes on the device; the result buffers are published in device slots.

#ifndef LMGS_SORT_ITEMS
#define LMGS_SORT_ITEMS 16
#endif
#ifndef LMGS_SORT_MIN_CTAS
#define LMGS_SORT_MIN_CTAS 3
#endif
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kMaxPasses = 8;
constexpr int kSortThreads = 256;
constexpr int kSortItems = LMGS_SORT_ITEMS;  // keys per thread per onesweep tile
constexpr int kSortTile = kSortThreads * kSortItems;

struct RadixPlan {
  int32_t n_passes;
  int32_t first_active;  // first non-trivial pass (-1: none)
  int32_t last_active;   // last non-trivial pass (-1: none)
  int32_t active[kMaxPasses];
  int32_t src[kMaxPasses];
  int32_t result;
  int32_t pad[5];
  uint32_t digit_start[kMaxPasses][kRadix];
};

struct RadixSortBuffers {
  void* keys[2];       // uint32_t or uint64_t keys, ping-pong
  int key_bytes;       // 4 or 8
  uint32_t* vals[2];   // vals[0] == nullptr -> keys only
  RadixPlan* plan;     // device
  uint32_t* hist;      // [kMaxPasses * kRadix]
  uint32_t* lookback;  // [kMaxPasses * blocks * kRadix]
  uint32_t* counters;  // [kMaxPasses]
  const int* gate;     // nullable: device flag, 0 -> the whole sort is a no-op
  void** keys_result;  // nullable: device slot receiving the result key buffer
  void** vals_result;  // nullable: device slot receiving the result value buffer
  bool hist_ready;     // hist already holds every digit histogram (the producer built it)
  bool iota_vals;      // vals[0] is implicit: value = input index (never read)
  // nullable: the last data-moving pass adds the length of every run of equal
  // (key >> seg_shift) to seg_counts[key >> seg_shift] (zeroed by the caller);
  // the sorted key bits must cover the segment bits (tile sort: ranges)
  uint32_t* seg_counts;
  int seg_shift;
  // nullable: the key count on the device (n is then an upper bound sizing
  // the grid and the look-back; kernels use min(n, *n_dev); the onesweep
  // grid becomes persistent)
  const unsigned long long* n_dev;
  unsigned long long* max_n;  // nullable: atomicMax(*max_n, *n_dev) (overflow check)
  bool concurrent;            // LMGS_FLAG_CONCURRENT: persistent grids sharing the SMs
};

size_t radix_lookback_words(int64_t capacity);
// sorts bits [begin_bit, begin_bit + 8*n_passes) of n keys (stable).
int radix_sort(const RadixSortBuffers& b, int64_t n, int begin_bit, int n_passes,
               cudaStream_t s);  // returns kernels launched
// K5: stable sort of k keys tile << 32 | id on the tile bits [32, 32 +
// tile_bits); every pass runs and the last one writes the ids alone (uint32_t,
// in the buffer keys_result names).  seg_counts (required) gets the per-tile
// counts.  keys[0] holds the input; both buffers hold k u64 keys.
// id_bits: bits of the largest id (the 2-pass sort then runs its second pass
// on packed 4-byte keys when (tile_bits - 8) + id_bits <= 32)
int tile_sort(const RadixSortBuffers& b, int64_t k, int tile_bits, int id_bits, cudaStream_t s);

// K4+K5 fused (LMGS_FLAG_FUSED_TILE_SORT; two tile passes, (tile bits - 8) +
// id bits <= 32): k_emit_ranks writes the rank records and both digit
// histograms, the first pass generates its instance keys from the records
// instead of reading an emitted array and writes packed u32 keys, the second
// ranks those and writes the ids with the range counts (kSegLo).
int tile_sort_fused(const RadixSortBuffers& b, int64_t k, int id_bits, const uint4* rrec,
                    const uint32_t* chunk_first, const unsigned long long* n_vis_dev, int tiles_x,
                    cudaStream_t s);  // kernels launched

// Device-side slots naming where a sort's result landed (written by the plan
// kernel, read by consumers) so the pipeline never syncs on it.
struct DevSlots {
  void* depth_keys;  // K2 result: fp32 depth keys in (depth, id) order
  void* depth_ids;   // K2 result: Gaussian ids in (depth, id) order
  void* inst_ids;    // K5 result: uint32_t ids, sorted by tile then depth rank
  void* unused;
};

// ---------------------------------------------------------------------------
// depth order + instance emission + tile ranges (tiles.cu)

constexpr int kMaxTilePasses = 3;  // tile ids < 2^24

// K2a: 24-bit depth keys quantised over the view's visible depth range
// (monotone in the fp64 depth; kDepthKeyNone = invisible) + their digit
// histograms for the radix sort (kDepthPasses passes of 8 bits)
constexpr int kDepthPasses = 3;
constexpr uint32_t kDepthKeyNone = (1u << (8 * kDepthPasses)) - 1;
int launch_depth_keys(const uint64_t* key64, const unsigned long long* zrange, int64_t n,
                      uint32_t* key32, uint32_t* hist, cudaStream_t s);

// K2b: order runs of equal 32-bit keys by (fp64 depth, id) — _sort_order's exact key
int launch_depth_fixup(void* const* keys_slot, void* const* ids_slot, int64_t n,
                        const uint64_t* key64, const int64_t* prim_ids, cudaStream_t s);

// K4: walk Gaussians in depth order, scan their tile counts (decoupled
// look-back) and emit one key (tile << 32 | id) per overlapped tile — the
// instance array comes out sorted by depth rank, so a stable sort by tile
// alone yields rasterize's per-tile (depth, id) lists.  Also builds the tile
// digit histograms of the K5 radix passes.
#ifndef LMGS_EMIT_ITEMS
#define LMGS_EMIT_ITEMS 4  // 4: emit 0.182 -> 0.152 ms/view over 8 (profiles/r07/emit_shape_variants.txt)
#endif
#ifndef LMGS_EMIT_THREADS
#define LMGS_EMIT_THREADS 256
#endif
constexpr int kEmitThreads = LMGS_EMIT_THREADS;
constexpr int kEmitItems = LMGS_EMIT_ITEMS;
constexpr int kEmitChunk = kEmitThreads * kEmitItems;
struct EmitArgs {
  void* const* order_slot;  // -> uint32_t[n_vis] Gaussian ids in depth order
  const uint64_t* rects;    // count = rect area (every splat in rank order is visible)
  int64_t n_vis;            // host bound of the visible count (grid)
  const unsigned long long* n_vis_dev;  // the count itself
  uint64_t cap;             // keys capacity: instances past it are dropped (no-sync overflow)
  int32_t tiles_x;
  int32_t n_tile_passes;
  uint64_t* keys;           // [K] out
  uint64_t* lookback;       // [chunks] status words
  uint32_t* ticket;         // chunk ticket counter (zeroed)
  uint32_t* hist;           // [kMaxTilePasses][256] digit histograms (zeroed)
  bool concurrent;          // LMGS_FLAG_CONCURRENT: a persistent grid sharing the SMs
  // k_emit_ranks (fused tile sort)
  uint4* rrec;              // [n_vis] {rect lo, rect hi, id, first slot}
  uint32_t* chunk_first;    // [n_sort_tiles] rank holding each sort tile's first slot
  int64_t n_sort_tiles;
  const unsigned long long* k_dev;  // K (no histogram when it exceeds cap)
};
int launch_emit_ranks(const EmitArgs& a, cudaStream_t s);
#ifndef LMGS_EMIT_PERSIST_CTAS
#define LMGS_EMIT_PERSIST_CTAS 4  // > 0: concurrent renders emit with this many CTAs per SM
#endif
inline int64_t emit_chunks(int64_t n_vis) { return (n_vis + kEmitChunk - 1) / kEmitChunk; }
int launch_emit(const EmitArgs& a, cudaStream_t s);

// K6: tile ranges [start, end) = exclusive scan of the per-tile counts the
// tile sort's last pass accumulated (empty tiles included)
// (ranges are clamped to cap: a capacity-bounded render never reads past it)
int launch_ranges_from_counts(const uint32_t* counts, int tiles, int2* ranges, int64_t cap,
                              cudaStream_t s);

struct InstanceExportArgs {
  const int2* ranges;
  void* const* keys_slot;
  const int64_t* prim_ids;  // nullable: original ids
  uint64_t* keys_out;
  int64_t* prims_out;
  int64_t k;
  int tiles;
};
void launch_export_instances(const InstanceExportArgs& a, cudaStream_t s);

// ---------------------------------------------------------------------------
// blend (blend.cu) and compositing (raster.cu)

struct BlendArgs {
  void* const* keys_slot;  // -> uint32_t[K] ids, per tile in list order
  const int2* ranges;
  const BlendRec* recs;
  int32_t width, height, tile_size, tiles_x, tiles_y;
  int32_t subs_x;  // set by launch_blend: 64x64 sub-blocks per tile edge (> 1 above 64 px)
  float bg[3];
  float* rgb;
  float* alpha;
  float* depth;
  float* trans;
  int32_t* touched;
  int32_t* n_processed;
  int* work_counter;  // device scalar for the persistent 16x16 kernel (nullable)
  bool concurrent;    // LMGS_FLAG_CONCURRENT: the persistent grid leaves room on each SM
  // strip targets (lmgs_render_strips): when n_strips > 0, pixel row y goes to
  // strip y / strip_rows at row y % strip_rows of srgb / strans / sdepth
  // (possibly peer-GPU pointers) instead of rgb / alpha / depth / trans
  int32_t n_strips, strip_rows;
  // exact-touched fix-up queue (nullable): pixels (y * W + x) for the fp64
  // replay; fix_list holds W * H entries
  uint32_t* fix_count;
  uint32_t* fix_list;
  float fix_band;  // relative band around TERM_EPS that queues a pixel
  // exact n_processed (launch_nproc_fix): pixels K7b corrected and their fp64
  // break index per pixel (-1 = none; reset after use)
  const uint32_t* np_count;
  const uint32_t* np_list;
  const uint8_t* np_need;
  int32_t* np_override;
  float* srgb[8];
  float* strans[8];
  float* sdepth[8];
};

// the one place the blend kernels write a finished pixel
__device__ __forceinline__ void put_pixel(const BlendArgs& a, int x, int y, float T, float c0,
                                          float c1, float c2, float d) {
  const float r = fmaf(T, a.bg[0], c0), g = fmaf(T, a.bg[1], c1), b = fmaf(T, a.bg[2], c2);
  if (a.n_strips == 0) {
    const int64_t o = (int64_t)y * a.width + x;
    a.rgb[3 * o + 0] = r;
    a.rgb[3 * o + 1] = g;
    a.rgb[3 * o + 2] = b;
    if (a.alpha) a.alpha[o] = 1.0f - T;
    if (a.depth) a.depth[o] = d;
    if (a.trans) a.trans[o] = T;
  } else {
    const int s = y / a.strip_rows;
    const int64_t o = (int64_t)(y - s * a.strip_rows) * a.width + x;
    float* rgb = a.srgb[s];
    rgb[3 * o + 0] = r;
    rgb[3 * o + 1] = g;
    rgb[3 * o + 2] = b;
    if (a.strans[s]) a.strans[s][o] = T;
    if (a.sdepth[s]) a.sdepth[s][o] = d;
  }
}
int launch_blend(const BlendArgs& a, cudaStream_t s);  // returns 0 or LMGS_ERR_UNSUPPORTED
// after K7b: n_processed of the tiles holding a corrected pixel, recomputed
// exactly (returns kernels launched)
int launch_nproc_fix(const BlendArgs& a, cudaStream_t s);

void launch_fill_background(float* rgb, float* alpha, float* depth, float* trans, int64_t n_pix,
                            const float bg[3], cudaStream_t s);

// K7b: exact touched counts for the pixels the blend queued (touched_fix.cu)
struct TouchedFixArgs {
  void* const* keys_slot;
  const int2* ranges;
  const BlendRec* recs;
  int32_t tile_size, tiles_x, width;
  const uint32_t* fix_count;
  const uint32_t* fix_list;  // pixels y * width + x
  int32_t* touched;
  const float* means;
  const float* quats;
  const float* scales;
  const float* logits;
  CamArgs cam;
  // nullable: a replayed pixel whose fp64 break index differs from the fp32
  // one is appended to np_list (np_need: its tile must be recomputed) and its
  // fp64 index stored in np_override; n_processed is corrected in place
  uint32_t* np_count;
  uint32_t* np_list;
  uint8_t* np_need;
  int32_t* np_override;
  int32_t* n_processed;
};
int launch_touched_fix(const TouchedFixArgs& a, cudaStream_t s);

// Backward of the blend + chain to SH / logits (backward.cu), over the tile
// lists of the preceding render of the same view on the same context.
struct __align__(32) BwRec {  // fp64 splat of one view; the first 32 B are the cull data
  double mx, my, r2, op;
  double ca, cb, cc;
  double col[3];
  double rop;  // 1 / op
  double pad;
};
struct BackwardArgs {
  const float* means;
  const float* quats;
  const float* scales;
  const float* logits;
  const float* sh;
  int64_t n;
  int32_t sh_coeffs;
  int32_t eval_degree;
  CamArgs cam;
  void* const* keys_slot;
  const int2* ranges;
  int32_t width, height, tile_size, tiles_x;
  int32_t blocks_x, blocks;            // 8x4 pixel blocks across / per tile
  double bg[3];
  BwRec* recs;                         // [n] scratch
  const float* image_grad;  // [H,W,3]
  double* d_colors;         // [n,3]  (zeroed per view)
  double* d_opacities;      // [n]
  double* d_mean2d;         // [n,2]
  int32_t* touched;         // [n]
  double* d_sh;             // [n,coeffs,3] accumulated (nullable)
  double* d_logits;         // [n] accumulated (nullable)
  double* grad_norm_sum;    // [n] DensifyStats, accumulated (nullable)
  int64_t* steps_seen;      // [n] DensifyStats, accumulated (nullable)
};
int launch_backward(const BackwardArgs& a, int tiles, cudaStream_t s);  // kernels launched or -err

// RenderRecord collect (backward_exact.cu): fp64 sigma / t_before per (tile,
// instance, pixel) and t_final per pixel, from the view's BwRec records
struct CollectArgs {
  const BwRec* recs;
  void* const* keys_slot;
  const int2* ranges;
  const int64_t* offsets;  // [T] start of each tile's (K_t, P_t) block
  int32_t width, height, tile_size, tiles_x;
  double* sigma;
  double* t_before;
  double* t_final;         // [H*W]
};
int launch_collect(const BackwardArgs& prep, const CollectArgs& a, int tiles, cudaStream_t s);
int launch_backward_replay(const BackwardArgs& a, int tiles, cudaStream_t s);  // backward.cu

constexpr int kMaxCompositeBlocks = 64;
// `order` is a host array (n_blocks <= kMaxCompositeBlocks), passed by value.
void launch_composite(const float* rgb, const float* trans, const float* depth, int n_blocks,
                      const int32_t* order, int64_t n_pix, const float bg[3], float* out_rgb,
                      float* out_alpha, float* out_depth, cudaStream_t s);

}  // namespace lmgs
