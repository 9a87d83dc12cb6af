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

struct CamArgs {
  double r[9], t[3], center[3];
  double fx, fy, cx, cy, lim_x, lim_y;
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
  // outputs
  uint32_t* depth_keys32;  // [n] bits(fp32 rd(depth)), 0xffffffff if culled
  uint64_t* depth_keys;    // [n] fp64 depth bits, kCulledKey if culled
  uint64_t* rects;         // [n]
  uint32_t* tile_counts;   // [n] tiles touched per Gaussian
  BlendRec* recs;          // [n]
  uint8_t* kept;           // [n] nullable
  unsigned long long* n_kept;  // scalar (atomic)
  uint64_t* sh_wait;           // set in-kernel: mbarrier guarding staged SH (TMA path)
  // optional fp64 dump for lmgs_project
  double* dbg_mean2d;
  double* dbg_cov2d;
  double* dbg_depth;
  double* dbg_radius;
  float* dbg_colors;
  float* dbg_opacity;
};

void launch_preprocess(const PreprocessArgs& a, cudaStream_t s);

// ---------------------------------------------------------------------------
// LSD radix sort (onesweep: one histogram pass + one scatter pass per digit
// with decoupled look-back), 8-bit digits, u32/u64 keys, optional u32 values.
// The plan kernel detects trivial digits (all keys share it) and skips those
// passes on the device; the result buffers are published in device slots.

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kMaxPasses = 8;
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;

struct RadixPlan {
  int32_t n_passes;
  int32_t active[kMaxPasses];
  int32_t src[kMaxPasses];
  int32_t result;
  int32_t pad[7];
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
};

size_t radix_lookback_words(int64_t capacity);
// sorts bits [begin_bit, begin_bit + 8*n_passes) of n keys (stable).
void radix_sort(const RadixSortBuffers& b, int64_t n, int begin_bit, int n_passes,
                cudaStream_t s);

// Device-side slots naming where a sort's result landed (written by the plan
// kernel, read by consumers) so the pipeline never syncs on it.
struct DevSlots {
  void* big_keys;  // oversized-bucket sort result keys
  void* big_vals;  // oversized-bucket sort result ids
};

// ---------------------------------------------------------------------------
// tile binning (tiles.cu)

// runs of equal fp32 depth keys up to this length are fixed up in registers
constexpr int kFixupRun = 32;
constexpr int kSmallTileCap = 2048;    // bucket sorted by a 256-thread CTA, 32 KB smem
constexpr int kMediumTileCap = 16384;  // bucket sorted by a 512-thread CTA, 208 KB smem

// K3a/K3b/K4: per-CTA (one per SM) tile histograms and placement
constexpr int kBinThreads = 1024;
constexpr int kSlabTiles = 49152;  // tile counters per shared-memory slab (192 KB)

struct BinArgs {
  const uint64_t* rects;
  const uint32_t* counts;   // tiles touched per Gaussian
  const uint32_t* key32;
  int64_t n;
  int32_t tiles_x;
  int32_t tiles;
  int32_t ctas;             // Gaussian slices (CTAs) of K3a / K4
  uint32_t* hist;           // [ctas][tiles] counts, then per-(cta, tile) offsets
  uint32_t* tile_count;     // [tiles] out of K3b
  const int2* ranges;       // K4 input
  uint32_t* bucket;         // [K] out of K4: Gaussian ids, arbitrary order within a tile
};
size_t bin_smem_bytes(int tiles);
void launch_bin_hist(const BinArgs& a, cudaStream_t s);   // K3a + K3b
void launch_bin_place(const BinArgs& a, cudaStream_t s);  // K4

struct TileScanArgs {
  const uint32_t* tile_count;  // [tiles]
  int tiles;
  int small_cap, medium_cap;
  int2* ranges;                // [tiles] out: [start, end)
  uint32_t* lists[3];          // [tiles] each: tile ids of class small/medium/big
  uint32_t* class_counts;      // [3]
  uint64_t* total;             // K
};
void launch_scan_tiles(const TileScanArgs& a, cudaStream_t s);

struct TileSortArgs {
  const uint32_t* bucket;
  const uint32_t* key32;  // [n] fp32 depth keys (L2-resident gather)
  const int2* ranges;
  const uint64_t* key64;  // [n] fp64 depth bits (exact tie order)
  uint32_t* sorted_ids;   // [K] out: per-tile lists in (depth, id) order
};
void launch_tile_sort(const TileSortArgs& a, const uint32_t* tile_list,
                      const uint32_t* list_count, int n_list, int cls, cudaStream_t s);
void launch_big_gather(const TileSortArgs& a, const uint32_t* big_list, int n_big,
                       const uint32_t* big_off, uint64_t* keys, uint32_t* vals, cudaStream_t s);
void launch_big_fixup(void* const* keys_ptr, void* const* vals_ptr, int64_t n,
                      const uint64_t* key64, cudaStream_t s);
void launch_big_scatter(const TileSortArgs& a, const uint32_t* big_list, int n_big,
                        const uint32_t* big_off, void* const* vals_ptr, cudaStream_t s);

struct InstanceExportArgs {
  const int2* ranges;
  const uint32_t* sorted_ids;
  const int64_t* prim_ids;  // nullable: original ids
  uint64_t* keys_out;
  int64_t* prims_out;
};
void launch_export_instances(const InstanceExportArgs& a, int tiles, cudaStream_t s);

// ---------------------------------------------------------------------------
// blend (blend.cu) and compositing (raster.cu)

struct BlendArgs {
  const uint32_t* sorted_ids;
  const int2* ranges;
  const BlendRec* recs;
  int32_t width, height, tile_size, tiles_x, tiles_y;
  float bg[3];
  float* rgb;
  float* alpha;
  float* depth;
  float* trans;
  int32_t* touched;
  int32_t* n_processed;
  int* work_counter;  // device scalar for the persistent 16x16 kernel (nullable)
};
int launch_blend(const BlendArgs& a, cudaStream_t s);  // returns 0 or LMGS_ERR_UNSUPPORTED

void launch_fill_background(float* rgb, float* alpha, float* depth, float* trans, int64_t n_pix,
                            const float bg[3], cudaStream_t s);

constexpr int kMaxCompositeBlocks = 64;
// `order` is a host array (n_blocks <= kMaxCompositeBlocks), passed by value.
void launch_composite(const float* rgb, const float* trans, const float* depth, int n_blocks,
                      const int32_t* order, int64_t n_pix, const float bg[3], float* out_rgb,
                      float* out_alpha, float* out_depth, cudaStream_t s);

}  // namespace lmgs
