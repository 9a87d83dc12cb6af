// K4 duplicate_with_keys, K6 identify_tile_ranges, background fill,
// instance export and K8 block composite.  (K7 blend lives in blend.cu.)
//
// Reference: rasterize (gaussian_core.py:340-403): tiles enumerated row-major
// (362-363) so tile_id = ty * tiles_x + tx; each tile's list is the splats
// whose bbox overlaps it (367-373) in (depth, prim_id) order (392).
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

// One thread per depth rank r: emit (tile << 32 | id) for every tile in the
// splat's rectangle, row-major, at its rank-order offset.  The stream is in
// depth order, so a stable sort on the tile bits alone yields per-tile lists
// in (depth, id) order; the low word carries the Gaussian row id so the blend
// reads its record without a rank -> id gather.
__global__ void __launch_bounds__(256) k_duplicate(DuplicateArgs a) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.n) return;
  const uint32_t* ids = static_cast<const uint32_t*>(a.slots->sorted_ids);
  const uint32_t id = ids[r];
  const uint32_t cnt = a.tile_counts[id];
  if (!cnt) return;
  const uint64_t rect = a.rects[id];
  const int x0 = (int)(rect & 0xffff), y0 = (int)((rect >> 16) & 0xffff);
  const int x1 = (int)((rect >> 32) & 0xffff), y1 = (int)((rect >> 48) & 0xffff);
  uint64_t off = a.offsets[r];
  for (int y = y0; y <= y1; ++y)
    for (int x = x0; x <= x1; ++x)
      a.keys_out[off++] = ((uint64_t)(uint32_t)(y * a.tiles_x + x) << 32) | (uint64_t)id;
}

__global__ void __launch_bounds__(256) k_tile_ranges(const DevSlots* slots, int64_t k,
                                                     int2* ranges) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const uint64_t* keys = static_cast<const uint64_t*>(slots->inst_keys);
  const uint32_t t = (uint32_t)(keys[i] >> 32);
  if (i == 0 || (uint32_t)(keys[i - 1] >> 32) != t) ranges[t].x = (int)i;
  if (i == k - 1 || (uint32_t)(keys[i + 1] >> 32) != t) ranges[t].y = (int)(i + 1);
}

__global__ void k_fill_bg(float* rgb, float* alpha, float* depth, float* trans, int64_t n,
                          float b0, float b1, float b2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  rgb[3 * i] = b0;
  rgb[3 * i + 1] = b1;
  rgb[3 * i + 2] = b2;
  if (alpha) alpha[i] = 0.0f;
  if (depth) depth[i] = 0.0f;
  if (trans) trans[i] = 1.0f;
}

__global__ void k_export(InstanceExportArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.k) return;
  const uint64_t key = static_cast<const uint64_t*>(a.slots->inst_keys)[i];
  if (a.keys_out) a.keys_out[i] = key;
  if (a.prims_out) {
    const uint32_t id = (uint32_t)key;
    a.prims_out[i] = a.prim_ids ? a.prim_ids[id] : (int64_t)id;
  }
}

struct BlockOrder {
  int32_t v[kMaxCompositeBlocks];
};

// Front-to-back "over" of per-block premultiplied renders (background 0):
// C = sum_b (prod_{b'<b} T_b') C_b + (prod_b T_b) bg.
__global__ void k_composite(const float* __restrict__ rgb, const float* __restrict__ trans,
                            const float* __restrict__ depth, int n_blocks, const BlockOrder order,
                            int64_t n_pix, float b0, float b1, float b2, float* out_rgb,
                            float* out_alpha, float* out_depth) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pix) return;
  float T = 1.0f, r = 0.f, g = 0.f, b = 0.f, d = 0.f;
  for (int k = 0; k < n_blocks; ++k) {
    const int64_t o = (int64_t)order.v[k] * n_pix + i;
    r = fmaf(T, rgb[3 * o + 0], r);
    g = fmaf(T, rgb[3 * o + 1], g);
    b = fmaf(T, rgb[3 * o + 2], b);
    if (depth) d = fmaf(T, depth[o], d);
    T *= trans[o];
  }
  out_rgb[3 * i + 0] = fmaf(T, b0, r);
  out_rgb[3 * i + 1] = fmaf(T, b1, g);
  out_rgb[3 * i + 2] = fmaf(T, b2, b);
  if (out_alpha) out_alpha[i] = 1.0f - T;
  if (out_depth) out_depth[i] = d;
}

}  // namespace

void launch_duplicate(const DuplicateArgs& a, cudaStream_t s) {
  if (a.n <= 0) return;
  k_duplicate<<<(unsigned)((a.n + 255) / 256), 256, 0, s>>>(a);
}

void launch_tile_ranges(const DevSlots* slots, int64_t k, int2* ranges, cudaStream_t s) {
  if (k <= 0) return;
  k_tile_ranges<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(slots, k, ranges);
}

void launch_fill_background(float* rgb, float* alpha, float* depth, float* trans, int64_t n_pix,
                            const float bg[3], cudaStream_t s) {
  if (n_pix <= 0) return;
  k_fill_bg<<<(unsigned)((n_pix + 255) / 256), 256, 0, s>>>(rgb, alpha, depth, trans, n_pix,
                                                            bg[0], bg[1], bg[2]);
}

void launch_export_instances(const InstanceExportArgs& a, cudaStream_t s) {
  if (a.k <= 0) return;
  k_export<<<(unsigned)((a.k + 255) / 256), 256, 0, s>>>(a);
}

void launch_composite(const float* rgb, const float* trans, const float* depth, int n_blocks,
                      const int32_t* order, int64_t n_pix, const float bg[3], float* out_rgb,
                      float* out_alpha, float* out_depth, cudaStream_t s) {
  if (n_pix <= 0) return;
  BlockOrder ord;
  for (int k = 0; k < n_blocks && k < kMaxCompositeBlocks; ++k) ord.v[k] = order[k];
  k_composite<<<(unsigned)((n_pix + 255) / 256), 256, 0, s>>>(
      rgb, trans, depth, n_blocks, ord, n_pix, bg[0], bg[1], bg[2], out_rgb, out_alpha,
      out_depth);
}

}  // namespace lmgs
