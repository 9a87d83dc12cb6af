// K4 duplicate_with_keys, K6 identify_tile_ranges, K7 blend_tiles, K8 composite.
//
// Reference: rasterize (gaussian_core.py:340-403) and _blend (286-332).
//
// K7 keeps the reference's per-pixel semantics exactly where they are
// discrete: the 3-sigma circle test d.d <= r^2 (314) is decided in fp32 with
// a certified guard band and falls back to the fp64 expression inside the
// band; "active" is T >= TERM_EPS before each splat (315); touched counts
// pixels with w > 0 (323) — judged from the exponent, since an fp32 exp2 can
// underflow where the fp64 exp does not; the tile stops at the first splat
// after which no pixel is active (324-325).  The continuous part (exponent,
// alpha compositing) runs in fp32 with MUFU ex2.
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

// smallest float >= 1e-4: (double)T >= 1e-4  <=>  T >= kTermEpsF for fp32 T
constexpr float kTermEpsF = 1.00000005e-4f;
constexpr float kSigmaMaxF = 0.9999f;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(256) k_duplicate(DuplicateArgs a) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.n) return;
  const uint32_t* ids = a.ids[a.plan->result];
  const uint32_t id = ids[r];
  const uint32_t cnt = a.tile_counts[id];
  if (!cnt) return;
  const uint64_t rect = a.rects[id];
  const int x0 = (int)(rect & 0xffff), y0 = (int)((rect >> 16) & 0xffff);
  const int x1 = (int)((rect >> 32) & 0xffff), y1 = (int)((rect >> 48) & 0xffff);
  uint64_t off = a.offsets[r];
  for (int y = y0; y <= y1; ++y)
    for (int x = x0; x <= x1; ++x)
      a.keys_out[off++] = ((uint64_t)(uint32_t)(y * a.tiles_x + x) << 32) | (uint64_t)r;
}

__global__ void __launch_bounds__(256) k_tile_ranges(const uint64_t* keys_a,
                                                     const uint64_t* keys_b,
                                                     const RadixPlan* plan, int64_t k,
                                                     int2* ranges) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const uint64_t* keys = plan->result ? keys_b : keys_a;
  const uint32_t t = (uint32_t)(keys[i] >> 32);
  if (i == 0 || (uint32_t)(keys[i - 1] >> 32) != t) ranges[t].x = (int)i;
  if (i == k - 1 || (uint32_t)(keys[i + 1] >> 32) != t) ranges[t].y = (int)(i + 1);
}

template <int PPT>
__global__ void __launch_bounds__(256) k_blend(BlendArgs a) {
  constexpr int kBatch = 256;
  __shared__ float4 s_geo[kBatch];   // mx_local, my_local, qa, qb
  __shared__ float4 s_geo2[kBatch];  // qc, log2_alpha, r2_lo, r2_hi
  __shared__ float4 s_col[kBatch];   // r, g, b, z
  __shared__ double s_mx[kBatch], s_my[kBatch], s_r2[kBatch];
  __shared__ uint32_t s_id[kBatch];
  __shared__ int s_cnt[kBatch];
  __shared__ int s_last[32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthreads = blockDim.x;
  const int tile = blockIdx.x;
  const int ts = a.tile_size;
  const int tile_x = tile % a.tiles_x, tile_y = tile / a.tiles_x;
  const int x0 = tile_x * ts, y0 = tile_y * ts;
  const int2 range = a.ranges[tile];
  const uint64_t* __restrict__ keys = a.keys[a.key_plan->result];
  const uint32_t* __restrict__ ids = a.ids[a.id_plan->result];

  float T[PPT], C0[PPT], C1[PPT], C2[PPT], D[PPT], px[PPT], py[PPT];
  int last[PPT];
  bool valid[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int pix = tid + p * nthreads;
    const int lx = pix % ts, ly = pix / ts;
    valid[p] = pix < ts * ts && x0 + lx < a.width && y0 + ly < a.height;
    T[p] = valid[p] ? 1.0f : 0.0f;  // invalid pixels never go active
    C0[p] = C1[p] = C2[p] = D[p] = 0.0f;
    px[p] = (float)lx + 0.5f;  // _pixel_centers (335-337), tile-local
    py[p] = (float)ly + 0.5f;
    last[p] = -1;
  }

  for (int b0 = range.x; b0 < range.y; b0 += kBatch) {
    bool mine_active = false;
#pragma unroll
    for (int p = 0; p < PPT; ++p) mine_active |= T[p] >= kTermEpsF;
    if (__syncthreads_count(mine_active) == 0) break;
    const int nb = min(kBatch, range.y - b0);
    for (int j = tid; j < nb; j += nthreads) {
      const uint64_t key = keys[b0 + j];
      const uint32_t id = ids[(uint32_t)key];
      const BlendRec rec = a.recs[id];
      const double mxl = rec.mx - (double)x0, myl = rec.my - (double)y0;
      const double ax = fabs(mxl) + ts, ay = fabs(myl) + ts;
      const double band = (rec.r2 + ax * ax + ay * ay) * 0x1p-18;
      s_geo[j] = make_float4((float)mxl, (float)myl, rec.qa, rec.qb);
      s_geo2[j] = make_float4(rec.qc, rec.log2_alpha, __double2float_rd(rec.r2 - band),
                              __double2float_ru(rec.r2 + band));
      s_col[j] = make_float4(rec.cr, rec.cg, rec.cb, rec.z);
      s_mx[j] = rec.mx;
      s_my[j] = rec.my;
      s_r2[j] = rec.r2;
      s_id[j] = id;
      s_cnt[j] = 0;
    }
    __syncthreads();
    for (int k = 0; k < nb; ++k) {
      const float4 g = s_geo[k];
      const float4 h = s_geo2[k];
      const float4 c = s_col[k];
      int cnt = 0;
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        if (T[p] >= kTermEpsF) {
          const float dx = px[p] - g.x, dy = py[p] - g.y;
          const float d2 = fmaf(dx, dx, dy * dy);
          bool inside = d2 <= h.z;
          if (!inside && d2 <= h.w) {
            // guard band: the reference's fp64 test, bit for bit
            const double ddx = ((double)(x0 + (int)(px[p] - 0.5f)) + 0.5) - s_mx[k];
            const double ddy = ((double)(y0 + (int)(py[p] - 0.5f)) + 0.5) - s_my[k];
            inside = __dadd_rn(__dmul_rn(ddx, ddx), __dmul_rn(ddy, ddy)) <= s_r2[k];
          }
          if (inside) {
            const float power = fmaf(fmaf(g.z, dx, g.w * dy), dx, fmaf(h.x * dy, dy, h.y));
            bool contrib = power > -1060.0f;
            if (!contrib && power >= -1080.0f)
              contrib = exp2((double)power) * (double)T[p] > 0.0;
            const float sig = fminf(ex2_approx(power), kSigmaMaxF);
            const float w = T[p] * sig;
            C0[p] = fmaf(w, c.x, C0[p]);
            C1[p] = fmaf(w, c.y, C1[p]);
            C2[p] = fmaf(w, c.z, C2[p]);
            D[p] = fmaf(w, c.w, D[p]);
            T[p] = T[p] * (1.0f - sig);
            cnt += contrib;
            if (T[p] < kTermEpsF) last[p] = b0 - range.x + k;
          }
        }
      }
      const int wsum = __reduce_add_sync(0xffffffffu, cnt);
      if (lane == 0 && wsum) atomicAdd(&s_cnt[k], wsum);
    }
    __syncthreads();
    if (a.touched)
      for (int j = tid; j < nb; j += nthreads)
        if (s_cnt[j]) atomicAdd(a.touched + s_id[j], s_cnt[j]);
  }

  // n_processed: the break index of _blend's loop (324-325)
  int my_last = -1;
  bool my_live = false;
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    my_last = max(my_last, last[p]);
    my_live |= valid[p] && T[p] >= kTermEpsF;
  }
  const int any_live = __syncthreads_or(my_live);
  if (a.n_processed) {
    int v = my_last;
#pragma unroll
    for (int off = 16; off; off >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) s_last[warp] = v;
    __syncthreads();
    if (tid == 0) {
      int m = -1;
      for (int w = 0; w < (nthreads + 31) / 32; ++w) m = max(m, s_last[w]);
      a.n_processed[tile] = any_live ? (range.y - range.x) : (m + 1);
    }
  }
  // outputs: C + T * bg (326), alpha = 1 - T_final, depth, T_final
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    if (!valid[p]) continue;
    const int pix = tid + p * nthreads;
    const int64_t o = (int64_t)(y0 + pix / ts) * a.width + (x0 + pix % ts);
    a.rgb[3 * o + 0] = fmaf(T[p], a.bg[0], C0[p]);
    a.rgb[3 * o + 1] = fmaf(T[p], a.bg[1], C1[p]);
    a.rgb[3 * o + 2] = fmaf(T[p], a.bg[2], C2[p]);
    if (a.alpha) a.alpha[o] = 1.0f - T[p];
    if (a.depth) a.depth[o] = D[p];
    if (a.trans) a.trans[o] = T[p];
  }
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
  const uint64_t key = a.keys[a.key_plan->result][i];
  if (a.keys_out) a.keys_out[i] = key;
  if (a.prims_out) {
    const uint32_t id = a.ids[a.id_plan->result][(uint32_t)key];
    a.prims_out[i] = a.prim_ids ? a.prim_ids[id] : (int64_t)id;
  }
}

// front-to-back "over" of per-block premultiplied renders
struct BlockOrder {
  int32_t v[kMaxCompositeBlocks];
};

__global__ void k_composite(const float* __restrict__ rgb, const float* __restrict__ trans,
                            const float* __restrict__ depth, int n_blocks,
                            const BlockOrder order, int64_t n_pix, float b0, float b1,
                            float b2, float* out_rgb, float* out_alpha, float* out_depth) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pix) return;
  float T = 1.0f, r = 0.f, g = 0.f, b = 0.f, d = 0.f;
  for (int k = 0; k < n_blocks; ++k) {
    const int64_t blk = order.v[k];
    const int64_t o = blk * n_pix + i;
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

void launch_tile_ranges(const uint64_t* keys_a, const uint64_t* keys_b, const RadixPlan* plan,
                        int64_t k, int2* ranges, cudaStream_t s) {
  if (k <= 0) return;
  k_tile_ranges<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(keys_a, keys_b, plan, k, ranges);
}

int launch_blend(const BlendArgs& a, cudaStream_t s) {
  const int ts = a.tile_size;
  const int tiles = a.tiles_x * a.tiles_y;
  if (tiles <= 0) return 0;
  if (ts <= 16) {
    const int threads = ((ts * ts + 31) / 32) * 32;
    k_blend<1><<<tiles, threads, 0, s>>>(a);
  } else if (ts <= 32) {
    k_blend<4><<<tiles, 256, 0, s>>>(a);
  } else if (ts <= 64) {
    k_blend<16><<<tiles, 256, 0, s>>>(a);
  } else {
    return LMGS_ERR_UNSUPPORTED;
  }
  return 0;
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
