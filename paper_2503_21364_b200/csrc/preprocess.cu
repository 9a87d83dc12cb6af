// K1 preprocess: near cull, fp64 EWA projection, tile rectangle + count,
// SH colour, blend record.  One thread per Gaussian.
//
// Reference: project_splats (gaussian_core.py:187-230), quat_to_rotmat
// (93-102), covariance_3d (105-117), eval_sh_colors (129-142), and the tile
// overlap predicate of rasterize (362-373) restated as an inclusive tile
// rectangle.
//
// This file is compiled with -fmad=false: every fp64 operation rounds exactly
// where torch's does.  The products torch hands to MKL dgemm (means @ r_wc.T,
// j @ r_wc) are written as the explicit FMA chain MKL evaluates; the bmm
// products (covariance, jw @ cov3d @ jw^T) as plain sequential sums.  The
// only deviation: sqrt here is IEEE-rounded while torch.sqrt (MKL VML) is
// <= 1 ulp low on ~0.7% of inputs.
#include "device_util.cuh"
#include "geometry.cuh"
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

// Inclusive tile index range [a, b] along one axis for lo/hi of a splat's
// bbox, identical to the reference comparisons hi >= t0 and lo <= t0 + tw
// with tw = min(ts, size - t0).  Empty when a > b.
__device__ __forceinline__ void axis_range(double lo, double hi, int size, int ts, double its,
                                           int nt, int* a, int* b) {
  int j;
  if (!(lo > -2.0 * ts)) j = 0;
  else if (lo > (double)size + 2.0 * ts) j = nt;
  else j = max((int)floor(lo * its) - 2, 0);  // a guess: the loops below are exact
  while (j < nt) {
    int end = min((j + 1) * ts, size);
    if (lo <= (double)end) break;
    ++j;
  }
  int k;
  if (!(hi < (double)size + 2.0 * ts)) k = nt - 1;
  else if (hi < -2.0 * ts) k = -1;
  else k = min((int)floor(hi * its) + 2, nt - 1);
  while (k >= 0 && !((double)(k * ts) <= hi)) --k;
  *a = j;
  *b = k;
}

// Colour along centre->mean; degree <= 1 is eval_sh_colors (129-142),
// degrees 2-3 extend it with the standard real SH basis, clamp(0,1), no +0.5.
template <bool SMEM>
__device__ __forceinline__ void sh_color(const float* __restrict__ sh, int ncoef, int deg,
                                         float x, float y, float z, float out[3]) {
  const float C0 = (float)kShC0, C1 = (float)kShC1;
  float c[3];
  const float4* sh4 = reinterpret_cast<const float4*>(sh);
  // coefficients 0..3 (12 floats = 3 float4)
  float v[48];
  int nload = ncoef * 3;
  if ((reinterpret_cast<uintptr_t>(sh) & 15) == 0 && (nload & 3) == 0) {
#pragma unroll
    for (int q = 0; q < 12; ++q) {
      if (4 * q < nload) {
        const float4 f = SMEM ? sh4[q] : __ldg(sh4 + q);
        v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < 48; ++q)
      if (q < nload) v[q] = SMEM ? sh[q] : __ldg(sh + q);
  }
  // fp32 colour (the image tolerance, 1e-4, not bit-exactness, applies): this
  // file is built with -fmad=false for the fp64 geometry, so the colour's
  // multiply-adds are written as explicit FMAs (half the instructions)
  const float b1 = -C1 * y, b2 = C1 * z, b3 = -C1 * x;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) c[ch] = C0 * v[ch];
  if (deg >= 1 && ncoef >= 4) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
      c[ch] = __fmaf_rn(b3, v[9 + ch], __fmaf_rn(b2, v[6 + ch], __fmaf_rn(b1, v[3 + ch], c[ch])));
  }
  if (deg >= 2 && ncoef >= 9) {
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    const float b[5] = {1.0925484305920792f * xy, -1.0925484305920792f * yz,
                        0.31539156525252005f * (2.0f * zz - xx - yy),
                        -1.0925484305920792f * xz, 0.5462742152960396f * (xx - yy)};
#pragma unroll
    for (int k = 0; k < 5; ++k)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) c[ch] = __fmaf_rn(b[k], v[12 + 3 * k + ch], c[ch]);
    if (deg >= 3 && ncoef >= 16) {
      const float d[7] = {-0.5900435899266435f * y * (3.0f * xx - yy),
                          2.890611442640554f * xy * z,
                          -0.4570457994644658f * y * (4.0f * zz - xx - yy),
                          0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy),
                          -0.4570457994644658f * x * (4.0f * zz - xx - yy),
                          1.445305721320277f * z * (xx - yy),
                          -0.5900435899266435f * x * (xx - 3.0f * yy)};
#pragma unroll
      for (int k = 0; k < 7; ++k)
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) c[ch] = __fmaf_rn(d[k], v[27 + 3 * k + ch], c[ch]);
    }
  }
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) out[ch] = fminf(fmaxf(c[ch], 0.0f), 1.0f);
}


// One Gaussian.  Inputs arrive as values (from shared memory staged by TMA or
// straight from global memory); `sh` points at its coefficients.
#ifndef LMGS_PRE_THREADS
#define LMGS_PRE_THREADS 128
#endif
#ifndef LMGS_PRE_MIN_CTAS
#define LMGS_PRE_MIN_CTAS 7
#endif
// Gaussians (threads) per CTA in both kernels; count_kept reduces over its warps.
// 128 x 7 CTAs per SM: 28 warps to hide the fp64 dependency chains, 7 x 30 KB
// of TMA-staged inputs in flight per SM.
constexpr int kPreThreads = LMGS_PRE_THREADS;
static_assert(kPreThreads == 128, "paged sets map one K1 block to one 128-row page");

// Returns the splat's tile count (0: culled or off-screen); *keep = near-kept.
// S (nullable): the Gaussian's world covariance, computed once for all the
// views of a block (covariance_3d is view-independent)
template <bool SMEM>
__device__ __forceinline__ uint32_t process_one(const PreprocessArgs& a, int64_t i, double m0, double m1,
                                            double m2, float4 q, double s0, double s1, double s2,
                                            float logit, const float* sh, uint64_t* sh_wait,
                                            bool* keep_out, uint64_t* zbits_out,
                                            const double* S = nullptr, uint32_t sh_phase = 0) {
  bool keep = false;
  uint32_t cnt = 0;
  uint64_t zb = 0;
  {
    const CamArgs& cam = a.cam;
    // p = means @ r_wc.T + t_wc (195): MKL FMA chain, then + t
    const double x = mkl_dot3(m0, cam.r[0], m1, cam.r[1], m2, cam.r[2]) + cam.t[0];
    const double y = mkl_dot3(m0, cam.r[3], m1, cam.r[4], m2, cam.r[5]) + cam.t[1];
    const double z = mkl_dot3(m0, cam.r[6], m1, cam.r[7], m2, cam.r[8]) + cam.t[2];
    keep = z > kNearCullZ;  // 196
    if (a.kept) a.kept[i] = keep;
    if (a.touched_zero) a.touched_zero[i] = 0;
    if (!keep) {
      a.depth_keys[i] = kCulledKey;
      a.rects[i] = kEmptyRect;
    } else {
      double mx, my, ca, cb, cc, radius;
      if (S) splat_projection(cam, x, y, z, S, &mx, &my, &ca, &cb, &cc, &radius);
      else splat_geometry(cam, x, y, z, q, s0, s1, s2, &mx, &my, &ca, &cb, &cc, &radius);
      // tile rectangle (362-373)
      int x0, x1, y0, y1;
      axis_range(mx - radius, mx + radius, cam.width, cam.tile_size, cam.inv_tile, cam.tiles_x, &x0,
                 &x1);
      axis_range(my - radius, my + radius, cam.height, cam.tile_size, cam.inv_tile, cam.tiles_y, &y0,
                 &y1);
      if (x0 <= x1 && y0 <= y1) cnt = (uint32_t)(x1 - x0 + 1) * (uint32_t)(y1 - y0 + 1);
      a.rects[i] = cnt ? pack_rect(x0, y0, x1, y1) : kEmptyRect;
      // off-screen splats sort behind every visible one (K2 orders only the
      // n_vis visible splats)
      zb = (uint64_t)__double_as_longlong(z);
      a.depth_keys[i] = cnt ? zb : kCulledKey;
      // conic (_blend 309-310), fp64 then pre-scaled to the exp2 domain in fp32
      // (the fp32 conic below is the blend's; one reciprocal instead of three
      // divisions changes it by < 1 fp64 ulp before the fp32 rounding)
      const double det = ca * cc - cb * cb;
      const double rdet = 1.0 / det;
      const double ica = cc * rdet, icb = -cb * rdet, icc = ca * rdet;
      const float log2_alpha =
          logit < -15.0f ? logit * (float)kLog2e : -log2f(1.0f + expf(-logit));
      float col[3] = {0.f, 0.f, 0.f};
      if (SMEM) mbar_wait(sh_wait, sh_phase);
      if (cnt || a.dbg_colors) {
        const double dx = m0 - cam.center[0], dy = m1 - cam.center[1], dz = m2 - cam.center[2];
        double nrm = sqrt((dx * dx + dy * dy) + dz * dz);
        nrm = fmax(nrm, 1e-12);
        const double rn = 1.0 / nrm;
        sh_color<SMEM>(sh, a.sh_coeffs, a.eval_degree,
                 (float)(dx * rn), (float)(dy * rn), (float)(dz * rn), col);
      }
      BlendRec rec;
      rec.mx = mx;
      rec.my = my;
      rec.r2 = radius * radius;
      rec.qa = (float)(-0.5 * kLog2e * ica);
      rec.qb = (float)(-kLog2e * icb);
      rec.qc = (float)(-0.5 * kLog2e * icc);
      rec.log2_alpha = log2_alpha;
      rec.cr = col[0];
      rec.cg = col[1];
      rec.cb = col[2];
      rec.z = (float)z;
      a.recs[i] = rec;
      if (a.dbg_mean2d) {
        a.dbg_mean2d[2 * i] = mx;
        a.dbg_mean2d[2 * i + 1] = my;
        a.dbg_cov2d[3 * i] = ca;
        a.dbg_cov2d[3 * i + 1] = cb;
        a.dbg_cov2d[3 * i + 2] = cc;
        a.dbg_depth[i] = z;
        a.dbg_radius[i] = radius;
        a.dbg_colors[3 * i] = col[0];
        a.dbg_colors[3 * i + 1] = col[1];
        a.dbg_colors[3 * i + 2] = col[2];
        a.dbg_opacity[i] = (float)(1.0 / (1.0 + exp(-(double)logit)));
      }
    }
  }
  *keep_out = keep;
  *zbits_out = zb;
  return cnt;
}

// block-aggregated counters: near-kept splats (M), visible splats, instances
// (K), and the visible depth range (positive fp64 bits order like integers).
// One atomic per counter per CTA: per-warp atomics on these five addresses
// serialised in L2 and doubled the kernel's time.  `slot` = the view within a
// multi-view block (its own shared partials, so views need no extra barrier).
// Warp sums and extrema are single REDUX instructions on 32-bit values: the
// per-warp instance count fits (< 32 * 2^24 tiles), and the depth range is
// kept at the resolution of the fp64 bits' high word, widened outward (min
// with low word 0, max with low word ~0).  K2 only needs a range that covers
// every visible depth: its keys stay monotone and the exact fp64 order is
// restored inside equal-key runs (k_depth_fixup).
__device__ __forceinline__ void count_kept(const PreprocessArgs& a, bool keep, uint32_t cnt,
                                           uint64_t zbits, int slot = 0) {
  __shared__ uint32_t s_acc_all[kMaxPreViews][kPreThreads / 32][5];
  auto& s_acc = s_acc_all[slot];
  const unsigned ballot = __ballot_sync(0xffffffffu, keep);
  const unsigned vis = __ballot_sync(0xffffffffu, cnt > 0);
  const uint32_t zh = (uint32_t)(zbits >> 32);
  const uint32_t k = __reduce_add_sync(0xffffffffu, cnt);
  const uint32_t zlo = __reduce_min_sync(0xffffffffu, cnt ? zh : 0xffffffffu);
  const uint32_t zhi = __reduce_max_sync(0xffffffffu, cnt ? zh : 0u);
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_acc[warp][0] = __popc(ballot);
    s_acc[warp][1] = __popc(vis);
    s_acc[warp][2] = k;
    s_acc[warp][3] = zlo;
    s_acc[warp][4] = zhi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long kept = 0, nv = 0, inst = 0;
    uint32_t lo = 0xffffffffu, hi = 0u;
    for (int w = 0; w < kPreThreads / 32; ++w) {
      kept += s_acc[w][0];
      nv += s_acc[w][1];
      inst += s_acc[w][2];
      lo = min(lo, s_acc[w][3]);
      hi = max(hi, s_acc[w][4]);
    }
    if (kept) atomicAdd(a.n_kept, kept);
    if (nv) {
      atomicAdd(a.n_vis, nv);
      atomicMin(a.zrange, (unsigned long long)lo << 32);
      atomicMax(a.zrange + 1, ((unsigned long long)hi << 32) | 0xffffffffull);
    }
    if (inst) atomicAdd(a.n_inst, inst);
  }
}

// a row of an inactive page (paged sets): culled
__device__ __forceinline__ void cull_row(const PreprocessArgs& a, int64_t i) {
  if (a.kept) a.kept[i] = 0;
  if (a.touched_zero) a.touched_zero[i] = 0;
  a.depth_keys[i] = kCulledKey;
  a.rects[i] = kEmptyRect;
}

// direct loads (tail block, unaligned inputs)
__global__ void __launch_bounds__(kPreThreads) k_preprocess_direct(
    const __grid_constant__ PreprocessMulti m, int64_t first) {
  const PreprocessArgs& a0 = m.v[0];
  const int64_t i = first + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < a0.n;
  const bool dead = live && a0.page_mask && (int)(i & 127) >= (int)a0.page_mask[i >> 7];
  for (int vi = 0; vi < m.nv; ++vi) {
    const PreprocessArgs& a = m.v[vi];
    bool keep = false;
    uint32_t cnt = 0;
    uint64_t zb = 0;
    if (dead) {
      cull_row(a, i);
    } else if (live) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(a.quats) + i);
      cnt = process_one<false>(a, i, a.means[3 * i], a.means[3 * i + 1], a.means[3 * i + 2], q,
                               a.scales[3 * i], a.scales[3 * i + 1], a.scales[3 * i + 2],
                               a.logits[i], a.sh + i * a.sh_coeffs * 3, nullptr, &keep, &zb);
    }
    count_kept(a, keep, cnt, zb, vi);
  }
}

// ---------------------------------------------------------------------------
// TMA-staged path: one thread issues cp.async.bulk copies of the block's
// means / quats / scales / logits (one mbarrier) and of its SH coefficients
// (a second mbarrier); the SH bytes stream into shared memory while the fp64
// geometry of the block is being computed.  With several views the staged
// block is projected once per view: the 236 B/Gaussian of inputs are read
// from HBM once per group of views instead of once per view.

// NV (= m.nv) is a template argument so that every view's camera and output
// pointers are constant-bank operands: with a runtime view index they would be
// loaded into registers (and spill).
// Views after the first keep more state in flight (the unrolled view bodies
// overlap); at 7 CTAs/SM (72 registers) they spill, so a multi-view block
// runs at LMGS_PRE_MULTI_MIN_CTAS.
#ifndef LMGS_PRE_VIEW_BARRIER
#define LMGS_PRE_VIEW_BARRIER 1
#endif
#ifndef LMGS_PRE_MULTI_MIN_CTAS
#define LMGS_PRE_MULTI_MIN_CTAS 5
#endif
template <int NV, bool LOOP>
__global__ void __launch_bounds__(kPreThreads, NV == 1 ? LMGS_PRE_MIN_CTAS : LMGS_PRE_MULTI_MIN_CTAS)
    k_preprocess_tma(
    const __grid_constant__ PreprocessMulti m) {
  const PreprocessArgs& a = m.v[0];  // inputs (shared by every view)
  extern __shared__ __align__(128) float smem_f[];
  float* s_means = smem_f;                       // [256*3]
  float* s_quats = s_means + kPreThreads * 3;    // [256*4]
  float* s_scales = s_quats + kPreThreads * 4;   // [256*3]
  float* s_logits = s_scales + kPreThreads * 3;  // [256]
  float* s_sh = s_logits + kPreThreads;          // [256*ncoef*3]
  __shared__ __align__(8) uint64_t s_bar[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_init_fence();
  }
  __syncthreads();
  // one block per CTA, or (m.blocks_per_cta: concurrent renders) a persistent
  // grid walking blocks, the barriers' phase flipping every block
  uint32_t phase = 0;
  for (int64_t blk = blockIdx.x; blk < m.n_blocks; blk += LOOP ? gridDim.x : m.n_blocks, phase ^= 1) {
  const int64_t i0 = blk * kPreThreads;
  if (a.page_mask && a.page_mask[i0 >> 7] == 0) {  // the block is one inactive page
#pragma unroll
    for (int vi = 0; vi < NV; ++vi) {
      cull_row(m.v[vi], i0 + tid);
      count_kept(m.v[vi], false, 0, 0, vi);
    }
    continue;
  }
  const uint32_t sh_bytes = (uint32_t)(kPreThreads * a.sh_coeffs * 3 * 4);
  if (tid == 0) {
    mbar_expect_tx(&s_bar[0], kPreThreads * (12 + 16 + 12 + 4));
    bulk_g2s(s_means, a.means + i0 * 3, kPreThreads * 12, &s_bar[0]);
    bulk_g2s(s_quats, a.quats + i0 * 4, kPreThreads * 16, &s_bar[0]);
    bulk_g2s(s_scales, a.scales + i0 * 3, kPreThreads * 12, &s_bar[0]);
    bulk_g2s(s_logits, a.logits + i0, kPreThreads * 4, &s_bar[0]);
    mbar_expect_tx(&s_bar[1], sh_bytes);
    bulk_g2s(s_sh, a.sh + i0 * a.sh_coeffs * 3, sh_bytes, &s_bar[1]);
  }
  mbar_wait(&s_bar[0], phase);
  const int64_t i = i0 + tid;
  const bool dead = a.page_mask && tid >= (int)a.page_mask[i0 >> 7];  // past the page's live rows
  // the world covariance once for the whole group of views
  double S[6];
  if (NV > 1 && !dead)
    covariance_3d(reinterpret_cast<const float4*>(s_quats)[tid], s_scales[3 * tid],
                  s_scales[3 * tid + 1], s_scales[3 * tid + 2], S);
#pragma unroll
  for (int vi = 0; vi < NV; ++vi) {
    // re-read the staged inputs every view (a compiler barrier keeps them
    // from being hoisted into registers that would live across views)
#if LMGS_PRE_VIEW_BARRIER
    asm volatile("" ::: "memory");
#endif
    const float4 q = reinterpret_cast<const float4*>(s_quats)[tid];
    const PreprocessArgs& av = m.v[vi];
    bool keep = false;
    uint32_t cnt = 0;
    uint64_t zb = 0;
    if (dead) {
      cull_row(av, i);
    } else {
      // the SH wait happens inside process_one just before the colour is needed
      cnt = process_one<true>(av, i, s_means[3 * tid], s_means[3 * tid + 1], s_means[3 * tid + 2],
                              q, s_scales[3 * tid], s_scales[3 * tid + 1], s_scales[3 * tid + 2],
                              s_logits[tid], s_sh + tid * a.sh_coeffs * 3, &s_bar[1], &keep, &zb,
                              NV > 1 ? S : nullptr, phase);
    }
    count_kept(av, keep, cnt, zb, vi);
  }
  // every thread must observe the SH barrier before the block may exit (or
  // the staging be refilled)
  mbar_wait(&s_bar[1], phase);
  if (!LOOP) break;
  fence_proxy_async_smem();  // this block's shared reads before the next block's TMA writes
  __syncthreads();
  }
}


}  // namespace

int launch_preprocess(const PreprocessArgs& a, cudaStream_t s) {
  PreprocessMulti m{};
  m.v[0] = a;
  m.nv = 1;
  return launch_preprocess_multi(m, s);
}

int launch_preprocess_multi(const PreprocessMulti& m, cudaStream_t s) {
  const PreprocessArgs& a = m.v[0];
  if (a.n <= 0 || m.nv < 1 || m.nv > kMaxPreViews) return 0;
  int launched = 0;
  // full blocks through TMA when every chunk is 16-byte aligned and sized
  const bool aligned =
      ((reinterpret_cast<uintptr_t>(a.means) | reinterpret_cast<uintptr_t>(a.quats) |
        reinterpret_cast<uintptr_t>(a.scales) | reinterpret_cast<uintptr_t>(a.logits) |
        reinterpret_cast<uintptr_t>(a.sh)) & 15) == 0;
  const int64_t full = aligned ? a.n / kPreThreads : 0;
  if (full > 0) {
    const size_t smem = sizeof(float) * kPreThreads * (3 + 4 + 3 + 1 + 3 * a.sh_coeffs);
    static size_t set[2 * kMaxPreViews][kMaxDevices] = {};
    const int dev = current_device();
    void (*kern)(PreprocessMulti) = nullptr;
    const bool loop = m.persist_ctas > 0;
    switch (m.nv) {
      case 1: kern = loop ? k_preprocess_tma<1, true> : k_preprocess_tma<1, false>; break;
      case 2: kern = loop ? k_preprocess_tma<2, true> : k_preprocess_tma<2, false>; break;
      case 3: kern = loop ? k_preprocess_tma<3, true> : k_preprocess_tma<3, false>; break;
      case 4: kern = loop ? k_preprocess_tma<4, true> : k_preprocess_tma<4, false>; break;
      case 5: kern = k_preprocess_tma<5, false>; break;
      case 6: kern = k_preprocess_tma<6, false>; break;
      case 7: kern = k_preprocess_tma<7, false>; break;
      default: kern = k_preprocess_tma<8, false>; break;
    }
    const int slot = (m.nv - 1) * 2 + (loop && m.nv <= 4 ? 1 : 0);
    if (smem > set[slot][dev]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      set_carveout(kern);
      set[slot][dev] = smem;
    }
    PreprocessMulti mm = m;
    mm.n_blocks = full;
    int64_t grid = full;
    if (loop && m.nv <= 4) {
      static int sms[kMaxDevices] = {};
      if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
      const int64_t p = (int64_t)sms[dev] * m.persist_ctas;
      if (grid > p) grid = p;
    }
    kern<<<(unsigned)grid, kPreThreads, smem, s>>>(mm);
    ++launched;
  }
  const int64_t first = full * kPreThreads;
  const int64_t rest = a.n - first;
  if (rest > 0) {
    k_preprocess_direct<<<(unsigned)((rest + kPreThreads - 1) / kPreThreads), kPreThreads, 0, s>>>(
        m, first);
    ++launched;
  }
  return launched;
}

}  // namespace lmgs
