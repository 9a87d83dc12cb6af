// Backward of the blend, the per-pixel replay:
// backward_render (gaussian_core.py:438-486) over the tile lists of the
// preceding render on the same context, from the fp64 splat records of
// backward_exact.cu.  fp64 throughout; this file is compiled with FMA
// contraction (the replay's sums are checked at rtol 1e-9, not bit for bit)
// except the circle test, which is written with explicit rounding so it
// decides exactly as the reference's (d.d).sum <= r^2.
//
// One 32-thread CTA per 8x4 pixel block of a tile, one pixel per lane:
//   pass A  the forward blend in fp64 -> every pixel's total colour C_tot
//           (including T_final * background);
//   pass B  the forward blend again; at each applied step the reference's
//           reverse-mode quantities: w = T_before sigma, suffix = C_tot - sum
//           of w c up to and including this step (the reference accumulates
//           the same suffix back to front), d_sigma = g . (c T_before -
//           suffix / max(1 - sigma, 1e-6)); the six per-splat sums (g w,
//           d_sigma sigma / alpha, d_sigma sigma (conic @ (pix - mean))) are
//           reduced across the warp with 8 fp64 shuffles and added to global
//           memory by six owner lanes; touched = popc(ballot(w > 0)).
// A pixel stops when its T < TERM_EPS (later steps have sigma = 0: no
// contribution), a block when all its pixels have.  Splats whose circle
// misses the box of a block's live pixels are skipped (exact).
#include <climits>

#include "device_util.cuh"
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

#ifdef LMGS_BW_COUNT
__device__ unsigned long long g_bw_count[2][4];
}  // namespace
}  // namespace lmgs
extern "C" int lmgs_debug_bw_count(unsigned long long* host_out) {
  return (int)cudaMemcpyFromSymbol(host_out, lmgs::g_bw_count, sizeof(lmgs::g_bw_count));
}
namespace lmgs {
namespace {
#endif
// exp(x) to ~1 ulp (the reference's libm exp is within 0.5-1 ulp): Cody-Waite
// reduction by ln 2 and a degree-13 Taylor polynomial in explicit FMAs
// (exact rounding whatever the contraction mode), scaled by 2^k in two steps when the
// result is subnormal.  About half the instructions of libdevice's exp.
__device__ __forceinline__ double exp_bw(double x) {
  if (!(x > -745.2)) return 0.0;
  const double kf = rint(x * 1.4426950408889634);
  double r = __fma_rn(-kf, 6.93147180369123816490e-01, x);  // ln2 hi (exact product)
  r = __fma_rn(-kf, 1.90821492927058770002e-10, r);         // ln2 lo
  double p = 1.6059043836821613e-10;                         // 1/13!
  p = __fma_rn(p, r, 2.08767569878680990e-09);               // 1/12!
  p = __fma_rn(p, r, 2.50521083854417188e-08);
  p = __fma_rn(p, r, 2.75573192239858907e-07);
  p = __fma_rn(p, r, 2.75573192239858907e-06);
  p = __fma_rn(p, r, 2.48015873015873016e-05);
  p = __fma_rn(p, r, 1.98412698412698413e-04);
  p = __fma_rn(p, r, 1.38888888888888889e-03);
  p = __fma_rn(p, r, 8.33333333333333333e-03);
  p = __fma_rn(p, r, 4.16666666666666667e-02);
  p = __fma_rn(p, r, 1.66666666666666667e-01);
  p = __fma_rn(p, r, 0.5);
  p = __fma_rn(p, r, 1.0);
  p = __fma_rn(p, r, 1.0);
  int k = (int)kf;
  if (k < -1020) {  // 2^k subnormal: scale in two normal steps
    p = __dmul_rn(p, __longlong_as_double((long long)(k + 600 + 1023) << 52));
    return __dmul_rn(p, __longlong_as_double((long long)(-600 + 1023) << 52));
  }
  if (k > 1023) return __longlong_as_double(0x7ff0000000000000LL);
  return __dmul_rn(p, __longlong_as_double((long long)(k + 1023) << 52));
}

// Sum six per-lane values over the warp with 8 fp64 shuffles (a transpose
// reduction: each exchange halves what a lane carries).  Returns the full sum
// of value bw_owner(lane) in the owner lanes.
__device__ __forceinline__ double warp_sum6(const double v[6], int lane) {
  const bool h = lane & 16, b = lane & 8, c = lane & 4;
  double a0 = (h ? v[3] : v[0]) + __shfl_xor_sync(~0u, h ? v[0] : v[3], 16);
  double a1 = (h ? v[4] : v[1]) + __shfl_xor_sync(~0u, h ? v[1] : v[4], 16);
  double a2 = (h ? v[5] : v[2]) + __shfl_xor_sync(~0u, h ? v[2] : v[5], 16);
  a2 = a2 + __shfl_xor_sync(~0u, a2, 8);
  const double k = (b ? a1 : a0) + __shfl_xor_sync(~0u, b ? a0 : a1, 8);
  double m = (c ? a2 : k) + __shfl_xor_sync(~0u, c ? k : a2, 4);
  m = m + __shfl_xor_sync(~0u, m, 2);
  m = m + __shfl_xor_sync(~0u, m, 1);
  return m;
}
// lanes 0,8,4,16,24,20 hold values 0..5
__device__ __forceinline__ int bw_owner(int lane) {
  if (lane & 3) return -1;
  const int base = (lane & 16) ? 3 : 0;
  if (lane & 4) return (lane & 8) ? -1 : base + 2;
  return base + ((lane & 8) ? 1 : 0);
}

// One warp (= one CTA) per 8x4 pixel block of a tile, one pixel per lane,
// pixel state in registers; no block-level synchronisation, so a block that
// has terminated frees its SM slot at once.  The tile list is walked in
// batches of 32: each lane loads one splat's cull data (mean, radius^2),
// prefetched a batch ahead; splats whose circle misses the bounding box of
// the still-active pixel centres are skipped (exact: sigma is 0 outside the
// circle and fp64 rounding is monotone); hit splats' full records are staged
// in the warp's shared buffer.  Gradients of a splat are warp-reduced and
// added to global memory by the owner lanes.
#ifndef LMGS_BW_MINB
#define LMGS_BW_MINB 32  // 64 registers (small spill): 1.65 vs 1.77 ms at 16
#endif
__global__ void __launch_bounds__(32, LMGS_BW_MINB) k_backward(BackwardArgs a) {
  __shared__ BwRec s_rec[32];
  const int lane = threadIdx.x;
  const int ts = a.tile_size;
  const int tile = blockIdx.x / a.blocks, blk = blockIdx.x % a.blocks;
  const int tx0 = (tile % a.tiles_x) * ts, ty0 = (tile / a.tiles_x) * ts;
  const int tx1 = min(tx0 + ts, a.width), ty1 = min(ty0 + ts, a.height);
  const int px = tx0 + (blk % a.blocks_x) * 8 + (lane & 7);
  const int py = ty0 + (blk / a.blocks_x) * 4 + (lane >> 3);
  const bool in_img = px < tx1 && py < ty1;
  const int2 range = a.ranges[tile];
  if (range.y <= range.x || !__any_sync(~0u, in_img)) return;
  const double pxd = (double)px + 0.5, pyd = (double)py + 0.5;
  const uint32_t* __restrict__ list = static_cast<const uint32_t*>(*a.keys_slot);
  const double4* __restrict__ cull = reinterpret_cast<const double4*>(a.recs);
  const int own = bw_owner(lane);

  double g0 = 0.0, g1 = 0.0, g2 = 0.0, t0 = 0.0, t1 = 0.0, t2 = 0.0;
  if (in_img) {
    const int64_t o = (int64_t)py * a.width + px;
    g0 = (double)a.image_grad[3 * o + 0];
    g1 = (double)a.image_grad[3 * o + 1];
    g2 = (double)a.image_grad[3 * o + 2];
  }
  for (int pass = 0; pass < 2; ++pass) {
    double T = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
    bool live = in_img;
    // prefetch of the first batch
    uint32_t nid = 0;
    double4 ncd = make_double4(0.0, 0.0, -1.0, 0.0);
    if (range.x + lane < range.y) {
      nid = list[range.x + lane];
      ncd = cull[3 * (size_t)nid];  // BwRec is 3 x 32 B, cull data first
    }
    for (int b0 = range.x; b0 < range.y; b0 += 32) {
      const uint32_t id = nid;
      const double4 cd = ncd;
      const int nb = min(32, range.y - b0);
      if (b0 + 32 + lane < range.y) {
        nid = list[b0 + 32 + lane];
        ncd = cull[3 * (size_t)nid];
      }
      // bounding box of the active pixel centres
      const int bx0 = __reduce_min_sync(~0u, live ? px : INT_MAX);
      const int bx1 = __reduce_max_sync(~0u, live ? px : INT_MIN);
      const int by0 = __reduce_min_sync(~0u, live ? py : INT_MAX);
      const int by1 = __reduce_max_sync(~0u, live ? py : INT_MIN);
      bool hit = false;
      if (lane < nb) {
        const double ex = fmax(fmax((bx0 + 0.5) - cd.x, cd.x - (bx1 + 0.5)), 0.0);
        const double ey = fmax(fmax((by0 + 0.5) - cd.y, cd.y - (by1 + 0.5)), 0.0);
        hit = __dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)) <= cd.z;  // as the pixel test
      }
      unsigned m = __ballot_sync(~0u, hit);
      __syncwarp();
      if (hit) {
        const double4* src = cull + 3 * (size_t)id;
        double4* dst = reinterpret_cast<double4*>(&s_rec[lane]);
        dst[0] = cd;
        dst[1] = src[1];
        dst[2] = src[2];
      }
      __syncwarp();
      while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        const BwRec& r = s_rec[k];
        double v[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        bool app = false, touch = false;
#ifdef LMGS_BW_COUNT
        {
          const double ddx = pxd - r.mx, ddy = pyd - r.my;
          const bool ins = live && (ddx * ddx + ddy * ddy) <= r.r2;
          const unsigned lv = __ballot_sync(~0u, live), iv = __ballot_sync(~0u, ins);
          if (lane == 0) {
            atomicAdd(&g_bw_count[pass][0], 1ull);
            atomicAdd(&g_bw_count[pass][1], (unsigned long long)__popc(lv));
            atomicAdd(&g_bw_count[pass][2], (unsigned long long)__popc(iv));
          }
        }
#endif
        if (live) {
          const double dx = pxd - r.mx, dy = pyd - r.my;  // 311
          const double maha = (r.ca * (dx * dx) + ((2.0 * r.cb) * dx) * dy) + r.cc * (dy * dy);
          double sig = r.op * exp_bw(-0.5 * maha);         // 313
          const bool inside = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) <= r.r2;  // 314
          sig = inside ? (sig > kSigmaMax ? kSigmaMax : sig) : 0.0;
          const double w = T * sig;
          c0 = c0 + w * r.col[0];
          c1 = c1 + w * r.col[1];
          c2 = c2 + w * r.col[2];
          if (pass == 1 && sig > 0.0) {  // backward_render 461-484
            const double s0 = t0 - c0, s1 = t1 - c1, s2 = t2 - c2;  // suffix
            double denom = 1.0 - sig;
            denom = denom < 1e-6 ? 1e-6 : denom;
            // x / denom as x * (1 / denom) and / alpha as * (1 / alpha): one
            // division instead of four, within 1 ulp of the reference's
            const double rd = 1.0 / denom;
            const double dsig = (g0 * (r.col[0] * T - s0 * rd) +
                                 g1 * (r.col[1] * T - s1 * rd)) +
                                g2 * (r.col[2] * T - s2 * rd);
            v[0] = g0 * w;
            v[1] = g1 * w;
            v[2] = g2 * w;
            v[3] = dsig * sig * r.rop;
            v[4] = dsig * (sig * (r.ca * dx + r.cb * dy));
            v[5] = dsig * (sig * (r.cb * dx + r.cc * dy));
            app = true;
            touch = w > 0.0;
          }
          T = T * (1.0 - sig);
          live = T >= kTermEps;
        }
        if (pass == 1) {
          if (__any_sync(~0u, app)) {  // all six terms are 0 unless sigma > 0
            const unsigned tm = __ballot_sync(~0u, touch);
            const double sum = warp_sum6(v, lane);
            const uint32_t sid = __shfl_sync(~0u, id, k);
            if (own >= 0 && sum != 0.0) {
              double* dst = own < 3 ? a.d_colors + 3 * (size_t)sid + own
                          : own == 3 ? a.d_opacities + sid
                                     : a.d_mean2d + 2 * (size_t)sid + (own - 4);
              atomicAdd(dst, sum);
            }
            if (lane == 1 && tm) atomicAdd(a.touched + sid, __popc(tm));
          }
        }
      }
      if (!__any_sync(~0u, live)) break;
    }
    // C_tot = sum w c + T_final * background (326)
    t0 = c0 + T * a.bg[0];
    t1 = c1 + T * a.bg[1];
    t2 = c2 + T * a.bg[2];
  }
}

}  // namespace

int launch_backward_replay(const BackwardArgs& a, int tiles, cudaStream_t s) {
  if (tiles <= 0) return 0;
  k_backward<<<(unsigned)((int64_t)tiles * a.blocks), 32, 0, s>>>(a);
  return 1;
}

}  // namespace lmgs
