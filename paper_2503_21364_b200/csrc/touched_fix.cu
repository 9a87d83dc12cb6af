// K7b: exact `touched` (rasterize's per-splat count of w > 0, gaussian_core.py
// 323) for the pixels whose fp32 transmittance crossed TERM_EPS within the
// blend's uncertainty band (blend.cu: crossing_uncertain).  Everywhere else
// the fp32 blend's decisions are the reference's: circle tests are exact
// (guard band + fp64), w > 0 is exact (exponent check + fp64), and a pixel
// far from TERM_EPS is active in both.  For a queued pixel one warp walks the
// tile list again: threads evaluate 256 splats at a time — the blend's fp32
// quantities with the blend's exact expressions, and for the splats the
// pixel is inside, sigma in fp64 from K1's geometry (geometry.cuh, this file
// is built with -fmad=false) as _blend (306-322) computes it — then thread 0
// runs both recurrences in list order over the inside splats and adds (fp64
// decision - fp32 decision) to each splat's count, until both transmittances
// are below TERM_EPS.
#include "device_util.cuh"
#include "geometry.cuh"
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

constexpr float kTermEpsF = 1.00000005e-4f;  // as blend.cu
constexpr float kSigmaMaxF = 0.9999f;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

#ifndef LMGS_FIX_THREADS
#define LMGS_FIX_THREADS 128  // 64: 663, 128: 671, 256: 667, 512: 637 frames/s (c3 bench)
#endif
constexpr int kFixThreads = LMGS_FIX_THREADS;
constexpr int kProdWarps = kFixThreads / 32 - 1;  // warps 1..7 produce, warp 0 scans
constexpr int kRound = 32 * kProdWarps;           // splats per round

#ifdef LMGS_FIX_STATS
// debug: histogram of |T32 / T64 - 1| at the end of each replayed pixel
__device__ unsigned int g_fix_hist[8];
#endif

// a list entry's id and first record sector (mx, my, r^2, qa, qb)
struct FixRec {
  uint32_t id;
  bool valid;
  double2 s0, s1;
};
// the circle test of one splat at the pixel and, when inside, what fp64 sigma
// needs: the blend's fp32 exponent terms and K1's inputs
struct FixIn {
  uint32_t id;
  bool inside;
  float dx, dy, qa, qb;
  float2 cl;  // qc, log2 alpha
  float4 q;
  float m0, m1, m2, sc0, sc1, sc2, logit;
};

__device__ __forceinline__ void load_rec(const TouchedFixArgs& a, const uint32_t* list,
                                         int2 range, int j, FixRec& r) {
  r.valid = j < range.y;
  if (r.valid) {
    r.id = list[j];
    const double2* r16 = reinterpret_cast<const double2*>(a.recs + r.id);
    r.s0 = r16[0];
    r.s1 = r16[1];
  }
}

__device__ __forceinline__ void test_and_load(const TouchedFixArgs& a, const FixRec& r, int x0,
                                              int y0, int ts, float px, float py, double pxd,
                                              double pyd, FixIn& f) {
  f.inside = false;
  f.id = r.id;
  if (!r.valid) return;
  const double rmx = r.s0.x, rmy = r.s0.y, rr2 = r.s1.x;
  const float2 qab = *reinterpret_cast<const float2*>(&r.s1.y);
  // the blend's fp32 view of the splat (blend.cu, same expressions)
  const double mxl = rmx - (double)x0, myl = rmy - (double)y0;
  const double ax = fabs(mxl) + (double)ts, ay = fabs(myl) + (double)ts;
  const double band =
      __dmul_rn(__dadd_rn(__dadd_rn(rr2, __dmul_rn(ax, ax)), __dmul_rn(ay, ay)), 0x1p-18);
  const float fx = (float)mxl, fy = (float)myl;
  const float dx = px - fx, dy = py - fy;
  const float d2 = fmaf(dx, dx, dy * dy);
  bool inside = d2 <= __double2float_rd(rr2 - band);
  if (!inside && d2 <= __double2float_ru(rr2 + band)) {
    const double ddx = pxd - rmx, ddy = pyd - rmy;
    inside = __dadd_rn(__dmul_rn(ddx, ddx), __dmul_rn(ddy, ddy)) <= rr2;
  }
  f.inside = inside;
  if (!inside) return;
  const uint32_t id = r.id;
  f.dx = dx;
  f.dy = dy;
  f.qa = qab.x;
  f.qb = qab.y;
  f.cl = reinterpret_cast<const float2*>(a.recs + id)[4];
  f.q = reinterpret_cast<const float4*>(a.quats)[id];
  f.m0 = a.means[3 * (size_t)id];
  f.m1 = a.means[3 * (size_t)id + 1];
  f.m2 = a.means[3 * (size_t)id + 2];
  f.sc0 = a.scales[3 * (size_t)id];
  f.sc1 = a.scales[3 * (size_t)id + 1];
  f.sc2 = a.scales[3 * (size_t)id + 2];
  f.logit = a.logits[id];
}

// One CTA per queued pixel, as a two-stage pipeline over rounds of 224
// consecutive splats of the tile list.  Producer warps (1..7) take 32 splats
// each: the blend's fp32 circle test and exponent, and for the splats the
// pixel is inside (a few percent) sigma in fp64 from K1's geometry, compacted
// in list order into the warp's slots of the round's buffer.  Meanwhile
// thread 0 runs the fp32 and fp64 recurrences over the previous round's
// buffer (double-buffered, one barrier per round).
__global__ void __launch_bounds__(kFixThreads) k_touched_fix(TouchedFixArgs a) {
  __shared__ float s_pow[2][kProdWarps][32];
  __shared__ double s_sig[2][kProdWarps][32];
  __shared__ uint32_t s_id[2][kProdWarps][32];
  __shared__ int s_pos[2][kProdWarps][32];  // list position (from the tile's start)
  __shared__ int s_cnt[2][kProdWarps];
  __shared__ int s_done;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t n = *a.fix_count;  // <= W * H = the queue's capacity
  const uint32_t* __restrict__ list = static_cast<const uint32_t*>(*a.keys_slot);
  const CamArgs& cam = a.cam;
  const int ts = a.tile_size;
  for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
    // blend.cu fix_entry: tile << 8 | ly << 4 | lx for 16x16 tiles, else y * W + x
    const uint32_t e = a.fix_list[i];
    int tile, lx, ly;
    if (ts == 16) {
      tile = (int)(e >> 8);
      ly = (int)((e >> 4) & 15);
      lx = (int)(e & 15);
    } else {
      const int gx = (int)(e % (uint32_t)a.width), gy = (int)(e / (uint32_t)a.width);
      tile = (gy / ts) * a.tiles_x + gx / ts;
      lx = gx % ts;
      ly = gy % ts;
    }
    const int x0 = (tile % a.tiles_x) * ts, y0 = (tile / a.tiles_x) * ts;
    const uint32_t v = (uint32_t)(y0 + ly) * (uint32_t)a.width + (uint32_t)(x0 + lx);  // pixel
    const float px = (float)lx + 0.5f, py = (float)ly + 0.5f;  // tile-local (blend)
    const double pxd = (double)(x0 + lx) + 0.5, pyd = (double)(y0 + ly) + 0.5;  // 335-337
    const int2 range = a.ranges[tile];
    const int nr = (range.y - range.x + kRound - 1) / kRound;
    float T32 = 1.0f;  // thread 0's recurrences
    double T64 = 1.0;
    int brk32 = -1, brk64 = -1;  // break indices: 1 + position of the crossing splat
    if (tid == 0) s_done = 0;
    // producer pipeline, three rounds deep: round r + 2's ids and first
    // record sectors load, round r + 1 takes the circle test and (inside
    // lanes) issues the loads of its geometry inputs, round r computes fp64
    // sigma from inputs that arrived during the previous round
    const int pt = 32 * (warp - 1) + lane;  // producer slot within a round
    FixRec ra{}, rb{};  // rounds r + 1 and r + 2: id + first record sector
    FixIn ia{};         // round r: circle test result and geometry inputs
    if (warp > 0) {
      load_rec(a, list, range, range.x + pt, ra);
      load_rec(a, list, range, range.x + kRound + pt, rb);
      test_and_load(a, ra, x0, y0, ts, px, py, pxd, pyd, ia);
      ra = rb;
    }
    __syncthreads();
#ifdef LMGS_FIX_STATS
    int rounds = 0;
#endif
    for (int r = 0; r <= nr; ++r) {
      const int buf = r & 1;
      if (warp > 0 && r < nr) {  // produce round r
        const FixIn cur = ia;
        FixRec nx{};
        load_rec(a, list, range, range.x + (r + 2) * kRound + pt, nx);
        test_and_load(a, ra, x0, y0, ts, px, py, pxd, pyd, ia);  // round r + 1
        ra = nx;
        const bool inside = cur.inside;
        const uint32_t m = __ballot_sync(0xffffffffu, inside);
        if (lane == 0) s_cnt[buf][warp - 1] = __popc(m);
        if (inside) {
          const int pos = __popc(m & lanemask_lt());
          const uint32_t id = cur.id;
          const float power = fmaf(fmaf(cur.qa, cur.dx, cur.qb * cur.dy), cur.dx,
                                   fmaf(cur.cl.x * cur.dy, cur.dy, cur.cl.y));
          // _blend 308-313 in fp64 from K1's geometry
          const double m0 = cur.m0, m1 = cur.m1, m2 = cur.m2;
          const double x = mkl_dot3(m0, cam.r[0], m1, cam.r[1], m2, cam.r[2]) + cam.t[0];
          const double y = mkl_dot3(m0, cam.r[3], m1, cam.r[4], m2, cam.r[5]) + cam.t[1];
          const double z = mkl_dot3(m0, cam.r[6], m1, cam.r[7], m2, cam.r[8]) + cam.t[2];
          double mx, my, c00, c01, c11, radius;
          splat_geometry(cam, x, y, z, cur.q, cur.sc0, cur.sc1, cur.sc2, &mx, &my, &c00, &c01,
                         &c11, &radius);
          const double det = c00 * c11 - c01 * c01;
          const double ca = c11 / det, cb = -c01 / det, cc = c00 / det;
          const double ddx = pxd - mx, ddy = pyd - my;
          const double maha = (ca * (ddx * ddx) + ((2.0 * cb) * ddx) * ddy) + cc * (ddy * ddy);
          const double op = 1.0 / (1.0 + exp(-(double)cur.logit));
          s_sig[buf][warp - 1][pos] = op * exp(-0.5 * maha);
          s_pow[buf][warp - 1][pos] = power;
          s_id[buf][warp - 1][pos] = id;
          s_pos[buf][warp - 1][pos] = r * kRound + pt;
        }
      }
      if (tid == 0 && r > 0 && !s_done) {  // scan round r - 1
        const int pb = buf ^ 1;
#ifdef LMGS_FIX_STATS
        ++rounds;
#endif
        for (int w = 0; w < kProdWarps && !s_done; ++w) {
          const int cnt = s_cnt[pb][w];
          for (int k = 0; k < cnt; ++k) {
            const float pw = s_pow[pb][w][k];
            // the blend's step (blend.cu k_blend16w / k_blend), inside = true
            const bool take32 = T32 >= kTermEpsF;
            bool c32 = take32 && pw > -1060.0f;
            if (take32 && !c32 && pw >= -1080.0f) c32 = exp2((double)pw) * (double)T32 > 0.0;
            const float sig32 = take32 ? fminf(ex2_approx(pw), kSigmaMaxF) : 0.0f;
            T32 = T32 * (1.0f - sig32);
            // the reference's step (_blend 314-323)
            const bool take64 = T64 >= kTermEps;
            const double sig64 = take64 ? fmin(s_sig[pb][w][k], kSigmaMax) : 0.0;
            const bool c64 = T64 * sig64 > 0.0;
            T64 = T64 * (1.0 - sig64);
            if (c64 != c32) atomicAdd(a.touched + s_id[pb][w][k], c64 ? 1 : -1);
            if (brk32 < 0 && T32 < kTermEpsF) brk32 = s_pos[pb][w][k] + 1;
            if (brk64 < 0 && T64 < kTermEps) brk64 = s_pos[pb][w][k] + 1;
            if (T32 < kTermEpsF && T64 < kTermEps) {
              s_done = 1;
              break;
            }
          }
        }
      }
      __syncthreads();
      if (s_done) break;
    }
#ifdef LMGS_FIX_STATS
    if (tid == 0) {
      const double rel = T64 > 0 ? fabs((double)T32 / T64 - 1.0) : 0.0;
      int bin = rel < 1e-7 ? 0 : rel < 1e-6 ? 1 : rel < 1e-5 ? 2 : rel < 1e-4 ? 3 : rel < 1e-3 ? 4 : 5;
      atomicAdd(&g_fix_hist[bin], 1u);
      atomicAdd(&g_fix_hist[6], (unsigned)rounds);
      atomicMax(&g_fix_hist[7], (unsigned)rounds);
    }
#endif
    if (tid == 0 && a.np_count) {
      const int len = range.y - range.x;
      if (brk32 < 0) brk32 = len;
      if (brk64 < 0) brk64 = len;
      if (brk32 != brk64) {
        // The blend's n_processed[tile] = max(others, brk32) with every other
        // pixel exact.  A later fp64 break only raises the max; an earlier one
        // changes it only if this pixel set it, and then the tile is
        // recomputed (launch_nproc_fix) with the fp64 index of every corrected
        // pixel (np_override).
        a.np_override[v] = brk64;
        uint8_t need = 0;
        if (brk64 > brk32) atomicMax(a.n_processed + tile, brk64);
        else need = atomicAdd(a.n_processed + tile, 0) == brk32;
        const uint32_t slot = atomicAdd(a.np_count, 1u);
        a.np_list[slot] = v;
        a.np_need[slot] = need;
      }
    }
    __syncthreads();
  }
}

}  // namespace

#ifdef LMGS_FIX_STATS
}  // namespace lmgs
extern "C" int lmgs_debug_fix_hist(unsigned int* out) {
  return (int)cudaMemcpyFromSymbol(out, lmgs::g_fix_hist, sizeof(lmgs::g_fix_hist));
}
namespace lmgs {
#endif

int launch_touched_fix(const TouchedFixArgs& a, cudaStream_t s) {
#ifndef LMGS_FIX_CTAS_PER_SM
#define LMGS_FIX_CTAS_PER_SM (2048 / kFixThreads)
#endif
  static bool once = false;
  if (!once) set_carveout(k_touched_fix), once = true;
  k_touched_fix<<<148 * LMGS_FIX_CTAS_PER_SM, kFixThreads, 0, s>>>(a);
  return 1;
}

}  // namespace lmgs
