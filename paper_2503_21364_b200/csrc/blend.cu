// K7 blend_tiles: per-tile front-to-back alpha blending.
//
// Reference: _blend (gaussian_core.py:286-332), background term (326),
// scatter into the image (396-397).
//
// One CTA per tile.  Per batch of up to 256 splats (in list order):
//   1. each thread stages one splat record into shared memory (fp32 conic and
//      colour, tile-local fp32 mean, guard-banded r^2 bounds, fp64 mean and
//      r^2 for the exact fallback, a conservative bbox);
//   2. each warp culls the batch against the bbox of its own pixels (8x4
//      pixel blocks for 16x16 tiles) — 32 splats per ballot — and keeps an
//      ordered list of the splats that can touch it;
//   3. each warp walks its list: per pixel the exact circle test, exponent,
//      MUFU ex2, front-to-back update; touched is counted with one ballot
//      per (warp, splat);
//   4. the CTA stops at the first batch boundary after which no pixel is
//      active; n_processed is the exact break index of the reference loop.
//
// Exactness: inside = d.d <= r^2 (314) is
// decided in fp32 with a certified guard band and re-done in fp64 inside the
// band; active = T >= TERM_EPS before each splat (315); touched counts w > 0
// (323) judged from the exponent (an fp32 ex2 underflows where fp64 exp
// does not).  The continuous part runs in fp32.
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

// smallest float >= 1e-4: (double)T >= 1e-4  <=>  T >= kTermEpsF for fp32 T
constexpr float kTermEpsF = 1.00000005e-4f;
constexpr float kSigmaMaxF = 0.9999f;

// Exact `touched` (K7b): a pixel whose fp32 transmittance passed TERM_EPS
// within a relative band of kFixBand — where fp32 and the reference's fp64
// could disagree on which splats the pixel still takes — is queued for an
// fp64 replay that corrects the counts.  Tc = T before the last splat the
// pixel took while active (its T before the crossing, once it crossed).
// The band is BlendArgs.fix_band: 1e-4 by default (10x the measured fp32/fp64
// T gap, < 1e-5 at the crossing), 1e-2 with LMGS_FLAG_WIDE_FIX_BAND (the
// check that the default band misses no disagreement).
//
// The crossing splat's own fp32 error widens the band per pixel: sigma is
// within ~1.5e-7 of the fp64 value (fp32 rounding + ex2.approx), so 1 - sigma
// — the factor T took at that splat — is relatively off by up to 1.5e-7 /
// (1 - sigma) = 1.5e-7 * Tc / T: negligible for translucent splats (c3: alpha
// <= 0.88 -> < 2e-6), up to ~2e-3 for a near-opaque one (sigma -> 0.9999);
// taken at 3e-7 * Tc / T (tests/test_gpu_parity.py::test_opaque_splats_*).
// (sigma <= SIGMA_MAX bounds Tc / T by ~1e4, so the widening stays below
// 1e-2: pixels outside band + 1e-2 are rejected before the division)
__device__ __forceinline__ bool crossing_uncertain(float T, float Tc, float band) {
  {
    const float hi = kTermEpsF * (1.01f + band), lo = kTermEpsF * (0.99f - band);
    if (!(T < kTermEpsF ? (Tc < hi || T >= lo) : T < hi)) return false;
  }
  band += 3e-7f * __fdividef(Tc, fmaxf(T, 1e-30f));  // (2x margin covers the approximation)
  const float hi = kTermEpsF * (1.0f + band), lo = kTermEpsF * (1.0f - band);
  if (T < kTermEpsF) return Tc < hi || T >= lo;
  return T < hi;
}
// The queue holds W * H entries (each pixel is queued at most once), so it
// cannot overflow.  Entry = fix_entry(): tile << 8 | ly << 4 | lx for 16x16
// tiles (tile < 2^24, the cheap form inside k_blend16w), else the pixel index
// y * W + x.
__device__ __forceinline__ uint32_t fix_entry16(int tile, int lx, int ly) {
  return ((uint32_t)tile << 8) | ((uint32_t)ly << 4) | (uint32_t)lx;
}
__device__ __forceinline__ void queue_fix(const BlendArgs& a, uint32_t entry) {
  const uint32_t slot = atomicAdd(a.fix_count, 1u);
  a.fix_list[slot] = entry;
}
constexpr int kBatch = 256;
constexpr int kMaxWarps = 8;
constexpr int kMaxBlockW = 64;  // k_blend pixel block edge (256 threads x 16 pixels)

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// PPT pixels per thread; SWZ: 16x16 tile on 256 threads with each warp owning
// an 8x4 pixel block (tighter warp bboxes than 16x2 rows).
// NPFIX: recompute n_processed of one tile exactly (no image outputs): each
// pixel's break index from the fp32 recurrence, except the pixels K7b found
// to cross TERM_EPS at a different splat in fp64, whose fp64 index
// (a.np_override) is taken instead.
template <int PPT, bool SWZ, bool NPFIX>
__device__ __forceinline__ void blend_block(const BlendArgs& a, const int tile, const int sub) {
  __shared__ float4 s_geo[kBatch];   // mx_local, my_local, qa, qb
  __shared__ float4 s_geo2[kBatch];  // qc, log2_alpha, r2_lo, r2_hi
  __shared__ float4 s_col[kBatch];   // r, g, b, z
  __shared__ float4 s_box[kBatch];   // conservative bbox: xmin, xmax, ymin, ymax (tile-local)
  __shared__ double s_mx[kBatch], s_my[kBatch], s_r2[kBatch];
  __shared__ uint32_t s_id[kBatch];
  __shared__ uint8_t s_list[kMaxWarps][kBatch];
  __shared__ uint16_t s_cnt[kMaxWarps][kBatch];
  __shared__ int s_last[kMaxWarps];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthreads = blockDim.x;
  const int nwarps = (nthreads + 31) >> 5;
  // tiles above 64 px are split into 64x64 sub-blocks, one CTA each, that
  // walk the same list (the tile's break index is the max of theirs)
  const int subs = a.subs_x * a.subs_x;
  const int ts = a.tile_size;
  const int bw = ts < kMaxBlockW ? ts : kMaxBlockW;
  const int sx0 = (sub % a.subs_x) * bw, sy0 = (sub / a.subs_x) * bw;
  const int tile_x = tile % a.tiles_x, tile_y = tile / a.tiles_x;
  const int x0 = tile_x * ts, y0 = tile_y * ts;
  const int2 range = a.ranges[tile];
  const uint32_t* __restrict__ list = static_cast<const uint32_t*>(*a.keys_slot);

  float T[PPT], C0[PPT], C1[PPT], C2[PPT], D[PPT], px[PPT], py[PPT], Tc[PPT];
  int lxs[PPT], lys[PPT], last[PPT];
  bool valid[PPT];
  float bx0 = 3.0e38f, bx1 = -3.0e38f, by0 = 3.0e38f, by1 = -3.0e38f;
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    int lx, ly, pix;
    if (SWZ) {
      lx = (warp & 1) * 8 + (lane & 7);
      ly = (warp >> 1) * 4 + (lane >> 3);
      pix = ly * 16 + lx;
    } else {
      pix = tid + p * nthreads;
      lx = sx0 + pix % bw;
      ly = sy0 + pix / bw;
    }
    lxs[p] = lx;
    lys[p] = ly;
    valid[p] = pix < bw * bw && lx < ts && ly < ts && x0 + lx < a.width && y0 + ly < a.height;
    T[p] = valid[p] ? 1.0f : 0.0f;  // invalid pixels never go active
    Tc[p] = 1.0f;
    C0[p] = C1[p] = C2[p] = D[p] = 0.0f;
    px[p] = (float)lx + 0.5f;  // _pixel_centers (335-337), tile-local
    py[p] = (float)ly + 0.5f;
    last[p] = -1;
    if (valid[p]) {
      bx0 = fminf(bx0, px[p]);
      bx1 = fmaxf(bx1, px[p]);
      by0 = fminf(by0, py[p]);
      by1 = fmaxf(by1, py[p]);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    bx0 = fminf(bx0, __shfl_xor_sync(0xffffffffu, bx0, o));
    bx1 = fmaxf(bx1, __shfl_xor_sync(0xffffffffu, bx1, o));
    by0 = fminf(by0, __shfl_xor_sync(0xffffffffu, by0, o));
    by1 = fmaxf(by1, __shfl_xor_sync(0xffffffffu, by1, o));
  }
  const uint32_t lt = lanemask_lt();

  for (int b0 = range.x; b0 < range.y; b0 += kBatch) {
    bool mine_active = false;
#pragma unroll
    for (int p = 0; p < PPT; ++p) mine_active |= T[p] >= kTermEpsF;
    if (__syncthreads_count(mine_active) == 0) break;
    const int nb = min(kBatch, range.y - b0);
    for (int j = tid; j < nb; j += nthreads) {
      const uint32_t id = list[b0 + j];
      const BlendRec rec = a.recs[id];
      const double mxl = rec.mx - (double)x0, myl = rec.my - (double)y0;
      const double ax = fabs(mxl) + ts, ay = fabs(myl) + ts;
      const double band =  // explicit rounding: touched_fix.cu recomputes it bit for bit
          __dmul_rn(__dadd_rn(__dadd_rn(rec.r2, __dmul_rn(ax, ax)), __dmul_rn(ay, ay)), 0x1p-18);
      const float fx = (float)mxl, fy = (float)myl;
      const float r = sqrtf((float)rec.r2) * 1.0001f + 1e-3f;
      s_geo[j] = make_float4(fx, fy, rec.qa, rec.qb);
      s_geo2[j] = make_float4(rec.qc, rec.log2_alpha, __double2float_rd(rec.r2 - band),
                              __double2float_ru(rec.r2 + band));
      s_col[j] = make_float4(rec.cr, rec.cg, rec.cb, rec.z);
      s_box[j] = make_float4(fx - r, fx + r, fy - r, fy + r);
      s_mx[j] = rec.mx;
      s_my[j] = rec.my;
      s_r2[j] = rec.r2;
      s_id[j] = id;
#pragma unroll
      for (int w = 0; w < kMaxWarps; ++w) s_cnt[w][j] = 0;
    }
    __syncthreads();
    // per-warp cull: ordered list of the batch's splats whose bbox meets ours
    int cnt = 0;
    if (__any_sync(0xffffffffu, mine_active)) {
      for (int j0 = 0; j0 < nb; j0 += 32) {
        const int j = j0 + lane;
        bool hit = false;
        if (j < nb) {
          const float4 bb = s_box[j];
          hit = bb.y >= bx0 && bb.x <= bx1 && bb.w >= by0 && bb.z <= by1;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, hit);
        if (hit) s_list[warp][cnt + __popc(m & lt)] = (uint8_t)j;
        cnt += __popc(m);
      }
    }
    __syncwarp();
    for (int q = 0; q < cnt; ++q) {
      const int k = s_list[warp][q];
      const float4 g = s_geo[k];
      const float4 h = s_geo2[k];
      const float4 c = s_col[k];
      int contrib_n = 0;
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        if (T[p] >= kTermEpsF) {
          const float dx = px[p] - g.x, dy = py[p] - g.y;
          const float d2 = fmaf(dx, dx, dy * dy);
          bool inside = d2 <= h.z;
          if (!inside && d2 <= h.w) {
            // guard band: the reference's fp64 test, bit for bit
            const double ddx = ((double)(x0 + lxs[p]) + 0.5) - s_mx[k];
            const double ddy = ((double)(y0 + lys[p]) + 0.5) - s_my[k];
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
            Tc[p] = T[p];
            T[p] = T[p] * (1.0f - sig);
            contrib_n += contrib;
            if (T[p] < kTermEpsF) last[p] = b0 - range.x + k;
          }
        }
      }
      int wsum;
      if (PPT == 1) wsum = __popc(__ballot_sync(0xffffffffu, contrib_n));
      else wsum = __reduce_add_sync(0xffffffffu, contrib_n);
      if (lane == 0) s_cnt[warp][k] = (uint16_t)wsum;
    }
    __syncthreads();
    if (!NPFIX && a.touched) {
      for (int j = tid; j < nb; j += nthreads) {
        int s = 0;
#pragma unroll
        for (int w = 0; w < kMaxWarps; ++w) s += w < nwarps ? s_cnt[w][j] : 0;
        if (s) atomicAdd(a.touched + s_id[j], s);
      }
    }
  }

  if (NPFIX) {
    // per pixel: its break index (list length while still active)
    const int len = range.y - range.x;
    int v = 0;
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
      if (!valid[p]) continue;
      const int o = a.np_override[(int64_t)(y0 + lys[p]) * a.width + x0 + lxs[p]];
      v = max(v, o >= 0 ? o : (T[p] >= kTermEpsF ? len : last[p] + 1));
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) s_last[warp] = v;
    __syncthreads();
    if (tid == 0) {
      int m = 0;
      for (int w = 0; w < nwarps; ++w) m = max(m, s_last[w]);
      // blocks of one tile run in sequence in this CTA (see k_nproc_fix)
      a.n_processed[tile] = sub == 0 ? m : max(a.n_processed[tile], m);
    }
    __syncthreads();
    return;
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
      for (int w = 0; w < nwarps; ++w) m = max(m, s_last[w]);
      const int v = any_live ? (range.y - range.x) : (m + 1);
      if (subs == 1) a.n_processed[tile] = v;
      else atomicMax(a.n_processed + tile, v);  // zeroed by launch_blend
    }
  }
  // outputs: C + T * bg (326), alpha = 1 - T_final, depth, T_final
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    if (NPFIX || !valid[p]) continue;
    put_pixel(a, x0 + lxs[p], y0 + lys[p], T[p], C0[p], C1[p], C2[p], D[p]);
    if (a.fix_count && crossing_uncertain(T[p], Tc[p], a.fix_band))
      queue_fix(a, ts == 16 ? fix_entry16(tile, lxs[p], lys[p])
                            : (uint32_t)(y0 + lys[p]) * (uint32_t)a.width + (uint32_t)(x0 + lxs[p]));
  }
}

template <int PPT, bool SWZ>
__global__ void __launch_bounds__(256) k_blend(BlendArgs a) {
  const int subs = a.subs_x * a.subs_x;
  blend_block<PPT, SWZ, false>(a, blockIdx.x / subs, blockIdx.x % subs);
}

// Exact n_processed for the tiles K7b flagged (np_need: a corrected pixel set
// the tile's fp32 break index; a tile listed twice is recomputed twice, to
// the same value).
template <int PPT, bool SWZ>
__global__ void __launch_bounds__(256) k_nproc_fix(BlendArgs a) {
  const uint32_t n = *a.np_count;
  for (uint32_t e = blockIdx.x; e < n; e += gridDim.x) {
    if (!a.np_need[e]) continue;
    const uint32_t pix = a.np_list[e];
    const int tile = (int)(pix / (uint32_t)a.width) / a.tile_size * a.tiles_x +
                     (int)(pix % (uint32_t)a.width) / a.tile_size;
    for (int sub = 0; sub < a.subs_x * a.subs_x; ++sub)
      blend_block<PPT, SWZ, true>(a, tile, sub);
  }
}

// the overrides are reset for the next view once k_nproc_fix has read them
__global__ void k_nproc_reset(BlendArgs a) {
  const uint32_t n = *a.np_count;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
    a.np_override[a.np_list[e]] = -1;
}

// ---------------------------------------------------------------------------
// 16x16 tiles: persistent warps over warp-granular work items.
//
// Item = (tile, 8x4 pixel block); 8 items per tile.  A warp takes items from
// a global counter, walks its tile's list 32 splats at a time (each lane
// loads one record's geometry sector, culls it against the warp's pixel box,
// and loads the colour sector only on a hit), blends the hits in list order,
// and stops as soon as its own 32 pixels are done — no CTA barriers, and a
// finished warp immediately starts the next item.  n_processed is the max of
// the warps' break indices (atomicMax); touched is one red.add per
// (warp, splat) with contributions.

constexpr int kWarpsPerBlock16 = 8;

// NP pixels per lane: the warp owns an 8 x (4*NP) block of its 16x16 tile
// (16 / (4*NP) * 2 items per tile); lane l holds pixels (l & 7, (l >> 3) + 4p).
// With NP = 2 the per-splat work (shared loads, ballots, the touched atomic,
// loop control) is shared by two pixels and the two pixels' dependency chains
// interleave.
// the first work item of a warp = its warp index (no counter round trip):
// blend 0.413 -> 0.43 ms/view (a static first item unbalances the persistent
// warps), off
#ifndef LMGS_BLEND_STATIC_FIRST
#define LMGS_BLEND_STATIC_FIRST 0
#endif
// list ids one batch further ahead than the records: blend 0.413 -> 0.398
// ms/view (profiles/r10/blend_prefetch_variants.txt)
#ifndef LMGS_BLEND_ID_AHEAD
#define LMGS_BLEND_ID_AHEAD 1
#endif
#ifndef LMGS_BLEND_SMEM_FP64
#define LMGS_BLEND_SMEM_FP64 0  // 1: hits' fp64 mean / r^2 staged in shared memory (6 KB per CTA)
#endif
#ifndef LMGS_BLEND_COMPACT
#define LMGS_BLEND_COMPACT 0  // 1: 264 -> 295 M warp instructions, 807 -> 799 frames/s (profiles/r10/blend_compact_variants.txt)
#endif
#ifndef LMGS_BLEND_PAIRS
#define LMGS_BLEND_PAIRS 0  // 1: two hits per trip, one break vote per pair (777.6 vs 777.3 frames/s: neutral, profiles/r10)
#endif
#ifndef LMGS_BLEND_CONCURRENT_CTAS
#define LMGS_BLEND_CONCURRENT_CTAS 2  // blend CTAs per SM under LMGS_FLAG_CONCURRENT (0: all)
#endif
#ifndef LMGS_BLEND_MINB
#define LMGS_BLEND_MINB 4  // 4 x 256 threads per SM (64 registers): measured best
#endif
#ifdef LMGS_BLEND_MAXREG  // experiment: a register cap between the MINB steps
#define LMGS_BLEND_BOUNDS __maxnreg__(LMGS_BLEND_MAXREG)
#else
#define LMGS_BLEND_BOUNDS __launch_bounds__(256, LMGS_BLEND_MINB)
#endif
template <int NP>
__global__ void LMGS_BLEND_BOUNDS k_blend16w(BlendArgs a, int n_items) {
  // per hit splat: {mx_local, my_local, qa, qb}, {qc, log2_alpha, r2_lo, r2_hi},
  // {r, g, b, z} side by side (one address per splat)
  __shared__ float4 s_rec[kWarpsPerBlock16][32][3];
#if LMGS_BLEND_SMEM_FP64
  __shared__ double s_mx[kWarpsPerBlock16][32], s_my[kWarpsPerBlock16][32],
      s_r2[kWarpsPerBlock16][32];
#endif
  __shared__ uint8_t s_lane[kWarpsPerBlock16][32];  // LMGS_BLEND_COMPACT: slot -> list lane
  constexpr int kItemsPerTile = 8 / NP;
  constexpr int kRows = 4 * NP;  // block height

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t* __restrict__ list = static_cast<const uint32_t*>(*a.keys_slot);
  const float4* __restrict__ rec4 = reinterpret_cast<const float4*>(a.recs);

#if LMGS_BLEND_STATIC_FIRST
  // the first item of every warp is its global warp index; the counter hands
  // out the rest (no round trip before the first list load)
  const int first_items = gridDim.x * kWarpsPerBlock16;
  bool first = true;
#endif
  while (true) {
    int item = 0;
#if LMGS_BLEND_STATIC_FIRST
    if (first) {
      item = blockIdx.x * kWarpsPerBlock16 + warp;
      first = false;
    } else {
      if (lane == 0) item = atomicAdd(a.work_counter, 1) + first_items;
      item = __shfl_sync(0xffffffffu, item, 0);
    }
#else
    if (lane == 0) item = atomicAdd(a.work_counter, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
#endif
    if (item >= n_items) break;
    const int tile = item / kItemsPerTile, sub = item % kItemsPerTile;
    const int tile_x = tile % a.tiles_x, tile_y = tile / a.tiles_x;
    const int x0 = tile_x * 16, y0 = tile_y * 16;
    const int lx = (sub & 1) * 8 + (lane & 7);
    int ly[NP];
    bool valid[NP];
    float T[NP], C0[NP], C1[NP], C2[NP], D[NP], Tc[NP];
    bool any_valid = false;
    float bx0 = 3.0e38f, bx1 = -3.0e38f, by0 = 3.0e38f, by1 = -3.0e38f;
    const float px = (float)lx + 0.5f;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      ly[q] = (sub >> 1) * kRows + (lane >> 3) + 4 * q;
      valid[q] = x0 + lx < a.width && y0 + ly[q] < a.height;
      T[q] = valid[q] ? 1.0f : 0.0f;  // invalid pixels never go active
      Tc[q] = 1.0f;
      C0[q] = C1[q] = C2[q] = D[q] = 0.0f;
      any_valid |= valid[q];
      if (valid[q]) {  // warp pixel box (pixel centres, tile-local)
        const float py = (float)ly[q] + 0.5f;
        bx0 = fminf(bx0, px);
        bx1 = fmaxf(bx1, px);
        by0 = fminf(by0, py);
        by1 = fmaxf(by1, py);
      }
    }
    if (!__any_sync(0xffffffffu, any_valid)) continue;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      bx0 = fminf(bx0, __shfl_xor_sync(0xffffffffu, bx0, o));
      bx1 = fmaxf(bx1, __shfl_xor_sync(0xffffffffu, bx1, o));
      by0 = fminf(by0, __shfl_xor_sync(0xffffffffu, by0, o));
      by1 = fmaxf(by1, __shfl_xor_sync(0xffffffffu, by1, o));
    }
    const int2 range = a.ranges[tile];
    int last = -1;     // list index after which no pixel of this warp is active
    bool live = true;  // some valid pixel still has T >= TERM_EPS
    // software pipeline: batch b's id and geometry sectors were loaded while
    // batch b - 32 was being blended
    uint32_t id = 0;
    float4 g0 = make_float4(0.f, 0.f, 0.f, 0.f), g1 = g0;
    if (range.x + lane < range.y) {
      id = list[range.x + lane];
      g0 = __ldg(rec4 + 4 * (size_t)id);
      g1 = __ldg(rec4 + 4 * (size_t)id + 1);
    }
#if LMGS_BLEND_ID_AHEAD
    // the ids run one batch further ahead than the records, so a batch's
    // record loads never wait on its id load
    uint32_t id_next = range.x + 32 + lane < range.y ? list[range.x + 32 + lane] : 0u;
#endif
    uint32_t box_mask = __ballot_sync(0xffffffffu, any_valid);  // lanes the box covers
    for (int b = range.x; b < range.y && live; b += 32) {
      const int j = b + lane;
      const bool have = j < range.y;
      const uint32_t cid = id;
      // shrink the cull box to the pixels still active (finished pixels need
      // no more splats); recomputed only when some lane has finished
      bool act_any = false;
#pragma unroll
      for (int q = 0; q < NP; ++q) act_any |= T[q] >= kTermEpsF;
      const uint32_t act_mask = __ballot_sync(0xffffffffu, act_any);
      if (act_mask != box_mask) {
        box_mask = act_mask;
        bx0 = 3.0e38f, bx1 = -3.0e38f, by0 = 3.0e38f, by1 = -3.0e38f;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          if (T[q] >= kTermEpsF) {
            const float py = (float)ly[q] + 0.5f;
            bx0 = fminf(bx0, px);
            bx1 = fmaxf(bx1, px);
            by0 = fminf(by0, py);
            by1 = fmaxf(by1, py);
          }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          bx0 = fminf(bx0, __shfl_xor_sync(0xffffffffu, bx0, o));
          bx1 = fmaxf(bx1, __shfl_xor_sync(0xffffffffu, bx1, o));
          by0 = fminf(by0, __shfl_xor_sync(0xffffffffu, by0, o));
          by1 = fmaxf(by1, __shfl_xor_sync(0xffffffffu, by1, o));
        }
      }
      const float4 c0 = g0, c1 = g1;
      if (j + 32 < range.y) {  // prefetch the next batch
#if LMGS_BLEND_ID_AHEAD
        id = id_next;
        if (j + 64 < range.y) id_next = list[j + 64];
#else
        id = list[j + 32];
#endif
        g0 = __ldg(rec4 + 4 * (size_t)id);
        g1 = __ldg(rec4 + 4 * (size_t)id + 1);
      }
      // (computed on every lane; a lane past the list end has no hit)
      const double mx = __hiloint2double(__float_as_int(c0.y), __float_as_int(c0.x));
      const double my = __hiloint2double(__float_as_int(c0.w), __float_as_int(c0.z));
      const double r2 = __hiloint2double(__float_as_int(c1.y), __float_as_int(c1.x));
      const double mxl = mx - (double)x0, myl = my - (double)y0;
      const float fx = (float)mxl, fy = (float)myl;
      // exact circle-vs-box cull (the reference's support is the circle
      // d.d <= r^2 around the mean) with a conservative radius margin
      const float r = sqrtf((float)r2) * 1.0001f + 1e-3f;
      const float ex = fx - fminf(fmaxf(fx, bx0), bx1);
      const float ey = fy - fminf(fmaxf(fy, by0), by1);
      const bool hit = have && fmaf(ex, ex, ey * ey) <= r * r;
#if LMGS_BLEND_COMPACT
      // hits staged in list order at consecutive slots: the hit loop walks
      // slots 0.. with a counter (no find-first-set per hit)
      const uint32_t hm = __ballot_sync(0xffffffffu, hit);
      const int slot = __popc(hm & lanemask_lt());
      if (hit) s_lane[warp][slot] = (uint8_t)lane;
#else
      const int slot = lane;
#endif
      if (hit) {
        const float4 g2 = __ldg(rec4 + 4 * (size_t)cid + 2);  // qc, log2a, r, g
        const float4 g3 = __ldg(rec4 + 4 * (size_t)cid + 3);  // b, z
        const double ax = fabs(mxl) + 16.0, ay = fabs(myl) + 16.0;
        const double band =  // explicit rounding (touched_fix.cu)
            __dmul_rn(__dadd_rn(__dadd_rn(r2, __dmul_rn(ax, ax)), __dmul_rn(ay, ay)), 0x1p-18);
        s_rec[warp][slot][0] = make_float4(fx, fy, c1.z, c1.w);
        s_rec[warp][slot][1] = make_float4(g2.x, g2.y, __double2float_rd(r2 - band),
                                           __double2float_ru(r2 + band));
        s_rec[warp][slot][2] = make_float4(g2.z, g2.w, g3.x, g3.y);
#if LMGS_BLEND_SMEM_FP64
        s_mx[warp][slot] = mx;
        s_my[warp][slot] = my;
        s_r2[warp][slot] = r2;
#endif
      }
      uint32_t m = __ballot_sync(0xffffffffu, hit);
      __syncwarp();
      uint32_t my_touch = 0;  // pixels with w > 0 for this lane's splat (cid)
      uint32_t my_ballot = 0;  // NP == 1: the pixels themselves
      // one hit splat k of the batch: the front-to-back update of this lane's
      // pixels; returns whether one of them is still active
      auto blend_one = [&](const int k) -> bool {
        const float4 g = s_rec[warp][k][0];
        const float4 h = s_rec[warp][k][1];
        const float4 c = s_rec[warp][k][2];
        const float dx = px - g.x;
        uint32_t contrib_bits = 0;  // NP > 1: pixels with w > 0
        bool contrib1 = false;      // NP == 1: the pixel has w > 0
        bool active = false;
        // Common path, branch-free: a pixel takes the splat when it is active
        // and certainly inside the circle (fp32 below the guard band); sigma
        // is 0 otherwise, which leaves C and T bit-identical (fmaf(0, c, C) =
        // C, T * (1 - 0) = T).  The rare fp64 decisions — d.d within the
        // guard band of r^2, or w > 0 where fp32 ex2 underflows — are flagged
        // and settled after the vote below, so this path carries no branch.
        bool any_rare = false;  // some pixel needs the exact path
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          const bool on = T[q] >= kTermEpsF;
          const float dy = ((float)ly[q] + 0.5f) - g.y;
          const float d2 = fmaf(dx, dx, dy * dy);
          const bool inside = d2 <= h.z;
          const float power = fmaf(fmaf(g.z, dx, g.w * dy), dx, fmaf(h.x * dy, dy, h.y));
          const bool take = on && inside;
          // fp64 circle test (guard band) or fp64 w > 0 test (fp32 ex2 underflow)
          // (inside implies d2 <= h.w: r2_lo <= r2_hi); bitwise, so no branch
          const bool tiny = power <= -1060.0f;
          any_rare |= on & (d2 <= h.w) & (!inside | tiny);
          const bool contrib = take && !tiny;
          const float sig = take ? fminf(ex2_approx(power), kSigmaMaxF) : 0.0f;
          const float w = T[q] * sig;
          C0[q] = fmaf(w, c.x, C0[q]);
          C1[q] = fmaf(w, c.y, C1[q]);
          C2[q] = fmaf(w, c.z, C2[q]);
          D[q] = fmaf(w, c.w, D[q]);
          Tc[q] = take ? T[q] : Tc[q];
          T[q] = T[q] * (1.0f - sig);
          if (NP == 1) contrib1 |= contrib;
          else contrib_bits += contrib;
        }
        if (__any_sync(0xffffffffu, any_rare)) {
#if !LMGS_BLEND_SMEM_FP64
          const uint32_t rare_id = __shfl_sync(0xffffffffu, cid, LMGS_BLEND_COMPACT ? s_lane[warp][k] : k);
#endif
#pragma unroll
          for (int q = 0; q < NP; ++q) {
            const float dy = ((float)ly[q] + 0.5f) - g.y;
            const float d2 = fmaf(dx, dx, dy * dy);
            const float power = fmaf(fmaf(g.z, dx, g.w * dy), dx, fmaf(h.x * dy, dy, h.y));
            // redone on the current state: a rare pixel's T was left unchanged
            // (not taken, or taken with sigma = 0); a pixel taken with sigma > 0
            // has power > -1060 and is inside, so the test is false for it
            const bool on = T[q] >= kTermEpsF;
            if (!(on && (d2 <= h.z ? power <= -1060.0f : d2 <= h.w))) continue;
            if (d2 <= h.z) {
              // taken above with sigma = 0 (ex2 underflow): only w > 0 is open,
              // judged in fp64 on T before the splat (unchanged)
              const bool cw = exp2((double)power) * (double)T[q] > 0.0;
              if (NP == 1) contrib1 |= cw;
              else contrib_bits += cw;
              continue;
            }
            // guard band: the reference's fp64 circle test
#if LMGS_BLEND_SMEM_FP64
            const double gmx = s_mx[warp][k], gmy = s_my[warp][k], gr2 = s_r2[warp][k];
#else
            // (rare path: the splat's fp64 mean and r^2 come back from its
            // record instead of 6 KB of shared staging per CTA)
            const double2 gm = __ldg(reinterpret_cast<const double2*>(a.recs + rare_id));
            const double gmx = gm.x, gmy = gm.y;
            const double gr2 = __ldg(&a.recs[rare_id].r2);
#endif
            const double ddx = ((double)(x0 + lx) + 0.5) - gmx;
            const double ddy = ((double)(y0 + ly[q]) + 0.5) - gmy;
            if (!(__dadd_rn(__dmul_rn(ddx, ddx), __dmul_rn(ddy, ddy)) <= gr2)) continue;
            bool contrib = power > -1060.0f;
            if (!contrib && power >= -1080.0f)  // fp32 ex2 underflows first
              contrib = exp2((double)power) * (double)T[q] > 0.0;
            const float sig = fminf(ex2_approx(power), kSigmaMaxF);
            const float w = T[q] * sig;
            C0[q] = fmaf(w, c.x, C0[q]);
            C1[q] = fmaf(w, c.y, C1[q]);
            C2[q] = fmaf(w, c.z, C2[q]);
            D[q] = fmaf(w, c.w, D[q]);
            Tc[q] = T[q];
            T[q] = T[q] * (1.0f - sig);
            if (NP == 1) contrib1 |= contrib;
            else contrib_bits += contrib;
          }
        }
#pragma unroll
        for (int q = 0; q < NP; ++q) active |= T[q] >= kTermEpsF;
        if (NP == 1) {  // the owner keeps its splat's ballot; counted after the batch
          const uint32_t bl = __ballot_sync(0xffffffffu, contrib1);
          my_ballot = hit && slot == k ? bl : my_ballot;
        } else {
          const int wsum = __reduce_add_sync(0xffffffffu, contrib_bits);
          if (hit && slot == k) my_touch += wsum;
        }
        return active;
      };
#if LMGS_BLEND_COMPACT
      const int nh = __popc(m);
      for (int h = 0; h < nh; ++h) {
        // pixels only go inactive on a splat they are inside: the warp's break
        // index is the first splat after which none of its pixels is active
        if (!__any_sync(0xffffffffu, blend_one(h))) {
          last = b - range.x + s_lane[warp][h];
          live = false;
          break;
        }
      }
#elif LMGS_BLEND_PAIRS
      // two hits per trip and one break vote per pair: a pixel that went
      // inactive takes nothing more (sigma 0, no w > 0), so blending the
      // second splat of a pair after the break changes nothing; when the pair
      // ends with no pixel active, the vote on the first splat's state tells
      // which of the two was the break
      while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        const bool act1 = blend_one(k);
        if (m) {
          const int k2 = __ffs(m) - 1;
          m &= m - 1;
          const bool act2 = blend_one(k2);
          if (!__any_sync(0xffffffffu, act2)) {
            last = b - range.x + (__any_sync(0xffffffffu, act1) ? k2 : k);
            live = false;
            break;
          }
        } else if (!__any_sync(0xffffffffu, act1)) {
          last = b - range.x + k;
          live = false;
          break;
        }
      }
#else
      while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        // pixels only go inactive on a splat they are inside: the warp's break
        // index is the first splat after which none of its pixels is active
        if (!__any_sync(0xffffffffu, blend_one(k))) {
          last = b - range.x + k;
          live = false;
          break;
        }
      }
#endif
      if (NP == 1) my_touch = __popc(my_ballot);
      if (my_touch && a.touched) atomicAdd(a.touched + cid, (int)my_touch);
      __syncwarp();
    }
    if (a.n_processed && lane == 0)
      atomicMax(a.n_processed + tile, live ? (range.y - range.x) : last + 1);
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      if (!valid[q]) continue;
      put_pixel(a, x0 + lx, y0 + ly[q], T[q], C0[q], C1[q], C2[q], D[q]);
      if (a.fix_count && crossing_uncertain(T[q], Tc[q], a.fix_band))
        queue_fix(a, fix_entry16(tile, lx, ly[q]));
    }
  }
}

#ifndef LMGS_BLEND_NP
#define LMGS_BLEND_NP 1
#endif
constexpr int kBlendNP = LMGS_BLEND_NP;

}  // namespace

int launch_nproc_fix(const BlendArgs& args, cudaStream_t s) {
  BlendArgs a = args;
  const int ts = a.tile_size;
  const int ext = ts < max(a.width, a.height) ? ts : max(a.width, a.height);
  a.subs_x = (ext + kMaxBlockW - 1) / kMaxBlockW;
  const int grid = 16;  // tiles to recompute are rare
  if (ts == 16) {
    k_nproc_fix<1, true><<<grid, 256, 0, s>>>(a);
  } else if (ts < 16) {
    k_nproc_fix<1, false><<<grid, ((ts * ts + 31) / 32) * 32, 0, s>>>(a);
  } else if (ts <= 32) {
    k_nproc_fix<4, false><<<grid, 256, 0, s>>>(a);
  } else {
    k_nproc_fix<16, false><<<grid, 256, 0, s>>>(a);
  }
  k_nproc_reset<<<16, 256, 0, s>>>(a);
  return 2;
}

int launch_blend(const BlendArgs& args, cudaStream_t s) {
  BlendArgs a = args;
  const int ts = a.tile_size;
  const int tiles = a.tiles_x * a.tiles_y;
  if (tiles <= 0) return 0;
  // the blocks of a tile larger than the image only need to cover the image
  const int ext = ts < max(a.width, a.height) ? ts : max(a.width, a.height);
  a.subs_x = (ext + kMaxBlockW - 1) / kMaxBlockW;
  if (ts == 16 && a.work_counter) {
    cudaMemsetAsync(a.work_counter, 0, sizeof(int), s);
    if (a.n_processed) cudaMemsetAsync(a.n_processed, 0, sizeof(int) * tiles, s);
    const int items = tiles * (8 / kBlendNP);
    static int bps_cache[kMaxDevices] = {}, sms_cache[kMaxDevices] = {};
    const int dev = current_device();
    if (!bps_cache[dev]) {
      int bps = 0, sms = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      set_carveout(k_blend16w<kBlendNP>);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_blend16w<kBlendNP>, 256, 0);
      sms_cache[dev] = sms > 0 ? sms : 148;
      bps_cache[dev] = bps > 0 ? bps : 1;
    }
#ifdef LMGS_BLEND_CTAS_PER_SM  // experiment: leave room for other streams' kernels
    int grid = sms_cache[dev] * min(bps_cache[dev], LMGS_BLEND_CTAS_PER_SM);
#else
    // concurrent renders: fewer resident blend CTAs (each holds a quarter of
    // the register file) so the other streams' kernels share the SMs
    int grid = sms_cache[dev] *
               (a.concurrent && LMGS_BLEND_CONCURRENT_CTAS > 0
                    ? min(bps_cache[dev], LMGS_BLEND_CONCURRENT_CTAS) : bps_cache[dev]);
#endif
    const int need = (items + kWarpsPerBlock16 - 1) / kWarpsPerBlock16;
    if (grid > need) grid = need;
    k_blend16w<kBlendNP><<<grid, 256, 0, s>>>(a, items);
  } else if (ts == 16) {
    k_blend<1, true><<<tiles, 256, 0, s>>>(a);
  } else if (ts < 16) {
    const int threads = ((ts * ts + 31) / 32) * 32;
    k_blend<1, false><<<tiles, threads, 0, s>>>(a);
  } else if (ts <= 32) {
    k_blend<4, false><<<tiles, 256, 0, s>>>(a);
  } else if (ts <= 64) {
    k_blend<16, false><<<tiles, 256, 0, s>>>(a);
  } else {
    const int64_t ctas = (int64_t)tiles * a.subs_x * a.subs_x;
    if (ctas >= ((int64_t)1 << 31)) return LMGS_ERR_UNSUPPORTED;
    if (a.n_processed) cudaMemsetAsync(a.n_processed, 0, sizeof(int) * tiles, s);
    k_blend<16, false><<<(unsigned)ctas, 256, 0, s>>>(a);
  }
  return 0;
}

}  // namespace lmgs
