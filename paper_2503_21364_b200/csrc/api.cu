// C-ABI entry points (include/lmgs.h): context, device arena, stage pipeline.
//
// One view (stream-ordered, one 24-byte D2H read of the counters):
//   K1 preprocess  fp64 geometry, tile rect + count, blend record, fp32 depth
//                  key; counts M (near-kept), visible splats and K
//   K2 depth sort  onesweep LSD radix of the fp32 depth keys (implicit id
//                  payload), then the exact fp64 fix-up of equal-key runs
//   K4 emit        splats in depth-rank order -> keys tile << 32 | id (scan by
//                  decoupled look-back) + tile-digit histograms
//   K5 tile sort   stable onesweep LSD radix on the tile bits (2 passes at 1080p)
//   K6 ranges      per-tile [start, end) from the sorted keys
//   K7 blend       persistent warps over (tile, 8x4 block) items
#include <cstdio>
#include <cstddef>
#include <cstring>
#include <string>
#include <vector>

#include "lmgs_internal.cuh"

using namespace lmgs;
static_assert(LMGS_MAX_GROUP == kMaxPreViews, "one K1 launch per group");

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

// Experiments only (bench_tools/stage_skip_probe.py): bit i of
// LMGS_SKIP_STAGES drops stage i's kernels (1 depth sort, 2 emit, 3 tile sort,
// 4 blend) so the batch's frame time without them can be measured; outputs
// are then garbage (stale but memory-safe arenas).
#ifndef LMGS_SKIP_STAGES
#define LMGS_SKIP_STAGES 0
#endif
constexpr unsigned kSkip = LMGS_SKIP_STAGES;
// concurrent renders: K1 as a persistent grid of this many CTAs per SM (0:
// one CTA per 128-row block)
#ifndef LMGS_PRE_PERSIST_CTAS
#define LMGS_PRE_PERSIST_CTAS 0  // 2-5: 749-780 vs 794 frames/s (profiles/r10/k1_persist_variants.txt)
#endif

const char* kStageNames[] = {"preprocess", "depth_sort", "emit", "tile_sort", "blend",
                             "touched_fix"};
constexpr int kNumStages = 6;

// grow-only device buffer
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaError_t reserve(size_t need) {
    if (need <= bytes) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    size_t want = need + need / 4;  // headroom against per-view jitter
    cudaError_t e = cudaMalloc(&ptr, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      e = cudaMalloc(&ptr, need);
      if (e != cudaSuccess) return e;
      want = need;
    }
    bytes = want;
    return cudaSuccess;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

struct Carver {
  char* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    T* p = reinterpret_cast<T*>(base + off);
    off += align_up(sizeof(T) * (count ? count : 1));
    return p;
  }
};

size_t gaussian_bytes(int64_t n) {
  size_t b = 0;
  b += 2 * align_up(sizeof(uint32_t) * n);  // fp32 depth keys (ping-pong)
  b += 2 * align_up(sizeof(uint32_t) * n);  // ids (ping-pong)
  b += align_up(sizeof(uint64_t) * n);      // fp64 depth keys
  b += align_up(sizeof(uint64_t) * n);      // rects
  b += align_up(sizeof(BlendRec) * n);      // records
  b += align_up(sizeof(uint4) * n);         // rank records (fused tile sort)
  b += align_up(sizeof(uint32_t) * radix_lookback_words(n));  // K2 look-back
  b += align_up(sizeof(uint64_t) * emit_chunks(n));            // K4 look-back
  return b + 10 * kAlign;
}
size_t tile_bytes(int64_t t) {
  return align_up(sizeof(int2) * t) + align_up(sizeof(uint32_t) * t) + 2 * kAlign;
}
size_t instance_bytes(int64_t k) {
  return 2 * align_up(sizeof(uint64_t) * k) + align_up(sizeof(uint32_t) * radix_lookback_words(k)) +
         align_up(sizeof(uint32_t) * (k / kSortTile + 2)) + 5 * kAlign;
}

struct Scalars {  // device-side small state
  RadixPlan depth_plan, tile_plan;
  uint32_t depth_hist[kMaxPasses * kRadix];
  uint32_t tile_hist[kMaxPasses * kRadix];
  uint32_t depth_counters[kMaxPasses];
  uint32_t tile_counters[kMaxPasses];
  unsigned long long counts[3];  // n_kept, n_vis, n_inst (one D2H copy)
  unsigned long long max_k;      // largest K of no-sync renders since lmgs_get_stats
  unsigned long long k_eff;      // fused tile sort: K, or 0 after a no-sync overflow
  unsigned long long zrange[2];  // min / max visible fp64 depth bits
  uint32_t emit_ticket[1];  // K4 chunk ticket
  int blend_counter;
  uint32_t fix_count;  // pixels queued for the exact-touched replay (K7b)
  uint32_t np_count;   // pixels whose fp64 break index differs (exact n_processed)
  DevSlots slots;
};

}  // namespace

struct lmgs_context {
  int device = 0;
  int sms = 148;
  std::string err;
  DevBuf gbuf, tbuf, ibuf, bwbuf, fixbuf, npbuf;  // npbuf: override (-1) + list, W*H each
  Scalars* d_scal = nullptr;
  uint64_t* h_pinned = nullptr;  // [0..2] = n_kept, n_vis, K
  cudaEvent_t ev[2 * kNumStages] = {};
  cudaEvent_t counts_ready = nullptr;
  cudaEvent_t ev_in = nullptr, ev_pre = nullptr;  // lmgs_render_group cross-stream order
  int pre_share = 1;  // views sharing the last K1 launch (its stage time is split)
  bool events_ok = false;
  int64_t cap_n = -1, cap_t = -1, cap_k = -1;
  // per-Gaussian arena
  uint32_t* key32[2] = {nullptr, nullptr};
  uint32_t* ids[2] = {nullptr, nullptr};
  uint64_t* key64 = nullptr;
  uint64_t* rects = nullptr;
  BlendRec* recs = nullptr;
  uint32_t* depth_lookback = nullptr;
  uint64_t* emit_lookback = nullptr;
  uint4* rrec = nullptr;
  // per-tile arena
  int2* ranges = nullptr;
  uint32_t* tile_count = nullptr;
  // per-instance arena
  uint64_t* inst_keys[2] = {nullptr, nullptr};
  uint32_t* tile_lookback = nullptr;
  uint32_t* chunk_first = nullptr;
  const int64_t* last_prim_ids = nullptr;
  const int2* last_ranges = nullptr;
  lmgs_stats stats{};
  bool last_timed = false;
  bool counts_pending = false;  // a no-sync render's counts are still on the device
  bool max_k_pending = false;   // no-sync renders ran since the last lmgs_get_stats
  int64_t host_max_k = 0;       // largest K of the host-synchronised renders since then
};

namespace {

int fail(lmgs_context* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define LMGS_CUDA(ctx, call)                                                          \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? LMGS_ERR_OOM : LMGS_ERR_CUDA, \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                \
    }                                                                                 \
  } while (0)

#ifndef LMGS_SERIAL_K1
#define LMGS_SERIAL_K1 0  // 1: 805.4 vs 807.4 frames/s (neutral, profiles/r10/k1_serial_variants.txt)
#endif
// one event per device ordering the K1 launches of concurrent renders
cudaEvent_t k1_serial_event(int dev) {
  static cudaEvent_t ev[kMaxDevices] = {};
  if (dev < 0 || dev >= kMaxDevices) return nullptr;
  if (!ev[dev] && cudaEventCreateWithFlags(&ev[dev], cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    ev[dev] = nullptr;
  }
  return ev[dev];
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int ensure_gaussians(lmgs_context* c, int64_t n, cudaStream_t s) {
  if (n <= c->cap_n && c->recs) return LMGS_OK;
  LMGS_CUDA(c, cudaStreamSynchronize(s));  // previous renders may still read the arena
  LMGS_CUDA(c, c->gbuf.reserve(gaussian_bytes(n)));
  const int64_t cap = (int64_t)(c->gbuf.bytes >= gaussian_bytes(n + n / 4) ? n + n / 4 : n);
  Carver cv{static_cast<char*>(c->gbuf.ptr)};
  for (int i = 0; i < 2; ++i) c->key32[i] = cv.take<uint32_t>(cap);
  for (int i = 0; i < 2; ++i) c->ids[i] = cv.take<uint32_t>(cap);
  c->key64 = cv.take<uint64_t>(cap);
  c->rects = cv.take<uint64_t>(cap);
  c->recs = cv.take<BlendRec>(cap);
  c->rrec = cv.take<uint4>(cap);
  c->depth_lookback = cv.take<uint32_t>(radix_lookback_words(cap));
  c->emit_lookback = cv.take<uint64_t>(emit_chunks(cap));
  c->cap_n = cap;
  return LMGS_OK;
}

int ensure_tiles(lmgs_context* c, int64_t t, cudaStream_t s) {
  if (t <= c->cap_t && c->ranges) return LMGS_OK;
  LMGS_CUDA(c, cudaStreamSynchronize(s));
  LMGS_CUDA(c, c->tbuf.reserve(tile_bytes(t)));
  Carver cv{static_cast<char*>(c->tbuf.ptr)};
  c->ranges = cv.take<int2>(t);
  c->tile_count = cv.take<uint32_t>(t);
  c->cap_t = t;
  return LMGS_OK;
}

int ensure_instances(lmgs_context* c, int64_t k, cudaStream_t s) {
  if (k <= c->cap_k && c->inst_keys[0]) return LMGS_OK;
  LMGS_CUDA(c, cudaStreamSynchronize(s));
  LMGS_CUDA(c, c->ibuf.reserve(instance_bytes(k)));
  const int64_t cap = (int64_t)(c->ibuf.bytes >= instance_bytes(k + k / 4) ? k + k / 4 : k);
  Carver cv{static_cast<char*>(c->ibuf.ptr)};
  c->inst_keys[0] = cv.take<uint64_t>(cap);
  c->inst_keys[1] = cv.take<uint64_t>(cap);
  c->tile_lookback = cv.take<uint32_t>(radix_lookback_words(cap));
  c->chunk_first = cv.take<uint32_t>(cap / kSortTile + 2);
  c->cap_k = cap;
  return LMGS_OK;
}

int validate(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cam,
             const lmgs_settings* s) {
  if (!c) return LMGS_ERR_INVALID;
  if (!g || !cam || !s) return fail(c, LMGS_ERR_INVALID, "null argument");
  if (g->count < 0) return fail(c, LMGS_ERR_INVALID, "count must be >= 0");
  if (g->count >= (int64_t)1 << 31) return fail(c, LMGS_ERR_INVALID, "count must be < 2^31");
  if (g->sh_degree < 0 || g->sh_degree > 3)
    return fail(c, LMGS_ERR_INVALID, "sh_degree must be in [0, 3]");
  if (g->sh_coeffs != (g->sh_degree + 1) * (g->sh_degree + 1))
    return fail(c, LMGS_ERR_INVALID, "SH coefficient count does not match degree");
  if (g->count > 0 && (!g->means || !g->quats || !g->scales || !g->opacity_logits || !g->sh))
    return fail(c, LMGS_ERR_INVALID, "null Gaussian array");
  if (g->count > 0 && (reinterpret_cast<uintptr_t>(g->quats) & 15))
    return fail(c, LMGS_ERR_INVALID, "quats must be 16-byte aligned");
  if (g->page_mask && g->page_shift != 7)
    return fail(c, LMGS_ERR_INVALID, "page_shift must be 7 (128-row pages)");
  if (s->tile_size < 1) return fail(c, LMGS_ERR_INVALID, "tile_size must be >= 1");
  if (cam->width < 1 || cam->height < 1) return fail(c, LMGS_ERR_INVALID, "bad image size");
  if ((int64_t)cam->width * cam->height >= ((int64_t)1 << 32))
    return fail(c, LMGS_ERR_UNSUPPORTED, "more than 2^32 pixels in one view");
  if (cam->width > 65535ll * s->tile_size || cam->height > 65535ll * s->tile_size)
    return fail(c, LMGS_ERR_UNSUPPORTED, "image too large for 16-bit tile coordinates");
  if (!(cam->fx > 0) || !(cam->fy > 0))
    return fail(c, LMGS_ERR_INVALID, "focal lengths must be positive");
  return LMGS_OK;
}

CamArgs make_cam(const lmgs_camera* cam, int ts) {
  CamArgs a;
  memcpy(a.r, cam->r_wc, sizeof(a.r));
  memcpy(a.t, cam->t_wc, sizeof(a.t));
  memcpy(a.center, cam->center, sizeof(a.center));
  a.fx = cam->fx;
  a.fy = cam->fy;
  a.cx = cam->cx;
  a.cy = cam->cy;
  a.lim_x = cam->lim_x;
  a.lim_y = cam->lim_y;
  a.width = cam->width;
  a.height = cam->height;
  a.tile_size = ts;
  a.inv_tile = 1.0 / ts;
  a.tiles_x = (cam->width + ts - 1) / ts;
  a.tiles_y = (cam->height + ts - 1) / ts;
  return a;
}

int bits_for(int64_t v) {  // bits needed to represent values in [0, v)
  int b = 0;
  while (((int64_t)1 << b) < v) ++b;
  return b;
}

PreprocessArgs make_pre(lmgs_context* c, const lmgs_gaussians* g, const CamArgs& ca,
                        const lmgs_settings* st, uint8_t* kept, int32_t* touched = nullptr) {
  PreprocessArgs pa{};
  pa.means = g->means;
  pa.quats = g->quats;
  pa.scales = g->scales;
  pa.logits = g->opacity_logits;
  pa.sh = g->sh;
  pa.n = g->count;
  pa.page_mask = g->page_mask;
  pa.page_shift = g->page_shift;
  pa.sh_coeffs = g->sh_coeffs;
  pa.eval_degree = st->sh_eval_degree < g->sh_degree ? st->sh_eval_degree : g->sh_degree;
  pa.cam = ca;
  pa.depth_keys = c->key64;
  pa.rects = c->rects;
  pa.recs = c->recs;
  pa.kept = kept;
  pa.touched_zero = touched;
  pa.n_kept = &c->d_scal->counts[0];
  pa.n_vis = &c->d_scal->counts[1];
  pa.n_inst = &c->d_scal->counts[2];
  pa.zrange = c->d_scal->zrange;
  return pa;
}

struct StageTimer {
  lmgs_context* c;
  cudaStream_t s;
  bool on;
  void begin(int i) {
    if (on) cudaEventRecord(c->ev[2 * i], s);
  }
  void end(int i) {
    if (on) cudaEventRecord(c->ev[2 * i + 1], s);
  }
};

// one view's launch state between its K1 and the rest of its pipeline
struct ViewPlan {
  CamArgs ca;
  int64_t n = 0, tiles = 0;
  int tile_passes = 1;
  int2* ranges = nullptr;
  bool timed = false;
  int launched = 0;
};

// stats, arenas and counter resets of one view (stream-ordered on s)
int view_prepare(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cam,
                 const lmgs_settings* st, const lmgs_frame* out, cudaStream_t s, ViewPlan* vp) {
  vp->timed = (st->flags & LMGS_FLAG_STAGE_TIMES) && c->events_ok;
  vp->ca = make_cam(cam, st->tile_size);
  const CamArgs& ca = vp->ca;
  const int64_t n = vp->n = g->count;
  const int64_t tiles = vp->tiles = (int64_t)ca.tiles_x * ca.tiles_y;
  c->stats = lmgs_stats{};
  c->stats.n_gaussians = n;
  c->stats.n_tiles = (int32_t)tiles;
  c->stats.tiles_x = ca.tiles_x;
  c->stats.tiles_y = ca.tiles_y;
  c->stats.n_stages = kNumStages;
  for (int i = 0; i < kNumStages; ++i) c->stats.stage_names[i] = kStageNames[i];
  c->last_timed = false;
  c->pre_share = 1;
  c->last_prim_ids = g->prim_ids;
  const int tile_bits = bits_for(tiles);
  if (tile_bits > 8 * kMaxTilePasses)
    return fail(c, LMGS_ERR_UNSUPPORTED, "more than 2^24 tiles in one view");
  vp->tile_passes = tile_bits ? (tile_bits + 7) / 8 : 1;

  if (int r = ensure_gaussians(c, n > 0 ? n : 1, s)) return r;
  if (int r = ensure_tiles(c, tiles, s)) return r;
  // ranges live in the context arena (lmgs_backward and lmgs_copy_instances
  // read them after the call, whatever the caller did with its buffers);
  // the caller's tile_ranges gets a copy
  vp->ranges = c->ranges;
  c->last_ranges = vp->ranges;
  Scalars* sc = c->d_scal;
  LMGS_CUDA(c, cudaMemsetAsync(sc->counts, 0, sizeof(sc->counts), s));
  LMGS_CUDA(c, cudaMemsetAsync(&sc->zrange[0], 0xff, sizeof(sc->zrange[0]), s));
  LMGS_CUDA(c, cudaMemsetAsync(&sc->zrange[1], 0, sizeof(sc->zrange[1]), s));
  // out->touched is zeroed by K1 (make_pre: touched_zero), one pass fewer
  return LMGS_OK;
}

int view_finish(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cam,
                const lmgs_settings* st, const lmgs_frame* out, cudaStream_t s, ViewPlan* vp,
                const lmgs_strip_targets* strips);

int render_one(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cam,
               const lmgs_settings* st, const lmgs_frame* out, cudaStream_t s,
               const lmgs_strip_targets* strips = nullptr) {
  ViewPlan vp;
  if (int r = view_prepare(c, g, cam, st, out, s, &vp)) return r;
  StageTimer tm{c, s, vp.timed};
  // K1
  tm.begin(0);
  vp.launched += launch_preprocess(make_pre(c, g, vp.ca, st, out->kept, out->touched), s);
  tm.end(0);
  return view_finish(c, g, cam, st, out, s, &vp, strips);
}

// K2..K7 of one view whose K1 has been enqueued before `s`'s current tail
int view_finish(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cam,
                const lmgs_settings* st, const lmgs_frame* out, cudaStream_t s, ViewPlan* vp,
                const lmgs_strip_targets* strips) {
  StageTimer tm{c, s, vp->timed};
  const CamArgs& ca = vp->ca;
  const int64_t n = vp->n, tiles = vp->tiles;
  const int tile_passes = vp->tile_passes;
  int2* ranges = vp->ranges;
  Scalars* sc = c->d_scal;
  int launched = vp->launched;
  const bool nosync = (st->flags & LMGS_FLAG_NO_HOST_SYNC) != 0;
  LMGS_CUDA(c, cudaMemcpyAsync(c->h_pinned, sc->counts, sizeof(sc->counts),
                               cudaMemcpyDeviceToHost, s));
  if (!nosync) LMGS_CUDA(c, cudaEventRecord(c->counts_ready, s));

  // K2: 32-bit depth keys + histograms, (key, id) radix sort of all splats,
  // then the fp64 fix-up of equal-key runs
  tm.begin(1);
  {
    LMGS_CUDA(c, cudaMemsetAsync(sc->depth_hist, 0, sizeof(sc->depth_hist), s));
    if (!(kSkip & 2)) launched += launch_depth_keys(c->key64, sc->zrange, n, c->key32[0], sc->depth_hist, s);
    RadixSortBuffers rb{};
    rb.keys[0] = c->key32[0];
    rb.keys[1] = c->key32[1];
    rb.key_bytes = 4;
    rb.vals[0] = c->ids[0];
    rb.vals[1] = c->ids[1];
    rb.plan = &sc->depth_plan;
    rb.hist = sc->depth_hist;
    rb.lookback = c->depth_lookback;
    rb.counters = sc->depth_counters;
    rb.keys_result = &sc->slots.depth_keys;
    rb.vals_result = &sc->slots.depth_ids;
    rb.iota_vals = true;
    rb.hist_ready = true;
    rb.concurrent = (st->flags & LMGS_FLAG_CONCURRENT) != 0;
    if (!(kSkip & 2)) {
      launched += radix_sort(rb, n, 0, kDepthPasses, s);
      launched += launch_depth_fixup(&sc->slots.depth_keys, &sc->slots.depth_ids, n, c->key64,
                                     g->prim_ids, s);
    }
  }
  tm.end(1);

  int64_t n_vis, k;  // exact (host wait) or upper bounds (no-sync)
  if (nosync) {
    // no host wait: grids are sized for the capacity, kernels read the counts
    k = st->max_instances > 0 ? st->max_instances : c->cap_k;
    if (k <= 0)
      return fail(c, LMGS_ERR_INVALID,
                  "LMGS_FLAG_NO_HOST_SYNC needs settings.max_instances or an earlier render");
    if (k >= ((int64_t)1 << 30)) return fail(c, LMGS_ERR_INVALID, "max_instances must be < 2^30");
    n_vis = n;
    c->counts_pending = true;
    c->max_k_pending = true;
    c->stats.n_kept = c->stats.n_visible = c->stats.n_instances = -1;
  } else {
    // the only host wait of the view: M, visible splats, K (the depth sort keeps
    // the device busy meanwhile)
    LMGS_CUDA(c, cudaGetLastError());
    LMGS_CUDA(c, cudaEventSynchronize(c->counts_ready));
    c->counts_pending = false;
    c->stats.n_kept = (int64_t)c->h_pinned[0];
    n_vis = (int64_t)c->h_pinned[1];
    c->stats.n_visible = n_vis;
    k = (int64_t)c->h_pinned[2];
    c->stats.n_instances = k;
    if (k > c->host_max_k) c->host_max_k = k;
    if (k >= ((int64_t)1 << 30))
      return fail(c, LMGS_ERR_UNSUPPORTED, "more than 2^30 tile instances in one view");
  }
  if (int r = ensure_instances(c, k > 0 ? k : 1, s)) return r;
  // the capacity this view renders with: K itself after a host wait
  const int64_t cap_view = nosync ? k : c->cap_k;
  c->stats.capacity = cap_view;

  // fused K4 + K5 on request (two tile passes whose packed second-pass key
  // fits 32 bits): rank records instead of instance keys
  const int tile_bits = bits_for(tiles);
  const int id_bits = n > 1 ? bits_for(n) : 1;
  const bool fused = (st->flags & LMGS_FLAG_FUSED_TILE_SORT) && tile_bits > 8 &&
                     tile_bits <= 16 && (tile_bits - 8) + id_bits <= 32;
  if (fused) {
    tm.begin(2);
    LMGS_CUDA(c, cudaMemsetAsync(sc->tile_hist, 0, sizeof(sc->tile_hist), s));
    LMGS_CUDA(c, cudaMemsetAsync(sc->emit_ticket, 0, sizeof(uint32_t), s));
    if (n_vis > 0) {
      LMGS_CUDA(c, cudaMemsetAsync(c->emit_lookback, 0, sizeof(uint64_t) * emit_chunks(n_vis), s));
      EmitArgs ea{};
      ea.order_slot = &sc->slots.depth_ids;
      ea.rects = c->rects;
      ea.n_vis = n_vis;
      ea.n_vis_dev = &sc->counts[1];
      ea.cap = (uint64_t)cap_view;
      ea.tiles_x = ca.tiles_x;
      ea.n_tile_passes = 2;
      ea.lookback = c->emit_lookback;
      ea.ticket = sc->emit_ticket;
      ea.hist = sc->tile_hist;
      ea.rrec = c->rrec;
      ea.chunk_first = c->chunk_first;
      ea.n_sort_tiles = (cap_view + kSortTile - 1) / kSortTile;
      ea.k_dev = &sc->counts[2];
      if (!(kSkip & 4)) launched += launch_emit_ranks(ea, s);
    }
    tm.end(2);
    tm.begin(3);
    RadixSortBuffers rb{};
    rb.keys[0] = c->inst_keys[0];
    rb.keys[1] = c->inst_keys[1];
    rb.key_bytes = 8;
    rb.plan = &sc->tile_plan;
    rb.hist = sc->tile_hist;
    rb.lookback = c->tile_lookback;
    rb.counters = sc->tile_counters;
    rb.keys_result = &sc->slots.inst_ids;
    rb.hist_ready = true;
    rb.seg_counts = c->tile_count;
    rb.seg_shift = 32;
    rb.concurrent = (st->flags & LMGS_FLAG_CONCURRENT) != 0;
    if (nosync) {
      rb.n_dev = &sc->counts[2];
      rb.max_n = &sc->max_k;
    }
    LMGS_CUDA(c, cudaMemsetAsync(c->tile_count, 0, sizeof(uint32_t) * tiles, s));
    if (!(kSkip & 8)) {
      launched += tile_sort_fused(rb, k, id_bits, c->rrec, c->chunk_first, &sc->counts[1],
                                  ca.tiles_x, s);
      launched += launch_ranges_from_counts(c->tile_count, (int)tiles, ranges, cap_view, s);
    }
  } else {
  // K4
  tm.begin(2);
  LMGS_CUDA(c, cudaMemsetAsync(sc->tile_hist, 0, sizeof(sc->tile_hist), s));
  LMGS_CUDA(c, cudaMemsetAsync(sc->emit_ticket, 0, sizeof(uint32_t), s));
  if (n_vis > 0) {
    LMGS_CUDA(c, cudaMemsetAsync(c->emit_lookback, 0, sizeof(uint64_t) * emit_chunks(n_vis), s));
    EmitArgs ea{};
    ea.order_slot = &sc->slots.depth_ids;
    ea.rects = c->rects;
    ea.n_vis = n_vis;  // the grid's bound; the kernel reads the device count
    ea.n_vis_dev = &sc->counts[1];
    ea.cap = (uint64_t)cap_view;
    ea.tiles_x = ca.tiles_x;
    ea.n_tile_passes = tile_passes;
    ea.keys = c->inst_keys[0];
    ea.lookback = c->emit_lookback;
    ea.ticket = sc->emit_ticket;
    ea.hist = sc->tile_hist;
    ea.concurrent = (st->flags & LMGS_FLAG_CONCURRENT) != 0;
    if (!(kSkip & 4)) launched += launch_emit(ea, s);
  }
  tm.end(2);

  // K5 + K6
  tm.begin(3);
  {
    RadixSortBuffers rb{};
    rb.keys[0] = c->inst_keys[0];
    rb.keys[1] = c->inst_keys[1];
    rb.key_bytes = 8;
    rb.plan = &sc->tile_plan;
    rb.hist = sc->tile_hist;
    rb.lookback = c->tile_lookback;
    rb.counters = sc->tile_counters;
    rb.keys_result = &sc->slots.inst_ids;
    rb.hist_ready = true;
    rb.seg_counts = c->tile_count;
    rb.seg_shift = 32;
    rb.concurrent = (st->flags & LMGS_FLAG_CONCURRENT) != 0;
    if (nosync) {  // K on the device; the grid covers the capacity
      rb.n_dev = &sc->counts[2];
      rb.max_n = &sc->max_k;
    }
    LMGS_CUDA(c, cudaMemsetAsync(c->tile_count, 0, sizeof(uint32_t) * tiles, s));
    if (!(kSkip & 8)) {
      launched += tile_sort(rb, k, bits_for(tiles), id_bits, s);
      launched += launch_ranges_from_counts(c->tile_count, (int)tiles, ranges, cap_view, s);
    }
  }
  }
  if (out->tile_ranges && tiles > 0)
    LMGS_CUDA(c, cudaMemcpyAsync(out->tile_ranges, ranges, sizeof(int2) * tiles,
                                 cudaMemcpyDeviceToDevice, s));
  tm.end(3);

  // K7
  tm.begin(4);
  BlendArgs ba{};
  ba.concurrent = (st->flags & LMGS_FLAG_CONCURRENT) != 0;
  ba.keys_slot = &sc->slots.inst_ids;
  ba.ranges = ranges;
  ba.recs = c->recs;
  ba.width = cam->width;
  ba.height = cam->height;
  ba.tile_size = st->tile_size;
  ba.tiles_x = ca.tiles_x;
  ba.tiles_y = ca.tiles_y;
  for (int i = 0; i < 3; ++i) ba.bg[i] = (float)st->background[i];
  ba.rgb = out->rgb;
  ba.alpha = out->alpha;
  ba.depth = out->depth;
  ba.trans = out->transmittance;
  ba.touched = out->touched;
  ba.n_processed = out->n_processed;
  ba.work_counter = &sc->blend_counter;
  const bool fix = out->touched != nullptr && !(st->flags & LMGS_FLAG_NO_TOUCHED_FIX);
  if (fix) {
    // one entry per pixel: a pixel is queued at most once, so the queue
    // cannot overflow
    const int64_t cap = (int64_t)cam->width * cam->height;
    if ((size_t)cap * 4 > c->fixbuf.bytes) {
      LMGS_CUDA(c, cudaStreamSynchronize(s));
      LMGS_CUDA(c, c->fixbuf.reserve((size_t)cap * 4));
    }
    LMGS_CUDA(c, cudaMemsetAsync(&sc->fix_count, 0, sizeof(uint32_t), s));
    ba.fix_count = &sc->fix_count;
    ba.fix_list = static_cast<uint32_t*>(c->fixbuf.ptr);
    ba.fix_band = (st->flags & LMGS_FLAG_WIDE_FIX_BAND) ? 1e-2f : 1e-4f;
    if (out->n_processed) {
      // override i32, list u32, need u8: W * H entries each
      const size_t third = align_up((size_t)cap * 4);
      if (3 * third > c->npbuf.bytes) {
        LMGS_CUDA(c, cudaStreamSynchronize(s));
        LMGS_CUDA(c, c->npbuf.reserve(3 * third));
        // every override entry is -1 between views (k_nproc_reset restores it)
        LMGS_CUDA(c, cudaMemsetAsync(c->npbuf.ptr, 0xff, c->npbuf.bytes, s));
      }
      char* nb = static_cast<char*>(c->npbuf.ptr);
      LMGS_CUDA(c, cudaMemsetAsync(&sc->np_count, 0, sizeof(uint32_t), s));
      ba.np_count = &sc->np_count;
      ba.np_override = reinterpret_cast<int32_t*>(nb);
      ba.np_list = reinterpret_cast<const uint32_t*>(nb + third);
      ba.np_need = reinterpret_cast<const uint8_t*>(nb + 2 * third);
    }
  }
  if (strips) {
    ba.n_strips = strips->n_strips;
    ba.strip_rows = strips->strip_rows;
    for (int i = 0; i < strips->n_strips; ++i) {
      ba.srgb[i] = strips->rgb[i];
      ba.strans[i] = strips->trans[i];
      ba.sdepth[i] = strips->depth[i];
    }
  }
  if (!(kSkip & 16))
    if (int r = launch_blend(ba, s)) return fail(c, r, "too many blend blocks for this tile size");
  launched += tiles > 0 ? 1 : 0;
  tm.end(4);
  // K7b
  tm.begin(5);
  if (fix && tiles > 0) {
    TouchedFixArgs fa{};
    fa.keys_slot = &sc->slots.inst_ids;
    fa.ranges = ranges;
    fa.recs = c->recs;
    fa.tile_size = st->tile_size;
    fa.tiles_x = ca.tiles_x;
    fa.fix_count = &sc->fix_count;
    fa.fix_list = ba.fix_list;
    fa.width = cam->width;
    fa.touched = out->touched;
    fa.means = g->means;
    fa.quats = g->quats;
    fa.scales = g->scales;
    fa.logits = g->opacity_logits;
    fa.cam = ca;
    if (ba.np_count) {
      fa.np_count = &sc->np_count;
      fa.np_list = const_cast<uint32_t*>(ba.np_list);
      fa.np_need = const_cast<uint8_t*>(ba.np_need);
      fa.np_override = ba.np_override;
      fa.n_processed = out->n_processed;
    }
    launched += launch_touched_fix(fa, s);
    if (ba.np_count) launched += launch_nproc_fix(ba, s);
  }
  tm.end(5);
  c->stats.n_launches = launched;
  c->last_timed = vp->timed;
  LMGS_CUDA(c, cudaGetLastError());
  return LMGS_OK;
}

}  // namespace

extern "C" {

int lmgs_abi_version(void) { return LMGS_ABI_VERSION; }

int lmgs_context_create(int device, lmgs_context** out) {
  if (!out) return LMGS_ERR_INVALID;
  *out = nullptr;
  lmgs_context* c = new lmgs_context();
  c->device = device;
  DeviceGuard guard(device);
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  if (c->sms < 1) c->sms = 1;
  cudaError_t e = cudaMalloc(&c->d_scal, sizeof(Scalars));
  if (e == cudaSuccess) e = cudaMemset(c->d_scal, 0, sizeof(Scalars));
  if (e == cudaSuccess) e = cudaHostAlloc(&c->h_pinned, 8 * sizeof(uint64_t), cudaHostAllocDefault);
  if (e != cudaSuccess) {
    cudaGetLastError();
    lmgs_context_destroy(c);
    return e == cudaErrorMemoryAllocation ? LMGS_ERR_OOM : LMGS_ERR_CUDA;
  }
  if (cudaEventCreateWithFlags(&c->counts_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_pre, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    lmgs_context_destroy(c);
    return LMGS_ERR_CUDA;
  }
  c->events_ok = true;
  for (int i = 0; i < 2 * kNumStages; ++i)
    if (cudaEventCreate(&c->ev[i]) != cudaSuccess) c->events_ok = false;
  *out = c;
  return LMGS_OK;
}

void lmgs_context_destroy(lmgs_context* c) {
  if (!c) return;
  DeviceGuard guard(c->device);
  cudaDeviceSynchronize();
  c->gbuf.release();
  c->tbuf.release();
  c->ibuf.release();
  c->bwbuf.release();
  c->fixbuf.release();
  c->npbuf.release();
  if (c->d_scal) cudaFree(c->d_scal);
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  for (int i = 0; i < 2 * kNumStages; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  if (c->counts_ready) cudaEventDestroy(c->counts_ready);
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  if (c->ev_pre) cudaEventDestroy(c->ev_pre);
  delete c;
}

const char* lmgs_last_error(const lmgs_context* c) { return c ? c->err.c_str() : "null context"; }

int lmgs_render(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cam,
                const lmgs_settings* s, const lmgs_frame* out, void* stream) {
  if (int r = validate(c, g, cam, s)) return r;
  if (!out || !out->rgb) return fail(c, LMGS_ERR_INVALID, "frame.rgb is required");
  DeviceGuard guard(c->device);
  return render_one(c, g, cam, s, out, static_cast<cudaStream_t>(stream));
}

int lmgs_touched_fix_count(lmgs_context* c, uint32_t* count) {
  if (!c || !count) return LMGS_ERR_INVALID;
  DeviceGuard guard(c->device);
  LMGS_CUDA(c, cudaMemcpy(count, &c->d_scal->fix_count, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return LMGS_OK;
}

int lmgs_render_strips(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cam,
                       const lmgs_settings* s, const lmgs_strip_targets* t, int32_t* touched,
                       void* stream) {
  if (int r = validate(c, g, cam, s)) return r;
  if (!t || t->n_strips < 1 || t->n_strips > LMGS_MAX_STRIPS || t->strip_rows < 1 ||
      (int64_t)t->n_strips * t->strip_rows < cam->height ||
      (int64_t)(t->n_strips - 1) * t->strip_rows >= cam->height)
    return fail(c, LMGS_ERR_INVALID, "strip targets must cover the image rows exactly");
  for (int i = 0; i < t->n_strips; ++i)
    if (!t->rgb[i]) return fail(c, LMGS_ERR_INVALID, "null strip rgb target");
  lmgs_frame f{};
  f.touched = touched;
  DeviceGuard guard(c->device);
  return render_one(c, g, cam, s, &f, static_cast<cudaStream_t>(stream), t);
}

int lmgs_render_batch(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cams,
                      int32_t n_views, const lmgs_settings* s, const lmgs_frame* out,
                      void* stream) {
  if (n_views < 0 || (n_views > 0 && (!cams || !out)))
    return fail(c, LMGS_ERR_INVALID, "bad view batch");
  for (int v = 0; v < n_views; ++v) {
    if (int r = lmgs_render(c, g, cams + v, s, out + v, stream)) return r;
  }
  return LMGS_OK;
}

int lmgs_render_group(lmgs_context* const* ctxs, int32_t n_views, const lmgs_gaussians* g,
                      const lmgs_camera* cams, const lmgs_settings* s, const lmgs_frame* out,
                      void* const* streams) {
  if (!ctxs || n_views < 1 || n_views > LMGS_MAX_GROUP || !cams || !out || !streams)
    return ctxs && ctxs[0] ? fail(ctxs[0], LMGS_ERR_INVALID, "bad view group (1..8 views)")
                           : LMGS_ERR_INVALID;
  for (int v = 0; v < n_views; ++v) {
    lmgs_context* c = ctxs[v];
    if (!c) return LMGS_ERR_INVALID;
    if (int r = validate(c, g, cams + v, s)) return r;
    if (!out[v].rgb) return fail(c, LMGS_ERR_INVALID, "frame.rgb is required");
    if (c->device != ctxs[0]->device)
      return fail(c, LMGS_ERR_INVALID, "group contexts must share one device");
    for (int u = 0; u < v; ++u)
      if (ctxs[u] == c) return fail(c, LMGS_ERR_INVALID, "group contexts must be distinct");
  }
  DeviceGuard guard(ctxs[0]->device);
  cudaStream_t s0 = static_cast<cudaStream_t>(streams[0]);
  ViewPlan vp[LMGS_MAX_GROUP];
  PreprocessMulti m{};
  m.nv = n_views;
  if (s->flags & LMGS_FLAG_CONCURRENT) m.persist_ctas = LMGS_PRE_PERSIST_CTAS;
  for (int v = 0; v < n_views; ++v) {
    lmgs_context* c = ctxs[v];
    cudaStream_t sv = static_cast<cudaStream_t>(streams[v]);
    if (int r = view_prepare(c, g, cams + v, s, out + v, sv, vp + v)) return r;
    m.v[v] = make_pre(c, g, vp[v].ca, s, out[v].kept, out[v].touched);
    if (sv != s0) {  // K1 (on streams[0]) follows each view's resets
      LMGS_CUDA(c, cudaEventRecord(c->ev_in, sv));
      LMGS_CUDA(c, cudaStreamWaitEvent(s0, c->ev_in, 0));
    }
  }
  for (int v = 0; v < n_views; ++v) {
    ctxs[v]->pre_share = n_views;
    if (vp[v].timed) LMGS_CUDA(ctxs[v], cudaEventRecord(ctxs[v]->ev[0], s0));
  }
  // concurrent renders: the K1 launches of the batch run one after another
  // (each waits for the previous group's K1, in host order), the other
  // streams' sorts and blends filling the SMs around them
  cudaEvent_t k1_done = nullptr;
  if ((s->flags & LMGS_FLAG_CONCURRENT) && LMGS_SERIAL_K1) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s0, &cap);
    if (cap == cudaStreamCaptureStatusNone) {
      k1_done = k1_serial_event(ctxs[0]->device);
      if (k1_done) LMGS_CUDA(ctxs[0], cudaStreamWaitEvent(s0, k1_done, 0));
    }
  }
  const int k1 = launch_preprocess_multi(m, s0);
  if (k1_done) LMGS_CUDA(ctxs[0], cudaEventRecord(k1_done, s0));
  for (int v = 0; v < n_views; ++v) {
    lmgs_context* c = ctxs[v];
    cudaStream_t sv = static_cast<cudaStream_t>(streams[v]);
    vp[v].launched = v == 0 ? k1 : 0;  // the shared launch is counted once
    if (vp[v].timed) LMGS_CUDA(c, cudaEventRecord(c->ev[1], s0));
    if (sv != s0) {
      LMGS_CUDA(c, cudaEventRecord(c->ev_pre, s0));
      LMGS_CUDA(c, cudaStreamWaitEvent(sv, c->ev_pre, 0));
    }
  }
  for (int v = 0; v < n_views; ++v) {
    if (int r = view_finish(ctxs[v], g, cams + v, s, out + v, static_cast<cudaStream_t>(streams[v]),
                            vp + v, nullptr))
      return r;
  }
  return LMGS_OK;
}

int lmgs_get_stats(lmgs_context* c, lmgs_stats* out) {
  if (!c || !out) return LMGS_ERR_INVALID;
  DeviceGuard guard(c->device);
  if (c->counts_pending) {  // a no-sync render (possibly replayed from a graph)
    LMGS_CUDA(c, cudaDeviceSynchronize());
    c->stats.n_kept = (int64_t)c->h_pinned[0];
    c->stats.n_visible = (int64_t)c->h_pinned[1];
    c->stats.n_instances = (int64_t)c->h_pinned[2];
    c->counts_pending = false;
  }
  {
    int64_t seen = c->host_max_k;
    if (c->max_k_pending) {  // the device-side maximum of the no-sync renders
      unsigned long long mk = 0;
      LMGS_CUDA(c, cudaMemcpy(&mk, &c->d_scal->max_k, sizeof(mk), cudaMemcpyDeviceToHost));
      LMGS_CUDA(c, cudaMemset(&c->d_scal->max_k, 0, sizeof(mk)));
      if ((int64_t)mk > seen) seen = (int64_t)mk;
      c->stats.overflow = (int64_t)mk > c->stats.capacity ? 1 : 0;
      c->max_k_pending = false;
    } else {
      c->stats.overflow = 0;
    }
    c->stats.max_instances_seen = seen;
    c->host_max_k = 0;
  }
  if (c->last_timed) {
    LMGS_CUDA(c, cudaEventSynchronize(c->ev[2 * kNumStages - 1]));
    for (int i = 0; i < kNumStages; ++i) {
      float ms = 0.f;
      LMGS_CUDA(c, cudaEventElapsedTime(&ms, c->ev[2 * i], c->ev[2 * i + 1]));
      c->stats.stage_ms[i] = i == 0 ? ms / (float)c->pre_share : ms;
    }
  }
  *out = c->stats;
  return LMGS_OK;
}

int lmgs_copy_instances(lmgs_context* c, uint64_t* keys, int64_t* prim_ids, void* stream) {
  if (!c) return LMGS_ERR_INVALID;
  DeviceGuard guard(c->device);
  if (c->counts_pending) {
    lmgs_stats tmp;
    if (int r = lmgs_get_stats(c, &tmp)) return r;
  }
  InstanceExportArgs a{};
  a.ranges = c->last_ranges;
  a.keys_slot = &c->d_scal->slots.inst_ids;
  a.prim_ids = c->last_prim_ids;
  a.keys_out = keys;
  a.prims_out = prim_ids;
  a.k = c->stats.n_instances;
  a.tiles = c->stats.n_tiles;
  launch_export_instances(a, static_cast<cudaStream_t>(stream));
  LMGS_CUDA(c, cudaGetLastError());
  return LMGS_OK;
}

int lmgs_backward(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cam,
                  const lmgs_settings* s, const float* image_grad, double* d_colors,
                  double* d_opacities, double* d_mean2d, int32_t* touched, double* d_sh,
                  double* d_logits, double* grad_norm_sum, int64_t* steps_seen,
                  void* stream) {
  if (int r = validate(c, g, cam, s)) return r;
  if (!image_grad || (g->count > 0 && (!d_colors || !d_opacities || !d_mean2d || !touched)))
    return fail(c, LMGS_ERR_INVALID, "null backward output");
  const CamArgs ca = make_cam(cam, s->tile_size);
  const int64_t tiles = (int64_t)ca.tiles_x * ca.tiles_y;
  if (c->stats.n_gaussians != g->count || c->stats.n_tiles != tiles || !c->last_ranges)
    return fail(c, LMGS_ERR_INVALID, "lmgs_backward needs the view's lmgs_render first");
  DeviceGuard guard(c->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = g->count;
  if ((size_t)n * sizeof(BwRec) > c->bwbuf.bytes) {
    LMGS_CUDA(c, cudaStreamSynchronize(st));  // an earlier backward may still read it
    LMGS_CUDA(c, c->bwbuf.reserve((size_t)(n > 0 ? n : 1) * sizeof(BwRec)));
  }
  BackwardArgs a{};
  a.recs = static_cast<BwRec*>(c->bwbuf.ptr);
  a.blocks_x = (s->tile_size + 7) / 8;
  a.blocks = a.blocks_x * ((s->tile_size + 3) / 4);
  a.means = g->means;
  a.quats = g->quats;
  a.scales = g->scales;
  a.logits = g->opacity_logits;
  a.sh = g->sh;
  a.n = n;
  a.sh_coeffs = g->sh_coeffs;
  a.eval_degree = s->sh_eval_degree < g->sh_degree ? s->sh_eval_degree : g->sh_degree;
  a.cam = ca;
  a.keys_slot = &c->d_scal->slots.inst_ids;
  a.ranges = c->last_ranges;
  a.width = cam->width;
  a.height = cam->height;
  a.tile_size = s->tile_size;
  a.tiles_x = ca.tiles_x;
  for (int i = 0; i < 3; ++i) a.bg[i] = s->background[i];
  a.image_grad = image_grad;
  a.d_colors = d_colors;
  a.d_opacities = d_opacities;
  a.d_mean2d = d_mean2d;
  a.touched = touched;
  a.d_sh = d_sh;
  a.d_logits = d_logits;
  a.grad_norm_sum = grad_norm_sum;
  a.steps_seen = steps_seen;
  launch_backward(a, (int)tiles, st);
  LMGS_CUDA(c, cudaGetLastError());
  return LMGS_OK;
}

int lmgs_record_collect(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cam,
                        const lmgs_settings* s, const int64_t* tile_offsets, double* sigma,
                        double* t_before, double* t_final, double* colors, double* opacities,
                        void* stream) {
  if (int r = validate(c, g, cam, s)) return r;
  if (!tile_offsets || !sigma || !t_before || !t_final)
    return fail(c, LMGS_ERR_INVALID, "null collect output");
  const CamArgs ca = make_cam(cam, s->tile_size);
  const int64_t tiles = (int64_t)ca.tiles_x * ca.tiles_y;
  if (c->stats.n_gaussians != g->count || c->stats.n_tiles != tiles || !c->last_ranges)
    return fail(c, LMGS_ERR_INVALID, "lmgs_record_collect needs the view's lmgs_render first");
  DeviceGuard guard(c->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = g->count;
  if ((size_t)n * sizeof(BwRec) > c->bwbuf.bytes) {
    LMGS_CUDA(c, cudaStreamSynchronize(st));
    LMGS_CUDA(c, c->bwbuf.reserve((size_t)(n > 0 ? n : 1) * sizeof(BwRec)));
  }
  BackwardArgs p{};
  p.recs = static_cast<BwRec*>(c->bwbuf.ptr);
  p.means = g->means;
  p.quats = g->quats;
  p.scales = g->scales;
  p.logits = g->opacity_logits;
  p.sh = g->sh;
  p.n = n;
  p.sh_coeffs = g->sh_coeffs;
  p.eval_degree = s->sh_eval_degree < g->sh_degree ? s->sh_eval_degree : g->sh_degree;
  p.cam = ca;
  CollectArgs a{};
  a.recs = p.recs;
  a.keys_slot = &c->d_scal->slots.inst_ids;
  a.ranges = c->last_ranges;
  a.offsets = tile_offsets;
  a.width = cam->width;
  a.height = cam->height;
  a.tile_size = s->tile_size;
  a.tiles_x = ca.tiles_x;
  a.sigma = sigma;
  a.t_before = t_before;
  a.t_final = t_final;
  launch_collect(p, a, (int)tiles, st);
  if (n > 0 && (colors || opacities)) {  // the records' fp64 colour and opacity
    if (colors)
      LMGS_CUDA(c, cudaMemcpy2DAsync(colors, 3 * sizeof(double),
                                     reinterpret_cast<const char*>(p.recs) + offsetof(BwRec, col),
                                     sizeof(BwRec), 3 * sizeof(double), (size_t)n,
                                     cudaMemcpyDeviceToDevice, st));
    if (opacities)
      LMGS_CUDA(c, cudaMemcpy2DAsync(opacities, sizeof(double),
                                     reinterpret_cast<const char*>(p.recs) + offsetof(BwRec, op),
                                     sizeof(BwRec), sizeof(double), (size_t)n,
                                     cudaMemcpyDeviceToDevice, st));
  }
  LMGS_CUDA(c, cudaGetLastError());
  return LMGS_OK;
}

int lmgs_project(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cam,
                 const lmgs_settings* s, double* mean2d, double* cov2d, double* depth,
                 double* radius, float* colors, float* opacity, uint8_t* kept, void* stream) {
  if (int r = validate(c, g, cam, s)) return r;
  if (g->count > 0 && (!mean2d || !cov2d || !depth || !radius || !colors || !opacity))
    return fail(c, LMGS_ERR_INVALID, "null output");
  DeviceGuard guard(c->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = g->count;
  if (int r = ensure_gaussians(c, n > 0 ? n : 1, st)) return r;
  PreprocessArgs pa = make_pre(c, g, make_cam(cam, s->tile_size), s, kept);
  pa.dbg_mean2d = mean2d;
  pa.dbg_cov2d = cov2d;
  pa.dbg_depth = depth;
  pa.dbg_radius = radius;
  pa.dbg_colors = colors;
  pa.dbg_opacity = opacity;
  launch_preprocess(pa, st);
  LMGS_CUDA(c, cudaGetLastError());
  return LMGS_OK;
}

int lmgs_composite_blocks(const float* rgb, const float* trans, const float* depth,
                          int32_t n_blocks, const int32_t* order_host, int64_t n_pixels,
                          const float* background_host, float* out_rgb, float* out_alpha,
                          float* out_depth, void* stream) {
  if (n_blocks < 0 || n_blocks > kMaxCompositeBlocks || n_pixels < 0) return LMGS_ERR_INVALID;
  if (!rgb || !trans || !out_rgb || (n_blocks > 0 && !order_host)) return LMGS_ERR_INVALID;
  for (int i = 0; i < n_blocks; ++i)
    if (order_host[i] < 0 || order_host[i] >= n_blocks) return LMGS_ERR_INVALID;
  float bg[3] = {0.f, 0.f, 0.f};
  if (background_host) memcpy(bg, background_host, sizeof(bg));
  launch_composite(rgb, trans, depth, n_blocks, order_host, n_pixels, bg, out_rgb, out_alpha,
                   out_depth, static_cast<cudaStream_t>(stream));
  return cudaGetLastError() == cudaSuccess ? LMGS_OK : LMGS_ERR_CUDA;
}

}  // extern "C"
