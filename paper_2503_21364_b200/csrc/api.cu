// C-ABI entry points (include/lmgs.h): context, device arena, stage pipeline.
//
// One view:
//   K1 preprocess  (fp64 geometry, tile rect, blend record)
//   K3 tile counts (per-SM shared-memory histograms + column scan) and tile
//      scan (one CTA: ranges, size classes, K) -> one 8-byte D2H read of K
//   K4 place       (shared-memory cursors: each instance into its tile bucket)
//   K5 tile sort   (per-tile smem LSD radix on the fp32 depth + exact fp64 fix-up;
//                   oversized buckets: onesweep radix + the same fix-up)
//   K7 blend       (persistent warps over (tile, 8x4 block) items)
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "lmgs_internal.cuh"

using namespace lmgs;

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

const char* kStageNames[] = {"preprocess", "tile_scan", "place", "tile_sort", "blend"};
constexpr int kNumStages = 5;

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
  b += align_up(sizeof(uint32_t) * n);  // fp32 depth keys
  b += align_up(sizeof(uint64_t) * n);  // fp64 depth keys
  b += align_up(sizeof(uint64_t) * n);  // rects
  b += align_up(sizeof(uint32_t) * n);  // tile counts
  b += align_up(sizeof(BlendRec) * n);  // records
  return b + 8 * kAlign;
}
size_t tile_bytes(int64_t t, int ctas) {
  return align_up(sizeof(uint32_t) * t * ctas) + 5 * align_up(sizeof(uint32_t) * t) +
         align_up(sizeof(int2) * t) + 8 * kAlign;
}
size_t instance_bytes(int64_t k) {
  return 2 * align_up(sizeof(uint32_t) * k) + 4 * kAlign;
}
size_t big_bytes(int64_t k) {
  return 2 * align_up(sizeof(uint64_t) * k) + 2 * align_up(sizeof(uint32_t) * k) +
         align_up(sizeof(uint32_t) * radix_lookback_words(k)) + 8 * kAlign;
}

struct Scalars {  // device-side small state
  RadixPlan big_plan;
  uint32_t hist[kMaxPasses * kRadix];
  uint32_t counters[kMaxPasses];
  uint32_t class_counts[4];
  unsigned long long n_kept;
  uint64_t total;
  unsigned long long big_total;
  int blend_counter;
  int pad;
  DevSlots slots;
};

}  // namespace

struct lmgs_context {
  int device = 0;
  int sms = 148;  // K3a / K4 CTA slices (one per SM)
  std::string err;
  DevBuf gbuf, tbuf, ibuf, bbuf;
  Scalars* d_scal = nullptr;
  uint64_t* h_pinned = nullptr;  // [0]=K [1]=kept [2]=class counts (3 x u32 packed)
  cudaEvent_t ev[kNumStages + 1] = {};
  bool events_ok = false;
  int64_t cap_n = -1, cap_t = -1, cap_k = -1, cap_big = -1;
  // per-Gaussian arena
  uint32_t* key32 = nullptr;
  uint64_t* key64 = nullptr;
  uint64_t* rects = nullptr;
  uint32_t* tile_counts = nullptr;
  BlendRec* recs = nullptr;
  // per-tile arena
  uint32_t* bin_hist = nullptr;   // [sms][tiles]
  uint32_t* tile_count = nullptr;
  uint32_t* lists[3] = {nullptr, nullptr, nullptr};
  uint32_t* big_off = nullptr;
  int2* ranges = nullptr;
  // per-instance arena
  uint32_t* bucket = nullptr;
  uint32_t* sorted_ids = nullptr;
  // oversized-bucket arena
  uint64_t* big_keys[2] = {nullptr, nullptr};
  uint32_t* big_vals[2] = {nullptr, nullptr};
  uint32_t* big_lookback = nullptr;
  const int64_t* last_prim_ids = nullptr;
  const int2* last_ranges = nullptr;
  int64_t big_views = 0;  // views that needed the oversized-bucket path
  lmgs_stats stats{};
  bool last_timed = false;
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
  c->key32 = cv.take<uint32_t>(cap);
  c->key64 = cv.take<uint64_t>(cap);
  c->rects = cv.take<uint64_t>(cap);
  c->tile_counts = cv.take<uint32_t>(cap);
  c->recs = cv.take<BlendRec>(cap);
  c->cap_n = cap;
  return LMGS_OK;
}

int ensure_tiles(lmgs_context* c, int64_t t, cudaStream_t s) {
  if (t <= c->cap_t && c->ranges) return LMGS_OK;
  LMGS_CUDA(c, cudaStreamSynchronize(s));
  LMGS_CUDA(c, c->tbuf.reserve(tile_bytes(t, c->sms)));
  Carver cv{static_cast<char*>(c->tbuf.ptr)};
  c->bin_hist = cv.take<uint32_t>(t * c->sms);
  c->tile_count = cv.take<uint32_t>(t);
  for (int i = 0; i < 3; ++i) c->lists[i] = cv.take<uint32_t>(t);
  c->big_off = cv.take<uint32_t>(t);
  c->ranges = cv.take<int2>(t);
  c->cap_t = t;
  return LMGS_OK;
}

int ensure_instances(lmgs_context* c, int64_t k, cudaStream_t s) {
  if (k <= c->cap_k && c->bucket) return LMGS_OK;
  LMGS_CUDA(c, cudaStreamSynchronize(s));
  LMGS_CUDA(c, c->ibuf.reserve(instance_bytes(k)));
  const int64_t cap = (int64_t)(c->ibuf.bytes >= instance_bytes(k + k / 4) ? k + k / 4 : k);
  Carver cv{static_cast<char*>(c->ibuf.ptr)};
  c->bucket = cv.take<uint32_t>(cap);
  c->sorted_ids = cv.take<uint32_t>(cap);
  c->cap_k = cap;
  return LMGS_OK;
}

int ensure_big(lmgs_context* c, int64_t k, cudaStream_t s) {
  if (k <= c->cap_big && c->big_keys[0]) return LMGS_OK;
  LMGS_CUDA(c, cudaStreamSynchronize(s));
  LMGS_CUDA(c, c->bbuf.reserve(big_bytes(k)));
  Carver cv{static_cast<char*>(c->bbuf.ptr)};
  c->big_keys[0] = cv.take<uint64_t>(k);
  c->big_keys[1] = cv.take<uint64_t>(k);
  c->big_vals[0] = cv.take<uint32_t>(k);
  c->big_vals[1] = cv.take<uint32_t>(k);
  c->big_lookback = cv.take<uint32_t>(radix_lookback_words(k));
  c->cap_big = k;
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
  if (s->tile_size < 1) return fail(c, LMGS_ERR_INVALID, "tile_size must be >= 1");
  if (s->tile_size > 64) return fail(c, LMGS_ERR_UNSUPPORTED, "tile_size > 64 not supported");
  if (cam->width < 1 || cam->height < 1) return fail(c, LMGS_ERR_INVALID, "bad image size");
  if (cam->width > 65535 * s->tile_size || cam->height > 65535 * s->tile_size)
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
                        const lmgs_settings* st, uint8_t* kept) {
  PreprocessArgs pa{};
  pa.means = g->means;
  pa.quats = g->quats;
  pa.scales = g->scales;
  pa.logits = g->opacity_logits;
  pa.sh = g->sh;
  pa.n = g->count;
  pa.sh_coeffs = g->sh_coeffs;
  pa.eval_degree = st->sh_eval_degree < g->sh_degree ? st->sh_eval_degree : g->sh_degree;
  pa.cam = ca;
  pa.depth_keys32 = c->key32;
  pa.depth_keys = c->key64;
  pa.rects = c->rects;
  pa.tile_counts = c->tile_counts;
  pa.recs = c->recs;
  pa.kept = kept;
  pa.n_kept = &c->d_scal->n_kept;
  return pa;
}

// oversized buckets: gather, onesweep on (bucket index << 32 | fp32 key), fix-up, scatter
int sort_big_tiles(lmgs_context* c, const TileSortArgs& ta, int n_big, cudaStream_t s) {
  // big list + ranges to host (rare path), offsets on host
  std::vector<uint32_t> tiles(n_big);
  std::vector<int2> rg(c->cap_t);
  LMGS_CUDA(c, cudaMemcpyAsync(tiles.data(), c->lists[2], sizeof(uint32_t) * n_big,
                               cudaMemcpyDeviceToHost, s));
  LMGS_CUDA(c, cudaMemcpyAsync(rg.data(), ta.ranges, sizeof(int2) * c->stats.n_tiles,
                               cudaMemcpyDeviceToHost, s));
  LMGS_CUDA(c, cudaStreamSynchronize(s));
  std::vector<uint32_t> off(n_big);
  int64_t total = 0;
  for (int b = 0; b < n_big; ++b) {
    off[b] = (uint32_t)total;
    total += rg[tiles[b]].y - rg[tiles[b]].x;
  }
  if (int r = ensure_big(c, total, s)) return r;
  LMGS_CUDA(c, cudaMemcpyAsync(c->big_off, off.data(), sizeof(uint32_t) * n_big,
                               cudaMemcpyHostToDevice, s));
  launch_big_gather(ta, c->lists[2], n_big, c->big_off, c->big_keys[0], c->big_vals[0], s);
  RadixSortBuffers rb{};
  rb.keys[0] = c->big_keys[0];
  rb.keys[1] = c->big_keys[1];
  rb.key_bytes = 8;
  rb.vals[0] = c->big_vals[0];
  rb.vals[1] = c->big_vals[1];
  rb.plan = &c->d_scal->big_plan;
  rb.hist = c->d_scal->hist;
  rb.lookback = c->big_lookback;
  rb.counters = c->d_scal->counters;
  rb.keys_result = &c->d_scal->slots.big_keys;
  rb.vals_result = &c->d_scal->slots.big_vals;
  radix_sort(rb, total, 0, (32 + bits_for(n_big) + 7) / 8, s);
  launch_big_fixup(&c->d_scal->slots.big_keys, &c->d_scal->slots.big_vals, total, ta.key64, s);
  launch_big_scatter(ta, c->lists[2], n_big, c->big_off, &c->d_scal->slots.big_vals, s);
  ++c->big_views;
  return LMGS_OK;
}

int render_one(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cam,
               const lmgs_settings* st, const lmgs_frame* out, cudaStream_t s) {
  const bool timed = (st->flags & LMGS_FLAG_STAGE_TIMES) && c->events_ok;
  const CamArgs ca = make_cam(cam, st->tile_size);
  const int64_t n = g->count;
  const int64_t tiles = (int64_t)ca.tiles_x * ca.tiles_y;
  c->stats = lmgs_stats{};
  c->stats.n_gaussians = n;
  c->stats.n_tiles = (int32_t)tiles;
  c->stats.tiles_x = ca.tiles_x;
  c->stats.tiles_y = ca.tiles_y;
  c->stats.n_stages = kNumStages;
  for (int i = 0; i < kNumStages; ++i) c->stats.stage_names[i] = kStageNames[i];
  c->last_timed = false;
  c->last_prim_ids = g->prim_ids;

  if (int r = ensure_gaussians(c, n > 0 ? n : 1, s)) return r;
  if (int r = ensure_tiles(c, tiles, s)) return r;
  int2* ranges = out->tile_ranges ? reinterpret_cast<int2*>(out->tile_ranges) : c->ranges;
  c->last_ranges = ranges;
  LMGS_CUDA(c, cudaMemsetAsync(&c->d_scal->n_kept, 0, sizeof(unsigned long long), s));
  if (out->touched && n > 0) LMGS_CUDA(c, cudaMemsetAsync(out->touched, 0, sizeof(int32_t) * n, s));

  if (timed) LMGS_CUDA(c, cudaEventRecord(c->ev[0], s));
  launch_preprocess(make_pre(c, g, ca, st, out->kept), s);
  if (timed) LMGS_CUDA(c, cudaEventRecord(c->ev[1], s));

  BinArgs bin{};
  bin.rects = c->rects;
  bin.counts = c->tile_counts;
  bin.key32 = c->key32;
  bin.n = n;
  bin.tiles_x = ca.tiles_x;
  bin.tiles = (int)tiles;
  bin.ctas = c->sms;
  bin.hist = c->bin_hist;
  bin.tile_count = c->tile_count;
  bin.ranges = ranges;
  launch_bin_hist(bin, s);

  TileScanArgs sa{};
  sa.tile_count = c->tile_count;
  sa.tiles = (int)tiles;
  sa.small_cap = kSmallTileCap;
  sa.medium_cap = kMediumTileCap;
  sa.ranges = ranges;
  for (int i = 0; i < 3; ++i) sa.lists[i] = c->lists[i];
  sa.class_counts = c->d_scal->class_counts;
  sa.total = &c->d_scal->total;
  launch_scan_tiles(sa, s);
  LMGS_CUDA(c, cudaMemcpyAsync(c->h_pinned, &c->d_scal->total, sizeof(uint64_t),
                               cudaMemcpyDeviceToHost, s));
  LMGS_CUDA(c, cudaMemcpyAsync(c->h_pinned + 1, &c->d_scal->n_kept, sizeof(uint64_t),
                               cudaMemcpyDeviceToHost, s));
  LMGS_CUDA(c, cudaMemcpyAsync(c->h_pinned + 2, c->d_scal->class_counts, 4 * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, s));
  LMGS_CUDA(c, cudaGetLastError());
  LMGS_CUDA(c, cudaStreamSynchronize(s));
  const int64_t k = (int64_t)c->h_pinned[0];
  c->stats.n_instances = k;
  c->stats.n_kept = (int64_t)c->h_pinned[1];
  const uint32_t* cls = reinterpret_cast<const uint32_t*>(c->h_pinned + 2);
  const int n_small = (int)cls[0], n_medium = (int)cls[1], n_big = (int)cls[2];
  if (k >= ((int64_t)1 << 31) - 1)
    return fail(c, LMGS_ERR_UNSUPPORTED, "more than 2^31 tile instances in one view");
  if (timed) LMGS_CUDA(c, cudaEventRecord(c->ev[2], s));

  if (int r = ensure_instances(c, k > 0 ? k : 1, s)) return r;
  bin.bucket = c->bucket;
  if (k > 0) launch_bin_place(bin, s);
  if (timed) LMGS_CUDA(c, cudaEventRecord(c->ev[3], s));

  TileSortArgs ta{};
  ta.bucket = c->bucket;
  ta.key32 = c->key32;
  ta.ranges = ranges;
  ta.key64 = c->key64;
  ta.sorted_ids = c->sorted_ids;
  launch_tile_sort(ta, c->lists[0], c->d_scal->class_counts + 0, n_small, 0, s);
  launch_tile_sort(ta, c->lists[1], c->d_scal->class_counts + 1, n_medium, 1, s);
  if (n_big > 0) {
    if (int r = sort_big_tiles(c, ta, n_big, s)) return r;
  }
  if (timed) LMGS_CUDA(c, cudaEventRecord(c->ev[4], s));

  BlendArgs ba{};
  ba.sorted_ids = c->sorted_ids;
  ba.ranges = ranges;
  ba.recs = c->recs;
  ba.width = cam->width;
  ba.height = cam->height;
  ba.tile_size = st->tile_size;
  ba.tiles_x = ca.tiles_x;
  ba.tiles_y = ca.tiles_y;
  for (int i = 0; i < 3; ++i) ba.bg[i] = st->background[i];
  ba.rgb = out->rgb;
  ba.alpha = out->alpha;
  ba.depth = out->depth;
  ba.trans = out->transmittance;
  ba.touched = out->touched;
  ba.n_processed = out->n_processed;
  ba.work_counter = &c->d_scal->blend_counter;
  if (int r = launch_blend(ba, s)) return fail(c, r, "unsupported tile size");
  if (timed) {
    LMGS_CUDA(c, cudaEventRecord(c->ev[5], s));
    c->last_timed = true;
  }
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
  c->events_ok = true;
  for (int i = 0; i <= kNumStages; ++i)
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
  c->bbuf.release();
  if (c->d_scal) cudaFree(c->d_scal);
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  for (int i = 0; i <= kNumStages; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
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

int lmgs_get_stats(lmgs_context* c, lmgs_stats* out) {
  if (!c || !out) return LMGS_ERR_INVALID;
  DeviceGuard guard(c->device);
  if (c->last_timed) {
    LMGS_CUDA(c, cudaEventSynchronize(c->ev[kNumStages]));
    for (int i = 0; i < kNumStages; ++i) {
      float ms = 0.f;
      LMGS_CUDA(c, cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]));
      c->stats.stage_ms[i] = ms;
    }
  }
  *out = c->stats;
  return LMGS_OK;
}

int lmgs_copy_instances(lmgs_context* c, uint64_t* keys, int64_t* prim_ids, void* stream) {
  if (!c) return LMGS_ERR_INVALID;
  DeviceGuard guard(c->device);
  InstanceExportArgs a{};
  a.ranges = c->last_ranges;
  a.sorted_ids = c->sorted_ids;
  a.prim_ids = c->last_prim_ids;
  a.keys_out = keys;
  a.prims_out = prim_ids;
  if (c->stats.n_instances > 0)
    launch_export_instances(a, c->stats.n_tiles, static_cast<cudaStream_t>(stream));
  LMGS_CUDA(c, cudaGetLastError());
  return LMGS_OK;
}

int lmgs_project(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cam,
                 const lmgs_settings* s, double* mean2d, double* cov2d, double* depth,
                 double* radius, float* colors, float* opacity, uint8_t* kept, void* stream) {
  if (int r = validate(c, g, cam, s)) return r;
  if (!mean2d || !cov2d || !depth || !radius || !colors || !opacity)
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
