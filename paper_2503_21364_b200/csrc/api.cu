// C-ABI entry points (include/lmgs.h): context, device arena, stage pipeline.
//
// One view = K1 preprocess -> K2 depth-rank radix sort -> K3 rank-order scan
// of tiles_touched -> (one 8-byte device->host read of K) -> K4 duplicate ->
// K5 tile radix sort -> K6 tile ranges -> K7 blend.
#include <cstdio>
#include <cstring>
#include <string>

#include "lmgs_internal.cuh"

using namespace lmgs;

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

const char* kStageNames[] = {"preprocess", "depth_sort", "scan", "duplicate",
                             "tile_sort",  "tile_ranges", "blend"};
constexpr int kNumStages = 7;

// grow-only device buffer
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaError_t reserve(size_t need) {
    if (need <= bytes) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    size_t want = need + need / 4;  // headroom against per-view K jitter
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

// sizes of the per-Gaussian arena for capacity n
size_t gaussian_bytes(int64_t n) {
  size_t b = 0;
  b += 2 * align_up(sizeof(uint32_t) * n);  // fp32 depth keys x2
  b += 2 * align_up(sizeof(uint64_t) * n);  // fp64 depth keys x2
  b += 3 * align_up(sizeof(uint32_t) * n);  // ids x3
  b += align_up(sizeof(uint64_t) * n);      // rects
  b += align_up(sizeof(uint32_t) * n);      // tile counts
  b += align_up(sizeof(BlendRec) * n);      // records
  b += align_up(sizeof(uint64_t) * n);      // offsets
  b += align_up(sizeof(uint32_t) * radix_lookback_words(n));
  b += align_up(sizeof(unsigned long long) * scan_status_words(n));
  return b + 16 * kAlign;
}
size_t instance_bytes(int64_t k) {
  size_t b = 0;
  b += 2 * align_up(sizeof(uint64_t) * k);
  b += align_up(sizeof(uint32_t) * radix_lookback_words(k));
  return b + 8 * kAlign;
}

struct Scalars {  // device-side small state
  RadixPlan depth_plan;
  RadixPlan fallback_plan;
  RadixPlan tile_plan;
  uint32_t hist[3][kMaxPasses * kRadix];
  uint32_t counters[3][kMaxPasses];
  uint32_t scan_counter;
  int blend_counter;
  unsigned long long n_kept;
  uint64_t total;
  DevSlots slots;
};

}  // namespace

struct lmgs_context {
  int device = 0;
  std::string err;
  DevBuf gbuf, ibuf, fbuf;
  Scalars* d_scal = nullptr;
  uint64_t* h_pinned = nullptr;  // [0] = K, [1] = kept, [2] = fallback flag
  cudaEvent_t ev[kNumStages + 1] = {};
  bool events_ok = false;
  // views into the arenas for the current / last render
  int64_t cap_n = -1, cap_k = -1;
  uint32_t* keys32[2] = {nullptr, nullptr};
  uint64_t* keys64[2] = {nullptr, nullptr};
  uint32_t* ids[3] = {nullptr, nullptr, nullptr};
  int64_t fallbacks = 0;  // views that needed the 64-bit depth sort
  uint64_t* rects = nullptr;
  uint32_t* tile_counts = nullptr;
  BlendRec* recs = nullptr;
  uint64_t* offsets = nullptr;
  uint32_t* depth_lookback = nullptr;
  unsigned long long* scan_status = nullptr;
  uint64_t* inst_keys[2] = {nullptr, nullptr};
  uint32_t* inst_lookback = nullptr;
  int2* ranges = nullptr;
  int64_t ranges_cap = -1;
  const int64_t* last_prim_ids = nullptr;
  // stats of the last render
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
  c->keys32[0] = cv.take<uint32_t>(cap);
  c->keys32[1] = cv.take<uint32_t>(cap);
  c->keys64[0] = cv.take<uint64_t>(cap);
  c->keys64[1] = cv.take<uint64_t>(cap);
  c->ids[0] = cv.take<uint32_t>(cap);
  c->ids[1] = cv.take<uint32_t>(cap);
  c->ids[2] = cv.take<uint32_t>(cap);
  c->rects = cv.take<uint64_t>(cap);
  c->tile_counts = cv.take<uint32_t>(cap);
  c->recs = cv.take<BlendRec>(cap);
  c->offsets = cv.take<uint64_t>(cap);
  c->depth_lookback = cv.take<uint32_t>(radix_lookback_words(cap));
  c->scan_status = cv.take<unsigned long long>(scan_status_words(cap));
  c->cap_n = cap;
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
  c->inst_lookback = cv.take<uint32_t>(radix_lookback_words(cap));
  c->cap_k = cap;
  return LMGS_OK;
}

int ensure_ranges(lmgs_context* c, int64_t tiles, cudaStream_t s) {
  if (tiles <= c->ranges_cap && c->ranges) return LMGS_OK;
  LMGS_CUDA(c, cudaStreamSynchronize(s));
  LMGS_CUDA(c, c->fbuf.reserve(align_up(sizeof(int2) * tiles)));
  c->ranges = static_cast<int2*>(c->fbuf.ptr);
  c->ranges_cap = (int64_t)(c->fbuf.bytes / sizeof(int2));
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

int render_one(lmgs_context* c, const lmgs_gaussians* g, const lmgs_camera* cam,
               const lmgs_settings* st, const lmgs_frame* out, cudaStream_t s) {
  const bool timed = (st->flags & LMGS_FLAG_STAGE_TIMES) && c->events_ok;
  const CamArgs ca = make_cam(cam, st->tile_size);
  const int64_t n = g->count;
  const int64_t tiles = (int64_t)ca.tiles_x * ca.tiles_y;
  const int64_t npix = (int64_t)cam->width * cam->height;
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
  if (int r = ensure_ranges(c, tiles, s)) return r;
  int2* ranges = out->tile_ranges ? reinterpret_cast<int2*>(out->tile_ranges) : c->ranges;
  LMGS_CUDA(c, cudaMemsetAsync(ranges, 0, sizeof(int2) * tiles, s));
  LMGS_CUDA(c, cudaMemsetAsync(&c->d_scal->n_kept, 0, sizeof(unsigned long long), s));
  LMGS_CUDA(c, cudaMemsetAsync(&c->d_scal->slots.fallback, 0, sizeof(int), s));
  if (out->touched && n > 0) LMGS_CUDA(c, cudaMemsetAsync(out->touched, 0, sizeof(int32_t) * n, s));

  if (timed) LMGS_CUDA(c, cudaEventRecord(c->ev[0], s));
  PreprocessArgs pa{};
  pa.means = g->means;
  pa.quats = g->quats;
  pa.scales = g->scales;
  pa.logits = g->opacity_logits;
  pa.sh = g->sh;
  pa.n = n;
  pa.sh_coeffs = g->sh_coeffs;
  pa.eval_degree = st->sh_eval_degree < g->sh_degree ? st->sh_eval_degree : g->sh_degree;
  pa.cam = ca;
  pa.depth_keys32 = c->keys32[0];
  pa.depth_keys = c->keys64[0];
  pa.ids = c->ids[0];
  pa.ids_fb = c->ids[2];
  pa.rects = c->rects;
  pa.tile_counts = c->tile_counts;
  pa.recs = c->recs;
  pa.kept = out->kept;
  pa.n_kept = &c->d_scal->n_kept;
  launch_preprocess(pa, s);
  if (timed) LMGS_CUDA(c, cudaEventRecord(c->ev[1], s));

  // K2: depth order = fp32-key radix sort + exact fp64 fix-up of equal-key runs
  DevSlots* slots = &c->d_scal->slots;
  RadixSortBuffers db{};
  db.keys[0] = c->keys32[0];
  db.keys[1] = c->keys32[1];
  db.key_bytes = 4;
  db.vals[0] = c->ids[0];
  db.vals[1] = c->ids[1];
  db.plan = &c->d_scal->depth_plan;
  db.hist = c->d_scal->hist[0];
  db.lookback = c->depth_lookback;
  db.counters = c->d_scal->counters[0];
  db.keys_result = &slots->depth_keys32;
  db.vals_result = &slots->sorted_ids;
  radix_sort(db, n, 0, 4, s);
  depth_fixup(&slots->depth_keys32, &slots->sorted_ids, n, c->keys64[0], &slots->fallback, s);
  if (timed) LMGS_CUDA(c, cudaEventRecord(c->ev[2], s));

  // K3: tiles_touched in depth order -> exclusive offsets and K
  scan_counts(c->tile_counts, &slots->sorted_ids, n, c->offsets, &c->d_scal->total,
              c->scan_status, &c->d_scal->scan_counter, s);
  LMGS_CUDA(c, cudaMemcpyAsync(c->h_pinned, &c->d_scal->total, sizeof(uint64_t),
                               cudaMemcpyDeviceToHost, s));
  LMGS_CUDA(c, cudaMemcpyAsync(c->h_pinned + 1, &c->d_scal->n_kept, sizeof(uint64_t),
                               cudaMemcpyDeviceToHost, s));
  LMGS_CUDA(c, cudaMemcpyAsync(c->h_pinned + 2, &slots->fallback, sizeof(int),
                               cudaMemcpyDeviceToHost, s));
  LMGS_CUDA(c, cudaGetLastError());
  LMGS_CUDA(c, cudaStreamSynchronize(s));
  const int64_t k = (int64_t)c->h_pinned[0];
  c->stats.n_instances = k;
  c->stats.n_kept = (int64_t)c->h_pinned[1];
  if (*reinterpret_cast<int*>(c->h_pinned + 2)) {
    // a run of > kFixupRun equal fp32 depths: exact 64-bit (depth, id) sort
    ++c->fallbacks;
    RadixSortBuffers fb{};
    fb.keys[0] = c->keys64[0];
    fb.keys[1] = c->keys64[1];
    fb.key_bytes = 8;
    fb.vals[0] = c->ids[2];
    fb.vals[1] = c->ids[0];
    fb.plan = &c->d_scal->fallback_plan;
    fb.hist = c->d_scal->hist[1];
    fb.lookback = c->depth_lookback;
    fb.counters = c->d_scal->counters[1];
    fb.keys_result = &slots->fb_keys;
    fb.vals_result = &slots->sorted_ids;
    radix_sort(fb, n, 0, 8, s);
    scan_counts(c->tile_counts, &slots->sorted_ids, n, c->offsets, &c->d_scal->total,
                c->scan_status, &c->d_scal->scan_counter, s);
  }
  if (k >= ((int64_t)1 << 30) - 1)
    return fail(c, LMGS_ERR_UNSUPPORTED, "more than 2^30 tile instances in one view");
  if (timed) LMGS_CUDA(c, cudaEventRecord(c->ev[3], s));

  if (int r = ensure_instances(c, k > 0 ? k : 1, s)) return r;
  DuplicateArgs da{};
  da.slots = slots;
  da.rects = c->rects;
  da.tile_counts = c->tile_counts;
  da.offsets = c->offsets;
  da.n = n;
  da.tiles_x = ca.tiles_x;
  da.keys_out = c->inst_keys[0];
  if (k > 0) launch_duplicate(da, s);
  if (timed) LMGS_CUDA(c, cudaEventRecord(c->ev[4], s));

  RadixSortBuffers kb{};
  kb.keys[0] = c->inst_keys[0];
  kb.keys[1] = c->inst_keys[1];
  kb.key_bytes = 8;
  kb.plan = &c->d_scal->tile_plan;
  kb.hist = c->d_scal->hist[2];
  kb.lookback = c->inst_lookback;
  kb.counters = c->d_scal->counters[2];
  kb.keys_result = &slots->inst_keys;
  const int tile_bits = bits_for(tiles);
  radix_sort(kb, k, 32, (tile_bits + 7) / 8, s);
  if (timed) LMGS_CUDA(c, cudaEventRecord(c->ev[5], s));

  launch_tile_ranges(slots, k, ranges, s);
  if (timed) LMGS_CUDA(c, cudaEventRecord(c->ev[6], s));

  BlendArgs ba{};
  ba.slots = slots;
  ba.work_counter = &c->d_scal->blend_counter;
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
  if (int r = launch_blend(ba, s)) return fail(c, r, "unsupported tile size");
  if (timed) {
    LMGS_CUDA(c, cudaEventRecord(c->ev[7], s));
    c->last_timed = true;
  }
  (void)npix;
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
  cudaError_t e = cudaMalloc(&c->d_scal, sizeof(Scalars));
  if (e == cudaSuccess) e = cudaMemset(c->d_scal, 0, sizeof(Scalars));
  if (e == cudaSuccess) e = cudaHostAlloc(&c->h_pinned, 4 * sizeof(uint64_t), cudaHostAllocDefault);
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
  c->ibuf.release();
  c->fbuf.release();
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
  a.slots = &c->d_scal->slots;
  a.prim_ids = c->last_prim_ids;
  a.k = c->stats.n_instances;
  a.keys_out = keys;
  a.prims_out = prim_ids;
  launch_export_instances(a, static_cast<cudaStream_t>(stream));
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
  PreprocessArgs pa{};
  pa.means = g->means;
  pa.quats = g->quats;
  pa.scales = g->scales;
  pa.logits = g->opacity_logits;
  pa.sh = g->sh;
  pa.n = n;
  pa.sh_coeffs = g->sh_coeffs;
  pa.eval_degree = s->sh_eval_degree < g->sh_degree ? s->sh_eval_degree : g->sh_degree;
  pa.cam = make_cam(cam, s->tile_size);
  pa.depth_keys32 = c->keys32[0];
  pa.depth_keys = c->keys64[0];
  pa.ids = c->ids[0];
  pa.ids_fb = c->ids[2];
  pa.rects = c->rects;
  pa.tile_counts = c->tile_counts;
  pa.recs = c->recs;
  pa.kept = kept;
  pa.n_kept = &c->d_scal->n_kept;
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
