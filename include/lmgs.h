/*
 * lmgs — B200-native (sm_100a) 3D Gaussian splatting forward rasterizer.
 * C ABI: plain pointers and sizes, no torch types.  All Gaussian / frame
 * pointers are DEVICE pointers unless the entry point says "host".
 *
 * Reference interfaces each entry point replaces (paths under
 * /root/reference/pkg/src/landmark/):
 *
 *   lmgs_render            gaussian_core.py:582-597  render_image(model, camera,
 *                          tile_size, background, with_record, subset)
 *                          = project_splats (187-230) + rasterize (340-403);
 *                          also the engine runtime switch
 *                          engine_api.py:291-299 Engine._render_gaussian
 *   lmgs_project           gaussian_core.py:187-230  project_splats (+ eval_sh_colors 129-142)
 *   lmgs_copy_instances    gaussian_core.py:256-263  TileRecord.order for every tile
 *                          (the per-tile lists the reference builds at 362-392)
 *   lmgs_render_batch      render_runtime.py:250-308 run_session's per-pose loop,
 *                          batched over camera views on one device
 *   lmgs_render_strips     (new) spatial-block render whose layers are stored
 *                          straight into the compositing GPUs' strip buffers;
 *                          lmgs_signal_flags / lmgs_wait_flags order it
 *   lmgs_composite_blocks  (new) front-to-back "over" of per-block premultiplied
 *                          images; replaces render_runtime.py:189-191 (BlockSession
 *                          concatenating resident cells into one model)
 *   lmgs_checkpoint_info_read / lmgs_checkpoint_load / lmgs_checkpoint_save
 *                          data_io.py:256-316 load_gaussian_checkpoint /
 *                          save_gaussian_checkpoint (LMGS format), into / from
 *                          device SoA arrays
 *   lmgs_backward          gaussian_core.py:438-486 backward_render (+ the chain
 *                          of render_loss_and_grads 600-629 to SH and logits)
 *   lmgs_record_collect    gaussian_core.py:256-274 RenderRecord / TileRecord
 *                          sigma, t_before, t_final (rasterize with_record)
 *   lmgs_encode_rgb8       render_runtime.py:397-401 encode_frame's pixels
 *                          (round(clip(rgb, 0, 1) * 255), half to even)
 *
 * Error behaviour: every entry point returns an lmgs_status; on failure
 * lmgs_last_error(ctx) holds a message.  Bad arguments map to the reference's
 * InvalidInputError / ShapeError in the Python wrapper (common.py:14-31).
 *
 * Threading: a context is bound to one device; calls on one context must be
 * serialised (use one context per concurrently-rendering stream).
 */
#ifndef LMGS_H_
#define LMGS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LMGS_ABI_VERSION 5

typedef enum lmgs_status {
  LMGS_OK = 0,
  LMGS_ERR_INVALID = 1,     /* bad argument (shape, size, null pointer)   */
  LMGS_ERR_CUDA = 2,        /* CUDA runtime error                         */
  LMGS_ERR_OOM = 3,         /* device allocation failed                   */
  LMGS_ERR_UNSUPPORTED = 4, /* e.g. more than 2^24 tiles in one view      */
  LMGS_ERR_FORMAT = 5,      /* malformed checkpoint (reference FormatError) */
  LMGS_ERR_IO = 6           /* file open / read / write failed             */
} lmgs_status;

typedef struct lmgs_context lmgs_context;

/* One pinhole view.  r_wc rows = (right, down, forward); center = -r_wc^T t_wc
 * and lim_x/lim_y = 1.3*max(cx, W-cx)/fx (gaussian_core.py:208-209) are
 * computed on the host in fp64 exactly as the reference does, and reach the
 * kernels as launch arguments (constant bank). */
typedef struct lmgs_camera {
  double r_wc[9];
  double t_wc[3];
  double center[3];
  double fx, fy, cx, cy;
  double lim_x, lim_y;
  int32_t width, height;
} lmgs_camera;

/* Structure-of-arrays Gaussian set, fp32, contiguous (GaussianModel,
 * gaussian_core.py:34-61).  sh: [count, sh_coeffs, 3]. */
typedef struct lmgs_gaussians {
  const float* means;           /* [count,3]                       */
  const float* quats;           /* [count,4] (w,x,y,z), unit       */
  const float* scales;          /* [count,3] > 0, linear           */
  const float* opacity_logits;  /* [count]                         */
  const float* sh;              /* [count, sh_coeffs, 3]           */
  const int64_t* prim_ids;      /* [count] original ids (render_image's `subset`,
                                   593-595; depth ties are broken by them) or
                                   NULL = row index                              */
  int64_t count;
  int32_t sh_degree;            /* model degree, sh_coeffs == (sh_degree+1)^2 */
  int32_t sh_coeffs;
  /* Paged sets (a device pool of 128-row pages, offload.py): row r takes
   * part only if (r & 127) < page_mask[r >> 7] (the live leading rows of its
   * page, 0..128); other rows are treated as culled.  NULL = every row.
   * page_shift must be 7. */
  const uint8_t* page_mask;
  int32_t page_shift;
  int32_t reserved;
} lmgs_gaussians;

typedef struct lmgs_settings {
  int32_t tile_size;       /* >= 1 (reference default 16; TileConfig 245-253) */
  int32_t sh_eval_degree;  /* 1 = reference eval_sh_colors; 3 = full degree 3 */
  double background[3];   /* fp64 like the reference (common.py DTYPE)     */
  uint32_t flags;          /* LMGS_FLAG_*                                    */
  int64_t max_instances;   /* LMGS_FLAG_NO_HOST_SYNC: tile-instance capacity
                              (0 = the context's current capacity)          */
} lmgs_settings;

#define LMGS_FLAG_STAGE_TIMES 1u  /* record per-stage CUDA events (lmgs_get_stats) */
/* Capacity-bounded render with no host wait: the instance count K is never
 * read back; every stage sizes its grid for settings.max_instances and reads
 * the true counts on the device, so a whole view batch can be captured in a
 * CUDA graph (after one ordinary render of the same configuration has sized
 * the context's arenas).  A view whose K exceeds the capacity is rendered
 * incompletely (memory-safe); lmgs_get_stats then reports it (overflow, the
 * largest K seen) and the caller re-renders with a larger capacity. */
#define LMGS_FLAG_NO_HOST_SYNC 8u
/* Queue pixels for the exact-touched replay within a relative band of 1e-2
 * around TERM_EPS instead of 1e-4 (100x more pixels replayed): the check that
 * the default band misses no fp32/fp64 disagreement (tests/test_gpu_parity). */
#define LMGS_FLAG_WIDE_FIX_BAND 16u
/* Build the tile lists with the fused emission + tile sort (K4c/K4r/K4p and a
 * first onesweep pass that generates its keys; tile ids < 2^16) instead of
 * the separate K4 emission + two-pass K5 tile sort: identical lists, fewer
 * DRAM bytes, measured slower at c3 (tests/test_gpu_fused.py). */
#define LMGS_FLAG_FUSED_TILE_SORT 32u
/* Other streams render concurrently (a view batch over several contexts):
 * the latency-bound radix-sort passes run as persistent grids of one CTA per
 * SM instead of one CTA per tile, leaving the other slots to the other
 * streams' kernels (BatchRenderer sets it; a lone view is faster without). */
#define LMGS_FLAG_CONCURRENT 64u
#define LMGS_FLAG_NO_TOUCHED_FIX 2u /* skip K7b: touched may then differ from the
                                       reference where fp32 and fp64 transmittance
                                       straddle TERM_EPS (a few per million)       */

/* Per-view outputs (device).  rgb is required; the rest may be NULL. */
typedef struct lmgs_frame {
  float* rgb;             /* [H,W,3] image incl. T_final * background          */
  float* alpha;           /* [H,W]   1 - T_final                               */
  float* depth;           /* [H,W]   sum_i w_i z_i (not in the reference)      */
  float* transmittance;   /* [H,W]   T_final (for block compositing)           */
  int32_t* touched;       /* [count] pixels with w > 0 per Gaussian (0 if culled) */
  uint8_t* kept;          /* [count] 1 if z > 0.01 (near cull, 196-198)        */
  int32_t* tile_ranges;   /* [T,2]   [start,end) of each tile's instance list  */
  int32_t* n_processed;   /* [T]     blend break index per tile (324-325)      */
} lmgs_frame;

#define LMGS_MAX_STAGES 8

typedef struct lmgs_stats {
  int64_t n_gaussians;
  int64_t n_kept;            /* M */
  int64_t n_instances;       /* K */
  int64_t n_visible;         /* splats touching >= 1 tile */
  int32_t n_tiles;           /* T */
  int32_t tiles_x, tiles_y;
  int32_t n_stages;
  int32_t n_launches;        /* liblmgs kernels launched by the last render */
  float stage_ms[LMGS_MAX_STAGES];  /* valid with LMGS_FLAG_STAGE_TIMES */
  const char* stage_names[LMGS_MAX_STAGES];
  int64_t capacity;          /* instance capacity of the last render           */
  int64_t max_instances_seen;/* largest K since the previous lmgs_get_stats    */
  int32_t overflow;          /* a view since then had K > its capacity         */
  int32_t reserved;
} lmgs_stats;

int lmgs_abi_version(void);
int lmgs_context_create(int device, lmgs_context** out);
void lmgs_context_destroy(lmgs_context* ctx);
const char* lmgs_last_error(const lmgs_context* ctx);

/* Render one view; stream is a cudaStream_t (NULL = legacy default stream).
 * Returns after the instance count is known (one device->host read of K);
 * the image kernels are enqueued on `stream` and not waited for. */
int lmgs_render(lmgs_context* ctx, const lmgs_gaussians* g, const lmgs_camera* cam,
                const lmgs_settings* s, const lmgs_frame* out, void* stream);

/* Render n_views views of the same Gaussians; out[v] receives view v. */
int lmgs_render_batch(lmgs_context* ctx, const lmgs_gaussians* g, const lmgs_camera* cams,
                      int32_t n_views, const lmgs_settings* s, const lmgs_frame* out,
                      void* stream);

/* Render a group of n_views (1..LMGS_MAX_GROUP) views of the same Gaussians,
 * view v on its own context ctxs[v] (distinct, one device) and stream
 * streams[v].  The preprocess of the whole group is ONE launch on streams[0]
 * that stages each block of Gaussians once and projects it for every view
 * (inputs read from HBM once per group, not once per view); each view's
 * depth sort, emission, tile sort and blend then run on its own stream.
 * Outputs are identical to n_views lmgs_render calls.  Same reference
 * interface as lmgs_render: the per-pose loop of run_session
 * (render_runtime.py:250-308) over render_image (gaussian_core.py:582-597). */
#define LMGS_MAX_GROUP 8
int lmgs_render_group(lmgs_context* const* ctxs, int32_t n_views, const lmgs_gaussians* g,
                      const lmgs_camera* cams, const lmgs_settings* s, const lmgs_frame* out,
                      void* const* streams);

/* Statistics of the last lmgs_render on this context (stage times require the
 * stream to have completed: call after synchronising).  After a
 * LMGS_FLAG_NO_HOST_SYNC render this synchronises the device first. */
int lmgs_get_stats(lmgs_context* ctx, lmgs_stats* out);

/* Copy the last render's sorted tile instances: keys[K] = tile << 32 | row
 * (the Gaussian's row in the input arrays), prim_ids[K] = original Gaussian id
 * (TileRecord.order mapped through splats.prim_id).  Lists are sorted by tile,
 * then by (fp64 depth, prim id).  Either pointer may be NULL.  Device buffers,
 * K entries.  The render's lmgs_gaussians.prim_ids array (when given) must
 * still be valid; everything else lives in the context. */
int lmgs_copy_instances(lmgs_context* ctx, uint64_t* keys, int64_t* prim_ids, void* stream);

/* Pixels the last render queued for the exact-touched replay (K7b):
 * synchronises with the render's stream. */
int lmgs_touched_fix_count(lmgs_context* ctx, uint32_t* count);

/* Backward of the blend for the view last rendered on ctx (same Gaussians,
 * camera and settings): backward_render (gaussian_core.py:
 * 438-486) in fp64 with the reference's semantics — d_colors [count,3],
 * d_opacities [count], d_mean2d [count,2], touched [count] (zeroed, rows of
 * non-rendered Gaussians stay 0) — and, when non-NULL, the chain rule of
 * render_loss_and_grads (600-629): d_sh [count,sh_coeffs,3] and d_logits
 * [count] are ACCUMULATED (+=) so several views can be summed, and so are
 * the DensifyStats increments (488-511) when grad_norm_sum / steps_seen are
 * non-NULL: += |d_mean2d| and += 1 for every Gaussian with touched > 0.
 * image_grad is the loss gradient w.r.t. the [H,W,3] image (fp32, device). */
int lmgs_backward(lmgs_context* ctx, const lmgs_gaussians* g, const lmgs_camera* cam,
                  const lmgs_settings* s, const float* image_grad, double* d_colors,
                  double* d_opacities, double* d_mean2d, int32_t* touched, double* d_sh,
                  double* d_logits, double* grad_norm_sum, int64_t* steps_seen,
                  void* stream);

/* RenderRecord with collect for the view last rendered on ctx (same
 * Gaussians, camera and settings): rasterize's per-tile TileRecord.sigma and
 * t_before (gaussian_core.py:256-263, _blend 306-322 over each tile's whole
 * list, no early break) in fp64 — tile t's (K_t, P_t) block, row-major over
 * its instances and its pixels (row-major within the tile), starts at
 * tile_offsets[t] (device int64, T entries) — t_final [H,W] fp64, and,
 * when non-NULL, each Gaussian's fp64 view colour [count,3] and opacity
 * [count] as the reference's RenderRecord.colors / opacities hold them. */
int lmgs_record_collect(lmgs_context* ctx, const lmgs_gaussians* g, const lmgs_camera* cam,
                        const lmgs_settings* s, const int64_t* tile_offsets, double* sigma,
                        double* t_before, double* t_final, double* colors, double* opacities,
                        void* stream);

/* The mean-squared-error step of render_loss_and_grads (gaussian_core.py:
 * 615-617) for one view: diff = rgb - gt over n_values = H*W*3 values,
 * loss_sum[0] += sum(diff^2) (fp64, device), image_grad = 2 diff / n_values
 * (fp32, the lmgs_backward input).  gt is fp64 when gt_is_f64, else fp32. */
int lmgs_mse_grad(const float* rgb, const void* gt, int gt_is_f64, int64_t n_values,
                  float* image_grad, double* loss_sum, void* stream);

/* Stage K1 alone (project_splats): per input Gaussian, fp64 geometry.
 * mean2d [count,2], cov2d [count,3] = (c00,c01,c11) incl. the 0.3 floor,
 * depth [count], radius [count], colors [count,3] (fp32), opacity [count]
 * (fp32), kept [count]; values of culled Gaussians are unspecified. */
int lmgs_project(lmgs_context* ctx, const lmgs_gaussians* g, const lmgs_camera* cam,
                 const lmgs_settings* s, double* mean2d, double* cov2d, double* depth,
                 double* radius, float* colors, float* opacity, uint8_t* kept, void* stream);

/* Spatial blocks over peer memory (the exchange fused into the blend).
 * lmgs_render_strips renders like lmgs_render with background 0 semantics
 * of a block layer, but writes every finished pixel of row y straight into
 * strip y / strip_rows of the targets — typically the receive buffers of
 * the GPUs that composite those strips, mapped into this process (NVLink
 * peer pointers from symmetric memory), so the exchange overlaps the blend
 * tile by tile and no separate collective moves the layers. */
#define LMGS_MAX_STRIPS 8
typedef struct lmgs_strip_targets {
  int32_t n_strips;               /* 1..LMGS_MAX_STRIPS                              */
  int32_t strip_rows;             /* rows per strip (the last may be shorter)         */
  float* rgb[LMGS_MAX_STRIPS];    /* [strip_rows, W, 3]: C + T_final * background      */
  float* trans[LMGS_MAX_STRIPS];  /* [strip_rows, W]: T_final (nullable)              */
  float* depth[LMGS_MAX_STRIPS];  /* [strip_rows, W]: sum w z (nullable)              */
} lmgs_strip_targets;
int lmgs_render_strips(lmgs_context* ctx, const lmgs_gaussians* g, const lmgs_camera* cam,
                       const lmgs_settings* s, const lmgs_strip_targets* targets,
                       int32_t* touched, void* stream);

/* Release-store `value` to n device flags (system scope, after a system
 * fence): tells the owners of the strips written by lmgs_render_strips that
 * this block's layers are complete.  flags is a host array of (peer) device
 * pointers, n <= 64. */
int lmgs_signal_flags(uint32_t* const* flags, int32_t n, uint32_t value, void* stream);

/* Stream-ordered wait until every flags[i] >= value (acquire, system scope),
 * i < n; the next work on `stream` (e.g. lmgs_composite_blocks over the
 * received layers) sees the peers' stores. */
int lmgs_wait_flags(const uint32_t* flags, int32_t n, uint32_t value, void* stream);

/* Front-to-back composite of n_blocks per-block renders (background 0):
 * rgb_b premultiplied [H*W*3], trans_b [H*W] (T_final), depth_b [H*W]
 * (nullable), stacked block-major: rgb[b*H*W*3 ...].  order[n_blocks] lists
 * block indices front to back.  out_rgb = sum_b (prod_{b'<b} T_b') C_b +
 * (prod T) bg; out_alpha = 1 - prod T; out_depth likewise (nullable). */
int lmgs_composite_blocks(const float* rgb, const float* trans, const float* depth,
                          int32_t n_blocks, const int32_t* order_host, int64_t n_pixels,
                          const float* background_host, float* out_rgb, float* out_alpha,
                          float* out_depth, void* stream);

/* LMGS checkpoint header (data_io.py:3-9): "<4sIIQ" then count rows of
 * row_floats f32, a grid flag byte and the optional grid block. */
typedef struct lmgs_checkpoint_info {
  uint32_t version;
  uint32_t sh_degree;
  int64_t count;
  int32_t row_floats;          /* 11 + 3 * (sh_degree + 1)^2               */
  int32_t has_grid;
  int64_t data_offset;         /* byte offset of the first row             */
  float grid_bbox[6];          /* (min xyz, max xyz) when has_grid         */
  uint32_t grid_nx, grid_ny;
  int64_t grid_table_offset;   /* byte offset of the nx*ny u32 table       */
} lmgs_checkpoint_info;

/* Parse and validate a checkpoint header (host only, no device work).  err
 * (nullable, err_len bytes) receives the message on failure.  A count the
 * file cannot hold fails with LMGS_ERR_FORMAT ("truncated"), before any size
 * arithmetic.  sh_degree > 3 returns LMGS_ERR_UNSUPPORTED: the reference loads
 * any degree, but the rasterizer evaluates SH up to degree 3. */
int lmgs_checkpoint_info_read(const char* path, lmgs_checkpoint_info* info, char* err,
                              int err_len);

/* Stream the rows into device SoA arrays sized from the header (means
 * [count,3], quats [count,4], scales [count,3], logits [count], sh
 * [count,(d+1)^2,3]); grid_table_host (nullable) receives the nx*ny submodel
 * ids.  Returns after the data is on the device. */
int lmgs_checkpoint_load(const char* path, float* means, float* quats, float* scales,
                         float* logits, float* sh, uint32_t* grid_table_host, void* stream,
                         char* err, int err_len);

/* Write device SoA Gaussians as an LMGS file (temp file, then rename);
 * grid (nullable or has_grid = 0: no grid block) with its host table. */
int lmgs_checkpoint_save(const char* path, const lmgs_gaussians* g,
                         const lmgs_checkpoint_info* grid, const uint32_t* grid_table_host,
                         void* stream, char* err, int err_len);

/* out[i] = round_half_even(clip(rgb[i], 0, 1) * 255) for n_values floats
 * (device pointers; the wire frame's pixel bytes). */
int lmgs_encode_rgb8(const float* rgb, int64_t n_values, uint8_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LMGS_H_ */
