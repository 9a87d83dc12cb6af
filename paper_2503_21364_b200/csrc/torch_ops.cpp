// Torch custom operators over the C ABI (include/lmgs.h): the drop-in boundary
// SURVEY.md §8(b) specifies for render_image (gaussian_core.py:582-597).
//
//   lmgs::render_fwd   every output buffer of one view
//   lmgs::render_image the reference's (image, touched[M]) pair
//
// Inputs are borrowed contiguous CUDA fp32 tensors; the camera is a packed
// host fp64 tensor (R 9, t 3, center 3, fx, fy, cx, cy, lim_x, lim_y) whose
// center and lim_* the caller computed in fp64 exactly as the reference does
// (data_io.py:65-67, gaussian_core.py:208-209).  Outputs come from the PyTorch
// caching allocator; the op runs on the current CUDA stream; scratch lives in
// one lmgs context per (device, stream), so the op is re-entrant across
// streams.  C-level errors surface as TORCH_CHECK -> RuntimeError.
#include <ATen/ATen.h>
#include <c10/cuda/CUDAGuard.h>
#include <c10/cuda/CUDAStream.h>
#include <torch/library.h>

#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include "../../include/lmgs.h"

namespace {

using at::Tensor;

constexpr int kCamValues = 21;

std::mutex g_mu;
std::map<std::pair<int, uintptr_t>, lmgs_context*> g_ctx;

lmgs_context* context_for(int device, cudaStream_t stream) {
  std::lock_guard<std::mutex> lock(g_mu);
  auto key = std::make_pair(device, reinterpret_cast<uintptr_t>(stream));
  auto it = g_ctx.find(key);
  if (it != g_ctx.end()) return it->second;
  lmgs_context* c = nullptr;
  const int st = lmgs_context_create(device, &c);
  TORCH_CHECK(st == LMGS_OK && c, "lmgs_context_create failed (status ", st, ")");
  g_ctx.emplace(key, c);
  return c;
}

void check(lmgs_context* c, int status, const char* what) {
  TORCH_CHECK(status == LMGS_OK, what, " failed (status ", status, "): ", lmgs_last_error(c));
}

void check_input(const Tensor& t, const char* name, int64_t rows, int64_t cols) {
  TORCH_CHECK(t.is_cuda(), name, " must be a CUDA tensor");
  TORCH_CHECK(t.scalar_type() == at::kFloat, name, " must be float32");
  TORCH_CHECK(t.is_contiguous(), name, " must be contiguous");
  TORCH_CHECK(t.size(0) == rows, name, " has ", t.size(0), " rows, expected ", rows);
  if (cols > 0) TORCH_CHECK(t.numel() == rows * cols, name, " must be (N, ", cols, ")");
}

lmgs_camera unpack_camera(const Tensor& cam, int64_t width, int64_t height) {
  TORCH_CHECK(cam.device().is_cpu() && cam.scalar_type() == at::kDouble &&
                  cam.numel() == kCamValues,
              "cam must be a host float64 tensor of 21 values (R 9, t 3, center 3, fx, fy, "
              "cx, cy, lim_x, lim_y)");
  const Tensor c = cam.contiguous();
  const double* v = c.data_ptr<double>();
  lmgs_camera out{};
  for (int i = 0; i < 9; ++i) out.r_wc[i] = v[i];
  for (int i = 0; i < 3; ++i) out.t_wc[i] = v[9 + i];
  for (int i = 0; i < 3; ++i) out.center[i] = v[12 + i];
  out.fx = v[15];
  out.fy = v[16];
  out.cx = v[17];
  out.cy = v[18];
  out.lim_x = v[19];
  out.lim_y = v[20];
  TORCH_CHECK(width >= 1 && height >= 1 && width < (1 << 30) && height < (1 << 30),
              "bad image size");
  out.width = (int32_t)width;
  out.height = (int32_t)height;
  return out;
}

using FwdResult = std::tuple<Tensor, Tensor, Tensor, Tensor, Tensor, Tensor, Tensor, Tensor>;

// render of one view; `kept` receives the near-cull mask when non-null
FwdResult render_impl(const Tensor& means_in, const Tensor& quats_in, const Tensor& scales_in,
                      const Tensor& logits_in, const Tensor& sh_in, int64_t sh_degree,
                      int64_t sh_eval_degree, const Tensor& cam, int64_t width, int64_t height,
                      int64_t tile_size, at::ArrayRef<double> background,
                      const c10::optional<Tensor>& subset, Tensor* kept_out) {
  TORCH_CHECK(background.size() == 3, "background must have 3 values");
  TORCH_CHECK(tile_size >= 1, "tile_size must be >= 1");
  const int64_t n_all = means_in.size(0);
  check_input(means_in, "means", n_all, 3);
  check_input(quats_in, "quats", n_all, 4);
  check_input(scales_in, "scales", n_all, 3);
  check_input(logits_in, "opacity_logits", n_all, 1);
  TORCH_CHECK(sh_in.dim() == 3 && sh_in.size(2) == 3, "sh must be (N, (deg+1)^2, 3)");
  check_input(sh_in, "sh", n_all, 0);
  TORCH_CHECK(sh_in.size(1) == (sh_degree + 1) * (sh_degree + 1),
              "SH coefficient count does not match degree");
  const c10::cuda::CUDAGuard guard(means_in.device());
  const int device = means_in.get_device();
  cudaStream_t stream = c10::cuda::getCurrentCUDAStream(device).stream();
  lmgs_context* ctx = context_for(device, stream);
  const auto dev_opts = means_in.options();

  // render_image's `subset` (gaussian_core.py:593-595): the selected rows in
  // ascending id order, original ids as the depth tie-break key
  Tensor means = means_in, quats = quats_in, scales = scales_in, logits = logits_in, sh = sh_in;
  Tensor prim_ids, inv;
  if (subset.has_value()) {
    Tensor ids = subset->to(means_in.device(), at::kLong).reshape({-1});
    if (ids.numel() > 0) {
      TORCH_CHECK(ids.min().item<int64_t>() >= 0 && ids.max().item<int64_t>() < n_all,
                  "subset ids out of range");
    }
    auto sorted = ids.sort(/*stable=*/true, /*dim=*/0, /*descending=*/false);
    prim_ids = std::get<0>(sorted).contiguous();
    inv = std::get<1>(sorted);
    means = means_in.index_select(0, prim_ids).contiguous();
    quats = quats_in.index_select(0, prim_ids).contiguous();
    scales = scales_in.index_select(0, prim_ids).contiguous();
    logits = logits_in.index_select(0, prim_ids).contiguous();
    sh = sh_in.index_select(0, prim_ids).contiguous();
  }
  const int64_t n = means.size(0);
  const int64_t tiles = ((width + tile_size - 1) / tile_size) * ((height + tile_size - 1) / tile_size);

  Tensor rgb = at::empty({height, width, 3}, dev_opts);
  Tensor alpha = at::empty({height, width}, dev_opts);
  Tensor depth = at::empty({height, width}, dev_opts);
  Tensor ranges = at::empty({tiles, 2}, dev_opts.dtype(at::kInt));
  Tensor touched = at::empty({n}, dev_opts.dtype(at::kInt));
  Tensor kept = at::empty({n}, dev_opts.dtype(at::kByte));
  Tensor nproc = at::empty({tiles}, dev_opts.dtype(at::kInt));

  lmgs_gaussians g{};
  g.means = means.data_ptr<float>();
  g.quats = quats.data_ptr<float>();
  g.scales = scales.data_ptr<float>();
  g.opacity_logits = logits.data_ptr<float>();
  g.sh = sh.data_ptr<float>();
  g.prim_ids = prim_ids.defined() ? prim_ids.data_ptr<int64_t>() : nullptr;
  g.count = n;
  g.sh_degree = (int32_t)sh_degree;
  g.sh_coeffs = (int32_t)sh.size(1);
  lmgs_camera c = unpack_camera(cam, width, height);
  lmgs_settings s{};
  s.tile_size = (int32_t)tile_size;
  s.sh_eval_degree = (int32_t)sh_eval_degree;
  for (int i = 0; i < 3; ++i) s.background[i] = background[i];
  lmgs_frame f{};
  f.rgb = rgb.data_ptr<float>();
  f.alpha = alpha.data_ptr<float>();
  f.depth = depth.data_ptr<float>();
  f.touched = touched.data_ptr<int32_t>();
  f.kept = kept.data_ptr<uint8_t>();
  f.tile_ranges = ranges.data_ptr<int32_t>();
  f.n_processed = nproc.data_ptr<int32_t>();
  check(ctx, lmgs_render(ctx, &g, &c, &s, &f, stream), "lmgs_render");
  lmgs_stats st{};
  check(ctx, lmgs_get_stats(ctx, &st), "lmgs_get_stats");
  const int64_t k = st.n_instances;
  Tensor keys = at::empty({k}, dev_opts.dtype(at::kLong));
  Tensor prims = at::empty({k}, dev_opts.dtype(at::kLong));
  check(ctx,
        lmgs_copy_instances(ctx, reinterpret_cast<uint64_t*>(keys.data_ptr<int64_t>()),
                            prims.data_ptr<int64_t>(), stream),
        "lmgs_copy_instances");
  Tensor vals = prims.to(at::kInt);
  if (inv.defined()) {  // per-row outputs back to the caller's subset order
    Tensor t2 = at::empty_like(touched);
    t2.index_put_({inv}, touched);
    touched = t2;
    Tensor k2 = at::empty_like(kept);
    k2.index_put_({inv}, kept);
    kept = k2;
  }
  if (kept_out) *kept_out = kept;
  return {rgb, alpha, depth, ranges, keys, vals, touched, nproc};
}

FwdResult render_fwd(const Tensor& means, const Tensor& quats, const Tensor& scales,
                     const Tensor& logits, const Tensor& sh, int64_t sh_degree,
                     int64_t sh_eval_degree, const Tensor& cam, int64_t width, int64_t height,
                     int64_t tile_size, at::ArrayRef<double> background,
                     const c10::optional<Tensor>& subset) {
  return render_impl(means, quats, scales, logits, sh, sh_degree, sh_eval_degree, cam, width,
                     height, tile_size, background, subset, nullptr);
}

std::tuple<Tensor, Tensor> render_image(const Tensor& means, const Tensor& quats,
                                        const Tensor& scales, const Tensor& logits,
                                        const Tensor& sh, int64_t sh_degree,
                                        int64_t sh_eval_degree, const Tensor& cam, int64_t width,
                                        int64_t height, int64_t tile_size,
                                        at::ArrayRef<double> background,
                                        const c10::optional<Tensor>& subset) {
  Tensor kept;
  auto r = render_impl(means, quats, scales, logits, sh, sh_degree, sh_eval_degree, cam, width,
                       height, tile_size, background, subset, &kept);
  // touched per kept splat (the reference's Splat2DBatch order), int64
  Tensor touched = std::get<6>(r).index({kept.to(at::kBool)}).to(at::kLong);
  return {std::get<0>(r), touched};
}

}  // namespace

TORCH_LIBRARY(lmgs, m) {
  m.def(
      "render_fwd(Tensor means, Tensor quats, Tensor scales, Tensor opacity_logits, Tensor sh, "
      "int sh_degree, int sh_eval_degree, Tensor cam, int width, int height, int tile_size, "
      "float[] background, Tensor? subset=None) -> (Tensor rgb, Tensor alpha, Tensor depth, "
      "Tensor tile_ranges, Tensor inst_keys, Tensor inst_vals, Tensor touched, "
      "Tensor n_processed)");
  m.def(
      "render_image(Tensor means, Tensor quats, Tensor scales, Tensor opacity_logits, "
      "Tensor sh, int sh_degree, int sh_eval_degree, Tensor cam, int width, int height, "
      "int tile_size, float[] background, Tensor? subset=None) -> (Tensor image, "
      "Tensor touched)");
}

TORCH_LIBRARY_IMPL(lmgs, CUDA, m) {
  m.impl("render_fwd", &render_fwd);
  m.impl("render_image", &render_image);
}
