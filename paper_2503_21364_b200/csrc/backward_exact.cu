// Backward of the blend, the parts that must round exactly like the
// reference (this file is compiled with -fmad=false): the per-view fp64 splat
// records (K1's projection code, geometry.cuh), the chain rule to SH
// coefficients and opacity logits with the reference's clamp gate, and the
// MSE loss step.  The per-pixel replay is in backward.cu.
//
// backward_render: gaussian_core.py:438-486; render_loss_and_grads: 600-629;
// sh_color_grad_to_coeffs: 145-166; eval_sh_colors: 129-142.
#include "geometry.cuh"
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

__constant__ double kShC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
__constant__ double kShC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

// unit view direction centre -> mean (eval_sh_colors 131-132)
__device__ __forceinline__ void view_dir(const CamArgs& cam, double m0, double m1, double m2,
                                         double* x, double* y, double* z) {
  const double dx = m0 - cam.center[0], dy = m1 - cam.center[1], dz = m2 - cam.center[2];
  double nrm = sqrt((dx * dx + dy * dy) + dz * dz);
  nrm = fmax(nrm, 1e-12);
  *x = dx / nrm;
  *y = dy / nrm;
  *z = dz / nrm;
}

// SH basis value of coefficient k (degree <= 3) along (x, y, z); degrees 0-1
// in the reference's sign convention (133-141)
__device__ __forceinline__ double sh_basis(int k, double x, double y, double z) {
  switch (k) {
    case 0: return kShC0;
    case 1: return -kShC1 * y;
    case 2: return kShC1 * z;
    case 3: return -kShC1 * x;
    case 4: return kShC2[0] * (x * y);
    case 5: return kShC2[1] * (y * z);
    case 6: return kShC2[2] * (2.0 * z * z - x * x - y * y);
    case 7: return kShC2[3] * (x * z);
    case 8: return kShC2[4] * (x * x - y * y);
    case 9: return kShC3[0] * y * (3.0 * x * x - y * y);
    case 10: return kShC3[1] * (x * y) * z;
    case 11: return kShC3[2] * y * (4.0 * z * z - x * x - y * y);
    case 12: return kShC3[3] * z * (2.0 * z * z - 3.0 * x * x - 3.0 * y * y);
    case 13: return kShC3[4] * x * (4.0 * z * z - x * x - y * y);
    case 14: return kShC3[5] * z * (x * x - y * y);
    default: return kShC3[6] * x * (x * x - 3.0 * y * y);
  }
}

// unclamped colour: degree <= 1 exactly as eval_sh_colors evaluates it
// (((C0 sh0 - (C1 y) sh1) + (C1 z) sh2) - (C1 x) sh3), higher degrees added
__device__ __forceinline__ void sh_raw(const float* sh, int deg, double x, double y, double z,
                                       double out[3]) {
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    double c = kShC0 * (double)sh[ch];
    if (deg >= 1)
      c = ((c - (kShC1 * y) * (double)sh[3 + ch]) + (kShC1 * z) * (double)sh[6 + ch]) -
          (kShC1 * x) * (double)sh[9 + ch];
    if (deg >= 2)
      for (int k = 4; k < (deg + 1) * (deg + 1); ++k)
        c = c + sh_basis(k, x, y, z) * (double)sh[3 * k + ch];
    out[ch] = c;
  }
}

// Per-Gaussian fp64 splat record of this view, computed once (K1's code):
// mean, conic, opacity, radius^2, clamped colour.
__global__ void k_bw_prep(BackwardArgs a) {
  const CamArgs& cam = a.cam;
  for (int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < a.n;
       id += (int64_t)gridDim.x * blockDim.x) {
    const double m0 = a.means[3 * id], m1 = a.means[3 * id + 1], m2 = a.means[3 * id + 2];
    const double x = mkl_dot3(m0, cam.r[0], m1, cam.r[1], m2, cam.r[2]) + cam.t[0];
    const double y = mkl_dot3(m0, cam.r[3], m1, cam.r[4], m2, cam.r[5]) + cam.t[1];
    const double z = mkl_dot3(m0, cam.r[6], m1, cam.r[7], m2, cam.r[8]) + cam.t[2];
    const float4 q = reinterpret_cast<const float4*>(a.quats)[id];
    double mx, my, ca, cb, cc, radius;
    splat_geometry(cam, x, y, z, q, a.scales[3 * id], a.scales[3 * id + 1], a.scales[3 * id + 2],
                   &mx, &my, &ca, &cb, &cc, &radius);
    const double det = ca * cc - cb * cb;  // _blend 308-310
    BwRec r;
    r.mx = mx;
    r.my = my;
    r.ca = cc / det;
    r.cb = -cb / det;
    r.cc = ca / det;
    r.op = 1.0 / (1.0 + exp(-(double)a.logits[id]));  // opacities (67-69)
    r.rop = 1.0 / r.op;
    r.r2 = radius * radius;
    double dx, dy, dz, raw[3];
    view_dir(cam, m0, m1, m2, &dx, &dy, &dz);
    sh_raw(a.sh + id * a.sh_coeffs * 3, a.eval_degree, dx, dy, dz, raw);
    r.col[0] = fmin(fmax(raw[0], 0.0), 1.0);
    r.col[1] = fmin(fmax(raw[1], 0.0), 1.0);
    r.col[2] = fmin(fmax(raw[2], 0.0), 1.0);
    a.recs[id] = r;
    if (!a.d_colors) continue;  // lmgs_record_collect: records only
    // this view's per-Gaussian outputs start at zero (k_backward adds into them)
    a.d_colors[3 * id] = a.d_colors[3 * id + 1] = a.d_colors[3 * id + 2] = 0.0;
    a.d_opacities[id] = 0.0;
    a.d_mean2d[2 * id] = a.d_mean2d[2 * id + 1] = 0.0;
    a.touched[id] = 0;
  }
}


// RenderRecord with collect (rasterize's TileRecord.sigma / t_before /
// t_final, gaussian_core.py:256-263, _blend 306-322 without the early break):
// one CTA per tile, one thread per pixel (chunks of 256 for tiles above 16x16),
// the tile's whole list in order, in fp64 from the view's splat records.
// sigma / t_before of tile t are (K_t, P_t) row-major at offsets[t].
__global__ void k_collect(CollectArgs a) {
  const int tile = blockIdx.x;
  const int ts = a.tile_size;
  const int tx0 = (tile % a.tiles_x) * ts, ty0 = (tile / a.tiles_x) * ts;
  const int tw = min(ts, a.width - tx0), th = min(ts, a.height - ty0);
  const int np = tw * th;
  const int2 range = a.ranges[tile];
  const int kt = range.y - range.x;
  const uint32_t* __restrict__ list = static_cast<const uint32_t*>(*a.keys_slot);
  const int64_t off = a.offsets[tile];
  for (int p = threadIdx.x; p < np; p += blockDim.x) {
    const int px = tx0 + p % tw, py = ty0 + p / tw;  // row-major within the tile
    const double pxd = (double)px + 0.5, pyd = (double)py + 0.5;
    double T = 1.0;
    for (int k = 0; k < kt; ++k) {
      const BwRec& r = a.recs[list[range.x + k]];
      const double dx = pxd - r.mx, dy = pyd - r.my;  // 311
      const double maha = (r.ca * (dx * dx) + ((2.0 * r.cb) * dx) * dy) + r.cc * (dy * dy);
      double sig = r.op * exp(-0.5 * maha);             // 313
      const bool inside = dx * dx + dy * dy <= r.r2;    // 314
      const bool active = T >= kTermEps;                // 315
      sig = inside && active ? (sig > kSigmaMax ? kSigmaMax : sig) : 0.0;
      const int64_t o = off + (int64_t)k * np + p;
      a.sigma[o] = sig;
      a.t_before[o] = T;
      T = T * (1.0 - sig);
    }
    a.t_final[(int64_t)py * a.width + px] = T;
  }
}

// render_loss_and_grads 617-622: d_sh += sh_color_grad_to_coeffs(d_colors),
// d_logit += d_opacity * alpha * (1 - alpha)
__global__ void k_backward_chain(BackwardArgs a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double dc0 = a.d_colors[3 * i], dc1 = a.d_colors[3 * i + 1],
                 dc2 = a.d_colors[3 * i + 2], dop = a.d_opacities[i];
    if (a.steps_seen && a.touched[i] > 0) {  // DensifyStats.accumulate (504-508)
      const double mx = a.d_mean2d[2 * i], my = a.d_mean2d[2 * i + 1];
      a.grad_norm_sum[i] += sqrt(mx * mx + my * my);
      a.steps_seen[i] += 1;
    }
    if (a.d_logits && dop != 0.0) {
      const double alpha = 1.0 / (1.0 + exp(-(double)a.logits[i]));
      a.d_logits[i] += (dop * alpha) * (1.0 - alpha);
    }
    if (!a.d_sh || (dc0 == 0.0 && dc1 == 0.0 && dc2 == 0.0)) continue;
    double x, y, z, raw[3];
    view_dir(a.cam, a.means[3 * i], a.means[3 * i + 1], a.means[3 * i + 2], &x, &y, &z);
    const int ncoef = a.sh_coeffs;
    sh_raw(a.sh + i * ncoef * 3, a.eval_degree, x, y, z, raw);
    const double dc[3] = {dc0, dc1, dc2};
    double gch[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) gch[ch] = (raw[ch] > 0.0 && raw[ch] < 1.0) ? dc[ch] : 0.0;
    const int nk = (a.eval_degree + 1) * (a.eval_degree + 1);
    for (int k = 0; k < nk && k < ncoef; ++k) {
      // grad[:,1] = -C1 * y * g etc. (157-161): ((+-C1) * coord) * g
      double bk;
      switch (k) {
        case 0: bk = kShC0; break;
        case 1: bk = -kShC1 * y; break;
        case 2: bk = kShC1 * z; break;
        case 3: bk = -kShC1 * x; break;
        default: bk = sh_basis(k, x, y, z);
      }
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) a.d_sh[(i * ncoef + k) * 3 + ch] += bk * gch[ch];
    }
  }
}

}  // namespace

int launch_collect(const BackwardArgs& prep, const CollectArgs& a, int tiles, cudaStream_t s) {
  if (prep.n > 0) {
    int64_t g = (prep.n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    k_bw_prep<<<(unsigned)g, 256, 0, s>>>(prep);
  }
  if (tiles > 0) k_collect<<<tiles, 256, 0, s>>>(a);
  return 2;
}

int launch_backward(const BackwardArgs& a, int tiles, cudaStream_t s) {
  int launched = 0;
  if (a.n > 0) {
    int64_t g = (a.n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    k_bw_prep<<<(unsigned)g, 256, 0, s>>>(a);
    ++launched;
  }
  launched += launch_backward_replay(a, tiles, s);
  if (a.n > 0 && (a.d_sh || a.d_logits || a.steps_seen)) {
    int64_t g = (a.n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    k_backward_chain<<<(unsigned)g, 256, 0, s>>>(a, a.n);
    ++launched;
  }
  return launched;
}

}  // namespace lmgs

namespace lmgs {
namespace {

template <typename G>
__global__ void k_mse_grad(const float* __restrict__ rgb, const G* __restrict__ gt, int64_t n,
                           float* __restrict__ grad, double* loss_sum) {
  double acc = 0.0;
  const double scale = 2.0 / (double)n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)rgb[i] - (double)gt[i];
    acc = acc + d * d;
    grad[i] = (float)(scale * d);
  }
  for (int o = 16; o; o >>= 1) acc = acc + __shfl_xor_sync(~0u, acc, o);
  __shared__ double part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = t + part[w];
    atomicAdd(loss_sum, t);
  }
}

}  // namespace
}  // namespace lmgs

extern "C" int lmgs_mse_grad(const float* rgb, const void* gt, int gt_is_f64, int64_t n_values,
                             float* image_grad, double* loss_sum, void* stream) {
  if (n_values < 0 || (n_values > 0 && (!rgb || !gt || !image_grad || !loss_sum)))
    return LMGS_ERR_INVALID;
  if (n_values == 0) return LMGS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int64_t g = (n_values + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  if (gt_is_f64)
    lmgs::k_mse_grad<double><<<(unsigned)g, 256, 0, s>>>(rgb, static_cast<const double*>(gt),
                                                         n_values, image_grad, loss_sum);
  else
    lmgs::k_mse_grad<float><<<(unsigned)g, 256, 0, s>>>(rgb, static_cast<const float*>(gt),
                                                        n_values, image_grad, loss_sum);
  return cudaGetLastError() == cudaSuccess ? LMGS_OK : LMGS_ERR_CUDA;
}

