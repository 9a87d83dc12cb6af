// Backward of the blend: backward_render
// (gaussian_core.py:438-486) and the chain rule of render_loss_and_grads
// (600-629) to SH coefficients (sh_color_grad_to_coeffs, 145-166) and opacity
// logits.  Reference semantics in fp64, op for op (this file is compiled with
// -fmad=false): each tile's splats are re-projected with K1's own fp64 code
// (geometry.cuh) so conic, opacity, mean and radius are bit-identical to the
// reference's, and colours are re-evaluated in fp64 (eval_sh_colors, 129-142).
//
// Per tile (one CTA, pixel state in shared memory), over the tile list of the
// preceding render on the same context:
//   pass A  the forward blend in fp64 -> every pixel's total colour C_tot
//           (including T_final * background);
//   pass B  the forward blend again; at each applied step the reference's
//           reverse-mode quantities: w = T_before sigma, suffix = C_tot - sum
//           of w c up to and including this step (the reference accumulates
//           the same suffix back to front), d_sigma = g . (c T_before -
//           suffix / max(1 - sigma, 1e-6)); per-splat sums of g w, d_sigma
//           sigma / alpha, d_sigma sigma (conic @ (pix - mean)) and w > 0 are
//           gathered in shared fp64 and flushed with one atomic per splat.
// A pixel stops when its T < TERM_EPS (later steps have sigma = 0: no
// contribution), a tile when all its pixels have.
#include "device_util.cuh"
#include "geometry.cuh"
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

constexpr int kBwThreads = 256;
constexpr int kBwBatch = 64;
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

__global__ void __launch_bounds__(kBwThreads) k_backward(BackwardArgs a) {
  extern __shared__ __align__(16) double s_px[];  // [7][np]: T, C0-2, Ctot0-2
  __shared__ double s_mx[kBwBatch], s_my[kBwBatch], s_ca[kBwBatch], s_cb[kBwBatch],
      s_cc[kBwBatch], s_op[kBwBatch], s_r2[kBwBatch], s_z[kBwBatch], s_col[kBwBatch][3];
  __shared__ double s_acc[kBwBatch][6];  // d_colors 3, d_opacity, d_mean 2
  __shared__ int s_touch[kBwBatch];
  __shared__ uint32_t s_id[kBwBatch];
  const int tid = threadIdx.x;
  const int ts = a.tile_size;
  const int tile = blockIdx.x;
  const int x0 = (tile % a.tiles_x) * ts, y0 = (tile / a.tiles_x) * ts;
  const int tw = min(ts, a.width - x0), th = min(ts, a.height - y0);
  const int np = tw * th;
  double* sT = s_px;
  double* sC = sT + np;           // [3][np] running colour
  double* sTot = sC + 3 * np;     // [3][np] total colour
  const int2 range = a.ranges[tile];
  if (range.y <= range.x) return;
  const uint64_t* __restrict__ list = static_cast<const uint64_t*>(*a.keys_slot);
  const CamArgs& cam = a.cam;
  const int ncoef = a.sh_coeffs;

  for (int pass = 0; pass < 2; ++pass) {
    for (int p = tid; p < np; p += kBwThreads) {
      sT[p] = 1.0;
      sC[p] = sC[np + p] = sC[2 * np + p] = 0.0;
    }
    __syncthreads();
    for (int b0 = range.x; b0 < range.y; b0 += kBwBatch) {
      const int nb = min(kBwBatch, range.y - b0);
      for (int j = tid; j < nb; j += kBwThreads) {  // re-project in fp64 (K1's code)
        const uint32_t id = (uint32_t)list[b0 + j];
        const double m0 = a.means[3 * (size_t)id], m1 = a.means[3 * (size_t)id + 1],
                     m2 = a.means[3 * (size_t)id + 2];
        const double x = mkl_dot3(m0, cam.r[0], m1, cam.r[1], m2, cam.r[2]) + cam.t[0];
        const double y = mkl_dot3(m0, cam.r[3], m1, cam.r[4], m2, cam.r[5]) + cam.t[1];
        const double z = mkl_dot3(m0, cam.r[6], m1, cam.r[7], m2, cam.r[8]) + cam.t[2];
        const float4 q = reinterpret_cast<const float4*>(a.quats)[id];
        double mx, my, ca, cb, cc, radius;
        splat_geometry(cam, x, y, z, q, a.scales[3 * (size_t)id], a.scales[3 * (size_t)id + 1],
                       a.scales[3 * (size_t)id + 2], &mx, &my, &ca, &cb, &cc, &radius);
        const double det = ca * cc - cb * cb;  // _blend 308-310
        s_ca[j] = cc / det;
        s_cb[j] = -cb / det;
        s_cc[j] = ca / det;
        s_op[j] = 1.0 / (1.0 + exp(-(double)a.logits[id]));  // opacities (67-69)
        s_mx[j] = mx;
        s_my[j] = my;
        s_r2[j] = radius * radius;
        s_z[j] = z;
        double dx, dy, dz, raw[3];
        view_dir(cam, m0, m1, m2, &dx, &dy, &dz);
        sh_raw(a.sh + (size_t)id * ncoef * 3, a.eval_degree, dx, dy, dz, raw);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) s_col[j][ch] = fmin(fmax(raw[ch], 0.0), 1.0);
        s_id[j] = id;
#pragma unroll
        for (int c = 0; c < 6; ++c) s_acc[j][c] = 0.0;
        s_touch[j] = 0;
      }
      __syncthreads();
      bool active = false;
      for (int p = tid; p < np; p += kBwThreads) {
        double T = sT[p];
        if (!(T >= kTermEps)) continue;
        double c0 = sC[p], c1 = sC[np + p], c2 = sC[2 * np + p];
        const int lx = p % tw, ly = p / tw;
        const double pxd = (double)(x0 + lx) + 0.5, pyd = (double)(y0 + ly) + 0.5;
        double g0 = 0.0, g1 = 0.0, g2 = 0.0, t0 = 0.0, t1 = 0.0, t2 = 0.0;
        if (pass == 1) {
          const int64_t o = (int64_t)(y0 + ly) * a.width + (x0 + lx);
          g0 = (double)a.image_grad[3 * o + 0];
          g1 = (double)a.image_grad[3 * o + 1];
          g2 = (double)a.image_grad[3 * o + 2];
          t0 = sTot[p];
          t1 = sTot[np + p];
          t2 = sTot[2 * np + p];
        }
        for (int k = 0; k < nb; ++k) {
          const double dx = pxd - s_mx[k], dy = pyd - s_my[k];  // 311
          const double maha =
              (s_ca[k] * (dx * dx) + ((2.0 * s_cb[k]) * dx) * dy) + s_cc[k] * (dy * dy);
          double sig = s_op[k] * exp(-0.5 * maha);  // 313
          const bool inside = (dx * dx + dy * dy) <= s_r2[k];  // 314 (active here)
          sig = inside ? (sig > kSigmaMax ? kSigmaMax : sig) : 0.0;
          const double w = T * sig;
          c0 = c0 + w * s_col[k][0];
          c1 = c1 + w * s_col[k][1];
          c2 = c2 + w * s_col[k][2];
          if (pass == 1 && sig > 0.0) {  // backward_render 461-484
            const double s0 = t0 - c0, s1 = t1 - c1, s2 = t2 - c2;  // suffix
            double denom = 1.0 - sig;
            denom = denom < 1e-6 ? 1e-6 : denom;
            const double dsig = (g0 * (s_col[k][0] * T - s0 / denom) +
                                 g1 * (s_col[k][1] * T - s1 / denom)) +
                                g2 * (s_col[k][2] * T - s2 / denom);
            atomicAdd(&s_acc[k][0], g0 * w);
            atomicAdd(&s_acc[k][1], g1 * w);
            atomicAdd(&s_acc[k][2], g2 * w);
            atomicAdd(&s_acc[k][3], dsig * sig / s_op[k]);
            atomicAdd(&s_acc[k][4], dsig * (sig * (s_ca[k] * dx + s_cb[k] * dy)));
            atomicAdd(&s_acc[k][5], dsig * (sig * (s_cb[k] * dx + s_cc[k] * dy)));
            if (w > 0.0) atomicAdd(&s_touch[k], 1);
          }
          T = T * (1.0 - sig);
          if (!(T >= kTermEps)) break;
        }
        sT[p] = T;
        sC[p] = c0;
        sC[np + p] = c1;
        sC[2 * np + p] = c2;
        active |= T >= kTermEps;
      }
      const int live = __syncthreads_or(active);
      if (pass == 1)
        for (int j = tid; j < nb; j += kBwThreads) {
          const uint32_t id = s_id[j];
          if (s_touch[j] || s_acc[j][3] != 0.0 || s_acc[j][0] != 0.0 || s_acc[j][1] != 0.0 ||
              s_acc[j][2] != 0.0) {
            atomicAdd(a.d_colors + 3 * (size_t)id + 0, s_acc[j][0]);
            atomicAdd(a.d_colors + 3 * (size_t)id + 1, s_acc[j][1]);
            atomicAdd(a.d_colors + 3 * (size_t)id + 2, s_acc[j][2]);
            atomicAdd(a.d_opacities + id, s_acc[j][3]);
            atomicAdd(a.d_mean2d + 2 * (size_t)id + 0, s_acc[j][4]);
            atomicAdd(a.d_mean2d + 2 * (size_t)id + 1, s_acc[j][5]);
            if (s_touch[j]) atomicAdd(a.touched + id, s_touch[j]);
          }
        }
      __syncthreads();
      if (!live) break;
    }
    if (pass == 0) {  // C_tot = sum w c + T_final * background (326)
      for (int p = tid; p < np; p += kBwThreads) {
        sTot[p] = sC[p] + sT[p] * a.bg[0];
        sTot[np + p] = sC[np + p] + sT[p] * a.bg[1];
        sTot[2 * np + p] = sC[2 * np + p] + sT[p] * a.bg[2];
      }
    }
    __syncthreads();
  }
}

// render_loss_and_grads 617-622: d_sh += sh_color_grad_to_coeffs(d_colors),
// d_logit += d_opacity * alpha * (1 - alpha)
__global__ void k_backward_chain(BackwardArgs a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double dc0 = a.d_colors[3 * i], dc1 = a.d_colors[3 * i + 1],
                 dc2 = a.d_colors[3 * i + 2], dop = a.d_opacities[i];
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

int launch_backward(const BackwardArgs& a, int tiles, cudaStream_t s) {
  if (a.tile_size > 32) return LMGS_ERR_UNSUPPORTED;
  int launched = 0;
  if (tiles > 0) {
    const size_t smem = sizeof(double) * 7 * (size_t)a.tile_size * a.tile_size;
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(k_backward, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(sizeof(double) * 7 * 32 * 32));
      set = true;
    }
    k_backward<<<tiles, kBwThreads, smem, s>>>(a);
    ++launched;
  }
  if (a.n > 0 && (a.d_sh || a.d_logits)) {
    int64_t g = (a.n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    k_backward_chain<<<(unsigned)g, 256, 0, s>>>(a, a.n);
    ++launched;
  }
  return launched;
}

}  // namespace lmgs
