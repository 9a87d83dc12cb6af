// Background fill and K8 block composite (the front-to-back "over" of
// per-block renders used by spatial-block rendering).
#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

__global__ void k_fill_bg(float* rgb, float* alpha, float* depth, float* trans, int64_t n,
                          float b0, float b1, float b2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  rgb[3 * i] = b0;
  rgb[3 * i + 1] = b1;
  rgb[3 * i + 2] = b2;
  if (alpha) alpha[i] = 0.0f;
  if (depth) depth[i] = 0.0f;
  if (trans) trans[i] = 1.0f;
}

struct BlockOrder {
  int32_t v[kMaxCompositeBlocks];
};

// Front-to-back "over" of per-block premultiplied renders (background 0):
// C = sum_b (prod_{b'<b} T_b') C_b + (prod_b T_b) bg.  Blocks are read four
// at a time (independent loads in flight) before the dependent "over" chain.
constexpr int kCompUnroll = 4;

__global__ void k_composite(const float* __restrict__ rgb, const float* __restrict__ trans,
                            const float* __restrict__ depth, int n_blocks, const BlockOrder order,
                            int64_t n_pix, float b0, float b1, float b2, float* out_rgb,
                            float* out_alpha, float* out_depth) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pix) return;
  float T = 1.0f, r = 0.f, g = 0.f, b = 0.f, d = 0.f;
  for (int k0 = 0; k0 < n_blocks; k0 += kCompUnroll) {
    float cr[kCompUnroll], cg[kCompUnroll], cb[kCompUnroll], ct[kCompUnroll], cd[kCompUnroll];
#pragma unroll
    for (int u = 0; u < kCompUnroll; ++u) {
      const bool on = k0 + u < n_blocks;
      const int64_t o = on ? (int64_t)order.v[k0 + u] * n_pix + i : i;
      cr[u] = on ? __ldg(rgb + 3 * o + 0) : 0.f;
      cg[u] = on ? __ldg(rgb + 3 * o + 1) : 0.f;
      cb[u] = on ? __ldg(rgb + 3 * o + 2) : 0.f;
      ct[u] = on ? __ldg(trans + o) : 1.f;
      cd[u] = (on && depth) ? __ldg(depth + o) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kCompUnroll; ++u) {
      r = fmaf(T, cr[u], r);
      g = fmaf(T, cg[u], g);
      b = fmaf(T, cb[u], b);
      d = fmaf(T, cd[u], d);
      T *= ct[u];
    }
  }
  out_rgb[3 * i + 0] = fmaf(T, b0, r);
  out_rgb[3 * i + 1] = fmaf(T, b1, g);
  out_rgb[3 * i + 2] = fmaf(T, b2, b);
  if (out_alpha) out_alpha[i] = 1.0f - T;
  if (out_depth) out_depth[i] = d;
}

}  // namespace

void launch_fill_background(float* rgb, float* alpha, float* depth, float* trans, int64_t n_pix,
                            const float bg[3], cudaStream_t s) {
  if (n_pix <= 0) return;
  k_fill_bg<<<(unsigned)((n_pix + 255) / 256), 256, 0, s>>>(rgb, alpha, depth, trans, n_pix,
                                                            bg[0], bg[1], bg[2]);
}

void launch_composite(const float* rgb, const float* trans, const float* depth, int n_blocks,
                      const int32_t* order, int64_t n_pix, const float bg[3], float* out_rgb,
                      float* out_alpha, float* out_depth, cudaStream_t s) {
  if (n_pix <= 0) return;
  BlockOrder ord;
  for (int k = 0; k < n_blocks && k < kMaxCompositeBlocks; ++k) ord.v[k] = order[k];
  k_composite<<<(unsigned)((n_pix + 255) / 256), 256, 0, s>>>(
      rgb, trans, depth, n_blocks, ord, n_pix, bg[0], bg[1], bg[2], out_rgb, out_alpha,
      out_depth);
}

}  // namespace lmgs

// ---------------------------------------------------------------------------
// Peer flags for the strip exchange (lmgs_render_strips): the producer
// fences its peer stores at system scope and release-stores the epoch into
// each owner's flag; the owner's stream spins on acquire loads before the
// composite reads the received layers.

namespace lmgs {
namespace {

constexpr int kMaxFlags = 64;
struct FlagPtrs {
  uint32_t* p[kMaxFlags];
};

__global__ void k_signal_flags(FlagPtrs f, int n, uint32_t value) {
  __threadfence_system();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.p[i]), "r"(value) : "memory");
}

__global__ void k_wait_flags(const uint32_t* flags, int n, uint32_t value) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    uint32_t v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + i) : "memory");
    } while ((int32_t)(v - value) < 0);  // wrap-safe v >= value
  }
  __syncthreads();
  __threadfence_system();
}

}  // namespace
}  // namespace lmgs

extern "C" int lmgs_signal_flags(uint32_t* const* flags, int32_t n, uint32_t value, void* stream) {
  if (n < 0 || n > lmgs::kMaxFlags || (n > 0 && !flags)) return LMGS_ERR_INVALID;
  if (n == 0) return LMGS_OK;
  lmgs::FlagPtrs f{};
  for (int i = 0; i < n; ++i) {
    if (!flags[i]) return LMGS_ERR_INVALID;
    f.p[i] = flags[i];
  }
  lmgs::k_signal_flags<<<1, 64, 0, static_cast<cudaStream_t>(stream)>>>(f, n, value);
  return cudaGetLastError() == cudaSuccess ? LMGS_OK : LMGS_ERR_CUDA;
}

extern "C" int lmgs_wait_flags(const uint32_t* flags, int32_t n, uint32_t value, void* stream) {
  if (n < 0 || (n > 0 && !flags)) return LMGS_ERR_INVALID;
  if (n == 0) return LMGS_OK;
  lmgs::k_wait_flags<<<1, 64, 0, static_cast<cudaStream_t>(stream)>>>(flags, n, value);
  return cudaGetLastError() == cudaSuccess ? LMGS_OK : LMGS_ERR_CUDA;
}
