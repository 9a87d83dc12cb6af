// LMGS checkpoint <-> device SoA, and RGB8 wire-frame encoding.
//
// Reference formats (pkg/src/landmark/):
//   data_io.py:3-9, 256-316  LMGS: "<4sIIQ" header (magic, version 1,
//       sh_degree, count), count rows of f32 [mean 3 | quat 4 (w,x,y,z) |
//       scale 3 | logit 1 | SH 3*(d+1)^2], grid flag u8, optional grid block
//       (bbox 6*f32, nx u32, ny u32, nx*ny u32 submodel ids), little-endian.
//   render_runtime.py:397-401  encode_frame: round(clip(rgb, 0, 1) * 255) as
//       uint8 (numpy rounds half to even) after a JSON header.
//
// Load: the host parses and validates the header, then streams the rows in
// chunks through two pinned buffers — fread of chunk i+1 overlaps the H2D
// copy and the de-interleave kernel of chunk i — into the caller's device
// SoA arrays (the layout GaussianModel holds).  Save is the mirror image.
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <string>

#include "lmgs_internal.cuh"

namespace lmgs {
namespace {

constexpr char kMagic[4] = {'L', 'M', 'G', 'S'};
constexpr uint32_t kVersion = 1;
constexpr size_t kHeaderBytes = 4 + 4 + 4 + 8;
constexpr size_t kChunkRows = 1 << 17;  // rows per streamed chunk

inline int row_floats(uint32_t sh_degree) { return 11 + 3 * (int)((sh_degree + 1) * (sh_degree + 1)); }

// AoS rows [n, stride] -> SoA fields (one thread per float of the chunk)
__global__ void k_rows_to_soa(const float* __restrict__ rows, int64_t n_rows, int stride,
                              int64_t row0, float* means, float* quats, float* scales,
                              float* logits, float* sh) {
  const int64_t total = n_rows * stride;
  const int shn = stride - 11;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / stride;
    const int c = (int)(e - r * stride);
    const int64_t g = row0 + r;
    const float v = rows[e];
    if (c < 3) means[3 * g + c] = v;
    else if (c < 7) quats[4 * g + (c - 3)] = v;
    else if (c < 10) scales[3 * g + (c - 7)] = v;
    else if (c == 10) logits[g] = v;
    else sh[(int64_t)shn * g + (c - 11)] = v;
  }
}

__global__ void k_soa_to_rows(float* __restrict__ rows, int64_t n_rows, int stride, int64_t row0,
                              const float* means, const float* quats, const float* scales,
                              const float* logits, const float* sh) {
  const int64_t total = n_rows * stride;
  const int shn = stride - 11;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / stride;
    const int c = (int)(e - r * stride);
    const int64_t g = row0 + r;
    float v;
    if (c < 3) v = means[3 * g + c];
    else if (c < 7) v = quats[4 * g + (c - 3)];
    else if (c < 10) v = scales[3 * g + (c - 7)];
    else if (c == 10) v = logits[g];
    else v = sh[(int64_t)shn * g + (c - 11)];
    rows[e] = v;
  }
}

// encode_frame's pixels: numpy computes clip/multiply in fp64 and rounds half
// to even; the same ops in fp64 (rint = round-half-even) give the same bytes.
__global__ void k_encode_rgb8(const float* __restrict__ rgb, int64_t n, uint8_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = fmin(fmax((double)rgb[i], 0.0), 1.0) * 255.0;
    out[i] = (uint8_t)rint(v);
  }
}

unsigned grid_of(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)(g > 0 ? g : 1);
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

int set_err(char* err, int err_len, int code, const std::string& msg) {
  if (err && err_len > 0) {
    strncpy(err, msg.c_str(), (size_t)err_len - 1);
    err[err_len - 1] = 0;
  }
  return code;
}

int read_info(FILE* f, const char* path, lmgs_checkpoint_info* info, char* err, int err_len) {
  memset(info, 0, sizeof(*info));
  unsigned char hdr[kHeaderBytes];
  if (fread(hdr, 1, kHeaderBytes, f) != kHeaderBytes)
    return set_err(err, err_len, LMGS_ERR_FORMAT,
                   std::string(path) + ": truncated at byte offset 0");
  if (memcmp(hdr, kMagic, 4) != 0)
    return set_err(err, err_len, LMGS_ERR_FORMAT, std::string(path) + ": bad magic");
  memcpy(&info->version, hdr + 4, 4);
  memcpy(&info->sh_degree, hdr + 8, 4);
  uint64_t count = 0;
  memcpy(&count, hdr + 12, 8);
  if (info->version != kVersion)
    return set_err(err, err_len, LMGS_ERR_FORMAT,
                   std::string(path) + ": unsupported version " + std::to_string(info->version));
  if (info->sh_degree > 3)
    return set_err(err, err_len, LMGS_ERR_UNSUPPORTED,
                   std::string(path) + ": sh_degree " + std::to_string(info->sh_degree));
  info->row_floats = row_floats(info->sh_degree);
  info->data_offset = (int64_t)kHeaderBytes;
  // the count is untrusted: bound it by the bytes the file holds before any
  // multiplication (the reference's reader fails with "truncated" there)
  if (fseek(f, 0, SEEK_END) != 0)
    return set_err(err, err_len, LMGS_ERR_IO, std::string(path) + ": seek failed");
  const int64_t file_bytes = (int64_t)ftell(f);
  const uint64_t row_bytes = 4ull * (uint64_t)info->row_floats;
  const uint64_t avail = file_bytes > info->data_offset ? (uint64_t)(file_bytes - info->data_offset) : 0;
  if (count > avail / row_bytes)
    return set_err(err, err_len, LMGS_ERR_FORMAT,
                   std::string(path) + ": truncated at byte offset " + std::to_string(file_bytes));
  info->count = (int64_t)count;
  const int64_t data_bytes = info->count * (int64_t)info->row_floats * 4;
  if (fseek(f, (long)(info->data_offset + data_bytes), SEEK_SET) != 0)
    return set_err(err, err_len, LMGS_ERR_FORMAT, std::string(path) + ": truncated rows");
  unsigned char flag = 0;
  if (fread(&flag, 1, 1, f) != 1)
    return set_err(err, err_len, LMGS_ERR_FORMAT,
                   std::string(path) + ": truncated at byte offset " +
                       std::to_string(info->data_offset + data_bytes));
  info->has_grid = flag ? 1 : 0;
  if (flag) {
    float bbox[6];
    uint32_t nxy[2];
    if (fread(bbox, 4, 6, f) != 6 || fread(nxy, 4, 2, f) != 2)
      return set_err(err, err_len, LMGS_ERR_FORMAT, std::string(path) + ": truncated grid");
    memcpy(info->grid_bbox, bbox, sizeof(bbox));
    info->grid_nx = nxy[0];
    info->grid_ny = nxy[1];
    info->grid_table_offset = info->data_offset + data_bytes + 1 + 24 + 8;
    if (fseek(f, (long)(info->grid_table_offset + 4 * (int64_t)nxy[0] * nxy[1]), SEEK_SET) != 0)
      return set_err(err, err_len, LMGS_ERR_FORMAT, std::string(path) + ": truncated grid");
  }
  // the reader takes exactly the bytes it needs; a shorter file fails above
  long end = ftell(f);
  fseek(f, 0, SEEK_END);
  if (ftell(f) < end)
    return set_err(err, err_len, LMGS_ERR_FORMAT, std::string(path) + ": truncated");
  return LMGS_OK;
}

}  // namespace
}  // namespace lmgs

using namespace lmgs;

extern "C" {

int lmgs_checkpoint_info_read(const char* path, lmgs_checkpoint_info* info, char* err,
                              int err_len) {
  if (!path || !info) return LMGS_ERR_INVALID;
  File file;
  file.f = fopen(path, "rb");
  if (!file.f)
    return set_err(err, err_len, LMGS_ERR_IO, std::string(path) + ": " + strerror(errno));
  return read_info(file.f, path, info, err, err_len);
}

int lmgs_checkpoint_load(const char* path, float* means, float* quats, float* scales,
                         float* logits, float* sh, uint32_t* grid_table_host, void* stream,
                         char* err, int err_len) {
  if (!path) return LMGS_ERR_INVALID;
  File file;
  file.f = fopen(path, "rb");
  if (!file.f)
    return set_err(err, err_len, LMGS_ERR_IO, std::string(path) + ": " + strerror(errno));
  lmgs_checkpoint_info info;
  if (int r = read_info(file.f, path, &info, err, err_len)) return r;
  if (info.count > 0 && (!means || !quats || !scales || !logits || !sh))
    return set_err(err, err_len, LMGS_ERR_INVALID, "null destination array");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int stride = info.row_floats;
  const size_t chunk_bytes = kChunkRows * (size_t)stride * 4;
  float* host[2] = {nullptr, nullptr};
  float* dev[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  int rc = LMGS_OK;
  auto cuda_fail = [&](cudaError_t e, const char* what) {
    cudaGetLastError();
    rc = set_err(err, err_len, e == cudaErrorMemoryAllocation ? LMGS_ERR_OOM : LMGS_ERR_CUDA,
                 std::string(what) + ": " + cudaGetErrorString(e));
  };
  for (int b = 0; b < 2 && rc == LMGS_OK; ++b) {
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&host[b]), chunk_bytes,
                                  cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&dev[b]), chunk_bytes);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
    if (e != cudaSuccess) cuda_fail(e, "checkpoint staging");
  }
  fseek(file.f, (long)info.data_offset, SEEK_SET);
  for (int64_t row0 = 0, it = 0; rc == LMGS_OK && row0 < info.count; row0 += kChunkRows, ++it) {
    const int b = (int)(it & 1);
    const int64_t rows = info.count - row0 < (int64_t)kChunkRows ? info.count - row0
                                                                 : (int64_t)kChunkRows;
    // the pinned buffer is reused only after its previous chunk was consumed
    cudaEventSynchronize(done[b]);
    const size_t bytes = (size_t)rows * stride * 4;
    if (fread(host[b], 1, bytes, file.f) != bytes) {
      rc = set_err(err, err_len, LMGS_ERR_FORMAT, std::string(path) + ": truncated rows");
      break;
    }
    cudaError_t e = cudaMemcpyAsync(dev[b], host[b], bytes, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
      k_rows_to_soa<<<grid_of(rows * stride), 256, 0, s>>>(dev[b], rows, stride, row0, means,
                                                          quats, scales, logits, sh);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaEventRecord(done[b], s);
    if (e != cudaSuccess) cuda_fail(e, "checkpoint upload");
  }
  if (rc == LMGS_OK && info.has_grid && grid_table_host) {
    const size_t nt = (size_t)info.grid_nx * info.grid_ny;
    fseek(file.f, (long)info.grid_table_offset, SEEK_SET);
    if (fread(grid_table_host, 4, nt, file.f) != nt)
      rc = set_err(err, err_len, LMGS_ERR_FORMAT, std::string(path) + ": truncated grid");
  }
  cudaStreamSynchronize(s);
  for (int b = 0; b < 2; ++b) {
    if (host[b]) cudaFreeHost(host[b]);
    if (dev[b]) cudaFree(dev[b]);
    if (done[b]) cudaEventDestroy(done[b]);
  }
  return rc;
}

int lmgs_checkpoint_save(const char* path, const lmgs_gaussians* g,
                         const lmgs_checkpoint_info* grid, const uint32_t* grid_table_host,
                         void* stream, char* err, int err_len) {
  if (!path || !g || g->count < 0) return LMGS_ERR_INVALID;
  if (g->sh_degree < 0 || g->sh_degree > 3 ||
      g->sh_coeffs != (g->sh_degree + 1) * (g->sh_degree + 1))
    return set_err(err, err_len, LMGS_ERR_INVALID, "bad SH degree / coefficient count");
  if (grid && grid->has_grid && !grid_table_host) return LMGS_ERR_INVALID;
  // atomic write: temp file then rename (data_io.py:222-227)
  const std::string tmp = std::string(path) + ".tmp";
  File file;
  file.f = fopen(tmp.c_str(), "wb");
  if (!file.f) return set_err(err, err_len, LMGS_ERR_IO, tmp + ": " + strerror(errno));
  unsigned char hdr[kHeaderBytes];
  memcpy(hdr, kMagic, 4);
  const uint32_t version = kVersion, deg = (uint32_t)g->sh_degree;
  const uint64_t count = (uint64_t)g->count;
  memcpy(hdr + 4, &version, 4);
  memcpy(hdr + 8, &deg, 4);
  memcpy(hdr + 12, &count, 8);
  int rc = fwrite(hdr, 1, kHeaderBytes, file.f) == kHeaderBytes
               ? LMGS_OK
               : set_err(err, err_len, LMGS_ERR_IO, tmp + ": write failed");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int stride = row_floats(deg);
  const size_t chunk_bytes = kChunkRows * (size_t)stride * 4;
  float* host = nullptr;
  float* dev = nullptr;
  if (rc == LMGS_OK && g->count > 0) {
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&host), chunk_bytes,
                                  cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&dev), chunk_bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      rc = set_err(err, err_len, LMGS_ERR_OOM, "checkpoint staging");
    }
  }
  for (int64_t row0 = 0; rc == LMGS_OK && row0 < g->count; row0 += kChunkRows) {
    const int64_t rows =
        g->count - row0 < (int64_t)kChunkRows ? g->count - row0 : (int64_t)kChunkRows;
    k_soa_to_rows<<<grid_of(rows * stride), 256, 0, s>>>(dev, rows, stride, row0, g->means,
                                                        g->quats, g->scales, g->opacity_logits,
                                                        g->sh);
    const size_t bytes = (size_t)rows * stride * 4;
    cudaError_t e = cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      cudaGetLastError();
      rc = set_err(err, err_len, LMGS_ERR_CUDA, std::string("checkpoint download: ") +
                                                     cudaGetErrorString(e));
      break;
    }
    if (fwrite(host, 1, bytes, file.f) != bytes)
      rc = set_err(err, err_len, LMGS_ERR_IO, tmp + ": write failed");
  }
  if (rc == LMGS_OK) {
    const unsigned char flag = (grid && grid->has_grid) ? 1 : 0;
    bool ok = fwrite(&flag, 1, 1, file.f) == 1;
    if (ok && flag) {
      const uint32_t nxy[2] = {grid->grid_nx, grid->grid_ny};
      ok = fwrite(grid->grid_bbox, 4, 6, file.f) == 6 && fwrite(nxy, 4, 2, file.f) == 2 &&
           fwrite(grid_table_host, 4, (size_t)nxy[0] * nxy[1], file.f) ==
               (size_t)nxy[0] * nxy[1];
    }
    if (!ok) rc = set_err(err, err_len, LMGS_ERR_IO, tmp + ": write failed");
  }
  if (host) cudaFreeHost(host);
  if (dev) cudaFree(dev);
  if (fclose(file.f) != 0 && rc == LMGS_OK) rc = set_err(err, err_len, LMGS_ERR_IO, tmp);
  file.f = nullptr;
  if (rc == LMGS_OK && rename(tmp.c_str(), path) != 0)
    rc = set_err(err, err_len, LMGS_ERR_IO, std::string(path) + ": " + strerror(errno));
  if (rc != LMGS_OK) remove(tmp.c_str());
  return rc;
}

int lmgs_encode_rgb8(const float* rgb, int64_t n_values, uint8_t* out, void* stream) {
  if (n_values < 0 || (n_values > 0 && (!rgb || !out))) return LMGS_ERR_INVALID;
  if (n_values == 0) return LMGS_OK;
  k_encode_rgb8<<<grid_of(n_values), 256, 0, static_cast<cudaStream_t>(stream)>>>(rgb, n_values,
                                                                                  out);
  return cudaGetLastError() == cudaSuccess ? LMGS_OK : LMGS_ERR_CUDA;
}

}  // extern "C"
