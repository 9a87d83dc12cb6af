// Calibration only (not shipped): CUB DeviceRadixSort on the two sort shapes
// of the pipeline, to size the headroom of our onesweep.
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>

int main() {
  const int n64 = 20900000, n32 = 6000000;
  std::vector<unsigned long long> h(n64);
  unsigned long long x = 88172645463325252ull;
  for (int i = 0; i < n64; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = ((x % 8160) << 32) | (unsigned)i; }
  unsigned long long *k0, *k1; cudaMalloc(&k0, n64 * 8); cudaMalloc(&k1, n64 * 8);
  cudaMemcpy(k0, h.data(), n64 * 8, cudaMemcpyHostToDevice);
  unsigned *a0, *a1, *v0, *v1; cudaMalloc(&a0, n32 * 4); cudaMalloc(&a1, n32 * 4); cudaMalloc(&v0, n32 * 4); cudaMalloc(&v1, n32 * 4);
  std::vector<unsigned> h4(n32); for (int i = 0; i < n32; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h4[i] = (unsigned)x & 0xffffff; }
  cudaMemcpy(a0, h4.data(), n32 * 4, cudaMemcpyHostToDevice);
  size_t t1 = 0, t2 = 0; void* tmp = nullptr;
  cub::DeviceRadixSort::SortKeys(nullptr, t1, k0, k1, n64, 32, 48);
  cub::DeviceRadixSort::SortPairs(nullptr, t2, a0, a1, v0, v1, n32, 0, 24);
  cudaMalloc(&tmp, t1 > t2 ? t1 : t2);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) {
    float best = 1e9, best2 = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(e0);
      cub::DeviceRadixSort::SortKeys(tmp, t1, k0, k1, n64, 32, 48);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      cudaEventRecord(e0);
      cub::DeviceRadixSort::SortPairs(tmp, t2, a0, a1, v0, v1, n32, 0, 24);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (ms < best2) best2 = ms;
    }
    if (w) printf("CUB u64 keys 20.9M bits 32-48: %.1f us | u32 pairs 6M bits 0-24: %.1f us\n", best * 1e3, best2 * 1e3);
  }
  return 0;
}
