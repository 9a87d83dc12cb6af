// Stand-alone timing + check of the K5 tile sort (sort.cu's tile_sort compiled
// into this TU): k keys tile << 32 | i with random tiles; checks that the ids
// come out grouped by tile in input order and that the per-tile counts match.
// usage: tile_sort_bench <k> <tiles>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2503_21364_b200/csrc/sort.cu"

using namespace lmgs;

static int bits_for(int64_t v) {
  int b = 0;
  while (((int64_t)1 << b) < v) ++b;
  return b;
}

int main(int argc, char** argv) {
  const int64_t k = argc > 1 ? atoll(argv[1]) : 20700000;
  const int tiles = argc > 2 ? atoi(argv[2]) : 8160;
  const int tile_bits = bits_for(tiles);
  std::vector<uint64_t> h(k);
  std::vector<uint32_t> cnt(tiles, 0);
  uint64_t x = 88172645463325252ull;
  for (int64_t i = 0; i < k; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const uint32_t t = (uint32_t)(x % tiles);
    h[i] = ((uint64_t)t << 32) | (uint64_t)i;
    ++cnt[t];
  }
  std::vector<uint32_t> hist(kMaxPasses * kRadix, 0);
  const int passes = tile_bits ? (tile_bits + 7) / 8 : 1;
  for (int64_t i = 0; i < k; ++i)
    for (int p = 0; p < passes; ++p) ++hist[p * kRadix + ((h[i] >> (32 + 8 * p)) & 0xff)];
  void *k0, *k1, *src;
  cudaMalloc(&k0, k * 8);
  cudaMalloc(&k1, k * 8);
  cudaMalloc(&src, k * 8);
  cudaMemcpy(src, h.data(), k * 8, cudaMemcpyHostToDevice);
  RadixPlan* plan; uint32_t *d_hist, *lb, *ctr, *seg;
  cudaMalloc(&plan, sizeof(RadixPlan));
  cudaMalloc(&d_hist, sizeof(uint32_t) * kMaxPasses * kRadix);
  cudaMemcpy(d_hist, hist.data(), sizeof(uint32_t) * kMaxPasses * kRadix, cudaMemcpyHostToDevice);
  cudaMalloc(&ctr, sizeof(uint32_t) * kMaxPasses);
  cudaMalloc(&lb, sizeof(uint32_t) * radix_lookback_words(k));
  cudaMalloc(&seg, sizeof(uint32_t) * tiles);
  void** slots; cudaMalloc(&slots, 2 * sizeof(void*));
  RadixSortBuffers b{};
  b.keys[0] = k0; b.keys[1] = k1; b.key_bytes = 8;
  b.plan = plan; b.hist = d_hist; b.lookback = lb; b.counters = ctr;
  b.keys_result = slots; b.hist_ready = true; b.seg_counts = seg; b.seg_shift = 32;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int it = 0; it < 8; ++it) {
    cudaMemcpy(k0, src, k * 8, cudaMemcpyDeviceToDevice);
    cudaMemset(seg, 0, sizeof(uint32_t) * tiles);
    cudaEventRecord(e0);
    tile_sort(b, k, tile_bits, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0 && ms < best) best = ms;
  }
  void* res; cudaMemcpy(&res, slots, sizeof(void*), cudaMemcpyDeviceToHost);
  std::vector<uint32_t> out(k), segs(tiles);
  cudaMemcpy(out.data(), res, k * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(segs.data(), seg, tiles * 4, cudaMemcpyDeviceToHost);
  int64_t bad = 0, badseg = 0, pos = 0;
  for (int t = 0; t < tiles; ++t) {
    if (segs[t] != cnt[t]) ++badseg;
    uint32_t prev = 0;
    for (uint32_t j = 0; j < cnt[t]; ++j, ++pos) {
      const uint32_t id = out[pos];
      if ((h[id] >> 32) != (uint64_t)t || (j && id <= prev)) ++bad;
      prev = id;
    }
  }
  printf("tile_sort k=%lld tiles=%d tile_bits=%d passes=%d: %.1f us  bad=%lld badseg=%lld err=%s\n",
         (long long)k, tiles, tile_bits, passes,
         best * 1e3, (long long)bad, (long long)badseg, cudaGetErrorString(cudaGetLastError()));
  return bad || badseg ? 1 : 0;
}
