// Stand-alone timing of the onesweep radix sort (sort.cu compiled into this
// TU with the variant's -D settings).  usage: sort_bench <n> <key_bytes> <passes>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2503_21364_b200/csrc/sort.cu"

using namespace lmgs;

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 20000000;
  const int kb = argc > 2 ? atoi(argv[2]) : 8;
  const int passes = argc > 3 ? atoi(argv[3]) : 2;
  const int vals = argc > 4 ? atoi(argv[4]) : 0;
  std::vector<uint64_t> h(n);
  uint64_t x = 88172645463325252ull;
  for (int64_t i = 0; i < n; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    h[i] = kb == 8 ? ((x % 8160) << 32) | (uint64_t)i : (uint32_t)x;
  }
  void *k0, *k1;
  uint32_t *v0 = nullptr, *v1 = nullptr;
  cudaMalloc(&k0, n * kb);
  cudaMalloc(&k1, n * kb);
  if (vals) { cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4); }
  if (kb == 8) cudaMemcpy(k0, h.data(), n * 8, cudaMemcpyHostToDevice);
  else {
    std::vector<uint32_t> h4(n);
    for (int64_t i = 0; i < n; ++i) h4[i] = (uint32_t)h[i];
    cudaMemcpy(k0, h4.data(), n * 4, cudaMemcpyHostToDevice);
  }
  void* src_copy;
  cudaMalloc(&src_copy, n * kb);
  cudaMemcpy(src_copy, k0, n * kb, cudaMemcpyDeviceToDevice);
  RadixPlan* plan; uint32_t *hist, *lb, *ctr;
  cudaMalloc(&plan, sizeof(RadixPlan));
  cudaMalloc(&hist, sizeof(uint32_t) * kMaxPasses * kRadix);
  cudaMalloc(&ctr, sizeof(uint32_t) * kMaxPasses);
  cudaMalloc(&lb, sizeof(uint32_t) * radix_lookback_words(n));
  void** slots; cudaMalloc(&slots, 2 * sizeof(void*));
  RadixSortBuffers b{};
  b.keys[0] = k0; b.keys[1] = k1; b.key_bytes = kb; b.vals[0] = v0; b.vals[1] = v1;
  b.plan = plan; b.hist = hist; b.lookback = lb; b.counters = ctr;
  b.keys_result = slots; b.vals_result = slots + 1; b.iota_vals = vals != 0;
  // optional 5th argument 1: device-side count -> persistent onesweep grid
  unsigned long long* d_n = nullptr;
  if (argc > 5 && atoi(argv[5])) {
    cudaMalloc(&d_n, sizeof(unsigned long long));
    unsigned long long hn = (unsigned long long)n;
    cudaMemcpy(d_n, &hn, sizeof(hn), cudaMemcpyHostToDevice);
    b.n_dev = d_n;
  }
  const int begin = kb == 8 ? 32 : 0;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int it = 0; it < 6; ++it) {
    cudaMemcpy(k0, src_copy, n * kb, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0);
    radix_sort(b, n, begin, passes, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0 && ms < best) best = ms;
  }
  // verify sortedness on the sorted bits
  void* res; cudaMemcpy(&res, slots, sizeof(void*), cudaMemcpyDeviceToHost);
  std::vector<uint64_t> out(n);
  if (kb == 8) cudaMemcpy(out.data(), res, n * 8, cudaMemcpyDeviceToHost);
  else { std::vector<uint32_t> o4(n); cudaMemcpy(o4.data(), res, n * 4, cudaMemcpyDeviceToHost);
         for (int64_t i = 0; i < n; ++i) out[i] = o4[i]; }
  int64_t bad = 0;
  const uint64_t mask = ((passes * 8 >= 64) ? ~0ull : ((1ull << (passes * 8)) - 1)) << begin;
  for (int64_t i = 1; i < n; ++i) {
    const uint64_t a = out[i - 1] & mask, c = out[i] & mask;
    if (a > c || (a == c && kb == 8 && (uint32_t)out[i - 1] > (uint32_t)out[i])) ++bad;
  }
  const double bytes = (double)n * (kb + (vals ? 4 : 0)) * 2 * passes;
  printf("items=%d ctas=%d win=%d n=%lld kb=%d vals=%d passes=%d: %.1f us  %.0f GB/s  %.1f us/pass  bad=%lld\n",
         LMGS_SORT_ITEMS, LMGS_SORT_MIN_CTAS, LMGS_LOOK_WINDOW, (long long)n, kb, vals, passes,
         best * 1e3, bytes / (best * 1e-3) / 1e9, best * 1e3 / passes, (long long)bad);
  return 0;
}
