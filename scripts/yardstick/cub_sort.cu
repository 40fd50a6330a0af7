// Yardstick only (never linked into the product): CUB onesweep SortPairs on
// cfg2-shaped data (10M uint64 keys, uint32 values) timed with CUDA events.
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <random>
int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 10000000;
  std::vector<unsigned long long> hk(n);
  std::mt19937_64 g(1);
  for (long i = 0; i < n; ++i) hk[i] = g();
  unsigned long long *k_in, *k_out; unsigned *v_in, *v_out;
  cudaMalloc(&k_in, n * 8); cudaMalloc(&k_out, n * 8); cudaMalloc(&v_in, n * 4); cudaMalloc(&v_out, n * 4);
  cudaMemcpy(k_in, hk.data(), n * 8, cudaMemcpyHostToDevice);
  void* tmp = nullptr; size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(tmp, tb, k_in, k_out, v_in, v_out, n);
  cudaMalloc(&tmp, tb);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9, sum = 0; int reps = 20;
  for (int r = 0; r < reps + 3; ++r) {
    cudaEventRecord(a);
    cub::DeviceRadixSort::SortPairs(tmp, tb, k_in, k_out, v_in, v_out, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r >= 3) { sum += ms; if (ms < best) best = ms; }
  }
  printf("cub SortPairs u64/u32 n=%ld: mean %.4f ms best %.4f ms (%.1f GB/s at 8 passes x 24 B)\n", n, sum / reps, best,
         8.0 * 24 * n / (sum / reps / 1e3) / 1e9);
  return 0;
}
