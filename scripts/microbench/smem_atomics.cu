// Shared-memory atomic throughput on B200: ops per clock per SM for random
// 32-bit atomicAdd (with / without return) over 32768 words and over 256
// bins, and random plain loads/stores for comparison.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a smem_atomics.cu -o smem_atomics
#include <cstdio>
#include <cstdint>

template <int MODE, int BINS>
__global__ void __launch_bounds__(1024, 1) k(uint32_t* out, int iters) {
  extern __shared__ uint32_t h[];
  for (int i = threadIdx.x; i < BINS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x * 97u + 1u, acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x = x * 1664525u + 1013904223u;
      const uint32_t b = (x >> 8) & (BINS - 1);
      if (MODE == 0) acc += atomicAdd(&h[b], 1u);   // with return
      if (MODE == 1) atomicAdd(&h[b], 1u);          // no return
      if (MODE == 2) acc += h[b];                   // random load
      if (MODE == 3) h[b] = x;                      // random store
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[0] + acc;
  else if (acc == 0x12345) out[blockIdx.x] = acc;
}

template <int MODE, int BINS>
void run(const char* name, int sms, double clk_ghz) {
  uint32_t* out;
  cudaMalloc(&out, sms * 4);
  const int iters = 512;
  auto kern = k<MODE, BINS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, BINS * 4);
  kern<<<sms, 1024, BINS * 4>>>(out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<sms, 1024, BINS * 4>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = double(sms) * 1024 * iters * 8;
  printf("%-34s %8.3f ms  %6.2f ops/clk/SM  (%.1f G ops/s)\n", name, ms, ops / sms / (ms * 1e-3 * clk_ghz * 1e9),
         ops / (ms * 1e-3) / 1e9);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int khz;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double ghz = khz / 1e6;
  printf("SMs %d, clock %.3f GHz\n", sms, ghz);
  run<0, 32768>("atomicAdd+ret, 32768 words", sms, ghz);
  run<1, 32768>("atomicAdd no ret, 32768 words", sms, ghz);
  run<0, 256>("atomicAdd+ret, 256 bins", sms, ghz);
  run<1, 256>("atomicAdd no ret, 256 bins", sms, ghz);
  run<0, 4096>("atomicAdd+ret, 4096 bins", sms, ghz);
  run<2, 32768>("random LDS, 32768 words", sms, ghz);
  run<3, 32768>("random STS, 32768 words", sms, ghz);
  return 0;
}
