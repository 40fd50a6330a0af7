// Random 8-byte gathers over a large source (1e9 rows = 8 GB): time and DRAM
// bytes per load flavour. Run under ncu --metrics dram__bytes_read.sum for the
// traffic. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a gather_flavors.cu -o gather_flavors
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return uint32_t(x);
}
__global__ void make_idx(uint32_t* idx, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    idx[i] = uint32_t((uint64_t(mix(i)) * n) >> 32);
}
template <int F>
__device__ __forceinline__ unsigned long long ld(const unsigned long long* p, uint64_t pol) {
  unsigned long long v;
  if constexpr (F == 0) v = *p;
  else if constexpr (F == 1) v = __ldcg(p);
  else if constexpr (F == 2) asm volatile("ld.global.nc.L1::no_allocate.b64 %0, [%1];" : "=l"(v) : "l"(p));
  else if constexpr (F == 3) v = __ldcs(p);
  else if constexpr (F == 4) asm volatile("ld.global.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  else if constexpr (F == 5) asm volatile("ld.global.cg.L2::64B.b64 %0, [%1];" : "=l"(v) : "l"(p));
  else if constexpr (F == 6) v = __ldlu(p);
  else asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
template <int F>
__global__ void gather(const uint32_t* __restrict__ idx, const unsigned long long* __restrict__ src,
                       unsigned long long* __restrict__ dst, uint64_t n) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  constexpr int U = 8;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * U;
  for (uint64_t b = blockIdx.x * uint64_t(blockDim.x) * U + threadIdx.x; b < n; b += stride) {
    unsigned long long v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = b + uint64_t(u) * blockDim.x;
      v[u] = i < n ? ld<F>(src + idx[i], pol) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = b + uint64_t(u) * blockDim.x;
      if (i < n) __stcs(dst + i, v[u]);
    }
  }
}
// two 8-byte columns by the same rows: separate source arrays (two random
// loads a row) vs one interleaved 16-byte source row (one load)
template <bool IL>
__global__ void gather2(const uint32_t* __restrict__ idx, const unsigned long long* __restrict__ a,
                        const unsigned long long* __restrict__ b, unsigned long long* __restrict__ da,
                        unsigned long long* __restrict__ db, uint64_t n) {
  constexpr int U = 4;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * U;
  for (uint64_t s = blockIdx.x * uint64_t(blockDim.x) * U + threadIdx.x; s < n; s += stride) {
    unsigned long long va[U], vb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = s + uint64_t(u) * blockDim.x;
      if (i < n) {
        const uint64_t r = idx[i];
        if constexpr (IL) {
          const ulonglong2 q = __ldcg(reinterpret_cast<const ulonglong2*>(a) + r);
          va[u] = q.x;
          vb[u] = q.y;
        } else {
          va[u] = __ldcg(a + r);
          vb[u] = __ldcg(b + r);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = s + uint64_t(u) * blockDim.x;
      if (i < n) {
        __stcs(da + i, va[u]);
        __stcs(db + i, vb[u]);
      }
    }
  }
}
template <bool IL>
float run2(const uint32_t* idx, const unsigned long long* a, const unsigned long long* b, unsigned long long* da,
           unsigned long long* db, uint64_t n, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  gather2<IL><<<sms * 4, 512>>>(idx, a, b, da, db, n);
  cudaEventRecord(e0);
  gather2<IL><<<sms * 4, 512>>>(idx, a, b, da, db, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}
template <int F>
float run(const uint32_t* idx, const unsigned long long* src, unsigned long long* dst, uint64_t n, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<F><<<sms * 4, 512>>>(idx, src, dst, n);
  cudaEventRecord(a);
  gather<F><<<sms * 4, 512>>>(idx, src, dst, n);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}
int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? uint64_t(atof(argv[1])) : 1000000000ull;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* idx;
  unsigned long long *src, *dst;
  if (cudaMalloc(&idx, n * 4) || cudaMalloc(&src, n * 8) || cudaMalloc(&dst, n * 8)) { printf("oom\n"); return 1; }
  cudaMemset(src, 1, n * 8);
  make_idx<<<sms * 8, 512>>>(idx, n);
  cudaDeviceSynchronize();
  const char* names[] = {"plain", "ldcg", "nc.no_allocate", "ldcs", "L2 evict_first hint", "cg.L2::64B", "ldlu", "nc.no_alloc+evict_first"};
  float t[8];
  t[0] = run<0>(idx, src, dst, n, sms);
  t[1] = run<1>(idx, src, dst, n, sms);
  t[2] = run<2>(idx, src, dst, n, sms);
  t[3] = run<3>(idx, src, dst, n, sms);
  t[4] = run<4>(idx, src, dst, n, sms);
  t[5] = run<5>(idx, src, dst, n, sms);
  t[6] = run<6>(idx, src, dst, n, sms);
  t[7] = run<7>(idx, src, dst, n, sms);
  for (int i = 0; i < 8; ++i) printf("%-26s %8.2f ms  %.2f G rows/s\n", names[i], t[i], n / (t[i] * 1e6));
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  if (argc > 2) {  // two columns: src = [2n] words (separate: a = src, b = src + n; interleaved: 16-byte rows)
    cudaFree(dst);
    unsigned long long *src2, *d2;
    if (cudaMalloc(&src2, n * 16) || cudaMalloc(&d2, n * 16)) { printf("oom2\n"); return 1; }
    cudaMemset(src2, 1, n * 16);
    const float ts = run2<false>(idx, src2, src2 + n, d2, d2 + n, n, sms);
    const float ti = run2<true>(idx, src2, nullptr, d2, d2 + n, n, sms);
    printf("two columns, separate arrays  %8.2f ms\ntwo columns, interleaved rows %8.2f ms\n", ts, ti);
  }
  return 0;
}
