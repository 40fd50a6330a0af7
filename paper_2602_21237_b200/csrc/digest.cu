// digest.cu — the reference's 128-bit multiset result digest, on the device.
//
// Replaces relation.py:319-330 (multiset_digest) + hashing.py:64-109
// (row_digests, combine_digests), bit-exactly:
//   * a row is serialised canonically (relation.py:138-151): columns in
//     schema order, Int64 as 8 little-endian bytes, Bytes(w) raw; width W;
//   * it is read as n_words = max(1, ceil(W/8)) little-endian 64-bit words,
//     zero padded;
//   * per lane L in {0x8C2F1D7A6E5B3940, 0x1F83D9ABFB41BD6B} (hashing.py:20):
//     (mult_j, off_j) come from a splitmix64 stream seeded with L ^ W
//     (mult_j = a | 1, off_j = b, two draws per word), the accumulator starts
//     at fmix64(L + W) and folds acc ^= (word_j ^ off_j) * mult_j; the lane
//     value is fmix64(acc);
//   * the relation digest is the XOR over rows of (lane0 << 64 | lane1).
// The row bytes never exist in memory: every thread assembles its row's
// words from the columns in registers, so a digest is one read of the
// columns (the reference serialises the whole relation first).
#include <vector>

#include "common.cuh"

namespace rl {
namespace digest {

constexpr uint64_t kLaneSeeds[2] = {0x8C2F1D7A6E5B3940ull, 0x1F83D9ABFB41BD6Bull};
constexpr int kMaxWords = 64;  // rows up to 512 bytes wide
constexpr int kThreads = 256;

struct Consts {
  uint64_t mult[2][kMaxWords];
  uint64_t off[2][kMaxWords];
  uint64_t init[2];
  int n_words;
};

static uint64_t splitmix_next(uint64_t& state) {
  state += 0x9E3779B97F4A7C15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ void fold(const Consts& k, uint64_t word, int j, uint64_t& a0, uint64_t& a1) {
  a0 ^= (word ^ k.off[0][j]) * k.mult[0][j];
  a1 ^= (word ^ k.off[1][j]) * k.mult[1][j];
}

// the per-word constants travel in the kernel parameters (no shared
// __constant__ state: concurrent digests on different streams are safe)
__global__ void __launch_bounds__(kThreads) digest_kernel(ColumnSet cols, const Consts k, int64_t n,
                                                          unsigned long long* out2) {
  uint64_t x0 = 0, x1 = 0;
  for (int64_t r = int64_t(blockIdx.x) * kThreads + threadIdx.x; r < n; r += int64_t(gridDim.x) * kThreads) {
    uint64_t a0 = k.init[0], a1 = k.init[1];
    uint64_t word = 0;
    int filled = 0, j = 0;  // bytes in the current word, word index
    for (int ci = 0; ci < cols.n; ++ci) {
      const int w = cols.c[ci].width;
      const uint8_t* src = static_cast<const uint8_t*>(cols.c[ci].src) + uint64_t(r) * w;
      int b = 0;
      if (filled == 0 && (w & 7) == 0 && (reinterpret_cast<uintptr_t>(src) & 7) == 0) {
        for (; b < w; b += 8) fold(k, *reinterpret_cast<const uint64_t*>(src + b), j++, a0, a1);  // aligned words
        continue;
      }
      for (; b < w; ++b) {
        word |= uint64_t(src[b]) << (8 * filled);
        if (++filled == 8) {
          fold(k, word, j++, a0, a1);
          word = 0;
          filled = 0;
        }
      }
    }
    if (filled || j == 0) fold(k, word, j++, a0, a1);  // zero padding; a width-0 row is one zero word
    x0 ^= fmix64(a0);
    x1 ^= fmix64(a1);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    x0 ^= __shfl_xor_sync(0xffffffffu, x0, o);
    x1 ^= __shfl_xor_sync(0xffffffffu, x1, o);
  }
  __shared__ uint64_t wx[2][kThreads / 32];  // one pair of global atomics per CTA
  if ((threadIdx.x & 31) == 0) {
    wx[0][threadIdx.x >> 5] = x0;
    wx[1][threadIdx.x >> 5] = x1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t y0 = 0, y1 = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      y0 ^= wx[0][w];
      y1 ^= wx[1][w];
    }
    atomicXor(&out2[0], (unsigned long long)y0);
    atomicXor(&out2[1], (unsigned long long)y1);
  }
}

int multiset_digest(const rl_column* columns, int n_columns, int64_t n, uint64_t* out2, cudaStream_t stream) {
  if (n < 0 || n_columns < 1 || n_columns > RL_MAX_COLUMNS || !columns || !out2) return RL_ERR_BAD_ARG;
  ColumnSet cs;
  cs.n = n_columns;
  int64_t width = 0;
  for (int i = 0; i < n_columns; ++i) {
    if (columns[i].width < 0 || (columns[i].width > 0 && n > 0 && !columns[i].src)) return RL_ERR_BAD_ARG;
    cs.c[i] = columns[i];
    width += columns[i].width;
  }
  const int n_words = int(std::max<int64_t>(1, (width + 7) / 8));
  if (n_words > kMaxWords) return RL_ERR_BAD_ARG;
  cudaError_t e = cudaMemsetAsync(out2, 0, 16, stream);
  if (e != cudaSuccess) return rl_cuda_status(e);
  if (n == 0) return RL_OK;  // relation.py:327-328: the empty digest is 0
  Consts k{};
  k.n_words = n_words;
  for (int lane = 0; lane < 2; ++lane) {
    uint64_t state = kLaneSeeds[lane] ^ uint64_t(width);
    for (int j = 0; j < n_words; ++j) {
      k.mult[lane][j] = splitmix_next(state) | 1ull;
      k.off[lane][j] = splitmix_next(state);
    }
    k.init[lane] = fmix64(kLaneSeeds[lane] + uint64_t(width));
  }
  const int grid = int(std::min<int64_t>((n + kThreads - 1) / kThreads, int64_t(device_sm_count()) * 8));
  digest_kernel<<<grid, kThreads, 0, stream>>>(cs, k, n, reinterpret_cast<unsigned long long*>(out2));
  count_launches(1);
  return rl_cuda_status(cudaGetLastError());
}

}  // namespace digest
}  // namespace rl

extern "C" RL_API int rl_multiset_digest(const rl_column* columns, int32_t n_columns, int64_t n, uint64_t* out2,
                                         void* stream) {
  return rl::digest::multiset_digest(columns, n_columns, n, out2, static_cast<cudaStream_t>(stream));
}
