// expand.cu — K6 run expansion fused with K7 column gathers, plus the
// standalone row gather used by tensor_sort.
//
// Replaces tensorpath.py:157-185:
//   local = arange(total) - repeat(cum[:-1], per_key)
//   li, ri = divmod(local, repeat(right_counts, per_key))
//   left_rows  = left_positions[repeat(left_starts, per_key) + li]
//   right_rows = right_positions[repeat(right_starts, per_key) + ri]
//   key column = repeat(matched_keys, per_key); other columns gathered.
//
// Output-space load balancing: CTA b owns output pairs
// [out_begin + b*2048, ...+2048). It locates the first and last matched key
// of its range with two binary searches over pair_offsets, stages that
// window of pair_offsets (at most 2049 entries: every matched key owns >= 1
// pair) in shared memory, and each thread resolves its pairs there. A
// Zipf-heavy key (1.24M x 1.24M pairs in BASELINE cfg3) is spread over as
// many CTAs as it has output tiles, so skew never serialises a thread.
// The numpy intermediates (local, cr, li/ri, expanded starts: 4 index
// arrays of `total` entries) are never materialised.
#include <algorithm>

#include "common.cuh"

namespace rl {
namespace expand {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;

// last index g in [0, m] with offs[g] <= t (offs is non-decreasing, offs[0] = 0 <= t)
__device__ __forceinline__ int64_t upper_bound_minus1(const uint64_t* __restrict__ offs, int64_t m, uint64_t t) {
  int64_t lo = 0, len = m + 1;
  while (len > 0) {
    const int64_t half = len >> 1;
    if (__ldg(reinterpret_cast<const unsigned long long*>(offs) + lo + half) <= t) {
      lo += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  return lo - 1;
}

struct ExpandArgs {
  const int64_t* matched_keys;
  const uint32_t* ls;
  const uint32_t* rs;
  const uint32_t* rc;
  const uint64_t* offs;
  int64_t m;
  const uint32_t* lpos;
  const uint32_t* rpos;
  uint64_t out_begin, out_end;
  uint32_t* lrows_out;
  uint32_t* rrows_out;
  uint64_t* checksum;  // checksum mode when non-null
};

template <bool kChecksum>
__global__ void __launch_bounds__(kThreads) expand_kernel(ExpandArgs a, ColumnSet cols) {
  __shared__ uint64_t so[kTile + 1];
  __shared__ int64_t s_g[2];
  const int tid = threadIdx.x;
  const uint64_t t0 = a.out_begin + uint64_t(blockIdx.x) * kTile;
  const uint64_t t1 = min(t0 + kTile, a.out_end);
  if (tid < 2) s_g[tid] = upper_bound_minus1(a.offs, a.m, tid == 0 ? t0 : t1 - 1);
  __syncthreads();
  const int64_t g0 = s_g[0];
  const int nk = int(s_g[1] - g0) + 1;  // <= kTile
  for (int i = tid; i <= nk; i += kThreads) so[i] = a.offs[g0 + i];
  __syncthreads();

  uint64_t sum = 0;
#pragma unroll 2
  for (int it = 0; it < kItems; ++it) {
    const uint64_t t = t0 + uint64_t(it) * kThreads + tid;
    if (t >= t1) break;
    // binary search in the staged window: last k with so[k] <= t
    int lo = 0, len = nk;
    while (len > 0) {
      const int half = len >> 1;
      if (so[lo + half] <= t) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    const int k = lo - 1;
    const int64_t g = g0 + k;
    const uint64_t local = t - so[k];
    const uint32_t c = __ldg(a.rc + g);
    uint64_t li, ri;
    if (local < (1ull << 32)) {
      const uint32_t l32 = uint32_t(local);
      li = l32 / c;
      ri = l32 - uint32_t(li) * c;
    } else {
      li = local / c;
      ri = local - li * c;
    }
    const uint32_t lrow = __ldg(a.lpos + __ldg(a.ls + g) + li);
    const uint32_t rrow = __ldg(a.rpos + __ldg(a.rs + g) + ri);
    if (kChecksum) {
      sum += fmix64((uint64_t(lrow) << 32) | rrow);
      continue;
    }
    const uint64_t o = t - a.out_begin;
    if (a.lrows_out) __stcs(a.lrows_out + o, lrow);
    if (a.rrows_out) __stcs(a.rrows_out + o, rrow);
    for (int ci = 0; ci < cols.n; ++ci) {
      const rl_column& col = cols.c[ci];
      const int w = col.width;
      uint8_t* dst = static_cast<uint8_t*>(col.dst) + o * uint64_t(w);
      if (col.side == RL_SIDE_KEY) {
        __stcs(reinterpret_cast<long long*>(dst), (long long)__ldg(reinterpret_cast<const long long*>(a.matched_keys) + g));
      } else {
        const uint64_t row = col.side == RL_SIDE_LEFT ? lrow : rrow;
        copy_row(static_cast<const uint8_t*>(col.src) + row * uint64_t(w), dst, w);
      }
    }
  }
  if (kChecksum) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((tid & 31) == 0 && sum) atomicAdd(reinterpret_cast<unsigned long long*>(a.checksum), (unsigned long long)sum);
  }
}

static int fill_columns(ColumnSet& cs, const rl_column* columns, int n_columns, bool allow_key) {
  if (n_columns < 0 || n_columns > RL_MAX_COLUMNS) return RL_ERR_BAD_ARG;
  if (n_columns > 0 && columns == nullptr) return RL_ERR_BAD_ARG;
  cs.n = n_columns;
  for (int i = 0; i < n_columns; ++i) {
    const rl_column& c = columns[i];
    if (c.width < 0) return RL_ERR_BAD_ARG;
    if (c.side == RL_SIDE_KEY) {
      if (!allow_key || c.width != 8 || c.dst == nullptr) return RL_ERR_BAD_ARG;
    } else if (c.side == RL_SIDE_LEFT || c.side == RL_SIDE_RIGHT) {
      if (c.width > 0 && (c.src == nullptr || c.dst == nullptr)) return RL_ERR_BAD_ARG;
      if (!allow_key && c.side != RL_SIDE_LEFT) return RL_ERR_BAD_ARG;
    } else {
      return RL_ERR_BAD_ARG;
    }
    cs.c[i] = c;
  }
  return RL_OK;
}

int join_expand(const int64_t* matched_keys, const uint32_t* ls, const uint32_t* rs, const uint32_t* rc,
                const uint64_t* offs, int64_t m, const uint32_t* lpos, const uint32_t* rpos, uint64_t out_begin,
                uint64_t out_end, uint32_t* lrows_out, uint32_t* rrows_out, const rl_column* columns,
                int n_columns, cudaStream_t stream) {
  if (out_end < out_begin || m < 0) return RL_ERR_BAD_ARG;
  ColumnSet cs;
  int st = fill_columns(cs, columns, n_columns, true);
  if (st != RL_OK) return st;
  if (out_end == out_begin) return RL_OK;
  if (m == 0) return RL_ERR_BAD_ARG;
  ExpandArgs a{matched_keys, ls, rs, rc, offs, m, lpos, rpos, out_begin, out_end, lrows_out, rrows_out, nullptr};
  const uint64_t blocks = (out_end - out_begin + kTile - 1) / kTile;
  if (blocks > 0x7fffffffull) return RL_ERR_BAD_ARG;
  expand_kernel<false><<<unsigned(blocks), kThreads, 0, stream>>>(a, cs);
  count_launches(1);
  return rl_cuda_status(cudaGetLastError());
}

int pair_checksum(const uint32_t* ls, const uint32_t* rs, const uint32_t* rc, const uint64_t* offs, int64_t m,
                  const uint32_t* lpos, const uint32_t* rpos, uint64_t out_begin, uint64_t out_end,
                  uint64_t* sum_out, cudaStream_t stream) {
  if (out_end < out_begin || m < 0 || sum_out == nullptr) return RL_ERR_BAD_ARG;
  if (out_end == out_begin) return RL_OK;
  if (m == 0) return RL_ERR_BAD_ARG;
  ExpandArgs a{nullptr, ls, rs, rc, offs, m, lpos, rpos, out_begin, out_end, nullptr, nullptr, sum_out};
  ColumnSet cs;
  cs.n = 0;
  const uint64_t blocks = (out_end - out_begin + kTile - 1) / kTile;
  if (blocks > 0x7fffffffull) return RL_ERR_BAD_ARG;
  expand_kernel<true><<<unsigned(blocks), kThreads, 0, stream>>>(a, cs);
  count_launches(1);
  return rl_cuda_status(cudaGetLastError());
}

// ---------------------------------------------------------------- K7 (sort)
__global__ void __launch_bounds__(kThreads) gather_kernel(const uint32_t* __restrict__ rows, int64_t m,
                                                          ColumnSet cols) {
  for (int64_t t = int64_t(blockIdx.x) * kThreads + threadIdx.x; t < m; t += int64_t(gridDim.x) * kThreads) {
    const uint64_t row = __ldg(rows + t);
    for (int ci = 0; ci < cols.n; ++ci) {
      const rl_column& col = cols.c[ci];
      const int w = col.width;
      copy_row(static_cast<const uint8_t*>(col.src) + row * uint64_t(w), static_cast<uint8_t*>(col.dst) + t * w, w);
    }
  }
}

int gather_rows(const uint32_t* rows, int64_t m, const rl_column* columns, int n_columns, cudaStream_t stream) {
  if (m < 0 || (m > 0 && rows == nullptr)) return RL_ERR_BAD_ARG;
  ColumnSet cs;
  int st = fill_columns(cs, columns, n_columns, false);
  if (st != RL_OK) return st;
  if (m == 0 || n_columns == 0) return RL_OK;
  const int grid = int(std::min<int64_t>((m + kThreads - 1) / kThreads, int64_t(device_sm_count()) * 16));
  gather_kernel<<<grid, kThreads, 0, stream>>>(rows, m, cs);
  count_launches(1);
  return rl_cuda_status(cudaGetLastError());
}

__global__ void widen_kernel(const uint32_t* __restrict__ src, int64_t n, int64_t* __restrict__ dst) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = int64_t(src[i]);
}

int widen_u32(const uint32_t* src, int64_t n, int64_t* dst, cudaStream_t stream) {
  if (n < 0 || (n > 0 && (src == nullptr || dst == nullptr))) return RL_ERR_BAD_ARG;
  if (n == 0) return RL_OK;
  const int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(device_sm_count()) * 16));
  widen_kernel<<<grid, 256, 0, stream>>>(src, n, dst);
  count_launches(1);
  return rl_cuda_status(cudaGetLastError());
}

}  // namespace expand
}  // namespace rl
