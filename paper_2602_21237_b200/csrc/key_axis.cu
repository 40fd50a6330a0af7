// key_axis.cu — K3 run bounds, K4+K5 key-axis alignment + join sizing.
//
//   K3  replaces tensorpath.py:84-92   (flatnonzero of key changes,
//       key_values = sk[bounds], offsets = concat(bounds, [n]))
//   K4  replaces tensorpath.py:109-128 (searchsorted(b, a), mask, compact)
//   K5  replaces tensorpath.py:149-161 (per_key = lc * rc, cumsum, total)
//
// Both are single-pass decoupled look-back compactions: one read of the
// input, one write of the compacted output, the device-side totals (D, M,
// total pairs) written by the last tile, so the host never waits between
// to_tensor, key_axis_align and the sizing pass.
#include <algorithm>

#include "common.cuh"

namespace rl {
namespace keyaxis {

constexpr int kThreads = 256;
constexpr int kRbItems = 16;
constexpr int kRbTile = kThreads * kRbItems;
constexpr int kAlItems = 8;
constexpr int kAlTile = kThreads * kAlItems;

// ---------------------------------------------------------------- K3
__global__ void __launch_bounds__(kThreads) run_bounds_kernel(const int64_t* __restrict__ sk, int64_t n,
                                                              int64_t* __restrict__ key_values,
                                                              uint32_t* __restrict__ offsets,
                                                              int64_t* __restrict__ d_out, uint32_t* counter,
                                                              uint64_t* status, uint32_t num_tiles) {
  __shared__ int64_t stage[kRbTile + 1];
  __shared__ uint32_t warp_sums[kThreads / 32 + 1];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_excl;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t begin = int64_t(tile) * kRbTile;
  const int64_t left = n - begin;
  const int count = left < kRbTile ? int(left) : kRbTile;

  // coalesced striped load into shared memory (+ the predecessor key)
  for (int i = tid; i < count; i += kThreads) stage[i + 1] = __ldcs(reinterpret_cast<const long long*>(sk) + begin + i);
  if (tid == 0) stage[0] = begin > 0 ? sk[begin - 1] : 0;
  __syncthreads();

  // blocked ownership: thread owns elements [tid*items, tid*items+items)
  uint32_t flags = 0, c = 0;
#pragma unroll
  for (int it = 0; it < kRbItems; ++it) {
    const int e = tid * kRbItems + it;
    if (e < count) {
      const bool head = (begin + e == 0) || (stage[e + 1] != stage[e]);
      flags |= uint32_t(head) << it;
      c += head;
    }
  }
  uint32_t tile_total;
  const uint32_t off = block_exclusive_scan<kThreads>(c, warp_sums, &tile_total);
  if (tid == 0) s_excl = lookback_publish(status, tile, 1, tile_total);
  __syncthreads();
  const uint64_t base = s_excl + off;
  uint32_t k = 0;
#pragma unroll
  for (int it = 0; it < kRbItems; ++it) {
    if (flags & (1u << it)) {
      const int e = tid * kRbItems + it;
      key_values[base + k] = stage[e + 1];
      offsets[base + k] = uint32_t(begin + e);
      ++k;
    }
  }
  if (tile == num_tiles - 1 && tid == 0) {
    const uint64_t d = s_excl + tile_total;
    *d_out = int64_t(d);
    offsets[d] = uint32_t(n);
  }
}

__global__ void empty_bounds_kernel(uint32_t* offsets, int64_t* d_out) {
  offsets[0] = 0;
  *d_out = 0;
}

size_t run_bounds_workspace_bytes(int64_t n) {
  const size_t tiles = size_t((std::max<int64_t>(n, 1) + kRbTile - 1) / kRbTile);
  CarveSize c;
  c.take<uint32_t>(1);
  c.take<uint64_t>(tiles);
  return c.used + 256;
}

int run_bounds(const int64_t* sk, int64_t n, int64_t* key_values, uint32_t* offsets, int64_t* d_out, void* ws,
               size_t ws_bytes, cudaStream_t stream) {
  if (n < 0 || offsets == nullptr || d_out == nullptr) return RL_ERR_BAD_ARG;
  if (n > RL_MAX_ROWS) return RL_ERR_TOO_MANY_ROWS;
  if (n == 0) {
    empty_bounds_kernel<<<1, 1, 0, stream>>>(offsets, d_out);
    count_launches(1);
    return rl_cuda_status(cudaGetLastError());
  }
  const uint32_t tiles = uint32_t((n + kRbTile - 1) / kRbTile);
  Carve c{static_cast<char*>(ws), ws_bytes};
  uint32_t* counter = c.take<uint32_t>(1);
  uint64_t* status = c.take<uint64_t>(tiles);
  if (!c.ok) return RL_ERR_WORKSPACE;
  cudaError_t e = cudaMemsetAsync(ws, 0, c.used, stream);
  if (e != cudaSuccess) return rl_cuda_status(e);
  run_bounds_kernel<<<tiles, kThreads, 0, stream>>>(sk, n, key_values, offsets, d_out, counter, status, tiles);
  count_launches(1);
  return rl_cuda_status(cudaGetLastError());
}

// ---------------------------------------------------------------- K4+K5
__device__ __forceinline__ uint32_t lower_bound_i64(const int64_t* __restrict__ a, uint32_t n, int64_t key) {
  uint32_t lo = 0, len = n;
  while (len > 0) {
    const uint32_t half = len >> 1;
    const int64_t v = __ldg(reinterpret_cast<const long long*>(a) + lo + half);
    if (v < key) {
      lo += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  return lo;
}

struct AlignArgs {
  const int64_t* lkeys;
  const uint32_t* loff;
  const int64_t* d_left;
  const int64_t* rkeys;
  const uint32_t* roff;
  const int64_t* d_right;
  int64_t* matched_keys;
  uint32_t* ls;
  uint32_t* lc;
  uint32_t* rs;
  uint32_t* rc;
  uint64_t* pair_offsets;
  int64_t* m_out;
  uint64_t* total_out;
  uint32_t* counter;
  uint64_t* status;      // packed flag | epoch | matches
  uint64_t* agg_pairs;   // per tile aggregate pairs (valid when flag >= AGG)
  uint64_t* incl_pairs;  // per tile inclusive pairs (valid when flag == INCL)
};

__global__ void __launch_bounds__(kThreads) align_kernel(AlignArgs a) {
  __shared__ uint32_t warp_m[kThreads / 32 + 1];
  __shared__ uint64_t warp_p[kThreads / 32 + 1];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_excl_m, s_excl_p;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(a.counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t dl = *a.d_left;
  const uint32_t dr = uint32_t(*a.d_right);
  const int64_t begin = int64_t(tile) * kAlTile;
  if (begin >= dl) {
    if (tile == 0 && tid == 0) {  // D_left == 0: empty alignment
      *a.m_out = 0;
      *a.total_out = 0;
      a.pair_offsets[0] = 0;
    }
    return;
  }
  const bool last = begin + kAlTile >= dl;

  uint32_t match_bits = 0, my_m = 0;
  uint64_t my_p = 0;
  uint32_t rj[kAlItems];
  uint32_t lcnt[kAlItems], rcnt[kAlItems];
#pragma unroll
  for (int it = 0; it < kAlItems; ++it) {
    const int64_t i = begin + tid * kAlItems + it;
    rj[it] = 0;
    lcnt[it] = rcnt[it] = 0;
    if (i < dl && dr > 0) {
      const int64_t key = a.lkeys[i];
      const uint32_t j = lower_bound_i64(a.rkeys, dr, key);
      if (j < dr && a.rkeys[j] == key) {
        match_bits |= 1u << it;
        rj[it] = j;
        lcnt[it] = a.loff[i + 1] - a.loff[i];
        rcnt[it] = a.roff[j + 1] - a.roff[j];
        ++my_m;
        my_p += uint64_t(lcnt[it]) * uint64_t(rcnt[it]);
      }
    }
  }
  uint32_t tot_m;
  uint64_t tot_p;
  const uint32_t off_m = block_exclusive_scan<kThreads>(my_m, warp_m, &tot_m);
  const uint64_t off_p = block_exclusive_scan<kThreads>(my_p, warp_p, &tot_p);

  if (tid == 0) {
    uint64_t excl_m = 0, excl_p = 0;
    if (tile == 0) {
      a.incl_pairs[0] = tot_p;
      st_release(&a.status[0], pack_status(kFlagIncl, 1, tot_m));
    } else {
      a.agg_pairs[tile] = tot_p;
      st_release(&a.status[tile], pack_status(kFlagAgg, 1, tot_m));
      int64_t p = int64_t(tile) - 1;
      while (true) {
        const uint64_t s = ld_acquire(&a.status[p]);
        const uint64_t f = s & kFlagMask;
        if (f == 0) continue;
        excl_m += s & kValueMask;
        if (f == kFlagIncl) {
          excl_p += ld_relaxed(&a.incl_pairs[p]);
          break;
        }
        excl_p += ld_relaxed(&a.agg_pairs[p]);
        --p;
      }
      a.incl_pairs[tile] = excl_p + tot_p;
      st_release(&a.status[tile], pack_status(kFlagIncl, 1, excl_m + tot_m));
    }
    s_excl_m = excl_m;
    s_excl_p = excl_p;
  }
  __syncthreads();
  uint64_t pos = s_excl_m + off_m;
  uint64_t pairs = s_excl_p + off_p;
#pragma unroll
  for (int it = 0; it < kAlItems; ++it) {
    if (match_bits & (1u << it)) {
      const int64_t i = begin + tid * kAlItems + it;
      a.matched_keys[pos] = a.lkeys[i];
      a.ls[pos] = a.loff[i];
      a.lc[pos] = lcnt[it];
      a.rs[pos] = a.roff[rj[it]];
      a.rc[pos] = rcnt[it];
      a.pair_offsets[pos] = pairs;
      pairs += uint64_t(lcnt[it]) * uint64_t(rcnt[it]);
      ++pos;
    }
  }
  if (last && tid == 0) {
    const uint64_t m = s_excl_m + tot_m, total = s_excl_p + tot_p;
    *a.m_out = int64_t(m);
    *a.total_out = total;
    a.pair_offsets[m] = total;
  }
}

__global__ void empty_align_kernel(uint64_t* pair_offsets, int64_t* m_out, uint64_t* total_out) {
  pair_offsets[0] = 0;
  *m_out = 0;
  *total_out = 0;
}

size_t align_workspace_bytes(int64_t cap) {
  const size_t tiles = size_t((std::max<int64_t>(cap, 1) + kAlTile - 1) / kAlTile);
  CarveSize c;
  c.take<uint32_t>(1);
  c.take<uint64_t>(tiles);
  c.take<uint64_t>(tiles);
  c.take<uint64_t>(tiles);
  return c.used + 256;
}

int key_axis_align(const int64_t* lkeys, const uint32_t* loff, const int64_t* d_left, int64_t cap,
                   const int64_t* rkeys, const uint32_t* roff, const int64_t* d_right, int64_t* matched_keys,
                   uint32_t* ls, uint32_t* lc, uint32_t* rs, uint32_t* rc, uint64_t* pair_offsets,
                   int64_t* m_out, uint64_t* total_out, void* ws, size_t ws_bytes, cudaStream_t stream) {
  if (cap < 0 || pair_offsets == nullptr || m_out == nullptr || total_out == nullptr) return RL_ERR_BAD_ARG;
  if (cap > RL_MAX_ROWS) return RL_ERR_TOO_MANY_ROWS;
  if (cap == 0) {
    empty_align_kernel<<<1, 1, 0, stream>>>(pair_offsets, m_out, total_out);
    count_launches(1);
    return rl_cuda_status(cudaGetLastError());
  }
  const uint32_t tiles = uint32_t((cap + kAlTile - 1) / kAlTile);
  Carve c{static_cast<char*>(ws), ws_bytes};
  AlignArgs a;
  a.counter = c.take<uint32_t>(1);
  a.status = c.take<uint64_t>(tiles);
  const size_t zero = c.used;
  a.agg_pairs = c.take<uint64_t>(tiles);
  a.incl_pairs = c.take<uint64_t>(tiles);
  if (!c.ok) return RL_ERR_WORKSPACE;
  cudaError_t e = cudaMemsetAsync(ws, 0, zero, stream);
  if (e != cudaSuccess) return rl_cuda_status(e);
  a.lkeys = lkeys;
  a.loff = loff;
  a.d_left = d_left;
  a.rkeys = rkeys;
  a.roff = roff;
  a.d_right = d_right;
  a.matched_keys = matched_keys;
  a.ls = ls;
  a.lc = lc;
  a.rs = rs;
  a.rc = rc;
  a.pair_offsets = pair_offsets;
  a.m_out = m_out;
  a.total_out = total_out;
  align_kernel<<<tiles, kThreads, 0, stream>>>(a);
  count_launches(1);
  return rl_cuda_status(cudaGetLastError());
}

}  // namespace keyaxis
}  // namespace rl
