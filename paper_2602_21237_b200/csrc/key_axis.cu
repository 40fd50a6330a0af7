// key_axis.cu — K3 run bounds, K4+K5 key-axis alignment + join sizing.
//
//   K3  replaces tensorpath.py:84-92   (flatnonzero of key changes,
//       key_values = sk[bounds], offsets = concat(bounds, [n]))
//   K4  replaces tensorpath.py:109-128 (searchsorted(b, a), mask, compact)
//   K5  replaces tensorpath.py:149-161 (per_key = lc * rc, cumsum, total)
//
// Both are single-pass decoupled look-back compactions (warp-parallel
// look-back: 32 predecessor tiles per round trip): one read of the input,
// one write of the compacted output, the device-side totals (D, M, total
// pairs) written by the last tile, so the host never waits between
// to_tensor, key_axis_align and the sizing pass.
//
// K4 is a tiled merge: a CTA stages 2048 consecutive left distinct keys,
// finds the matching window of right distinct keys with two warp-parallel
// 32-ary searches (4 round trips for ~1e6 keys instead of 20 dependent
// loads per key), stages that window in shared memory and searches it there.
#include <algorithm>

#include "common.cuh"

namespace rl {
namespace keyaxis {

constexpr int kThreads = 256;
constexpr int kRbItems = 16;
constexpr int kRbTile = kThreads * kRbItems;
constexpr int kAlItems = 8;
constexpr int kAlTile = kThreads * kAlItems;
constexpr int kAlWindow = 3584;  // right keys staged per CTA (larger windows search global memory)

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

  // warp w owns the 512 consecutive elements [512 w, 512 w + 512), 32 per
  // round (conflict-free 8-byte reads); run heads by ballot, so each round
  // writes its heads to consecutive slots (coalesced)
  constexpr int kSeg = 32 * kRbItems;
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t lt = lanemask_lt();
  uint32_t bal[kRbItems];
  uint32_t c = 0;
#pragma unroll
  for (int it = 0; it < kRbItems; ++it) {
    const int e = warp * kSeg + it * 32 + lane;
    const bool head = e < count && ((begin + e == 0) || (stage[e + 1] != stage[e]));
    bal[it] = __ballot_sync(0xffffffffu, head);
    c += __popc(bal[it]);
  }
  if (lane == 0) warp_sums[warp] = c;
  __syncthreads();
  if (tid < 32) {
    const uint32_t v = tid < kThreads / 32 ? warp_sums[tid] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (tid >= o) incl += x;
    }
    const uint32_t tile_total = __shfl_sync(0xffffffffu, incl, kThreads / 32 - 1);
    if (tid < kThreads / 32) warp_sums[tid] = incl - v;  // exclusive warp offsets
    if (tile == 0) {
      if (tid == 0) st_relaxed(&status[0], pack_status(kFlagIncl, 1, tile_total));
      if (tid == 0) s_excl = 0;
    } else {
      if (tid == 0) st_relaxed(&status[tile], pack_status(kFlagAgg, 1, tile_total));
      const uint64_t excl = warp_lookback(status, tile, 1);
      if (tid == 0) {
        st_relaxed(&status[tile], pack_status(kFlagIncl, 1, excl + tile_total));
        s_excl = excl;
      }
    }
    if (tid == 0) warp_sums[kThreads / 32] = tile_total;
  }
  __syncthreads();
  const uint32_t tile_total = warp_sums[kThreads / 32];
  uint64_t pos = s_excl + warp_sums[warp];
#pragma unroll
  for (int it = 0; it < kRbItems; ++it) {
    const int e = warp * kSeg + it * 32 + lane;
    if (bal[it] & (1u << lane)) {
      const uint64_t o = pos + __popc(bal[it] & lt);
      key_values[o] = stage[e + 1];
      offsets[o] = uint32_t(begin + e);
    }
    pos += __popc(bal[it]);
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
// first index in a[lo, hi) with a[i] >= x (strict = false) or a[i] > x
// (strict = true); one warp, 32 probes per round trip.
__device__ __forceinline__ uint32_t warp_bound(const int64_t* __restrict__ a, uint32_t lo, uint32_t hi, int64_t x,
                                               bool strict) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t idx = lo + uint32_t(lane) * step;
    bool pred = false;
    if (idx < hi) {
      const int64_t v = __ldg(reinterpret_cast<const long long*>(a) + idx);
      pred = strict ? v <= x : v < x;
    }
    const uint32_t c = __popc(__ballot_sync(0xffffffffu, pred));
    const uint32_t nlo = c == 0 ? lo : lo + (c - 1) * step + 1;
    const uint32_t nhi = min(hi, lo + c * step);
    lo = nlo;
    hi = nhi;
  }
  bool pred = false;
  if (lo + lane < hi) {
    const int64_t v = __ldg(reinterpret_cast<const long long*>(a) + lo + lane);
    pred = strict ? v <= x : v < x;
  }
  return lo + __popc(__ballot_sync(0xffffffffu, pred));
}

__device__ __forceinline__ uint32_t lower_bound_i64(const int64_t* a, uint32_t lo, uint32_t hi, int64_t key) {
  uint32_t len = hi - lo;
  while (len > 0) {
    const uint32_t half = len >> 1;
    if (a[lo + half] < key) {
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

// Two-value warp look-back: matches packed in the status word, pairs in a
// side array published before the flag (release) and read after it (acquire).
__device__ __forceinline__ void warp_lookback2(const AlignArgs& a, uint32_t tile, uint64_t* excl_m,
                                               uint64_t* excl_p) {
  const int lane = threadIdx.x & 31;
  uint64_t em = 0, ep = 0;
  int64_t base = int64_t(tile) - 1;
  while (true) {
    const int64_t p = base - lane;
    uint64_t s = kFlagIncl;  // virtual tile -1: inclusive zero
    uint64_t pv = 0;
    if (p >= 0) {
      s = ld_acquire(&a.status[p]);
      if ((s & kFlagMask) == kFlagIncl) pv = ld_relaxed(&a.incl_pairs[p]);
      else if ((s & kFlagMask) == kFlagAgg) pv = ld_relaxed(&a.agg_pairs[p]);
    }
    const bool ready = (s & kFlagMask) != 0;
    const uint32_t incl = __ballot_sync(0xffffffffu, ready && (s & kFlagMask) == kFlagIncl);
    const uint32_t notready = __ballot_sync(0xffffffffu, !ready);
    const int stop = incl ? __ffs(incl) - 1 : 31;
    const uint32_t need = stop == 31 ? 0xffffffffu : ((2u << stop) - 1u);
    if (notready & need) {
      __nanosleep(32);
      continue;
    }
    uint64_t vm = lane <= stop ? (s & kValueMask) : 0;
    uint64_t vp = lane <= stop ? pv : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      vm += __shfl_xor_sync(0xffffffffu, vm, o);
      vp += __shfl_xor_sync(0xffffffffu, vp, o);
    }
    em += vm;
    ep += vp;
    if (incl) break;
    base -= 32;
  }
  *excl_m = em;
  *excl_p = ep;
}

__global__ void __launch_bounds__(kThreads) align_kernel(AlignArgs a) {
  __shared__ int64_t sl[kAlTile];        // this tile's left distinct keys
  __shared__ int64_t sr[kAlWindow];      // the matching window of right distinct keys
  __shared__ uint32_t warp_m[kThreads / 32 + 1];
  __shared__ uint64_t warp_p[kThreads / 32 + 1];
  __shared__ uint32_t s_tile, s_lo, s_hi;
  __shared__ uint64_t s_excl_m, s_excl_p;
  const int tid = threadIdx.x, warp = tid >> 5;
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
  const int count = dl - begin < kAlTile ? int(dl - begin) : kAlTile;
  const bool last = begin + kAlTile >= dl;
  for (int i = tid; i < count; i += kThreads) sl[i] = __ldg(reinterpret_cast<const long long*>(a.lkeys) + begin + i);
  // right window [lo, hi): keys in [first left key, last left key]
  if (warp == 0) {
    const uint32_t lo = dr ? warp_bound(a.rkeys, 0, dr, a.lkeys[begin], false) : 0;
    if (tid == 0) s_lo = lo;
  } else if (warp == 1) {
    const uint32_t hi = dr ? warp_bound(a.rkeys, 0, dr, a.lkeys[begin + count - 1], true) : 0;
    if ((tid & 31) == 0) s_hi = hi;
  }
  __syncthreads();
  const uint32_t lo = s_lo, hi = max(s_lo, s_hi);
  const bool staged = hi - lo <= uint32_t(kAlWindow);
  if (staged)
    for (uint32_t i = tid; i < hi - lo; i += kThreads) sr[i] = __ldg(reinterpret_cast<const long long*>(a.rkeys) + lo + i);
  __syncthreads();

  uint32_t match_bits = 0, my_m = 0;
  uint64_t my_p = 0;
  uint32_t rj[kAlItems];
  uint32_t lcnt[kAlItems], rcnt[kAlItems];
  uint32_t from = 0;  // search start inside the window (this thread's keys increase)
#pragma unroll
  for (int it = 0; it < kAlItems; ++it) {
    const int e = tid * kAlItems + it;
    rj[it] = 0;
    lcnt[it] = rcnt[it] = 0;
    if (e < count && hi > lo) {
      const int64_t key = sl[e];
      uint32_t j;
      bool hit;
      if (staged) {
        j = lower_bound_i64(sr, from, hi - lo, key);
        hit = j < hi - lo && sr[j] == key;
        from = j;
        j += lo;
      } else {
        j = lower_bound_i64(a.rkeys, lo, hi, key);
        hit = j < hi && a.rkeys[j] == key;
      }
      if (hit) {
        match_bits |= 1u << it;
        rj[it] = j;
        lcnt[it] = a.loff[begin + e + 1] - a.loff[begin + e];
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

  if (warp == 0) {
    uint64_t excl_m = 0, excl_p = 0;
    if (tile == 0) {
      if (tid == 0) {
        a.incl_pairs[0] = tot_p;
        st_release(&a.status[0], pack_status(kFlagIncl, 1, tot_m));
      }
    } else {
      if (tid == 0) {
        a.agg_pairs[tile] = tot_p;
        st_release(&a.status[tile], pack_status(kFlagAgg, 1, tot_m));
      }
      warp_lookback2(a, tile, &excl_m, &excl_p);
      if (tid == 0) {
        a.incl_pairs[tile] = excl_p + tot_p;
        st_release(&a.status[tile], pack_status(kFlagIncl, 1, excl_m + tot_m));
      }
    }
    if (tid == 0) {
      s_excl_m = excl_m;
      s_excl_p = excl_p;
    }
  }
  __syncthreads();
  uint64_t pos = s_excl_m + off_m;
  uint64_t pairs = s_excl_p + off_p;
#pragma unroll
  for (int it = 0; it < kAlItems; ++it) {
    if (match_bits & (1u << it)) {
      const int e = tid * kAlItems + it;
      a.matched_keys[pos] = sl[e];
      a.ls[pos] = a.loff[begin + e];
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
