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
#ifndef RL_AL_WINDOW
#define RL_AL_WINDOW 2560  // 52 KB of shared memory per CTA: 4 CTAs per SM (3584: 60 KB, 3 per SM; 1e8 join 11.89 -> 11.64 ms)
#endif
constexpr int kAlWindow = RL_AL_WINDOW;  // right keys staged per CTA (larger windows search global memory)

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
  uint32_t* wlo;         // per tile right window [wlo, whi) from align_bounds_kernel (NULL: searched in-tile)
  uint32_t* whi;
};

// The right-key window of every tile, one thread per tile: the two binary
// searches over the right keys (~6 dependent global round trips each) leave
// the tile's own latency chain, and the searches of all tiles overlap. Used
// when the tiles span several waves (1e8 rows: ~31K tiles).
__global__ void __launch_bounds__(kThreads) align_bounds_kernel(AlignArgs a, uint32_t tiles) {
  const uint32_t t = blockIdx.x * kThreads + threadIdx.x;
  if (t >= tiles) return;
  const int64_t dl = *a.d_left;
  const uint32_t dr = uint32_t(*a.d_right);
  const int64_t begin = int64_t(t) * kAlTile;
  if (begin >= dl) return;
  const int64_t end = begin + kAlTile < dl ? begin + kAlTile : dl;
  const int64_t k0 = __ldg(reinterpret_cast<const long long*>(a.lkeys) + begin);
  const int64_t k1 = __ldg(reinterpret_cast<const long long*>(a.lkeys) + end - 1);
  uint32_t lo = 0, len = dr;  // first right key >= k0
  while (len > 0) {
    const uint32_t half = len >> 1;
    if (__ldg(reinterpret_cast<const long long*>(a.rkeys) + lo + half) < k0) {
      lo += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  uint32_t hi = lo;
  len = dr - lo;  // first right key > k1
  while (len > 0) {
    const uint32_t half = len >> 1;
    if (__ldg(reinterpret_cast<const long long*>(a.rkeys) + hi + half) <= k1) {
      hi += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  a.wlo[t] = lo;
  a.whi[t] = hi;
}

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

// Dynamic shared memory of align_kernel.
constexpr size_t kAlSl = 0;                                   // int64 [kAlTile] left keys of the tile
constexpr size_t kAlSr = kAlSl + size_t(kAlTile) * 8;         // int64 [kAlWindow] right window
constexpr size_t kAlMi = kAlSr + size_t(kAlWindow) * 8;       // uint32 [kAlTile] match: tile-local left index
constexpr size_t kAlMj = kAlMi + size_t(kAlTile) * 4;         // uint32 [kAlTile] match: right index
constexpr size_t kAlSmem = kAlMj + size_t(kAlTile) * 4;

// One tile of kAlTile left distinct keys. The matching window of right
// distinct keys is staged, then merge path: thread t takes diagonals
// [t E, (t+1) E) of the merged (left, right) order — one binary search for
// its split, then a sequential walk (a key present on both sides is a
// match) — so the tile costs ~log(window) + E shared reads per thread
// instead of a binary search per key. Matches are listed in shared memory
// in left order, then resolved and written striped (coalesced), with the
// pair prefix from per-round block scans and a two-value look-back.
__global__ void __launch_bounds__(kThreads) align_kernel(AlignArgs a) {
  extern __shared__ __align__(16) uint8_t asmem[];
  int64_t* sl = reinterpret_cast<int64_t*>(asmem + kAlSl);
  int64_t* sr = reinterpret_cast<int64_t*>(asmem + kAlSr);
  uint32_t* mi = reinterpret_cast<uint32_t*>(asmem + kAlMi);
  uint32_t* mj = reinterpret_cast<uint32_t*>(asmem + kAlMj);
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
  if (a.wlo) {
    if (tid == 0) {
      s_lo = __ldg(a.wlo + tile);
      s_hi = __ldg(a.whi + tile);
    }
  } else if (warp == 0) {
    const uint32_t lo = dr ? warp_bound(a.rkeys, 0, dr, a.lkeys[begin], false) : 0;
    if (tid == 0) s_lo = lo;
  } else if (warp == 1) {
    const uint32_t hi = dr ? warp_bound(a.rkeys, 0, dr, a.lkeys[begin + count - 1], true) : 0;
    if ((tid & 31) == 0) s_hi = hi;
  }
  __syncthreads();
  const uint32_t lo = s_lo, hi = max(s_lo, s_hi);
  const uint32_t w = hi - lo;
  const bool staged = w <= uint32_t(kAlWindow);
  if (staged)
    for (uint32_t i = tid; i < w; i += kThreads) sr[i] = __ldg(reinterpret_cast<const long long*>(a.rkeys) + lo + i);
  __syncthreads();

  // ---- phase 1: this thread's matches (count, then list them in order)
  const uint32_t T = uint32_t(count) + (staged ? w : 0u);
  const uint32_t E = (T + kThreads - 1) / kThreads;
  uint32_t d0 = min(uint32_t(tid) * E, T), d1 = min(d0 + E, T);
  uint32_t i0 = 0, j0 = 0;
  if (staged) {
    uint32_t l = d0 > w ? d0 - w : 0u, h = min(d0, uint32_t(count));
    while (l < h) {  // smallest i whose left key comes after right key d0-1-i
      const uint32_t mid = (l + h) >> 1;
      if (sl[mid] <= sr[d0 - 1 - mid]) l = mid + 1;
      else h = mid;
    }
    i0 = l;
    j0 = d0 - l;
  }
  auto walk = [&](auto&& on_match) {
    if (staged) {
      uint32_t i = i0, j = j0;
      for (uint32_t d = d0; d < d1; ++d) {
        if (i < uint32_t(count) && (j >= w || sl[i] <= sr[j])) {
          if (j < w && sl[i] == sr[j]) on_match(i, lo + j);
          ++i;
        } else {
          ++j;
        }
      }
    } else if (hi > lo) {  // window too wide to stage: per-key searches in global memory
      for (int it = 0; it < kAlItems; ++it) {
        const int e = tid * kAlItems + it;
        if (e < count) {
          const uint32_t j = lower_bound_i64(a.rkeys, lo, hi, sl[e]);
          if (j < hi && a.rkeys[j] == sl[e]) on_match(uint32_t(e), j);
        }
      }
    }
  };
  uint32_t my_m = 0;
  walk([&](uint32_t, uint32_t) { ++my_m; });
  uint32_t tot_m;
  uint32_t q = block_exclusive_scan<kThreads>(my_m, warp_m, &tot_m);
  walk([&](uint32_t i, uint32_t j) {
    mi[q] = i;
    mj[q] = j;
    ++q;
  });
  __syncthreads();

  // ---- phase 2: the tile's pair total (for the look-back), striped over matches
  uint64_t my_p = 0;
  for (uint32_t t = tid; t < tot_m; t += kThreads) {
    const uint32_t i = mi[t], j = mj[t];
    my_p += uint64_t(__ldg(a.loff + begin + i + 1) - __ldg(a.loff + begin + i)) *
            uint64_t(__ldg(a.roff + j + 1) - __ldg(a.roff + j));
  }
  uint64_t tot_p;
  block_exclusive_scan<kThreads>(my_p, warp_p, &tot_p);
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

  // ---- phase 3: resolve and write the matches, striped (coalesced), the
  // pair prefix carried across rounds of kThreads matches
  uint64_t pairs_base = s_excl_p;
  const uint64_t mbase = s_excl_m;
  for (uint32_t r0 = 0; r0 < tot_m; r0 += kThreads) {
    const uint32_t t = r0 + tid;
    uint32_t l0 = 0, lcount = 0, rr0 = 0, rcount = 0, i = 0;
    if (t < tot_m) {
      i = mi[t];
      const uint32_t j = mj[t];
      l0 = __ldg(a.loff + begin + i);
      lcount = __ldg(a.loff + begin + i + 1) - l0;
      rr0 = __ldg(a.roff + j);
      rcount = __ldg(a.roff + j + 1) - rr0;
    }
    const uint64_t p = uint64_t(lcount) * uint64_t(rcount);
    uint64_t round_total;
    const uint64_t pre = block_exclusive_scan<kThreads>(p, warp_p, &round_total);
    if (t < tot_m) {
      const uint64_t o = mbase + t;
      a.matched_keys[o] = sl[i];
      a.ls[o] = l0;
      a.lc[o] = lcount;
      a.rs[o] = rr0;
      a.rc[o] = rcount;
      a.pair_offsets[o] = pairs_base + pre;
    }
    pairs_base += round_total;
    __syncthreads();  // warp_p reuse by the next round's scan
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
  c.take<uint32_t>(tiles);
  c.take<uint32_t>(tiles);
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
  a.wlo = c.take<uint32_t>(tiles);
  a.whi = c.take<uint32_t>(tiles);
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
  static int attr[kMaxDevices] = {};  // per device: 1 = opted in, -1 = refused
  if (per_device(attr, [] {
        if (cudaFuncSetAttribute(align_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kAlSmem)) ==
            cudaSuccess)
          return 1;
        cudaGetLastError();
        return -1;
      }) < 0)
    return rl_cuda_status(cudaErrorInvalidConfiguration);
  // window pre-pass when the tiles span more than ~4 waves (3 CTAs per SM)
  const char* force = getenv("RL_ALIGN_PREPASS");  // "1" / "0": force on / off (tests, A/B)
  const bool prepass = force && force[0] ? force[0] == '1' : tiles > uint32_t(device_sm_count()) * 12;
  if (prepass) {
    align_bounds_kernel<<<(tiles + kThreads - 1) / kThreads, kThreads, 0, stream>>>(a, tiles);
  } else {
    a.wlo = a.whi = nullptr;
  }
  align_kernel<<<tiles, kThreads, kAlSmem, stream>>>(a);
  count_launches(prepass ? 2 : 1);
  return rl_cuda_status(cudaGetLastError());
}

}  // namespace keyaxis
}  // namespace rl
