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
#include <cstdlib>

#include "common.cuh"

namespace rl {
namespace expand {

constexpr int kThreads = 256;
#ifndef RL_EXPAND_ITEMS
#define RL_EXPAND_ITEMS 4
#endif
constexpr int kItems = RL_EXPAND_ITEMS;
#ifndef RL_EXPAND_MIN_BLOCKS
#define RL_EXPAND_MIN_BLOCKS 4
#endif
constexpr int kTile = kThreads * kItems;

// last index g in [0, m] with offs[g] <= t (offs is non-decreasing,
// offs[0] = 0 <= t); one warp, 32 probes per round trip.
__device__ __forceinline__ int64_t warp_last_le(const uint64_t* __restrict__ offs, int64_t lo, int64_t m,
                                                uint64_t t) {
  const int lane = threadIdx.x & 31;
  int64_t hi = m + 1;  // answer + 1 = first index with offs[i] > t, in [lo, hi]; offs[lo] <= t
  {  // gallop: the answer is usually within 32 keys of the hint (consecutive output tiles)
    const bool pred = lo + lane < hi && __ldg(reinterpret_cast<const unsigned long long*>(offs) + lo + lane) <= t;
    const uint32_t bal = __ballot_sync(0xffffffffu, pred);
    if (bal != 0xffffffffu) return lo + __popc(bal) - 1;
    lo += 31;
  }
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t idx = lo + int64_t(lane) * step;
    const bool pred = idx < hi && __ldg(reinterpret_cast<const unsigned long long*>(offs) + idx) <= t;
    const int64_t c = __popc(__ballot_sync(0xffffffffu, pred));
    const int64_t nlo = c == 0 ? lo : lo + (c - 1) * step + 1;
    const int64_t nhi = min(hi, lo + c * step);
    lo = nlo;
    hi = nhi;
  }
  const bool pred = lo + lane < hi && __ldg(reinterpret_cast<const unsigned long long*>(offs) + lo + lane) <= t;
  return lo + __popc(__ballot_sync(0xffffffffu, pred)) - 1;
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

// Gather one column for this thread's items: all loads first, then all
// stores, so the kItems random reads are in flight together.
template <typename T>
__device__ __forceinline__ void gather_items(const rl_column& col, const uint32_t (&row)[kItems], uint64_t o0,
                                             uint32_t valid) {
  const T* src = static_cast<const T*>(col.src);
  T* dst = static_cast<T*>(col.dst) + o0;  // item it writes dst[it * kThreads]
  T v[kItems];
#pragma unroll
  for (int it = 0; it < kItems; ++it)
    if (valid & (1u << it)) v[it] = ld_row(src + row[it]);
#pragma unroll
  for (int it = 0; it < kItems; ++it)
    if (valid & (1u << it)) __stcs(dst + it * kThreads, v[it]);
}

__device__ __forceinline__ void gather_column(const rl_column& col, const uint32_t (&row)[kItems], uint64_t o0,
                                              uint32_t valid) {
  const int w = col.width;
  if (w == 8) {
    gather_items<unsigned long long>(col, row, o0, valid);
  } else if (w == 4) {
    gather_items<unsigned int>(col, row, o0, valid);
  } else if (w == 16) {
    gather_items<uint4>(col, row, o0, valid);
  } else {
#pragma unroll 1
    for (int it = 0; it < kItems; ++it)
      if (valid & (1u << it))
        copy_row(static_cast<const uint8_t*>(col.src) + uint64_t(row[it]) * w,
                 static_cast<uint8_t*>(col.dst) + (o0 + uint64_t(it) * kThreads) * uint64_t(w), w);
  }
}

// Output-space load-balanced expansion. Each CTA owns kTile consecutive
// output pairs; it locates its window of matched keys with two warp-parallel
// searches and stages the window's pair offsets and per-key starts/counts in
// shared memory. Each thread then resolves its kItems pairs in phases —
// window search, row-id loads, column loads, stores — so the dependent
// global reads of all its pairs overlap instead of running one pair at a time.
template <bool kChecksum>
__global__ void __launch_bounds__(kThreads, RL_EXPAND_MIN_BLOCKS) expand_kernel(ExpandArgs a, ColumnSet cols,
                                                                               uint32_t tiles_per_cta) {
  __shared__ uint64_t so[kTile + 1];
  __shared__ uint32_t sls[kTile], srs[kTile], src_[kTile];
  __shared__ int64_t s_g[2];
  const int tid = threadIdx.x, warp = tid >> 5;
  uint64_t sum = 0;  // checksum mode
  int64_t hint = 0;  // the next sub-tile's first key is at or after this one's last
  bool reuse = false;  // the first tile's key window = the streaming check's search

  // ---- streaming mode: the CTA's whole output range is covered by few heavy
  // keys (>= 1024 pairs per key on average, e.g. the Zipf head of BASELINE
  // cfg3). Each key's block of lc x rc pairs is walked with a
  // division-free (li, ri) stride, no shared-memory staging, no barriers.
  {
    const uint64_t c0 = a.out_begin + uint64_t(blockIdx.x) * tiles_per_cta * kTile;
    const uint64_t c1 = min(c0 + uint64_t(tiles_per_cta) * kTile, a.out_end);
    if (warp < 2) {
      const int64_t g = warp_last_le(a.offs, 0, a.m, warp == 0 ? c0 : c1 - 1);
      if ((tid & 31) == 0) s_g[warp] = g;
    }
    __syncthreads();
    const int64_t ga = s_g[0], gb = s_g[1];
    hint = ga;
    if (uint64_t(gb - ga + 1) * kTile <= c1 - c0) {
      for (int64_t g = ga; g <= gb; ++g) {
        const uint64_t kbeg = __ldg(reinterpret_cast<const unsigned long long*>(a.offs) + g);
        const uint64_t kend = __ldg(reinterpret_cast<const unsigned long long*>(a.offs) + g + 1);
        const uint64_t s0 = max(kbeg, c0), s1 = min(kend, c1);
        const uint32_t c = __ldg(a.rc + g);
        const uint32_t* lp = a.lpos + __ldg(a.ls + g);
        const uint32_t* rp = a.rpos + __ldg(a.rs + g);
        if (!kChecksum && cols.n == 0 && a.lrows_out && a.rrows_out && s1 - s0 >= 8 * kThreads) {
          // pairs only (cfg3 materialisation): 4 consecutive outputs per thread
          // per step, one 16-byte store per row-id array (scalar head / tail)
          const uint64_t oa = s0 - a.out_begin;
          const uint64_t head = (4 - (oa & 3)) & 3;  // outputs before the first 16-byte boundary
          auto scalar_at = [&](uint64_t u) {
            const uint64_t local = u - kbeg;
            const uint64_t li = local / c;
            const uint32_t ri = uint32_t(local - li * c);
            __stcs(a.lrows_out + (u - a.out_begin), __ldg(lp + li));
            __stcs(a.rrows_out + (u - a.out_begin), __ldg(rp + ri));
          };
          if (tid < head) scalar_at(s0 + tid);
          const uint64_t v0 = s0 + head;                   // first vector output
          const uint64_t nvec = (s1 - v0) / 4;             // whole 4-output groups
          const uint64_t tail0 = v0 + nvec * 4;
          if (tid < s1 - tail0) scalar_at(tail0 + tid);
          uint64_t u = v0 + uint64_t(tid) * 4;
          if (u < tail0) {
            const uint64_t local = u - kbeg;
            uint64_t li = local / c;
            uint32_t ri = uint32_t(local - li * c);
            constexpr uint32_t kStep = 4 * kThreads;
            const uint32_t q = kStep / c, r = kStep % c;
            for (; u < tail0; u += kStep) {
              uint32_t lv[4], rv[4];
              uint64_t li2 = li;
              uint32_t ri2 = ri;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                lv[e] = __ldg(lp + li2);
                rv[e] = __ldg(rp + ri2);
                if (++ri2 == c) {
                  ri2 = 0;
                  ++li2;
                }
              }
              const uint64_t o = u - a.out_begin;
              __stcs(reinterpret_cast<uint4*>(a.lrows_out + o), make_uint4(lv[0], lv[1], lv[2], lv[3]));
              __stcs(reinterpret_cast<uint4*>(a.rrows_out + o), make_uint4(rv[0], rv[1], rv[2], rv[3]));
              li += q;
              ri += r;
              if (ri >= c) {
                ri -= c;
                ++li;
              }
            }
          }
          continue;
        }
        const uint64_t t = s0 + tid;
        if (t >= s1) continue;
        const uint64_t local = t - kbeg;
        uint64_t li = local / c;
        uint32_t ri = uint32_t(local - li * c);
        const uint32_t q = uint32_t(kThreads) / c, r = uint32_t(kThreads) % c;
        for (uint64_t u = t; u < s1; u += kThreads) {
          const uint32_t lrow = __ldg(lp + li), rrow = __ldg(rp + ri);
          if (kChecksum) {
            sum += fmix64((uint64_t(lrow) << 32) | rrow);
          } else {
            const uint64_t o = u - a.out_begin;
            if (a.lrows_out) __stcs(a.lrows_out + o, lrow);
            if (a.rrows_out) __stcs(a.rrows_out + o, rrow);
            for (int ci = 0; ci < cols.n; ++ci) {
              const rl_column& col = cols.c[ci];
              const int w = col.width;
              uint8_t* dst = static_cast<uint8_t*>(col.dst) + o * uint64_t(w);
              if (col.side == RL_SIDE_KEY)
                __stcs(reinterpret_cast<long long*>(dst), (long long)__ldg(reinterpret_cast<const long long*>(a.matched_keys) + g));
              else
                copy_row(static_cast<const uint8_t*>(col.src) + uint64_t(col.side == RL_SIDE_LEFT ? lrow : rrow) * w, dst, w);
            }
          }
          li += q;
          ri += r;
          if (ri >= c) {
            ri -= c;
            ++li;
          }
        }
      }
      tiles_per_cta = 0;  // skip the tile loop
    }
    // a one-tile CTA's tile is the range just searched: reuse [ga, gb]
    reuse = tiles_per_cta == 1 && c1 - c0 <= uint64_t(kTile);
    __syncthreads();
  }

  for (uint32_t sub = 0; sub < tiles_per_cta; ++sub) {
  const uint64_t t0 = a.out_begin + (uint64_t(blockIdx.x) * tiles_per_cta + sub) * kTile;
  if (t0 >= a.out_end) break;
  const uint64_t t1 = min(t0 + kTile, a.out_end);
  if (warp < 2 && !(reuse && sub == 0)) {
    const int64_t g = warp_last_le(a.offs, hint, a.m, warp == 0 ? t0 : t1 - 1);
    if ((tid & 31) == 0) s_g[warp] = g;
  }
  __syncthreads();
  const int64_t g0 = s_g[0];
  hint = s_g[1];
  const int nk = int(s_g[1] - g0) + 1;  // <= kTile: every matched key owns >= 1 pair
  for (int i = tid; i <= nk; i += kThreads) so[i] = a.offs[g0 + i];
  for (int i = tid; i < nk; i += kThreads) {
    sls[i] = __ldg(a.ls + g0 + i);
    srs[i] = __ldg(a.rs + g0 + i);
    src_[i] = __ldg(a.rc + g0 + i);
  }
  __syncthreads();

  // phase 1: window slot of each pair (binary search in shared memory)
  uint32_t kk[kItems], lrow[kItems], rrow[kItems];
  const uint64_t o0 = t0 + tid - a.out_begin;  // output index of item 0; item it is o0 + it * kThreads
  uint32_t valid = 0;
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const uint64_t t = t0 + uint64_t(it) * kThreads + tid;
    kk[it] = 0;
    if (t < t1) {
      valid |= 1u << it;
      if (nk == 1) continue;
      int lo = 0, len = nk;
      while (len > 0) {
        const int half = len >> 1;
        if (so[lo + half + 1] <= t) {
          lo += half + 1;
          len -= half + 1;
        } else {
          len = half;
        }
      }
      kk[it] = uint32_t(lo);
    }
  }
  // phase 2: divmod by the right count, then the two row-id loads of every pair
  if (nk == 1) {
    // the whole tile lies inside one (heavy) key: one division, then step the
    // (li, ri) pair by kThreads outputs per item without dividing again
    const uint32_t c = src_[0];
    const uint64_t local0 = t0 + tid - so[0];
    uint64_t li = local0 / c;
    uint32_t ri = uint32_t(local0 - li * c);
    const uint32_t q = uint32_t(kThreads) / c, r = uint32_t(kThreads) % c;
    const uint32_t* lp = a.lpos + sls[0];
    const uint32_t* rp = a.rpos + srs[0];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      if (valid & (1u << it)) {
        lrow[it] = __ldg(lp + li);
        rrow[it] = __ldg(rp + ri);
      }
      li += q;
      ri += r;
      if (ri >= c) {
        ri -= c;
        ++li;
      }
    }
  } else {
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      if (!(valid & (1u << it))) continue;
      const uint32_t k = kk[it];
      const uint64_t local = t0 + uint64_t(it) * kThreads + tid - so[k];
      const uint32_t c = src_[k];
      uint64_t li, ri;
      if (local < (1ull << 32)) {
        const uint32_t l32 = uint32_t(local);
        li = l32 / c;
        ri = l32 - uint32_t(li) * c;
      } else {
        li = local / c;
        ri = local - li * c;
      }
      lrow[it] = __ldg(a.lpos + sls[k] + li);
      rrow[it] = __ldg(a.rpos + srs[k] + ri);
    }
  }
  if (kChecksum) {
#pragma unroll
    for (int it = 0; it < kItems; ++it)
      if (valid & (1u << it)) sum += fmix64((uint64_t(lrow[it]) << 32) | rrow[it]);
    __syncthreads();  // the staged window is rewritten by the next sub-tile
    continue;
  }
  // phase 3: pair outputs and column gathers (loads of a column batched)
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    if (!(valid & (1u << it))) continue;
    if (a.lrows_out) __stcs(a.lrows_out + o0 + it * kThreads, lrow[it]);
    if (a.rrows_out) __stcs(a.rrows_out + o0 + it * kThreads, rrow[it]);
  }
  for (int ci = 0; ci < cols.n; ++ci) {
    const rl_column& col = cols.c[ci];
    const int w = col.width;
    if (col.side == RL_SIDE_KEY) {
#pragma unroll
      for (int it = 0; it < kItems; ++it)
        if (valid & (1u << it))
          __stcs(reinterpret_cast<long long*>(col.dst) + o0 + it * kThreads,
                 (long long)__ldg(reinterpret_cast<const long long*>(a.matched_keys) + g0 + kk[it]));
      continue;
    }
    if (col.side == RL_SIDE_LEFT) gather_column(col, lrow, o0, valid);
    else gather_column(col, rrow, o0, valid);
  }
  __syncthreads();  // the staged window is rewritten by the next sub-tile
  }
  if (kChecksum) {  // one global atomic per CTA (per warp, thousands queue on one address at the end)
    __shared__ uint64_t wsum[kThreads / 32];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if ((tid & 31) == 0) wsum[tid >> 5] = sum;
    __syncthreads();
    if (tid == 0) {
      uint64_t t = 0;
      for (int w = 0; w < kThreads / 32; ++w) t += wsum[w];
      if (t) atomicAdd(reinterpret_cast<unsigned long long*>(a.checksum), (unsigned long long)t);
    }
  }
}
// One CTA per output tile while that fills ~8 CTAs per SM; beyond, each CTA
// walks a contiguous run of tiles (the key-window search then continues
// from where the previous tile ended instead of starting over).
static unsigned expand_grid(uint64_t outputs, uint32_t* per_cta) {
  const uint64_t tiles = (outputs + kTile - 1) / kTile;
  const uint64_t target = uint64_t(device_sm_count()) * 8;
  uint64_t per = tiles <= target ? 1 : (tiles + target - 1) / target;
  *per_cta = uint32_t(per);
  return unsigned((tiles + per - 1) / per);
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
  // the pairs-only path stores four row ids at a time (16-byte stores)
  if ((reinterpret_cast<uintptr_t>(lrows_out) | reinterpret_cast<uintptr_t>(rrows_out)) & 15) return RL_ERR_BAD_ARG;
  ExpandArgs a{matched_keys, ls, rs, rc, offs, m, lpos, rpos, out_begin, out_end, lrows_out, rrows_out, nullptr};
  uint32_t per_cta;
  const unsigned blocks = expand_grid(out_end - out_begin, &per_cta);
  expand_kernel<false><<<blocks, kThreads, 0, stream>>>(a, cs, per_cta);
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
  uint32_t per_cta;
  const unsigned blocks = expand_grid(out_end - out_begin, &per_cta);
  expand_kernel<true><<<blocks, kThreads, 0, stream>>>(a, cs, per_cta);
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

// The same for 4- and 8-byte columns, four consecutive output rows a thread:
// one 16-byte load of their row ids, every random row load of a column in
// flight before its 16-byte stores (kGU groups of four a thread). A gather
// from an L2-resident source is bound by random-load latency x loads in
// flight, not bytes: cfg2's 10M-row payload gather took 55 us one row a
// thread with the source already in L2.
constexpr int kGU = 2;
__global__ void __launch_bounds__(kThreads) gather_vec_kernel(const uint32_t* __restrict__ rows, int64_t m,
                                                              ColumnSet cols) {
  const int64_t m4 = m >> 2;
  const int64_t stride = int64_t(gridDim.x) * kThreads * kGU;
  for (int64_t g0 = int64_t(blockIdx.x) * kThreads * kGU + threadIdx.x; g0 < m4; g0 += stride) {
    uint4 r[kGU];
#pragma unroll
    for (int u = 0; u < kGU; ++u) {
      const int64_t g = g0 + int64_t(u) * kThreads;
      r[u] = g < m4 ? __ldcs(reinterpret_cast<const uint4*>(rows) + g) : make_uint4(0, 0, 0, 0);
    }
    for (int ci = 0; ci < cols.n; ++ci) {
      const rl_column& c = cols.c[ci];
      if (c.width == 4) {
        const unsigned int* src = static_cast<const unsigned int*>(c.src);
        uint4 v[kGU];
#pragma unroll
        for (int u = 0; u < kGU; ++u) {
          if (g0 + int64_t(u) * kThreads < m4) {
            v[u].x = ld_row(src + r[u].x);
            v[u].y = ld_row(src + r[u].y);
            v[u].z = ld_row(src + r[u].z);
            v[u].w = ld_row(src + r[u].w);
          }
        }
#pragma unroll
        for (int u = 0; u < kGU; ++u) {
          const int64_t g = g0 + int64_t(u) * kThreads;
          if (g < m4) __stcs(static_cast<uint4*>(c.dst) + g, v[u]);
        }
      } else {  // 8 bytes
        const unsigned long long* src = static_cast<const unsigned long long*>(c.src);
        ulonglong2 v[kGU][2];
#pragma unroll
        for (int u = 0; u < kGU; ++u) {
          if (g0 + int64_t(u) * kThreads < m4) {
            v[u][0].x = ld_row(src + r[u].x);
            v[u][0].y = ld_row(src + r[u].y);
            v[u][1].x = ld_row(src + r[u].z);
            v[u][1].y = ld_row(src + r[u].w);
          }
        }
#pragma unroll
        for (int u = 0; u < kGU; ++u) {
          const int64_t g = g0 + int64_t(u) * kThreads;
          if (g < m4) {
            __stcs(static_cast<ulonglong2*>(c.dst) + 2 * g, v[u][0]);
            __stcs(static_cast<ulonglong2*>(c.dst) + 2 * g + 1, v[u][1]);
          }
        }
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < uint32_t(m & 3)) {  // the last m % 4 rows
    const int64_t t = (m4 << 2) + threadIdx.x;
    const uint64_t row = rows[t];
    for (int ci = 0; ci < cols.n; ++ci) {
      const rl_column& c = cols.c[ci];
      copy_row(static_cast<const uint8_t*>(c.src) + row * uint64_t(c.width),
               static_cast<uint8_t*>(c.dst) + t * c.width, c.width);
    }
  }
}

int gather_rows(const uint32_t* rows, int64_t m, const rl_column* columns, int n_columns, cudaStream_t stream) {
  if (m < 0 || (m > 0 && rows == nullptr)) return RL_ERR_BAD_ARG;
  ColumnSet cs;
  int st = fill_columns(cs, columns, n_columns, false);
  if (st != RL_OK) return st;
  if (m == 0 || n_columns == 0) return RL_OK;
  bool vec = (reinterpret_cast<uintptr_t>(rows) & 15) == 0 && m >= 4 && std::getenv("RL_GATHER_SCALAR") == nullptr;
  for (int i = 0; i < n_columns && vec; ++i) {
    const rl_column& c = cs.c[i];
    vec = (c.width == 4 || c.width == 8) && (reinterpret_cast<uintptr_t>(c.src) % uintptr_t(c.width)) == 0 &&
          (reinterpret_cast<uintptr_t>(c.dst) & 15) == 0;
  }
  if (vec) {
    const int64_t groups = (m >> 2) + kThreads * kGU - 1;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(groups / (kThreads * kGU), int64_t(device_sm_count()) * 8)));
    gather_vec_kernel<<<grid, kThreads, 0, stream>>>(rows, m, cs);
    count_launches(1);
    return rl_cuda_status(cudaGetLastError());
  }
  const int grid = int(std::min<int64_t>((m + kThreads - 1) / kThreads, int64_t(device_sm_count()) * 16));
  gather_kernel<<<grid, kThreads, 0, stream>>>(rows, m, cs);
  count_launches(1);
  return rl_cuda_status(cudaGetLastError());
}

// Relation.take of two 8-byte columns stored row-interleaved (16-byte rows,
// e.g. a join's output written that way for the ORDER BY behind it): ONE
// random 16-byte load a row instead of two 8-byte loads from two arrays —
// random gathers over a large source are bound by the access rate, not the
// bytes (scripts/microbench/gather_flavors.cu: 27.6 vs 56.5 ms for 1e9 rows).
__global__ void __launch_bounds__(kThreads) gather_split16_kernel(const uint32_t* __restrict__ rows, int64_t m,
                                                                  const ulonglong2* __restrict__ src,
                                                                  unsigned long long* __restrict__ lo,
                                                                  unsigned long long* __restrict__ hi) {
  constexpr int U = 4;  // rows in flight a thread
  const int64_t stride = int64_t(gridDim.x) * kThreads * U;
  for (int64_t s = int64_t(blockIdx.x) * kThreads * U + threadIdx.x; s < m; s += stride) {
    uint32_t r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = s + int64_t(u) * kThreads;
      r[u] = t < m ? __ldcs(rows + t) : 0u;
    }
    ulonglong2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = s + int64_t(u) * kThreads;
      v[u] = t < m ? ld_row(src + r[u]) : make_ulonglong2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = s + int64_t(u) * kThreads;
      if (t < m) {
        __stcs(lo + t, v[u].x);
        __stcs(hi + t, v[u].y);
      }
    }
  }
}

int gather_split16(const uint32_t* rows, int64_t m, const void* src, void* lo, void* hi, cudaStream_t stream) {
  if (m < 0 || (m > 0 && (!rows || !src || !lo || !hi))) return RL_ERR_BAD_ARG;
  if ((reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(lo) & 7) ||
      (reinterpret_cast<uintptr_t>(hi) & 7))
    return RL_ERR_BAD_ARG;
  if (m == 0) return RL_OK;
  const int grid = int(std::min<int64_t>((m + kThreads * 4 - 1) / (kThreads * 4), int64_t(device_sm_count()) * 8));
  gather_split16_kernel<<<grid, kThreads, 0, stream>>>(rows, m, static_cast<const ulonglong2*>(src),
                                                       static_cast<unsigned long long*>(lo),
                                                       static_cast<unsigned long long*>(hi));
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
