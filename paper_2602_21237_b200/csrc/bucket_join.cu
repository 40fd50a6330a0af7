// bucket_join.cu — the equi-join as a partitioned join on chip.
//
// Replaces, for join keys with <= 32 varying bits (cfg1, cfg4, cfg5 keys), the
// reference's to_tensor x 2 + key_axis_align + expansion
// (/root/reference/pkg/src/relab/tensorpath.py:78-93, 109-128, 131-185) with
// a plan that never materialises the sorted key axes:
//
//   1. bj_partition (radix_sort.cu): one joint key packing for both sides
//      (the varying bits of both, against the left side's first key), then per
//      side the scatter path's chunk counts + two counting passes in packed-row
//      mode: every row becomes ONE u64 (packed key << 32 | row id) and lands
//      in its sub-bucket (top 16 bits of the packed key). Equal keys of the two
//      sides land in the same sub-bucket index.
//   2. bj_count_kernel: per run (consecutive sub-buckets of a 16-sub-bucket
//      group with <= kBjCap rows per side) the right rows are binned on chip
//      by (sub-bucket, next bits), every left row counts the right rows of its
//      bin with an equal key -> the run's pair count.
//   3. bj_scan_kernel: exclusive scan of the 65536 run counts -> every run's
//      first output row, the total (the one host sync of a join) and the
//      "applies" flag (no side fell back).
//   4. bj_emit_kernel: per run, both sides sorted on chip by their packed
//      words (= by key, then row id), every left row's matching right range
//      found in its bin, a prefix over the left rows gives each row's first
//      output, and the outputs are written in output order: key, left row,
//      right row — the reference order (tensorpath.py:162-172) — with every
//      column gathered (key = the matched key itself, left / right columns by
//      row id, or read beside the row when carried through the passes),
//      optionally only the slice [out_begin, out_end) and optionally
//      row-interleaved (a destination stride per column). Both sides are sorted
//      in one set of barrier phases (packed left / right bin counters); a run
//      with few pairs (<= 512 and <= 1/8 of its rows: selective joins) bins
//      only the right side, lists its matches and writes each at its rank
//      (two-level plans: the count kernel lists them; runs of <= 32 pairs are
//      written a warp each, ranked by shuffles).
//
// DRAM traffic per side: 8n (counts) + 16n (digit-7 pass) + 16n (digit-6
// pass) + 8n (count) + 8n (emit); no position, key-value, offset or
// alignment arrays are written. A sub-bucket above kBjCap rows (skewed keys),
// keys with more than 32 varying bits or a varying bit the joint sample missed
// make the plan report "does not apply" (scalars[1] == 0) and the caller runs
// the sort-based plan (plan.cu) instead.
#include <algorithm>
#include <cstdlib>

#include "bjoin.cuh"
#include "common.cuh"
#include "keypack.cuh"

namespace rl {
namespace bjoin {

using radix::BjSide;
using radix::kBjCap;
using radix::kBjSubBuckets;

constexpr int kThreads = 512;
// Work items: G consecutive sub-buckets — 16 of the 2^16 (two levels), or the
// 256 sub-sub-buckets of one level-2 sub-bucket (three levels: 2^24 of them)
template <int LEVELS>
struct Geo {
  static constexpr int G = LEVELS == 3 ? 256 : 16;
  static constexpr uint32_t kGroups = (LEVELS == 3 ? (1u << 24) : uint32_t(kBjSubBuckets)) / G;
  static constexpr int kShift = LEVELS == 3 ? 40 : 48;  // the sub-bucket index: top 24 / 16 bits
};
constexpr uint32_t kMaxGroups = 1u << 16;  // (three levels)
constexpr int kMaxG = 256;
constexpr int kMaxBins = 4096;
constexpr int kRowsPerThread = (kBjCap + kThreads - 1) / kThreads;  // 5
static_assert(kRowsPerThread <= 32, "the count kernel keeps a row-hit bit mask in one word");
constexpr int kRankMax = 48;  // bins above this: a warp's bitonic network
constexpr uint32_t kSelMax = 512;  // emit: a run with at most this many pairs (and <= 1/8 of its rows) lists its matches instead of sorting

struct PlanArgs {
  const uint64_t* rows_l;
  const uint64_t* rows_r;
  const uint32_t* off_l;
  const uint32_t* off_r;
  const uint32_t* flags_l;
  const uint32_t* flags_r;
  uint32_t* counts;  // [groups * G] pairs per (group, run slot)
  uint64_t* gtot;    // [groups] pairs per group -> (bj_scan_kernel) first output row of the group
  int levels;
  int64_t* scalars;  // [0] total pairs, [1] 1 = the bucket join applies
  const long long* k0_src;  // the left side's first key (constant bits of every key)
  const uint64_t* pay_l;    // carried payload words, parallel to rows_l (words_l per row)
  const uint64_t* pay_r;
  int words_l, words_r;
  // selective runs listed by the count kernel (two levels; null / 0 = off): the
  // run's matches (left word, right word) and load indexes (left | right << 16)
  // at run_sel[run] in sel_pairs / sel_idx (~0u: not listed), sel_cursor the fill
  ulonglong2* sel_pairs;
  uint32_t* sel_idx;
  uint32_t* run_sel;
  unsigned long long* sel_cursor;
  uint32_t sel_cap;
};

// Runs of one group: consecutive sub-buckets [s, e) with at most kBjCap rows
// on each side (every single sub-bucket fits: the scatter passes check it);
// encoded (s << 16) | e; greedy (a run from s takes the most sub-buckets that
// fit, at least one). The same cut in the count and emit kernels,
// by one warp (all 32 lanes, converged): a run's end is found by
// two ballots instead of a binary search — ends s + 8, s + 16, ... (the fit is
// monotone in the end: the count of fitting lanes places it within 8), then the
// 7 ends after that; G <= 256. Returns the run count in every lane.
template <int G>
__device__ __forceinline__ uint32_t cut_runs_warp(const uint32_t* ol, const uint32_t* orr, uint32_t* ends) {
  static_assert(G <= 256, "one ballot covers 32 x 8 ends");
  const uint32_t lane = threadIdx.x & 31;
  if (ol[G] - ol[0] <= uint32_t(kBjCap) && orr[G] - orr[0] <= uint32_t(kBjCap)) {  // the whole group
    if (lane == 0) ends[0] = uint32_t(G);
    return 1;
  }
  uint32_t nr = 0, s = 0;
  while (s < uint32_t(G)) {
    const uint32_t bl = ol[s], br = orr[s];
    auto fits = [&](uint32_t e) { return ol[e] - bl <= uint32_t(kBjCap) && orr[e] - br <= uint32_t(kBjCap); };
    const uint32_t e1 = s + 8 * (lane + 1);
    const uint32_t k1 = __popc(__ballot_sync(0xffffffffu, e1 <= uint32_t(G) && fits(e1)));
    const uint32_t base = s + 8 * k1;
    const uint32_t e2 = base + 1 + lane;
    const uint32_t k2 = __popc(__ballot_sync(0xffffffffu, lane < 7 && e2 <= uint32_t(G) && fits(e2)));
    const uint32_t e = max(base + k2, s + 1);  // (at least one sub-bucket)
    if (lane == 0) ends[nr] = (s << 16) | e;
    ++nr;
    s = e;
  }
  return nr;
}

__device__ __forceinline__ uint32_t bin_bits(uint32_t nsb) {
  return 12u - (nsb > 1 ? 32u - uint32_t(__clz(int(nsb - 1))) : 0u);
}

struct Bins {
  uint32_t first, bb, shift;
  __device__ __forceinline__ Bins(uint32_t first_sub, uint32_t nsb, uint32_t sub_shift) {
    first = first_sub;
    bb = bin_bits(nsb);
    shift = sub_shift;
  }
  __device__ __forceinline__ uint32_t count(uint32_t nsb) const { return nsb << bb; }
  // (sub-bucket - first, the next bb key bits): bins ordered like the keys
  __device__ __forceinline__ uint32_t of(uint64_t w) const {
    return ((uint32_t(w >> shift) - first) << bb) | (uint32_t(w >> (shift - bb)) & ((1u << bb) - 1u));
  }
};

__device__ __forceinline__ bool fell_back(const PlanArgs& a) {
  return __syncthreads_or(threadIdx.x == 0 && (*reinterpret_cast<volatile const uint32_t*>(a.flags_l) |
                                               *reinterpret_cast<volatile const uint32_t*>(a.flags_r)) != 0) != 0;
}

// Bin `cnt` rows (this thread's rows in w[]) into dst[] grouped by bin; hist[]
// ends as each bin's END. hist must be zero for the nbins bins on entry.
__device__ __forceinline__ void bin_rows(const uint64_t (&w)[kRowsPerThread], uint32_t cnt, const Bins& bins,
                                         uint32_t nbins, uint32_t* hist, uint64_t* dst, uint64_t* scan_scratch,
                                         uint16_t* dst_idx = nullptr) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int u = 0; u < kRowsPerThread; ++u)
    if (tid + u * kThreads < int(cnt)) atomicAdd(&hist[bins.of(w[u])], 1u);
  __syncthreads();
  scan_counters<kThreads, kMaxBins>(hist, nbins, reinterpret_cast<uint32_t*>(scan_scratch));  // (synchronised)
#pragma unroll
  for (int u = 0; u < kRowsPerThread; ++u) {
    if (tid + u * kThreads < int(cnt)) {
      const uint32_t at = atomicAdd(&hist[bins.of(w[u])], 1u);
      dst[at] = w[u];
      if (dst_idx) dst_idx[at] = uint16_t(tid + u * kThreads);  // the row's load index in its run
    }
  }
  __syncthreads();
}

// L2 prefetch of the rows of the run after r in this group (both sides), issued
// while run r is processed: the next run's first loads then hit L2.
template <int G>
__device__ __forceinline__ void prefetch_next_run(const PlanArgs& a, const uint32_t* offl, const uint32_t* offr,
                                                  const uint32_t* ends, uint32_t r, uint32_t nr) {
  if (r + 1 >= nr) return;
  const uint32_t s = ends[r + 1] >> 16, e = ends[r + 1] & 0xFFFFu;
  const uint32_t l0 = offl[s], r0 = offr[s];
  const uint32_t lines_l = ((offl[e] - l0) * 8 + 127) / 128, lines_r = ((offr[e] - r0) * 8 + 127) / 128;
  for (uint32_t i = threadIdx.x; i < lines_l + lines_r; i += kThreads) {
    const uint64_t* p = i < lines_l ? a.rows_l + l0 + size_t(i) * 16 : a.rows_r + r0 + size_t(i - lines_l) * 16;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  }
}

__device__ __forceinline__ void load_rows(const uint64_t* rows, uint32_t r0, uint32_t cnt,
                                          uint64_t (&w)[kRowsPerThread]) {
#pragma unroll
  for (int u = 0; u < kRowsPerThread; ++u) {
    const uint32_t j = threadIdx.x + u * kThreads;
    w[u] = j < cnt ? __ldcs(rows + r0 + j) : 0ull;
  }
}

// ---------------------------------------------------------------- count
template <int LEVELS>
__global__ void __launch_bounds__(kThreads, 3) bj_count_kernel(PlanArgs a) {
  using Q = Geo<LEVELS>;
  constexpr int G = Q::G;
  __shared__ uint64_t br[kBjCap];
  __shared__ __align__(16) uint32_t hist[kMaxBins];
  __shared__ uint32_t offl[G + 1], offr[G + 1], ends[G];
  __shared__ uint64_t scratch[kThreads / 32 + 2];
  __shared__ uint32_t nruns;
  __shared__ unsigned long long gsum;
  __shared__ unsigned long long runsum[2];  // pair counts of the current / next run
  __shared__ uint16_t bidx[kBjCap];            // right rows' load indexes (listing)
  __shared__ uint32_t selbase, lcount;
  const int tid = threadIdx.x;
  if (fell_back(a)) return;
  // packed key length: a bin covering all of its bits holds ONE key
  const uint32_t code = __ldcg(a.flags_l + 6);
  const uint32_t keybits = (code >> 14 & 127) + (code & 127);
  for (uint32_t g = blockIdx.x; g < Q::kGroups; g += gridDim.x) {
    for (uint32_t i = tid; i <= uint32_t(G); i += kThreads) {
      offl[i] = __ldcg(a.off_l + size_t(g) * G + i);
      offr[i] = __ldcg(a.off_r + size_t(g) * G + i);
    }
    if (tid == 0) {
      gsum = 0;
      runsum[0] = 0;
    }
    __syncthreads();
    if (tid < 32) {
      const uint32_t n = cut_runs_warp<G>(offl, offr, ends);
      if (tid == 0) nruns = n;
    }
    __syncthreads();
    const uint32_t nr = nruns;
    for (uint32_t r = 0; r < nr; ++r) {
      const uint32_t s = ends[r] >> 16, e = ends[r] & 0xFFFFu;
      const uint32_t l0 = offl[s], nl = offl[e] - l0, r0 = offr[s], nrr = offr[e] - r0;
      prefetch_next_run<G>(a, offl, offr, ends, r, nr);
      uint64_t cnt = 0;
      const Bins bins(g * G + s, e - s, Q::kShift);
      const bool key_bins = (64u - uint32_t(Q::kShift)) + bins.bb >= keybits;  // bins = keys
      if (nl && nrr && key_bins) {
        // one key a bin: pairs = sum over bins of left rows x right rows (both
        // counts in one word: left in the low 16 bits, right in the high 16)
        const uint32_t nbins = bins.count(e - s);
        for (uint32_t i = tid; i < nbins / 4; i += kThreads) reinterpret_cast<uint4*>(hist)[i] = make_uint4(0, 0, 0, 0);
        uint64_t w[kRowsPerThread], wl[kRowsPerThread];
        load_rows(a.rows_r, r0, nrr, w);
        load_rows(a.rows_l, l0, nl, wl);
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u) {
          if (tid + u * kThreads < int(nl)) atomicAdd(&hist[bins.of(wl[u])], 1u);
          if (tid + u * kThreads < int(nrr)) atomicAdd(&hist[bins.of(w[u])], 1u << 16);
        }
        __syncthreads();
        for (uint32_t i = tid; i < nbins; i += kThreads) {
          const uint32_t h = hist[i];
          cnt += uint64_t(h & 0xFFFFu) * (h >> 16);
        }
      } else if (nl && nrr) {
        const uint32_t nbins = bins.count(e - s);
        for (uint32_t i = tid; i < nbins; i += kThreads) hist[i] = 0;
        uint64_t w[kRowsPerThread], wl[kRowsPerThread];
        load_rows(a.rows_r, r0, nrr, w);
        load_rows(a.rows_l, l0, nl, wl);  // in flight while the right side is binned
        __syncthreads();
        bin_rows(w, nrr, bins, nbins, hist, br, scratch, bidx);
        uint32_t hits = 0;  // bit u: left row u matched (the listing re-probes only those)
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u) {
          if (tid + u * kThreads < int(nl)) {
            const uint32_t b = bins.of(wl[u]);
            const uint32_t b0 = b ? hist[b - 1] : 0u, b1 = hist[b];
            const uint32_t key = uint32_t(wl[u] >> 32);
            uint32_t c = 0;
            for (uint32_t i = b0; i < b1; ++i) c += uint32_t(br[i] >> 32) == key ? 1u : 0u;
            cnt += c;
            hits |= (c != 0 ? 1u : 0u) << u;
          }
        }
        if (a.sel_cap) {
          // a selective run (few pairs: <= kSelMax and <= 1/8 of its rows, the
          // emit's own rule) lists its matches for the emit, which then needs
          // neither side's rows (the 1/8 rule bounds the buffer: sel_cap >= rows / 8)
          uint64_t wc = cnt;
          for (int o = 16; o > 0; o >>= 1) wc += __shfl_xor_sync(0xffffffffu, wc, o);
          if ((tid & 31) == 0 && wc) atomicAdd(&runsum[r & 1], (unsigned long long)wc);
          __syncthreads();
          const uint64_t tot = runsum[r & 1];
          const bool list = tot > 0 && tot <= kSelMax && tot * 8 <= uint64_t(nl) + nrr;
          if (list) {
            if (tid == 0) {
              selbase = uint32_t(atomicAdd(a.sel_cursor, (unsigned long long)tot));
              lcount = 0;
            }
            __syncthreads();
            const uint32_t sb = selbase;
#pragma unroll
            for (int u = 0; u < kRowsPerThread; ++u) {
              const uint32_t j = tid + u * kThreads;
              if (hits >> u & 1u) {
                const uint32_t b = bins.of(wl[u]);
                const uint32_t b0 = b ? hist[b - 1] : 0u, b1 = hist[b];
                const uint32_t key = uint32_t(wl[u] >> 32);
                for (uint32_t i = b0; i < b1; ++i) {
                  if (uint32_t(br[i] >> 32) == key) {
                    const uint32_t k = atomicAdd(&lcount, 1u);
                    a.sel_pairs[sb + k] = make_ulonglong2(wl[u], br[i]);
                    a.sel_idx[sb + k] = j | (uint32_t(bidx[i]) << 16);
                  }
                }
              }
            }
          }
          if (tid == 0) a.run_sel[size_t(g) * G + r] = list ? selbase : ~0u;
          cnt = 0;  // (already in runsum)
        }
      }
      if (a.sel_cap && !(nl && nrr && !key_bins) && tid == 0) a.run_sel[size_t(g) * G + r] = ~0u;
      // the run's pair count: a warp sum, one shared atomic a warp
      for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      if ((tid & 31) == 0 && cnt) atomicAdd(&runsum[r & 1], (unsigned long long)cnt);
      __syncthreads();  // (also: hist / br reused by the next run)
      if (tid == 0) {
        const uint64_t tot = runsum[r & 1];
        a.counts[size_t(g) * G + r] = uint32_t(tot);
        gsum += tot;
        runsum[(r + 1) & 1] = 0;  // the next run's slot (its atomics come after a later barrier)
      }
    }
    if (tid == 0) a.gtot[g] = gsum;
    __syncthreads();
  }
}

// ---------------------------------------------------------------- scan
// One CTA: the group totals (4096 or 65536) in chunks staged through shared
// memory (coalesced loads), an exclusive scan carried from chunk to chunk —
// in place: gtot[g] becomes the group's first output row.
__global__ void __launch_bounds__(1024) bj_scan_kernel(PlanArgs a, uint32_t groups) {
  constexpr int kChunk = 4096, kPer = kChunk / 1024;
  __shared__ uint64_t buf[kChunk];
  __shared__ uint64_t scratch[34];
  const int tid = threadIdx.x;
  const bool ok = *reinterpret_cast<volatile const uint32_t*>(a.flags_l) == 0 &&
                  *reinterpret_cast<volatile const uint32_t*>(a.flags_r) == 0;
  uint64_t carry = 0;
  for (uint32_t c0 = 0; c0 < groups; c0 += kChunk) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) buf[i * 1024 + tid] = ok ? __ldcg(a.gtot + c0 + i * 1024 + tid) : 0ull;
    __syncthreads();
    uint64_t run = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) run += buf[tid * kPer + i];
    uint64_t total;
    uint64_t start = carry + block_exclusive_scan<1024>(run, scratch, &total);
    if (ok) {
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        a.gtot[c0 + tid * kPer + i] = start;
        start += buf[tid * kPer + i];
      }
    }
    carry += total;
    __syncthreads();  // buf and scratch reused by the next chunk
  }
  if (tid == 0) {
    a.scalars[0] = ok ? int64_t(carry) : 0;
    a.scalars[1] = ok ? 1 : 0;
  }
}

// ---------------------------------------------------------------- emit
struct EmitArgs {
  PlanArgs p;
  uint64_t out_begin, out_end;
  int no_sel;  // RL_BJ_NO_SEL=1: every run takes the sorting path (A/B, tests)
  uint32_t* lrows_out;
  uint32_t* rrows_out;
  unsigned long long* checksum;
};

constexpr int kMaxCols = RL_MAX_COLUMNS;
struct EmitCol {
  const uint8_t* src;  // gathered by row id (carry_off < 0)
  uint8_t* dst;
  int width;
  int side;
  int carry_off;       // >= 0: the bytes at this offset of the row's carried payload words
  int vec;             // 8 / 16: every source row of the column is one aligned 8- / 16-byte load (host-checked)
  int64_t dstride;     // bytes between output rows (the width, or a row-interleaved layout's row size)
};
struct Cols {
  EmitCol c[kMaxCols];
  int n;
};

// Sort the rows of dst[0, cnt) — grouped by bin, hist[] = bin ends — into
// sorted[] by packed word (unique: key bits, then row id). Rows rank among
// their bin-mates; bins above kRankMax rows go through a warp's bitonic
// network in place first.
__device__ __forceinline__ void finish_sort(uint64_t* grouped, uint64_t* sorted, const uint32_t* hist,
                                            const Bins& bins, uint32_t cnt, uint32_t* big, uint32_t* nbig,
                                            uint16_t* gidx, uint16_t* sidx) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) *nbig = 0;
  __syncthreads();
  for (uint32_t p = tid; p < cnt; p += kThreads) {
    const uint64_t w = grouped[p];
    const uint32_t b = bins.of(w);
    const uint32_t b0 = b ? hist[b - 1] : 0u, b1 = hist[b];
    if (b1 - b0 > uint32_t(kRankMax)) {
      if (p == b0) {
        const uint32_t slot = atomicAdd(nbig, 1u);
        if (slot < 64u) big[slot] = b;
      }
      continue;
    }
    uint32_t rk = 0;
    for (uint32_t i = b0; i < b1; ++i) rk += grouped[i] < w ? 1u : 0u;
    sorted[b0 + rk] = w;
    sidx[b0 + rk] = gidx[p];
  }
  __syncthreads();
  const uint32_t nb = *nbig;  // <= kBjCap / (kRankMax + 1) = 52 < 64
  for (uint32_t t = warp; t < min(nb, 64u); t += kThreads / 32) {
    const uint32_t b = big[t];
    const uint32_t b0 = b ? hist[b - 1] : 0u, b1 = hist[b];
    // bitonic over [b0, b1) in `grouped`, padded to a power of two with +inf
    const uint32_t sz = b1 - b0;
    uint32_t p2 = 1;
    while (p2 < sz) p2 <<= 1;
    for (uint32_t k = 2; k <= p2; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t x = lane; x < (p2 >> 1); x += 32) {
          const uint32_t i = (x / j) * (2 * j) + (x % j);
          const uint32_t q = j == (k >> 1) ? (i ^ (k - 1)) : (i + j);
          if (q < sz) {
            const uint64_t u = grouped[b0 + i], v = grouped[b0 + q];
            if (v < u) {
              grouped[b0 + i] = v;
              grouped[b0 + q] = u;
              const uint16_t t = gidx[b0 + i];
              gidx[b0 + i] = gidx[b0 + q];
              gidx[b0 + q] = t;
            }
          }
        }
        __syncwarp();
      }
    }
    for (uint32_t p = b0 + lane; p < b1; p += 32) {
      sorted[p] = grouped[p];
      sidx[p] = gidx[p];
    }
  }
  __syncthreads();
}

// Both sides of a run sorted by packed word in ONE set of barrier phases: the
// bin counters hold the left count in the low 16 bits and the right count in
// the high 16 (<= kBjCap rows a side, so one packed scan gives both sides'
// starts), and the left rows go grouped-by-bin into `grouped` and then ranked
// into `sl` while the right rows are grouped straight into `sr` and ranked in
// place (new slots kept in registers across the barrier). On return hist[b]
// holds both sides' bin ends (left: low half, right: high half).
__device__ __forceinline__ void sort_both(const uint64_t (&wl)[kRowsPerThread], uint32_t nl,
                                          const uint64_t (&wr)[kRowsPerThread], uint32_t nrr, const Bins& bins,
                                          uint32_t nbins, uint32_t* hist, uint64_t* grouped, uint64_t* sl,
                                          uint64_t* sr, uint16_t* gidx, uint16_t* lidx, uint16_t* ridx,
                                          uint64_t* scan_scratch, uint32_t* big, uint32_t* nbig) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int u = 0; u < kRowsPerThread; ++u) {
    if (tid + u * kThreads < int(nl)) atomicAdd(&hist[bins.of(wl[u])], 1u);
    if (tid + u * kThreads < int(nrr)) atomicAdd(&hist[bins.of(wr[u])], 1u << 16);
  }
  if (tid == 0) *nbig = 0;
  __syncthreads();
  scan_counters<kThreads, kMaxBins>(hist, nbins, reinterpret_cast<uint32_t*>(scan_scratch));  // (synchronised)
#pragma unroll
  for (int u = 0; u < kRowsPerThread; ++u) {
    const uint16_t j = uint16_t(tid + u * kThreads);  // the row's load index in its run
    if (j < nl) {
      const uint32_t at = atomicAdd(&hist[bins.of(wl[u])], 1u) & 0xFFFFu;
      grouped[at] = wl[u];
      gidx[at] = j;
    }
    if (j < nrr) {
      const uint32_t at = atomicAdd(&hist[bins.of(wr[u])], 1u << 16) >> 16;
      sr[at] = wr[u];
      ridx[at] = j;
    }
  }
  __syncthreads();
  // rank among bin-mates (the packed words are unique); bins above kRankMax
  // rows are listed (bit 31: right side) for a warp's bitonic network
  uint64_t mv[kRowsPerThread];
  uint32_t mp[kRowsPerThread];  // right rows: new slot << 16 | load index, or ~0u (stays)
#pragma unroll
  for (int u = 0; u < kRowsPerThread; ++u) {
    const uint32_t p = tid + u * kThreads;
    if (p < nl) {
      const uint64_t w = grouped[p];
      const uint32_t b = bins.of(w);
      const uint32_t b0 = b ? hist[b - 1] & 0xFFFFu : 0u, b1 = hist[b] & 0xFFFFu;
      if (b1 - b0 > uint32_t(kRankMax)) {
        if (p == b0) {
          const uint32_t slot = atomicAdd(nbig, 1u);
          if (slot < 128u) big[slot] = b;
        }
      } else {
        uint32_t rk = 0;
        if (b1 - b0 > 1)
          for (uint32_t i = b0; i < b1; ++i) rk += grouped[i] < w ? 1u : 0u;
        sl[b0 + rk] = w;
        lidx[b0 + rk] = gidx[p];
      }
    }
    mp[u] = ~0u;
    mv[u] = 0;
    if (p < nrr) {
      const uint64_t w = sr[p];
      const uint32_t b = bins.of(w);
      const uint32_t b0 = b ? hist[b - 1] >> 16 : 0u, b1 = hist[b] >> 16;
      if (b1 - b0 > uint32_t(kRankMax)) {
        if (p == b0) {
          const uint32_t slot = atomicAdd(nbig, 1u);
          if (slot < 128u) big[slot] = b | 0x80000000u;
        }
      } else if (b1 - b0 > 1) {
        uint32_t rk = 0;
        for (uint32_t i = b0; i < b1; ++i) rk += sr[i] < w ? 1u : 0u;
        if (b0 + rk != p) {
          mv[u] = w;
          mp[u] = ((b0 + rk) << 16) | ridx[p];
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kRowsPerThread; ++u) {
    if (mp[u] != ~0u) {
      sr[mp[u] >> 16] = mv[u];
      ridx[mp[u] >> 16] = uint16_t(mp[u]);
    }
  }
  const uint32_t nb = min(*nbig, 128u);  // <= 2 x kBjCap / (kRankMax + 1) = 104
  for (uint32_t t = warp; t < nb; t += kThreads / 32) {
    const uint32_t e = big[t];
    const bool right = e >> 31;
    const uint32_t b = e & 0x7FFFFFFFu;
    const uint32_t sh = right ? 16u : 0u;
    const uint32_t b0 = b ? (hist[b - 1] >> sh) & 0xFFFFu : 0u, b1 = (hist[b] >> sh) & 0xFFFFu;
    uint64_t* arr = right ? sr : grouped;
    uint16_t* ix = right ? ridx : gidx;
    // bitonic over [b0, b1), padded to a power of two with +inf; the rows of a
    // big bin are not moved by the rank writes above (disjoint slots)
    const uint32_t sz = b1 - b0;
    uint32_t p2 = 1;
    while (p2 < sz) p2 <<= 1;
    for (uint32_t k = 2; k <= p2; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t x = lane; x < (p2 >> 1); x += 32) {
          const uint32_t i = (x / j) * (2 * j) + (x % j);
          const uint32_t q = j == (k >> 1) ? (i ^ (k - 1)) : (i + j);
          if (q < sz) {
            const uint64_t a = arr[b0 + i], c = arr[b0 + q];
            if (c < a) {
              arr[b0 + i] = c;
              arr[b0 + q] = a;
              const uint16_t t2 = ix[b0 + i];
              ix[b0 + i] = ix[b0 + q];
              ix[b0 + q] = t2;
            }
          }
        }
        __syncwarp();
      }
    }
    if (!right)
      for (uint32_t p = b0 + lane; p < b1; p += 32) {
        sl[p] = grouped[p];
        lidx[p] = gidx[p];
      }
  }
  __syncthreads();
}

#ifdef RL_BJ_PROFILE  // per-phase clock totals of the emit (A/B builds only)
__device__ unsigned long long g_bj_prof[16];
#define BJPROF(i) do { if (threadIdx.x == 0) { const long long c_ = clock64(); atomicAdd(&g_bj_prof[i], (unsigned long long)(c_ - bjt)); bjt = c_; } } while (0)
#else
#define BJPROF(i) do { } while (0)
#endif

template <bool CHECKSUM, int LEVELS>  // CHECKSUM: sum fmix64(l << 32 | r) over the pairs into *e.checksum instead
__global__ void __launch_bounds__(kThreads, 2) bj_emit_kernel(EmitArgs e, Cols cols) {
  using Q = Geo<LEVELS>;
  constexpr int G = Q::G;
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* sl = reinterpret_cast<uint64_t*>(smem);  // [kBjCap] left rows, sorted
  uint64_t* sr = sl + kBjCap;                         // [kBjCap] right rows, sorted
  uint64_t* gx = sr + kBjCap;                         // [kBjCap] grouped-by-bin scratch / per-left-row arrays
  uint32_t* hr = reinterpret_cast<uint32_t*>(gx + kBjCap);  // [kMaxBins] bin counters (right bin ends for the match)
  uint32_t* omap = hr + kMaxBins;                           // [kMaxBins] output -> left row
  uint16_t* gidx = reinterpret_cast<uint16_t*>(omap + kMaxBins);  // [kBjCap] load index of grouped rows
  uint16_t* lidx = gidx + kBjCap;                                 // [kBjCap] load index of sorted left rows
  uint16_t* ridx = lidx + kBjCap;                                 // [kBjCap] ... right rows
  uint64_t* scratch = reinterpret_cast<uint64_t*>(ridx + kBjCap);  // [kThreads / 32 + 2]
  uint64_t* rpre = scratch + kThreads / 32 + 2;                    // [kMaxG + 1] run starts in the group
  uint32_t* misc = reinterpret_cast<uint32_t*>(rpre + kMaxG + 1);  // offsets, runs, big bins
  uint32_t* offl = misc;                     // [kMaxG + 1]
  uint32_t* offr = misc + (kMaxG + 1);       // [kMaxG + 1]
  uint32_t* ends = misc + 2 * (kMaxG + 1);   // [kMaxG]
  uint32_t* big = ends + kMaxG;              // [128] big bins of both sides
  uint32_t* nbig = big + 128;
  uint32_t* nruns = nbig + 1;
  const PlanArgs& a = e.p;
  const int tid = threadIdx.x;
  uint64_t sum = 0;
  const uint32_t code = __ldcg(a.flags_l + 6);
  const uint64_t k0 = radix::xform(uint64_t(__ldg(a.k0_src)), 0);
  const uint64_t constbits = k0 & ~radix::pack_mask(code);
  const int mode = radix::pack_mode(code);
  const uint32_t shl = radix::pack_shift(code);
  const uint32_t keybits = (code >> 14 & 127) + (code & 127);  // packed key length
  auto key_of = [&](uint64_t w) -> long long {
    const uint64_t v = w & ~0xFFFFFFFFull;
    const uint64_t u = mode == 1 ? (v >> shl) | constbits : radix::unpack_key(v, code, constbits);
    return (long long)radix::xform(u, 0);
  };
  // one listed pair at output row t (l0 / r0: its run's first rows, for carried payloads)
  auto write_pair = [&](uint64_t t, uint32_t l0, uint32_t r0, const ulonglong2& me, uint32_t pi) {
    const uint32_t lrow = uint32_t(me.x), rrow = uint32_t(me.y);
    if constexpr (CHECKSUM) {
      sum += fmix64((uint64_t(lrow) << 32) | rrow);
      return;
    }
    const uint64_t o = t - e.out_begin;
    if (e.lrows_out) __stcs(e.lrows_out + o, lrow);
    if (e.rrows_out) __stcs(e.rrows_out + o, rrow);
    const uint32_t lj = pi & 0xFFFFu, rj = pi >> 16;
    for (int ci = 0; ci < cols.n; ++ci) {
      const EmitCol& c = cols.c[ci];
      uint8_t* dst = c.dst + o * uint64_t(c.dstride);
      if (c.side == RL_SIDE_KEY) {
        __stcs(reinterpret_cast<long long*>(dst), key_of(me.x));
      } else if (c.carry_off >= 0) {
        const bool left = c.side == RL_SIDE_LEFT;
        const uint64_t* pay = left ? a.pay_l : a.pay_r;
        const int words = left ? a.words_l : a.words_r;
        const uint64_t at = left ? uint64_t(l0) + lj : uint64_t(r0) + rj;
        copy_row(reinterpret_cast<const uint8_t*>(pay + at * words) + c.carry_off, dst, c.width);
      } else {
        copy_row(c.src + uint64_t(c.side == RL_SIDE_LEFT ? lrow : rrow) * c.width, dst, c.width);
      }
    }
  };
#ifdef RL_BJ_PROFILE
  long long bjt = clock64();
#endif
  for (uint32_t g = blockIdx.x; g < Q::kGroups; g += gridDim.x) {
    const uint64_t gbase = __ldcg(a.gtot + g);  // the group's first output row (scanned)
    for (uint32_t i = tid; i <= uint32_t(G); i += kThreads) {
      offl[i] = __ldcg(a.off_l + size_t(g) * G + i);
      offr[i] = __ldcg(a.off_r + size_t(g) * G + i);
    }
    __syncthreads();
    if (tid < 32) {
      const uint32_t n = cut_runs_warp<G>(offl, offr, ends);
      if (tid == 0) *nruns = n;
    }
    __syncthreads();
    const uint32_t nr = *nruns;
    {  // run starts inside the group (and the run's pair count: rpre[r + 1] - rpre[r])
      const uint64_t c = tid < int(nr) ? uint64_t(__ldcg(a.counts + size_t(g) * G + tid)) : 0ull;
      uint64_t tot;
      const uint64_t ex = block_exclusive_scan<kThreads>(c, scratch, &tot);
      if (tid < int(nr)) rpre[tid] = ex;
      if (tid == 0) rpre[nr] = tot;
      __syncthreads();
    }
    if (LEVELS == 2 && a.run_sel) {  // (three-level plans list nothing: sel_cap_of)
      // listed runs of at most 32 pairs: a warp each, the CTA's warps on different
      // runs at once (the run loop below would take them one at a time, each a
      // load -> barrier -> gather round trip); lane q ranks pair q by shuffles
      const uint32_t lane = tid & 31;
      for (uint32_t r = tid >> 5; r < nr; r += kThreads / 32) {
        const uint32_t np = uint32_t(rpre[r + 1] - rpre[r]);
        const uint64_t base = gbase + rpre[r];
        if (np == 0 || np > 32 || base + np <= e.out_begin || base >= e.out_end) continue;
        const uint32_t so = __ldcg(a.run_sel + size_t(g) * G + r);
        if (so == ~0u) continue;
        // the run's first rows from global, not offl / offr: a warp still here may
        // overlap the next group's rewrite of those (no barrier after this loop)
        const uint32_t s = ends[r] >> 16;
        const uint32_t l0 = __ldcg(a.off_l + size_t(g) * G + s), r0 = __ldcg(a.off_r + size_t(g) * G + s);
        ulonglong2 me = make_ulonglong2(~0ull, ~0ull);
        uint32_t pi = 0;
        if (lane < np) {
          me = __ldcg(a.sel_pairs + so + lane);
          pi = __ldcg(a.sel_idx + so + lane);
        }
        uint32_t rk = 0;
        for (uint32_t i = 0; i < np; ++i) {
          const unsigned long long ox = __shfl_sync(0xffffffffu, me.x, i), oy = __shfl_sync(0xffffffffu, me.y, i);
          rk += (ox < me.x || (ox == me.x && oy < me.y)) ? 1u : 0u;
        }
        const uint64_t t = base + rk;
        if (lane < np && t >= e.out_begin && t < e.out_end) write_pair(t, l0, r0, me, pi);
      }
    }
    for (uint32_t r = 0; r < nr; ++r) {
      const uint32_t cnt_pairs = uint32_t(rpre[r + 1] - rpre[r]);
      const uint64_t base = gbase + rpre[r];
      if (cnt_pairs == 0 || base + cnt_pairs <= e.out_begin || base >= e.out_end) continue;  // uniform
      const uint32_t s = ends[r] >> 16, en = ends[r] & 0xFFFFu;
      const uint32_t l0 = offl[s], nl = offl[en] - l0, r0 = offr[s], nrr = offr[en] - r0;
      const Bins bins(g * G + s, en - s, Q::kShift);
      const uint32_t nbins = bins.count(en - s);
      const bool key_bins = (64u - uint32_t(Q::kShift)) + bins.bb >= keybits;  // bins = keys
      // listed pairs of a selective run: each writes itself at output row base +
      // its rank in (left word, right word) order = (key, left row, right row)
      auto rank_write = [&](const ulonglong2* pairs, const uint32_t* pidx, uint32_t np) {
          for (uint32_t q = tid; q < np; q += kThreads) {
            const ulonglong2 me = pairs[q];
            uint32_t rk = 0;
            for (uint32_t i = 0; i < np; ++i) {
              const ulonglong2 o = pairs[i];
              rk += (o.x < me.x || (o.x == me.x && o.y < me.y)) ? 1u : 0u;
            }
            const uint64_t t = base + rk;  // the pair's output row
            if (t < e.out_begin || t >= e.out_end) continue;
            write_pair(t, l0, r0, me, pidx[q]);
          }
      };
      if (a.run_sel) {  // listed by the count kernel: neither side's rows are needed
        const uint32_t so = __ldcg(a.run_sel + size_t(g) * G + r);
        if (so != ~0u) {
          if (cnt_pairs <= 32) continue;  // (written by a warp above)
          ulonglong2* pairs = reinterpret_cast<ulonglong2*>(gx);
          uint32_t* pidx = omap;
          for (uint32_t q = tid; q < cnt_pairs; q += kThreads) {
            pairs[q] = __ldcg(a.sel_pairs + so + q);
            pidx[q] = __ldcg(a.sel_idx + so + q);
          }
          __syncthreads();
          rank_write(pairs, pidx, cnt_pairs);
          __syncthreads();  // smem reused by the next run
          continue;
        }
      }
      for (uint32_t i = tid; i < nbins / 4; i += kThreads) reinterpret_cast<uint4*>(hr)[i] = make_uint4(0, 0, 0, 0);  // (nbins % 16 == 0)
      prefetch_next_run<G>(a, offl, offr, ends, r, nr);
      if constexpr (!CHECKSUM) {  // the carried payload windows of this run: into L2 while the rows are sorted
        const uint32_t lines_l = (nl * uint32_t(a.words_l) * 8 + 127) / 128, lines_r = (nrr * uint32_t(a.words_r) * 8 + 127) / 128;
        for (uint32_t i = tid; i < lines_l + lines_r; i += kThreads) {
          const uint64_t* p = i < lines_l ? a.pay_l + size_t(l0) * a.words_l + size_t(i) * 16
                                          : a.pay_r + size_t(r0) * a.words_r + size_t(i - lines_l) * 16;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
        }
      }
      uint64_t w[kRowsPerThread], wl[kRowsPerThread];
      BJPROF(7);  // group setup / skipped runs
      load_rows(a.rows_l, l0, nl, wl);
      load_rows(a.rows_r, r0, nrr, w);
      __syncthreads();
      BJPROF(0);  // run setup, prefetch issue, row loads
      // (measured: with pairs about as many as rows, e.g. 240 a run, listing and
      // ranking them cost more than the two sorts — 1M-row joins 0.44 -> 0.57 ms)
      if (cnt_pairs <= kSelMax && cnt_pairs * 8 <= nl + nrr && !e.no_sel) {
        // a selective run (few pairs, e.g. cfg4): only the right side is binned;
        // every left row lists its matches (left word, right word, load indexes),
        // and each listed pair's output row is its rank in (left word, right
        // word) order = (key, left row, right row) — no sort of either side
        bin_rows(w, nrr, bins, nbins, hr, sr, scratch, ridx);
        if (tid == 0) *nbig = 0;
        __syncthreads();
        ulonglong2* pairs = reinterpret_cast<ulonglong2*>(gx);  // [kSelMax] (left word, right word)
        uint32_t* pidx = omap;                                  // [kSelMax] left | right load index << 16
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u) {
          const uint32_t j = tid + u * kThreads;
          if (j < nl) {
            const uint64_t wv = wl[u];
            const uint32_t b = bins.of(wv);
            const uint32_t b0 = b ? hr[b - 1] : 0u, b1 = hr[b];
            const uint32_t key = uint32_t(wv >> 32);
            for (uint32_t i = b0; i < b1; ++i) {
              const uint64_t wr = sr[i];
              if (key_bins || uint32_t(wr >> 32) == key) {
                const uint32_t at = atomicAdd(nbig, 1u);
                if (at < kSelMax) {
                  pairs[at] = make_ulonglong2(wv, wr);
                  pidx[at] = j | (uint32_t(ridx[i]) << 16);
                }
              }
            }
          }
        }
        __syncthreads();
        const uint32_t np = min(*nbig, kSelMax);  // (== cnt_pairs)
        rank_write(pairs, pidx, np);
        __syncthreads();  // smem reused by the next run
        continue;
      }
      // left side sorted first; the bin counters then serve the right side and
      // keep its bin ends for the match
#ifdef RL_BJ_SEPARATE_SORTS  // (A/B: one side after the other)
      bin_rows(wl, nl, bins, nbins, hr, gx, scratch, gidx);
      finish_sort(gx, sl, hr, bins, nl, big, nbig, gidx, lidx);
      BJPROF(1);  // left side binned + sorted
      for (uint32_t i = tid; i < nbins; i += kThreads) hr[i] = 0;
      __syncthreads();
      bin_rows(w, nrr, bins, nbins, hr, gx, scratch, gidx);
      finish_sort(gx, sr, hr, bins, nrr, big, nbig, gidx, ridx);
      for (uint32_t i = tid; i < nbins; i += kThreads) hr[i] <<= 16;  // (the right ends in the high half)
      __syncthreads();
#else
      sort_both(wl, nl, w, nrr, bins, nbins, hr, gx, sl, sr, gidx, lidx, ridx, scratch, big, nbig);
#endif
      BJPROF(2);  // both sides binned + sorted
      // every left row (sorted index p): its matching right range [rs, rs + m) in sr
      uint32_t* m_arr = reinterpret_cast<uint32_t*>(gx);
      uint32_t* rs_arr = m_arr + kBjCap;
      constexpr int kPer = kRowsPerThread;
      uint32_t mloc[kPer], run = 0, mmax = 0;
#pragma unroll
      for (int u = 0; u < kPer; ++u) {  // thread owns left rows tid * kPer + u (consecutive: the scan below)
        const uint32_t p = tid * kPer + u;
        uint32_t m = 0, rs = 0;
        if (p < nl) {
          const uint64_t wv = sl[p];
          const uint32_t b = bins.of(wv);
          const uint32_t b0 = b ? hr[b - 1] >> 16 : 0u, b1 = hr[b] >> 16;
          if (key_bins) {  // one key a bin: the whole right bin matches
            rs = b0;
            m = b1 - b0;
          } else {
            const uint32_t key = uint32_t(wv >> 32);
            uint32_t i = b0;
            while (i < b1 && uint32_t(sr[i] >> 32) < key) ++i;
            rs = i;
            while (i < b1 && uint32_t(sr[i] >> 32) == key) ++i;
            m = i - rs;
          }
          rs_arr[p] = rs;
        }
        mloc[u] = m;
        run += m;
        mmax = max(mmax, m);
      }
      uint32_t total;
      uint32_t start = block_exclusive_scan<kThreads>(run, reinterpret_cast<uint32_t*>(scratch), &total);
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const uint32_t p = tid * kPer + u;
        if (p < nl) m_arr[p] = start;  // exclusive prefix: the first output of left row p
        start += mloc[u];
      }
      // few pairs per left row (unique-ish keys): one thread per left row writes
      // its outputs (consecutive rows -> consecutive outputs, no search);
      // otherwise output-space: every thread takes outputs t and finds its
      // left row by binary search over the prefixes
      __syncthreads();  // prefixes (m_arr) and right starts (rs_arr) complete
      BJPROF(3);  // match ranges + prefix
      // (measured: one thread per left row writing its pairs was slower than the
      // search — divergent pair counts, gaps in the output runs)
      constexpr bool per_row = false;
      const uint64_t lo = e.out_begin > base ? e.out_begin - base : 0;
      const uint64_t hi = min(uint64_t(total), e.out_end - base);
      auto write = [&](uint32_t x, uint32_t t) {
        const uint64_t wv = sl[x];
        const uint32_t jr = rs_arr[x] + (t - m_arr[x]);
        const uint64_t wr = sr[jr];
        const uint32_t lrow = uint32_t(wv), rrow = uint32_t(wr);
        if constexpr (CHECKSUM) {
          sum += fmix64((uint64_t(lrow) << 32) | rrow);
          return;
        }
        const uint64_t o = base + t - e.out_begin;
        if (e.lrows_out) __stcs(e.lrows_out + o, lrow);
        if (e.rrows_out) __stcs(e.rrows_out + o, rrow);
        for (int ci = 0; ci < cols.n; ++ci) {
          const EmitCol& c = cols.c[ci];
          const int wd = c.width;
          uint8_t* dst = c.dst + o * uint64_t(c.dstride);
          if (c.side == RL_SIDE_KEY) {
            __stcs(reinterpret_cast<long long*>(dst), key_of(wv));
          } else if (c.carry_off >= 0) {  // carried: the run's payload window (L1 / L2 resident)
            const bool left = c.side == RL_SIDE_LEFT;
            const uint64_t* pay = left ? a.pay_l : a.pay_r;
            const int words = left ? a.words_l : a.words_r;
            const uint64_t at = left ? uint64_t(l0) + lidx[x] : uint64_t(r0) + ridx[jr];
            copy_row(reinterpret_cast<const uint8_t*>(pay + at * words) + c.carry_off, dst, wd);
          } else {
            copy_row(c.src + uint64_t(c.side == RL_SIDE_LEFT ? lrow : rrow) * wd, dst, wd);
          }
        }
      };
      if (per_row) {
        for (uint32_t x = tid; x < nl; x += kThreads) {
          const uint32_t t0 = m_arr[x], t1 = x + 1 < nl ? m_arr[x + 1] : total;
          for (uint32_t t = max(t0, uint32_t(lo)); t < min(t1, uint32_t(hi)); ++t) write(x, t);
        }
      } else if (total <= uint32_t(kMaxBins)) {
        // output -> left row map in shared memory (the left bin ends are free now):
        // every row with pairs marks its first output, an inclusive max-scan fills
        // the rest — one lookup per output instead of a binary search
        uint32_t* map = omap;
        const uint32_t total4 = (total + 3) / 4;  // (whole uint4s zeroed: the scan reads them)
        for (uint32_t t = tid; t < total4; t += kThreads) reinterpret_cast<uint4*>(map)[t] = make_uint4(0, 0, 0, 0);
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const uint32_t x = tid * kPer + u;
          if (x < nl && mloc[u]) map[m_arr[x]] = x;
        }
        __syncthreads();
        {  // inclusive max-scan; warp w owns entries [w W, (w + 1) W), read as uint4 by
           // consecutive lanes (conflict-free)
          constexpr uint32_t W = uint32_t(kMaxBins / (kThreads / 32)), C = W / 128;
          const uint32_t lane = tid & 31, wp = tid >> 5;
          uint4* m4 = reinterpret_cast<uint4*>(map) + wp * (W / 4);
          const uint32_t lo4 = wp * (W / 4), lim4 = total4 > lo4 ? total4 - lo4 : 0u;
          uint32_t* wmax = reinterpret_cast<uint32_t*>(scratch);
          uint32_t wm = 0;
#pragma unroll
          for (uint32_t i = 0; i < C; ++i) {
            const uint32_t q = i * 32 + lane;
            if (q < lim4) {
              const uint4 c = m4[q];
              wm = max(wm, max(max(c.x, c.y), max(c.z, c.w)));
            }
          }
          wm = __reduce_max_sync(0xffffffffu, wm);
          if (lane == 0) wmax[wp] = wm;
          __syncthreads();
          uint32_t run_max = 0;
          for (uint32_t w2 = 0; w2 < wp; ++w2) run_max = max(run_max, wmax[w2]);
#pragma unroll
          for (uint32_t i = 0; i < C; ++i) {
            const uint32_t q = i * 32 + lane;
            const uint4 c = q < lim4 ? m4[q] : make_uint4(0, 0, 0, 0);
            uint32_t incl = max(max(c.x, c.y), max(c.z, c.w));
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= uint32_t(o)) incl = max(incl, x);
            }
            uint32_t excl = __shfl_up_sync(0xffffffffu, incl, 1);
            if (lane == 0) excl = 0;
            if (q < lim4) {
              uint4 o4;
              o4.x = max(max(run_max, excl), c.x);
              o4.y = max(o4.x, c.y);
              o4.z = max(o4.y, c.z);
              o4.w = max(o4.z, c.w);
              m4[q] = o4;
            }
            run_max = max(run_max, __shfl_sync(0xffffffffu, incl, 31));
          }
        }
        __syncthreads();
        BJPROF(4);  // output -> left row map
        if (CHECKSUM || hi - lo < uint64_t(2 * kThreads)) {  // (a selective run: a few outputs)
          for (uint64_t t = lo + tid; t < hi; t += kThreads) write(map[t], uint32_t(t));
        } else {
          // kU outputs a thread at a time, column by column: every load of a column
          // (carried words from the run's window, gathered rows) issued before its
          // stores, instead of one dependent load -> store chain per output
          constexpr int kU = 4;
          for (uint64_t t0 = lo + tid; t0 < hi; t0 += uint64_t(kU) * kThreads) {
            uint32_t xs[kU], jrs[kU];
            bool ok[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              const uint64_t t = t0 + uint64_t(u) * kThreads;
              ok[u] = t < hi;
              const uint32_t x = ok[u] ? map[t] : 0u;
              xs[u] = x;
              jrs[u] = ok[u] ? rs_arr[x] + (uint32_t(t) - m_arr[x]) : 0u;
            }
            auto out_row = [&](int u) { return base + t0 + uint64_t(u) * kThreads - e.out_begin; };
            if (e.lrows_out) {
#pragma unroll
              for (int u = 0; u < kU; ++u)
                if (ok[u]) __stcs(e.lrows_out + out_row(u), uint32_t(sl[xs[u]]));
            }
            if (e.rrows_out) {
#pragma unroll
              for (int u = 0; u < kU; ++u)
                if (ok[u]) __stcs(e.rrows_out + out_row(u), uint32_t(sr[jrs[u]]));
            }
            for (int ci = 0; ci < cols.n; ++ci) {
              const EmitCol& c = cols.c[ci];
              const int wd = c.width;
              if (c.side == RL_SIDE_KEY) {
#pragma unroll
                for (int u = 0; u < kU; ++u)
                  if (ok[u]) __stcs(reinterpret_cast<long long*>(c.dst + out_row(u) * uint64_t(c.dstride)), key_of(sl[xs[u]]));
                continue;
              }
              const bool left = c.side == RL_SIDE_LEFT;
              auto src_of = [&](int u) -> const uint8_t* {
                if (c.carry_off >= 0) {
                  const uint64_t* pay = left ? a.pay_l : a.pay_r;
                  const int words = left ? a.words_l : a.words_r;
                  const uint64_t at = left ? uint64_t(l0) + lidx[xs[u]] : uint64_t(r0) + ridx[jrs[u]];
                  return reinterpret_cast<const uint8_t*>(pay + at * words) + c.carry_off;
                }
                const uint32_t row = left ? uint32_t(sl[xs[u]]) : uint32_t(sr[jrs[u]]);
                return c.src + uint64_t(row) * wd;
              };
              if (c.vec == 8) {
                unsigned long long v[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u)
                  v[u] = ok[u] ? ld_row(reinterpret_cast<const unsigned long long*>(src_of(u))) : 0ull;
#pragma unroll
                for (int u = 0; u < kU; ++u)
                  if (ok[u]) __stcs(reinterpret_cast<unsigned long long*>(c.dst + out_row(u) * uint64_t(c.dstride)), v[u]);
              } else if (c.vec == 16) {
                uint4 v[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u)
                  v[u] = ok[u] ? ld_row(reinterpret_cast<const uint4*>(src_of(u))) : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int u = 0; u < kU; ++u)
                  if (ok[u]) __stcs(reinterpret_cast<uint4*>(c.dst + out_row(u) * uint64_t(c.dstride)), v[u]);
              } else {
#pragma unroll
                for (int u = 0; u < kU; ++u)
                  if (ok[u]) copy_row(src_of(u), c.dst + out_row(u) * uint64_t(c.dstride), wd);
              }
            }
          }
        }
      } else {
        for (uint64_t t = lo + tid; t < hi; t += kThreads) {
          uint32_t x = 0, y = nl;  // largest p with pre[p] <= t
          while (y - x > 1) {
            const uint32_t mid = (x + y) >> 1;
            if (m_arr[mid] <= uint32_t(t)) x = mid;
            else y = mid;
          }
          write(x, uint32_t(t));
        }
      }
      __syncthreads();  // smem reused by the next run
      BJPROF(5);  // outputs written
#ifdef RL_BJ_PROFILE
      if (threadIdx.x == 0) atomicAdd(&g_bj_prof[8], 1ull);
#endif
    }
  }
  if constexpr (CHECKSUM) {  // mod 2^64: one atomic per warp
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if ((tid & 31) == 0 && sum) atomicAdd(e.checksum, (unsigned long long)sum);
  }
}

constexpr size_t kEmitSmem = size_t(kBjCap) * 8 * 3 + size_t(kMaxBins) * 4 * 2 + size_t(kBjCap) * 2 * 3 +
                             (kThreads / 32 + 2) * 8 + size_t(kMaxG + 1) * 8 + (3 * kMaxG + 2 + 128 + 4) * 4;

// ---------------------------------------------------------------- host
static size_t side_bytes(int64_t n, int words, int levels) {
  return align_up(radix::bj_side_workspace_bytes(n, words, levels), 256);
}
static uint32_t groups_of(int levels) { return levels == 3 ? Geo<3>::kGroups : Geo<2>::kGroups; }
static int group_size(int levels) { return levels == 3 ? Geo<3>::G : Geo<2>::G; }

// The listed matches of selective runs (two levels only): a listed run holds at
// most 1/8 of its rows in pairs, so (nl + nr) / 8 entries always suffice.
static size_t sel_cap_of(int64_t nl, int64_t nr, int levels) {
  return levels == 2 ? size_t((nl + nr) / 8) + kSelMax : 0;
}
static size_t sel_bytes(int64_t nl, int64_t nr, int levels) {
  const size_t cap = sel_cap_of(nl, nr, levels);
  if (!cap) return 0;
  const size_t runs = size_t(groups_of(levels)) * group_size(levels);
  return align_up(16 * cap, 256) + align_up(4 * cap, 256) + align_up(4 * runs, 256);
}

size_t workspace_bytes(int64_t nl, int64_t nr, int lwords, int rwords) {
  const int lv = radix::bj_levels(nl, nr);
  const size_t runs = size_t(groups_of(lv)) * group_size(lv);
  return side_bytes(nl, lwords, lv) + side_bytes(nr, rwords, lv) + align_up(sizeof(uint32_t) * runs, 256) +
         align_up(sizeof(uint64_t) * groups_of(lv), 256) + align_up(sizeof(int64_t) * 4, 256) +
         sel_bytes(nl, nr, lv) + 256;
}

template <bool CK, int LV>
static int emit_grid_of() {
  static int cache[kMaxDevices] = {};
  return per_device(cache, [] {
    if (cudaFuncSetAttribute(bj_emit_kernel<CK, LV>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kEmitSmem)) !=
        cudaSuccess) {
      cudaGetLastError();
      return -1;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bj_emit_kernel<CK, LV>, kThreads, kEmitSmem) !=
            cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    return per_sm * device_sm_count();
  });
}

// A side's carried columns: natural alignment inside <= 16 bytes of payload
// words, widest first; all of them or none (-> gathered by row id).
static int make_carry(const rl_column* cols, int n, radix::BjCarry* cy, int32_t* offs) {
  *cy = radix::BjCarry{};
  if (n <= 0) return RL_OK;
  if (!cols || n > radix::kBjMaxCarryCols) return n > radix::kBjMaxCarryCols ? RL_OK : RL_ERR_BAD_ARG;
  int order[radix::kBjMaxCarryCols];
  for (int i = 0; i < n; ++i) {
    if (!cols[i].src || cols[i].width <= 0) return RL_ERR_BAD_ARG;
    order[i] = i;
  }
  std::sort(order, order + n, [&](int x, int y) { return cols[x].width > cols[y].width; });
  int at = 0;
  for (int k = 0; k < n; ++k) {
    const int w = cols[order[k]].width;
    const int al = (w % 8 == 0) ? 8 : (w % 4 == 0) ? 4 : 1;
    at = (at + al - 1) / al * al;
    offs[order[k]] = at;
    at += w;
  }
  if (at > 8 * radix::kBjMaxCarryWords) return RL_OK;  // too wide: gather instead
  cy->n = n;
  cy->words = (at + 7) / 8;
  for (int i = 0; i < n; ++i) {
    cy->src[i] = static_cast<const uint8_t*>(cols[i].src);
    cy->width[i] = cols[i].width;
    cy->off[i] = offs[i];
  }
  return RL_OK;
}

int plan(const int64_t* lkeys, int64_t nl, const int64_t* rkeys, int64_t nr, const rl_column* lcarry, int nlc,
         const rl_column* rcarry, int nrc, void* ws, size_t ws_bytes, rl_bjoin_plan* out, cudaStream_t stream) {
  if (!out || nl < 1 || nr < 1 || nlc < 0 || nrc < 0) return RL_ERR_BAD_ARG;
  *out = rl_bjoin_plan{};
  radix::BjCarry lc, rc;
  int st = make_carry(lcarry, nlc, &lc, out->carry_off_left);
  if (st == RL_OK) st = make_carry(rcarry, nrc, &rc, out->carry_off_right);
  if (st != RL_OK) return st;
  if (reinterpret_cast<uintptr_t>(ws) % 256 != 0 || ws_bytes < workspace_bytes(nl, nr, lc.words, rc.words))
    return RL_ERR_WORKSPACE;
  const int lv = radix::bj_levels(nl, nr);
  const size_t runs = size_t(groups_of(lv)) * group_size(lv);
  char* base = static_cast<char*>(ws);
  const size_t wl = side_bytes(nl, lc.words, lv), wr = side_bytes(nr, rc.words, lv);
  uint32_t* counts = reinterpret_cast<uint32_t*>(base + wl + wr);
  uint64_t* gtot = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(counts) + align_up(sizeof(uint32_t) * runs, 256));
  int64_t* scalars = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(gtot) +
                                                align_up(sizeof(uint64_t) * groups_of(lv), 256));
  BjSide L, R;
  st = radix::bj_partition(lkeys, nl, rkeys, nr, lc, rc, base, wl, base + wl, wr, stream, &L, &R);
  if (st != RL_OK) return st;
  PlanArgs a{L.rows, R.rows, L.sub_off, R.sub_off, L.flags, R.flags, counts, gtot, lv, scalars,
             reinterpret_cast<const long long*>(lkeys), L.pay, R.pay, L.words, R.words};
  const size_t cap = sel_cap_of(nl, nr, lv);
  if (cap && std::getenv("RL_BJ_NO_SEL") == nullptr) {
    char* sb = reinterpret_cast<char*>(scalars) + align_up(sizeof(int64_t) * 4, 256);
    a.sel_pairs = reinterpret_cast<ulonglong2*>(sb);
    a.sel_idx = reinterpret_cast<uint32_t*>(sb + align_up(16 * cap, 256));
    a.run_sel = reinterpret_cast<uint32_t*>(sb + align_up(16 * cap, 256) + align_up(4 * cap, 256));
    a.sel_cursor = reinterpret_cast<unsigned long long*>(scalars + 2);
    a.sel_cap = uint32_t(std::min<size_t>(cap, 0xFFFFFFFFu));
    if (cudaMemsetAsync(scalars + 2, 0, sizeof(int64_t), stream) != cudaSuccess) return rl_cuda_status(cudaGetLastError());
  }
  const int grid = device_sm_count() * 3;
  if (lv == 3) bj_count_kernel<3><<<grid, kThreads, 0, stream>>>(a);
  else bj_count_kernel<2><<<grid, kThreads, 0, stream>>>(a);
  bj_scan_kernel<<<1, 1024, 0, stream>>>(a, groups_of(lv));
  count_launches(2);
  out->rows_left = L.rows;
  out->rows_right = R.rows;
  out->sub_off_left = L.sub_off;
  out->sub_off_right = R.sub_off;
  out->flags_left = L.flags;
  out->flags_right = R.flags;
  out->counts = counts;
  out->offsets = gtot;
  out->scalars = scalars;
  out->levels = lv;
  out->left_keys = lkeys;
  out->pay_left = L.pay;
  out->pay_right = R.pay;
  out->sel_pairs = a.sel_pairs;
  out->sel_idx = a.sel_idx;
  out->run_sel = a.run_sel;
  out->words_left = L.words;
  out->words_right = R.words;
  out->carry_cols_left = lc.n;
  out->carry_cols_right = rc.n;
  for (int i = 0; i < lc.n; ++i) {
    out->carry_src_left[i] = lc.src[i];
    out->carry_width_left[i] = lc.width[i];
  }
  for (int i = 0; i < rc.n; ++i) {
    out->carry_src_right[i] = rc.src[i];
    out->carry_width_right[i] = rc.width[i];
  }
  return rl_cuda_status(cudaGetLastError());
}

// The carried payload offset of an output column, or -1 (gathered by row id).
static int carried_offset(const rl_bjoin_plan* p, const rl_column& c) {
  const bool left = c.side == RL_SIDE_LEFT;
  const int n = left ? p->carry_cols_left : p->carry_cols_right;
  for (int i = 0; i < n; ++i) {
    const void* src = left ? p->carry_src_left[i] : p->carry_src_right[i];
    const int w = left ? p->carry_width_left[i] : p->carry_width_right[i];
    if (src == c.src && w == c.width) return left ? p->carry_off_left[i] : p->carry_off_right[i];
  }
  return -1;
}

int emit(const rl_bjoin_plan* p, uint64_t out_begin, uint64_t out_end, uint32_t* lrows_out, uint32_t* rrows_out,
         const rl_column* columns, int n_columns, cudaStream_t stream, uint64_t* checksum = nullptr,
         const int32_t* dst_strides = nullptr) {
  if (!p || out_end < out_begin || n_columns < 0 || n_columns > kMaxCols || (n_columns && !columns))
    return RL_ERR_BAD_ARG;
  if (out_end == out_begin) return RL_OK;
  Cols cs;
  cs.n = n_columns;
  for (int i = 0; i < n_columns; ++i) {
    const rl_column& c = columns[i];
    if (c.width < 0 || !c.dst) return RL_ERR_BAD_ARG;
    if (c.side == RL_SIDE_KEY) {
      if (c.width != 8) return RL_ERR_BAD_ARG;
    } else if (c.side != RL_SIDE_LEFT && c.side != RL_SIDE_RIGHT) {
      return RL_ERR_BAD_ARG;
    } else if (c.width > 0 && !c.src) {
      return RL_ERR_BAD_ARG;
    }
    const int co = c.side == RL_SIDE_KEY ? -1 : carried_offset(p, c);
    // one aligned vector load a source row: carried words are 8-byte aligned rows
    // of 8 x words bytes in 256-byte-aligned workspace; gathered rows are src + row x width
    int vec = 0;
    if (c.side != RL_SIDE_KEY && (c.width == 8 || c.width == 16)) {
      if (co >= 0) {
        const int words = c.side == RL_SIDE_LEFT ? p->words_left : p->words_right;
        const uintptr_t pay = reinterpret_cast<uintptr_t>(c.side == RL_SIDE_LEFT ? p->pay_left : p->pay_right);
        if (((pay | uintptr_t(co)) % uintptr_t(c.width)) == 0 && (8 * words) % c.width == 0) vec = c.width;
      } else if (reinterpret_cast<uintptr_t>(c.src) % uintptr_t(c.width) == 0) {
        vec = c.width;
      }
    }
    // a row-interleaved destination: stride >= width, naturally aligned for the vector stores
    const int64_t stride = dst_strides && dst_strides[i] ? dst_strides[i] : c.width;
    if (stride < c.width || (stride != c.width && (c.width != 8 && c.width != 16)) ||
        (stride != c.width && (stride % c.width != 0 || reinterpret_cast<uintptr_t>(c.dst) % uintptr_t(c.width) != 0)))
      return RL_ERR_BAD_ARG;
    cs.c[i] = EmitCol{static_cast<const uint8_t*>(c.src), static_cast<uint8_t*>(c.dst), c.width, c.side, co, vec, stride};
  }
  const int lv = p->levels == 3 ? 3 : 2;
  const int grid = lv == 3 ? (checksum ? emit_grid_of<true, 3>() : emit_grid_of<false, 3>())
                           : (checksum ? emit_grid_of<true, 2>() : emit_grid_of<false, 2>());
  if (grid < 1) return rl_cuda_status(cudaErrorInvalidConfiguration);
  EmitArgs e;
  e.p = PlanArgs{p->rows_left, p->rows_right, p->sub_off_left, p->sub_off_right, p->flags_left, p->flags_right,
                 p->counts, p->offsets, lv, p->scalars, reinterpret_cast<const long long*>(p->left_keys),
                 p->pay_left, p->pay_right, p->words_left, p->words_right};
  e.p.sel_pairs = static_cast<ulonglong2*>(const_cast<void*>(p->sel_pairs));
  e.p.sel_idx = const_cast<uint32_t*>(p->sel_idx);
  e.p.run_sel = const_cast<uint32_t*>(p->run_sel);
  e.out_begin = out_begin;
  e.out_end = out_end;
  e.no_sel = std::getenv("RL_BJ_NO_SEL") != nullptr ? 1 : 0;
  e.lrows_out = lrows_out;
  e.rrows_out = rrows_out;
  e.checksum = reinterpret_cast<unsigned long long*>(checksum);
  if (lv == 3) {
    if (checksum) bj_emit_kernel<true, 3><<<grid, kThreads, kEmitSmem, stream>>>(e, cs);
    else bj_emit_kernel<false, 3><<<grid, kThreads, kEmitSmem, stream>>>(e, cs);
  } else {
    if (checksum) bj_emit_kernel<true, 2><<<grid, kThreads, kEmitSmem, stream>>>(e, cs);
    else bj_emit_kernel<false, 2><<<grid, kThreads, kEmitSmem, stream>>>(e, cs);
  }
  count_launches(1);
  return rl_cuda_status(cudaGetLastError());
}

}  // namespace bjoin
}  // namespace rl

extern "C" {

RL_API size_t rl_bjoin_workspace_bytes(int64_t n_left, int64_t n_right, int32_t left_words, int32_t right_words) {
  return rl::bjoin::workspace_bytes(std::max<int64_t>(n_left, 1), std::max<int64_t>(n_right, 1), left_words,
                                    right_words);
}

RL_API int rl_bjoin_carry_words(const rl_column* columns, int32_t n_columns) {
  rl::radix::BjCarry cy;
  int32_t offs[rl::radix::kBjMaxCarryCols];
  if (rl::bjoin::make_carry(columns, n_columns, &cy, offs) != RL_OK) return -1;
  return cy.words;
}

RL_API int rl_bjoin_plan_build(const int64_t* left_keys, int64_t n_left, const int64_t* right_keys, int64_t n_right,
                               const rl_column* left_carry, int32_t n_left_carry, const rl_column* right_carry,
                               int32_t n_right_carry, void* ws, size_t ws_bytes, rl_bjoin_plan* plan, void* stream) {
  return rl::bjoin::plan(left_keys, n_left, right_keys, n_right, left_carry, n_left_carry, right_carry, n_right_carry,
                         ws, ws_bytes, plan, static_cast<cudaStream_t>(stream));
}

RL_API int rl_bjoin_expand(const rl_bjoin_plan* plan, uint64_t out_begin, uint64_t out_end, uint32_t* left_rows_out,
                           uint32_t* right_rows_out, const rl_column* columns, int32_t n_columns, void* stream) {
  return rl::bjoin::emit(plan, out_begin, out_end, left_rows_out, right_rows_out, columns, n_columns,
                         static_cast<cudaStream_t>(stream));
}

RL_API int rl_bjoin_expand_strided(const rl_bjoin_plan* plan, uint64_t out_begin, uint64_t out_end,
                                   uint32_t* left_rows_out, uint32_t* right_rows_out, const rl_column* columns,
                                   int32_t n_columns, const int32_t* dst_strides, void* stream) {
  return rl::bjoin::emit(plan, out_begin, out_end, left_rows_out, right_rows_out, columns, n_columns,
                         static_cast<cudaStream_t>(stream), nullptr, dst_strides);
}

RL_API int rl_bjoin_pair_checksum(const rl_bjoin_plan* plan, uint64_t out_begin, uint64_t out_end, uint64_t* sum_out,
                                  void* stream) {
  if (!sum_out) return RL_ERR_BAD_ARG;
  return rl::bjoin::emit(plan, out_begin, out_end, nullptr, nullptr, nullptr, 0, static_cast<cudaStream_t>(stream),
                         sum_out);
}

}  // extern "C"

#ifdef RL_BJ_PROFILE
extern "C" __attribute__((visibility("default"))) int rl_debug_bj_prof(unsigned long long* out16, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out16, rl::bjoin::g_bj_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(rl::bjoin::g_bj_prof, z, sizeof(z));
  }
  return 0;
}
#endif
