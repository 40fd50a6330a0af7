// radix_sort.cu — K1 (digit histograms) + K2 (onesweep digit passes), fused
// into ONE persistent cooperative kernel per sort.
//
// Stable LSD radix sort of 64-bit key words carrying uint32 row ids. It
// replaces the reference's stable argsorts:
//   _stable_key_order   /root/reference/pkg/src/relab/tensorpath.py:62-75
//   _stable_axis_order  /root/reference/pkg/src/relab/tensorpath.py:206-229
//
// Design (B200, HBM/shared-memory bound integer work — no tensor cores):
//   * One cooperative launch of 2 CTAs per SM (all co-resident). Phases are
//     separated by a grid barrier instead of kernel boundaries, so a sort is
//     a single launch: digits that are constant over the input (pass
//     skipping: a 1e6-domain key has only 3 active 8-bit digits of 8) cost
//     nothing, and no launch gaps separate the passes.
//   * Phase H reads the keys once and builds all eight 8-bit digit
//     histograms (shared-memory counters, one global atomic per bin per
//     CTA). For a gathered key (a refinement step of a multi-key sort, or a
//     Bytes word) it also materialises the transformed key words so the
//     first digit pass streams them contiguously.
//   * Every CTA then derives the pass plan itself from the global
//     histograms (active digits, ping-pong buffers, global digit bases): no
//     plan kernel, no host synchronisation.
//   * Each active digit pass is a onesweep pass over tiles of 3072 keys that
//     CTAs claim in increasing order from an atomic counter. A CTA prefetches
//     its next tile with TMA bulk copies (cp.async.bulk → shared memory,
//     mbarrier completion) while it ranks and scatters the current one:
//       - early counts: per-warp digit histograms (shared atomics) published
//         as the tile's aggregate before ranking (decoupled look-back);
//       - stable warp multisplit rank: peers of a digit from a shared
//         atomicOr mask, the leader bumps the warp's running digit offset;
//       - the tile is staged in digit order in place, the look-back resolves
//         the global digit offsets (a window of predecessor status words per
//         round trip), and the staged tile is written out so every digit run
//         is a contiguous burst.
//
// Wide-key hybrid (raw int64 keys, n >= 2^18): when the top 16 key bits
// spread the input into sub-buckets that fit on chip, the sort runs only
// two onesweep passes — digit 6 then digit 7, i.e. stably by the top 16
// bits; the digit-7 pass also writes the 65536 sub-bucket starts from its
// look-back prefixes (its input is digit-6 ordered). A local phase then
// sorts every sub-bucket in shared memory ((sub-bucket, d5) counting
// scatter, then each row's rank by (key, row id) among the rows equal in
// their top 24 bits) and writes the final keys, permutation and fused
// gathers: 2 passes + 1 streaming phase over HBM instead of 8 passes. A
// sub-bucket larger than kLocalCap (skewed top bits) is caught after the
// two passes and the same launch runs the LSD passes instead.
//
// Scatter hybrid (raw int64 keys, n >= 2^22 — the cfg2 path): the rows reach
// their sub-buckets by exact per-chunk counts and two NON-stable counting
// passes (the local phase orders every sub-bucket by (key, row id) anyway),
// keys packed to their varying bits first; see "scatter hybrid" below.
//
// Key transform (self-inverse): int64 ascending  u = x ^ 2^63;
// descending u = ~x ^ 2^63 (the reference's np.invert, tensorpath.py:215,
// keeps ties in ascending row order). Bytes words are built big-endian
// from (complemented when descending) bytes, zero padded
// (tensorpath.py:220-225).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "keypack.cuh"
#include "bjoin.cuh"

namespace rl {
namespace radix {

#ifndef RL_ONESWEEP_ITEMS
#define RL_ONESWEEP_ITEMS 14
#endif
#ifndef RL_ONESWEEP_MIN_BLOCKS
#define RL_ONESWEEP_MIN_BLOCKS 2
#endif
#ifndef RL_LOOKBACK_WINDOW
#define RL_LOOKBACK_WINDOW 4
#endif
#ifndef RL_RANK_MODE
#define RL_RANK_MODE 2  // 1: ballot match_any, 2: shared atomicOr match (fewest instructions)
#endif

constexpr int kBits = 8;
constexpr int kBins = 1 << kBits;
constexpr int kPasses = 64 / kBits;
constexpr int kThreads = 256;  // == kBins: one digit per thread in the tile scan
constexpr int kItems = RL_ONESWEEP_ITEMS;
constexpr int kTile = kThreads * kItems;
constexpr int kWarps = kThreads / 32;
constexpr int kLookback = RL_LOOKBACK_WINDOW;
#ifndef RL_HIST_UNROLL
#define RL_HIST_UNROLL 16
#endif
constexpr int kHistUnroll = RL_HIST_UNROLL;
constexpr int kStamps = 2 + kPasses + 2;  // per-phase globaltimer stamps + the path taken (profiling)
// wide-key hybrid
#ifndef RL_LOCAL_CAP
#define RL_LOCAL_CAP 2560
#endif
constexpr int kLocalCap = RL_LOCAL_CAP;    // rows of one on-chip local run (and the largest sub-bucket)
constexpr int kSubBuckets = 1 << 16;       // (d7, d6) sub-buckets
constexpr int kGroupSubs = 16;             // sub-buckets claimed per local work item
constexpr int64_t kHybridMinRows = 1 << 18;
constexpr int64_t kCountAllRows = int64_t(1) << 22;  // raw keys below this: all 8 histograms up front
constexpr uint32_t kHybridEpoch = kPasses; // LSD after a hybrid fallback publishes epoch PASS + 1 + 8

static_assert(kThreads == kBins, "tile scan maps one digit per thread");
static_assert(kStamps == RL_SORT_STAMPS, "stamp layout is part of the ABI");

enum KeyMode : int { kRawAsc = 0, kRawDesc = 1, kMaterialized = 2 };
enum SortMode : int { kModeLsd = 0, kModeHybrid = 1, kModeScatter = 2 };  // hybrid/scatter: try the wide-key path first

// scatter hybrid: exact per-chunk 16-bit counts, then two non-stable
// counting passes (digit 7; digit 6 inside every digit-7 bucket), then the local phase
constexpr int kScatThreads = 1024;                 // histogram kernel: one CTA per SM
constexpr int kScatWords = (1 << 16) / 2;          // sub-bucket counters, packed u16 pairs
constexpr int kMaxChunks = 160;
constexpr int kHistReps = 8;                       // digit-histogram replicas: no grid-deep same-address atomics
constexpr int kD7Reps = 8;                         // digit-7 count replicas: no 148-deep same-address atomics
constexpr int64_t kScatterMinRows = int64_t(1) << 22;  // below: the histogram kernel counts every digit at once
constexpr int64_t kChunkMinRows = 32768;            // small inputs: fewer chunk histograms (128 KB each)
#ifndef RL_PASS_THREADS
#define RL_PASS_THREADS 512
#endif
#ifndef RL_PASS_CTAS_PER_SM
#define RL_PASS_CTAS_PER_SM 2
#endif
constexpr int kPThreads = RL_PASS_THREADS;         // counting passes
#ifndef RL_PASS_ITEMS
#define RL_PASS_ITEMS 8
#endif
constexpr int kPItems = RL_PASS_ITEMS;
constexpr int kPTile = kPThreads * kPItems;        // rows per staged tile
constexpr size_t kPStage = size_t(kPTile) * 12;    // staged keys + row ids (also reduction scratch)
constexpr size_t kPSmem = kPStage + 3 * 256 * 4 + 64 * 4;
enum SrcMode : int { kSrcInt64 = 0, kSrcInt64Gather = 1, kSrcBytes = 2, kSrcWords = 3 };


__device__ __forceinline__ uint64_t bytes_word(const uint8_t* row, int width, int word, int desc) {
  uint64_t v = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    int idx = word * 8 + b;
    uint32_t byte = 0;
    if (idx < width) {
      byte = row[idx];
      if (desc) byte = (~byte) & 0xFFu;
    }
    v = (v << 8) | byte;
  }
  return v;
}

constexpr int kMaxFusedColumns = 8;
struct FusedColumns {
  rl_column c[kMaxFusedColumns];
  int n;
};

__device__ __forceinline__ void gather_fused(const FusedColumns& g, uint32_t row, uint64_t o) {
  for (int ci = 0; ci < g.n; ++ci) {
    const int w = g.c[ci].width;
    copy_row(static_cast<const uint8_t*>(g.c[ci].src) + uint64_t(row) * w, static_cast<uint8_t*>(g.c[ci].dst) + o * w, w);
  }
}

struct SortArgs {
  // phase H source
  const void* col;
  const uint32_t* perm_in;   // row ids of the input slots (NULL = identity)
  uint64_t* materialized;    // gathered/bytes modes: transformed key words
  int64_t n;
  int width, word, desc, src_mode, key_mode;
  // passes
  const void* orig_keys;     // what the first active pass streams (raw int64 or materialised words)
  uint64_t* keys_a;
  uint64_t* keys_b;
  uint32_t* vals_a;
  uint32_t* vals_b;
  int64_t* out_keys;         // final sorted int64 keys (optional, raw modes)
  uint32_t* out_vals;        // final permutation
  int mode;                  // SortMode
  int count_all;             // raw keys: the histogram kernel counted every digit (small n)
  // zeroed per call
  uint32_t* ghist;           // [kHistReps][kPasses][kBins]: CTA c adds into replica c % kHistReps
  uint32_t* tile_counter;    // [2][kPasses] (first attempt, LSD after a hybrid fallback)
  uint32_t* grid_bar;        // grid barrier arrivals
  uint32_t* flags;           // [0] LSD fallback (a sub-bucket exceeds kLocalCap, ...), [1] local work-item counter,
                             // [3] scatter path: pass-B tile counter,
                             // [4..5] raw int64 keys: OR of (key ^ first key) = the varying bits (u64),
  uint32_t* sub_off;         // [kSubBuckets + 1] sub-bucket starts, hybrid (not zeroed)
  uint64_t* status;          // [num_tiles][kBins] look-back words (epoch = pass + 1)
  unsigned long long* stamps;  // optional [kStamps] globaltimer ns (device)
  // columns gathered by the final permutation inside the last pass
  // (Relation.take fused into the sort: dst row o = src row perm[o])
  FusedColumns gather;
  // scatter hybrid (kModeScatter)
  uint32_t* chunk_cnt;       // [kMaxChunks][kScatWords] rows per (chunk, sub-bucket), packed u16 pairs
  uint32_t* cur7;            // [kBins] rows placed per digit-7 bucket so far (zeroed)
  uint32_t* d7rep;           // [kD7Reps][kBins] digit-7 counts, CTA c adds into replica c % kD7Reps (zeroed)
  uint32_t* cur16;           // [kSubBuckets] rows placed per sub-bucket so far (zeroed)
  uint32_t* d7_base;         // [kBins + 1] digit-7 bucket starts
  uint4* items;              // pass-B tiles (digit-7 bucket, first row, end row)
  uint32_t* meta;            // [0] pass-B tiles
  int chunks;                // input chunks = CTAs of the histogram and digit-7 kernels
  int allow_pk;              // scatter path: packed rows allowed (RL_NO_PACKED_ROWS=1 turns them off)
  // bucket join (bj_partition): both sides share one pack code, set in flags[6]
  // before the chunk counts, checked against the LEFT side's first key
  int pack_given;
  const long long* k0_src;   // the key whose constant bits every key must share (default: col[0])
  int bj;                    // keep going with < 4 varying digits (the join needs the sub-buckets)
  // bucket join: payload words carried with every row through the counting
  // passes (CW u64 words per row; the side's output columns packed in)
  int carry_n;               // carried columns
  const uint8_t* carry_src[4];
  int carry_width[4];
  int carry_off[4];          // byte offset in the row's payload words
  uint8_t* carry_dst[4];     // sort with carried columns: where the local phase writes them (dst row o)
  int cw;                    // sort with carried columns: payload words a row (0: none)
  int idw;                   // carried columns of <= 4 bytes: keys that do not pack carry the row id in the
                             // word's low half, the columns' bytes in its high half (no row-id stream)
  uint64_t* pay_a;           // [n * CW] parallel to keys_a
  uint64_t* pay_b;           // [n * CW] parallel to keys_b
  // three-level scatter (n above ~65536 x kLocalCap): digit 5 inside every
  // (d7, d6) sub-bucket, the local phase over 2^24 sub-sub-buckets
  int levels;                // 2 or 3
  uint32_t* sub3_off;        // [kSub3 + 1] sub-sub-bucket starts
  uint32_t* cur24;           // [kSub3] rows placed per sub-sub-bucket so far (zeroed)
  uint32_t* tile3;           // [kSubBuckets + 1] first level-3 tile of every sub-bucket (prefix)
  uint32_t* tmap;            // [level-3 tiles] uint4 (sub-bucket, first row, end row) of every tile
};
constexpr int kSub3 = 1 << 24;  // (d7, d6, d5) sub-sub-buckets

// Global digit count (pass p, digit d): the sum of the histogram replicas.
__device__ __forceinline__ uint32_t ghist_at(const SortArgs& a, int p, int d) {
  uint32_t c = 0;
#pragma unroll
  for (int r = 0; r < kHistReps; ++r) c += __ldcg(a.ghist + (r * kPasses + p) * kBins + d);
  return c;
}

__device__ __forceinline__ uint64_t load_key(const SortArgs& a, int64_t i) {
  if (a.src_mode == kSrcInt64) return xform(uint64_t(__ldg(static_cast<const long long*>(a.col) + i)), a.desc);
  if (a.src_mode == kSrcWords) return __ldg(static_cast<const unsigned long long*>(a.col) + i);
  const uint64_t row = a.perm_in ? uint64_t(__ldg(a.perm_in + i)) : uint64_t(i);
  if (a.src_mode == kSrcInt64Gather) return xform(uint64_t(ld_row(static_cast<const long long*>(a.col) + row)), a.desc);
  return bytes_word(static_cast<const uint8_t*>(a.col) + row * uint64_t(a.width), a.width, a.word, a.desc);
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Grid-wide barrier for the co-resident cooperative grid: the k-th barrier
// completes when k * gridDim.x arrivals have been counted.
__device__ __forceinline__ void grid_sync(uint32_t* arrivals, uint32_t k) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(arrivals, 1u);
    const uint32_t target = k * gridDim.x;
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(arrivals) : "memory");
      if (v >= target) break;
      __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// Shared memory of one CTA during a pass: two tile buffers (one being
// processed — loaded by TMA, then reused as the digit-ordered staging area —
// and one being prefetched), per-warp digit counters and match masks.
constexpr size_t kBufBytes = size_t(kTile) * 12;  // keys (8 B) then row ids (4 B)
constexpr size_t kBarOffset = 2 * kBufBytes + size_t(kWarps) * kBins * 4 * 2 + size_t(kBins) * 4 + 64 * 4;
constexpr size_t kPassSmemBytes = kBarOffset + 64;
// + the plan kept for the whole kernel: global digit bases [kPasses][kBins] + flags
// ---------------------------------------------------------------- hybrid
// Shared memory of the local phase (reuses the pass buffers): load buffer
// A, scattered buffer B, the (sub-bucket, d5) bin counters/cursors, the
// list of bins too long for a one-thread fix-up, and scalars.
constexpr int kLocalBins = kGroupSubs * kBins;  // (top16 - first of group, d5)
constexpr int kBigList = 128;
constexpr size_t kLocAKeys = size_t(kLocalCap + 2) * 8;  // +2 / +4: TMA copies start 16-byte aligned
constexpr size_t kLocAVals = size_t(kLocalCap + 4) * 4;
constexpr size_t kLocABytes = (kLocAKeys + kLocAVals + 15) / 16 * 16;
constexpr size_t kLocA = 0;  // two run buffers (double-buffered TMA loads)
constexpr size_t kLocBk = kLocA + 2 * kLocABytes;
constexpr size_t kLocBv = kLocBk + size_t(kLocalCap) * 8;
constexpr size_t kLocHist = kLocBv + size_t(kLocalCap) * 4;
constexpr size_t kLocBig = kLocHist + size_t(kLocalBins) * 4;
// the scatter path's local phase (BAL) scatters the keys inside their own load
// buffer (every key is in registers before the first barrier), so B's key
// half and the 4096 counters give way to B's row ids + 8192 counters
#ifndef RL_LOCAL_BAL_BITS
#define RL_LOCAL_BAL_BITS 12
#endif
constexpr int kLocalBinsBal = 1 << RL_LOCAL_BAL_BITS;
constexpr size_t kLocBvBal = kLocBk;
constexpr size_t kLocHistBal = kLocBvBal + (size_t(kLocalCap) * 4 + 15) / 16 * 16;
static_assert(kLocHistBal + size_t(kLocalBinsBal) * 4 <= kLocBig, "8192 counters fit in B + the 4096 counters");
constexpr size_t kLocMisc = kLocBig + size_t(kBigList) * 4;
// idw (keys that do not pack, <= 4 carried bytes): a run buffer holds the keys
// and the carried words (row id | columns), 8 bytes each; bv holds every
// bin-ordered row's u16 load index; the counters follow (big list, misc and the
// barriers stay where they are)
constexpr size_t kLocABytesW = (2 * kLocAKeys + 15) / 16 * 16;
constexpr size_t kLocBvW = kLocA + 2 * kLocABytesW;
constexpr size_t kLocHistW = kLocBvW + (size_t(kLocalCap) * 2 + 15) / 16 * 16;
static_assert(kLocHistW + size_t(kLocalBinsBal) * 4 <= kLocBig, "idw: the counters end before the big-bin list");
// misc: [0] big count, [2..3] run-list sizes, [8..] scan scratch, [32..65] group offsets (x2),
// [72..103] run ends (x2), [112..] run descriptors
constexpr size_t kLocBars = kLocMisc + 128 * 4;
constexpr size_t kLocalSmemBytes = kLocBars + 4 * 8;  // full[2], empty[2] (the producer-warp kernels)
// local_kernel only (not the cooperative kernel's budget): the three-level
// path's group offsets and runs, [2][257] + [2][256]
constexpr size_t kLocGrp = (kLocalSmemBytes + 15) / 16 * 16;
constexpr size_t kLocalKernelSmem = kLocGrp + (2 * 257 + 2 * 256) * 4;
constexpr size_t kSmemBytes = std::max(kPassSmemBytes + size_t(kPasses) * kBins * 4 + 128, kLocalSmemBytes);

struct PassState {  // per-CTA mbarrier phase parities, carried across passes
  uint32_t phase0, phase1;
};

// Stable rank of every item of this warp within its digit, offset by the
// warp's base for that digit (wh[] holds the bases on entry). Warp-striped
// items: element order is (item, lane), so lanes of one item are ranked by
// peer mask and items by the in-order shared atomics on wh[].
template <int SHIFT>
__device__ __forceinline__ void rank_items(const uint64_t (&k)[kItems], uint32_t (&rank2)[kItems / 2],
                                           uint32_t* wh, uint32_t* wm, uint32_t e0, uint32_t count, int lane) {
  const uint32_t lt = lanemask_lt();
  const uint32_t me = 1u << lane;
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const bool valid = (e0 + it * 32) < count;
    const uint32_t d = uint32_t(k[it] >> SHIFT) & (kBins - 1);
#if RL_RANK_MODE == 1
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
    if (!valid) peers = me;
#pragma unroll
    for (int b = 0; b < kBits; ++b) {
      const bool bit = (d >> b) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bal : ~bal;
    }
    const int leader = 31 - __clz(peers);
    uint32_t base = 0;
    if (valid && lane == leader) base = atomicAdd(&wh[d], uint32_t(__popc(peers)));
    base = __shfl_sync(0xffffffffu, base, leader);
#else
    // match via shared atomicOr (wm[] is all-zero between items)
    if (valid) atomicOr(&wm[d], me);
    __syncwarp();
    const uint32_t peers = valid ? wm[d] : me;
    const int leader = 31 - __clz(peers);
    uint32_t base = 0;
    if (valid && lane == leader) base = atomicAdd(&wh[d], uint32_t(__popc(peers)));
    base = __shfl_sync(0xffffffffu, base, leader);  // also orders every read of wm before the clear
    if (valid && lane == leader) wm[d] = 0;
    __syncwarp();
#endif
    const uint32_t r = base + __popc(peers & lt);
    if (it & 1) rank2[it >> 1] |= r << 16;
    else rank2[it >> 1] = r;
  }
}

// Issue the TMA bulk loads of one tile into `buf` (full 16-byte chunks; a
// ragged tail is finished with plain loads after the wait).
__device__ __forceinline__ void prefetch_tile(int64_t n, const uint64_t* kin, const uint32_t* vin, uint32_t tile,
                                              uint8_t* buf, uint64_t* bar) {
  const int64_t begin = int64_t(tile) * kTile;
  const int64_t left = n - begin;
  const uint32_t count = left < kTile ? uint32_t(left) : uint32_t(kTile);
  const uint32_t kbytes = (count * 8u) & ~15u;
  const uint32_t vbytes = vin ? ((count * 4u) & ~15u) : 0u;
  mbar_expect_tx(bar, kbytes + vbytes);
  if (kbytes) bulk_g2s(buf, kin + begin, kbytes, bar);
  if (vbytes) bulk_g2s(buf + size_t(kTile) * 8, vin + begin, vbytes, bar);
}

// One stable 8-bit onesweep digit pass (PASS selects the digit). Persistent:
// the CTA claims tiles in increasing order and prefetches tile i+1 while it
// processes tile i. Progress: the smallest unfinished tile's predecessors
// are all finished, and it is either being processed or queued behind a
// smaller tile of the same CTA.
//
// SUBOFF (the hybrid's digit-7 pass, whose input is ordered by digit 6):
// a tile holding the first rows of digit-6 values c in (lo, hi] writes
// every sub-bucket start (d7, c) = d7's base + its look-back prefix + the
// rows of d7 in this tile with d6 < c (a binary search in the staged run,
// which keeps input order, i.e. d6 order). No extra pass over the data.
template <int PASS, bool SUBOFF = false>
__device__ __forceinline__ void run_pass(const SortArgs& a, uint8_t* smem, uint32_t src, uint32_t dst,
                                      const uint32_t* bin_off, PassState& ps, const uint32_t kEpoch,
                                      uint32_t* tile_counter) {
  constexpr int kShift = PASS * kBits;
  uint8_t* bufs = smem;
  uint32_t* whist = reinterpret_cast<uint32_t*>(smem + 2 * kBufBytes);
  uint32_t* wmatch = whist + kWarps * kBins;
  uint32_t* gbase = wmatch + kWarps * kBins;
  uint32_t* misc = gbase + kBins;  // [0],[1] claimed tile ids (by iteration parity), [4..] scan scratch
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOffset);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t num_tiles = uint32_t((a.n + kTile - 1) / kTile);
  const uint64_t* kin = src == 1 ? a.keys_a : src == 2 ? a.keys_b : static_cast<const uint64_t*>(a.orig_keys);
  const uint32_t* vin = src == 1 ? a.vals_a : src == 2 ? a.vals_b : a.perm_in;
  const bool xf = src == 0 && a.key_mode != kMaterialized;
  const int desc_in = a.key_mode == kRawDesc;

  for (int i = tid; i < 2 * kWarps * kBins; i += kThreads) whist[i] = 0;  // whist + wmatch
  if (tid == 0) {
    const uint32_t t = atomicAdd(&tile_counter[PASS], 1u);
    misc[0] = t;
    if (t < num_tiles) {
      fence_proxy_async_smem();  // buffer 0 was last written by generic stores
      prefetch_tile(a.n, kin, vin, t, bufs, &bars[0]);
    }
  }
  __syncthreads();
  uint32_t tile = misc[0];
  uint32_t cb = 0;  // buffer + claim slot of this iteration
  uint32_t* wh = whist + warp * kBins;
  const uint32_t e0 = uint32_t(warp) * (32 * kItems) + lane;

  while (tile < num_tiles) {
    uint8_t* buf = bufs + cb * kBufBytes;
    uint64_t* skeys = reinterpret_cast<uint64_t*>(buf);
    uint32_t* svals = reinterpret_cast<uint32_t*>(buf + size_t(kTile) * 8);
    if (tid == 0) {  // claim + prefetch the next tile into the other buffer
      const uint32_t nt = atomicAdd(&tile_counter[PASS], 1u);
      misc[cb ^ 1] = nt;  // slot cb^1: its previous value was read before the last barrier
      if (nt < num_tiles) {
        fence_proxy_async_smem();
        prefetch_tile(a.n, kin, vin, nt, bufs + (cb ^ 1) * kBufBytes, &bars[cb ^ 1]);
      }
    }
    const int64_t tile_begin = int64_t(tile) * kTile;
    const int64_t left = a.n - tile_begin;
    const uint32_t count = left < kTile ? uint32_t(left) : uint32_t(kTile);
    uint64_t before = 0;  // SUBOFF: the row ahead of this tile
    if (SUBOFF && tid == 0 && tile_begin > 0) before = __ldcg(reinterpret_cast<const unsigned long long*>(kin) + tile_begin - 1);
    mbar_wait(&bars[cb], cb ? ps.phase1 : ps.phase0);
    if (cb) ps.phase1 ^= 1;
    else ps.phase0 ^= 1;
    if (count < kTile) {  // ragged tail: the bytes TMA did not move
      const uint32_t kdone = ((count * 8u) & ~15u) / 8u;
      for (uint32_t i = kdone + tid; i < count; i += kThreads) skeys[i] = kin[tile_begin + i];
      if (vin) {
        const uint32_t vdone = ((count * 4u) & ~15u) / 4u;
        for (uint32_t i = vdone + tid; i < count; i += kThreads) svals[i] = vin[tile_begin + i];
      }
      __syncthreads();
    }

    if (SUBOFF && tid == 0) {  // d6 range of this tile's rows: (lo, hi]
      const uint64_t last = skeys[count - 1];
      misc[16] = tile_begin > 0 ? uint32_t((xf ? xform(before, desc_in) : before) >> 48) & (kBins - 1u) : 0xFFFFFFFFu;
      misc[17] = uint32_t((xf ? xform(last, desc_in) : last) >> 48) & (kBins - 1u);
    }
    // ---- keys + row ids into registers (warp-striped; conflict-free 8-byte reads)
    uint64_t k[kItems];
    uint32_t v[kItems];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const uint32_t e = e0 + it * 32;
      const uint64_t x = skeys[e];
      k[it] = xf ? xform(x, desc_in) : x;
      v[it] = vin ? svals[e] : uint32_t(tile_begin + e);
    }

    // ---- early counts: per-warp digit histograms (order-free shared
    // reductions), so the tile publishes its aggregate before ranking.
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      if ((e0 + it * 32) < count) atomicAdd(&wh[uint32_t(k[it] >> kShift) & (kBins - 1)], 1u);
    }
    __syncthreads();  // counts complete; every thread has read its keys out of buf

    // ---- per-digit tile counts → warp base offsets; publish the aggregate
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = whist[w * kBins + tid];
      whist[w * kBins + tid] = run;
      run += c;
    }
    uint64_t* my_status = a.status + uint64_t(tile) * kBins + tid;
    st_relaxed(my_status, pack_status(tile == 0 ? kFlagIncl : kFlagAgg, kEpoch, run));
    uint32_t tile_total;
    const uint32_t ls = block_exclusive_scan<kThreads>(run, misc + 4, &tile_total);  // syncs: bases visible
    // fold the tile-local digit start into every warp's base, so a rank is
    // directly the item's slot in the digit-ordered staging buffer
#pragma unroll
    for (int w = 0; w < kWarps; ++w) whist[w * kBins + tid] += ls;
    __syncthreads();

    // ---- warp-level stable ranking
    uint32_t rank2[kItems / 2];  // two 16-bit tile-local slots per register (slot < kTile)
    rank_items<kShift>(k, rank2, wh, wmatch + warp * kBins, e0, count, lane);

    // ---- stage the tile in digit order (stable local positions), in place
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      if ((e0 + it * 32) < count) {
        const uint32_t pos = (rank2[it >> 1] >> ((it & 1) * 16)) & 0xFFFFu;
        skeys[pos] = k[it];
        svals[pos] = v[it];
      }
    }

    // ---- decoupled look-back for this thread's digit, kLookback predecessor
    // status words per round trip, from the nearest tile back to the first
    // inclusive prefix; a not-yet-published predecessor is polled alone.
    uint64_t excl = 0;
    if (tile > 0) {
      int64_t p = int64_t(tile) - 1;
      bool done = false;
      while (!done) {
        uint64_t st[kLookback];
#pragma unroll
        for (int j = 0; j < kLookback; ++j)
          st[j] = (p - j >= 0) ? ld_relaxed(a.status + uint64_t(p - j) * kBins + tid) : 0;
        int used = 0;
#pragma unroll
        for (int j = 0; j < kLookback; ++j) {
          if (done) break;
          const uint64_t sj = st[j];
          if ((sj & kFlagMask) == 0 || status_epoch(sj) != kEpoch) break;  // not published yet
          excl += sj & kValueMask;
          ++used;
          done = (sj & kFlagMask) == kFlagIncl;
        }
        if (done) break;
        p -= used;
        if (used < kLookback) {  // tile p not published yet: poll it alone, backing off
          uint64_t sp;
          uint32_t ns = 32;
          while (true) {
            sp = ld_relaxed(a.status + uint64_t(p) * kBins + tid);
            if ((sp & kFlagMask) != 0 && status_epoch(sp) == kEpoch) break;
            __nanosleep(ns);
            ns = ns < 256 ? ns * 2 : ns;
          }
          excl += sp & kValueMask;
          done = (sp & kFlagMask) == kFlagIncl;
          --p;
        }
      }
      st_relaxed(my_status, pack_status(kFlagIncl, kEpoch, excl + run));
    }
    gbase[tid] = bin_off[PASS * kBins + tid] + uint32_t(excl) - ls;
    __syncthreads();  // every warp is past its ranking: whist may be reset
    for (int i = tid; i < kWarps * kBins; i += kThreads) whist[i] = 0;  // for the next tile
    if constexpr (SUBOFF) {
      const int lo = int(misc[16]), hi = int(misc[17]);  // lo = -1 (0xFFFFFFFF) for tile 0
      const bool last_tile = tile == num_tiles - 1;
      if (hi > lo || last_tile) {
        const uint32_t base7 = bin_off[PASS * kBins + tid] + uint32_t(excl);
        const uint32_t row = uint32_t(tid) << kBits;
        for (int c = lo + 1; c <= hi; ++c) {
          uint32_t l = ls, r = ls + run;
          while (l < r) {
            const uint32_t m = (l + r) >> 1;
            if (int(uint32_t(skeys[m] >> 48) & (kBins - 1)) < c) l = m + 1;
            else r = m;
          }
          a.sub_off[row | uint32_t(c)] = base7 + (l - ls);
        }
        if (last_tile) {
          for (int c = hi + 1; c < kBins; ++c) a.sub_off[row | uint32_t(c)] = base7 + run;
          if (tid == 0) a.sub_off[kSubBuckets] = uint32_t(a.n);
        }
      }
    }

    // ---- write the staged tile: consecutive threads → consecutive slots
    if (dst == 3) {
      const int desc = a.key_mode == kRawDesc;
#pragma unroll 4
      for (int it = 0; it < kItems; ++it) {
        const uint32_t j = uint32_t(it) * kThreads + tid;
        if (j < count) {
          const uint64_t key = skeys[j];
          const uint32_t o = gbase[uint32_t(key >> kShift) & (kBins - 1)] + j;
          if (a.out_keys) __stcs(reinterpret_cast<long long*>(a.out_keys) + o, (long long)xform(key, desc));
          const uint32_t row = svals[j];
          __stcs(a.out_vals + o, row);
          gather_fused(a.gather, row, o);
        }
      }
    } else {
      uint64_t* kout = dst == 1 ? a.keys_a : a.keys_b;
      uint32_t* vout = dst == 1 ? a.vals_a : a.vals_b;
#pragma unroll 4
      for (int it = 0; it < kItems; ++it) {
        const uint32_t j = uint32_t(it) * kThreads + tid;
        if (j < count) {
          const uint64_t key = skeys[j];
          const uint32_t o = gbase[uint32_t(key >> kShift) & (kBins - 1)] + j;
          kout[o] = key;
          vout[o] = svals[j];
        }
      }
    }
    __syncthreads();  // buf free for the prefetch two tiles ahead; next tile id visible
    cb ^= 1;
    tile = misc[cb];
  }
}

// K1: all eight digit histograms in one read of the keys (its own launch:
// shared-atomic bound, it wants 4x the resident threads of the passes).
// RAW: contiguous int64 keys, read as 16-byte vectors with every load of a
// step in flight before the first use; otherwise the generic loader
// (gathered rows, Bytes words; materialises the transformed words).
constexpr int kHistThreads = 512;
template <bool RAW, bool ALL = !RAW>
__global__ void __launch_bounds__(kHistThreads) hist_kernel(SortArgs a) {
  __shared__ uint32_t h[kPasses * kBins];
  const int tid = threadIdx.x;
  if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[0] = globaltimer();
  pdl_launch_dependents();  // the sort kernel may be scheduled now; it waits for these counts
  for (int i = tid; i < kPasses * kBins; i += kHistThreads) h[i] = 0;
  __syncthreads();
  // RAW counts only the top two digits (the hybrid's passes) and ORs the
  // varying bits: which digits an LSD sort needs, counted later in the sort
  // kernel only if it goes LSD, and only for digits that vary
  uint64_t vary = 0, k0 = 0;
  if constexpr (RAW) k0 = xform(uint64_t(__ldg(static_cast<const long long*>(a.col))), a.desc);
  auto count = [&](uint64_t k) {
    if constexpr (RAW) vary |= k ^ k0;
    if constexpr (RAW && !ALL) {
      atomicAdd(&h[6 * kBins + ((k >> (6 * kBits)) & (kBins - 1))], 1u);
      atomicAdd(&h[7 * kBins + ((k >> (7 * kBits)) & (kBins - 1))], 1u);
    } else {
#pragma unroll
      for (int p = 0; p < kPasses; ++p) atomicAdd(&h[p * kBins + ((k >> (p * kBits)) & (kBins - 1))], 1u);
    }
  };
  if constexpr (RAW) {
    const ulonglong2* v2 = static_cast<const ulonglong2*>(a.col);  // 16-byte aligned (checked by the caller)
    const int64_t pairs = a.n >> 1;
    constexpr int kV = kHistUnroll / 2;
    const int64_t stride = int64_t(gridDim.x) * kHistThreads * kV;
    for (int64_t base = int64_t(blockIdx.x) * kHistThreads * kV + tid; base < pairs; base += stride) {
      ulonglong2 q[kV];
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const int64_t i = base + int64_t(u) * kHistThreads;
        q[u] = i < pairs ? __ldcs(v2 + i) : make_ulonglong2(0, 0);
      }
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        if (base + int64_t(u) * kHistThreads < pairs) {
          count(xform(q[u].x, a.desc));
          count(xform(q[u].y, a.desc));
        }
      }
    }
    if ((a.n & 1) && blockIdx.x == 0 && tid == 0)
      count(xform(uint64_t(static_cast<const long long*>(a.col)[a.n - 1]), a.desc));
  } else {
    const int64_t stride = int64_t(gridDim.x) * kHistThreads * kHistUnroll;
    for (int64_t base = int64_t(blockIdx.x) * kHistThreads * kHistUnroll + tid; base < a.n; base += stride) {
      uint64_t k[kHistUnroll];
#pragma unroll
      for (int u = 0; u < kHistUnroll; ++u) {
        const int64_t i = base + int64_t(u) * kHistThreads;
        k[u] = i < a.n ? load_key(a, i) : 0;
      }
#pragma unroll
      for (int u = 0; u < kHistUnroll; ++u) {
        const int64_t i = base + int64_t(u) * kHistThreads;
        if (i >= a.n) continue;
        if (a.materialized) a.materialized[i] = k[u];
        count(k[u]);
      }
    }
  }
  __shared__ uint32_t vparts[2 * (kHistThreads / 32)];
  if constexpr (RAW) {  // varying bits: one global atomic per CTA
    const uint32_t hi = __reduce_or_sync(0xffffffffu, uint32_t(vary >> 32));
    const uint32_t lo = __reduce_or_sync(0xffffffffu, uint32_t(vary));
    if ((tid & 31) == 0) {
      vparts[2 * (tid >> 5)] = hi;
      vparts[2 * (tid >> 5) + 1] = lo;
    }
  }
  __syncthreads();
  if constexpr (RAW) {
    if (tid < 32) {
      const uint32_t hi = __reduce_or_sync(0xffffffffu, tid < kHistThreads / 32 ? vparts[2 * tid] : 0u);
      const uint32_t lo = __reduce_or_sync(0xffffffffu, tid < kHistThreads / 32 ? vparts[2 * tid + 1] : 0u);
      if (tid == 0 && (hi | lo)) atomicOr(reinterpret_cast<unsigned long long*>(a.flags + 4), (uint64_t(hi) << 32) | lo);
    }
  }
  uint32_t* gh = a.ghist + size_t(blockIdx.x % kHistReps) * kPasses * kBins;
  for (int i = RAW && !ALL ? 6 * kBins + tid : tid; i < kPasses * kBins; i += kHistThreads) {
    const uint32_t c = h[i];
    if (c) atomicAdd(&gh[i], c);
  }
}

// In-kernel histograms of the varying digits in `digits` (bit p = digit p)
// of raw int64 keys, by every CTA of the cooperative kernel (the LSD path
// after the RAW histogram kernel, which counted only digits 6 and 7).
__device__ void count_digits(const SortArgs& a, uint8_t* smem, uint32_t digits) {
  uint32_t* h = reinterpret_cast<uint32_t*>(smem);  // [kPasses][kBins]; pass buffers are free here
  const int tid = threadIdx.x;
  for (int i = tid; i < kPasses * kBins; i += kThreads) h[i] = 0;
  __syncthreads();
  const ulonglong2* v2 = static_cast<const ulonglong2*>(a.col);
  const int64_t pairs = a.n >> 1;
  constexpr int kV = 8;
  auto count = [&](uint64_t k) {
#pragma unroll
    for (int p = 0; p < kPasses; ++p)
      if ((digits >> p) & 1u) atomicAdd(&h[p * kBins + ((k >> (p * kBits)) & (kBins - 1))], 1u);
  };
  const int64_t stride = int64_t(gridDim.x) * kThreads * kV;
  for (int64_t base = int64_t(blockIdx.x) * kThreads * kV + tid; base < pairs; base += stride) {
    ulonglong2 q[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int64_t i = base + int64_t(u) * kThreads;
      q[u] = i < pairs ? __ldcs(v2 + i) : make_ulonglong2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      if (base + int64_t(u) * kThreads < pairs) {
        count(xform(q[u].x, a.desc));
        count(xform(q[u].y, a.desc));
      }
    }
  }
  if ((a.n & 1) && blockIdx.x == 0 && tid == 0) count(xform(uint64_t(static_cast<const long long*>(a.col)[a.n - 1]), a.desc));
  __syncthreads();
  for (int i = tid; i < kPasses * kBins; i += kThreads) {
    const uint32_t c = h[i];
    if (c && ((digits >> (i / kBins)) & 1u)) atomicAdd(&a.ghist[size_t(blockIdx.x % kHistReps) * kPasses * kBins + i], c);
  }
}

// ---------------------------------------------------------------- scatter hybrid
// Wide raw int64 keys, n >= kScatterMinRows. The local phase ranks every row
// by (key, row id) inside its sub-bucket (top 16 bits of the packed key, see
// below), so the rows only
// have to reach their sub-bucket, in any order — two non-stable counting
// passes with exact, precomputed bucket starts instead of two stable
// onesweep passes (no look-back, no stable multisplit):
//   sub_hist_kernel     chunk c (one CTA per SM) counts its rows per
//                       sub-bucket in shared memory (packed u16 pairs, 128 KB)
//                       into chunk_cnt[c], adds its digit-7 counts into one
//                       of kD7Reps replicas (148 CTAs adding into the same
//                       256 counters at once queue ~8 us of same-address
//                       atomics behind the kernel's end), ORs the varying
//                       key bits (one atomic per CTA)
//   top_scatter_kernel  every CTA: the digit-7 bucket starts; CTA g also the
//                       starts of bucket g's 256 sub-buckets (totals over the
//                       chunk counts; > kLocalCap -> LSD fallback); CTA 0 the
//                       pass-B tile list. Then tiles of 4096 rows: ranked by
//                       shared atomics, staged in digit order, one global
//                       atomic per (tile, digit) reserves the run, written as
//                       contiguous runs (keys_b / vals_b)
//   sub_scatter_kernel  tiles of one digit-7 bucket each, claimed in bucket
//                       order: the same staged scatter by digit 6 into the
//                       sub-buckets (keys_a / vals_a)
//   local_kernel        the local phase (512-thread CTAs)
// Bucket-ordered claiming keeps the sub-buckets being written within a few
// MB, so every sector completes in L2. The cooperative kernel launched last
// returns at once — unless the fallback flag is set (a sub-bucket above
// kLocalCap, a wrapped chunk counter, < 4 varying digits, a varying bit the
// key sample missed): then it runs the LSD passes from the original input.
// Each kernel after the first is a programmatic dependent of the one before
// when the sort has the device to itself.

// Packed rows: the packed key occupies the top len1 + len2 bits; with at most
// 32 of them the low 32 bits are free for the row id (n <= 2^32), so a row is
// ONE u64 (key | row id) through the counting passes and the local phase.
// Every packed word is distinct and orders rows by (key, row id).
__device__ __forceinline__ bool packed_rows(uint32_t c, const SortArgs& a) {
  return a.allow_pk && pack_mode(c) != 0 && (c >> 14 & 127) + (c & 127) <= 32u;
}
template <int MODE>
__device__ __forceinline__ uint64_t pack_as(uint64_t u, uint32_t c, uint32_t shl) {
  if constexpr (MODE == 0) return u;
  else if constexpr (MODE == 1) return u << shl;
  else return pack_key(u, c);
}
template <int MODE>
__device__ __forceinline__ uint64_t unpack_as(uint64_t v, uint32_t c, uint32_t shl, uint64_t constbits) {
  if constexpr (MODE == 0) return v;
  else if constexpr (MODE == 1) return (v >> shl) | constbits;
  else return unpack_key(v, c, constbits);
}

// The bits every key shares (from the first key) where the code drops them.
__device__ __forceinline__ uint64_t key_constbits(const SortArgs& a, uint32_t c) {
  const uint64_t u0 = xform(uint64_t(__ldg(static_cast<const long long*>(a.col))), a.desc);
  return u0 & ~pack_mask(c);
}

// The fallback flag, read ONCE per CTA: other CTAs of the same kernel may
// set it meanwhile, and a per-thread read could split the CTA at a barrier.
__device__ __forceinline__ bool fallback_flag(const SortArgs& a) {
  return __syncthreads_or(threadIdx.x == 0 && *reinterpret_cast<volatile const uint32_t*>(a.flags) != 0) != 0;
}

// The local phase's view of the fallback flag (final before its launch: uniform).
// (A CUDA-graph IF node around the fallback launch, armed here, replayed ~10 us
// slower than the no-op cooperative launch it would skip: not used.)
__device__ __forceinline__ bool local_fallback(const SortArgs& a) {
  return *reinterpret_cast<volatile const uint32_t*>(a.flags) != 0;
}

__device__ __forceinline__ int64_t chunk_lo(int64_t n, int chunks, int c) {
  const int64_t per = (((n + chunks - 1) / chunks) + 1) & ~int64_t(1);  // even: 16-byte pair loads
  return per * c < n ? per * c : n;
}

// Exclusive scan of one value per thread over threads 0..255 (every thread
// of the CTA calls it; the result is meaningful for tid < 256).
__device__ __forceinline__ uint32_t scan256(uint32_t c, uint32_t* scratch) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t incl = c;
  if (tid < 256) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) scratch[warp] = incl;
  }
  __syncthreads();
  uint32_t pre = 0;
  if (tid < 256)
    for (int w = 0; w < warp; ++w) pre += scratch[w];
  __syncthreads();
  return pre + incl - c;
}

struct PTile {  // shared memory of the counting passes
  uint64_t* sk;       // [kPTile] staged keys
  uint32_t* sv;       // [kPTile] staged row ids (CW == 0)
  uint64_t* sp;       // [kPTile * CW] staged carried payload words (CW > 0)
  uint32_t* hist;     // [256] tile digit counts -> tile digit starts
  uint32_t* base;     // [256] output position of staged row 0 of each digit
  uint32_t* aux;      // [256] pass A: digit-7 bucket starts
  uint32_t* scratch;  // [64]
};

// Staging bytes of a counting pass: keys + row ids, or (bucket join) keys +
// CW carried payload words per row (packed rows: no row-id stream).
constexpr size_t pstage_bytes(int cw) { return cw ? size_t(kPTile) * 8 * (1 + cw) : kPStage; }
constexpr size_t psmem_bytes(int cw) { return pstage_bytes(cw) + 3 * 256 * 4 + 64 * 4; }
static_assert(psmem_bytes(0) == kPSmem, "the sort's pass layout is unchanged");

template <int CW>  // carried payload words per row; arrays of CW == 0 keep one dummy slot
struct Carry {
  uint64_t p[kPItems][CW > 0 ? CW : 1];
};

template <int CW = 0>
__device__ __forceinline__ PTile ptile(uint8_t* sm) {
  PTile t;
  t.sk = reinterpret_cast<uint64_t*>(sm);
  t.sv = reinterpret_cast<uint32_t*>(sm + size_t(kPTile) * 8);
  t.sp = reinterpret_cast<uint64_t*>(sm + size_t(kPTile) * 8);
  t.hist = reinterpret_cast<uint32_t*>(sm + pstage_bytes(CW));
  t.base = t.hist + 256;
  t.aux = t.base + 256;
  t.scratch = t.aux + 256;
  return t;
}

// One tile of a non-stable counting scatter by the 8-bit digit at SHIFT:
// rank by shared atomics, reserve every digit's run with one global atomic
// (reserve(d, count) -> first output position; in flight during the scan and
// the staging), stage in digit order, write every run contiguously. s.hist
// is zero on entry and on exit. Once the tile is staged, next(k, v) loads the
// following tile into the same registers, in flight during the write-out.
// PK (packed rows): the row id travels in the key word's low 32 bits — no
// separate row-id stream (v[] unused). mid() runs on every thread after the
// counting barrier, beside the digit scan (warps 8..15 only reserve there).
// CW > 0 (bucket join): CW payload words ride with every row (c.p), staged and
// written to out_p[o * CW + w] beside the key.
#ifdef RL_PASS_PROFILE  // per-phase clock totals of the counting passes and the local phase (A/B builds only)
__device__ unsigned long long g_pass_prof[32];
#define PPROF(i, t) do { if (threadIdx.x == 0) { const long long c_ = clock64(); atomicAdd(&g_pass_prof[i], (unsigned long long)(c_ - t)); t = c_; } } while (0)
#else
#define PPROF(i, t) do { } while (0)
#endif

struct NoMid {
  __device__ void operator()() const {}
};
template <int SHIFT, bool PK, int CW = 0, typename Reserve, typename Next, typename Mid = NoMid>
__device__ __forceinline__ void ptile_scatter(uint64_t (&k)[kPItems], uint32_t (&v)[kPItems], Carry<CW>& cr, int tn,
                                              const PTile& s, uint64_t* out_k, uint32_t* out_v, uint64_t* out_p,
                                              Reserve reserve, Next next, Mid mid = Mid()) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef RL_PASS_PROFILE
  long long pt = clock64();
#endif
  uint32_t r[kPItems];
#pragma unroll
  for (int u = 0; u < kPItems; ++u)
    if (u * kPThreads + tid < tn) r[u] = atomicAdd(&s.hist[uint32_t(k[u] >> SHIFT) & 255u], 1u);
  __syncthreads();
  PPROF(SHIFT == 56 ? 0 : 8, pt);
  mid();  // the caller's work beside the digit scan (the next tile's descriptor)
  const uint32_t c = tid < 256 ? s.hist[tid] : 0u;
  // the digit runs: reserve(d, c) = {static start, atomic reservation}, issued
  // by warps 8..15 (thread 256 + d) while warps 0..7 scan, in flight until
  // s.base is written after the staging (empty digits reserve 0)
  static_assert(kPThreads >= 512, "digit scan on threads 0..255, reservations on 256..511");
  uint2 res;
  if (tid >= 256 && tid < 512) res = reserve(uint32_t(tid - 256), s.hist[tid - 256]);
  uint32_t incl = c;  // digit scan: warps 0..7, one barrier (the next scratch write is behind two more)
  if (tid < 256) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    if (lane == 31) s.scratch[warp] = incl;
  }
  __syncthreads();
  uint32_t excl = incl - c;
  if (tid < 256) {
    for (int w = 0; w < warp; ++w) excl += s.scratch[w];
    s.hist[tid] = excl;
  }
  __syncthreads();
  PPROF(SHIFT == 56 ? 1 : 9, pt);
  // staging: every digit start read before the first staged store (a store
  // could alias a later start, so the compiler keeps written order)
  uint32_t sp[kPItems];
#pragma unroll
  for (int u = 0; u < kPItems; ++u) sp[u] = s.hist[uint32_t(k[u] >> SHIFT) & 255u] + r[u];
#pragma unroll
  for (int u = 0; u < kPItems; ++u) {
    if (u * kPThreads + tid < tn) {
      const uint32_t p = sp[u];
      if constexpr (CW == 1) {  // key + carried word interleaved (read back as one 16-byte load)
        s.sk[2 * p] = k[u];
        s.sk[2 * p + 1] = cr.p[u][0];
        continue;
      }
      s.sk[p] = k[u];
      if constexpr (CW > 0) {
#pragma unroll
        for (int w = 0; w < CW; ++w) s.sp[p * CW + w] = cr.p[u][w];
      } else if constexpr (!PK) {
        s.sv[p] = v[u];
      }
    }
  }
  if (tid >= 256 && tid < 512) s.base[tid - 256] = res.x + res.y - s.hist[tid - 256];  // (s.hist = digit starts)
  __syncthreads();
  PPROF(SHIFT == 56 ? 2 : 10, pt);
  next(k, v, cr);
  PPROF(SHIFT == 56 ? 5 : 13, pt);
  if (tid < 256) s.hist[tid] = 0;  // for the next tile (the write-out reads only s.base)
  // write-out in batches of kWB rows a thread: the staged keys, then their
  // digit bases, then the global stores (st.global: no ordering against the
  // shared loads of the next batch)
  constexpr int kWB = CW >= 2 ? 1 : 4;  // (two carried words: batches spill)
  for (int i0 = tid; i0 < tn; i0 += kWB * kPThreads) {
    if constexpr (CW == 1) {  // key + carried word: one 16-byte shared load a row
      ulonglong2 q[kWB];
      uint32_t o[kWB];
#pragma unroll
      for (int u = 0; u < kWB; ++u) {
        const int i = i0 + u * kPThreads;
        q[u] = i < tn ? reinterpret_cast<const ulonglong2*>(s.sk)[i] : make_ulonglong2(0, 0);
        o[u] = s.base[uint32_t(q[u].x >> SHIFT) & 255u] + uint32_t(i);
      }
#pragma unroll
      for (int u = 0; u < kWB; ++u) {
        if (i0 + u * kPThreads < tn) {
          __stwb(reinterpret_cast<unsigned long long*>(out_k) + o[u], q[u].x);
          __stwb(reinterpret_cast<unsigned long long*>(out_p) + o[u], q[u].y);
        }
      }
      continue;
    }
    uint64_t kk[kWB];
    uint32_t o[kWB];
#pragma unroll
    for (int u = 0; u < kWB; ++u) {
      const int i = i0 + u * kPThreads;
      kk[u] = i < tn ? s.sk[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kWB; ++u) o[u] = s.base[uint32_t(kk[u] >> SHIFT) & 255u] + uint32_t(i0 + u * kPThreads);
    if constexpr (CW > 0) {
      uint64_t pw[kWB][CW];
#pragma unroll
      for (int u = 0; u < kWB; ++u) {
        const int i = i0 + u * kPThreads;
#pragma unroll
        for (int w = 0; w < CW; ++w) pw[u][w] = i < tn ? s.sp[i * CW + w] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < kWB; ++u) {
        if (i0 + u * kPThreads < tn) {
          __stwb(reinterpret_cast<unsigned long long*>(out_k) + o[u], kk[u]);
#pragma unroll
          for (int w = 0; w < CW; ++w) __stwb(reinterpret_cast<unsigned long long*>(out_p) + size_t(o[u]) * CW + w, pw[u][w]);
        }
      }
    } else {
      uint32_t vv[kWB];
#pragma unroll
      for (int u = 0; u < kWB; ++u) {
        const int i = i0 + u * kPThreads;
        vv[u] = !PK && i < tn ? s.sv[i] : 0u;
      }
#pragma unroll
      for (int u = 0; u < kWB; ++u) {
        if (i0 + u * kPThreads < tn) {
          __stwb(reinterpret_cast<unsigned long long*>(out_k) + o[u], kk[u]);
          if constexpr (!PK) __stwb(out_v + o[u], vv[u]);
        }
      }
    }
  }
  __syncthreads();  // staging and s.base reused by the next tile
  PPROF(SHIFT == 56 ? 3 : 11, pt);
#ifdef RL_PASS_PROFILE
  if (tid == 0) atomicAdd(&g_pass_prof[SHIFT == 56 ? 4 : 12], 1ull);
#endif
}

__global__ void __launch_bounds__(kScatThreads, 1) sub_hist_kernel(SortArgs a) {
  extern __shared__ __align__(16) uint32_t w[];  // [kScatWords] + [kScatThreads] reduction scratch
  uint32_t* red = w + kScatWords;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[0] = globaltimer();
  pdl_launch_dependents();
  if (a.bj && fallback_flag(a)) return;  // the bucket join's plan already declined (bj_pack_kernel)
  // this thread's key sample, in flight while the histogram is zeroed
  const long long sample = __ldg(static_cast<const long long*>(a.col) + int64_t(tid) * a.n / kScatThreads);
  for (int i = tid; i < kScatWords / 4; i += kScatThreads) reinterpret_cast<uint4*>(w)[i] = make_uint4(0, 0, 0, 0);
  if (tid < 2) red[kScatThreads - 4 + tid] = 0u;  // the sample's varying-bit OR
  __syncthreads();
#ifdef RL_K1_PROFILE
  if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[4] = globaltimer();
#endif
  const int64_t lo = chunk_lo(a.n, a.chunks, blockIdx.x), hi = chunk_lo(a.n, a.chunks, blockIdx.x + 1);
  const long long* col = static_cast<const long long*>(a.col);
  const uint64_t k0 = xform(uint64_t(__ldg(a.k0_src ? a.k0_src : col)), a.desc);
  uint32_t sh;
  if (a.pack_given) {  // bucket join: the joint code of both sides (bj_pack_kernel)
    sh = __ldcg(a.flags + 6);
  } else {  // the key shift from 1024 strided samples — the same in every CTA (mostly L2
     // hits); a varying bit they miss is caught by the full check below (-> LSD)
    const uint64_t v = xform(uint64_t(sample), a.desc) ^ k0;
    const uint32_t vh = __reduce_or_sync(0xffffffffu, uint32_t(v >> 32));
    const uint32_t vl = __reduce_or_sync(0xffffffffu, uint32_t(v));
    if (lane == 0) {  // (red[1020..1021] zeroed with the histogram)
      atomicOr(&red[kScatThreads - 4], vh);
      atomicOr(&red[kScatThreads - 3], vl);
    }
    __syncthreads();
    sh = pack_code_of((uint64_t(red[kScatThreads - 4]) << 32) | red[kScatThreads - 3]);
    if (blockIdx.x == 0 && tid == 0) a.flags[6] = sh;  // the pack code, for the later kernels
  }
  uint64_t vary = 0;
  // the counting loop, compiled per key-packing mode (chosen once)
  const uint32_t shl = pack_shift(sh);
  auto counting = [&](auto packed) {
    auto count = [&](uint64_t u) {  // a wrapped 16-bit counter shows up in the chunk total below
      vary |= u ^ k0;
      const uint32_t b = uint32_t(pack_as<decltype(packed)::value>(u, sh, shl) >> 48);
      atomicAdd(&w[b >> 1], 1u << ((b & 1u) << 4));
    };
    const ulonglong2* v2 = reinterpret_cast<const ulonglong2*>(col);
    constexpr int kV = 4;
    constexpr int64_t kStep = int64_t(kScatThreads) * kV;
    const int64_t p1 = hi >> 1;
    // two batches alternate: one is counted while the other's loads are in flight
    ulonglong2 qa[kV], qb[kV];
    auto fetch = [&](ulonglong2 (&q)[kV], int64_t base) {
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const int64_t i = base + int64_t(u) * kScatThreads;
        q[u] = i < p1 ? __ldg(v2 + i) : make_ulonglong2(0, 0);
      }
    };
    auto consume = [&](const ulonglong2 (&q)[kV], int64_t base) {
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        if (base + int64_t(u) * kScatThreads < p1) {
          count(xform(q[u].x, a.desc));
          count(xform(q[u].y, a.desc));
        }
      }
    };
    int64_t base = (lo >> 1) + tid;
    fetch(qa, base);
    while (base < p1) {
      fetch(qb, base + kStep);
      consume(qa, base);
      base += kStep;
      if (base >= p1) break;
      fetch(qa, base + kStep);
      consume(qb, base);
      base += kStep;
    }
    if ((hi & 1) && hi > lo && tid == 0) count(xform(uint64_t(col[hi - 1]), a.desc));
  };
  switch (pack_mode(sh)) {
    case 0: counting(std::integral_constant<int, 0>{}); break;
    case 1: counting(std::integral_constant<int, 1>{}); break;
    default: counting(std::integral_constant<int, 2>{}); break;
  }
  // varying key bits: one global atomic per CTA (one per warp serialised ~4700
  // same-address atomics at one L2 slice: a 15 us tail)
  const uint32_t vhi = __reduce_or_sync(0xffffffffu, uint32_t(vary >> 32));
  const uint32_t vlo = __reduce_or_sync(0xffffffffu, uint32_t(vary));
  if (lane == 0) {
    red[2 * warp] = vhi;
    red[2 * warp + 1] = vlo;
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t h2 = __reduce_or_sync(0xffffffffu, red[2 * lane]);
    const uint32_t l2 = __reduce_or_sync(0xffffffffu, red[2 * lane + 1]);
    const uint64_t v2 = (uint64_t(h2) << 32) | l2;
    if (lane == 0 && v2) atomicOr(reinterpret_cast<unsigned long long*>(a.flags + 4), v2);
    if (lane == 0 && (v2 & ~pack_mask(sh))) atomicOr(a.flags, 1u);  // the sample missed a varying bit: LSD
  }
#ifdef RL_K1_PROFILE
  __syncthreads();
  if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[5] = globaltimer();
  if (a.stamps && tid == 0) atomicMax(a.stamps + 7, globaltimer());  // last count loop to end
#endif
  uint4* dst = reinterpret_cast<uint4*>(a.chunk_cnt + size_t(blockIdx.x) * kScatWords);
  for (int i = tid; i < kScatWords / 4; i += kScatThreads) dst[i] = reinterpret_cast<const uint4*>(w)[i];
#ifdef RL_K1_PROFILE
  __syncthreads();
  if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[6] = globaltimer();
#endif
  // digit 7: a warp sums the 128 words of one bucket at a time; the chunk
  // total exposes a 16-bit counter that wrapped (> 65535 rows of one
  // sub-bucket in this chunk: far above kLocalCap, so the LSD runs)
  uint32_t mine = 0;
  for (int g = warp; g < kBins; g += kScatThreads / 32) {
    uint32_t t = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t x = w[g * 128 + j * 32 + lane];
      t += (x & 0xFFFFu) + (x >> 16);
    }
    t = __reduce_add_sync(0xffffffffu, t);
    mine += t;
    if (lane == 0 && t) atomicAdd(&a.d7rep[(blockIdx.x % kD7Reps) * kBins + g], t);
  }
  if (lane == 0) red[64 + warp] = mine;  // (slots 0..63 held the varying-bit parts)
  __syncthreads();
  if (tid == 0) {
    uint32_t tot = 0;
    for (int i = 0; i < kScatThreads / 32; ++i) tot += red[64 + i];
    if (tot != uint32_t(hi - lo)) atomicOr(a.flags, 1u);  // LSD fallback
#ifdef RL_K1_PROFILE
    if (a.stamps) atomicMax(a.stamps + 8, globaltimer());  // last CTA to end
#endif
  }
}

// The carried payload words of input row `row` (bucket join): the carried
// columns' bytes packed at their offsets; 8-byte-aligned 8 / 16-byte columns
// with whole-word loads, anything else byte by byte.
template <int CW>
__device__ __forceinline__ void load_carry(const SortArgs& a, uint64_t row, uint64_t (&w)[CW > 0 ? CW : 1]) {
  if (a.carry_n == 1 && a.carry_width[0] == 8 * CW) {  // one column filling the words: whole-word loads
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(a.carry_src[0]) + row * CW;
#pragma unroll
    for (int i = 0; i < CW; ++i) w[i] = __ldcs(src + i);
    return;
  }
  if (a.carry_n == 1 && a.carry_width[0] == 4 && a.carry_off[0] == 0) {  // one 4-byte column (cfg2's payload)
    w[0] = __ldcs(reinterpret_cast<const unsigned int*>(a.carry_src[0]) + row);
#pragma unroll
    for (int i = 1; i < CW; ++i) w[i] = 0;
    return;
  }
  // general layout: the words as two scalars (a dynamic index into w[] would
  // put the caller's carry registers on the stack)
  uint64_t w0 = 0, w1 = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (c >= a.carry_n) break;
    const int wd = a.carry_width[c], off = a.carry_off[c];
    const uint8_t* src = a.carry_src[c] + row * uint64_t(wd);
    if ((wd == 8 || wd == 16) && (off & 7) == 0) {
      const uint64_t x = __ldcs(reinterpret_cast<const unsigned long long*>(src));
      if (off == 0) w0 = x;
      else w1 = x;
      if (wd == 16 && off == 0) w1 = __ldcs(reinterpret_cast<const unsigned long long*>(src) + 1);
    } else {
      for (int b = 0; b < wd; ++b) {
        const int at = off + b;
        const uint64_t x = uint64_t(__ldg(src + b));
        if (at < 8) w0 |= x << (at * 8);
        else if (at < 16) w1 |= x << ((at - 8) * 8);
      }
    }
  }
  w[0] = w0;
  if constexpr (CW > 1) w[1] = w1;
}

template <int CW = 0>
__global__ void __launch_bounds__(kPThreads, RL_PASS_CTAS_PER_SM) top_scatter_kernel(SortArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  const PTile s = ptile<CW>(sm);
  const int tid = threadIdx.x;
  pdl_wait();  // the chunk counts
  pdl_launch_dependents();
  if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[2] = globaltimer();
  if (tid == 0) s.scratch[50] = __ldcg(a.flags + 6);  // the key pack code, read after the prologue's barriers
  if (fallback_flag(a)) return;  // a chunk counter wrapped: LSD
  // digit-7 bucket starts (every CTA)
  uint32_t t7 = 0;
  if (tid < 256) {
#pragma unroll
    for (int r = 0; r < kD7Reps; ++r) t7 += __ldcg(a.d7rep + r * kBins + tid);
  }
  {  // certain fallbacks, decided by every CTA alike before any work: fewer than 4
     // varying digits (LSD is as cheap), or a digit-7 bucket too big for 256 sub-buckets
    const uint64_t vary = __ldcg(reinterpret_cast<const unsigned long long*>(a.flags + 4));
    int na = 0;
    for (int q = 0; q < kPasses; ++q) na += ((vary >> (q * kBits)) & (kBins - 1)) ? 1 : 0;
    const uint64_t cap7 = uint64_t(a.levels == 3 ? kSubBuckets : kBins) * kLocalCap;
    const bool too_big = __syncthreads_or(tid < 256 && uint64_t(t7) > cap7) != 0;
    if (too_big || (na < 4 && !a.bj)) {
      if (blockIdx.x == 0 && tid == 0) atomicOr(a.flags, 1u);
      return;
    }
  }
  const uint32_t b7 = scan256(t7, s.scratch);
  if (tid < 256) s.aux[tid] = b7;
  if (blockIdx.x == 0) {
    // pass-B tiles: a bucket's rows cut into tiles of kPTile
    const uint32_t k = tid < 256 ? (t7 + kPTile - 1) / kPTile : 0u;
    const uint32_t first = scan256(k, s.scratch);
    if (tid < 256) {
      a.d7_base[tid] = b7;
      for (uint32_t j = 0; j < k; ++j) {
        const uint32_t r0 = b7 + j * kPTile, r1 = min(b7 + t7, r0 + kPTile);
        a.items[first + j] = make_uint4(uint32_t(tid), r0, r1, 0u);
      }
    }
    if (tid == 255) {
      a.d7_base[kBins] = uint32_t(a.n);
      a.meta[0] = first + k;
    }
  }
  // this CTA's rows; the first tile's lines are requested into L2 now, so that
  // they arrive during the sub-bucket totals below (prefetching every next tile
  // this way, here and in the digit-6 pass, measured no faster: 0.297 -> 0.303 ms)
  const int64_t lo = chunk_lo(a.n, gridDim.x, blockIdx.x), hi = chunk_lo(a.n, gridDim.x, blockIdx.x + 1);
  const long long* col = static_cast<const long long*>(a.col);
  if (tid == 0) bulk_prefetch_l2(col + lo, size_t(min(hi - lo, int64_t(kPTile))) * 8);
  // sub-bucket starts of bucket g = this CTA (totals over the chunk counts):
  // lane q sums the uint4 column q (sub-buckets 8q .. 8q+7) of one chunk slice,
  // every load of the slice in flight at once
  uint32_t* red = reinterpret_cast<uint32_t*>(s.sk);  // staging is free here
  for (uint32_t g = blockIdx.x; g < uint32_t(kBins); g += gridDim.x) {
    constexpr int kSl = kPThreads / 32;
    constexpr int kU = (kMaxChunks + kSl - 1) / kSl;
    const int q = tid & 31, sl = tid >> 5;
    const uint4* col_g = reinterpret_cast<const uint4*>(a.chunk_cnt + g * 128) + q;
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint4 x[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int cc = sl + u * kSl;
      x[u] = cc < a.chunks ? __ldcg(col_g + size_t(cc) * (kScatWords / 4)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      acc[0] += x[u].x & 0xFFFFu;
      acc[1] += x[u].x >> 16;
      acc[2] += x[u].y & 0xFFFFu;
      acc[3] += x[u].y >> 16;
      acc[4] += x[u].z & 0xFFFFu;
      acc[5] += x[u].z >> 16;
      acc[6] += x[u].w & 0xFFFFu;
      acc[7] += x[u].w >> 16;
    }
    uint4* r4 = reinterpret_cast<uint4*>(red + sl * 256 + q * 8);
    r4[0] = make_uint4(acc[0], acc[1], acc[2], acc[3]);
    r4[1] = make_uint4(acc[4], acc[5], acc[6], acc[7]);
    __syncthreads();
    uint32_t tb = 0;
    if (tid < 256)
#pragma unroll
      for (int j = 0; j < kSl; ++j) tb += red[j * 256 + tid];
    const uint32_t ex = scan256(tb, s.scratch);
    if (tid < 256) {
      a.sub_off[g * 256 + tid] = s.aux[g] + ex;
      if (tb > uint32_t(kLocalCap) && a.levels != 3) atomicOr(a.flags, 1u);  // (3 levels: checked per sub-sub-bucket)
    }
    if (g == kBins - 1 && tid == 0) a.sub_off[kSubBuckets] = uint32_t(a.n);
  }
#ifdef RL_TOP_PROFILE
  if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[4] = globaltimer();
  if (a.stamps && tid == 0) atomicMax(reinterpret_cast<unsigned long long*>(a.stamps) + 5, globaltimer());
#endif
  // a fallback already found (here or by an earlier CTA's prologue): skip the scatter
  if (fallback_flag(a)) return;
  // this CTA's rows by digit 7 -> keys_b / vals_b
  const uint32_t sh = s.scratch[50];
  auto reserve = [&](uint32_t d, uint32_t c) { return make_uint2(s.aux[d], atomicAdd(a.cur7 + d, c)); };
  // the tile loop, compiled per key-packing mode (chosen once)
  const uint32_t shl = pack_shift(sh);
  auto tiles = [&](auto packed, auto pkc) {
    constexpr bool PK = decltype(pkc)::value;
    // every load of a tile is issued during the previous tile's write-out (the
    // payload loads of the common one-column case too); the keys are transformed
    // (finish) only when the tile is ranked, so that nothing waits for them there
    const bool whole_words = CW > 0 && a.carry_n == 1 && a.carry_width[0] == 8 * CW;
    auto load = [&](uint64_t (&k)[kPItems], uint32_t (&v)[kPItems], Carry<CW>& cr, int64_t t0) {
      const int tn = int(hi - t0 < kPTile ? hi - t0 : kPTile);
#pragma unroll
      for (int u = 0; u < kPItems; ++u) {
        const int j = u * kPThreads + tid;
        k[u] = j < tn ? uint64_t(__ldcs(col + t0 + j)) : 0ull;
      }
      if constexpr (CW > 0) {
        if (whole_words) {
          const unsigned long long* src = reinterpret_cast<const unsigned long long*>(a.carry_src[0]);
#pragma unroll
          for (int u = 0; u < kPItems; ++u) {
            const int j = u * kPThreads + tid;
#pragma unroll
            for (int w = 0; w < CW; ++w) cr.p[u][w] = j < tn ? __ldcs(src + (t0 + j) * CW + w) : 0ull;
          }
        } else {
#pragma unroll
          for (int u = 0; u < kPItems; ++u) {
            const int j = u * kPThreads + tid;
            if (j < tn) load_carry<CW>(a, uint64_t(t0 + j), cr.p[u]);
          }
        }
      }
    };
    auto finish = [&](uint64_t (&k)[kPItems], uint32_t (&v)[kPItems], Carry<CW>& cr, int64_t t0) {
      const int tn = int(hi - t0 < kPTile ? hi - t0 : kPTile);
#pragma unroll
      for (int u = 0; u < kPItems; ++u) {
        const int j = u * kPThreads + tid;
        k[u] = j < tn ? pack_as<decltype(packed)::value>(xform(k[u], a.desc), sh, shl) : 0ull;
        if constexpr (PK) k[u] |= uint64_t(uint32_t(t0 + j));
        else if constexpr (CW > 0) cr.p[u][0] = (cr.p[u][0] << 32) | uint32_t(t0 + j);  // idw: (columns, row id)
        else v[u] = uint32_t(t0 + j);
      }
    };
    uint64_t k[kPItems];
    uint32_t v[kPItems];
    Carry<CW> cr;
    if (lo < hi) load(k, v, cr, lo);
    if (tid < 256) s.hist[tid] = 0;
    __syncthreads();
    for (int64_t t0 = lo; t0 < hi; t0 += kPTile) {
      const int tn = int(hi - t0 < kPTile ? hi - t0 : kPTile);
      const int64_t nt = t0 + kPTile;
      finish(k, v, cr, t0);
      ptile_scatter<7 * kBits, PK, CW>(k, v, cr, tn, s, a.keys_b, a.vals_b, a.pay_b, reserve,
                                       [&](uint64_t (&kk)[kPItems], uint32_t (&vv)[kPItems], Carry<CW>& cc) {
                                         if (nt < hi) load(kk, vv, cc, nt);
                                       });
    }
  };
  using F = std::false_type;
  using T = std::true_type;
  const bool pk = packed_rows(sh, a);
  if constexpr (CW > 0) {  // carried payload rides with packed rows (the bucket join's plan checks the code)
    if (!packed_rows(sh, a)) {
      // keys that do not pack: one word of <= 4 carried bytes holds the row id
      // too (idw); wider carried columns: the LSD passes gather them instead
      if (CW != 1 || !a.idw) {
        if (tid == 0) atomicOr(a.flags, 1u);
        return;
      }
      switch (pack_mode(sh)) {
        case 0: tiles(std::integral_constant<int, 0>{}, F{}); break;
        case 1: tiles(std::integral_constant<int, 1>{}, F{}); break;
        default: tiles(std::integral_constant<int, 2>{}, F{}); break;
      }
      return;
    }
    if (pack_mode(sh) == 1) tiles(std::integral_constant<int, 1>{}, T{});
    else tiles(std::integral_constant<int, 2>{}, T{});
    return;
  }
  switch (pack_mode(sh)) {
    case 0: tiles(std::integral_constant<int, 0>{}, F{}); break;
    case 1:
      if (pk) tiles(std::integral_constant<int, 1>{}, T{});
      else tiles(std::integral_constant<int, 1>{}, F{});
      break;
    default:
      if (pk) tiles(std::integral_constant<int, 2>{}, T{});
      else tiles(std::integral_constant<int, 2>{}, F{});
      break;
  }
#ifdef RL_TOP_PROFILE
  if (a.stamps && tid == 0) atomicMax(reinterpret_cast<unsigned long long*>(a.stamps) + 6, globaltimer());
#endif
}

template <bool PK, int CW>
__device__ __forceinline__ void sub_scatter_tiles(const SortArgs& a, const PTile& s);

template <int CW = 0>
__global__ void __launch_bounds__(kPThreads, RL_PASS_CTAS_PER_SM) sub_scatter_kernel(SortArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  const PTile s = ptile<CW>(sm);
  const int tid = threadIdx.x;
  pdl_wait();  // the digit-7 pass
  pdl_launch_dependents();
  if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[3] = globaltimer();
  if (tid == 0) s.scratch[50] = __ldcg(a.flags + 6);  // the key pack code
  if (fallback_flag(a)) return;  // LSD fallback (the barrier also publishes scratch[50])
  if constexpr (CW > 0) {
    if (packed_rows(s.scratch[50], a)) sub_scatter_tiles<true, CW>(a, s);
    else if constexpr (CW == 1) sub_scatter_tiles<false, CW>(a, s);  // idw (the digit-7 pass declined otherwise)
  } else {
    if (packed_rows(s.scratch[50], a)) sub_scatter_tiles<true, 0>(a, s);
    else sub_scatter_tiles<false, 0>(a, s);
  }
#ifdef RL_TOP_PROFILE
  if (a.stamps && tid == 0) atomicMax(reinterpret_cast<unsigned long long*>(a.stamps) + 7, globaltimer());
#endif
}

// The tiles of the digit-6 / digit-5 passes are claimed from a counter in
// bucket order (the runs being written span a few MB: every sector completes
// in L2). One thread (kClaimer: warp 15, idle beside the digit scan) keeps the
// claims two tiles ahead: during tile t (mid) it reads the descriptor of tile
// t + 1 into slot[(t + 1) & 1] and claims tile t + 2, so the next tile's loads
// (issued at the staging barrier) wait for no atomic or descriptor round trip.
constexpr int kClaimer = kPThreads - 1;
__device__ __forceinline__ uint4 no_tile() { return make_uint4(~0u, 0u, 0u, 0u); }

template <bool PK, int CW>
__device__ __forceinline__ void sub_scatter_tiles(const SortArgs& a, const PTile& s) {
  const int tid = threadIdx.x;
  const uint32_t n_items = __ldcg(a.meta);
  uint4* slot = reinterpret_cast<uint4*>(s.scratch + 52);  // [2] descriptors (bucket, first row, end row)
  auto load = [&](uint64_t (&k)[kPItems], uint32_t (&v)[kPItems], Carry<CW>& cr, const uint4& item) {
    const int tn = int(item.z - item.y);
#pragma unroll
    for (int u = 0; u < kPItems; ++u) {
      const int j = u * kPThreads + tid;
      k[u] = j < tn ? __ldcs(a.keys_b + item.y + j) : 0ull;
      if constexpr (!PK && CW == 0) v[u] = j < tn ? __ldcs(a.vals_b + item.y + j) : 0u;
      if constexpr (CW > 0) {
#pragma unroll
        for (int w = 0; w < CW; ++w) cr.p[u][w] = j < tn ? __ldcs(a.pay_b + (size_t(item.y) + j) * CW + w) : 0ull;
      }
    }
  };
  uint32_t ahead = 0;  // (kClaimer) the claim two tiles ahead
  if (tid == kClaimer) {
    const uint32_t c0 = atomicAdd(a.flags + 3, 1u);
    slot[0] = c0 < n_items ? __ldcg(a.items + c0) : no_tile();
    ahead = atomicAdd(a.flags + 3, 1u);
  }
  if (tid < 256) s.hist[tid] = 0;
  __syncthreads();
  uint32_t par = 0;
  uint4 item = slot[0];
  uint64_t k[kPItems];
  uint32_t v[kPItems];
  Carry<CW> cr;
  if (item.x != ~0u) load(k, v, cr, item);
  while (item.x != ~0u) {
    const uint32_t g = item.x;
    uint4 nitem = no_tile();
    auto reserve = [&](uint32_t d, uint32_t c) {
      return make_uint2(__ldcg(a.sub_off + g * 256 + d), atomicAdd(a.cur16 + g * 256 + d, c));
    };
    ptile_scatter<6 * kBits, PK, CW>(
        k, v, cr, int(item.z - item.y), s, a.keys_a, a.vals_a, a.pay_a, reserve,
        [&](uint64_t (&kk)[kPItems], uint32_t (&vv)[kPItems], Carry<CW>& cc) {
          nitem = slot[par ^ 1];
          if (nitem.x != ~0u) load(kk, vv, cc, nitem);
        },
        [&]() {
          if (tid == kClaimer) {
            slot[par ^ 1] = ahead < n_items ? __ldcg(a.items + ahead) : no_tile();
            if (ahead < n_items) ahead = atomicAdd(a.flags + 3, 1u);
          }
        });
    item = nitem;
    par ^= 1;
  }
}

// ---------------------------------------------------------------- third level
// Above ~65536 x kLocalCap rows the (d7, d6) sub-buckets no longer fit on chip:
// digit 5 splits each of them (2^24 sub-sub-buckets). The level-2 pass leaves
// every sub-bucket contiguous in keys_a, so its digit-5 counts need no global
// atomics: count3_kernel reads each sub-bucket once (a CTA per sub-bucket at a
// time), writes its 256 sub-sub-bucket starts and its tile count (a sub-sub-
// bucket above kLocalCap sets the LSD fallback); tile_scan_kernel turns the
// tile counts into a prefix; sub3_scatter_kernel scatters every tile of a
// sub-bucket by digit 5 into keys_b (reservations from the starts + per-
// sub-sub-bucket cursors); the local phase then sorts runs of sub-sub-buckets.
__global__ void __launch_bounds__(kPThreads, RL_PASS_CTAS_PER_SM) count3_kernel(SortArgs a) {
  __shared__ uint32_t h[256];
  __shared__ uint32_t scratch[64];
  const int tid = threadIdx.x;
  pdl_wait();  // the digit-6 pass
  pdl_launch_dependents();
  if (fallback_flag(a)) return;
  for (uint32_t sb = blockIdx.x; sb < uint32_t(kSubBuckets); sb += gridDim.x) {
    const uint32_t lo = __ldcg(a.sub_off + sb), hi = __ldcg(a.sub_off + sb + 1);
    if (tid < 256) h[tid] = 0;
    __syncthreads();
    uint32_t i = lo + tid;
    for (; i + 3 * kPThreads < hi; i += 4 * kPThreads) {  // four loads in flight
      uint64_t k4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) k4[u] = __ldcs(a.keys_a + i + u * kPThreads);
#pragma unroll
      for (int u = 0; u < 4; ++u) atomicAdd(&h[uint32_t(k4[u] >> 40) & 255u], 1u);
    }
    for (; i < hi; i += kPThreads) atomicAdd(&h[uint32_t(__ldcs(a.keys_a + i) >> 40) & 255u], 1u);
    __syncthreads();
    const uint32_t c = tid < 256 ? h[tid] : 0u;
    const uint32_t ex = scan256(c, scratch);
    if (tid < 256) {
      a.sub3_off[sb * 256 + tid] = lo + ex;
      if (c > uint32_t(kLocalCap)) atomicOr(a.flags, 1u);
    }
    if (tid == 0) a.tile3[sb] = (hi - lo + kPTile - 1) / kPTile;
    if (sb == uint32_t(kSubBuckets) - 1 && tid == 0) a.sub3_off[kSub3] = uint32_t(a.n);
    __syncthreads();
  }
}

// One CTA: the 65536 tile counts -> exclusive prefix in place, total in meta[1].
__global__ void __launch_bounds__(1024) tile_scan_kernel(SortArgs a) {
  constexpr int kChunk = 8192, kPer = kChunk / 1024;
  __shared__ uint32_t buf[kChunk];
  __shared__ uint32_t scratch[40];
  const int tid = threadIdx.x;
  pdl_wait();
  pdl_launch_dependents();
  if (fallback_flag(a)) return;
  uint32_t carry = 0;
  for (int c0 = 0; c0 < kSubBuckets; c0 += kChunk) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) buf[i * 1024 + tid] = __ldcg(a.tile3 + c0 + i * 1024 + tid);
    __syncthreads();
    uint32_t run = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) run += buf[tid * kPer + i];
    uint32_t total;
    uint32_t start = carry + block_exclusive_scan<1024>(run, scratch, &total);
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const uint32_t v = buf[tid * kPer + i];
      const uint32_t sb = uint32_t(c0 + tid * kPer + i);
      a.tile3[sb] = start;
      if (v) {  // the sub-bucket's tiles: (sub-bucket, first row, end row)
        const uint32_t lo = __ldcg(a.sub_off + sb), hi = __ldcg(a.sub_off + sb + 1);
        uint4* td = reinterpret_cast<uint4*>(a.tmap);
        for (uint32_t j = 0; j < v; ++j) td[start + j] = make_uint4(sb, lo + j * kPTile, min(hi, lo + (j + 1) * kPTile), 0u);
      }
      start += v;
    }
    carry += total;
    __syncthreads();
  }
  if (tid == 0) {
    a.tile3[kSubBuckets] = carry;
    a.meta[1] = carry;
  }
}

template <bool PK, int CW = 0>
__device__ __forceinline__ void sub3_scatter_tiles(const SortArgs& a, const PTile& s) {
  const int tid = threadIdx.x;
  const uint32_t n_tiles = __ldcg(a.meta + 1);
  const uint4* tdesc = reinterpret_cast<const uint4*>(a.tmap);  // (sub-bucket, first row, end row) a tile
  uint4* slot = reinterpret_cast<uint4*>(s.scratch + 52);
  auto load = [&](uint64_t (&k)[kPItems], uint32_t (&v)[kPItems], Carry<CW>& cc, const uint4& d) {
    const int tn = int(d.z - d.y);
#pragma unroll
    for (int u = 0; u < kPItems; ++u) {
      const int j = u * kPThreads + tid;
      k[u] = j < tn ? __ldcs(a.keys_a + d.y + j) : 0ull;
      if constexpr (!PK && CW == 0) v[u] = j < tn ? __ldcs(a.vals_a + d.y + j) : 0u;
      if constexpr (CW > 0) {
#pragma unroll
        for (int w = 0; w < CW; ++w) cc.p[u][w] = j < tn ? __ldcs(a.pay_a + (size_t(d.y) + j) * CW + w) : 0ull;
      }
    }
  };
  uint32_t ahead = 0;  // (kClaimer) the claim two tiles ahead (see sub_scatter_tiles)
  if (tid == kClaimer) {
    const uint32_t c0 = atomicAdd(a.flags + 2, 1u);
    slot[0] = c0 < n_tiles ? __ldcg(tdesc + c0) : no_tile();
    ahead = atomicAdd(a.flags + 2, 1u);
  }
  if (tid < 256) s.hist[tid] = 0;
  __syncthreads();
  uint32_t par = 0;
  uint4 d = slot[0];
  uint64_t k[kPItems];
  uint32_t v[kPItems];
  Carry<CW> cr;
  if (d.x != ~0u) load(k, v, cr, d);
  while (d.x != ~0u) {
    const uint32_t g = d.x;
    uint4 nd = no_tile();
    auto reserve = [&](uint32_t dg, uint32_t c) {
      return make_uint2(__ldcg(a.sub3_off + g * 256 + dg), atomicAdd(a.cur24 + g * 256 + dg, c));
    };
    ptile_scatter<5 * kBits, PK, CW>(
        k, v, cr, int(d.z - d.y), s, a.keys_b, a.vals_b, a.pay_b, reserve,
        [&](uint64_t (&kk)[kPItems], uint32_t (&vv)[kPItems], Carry<CW>& cc) {
          nd = slot[par ^ 1];
          if (nd.x != ~0u) load(kk, vv, cc, nd);
        },
        [&]() {
          if (tid == kClaimer) {
            slot[par ^ 1] = ahead < n_tiles ? __ldcg(tdesc + ahead) : no_tile();
            if (ahead < n_tiles) ahead = atomicAdd(a.flags + 2, 1u);
          }
        });
    d = nd;
    par ^= 1;
  }
}

template <int CW = 0>  // CW > 0: the bucket join's carried payload words (packed rows)
__global__ void __launch_bounds__(kPThreads, RL_PASS_CTAS_PER_SM) sub3_scatter_kernel(SortArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  const PTile s = ptile<CW>(sm);
  const int tid = threadIdx.x;
  pdl_wait();  // the tile prefix
  pdl_launch_dependents();
  if (tid == 0) s.scratch[50] = __ldcg(a.flags + 6);
  if (fallback_flag(a)) return;
  if constexpr (CW > 0) {
    if (packed_rows(s.scratch[50], a)) sub3_scatter_tiles<true, CW>(a, s);
    else if constexpr (CW == 1) sub3_scatter_tiles<false, CW>(a, s);  // idw
  } else {
    if (packed_rows(s.scratch[50], a)) sub3_scatter_tiles<true>(a, s);
    else sub3_scatter_tiles<false>(a, s);
  }
}

__device__ __forceinline__ bool row_less(uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
  return ka < kb || (ka == kb && va < vb);
}

// Sort rows [lo, hi) of B by (key, row id) — one warp, bitonic network
// with mirrored first steps (every comparator ascending), so rows past hi
// act as +inf padding and their comparators are skipped.
template <bool PK = false, bool MOVE_V = false>  // PK: the key word alone orders rows; MOVE_V: bv moves along
__device__ void warp_bitonic(uint64_t* bk, uint32_t* bv, uint32_t lo, uint32_t hi, int lane) {
  const uint32_t sz = hi - lo;
  uint32_t p2 = 1;
  while (p2 < sz) p2 <<= 1;
  for (uint32_t k = 2; k <= p2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t t = lane; t < (p2 >> 1); t += 32) {
        const uint32_t i = (t / j) * (2 * j) + (t % j);
        const uint32_t q = j == (k >> 1) ? (i ^ (k - 1)) : (i + j);
        if (q < sz) {
          const uint64_t ka = bk[lo + i], kb = bk[lo + q];
          if constexpr (PK) {
            if (kb < ka) {
              bk[lo + i] = kb; bk[lo + q] = ka;
              if constexpr (MOVE_V) {
                const uint32_t t = bv[lo + i];
                bv[lo + i] = bv[lo + q];
                bv[lo + q] = t;
              }
            }
          } else {
            const uint32_t va = bv[lo + i], vb = bv[lo + q];
            if (row_less(kb, vb, ka, va)) {
              bk[lo + i] = kb; bk[lo + q] = ka;
              bv[lo + i] = vb; bv[lo + q] = va;
            }
          }
        }
      }
      __syncwarp();
    }
  }
}

// warp_bitonic for idw runs: rows ordered by (key, row id), the id read from
// the run's carried word behind each row's u16 load index.
__device__ void warp_bitonic_idw(uint64_t* bk, uint16_t* bi, const uint64_t* aw, uint32_t lo, uint32_t hi, int lane) {
  const uint32_t sz = hi - lo;
  uint32_t p2 = 1;
  while (p2 < sz) p2 <<= 1;
  for (uint32_t k = 2; k <= p2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t t = lane; t < (p2 >> 1); t += 32) {
        const uint32_t i = (t / j) * (2 * j) + (t % j);
        const uint32_t q = j == (k >> 1) ? (i ^ (k - 1)) : (i + j);
        if (q < sz) {
          const uint64_t ka = bk[lo + i], kb = bk[lo + q];
          const uint16_t ia = bi[lo + i], ib = bi[lo + q];
          if (kb < ka || (kb == ka && uint32_t(aw[ib]) < uint32_t(aw[ia]))) {
            bk[lo + i] = kb; bk[lo + q] = ka;
            bi[lo + i] = ib; bi[lo + q] = ia;
          }
        }
      }
      __syncwarp();
    }
  }
}

// The local phase. CTA c owns groups c, c + grid, ... of kGroupSubs
// consecutive sub-buckets; each group is cut into runs of whole sub-buckets
// of at most kLocalCap rows. Runs are double-buffered: while one is sorted
// the next streams in with TMA bulk copies, and the offsets of the next
// group are loaded a group ahead. A run is sorted on chip by (top16, d5)
// with a counting scatter (one shared atomic per row: the order inside a
// bin is settled next), then each row takes its rank by (key, row id)
// inside its bin — rows equal in their top 24 bits, ~1 for uniform keys; a
// warp's bitonic network for bins above 32 rows — and goes straight to its
// final position in the outputs, with the fused gathers.

// Greedy cut of one group (offsets off[0..G]) into runs of whole sub-buckets
// of at most kLocalCap rows; run = (first << 16) | end; returns the count.
template <int G>
__device__ __forceinline__ uint32_t cut_group(const uint32_t* off, uint32_t* ends) {
  if (off[G] - off[0] <= uint32_t(kLocalCap)) {  // the common case: the whole group is one run
    if (off[G] == off[0]) return 0;
    ends[0] = uint32_t(G);  // (0 << 16) | G
    return 1;
  }
  uint32_t nr = 0, s = 0;
  while (s < uint32_t(G)) {
    const uint32_t base = off[s];
    uint32_t e = s + 1;
    while (e < uint32_t(G) && off[e + 1] - base <= uint32_t(kLocalCap)) ++e;
    if (off[e] > base) ends[nr++] = (s << 16) | e;
    s = e;
  }
  return nr;
}

__device__ __forceinline__ void issue_run(const uint64_t* kin, const uint32_t* vin, uint32_t base, uint32_t cnt,
                                          uint8_t* abuf, uint64_t* bar) {
  const uint32_t k0 = base & ~1u, v0 = base & ~3u;
  const uint32_t kbytes = ((base + cnt - k0) * 8u + 15u) & ~15u;
  const uint32_t vbytes = vin ? ((base + cnt - v0) * 4u + 15u) & ~15u : 0u;  // packed rows: keys only
  fence_proxy_async_smem();
  mbar_expect_tx(bar, kbytes + vbytes);
  bulk_g2s(abuf, kin + k0, kbytes, bar);
  if (vbytes) bulk_g2s(abuf + kLocAKeys, vin + v0, vbytes, bar);
}

// idw: the run's keys and carried words (same alignment: both 8 bytes a row)
__device__ __forceinline__ void issue_run_w(const uint64_t* kin, const uint64_t* win, uint32_t base, uint32_t cnt,
                                            uint8_t* abuf, uint64_t* bar) {
  const uint32_t k0 = base & ~1u;
  const uint32_t bytes = ((base + cnt - k0) * 8u + 15u) & ~15u;
  fence_proxy_async_smem();
  mbar_expect_tx(bar, 2 * bytes);
  bulk_g2s(abuf, kin + k0, bytes, bar);
  bulk_g2s(abuf + kLocAKeys, win + k0, bytes, bar);
}

// BAL (the scatter path's large runs): a thread's rows in registers across
// count + scatter, and the claimed group tail. The onesweep hybrid's short
// runs (n < 4M) are faster without both (+1-5 us each at 0.3-2M rows).
// PROD (the scatter path's kernels, THREADS + 32 threads): warp THREADS / 32
// is a producer — it walks the groups, cuts the runs and issues every run's
// TMA into a free buffer (full / empty mbarriers) — so the group bookkeeping
// and the copy issue (~15 % of a run, measured) leave the consumers' path; the
// consumers synchronise on named barrier 1.
template <int THREADS, int PACK = 0, bool BAL = false, bool PK = false, int LEVELS = 2, int CW = 0, bool PROD = false>
__device__ void local_phase(const SortArgs& a, uint8_t* smem, uint32_t src) {
  // CW > 0 (packed rows): every row's payload words ride in pay_a / pay_b beside
  // its key; bv holds the row's load index in its run, and the emit copies the
  // carried columns out of the run's payload window (no gather by row id)
  // idw (CW == 1, keys that do not pack): the carried word holds the row id
  // (low half) and the columns' bytes (high half); it is staged with the key
  // by TMA, bv holds the load index, ties compare the ids behind the indexes
  constexpr bool IDW = CW == 1 && !PK;
  static_assert(CW == 0 || PK || IDW, "carried payload rides with packed rows, or as idw words");
  static_assert(!IDW || BAL, "idw runs use the in-place layout");
  constexpr size_t kABytes = IDW ? kLocABytesW : kLocABytes;
  const uint64_t* pay = CW ? (src == 1 ? a.pay_a : a.pay_b) : nullptr;
  // sub-buckets of the runs: (d7, d6) or, with three levels, (d7, d6, d5)
  constexpr int kSubShift = LEVELS == 3 ? 40 : 48;
  const uint32_t* sub_off = LEVELS == 3 ? a.sub3_off : a.sub_off;
  constexpr int kLWarps = THREADS / 32;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + (IDW ? kLocHistW : BAL ? kLocHistBal : kLocHist));
  uint32_t* bv = reinterpret_cast<uint32_t*>(smem + (BAL ? kLocBvBal : kLocBv));
  uint16_t* bv16 = reinterpret_cast<uint16_t*>(smem + kLocBvW);  // idw
  uint32_t* big = reinterpret_cast<uint32_t*>(smem + kLocBig);
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + kLocMisc);
  // a work item: G consecutive sub-buckets (three levels: the 256 sub-sub-buckets
  // of one (d7, d6) sub-bucket), its offsets and runs in two slots
  constexpr int G = LEVELS == 3 ? 256 : kGroupSubs;
  constexpr int GO = G + 1;
  uint32_t* goff = LEVELS == 3 ? reinterpret_cast<uint32_t*>(smem + kLocGrp) : misc + 32;  // [2][G + 1]
  uint32_t* gends = LEVELS == 3 ? goff + 2 * GO : misc + 72;                              // [2][G]
  uint32_t* runs = misc + 112;  // [2][4] descriptors of the run in each buffer
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kLocBars);  // [0..1] full (data landed), PROD: [2..3] empty
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  static_assert(!PROD || BAL, "the producer warp serves the in-place runs");
  constexpr int kPW = PROD ? THREADS / 32 : 0;  // the warp that walks the groups
  auto csync = [&]() {  // the run's threads (PROD: the consumers only)
    if constexpr (PROD) asm volatile("bar.sync 1, %0;" ::"n"(THREADS) : "memory");
    else __syncthreads();
  };
  const uint64_t* kin = src == 1 ? a.keys_a : a.keys_b;
  const uint32_t* vin = PK ? nullptr : src == 1 ? a.vals_a : a.vals_b;
  const int desc = a.key_mode == kRawDesc;
  constexpr uint32_t kGroups = (LEVELS == 3 ? kSub3 : kSubBuckets) / G;
  constexpr int kNBins = BAL ? kLocalBinsBal : kLocalBins;
  constexpr uint32_t kBinBits = BAL ? uint32_t(RL_LOCAL_BAL_BITS) : 12u;
  const uint32_t g0 = blockIdx.x;
  if (g0 >= kGroups) return;
  // group schedule: the first nstat groups of every CTA on a static stride
  // (no atomic on warp 0's path: it issues the next run's TMA while the other
  // warps wait), the last ~2 rounds claimed from a counter (flags[1], zeroed
  // per sort) so that CTAs which drew short groups take more — the static
  // stride alone left the last CTA ~15 us behind the first at 10M rows; claims
  // throughout cost ~0.6 us of warp-0 latency per group (+9 us at 1M rows).
  uint32_t* gid = misc + 120;  // [2] the group whose offsets are in goff slot s (warp 0 only)
  // groups below lim go by the static stride, the rest are claimed
  const uint32_t lim = !BAL ? 0xFFFFFFFFu
                            : (max(1u, kGroups / gridDim.x) - (kGroups / gridDim.x > 1 ? 1u : 0u)) * gridDim.x;
  auto claim = [&](uint32_t last) -> uint32_t {  // warp 0, converged; last = the group claimed before
    if constexpr (!BAL) return last + gridDim.x;
    if (last + gridDim.x < lim) return last + gridDim.x;
    uint32_t g = 0;
    if (lane == 0) g = lim + atomicAdd(a.flags + 1, 1u);
    return __shfl_sync(0xffffffffu, g, 0);
  };

  // ---- prologue (warp 0): offsets of the first group, its runs, the first
  // TMA; the next group is claimed and its offsets requested into registers
  // warp 0: the sub-bucket offsets of group next_g, requested into a register
  // a group ahead (groups of 16); the three-level path's 257 offsets are read
  // when the group is moved into its slot (its groups are ~256x larger)
  uint32_t next_off = 0;
  uint32_t next_g = g0;
  auto fetch_next = [&]() {
    if constexpr (G <= 31) next_off = lane <= uint32_t(G) && next_g < kGroups ? __ldcg(sub_off + size_t(next_g) * G + lane) : 0u;
  };
  if (warp == kPW) {
    if (lane == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      if constexpr (PROD) {
        mbar_init(&bars[2], 1);
        mbar_init(&bars[3], 1);
      }
      gid[0] = g0;
    }
    for (uint32_t i = lane; i <= uint32_t(G); i += 32) goff[i] = __ldcg(sub_off + size_t(g0) * G + i);
    next_g = claim(next_g);
    fetch_next();
    __syncwarp();
    if (lane == 0) misc[2] = cut_group<G>(goff, gends);
    __syncwarp();
  }
  // warp 0: move the claimed group's offsets into goff slot s, claim the next;
  // false when no group is left
  auto advance = [&](uint32_t s) -> bool {
    const uint32_t gn = next_g;
    if (gn >= kGroups) return false;
    if constexpr (G <= 31) {
      if (lane <= uint32_t(G)) goff[s * GO + lane] = next_off;
    } else {
      for (uint32_t i = lane; i <= uint32_t(G); i += 32) goff[s * GO + i] = __ldcg(sub_off + size_t(gn) * G + i);
    }
    if (lane == 0) gid[s] = gn;
    next_g = claim(next_g);
    fetch_next();
    __syncwarp();
    if (lane == 0) misc[2 + s] = cut_group<G>(goff + s * GO, gends + s * G);
    __syncwarp();
    return true;
  };
  __syncthreads();
  // the scatter path's key pack code and constant bits (staged in misc[125..127] by the caller)
  const uint32_t pcode = PACK ? misc[125] : 0u;
  const uint64_t constbits = PACK ? (uint64_t(misc[127]) << 32) | misc[126] : 0ull;
  const uint32_t pshl = pack_shift(pcode);
  // run cursor: group k (g = g0 + k gstep), run r of that group; identical in every thread
  uint32_t k = 0, r = 0, buf = 0, phase0 = 0, phase1 = 0;
  if constexpr (PROD) {
    if (warp == kPW) {  // ---- the producer: run q goes into buffer q & 1 once run q - 2 released it
      for (uint32_t q = 0;; ++q, ++r) {
        bool ok = true;
        while (r >= misc[2 + (k & 1)]) {  // past the group's runs (or an empty group): the next group
          if (!advance((k + 1) & 1)) {
            ok = false;
            break;
          }
          ++k;
          r = 0;
        }
        const uint32_t b = q & 1;
        if (q >= 2) mbar_wait(&bars[2 + b], ((q >> 1) + 1) & 1);
        if (lane == 0) {
          uint32_t* d = runs + b * 4;
          if (ok) {
            const uint32_t* off = goff + (k & 1) * GO;
            const uint32_t se = gends[(k & 1) * G + r];
            const uint32_t base = off[se >> 16], cnt = off[se & 0xFFFFu] - base;
            d[0] = base;
            d[1] = cnt;
            d[2] = gid[k & 1] * G + (se >> 16);
            d[3] = (se & 0xFFFFu) - (se >> 16);
            if constexpr (IDW) issue_run_w(kin, pay, base, cnt, smem + kLocA + b * kABytes, &bars[b]);
            else issue_run(kin, vin, base, cnt, smem + kLocA + b * kLocABytes, &bars[b]);
          } else {
            d[1] = ~0u;  // no run left: the consumers stop
            mbar_arrive(&bars[b]);
          }
        }
        __syncwarp();
        if (!ok) return;
      }
    }
  }
  bool have = PROD || misc[2] > 0;
  // an empty first group: advance (rare; only tiny inputs have empty groups)
  while (!have) {
    __syncthreads();
    if (warp == 0) {
      const bool got = advance((k + 1) & 1);
      if (lane == 0) misc[7] = got ? 1u : 0u;
    }
    __syncthreads();
    ++k;
    if (!misc[7]) return;
    have = misc[2 + (k & 1)] > 0;
  }
  if (!PROD && tid == 0) {
    const uint32_t* off = goff + (k & 1) * GO;
    const uint32_t se = gends[(k & 1) * G];
    const uint32_t base = off[se >> 16], cnt = off[se & 0xFFFFu] - base;
    runs[0] = base;
    runs[1] = cnt;
    runs[2] = gid[k & 1] * G + (se >> 16);
    runs[3] = (se & 0xFFFFu) - (se >> 16);
    if constexpr (IDW) issue_run_w(kin, pay, base, cnt, smem + kLocA, &bars[0]);
    else issue_run(kin, vin, base, cnt, smem + kLocA, &bars[0]);
  }
  if constexpr (!PROD) __syncthreads();  // the first run's descriptor is visible to every thread
  uint32_t q = 0;  // PROD: runs taken

#ifdef RL_PASS_PROFILE
  long long lpt = clock64();
#define LPROF(i) do { if (BAL && CW == 0 && LEVELS == 2) PPROF(16 + (i), lpt); } while (0)
#else
#define LPROF(i) do { } while (0)
#endif
  while (true) {
    LPROF(7);  // (the end of the previous run's big bins)
    uint32_t first, nsb, bb, nbins, next_k = 0, next_r = 0;
    bool more = false;
    if constexpr (PROD) {  // the producer's run q (or the stop mark) in buffer q & 1
      buf = q & 1;
      for (uint32_t i = tid; i < uint32_t(kNBins / 4); i += THREADS) reinterpret_cast<uint4*>(hist)[i] = make_uint4(0, 0, 0, 0);
      mbar_wait(&bars[buf], (q >> 1) & 1);
      if (runs[buf * 4 + 1] == ~0u) break;
      first = runs[buf * 4 + 2];
      nsb = runs[buf * 4 + 3];
      bb = kBinBits - (nsb > 1 ? 32u - uint32_t(__clz(int(nsb - 1))) : 0u);
      nbins = nsb << bb;
      csync();  // hist zeroed
    } else {
    // ---- warp 0: find and prefetch the next run into the other buffer
    if (warp == 0) {
      uint32_t nk = k, nr = r + 1;
      bool ok = true;
      while (nr >= misc[2 + (nk & 1)]) {  // past the group's runs: the next group (offsets were prefetched)
        if (!advance((nk + 1) & 1)) {
          ok = false;
          break;
        }
        ++nk;
        nr = 0;
      }
      LPROF(6);  // (warp 0: the next group's offsets and runs)
      if (lane == 0) {
        misc[4] = ok ? 1u : 0u;
        misc[5] = nk;
        misc[6] = nr;
        if (ok) {
          const uint32_t* off = goff + (nk & 1) * GO;
          const uint32_t se = gends[(nk & 1) * G + nr];
          const uint32_t base = off[se >> 16], cnt = off[se & 0xFFFFu] - base;
          uint32_t* d = runs + (buf ^ 1) * 4;
          d[0] = base;
          d[1] = cnt;
          d[2] = gid[nk & 1] * G + (se >> 16);
          d[3] = (se & 0xFFFFu) - (se >> 16);
          if constexpr (IDW) issue_run_w(kin, pay, base, cnt, smem + kLocA + (buf ^ 1) * kABytes, &bars[buf ^ 1]);
          else issue_run(kin, vin, base, cnt, smem + kLocA + (buf ^ 1) * kLocABytes, &bars[buf ^ 1]);
        }
      }
    }
    // ---- this run: only the bins of its sub-buckets are zeroed and scanned
    // bins of this run: (sub-bucket, the next bb key bits), run-relative; the
    // fewer sub-buckets a run holds, the more bits each gets (4096 bins at most:
    // a run of one big sub-bucket is split 4096 ways, not 256)
    first = runs[buf * 4 + 2];
    nsb = runs[buf * 4 + 3];
    bb = kBinBits - (nsb > 1 ? 32u - uint32_t(__clz(int(nsb - 1))) : 0u);
    nbins = nsb << bb;
    LPROF(0);  // warp 0's prefetch of the next run
    for (uint32_t i = tid; i < nbins / 4; i += THREADS) reinterpret_cast<uint4*>(hist)[i] = make_uint4(0, 0, 0, 0);
    mbar_wait(&bars[buf], buf ? phase1 : phase0);
    if (buf) phase1 ^= 1;
    else phase0 ^= 1;
    __syncthreads();  // hist zeroed, run descriptors and next-run fields visible
    LPROF(1);  // zeroing + this run's data + barrier
    // the next-run fields go to registers now: warp 0 rewrites them at the top
    // of the next run, with no barrier at the end of this one
    more = misc[4] != 0;
    next_k = misc[5];
    next_r = misc[6];
    }
    if (tid == 0) misc[0] = 0;  // big-bin list: appended after later barriers, read after the rank loop
    const uint32_t base = runs[buf * 4], cnt = runs[buf * 4 + 1];
    uint8_t* abuf = smem + kLocA + buf * kABytes;
    const uint64_t* ak = reinterpret_cast<const uint64_t*>(abuf) + (base & 1u);
    const uint32_t* av = reinterpret_cast<const uint32_t*>(abuf + kLocAKeys) + (base & 3u);
    const uint64_t* aw = reinterpret_cast<const uint64_t*>(abuf + kLocAKeys) + (base & 1u);  // idw
    // the bin-ordered keys: BAL, in this run's own key buffer (read into registers first)
    uint64_t* bk = reinterpret_cast<uint64_t*>(BAL ? abuf : smem + kLocBk);
    auto bin_of = [&](uint64_t key) {
      return int(((uint32_t(key >> kSubShift) - first) << bb) | (uint32_t(key >> (kSubShift - bb)) & ((1u << bb) - 1u)));
    };
    // BAL: a thread's rows of the run (at most kRows: kLocalCap / THREADS),
    // loaded once into registers — the loads issue together instead of one per
    // shared atomic (which they may not pass: same memory) — kept for the scatter
    constexpr int kRows = BAL ? (kLocalCap + THREADS - 1) / THREADS : 1;
    uint64_t rk[kRows];
    if constexpr (BAL) {
#pragma unroll
      for (int u = 0; u < kRows; ++u) {
        const uint32_t j = tid + u * THREADS;
        rk[u] = j < cnt ? ak[j] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < kRows; ++u)
        if (tid + u * THREADS < cnt) atomicAdd(&hist[bin_of(rk[u])], 1u);
    } else {
      for (uint32_t j = tid; j < cnt; j += THREADS) atomicAdd(&hist[bin_of(ak[j])], 1u);
    }
    csync();
    LPROF(2);  // counting
    scan_counters<THREADS, kNBins, PROD ? 1 : 0>(hist, nbins, misc + 8);  // (ends synchronised)
    LPROF(3);  // scan
    if constexpr (BAL) {
      uint32_t pos[kRows];
#pragma unroll
      for (int u = 0; u < kRows; ++u)
        if (tid + u * THREADS < cnt) pos[u] = atomicAdd(&hist[bin_of(rk[u])], 1u);
#pragma unroll
      for (int u = 0; u < kRows; ++u) {
        const uint32_t j = tid + u * THREADS;
        if (j < cnt) {
          bk[pos[u]] = rk[u];
          if constexpr (IDW) bv16[pos[u]] = uint16_t(j);
          else if constexpr (!PK) bv[pos[u]] = av[j];
          else if constexpr (CW > 0) bv[pos[u]] = j;
        }
      }
    } else {
      for (uint32_t j = tid; j < cnt; j += THREADS) {
        const uint64_t key = ak[j];
        const uint32_t pos = atomicAdd(&hist[bin_of(key)], 1u);
        bk[pos] = key;
        if constexpr (!PK) bv[pos] = av[j];
        else if constexpr (CW > 0) bv[pos] = j;
      }
    }
    csync();
    LPROF(4);  // scatter into bins
    // hist[b] is now the end of bin b; a bin holds the rows equal in their
    // top 24 bits (~1 for uniform keys). Each row takes its rank by (key,
    // row id) among its bin's rows and goes straight to its final position;
    // bins above 32 rows are sorted by a warp's bitonic network first.
    constexpr uint32_t kRankMax = 32;
    auto emit = [&](uint32_t p, uint64_t key, uint32_t v) {
      const uint64_t o = uint64_t(base) + p;
      const uint32_t j = v;  // CW > 0: the row's load index in the run
      if constexpr (PK) {  // packed row: row id in the low 32 bits
        v = uint32_t(key);
        key &= ~0xFFFFFFFFull;
      }
      uint64_t wd = 0;
      if constexpr (IDW) {
        wd = aw[j];
        v = uint32_t(wd);
      }
      if (a.out_keys) __stcs(reinterpret_cast<long long*>(a.out_keys) + o, (long long)xform(unpack_as<PACK>(key, pcode, pshl, constbits), desc));
      __stcs(a.out_vals + o, v);
      if constexpr (IDW) {  // the columns' bytes: the word's high half
        const uint32_t pw = uint32_t(wd >> 32);
        for (int c = 0; c < a.carry_n; ++c) {
          const int w = a.carry_width[c], off = a.carry_off[c];
          uint8_t* dst = a.carry_dst[c] + o * uint64_t(w);
          if (w == 4) __stcs(reinterpret_cast<unsigned int*>(dst), pw);
          else
            for (int b = 0; b < w; ++b) dst[b] = uint8_t(pw >> (8 * (off + b)));
        }
      } else if constexpr (CW > 0) {
        const uint8_t* row = reinterpret_cast<const uint8_t*>(pay + (size_t(base) + j) * CW);
        for (int c = 0; c < a.carry_n; ++c)
          copy_row(row + a.carry_off[c], a.carry_dst[c] + o * uint64_t(a.carry_width[c]), a.carry_width[c]);
      } else {
        gather_fused(a.gather, v, o);
      }
    };
    for (uint32_t p = tid; p < cnt; p += THREADS) {
      const uint64_t key = bk[p];
      const uint32_t v = IDW ? uint32_t(bv16[p]) : PK && CW == 0 ? 0u : bv[p];
      const int b = bin_of(key);
      const uint32_t b0 = b > 0 ? hist[b - 1] : 0u, b1 = hist[b];
      uint32_t pos = p;
      if (b1 - b0 > kRankMax) {
        if (p == b0) {
          const uint32_t slot = atomicAdd(&misc[0], 1u);
          if (slot < kBigList) big[slot] = uint32_t(b);
        }
        continue;
      }
      if (b1 - b0 > 1) {
        uint32_t rk = 0;
        if constexpr (PK) {
          for (uint32_t i = b0; i < b1; ++i) rk += bk[i] < key ? 1u : 0u;
        } else if constexpr (IDW) {  // the row ids only for equal keys
          for (uint32_t i = b0; i < b1; ++i) {
            const uint64_t ki = bk[i];
            rk += ki < key || (ki == key && uint32_t(aw[bv16[i]]) < uint32_t(aw[v])) ? 1u : 0u;
          }
        } else {
          for (uint32_t i = b0; i < b1; ++i) rk += row_less(bk[i], bv[i], key, v) ? 1u : 0u;
        }
        pos = b0 + rk;
      }
      emit(pos, key, v);
    }
    csync();
    LPROF(5);  // rank + emit
#ifdef RL_PASS_PROFILE
    if (BAL && CW == 0 && LEVELS == 2 && tid == 0) atomicAdd(&g_pass_prof[24], 1ull);
#endif
    const uint32_t nbig = min(misc[0], uint32_t(kBigList));
    for (uint32_t t = warp; t < nbig; t += kLWarps) {
      const int b = int(big[t]);
      const uint32_t b0 = b > 0 ? hist[b - 1] : 0u, b1 = hist[b];
      if constexpr (IDW) {
        warp_bitonic_idw(bk, bv16, aw, b0, b1, lane);
        for (uint32_t p = b0 + lane; p < b1; p += 32) emit(p, bk[p], uint32_t(bv16[p]));
      } else {
        warp_bitonic<PK, (CW > 0)>(bk, bv, b0, b1, lane);
        for (uint32_t p = b0 + lane; p < b1; p += 32) emit(p, bk[p], PK && CW == 0 ? 0u : bv[p]);
      }
    }
    if (nbig) csync();  // (the rank loop's reads of B/hist ended at the barrier before nbig)
    if constexpr (PROD) {  // this run's buffer is free for the producer
      if (tid == 0) mbar_arrive(&bars[2 + buf]);
      ++q;
      continue;
    }
    if (!more) break;
    k = next_k;
    r = next_r;
    buf ^= 1;
  }
  if (tid == 0) {
    mbar_inval(&bars[0]);
    mbar_inval(&bars[1]);
  }
}


// The whole sort after the histograms: plan, every active digit pass,
// copy-through — one cooperative launch. Hybrid (wide raw int64 keys):
// the two top-digit passes, the boundary scan, then the local phase — or,
// if a sub-bucket turned out larger than kLocalCap, the LSD passes from
// the original input (fresh epochs and tile counters), in the same launch.
__device__ void run_passes(const SortArgs& a, uint8_t* smem, const uint32_t* bin_off, const uint32_t* active,
                           uint32_t n_active, bool to_final, bool suboff, PassState& ps, uint32_t epoch_base,
                           uint32_t* tile_counter, uint32_t* grid_bar, uint32_t& barrier_no, uint32_t& src,
                           bool stamper) {
  uint32_t seen = 0;
  src = 0;
  for (int p = 0; p < kPasses; ++p) {
    if (!active[p]) continue;
    ++seen;
    const bool last = seen == n_active;
    const uint32_t dst = last && to_final ? 3u : (src == 1 ? 2u : 1u);
    const uint32_t ep = epoch_base + p + 1;
    switch (p) {
      case 0: run_pass<0>(a, smem, src, dst, bin_off, ps, ep, tile_counter); break;
      case 1: run_pass<1>(a, smem, src, dst, bin_off, ps, ep, tile_counter); break;
      case 2: run_pass<2>(a, smem, src, dst, bin_off, ps, ep, tile_counter); break;
      case 3: run_pass<3>(a, smem, src, dst, bin_off, ps, ep, tile_counter); break;
      case 4: run_pass<4>(a, smem, src, dst, bin_off, ps, ep, tile_counter); break;
      case 5: run_pass<5>(a, smem, src, dst, bin_off, ps, ep, tile_counter); break;
      case 6: run_pass<6>(a, smem, src, dst, bin_off, ps, ep, tile_counter); break;
      default:
        if (suboff) run_pass<7, true>(a, smem, src, dst, bin_off, ps, ep, tile_counter);
        else run_pass<7>(a, smem, src, dst, bin_off, ps, ep, tile_counter);
        break;
    }
    src = dst;
    if (!last || !to_final) grid_sync(grid_bar, ++barrier_no);  // the next phase reads what this one wrote
    if (stamper) a.stamps[2 + p] = globaltimer();
  }
}

// The scatter hybrid's local phase on its own launch (512 threads: twice the
// warps of the cooperative kernel's 256-thread CTAs for this latency-bound
// phase); the cooperative kernel behind it runs only on the fallback flag.
#ifndef RL_LOCAL_THREADS
#define RL_LOCAL_THREADS 512
#endif
constexpr int kLocalThreads = RL_LOCAL_THREADS;
__global__ void __launch_bounds__(kLocalThreads, 1024 / kLocalThreads) local_kernel(SortArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const bool stamper = a.stamps && blockIdx.x == 0 && threadIdx.x == 0;
  pdl_wait();  // the digit-6 pass
  pdl_launch_dependents();
  const bool scatter = a.mode == kModeScatter;
  if (stamper && scatter) a.stamps[1] = globaltimer();
  // scatter path: flags[0] = LSD fallback; onesweep hybrid: flags[7] = the
  // cooperative kernel took the hybrid and every sub-bucket fits (else it sorted
  // LSD). Both final before this launch: uniform.
  if (scatter ? local_fallback(a) : *reinterpret_cast<volatile const uint32_t*>(a.flags + 7) == 0) return;
  // the rows sit in their sub-buckets in keys_a / vals_a (scatter path: the
  // digit-6 pass) or keys_b / vals_b (onesweep hybrid: its digit-7 pass)
  const uint32_t src = scatter ? 1u : 2u;
  if (threadIdx.x == 0) {  // key pack code and constant bits, read by the local phase after its first barrier
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + kLocMisc);
    const uint32_t pc = __ldcg(a.flags + 6);
    const uint64_t cb = pack_mode(pc) ? key_constbits(a, pc) : 0ull;  // (a.col is null for encoded keys)
    misc[125] = pc;
    misc[126] = uint32_t(cb);
    misc[127] = uint32_t(cb >> 32);
  }
  if (!scatter) {
    local_phase<kLocalThreads, 0, false>(a, smem, src);  // (the onesweep hybrid packs no keys)
  } else {
    const uint32_t pc = __ldcg(a.flags + 6);
    const bool pk = packed_rows(pc, a);
    {
      switch (pack_mode(pc)) {
        case 0: local_phase<kLocalThreads, 0, true>(a, smem, src); break;
        case 1:
          if (pk) local_phase<kLocalThreads, 1, true, true>(a, smem, src);
          else local_phase<kLocalThreads, 1, true>(a, smem, src);
          break;
        default:
          if (pk) local_phase<kLocalThreads, 2, true, true>(a, smem, src);
          else local_phase<kLocalThreads, 2, true>(a, smem, src);
          break;
      }
    }
  }
  if (a.stamps && scatter && threadIdx.x == 0)  // (profiling: the last CTA's end, pass-6 slot unused here)
    atomicMax(reinterpret_cast<unsigned long long*>(a.stamps + 8), (unsigned long long)globaltimer());
  if (stamper) {
    a.stamps[kStamps - 2] = globaltimer();
    a.stamps[kStamps - 1] = scatter ? 3 : 1;
  }
}

// The scatter path's two-level local phase with a producer warp (kLocalThreads
// consumers + 32): the rows sit in their sub-buckets in keys_a / vals_a.
constexpr int kLocalWsThreads = kLocalThreads + 32;
__global__ void __launch_bounds__(kLocalWsThreads, 1024 / kLocalThreads) local_ws_kernel(SortArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const bool stamper = a.stamps && blockIdx.x == 0 && threadIdx.x == 0;
  pdl_wait();  // the digit-6 pass
  pdl_launch_dependents();
  if (stamper) a.stamps[1] = globaltimer();
  if (local_fallback(a)) return;  // (final before this launch: uniform)
  const uint32_t pc = __ldcg(a.flags + 6);
  if (threadIdx.x == 0) {  // key pack code and constant bits, read by the local phase after its first barrier
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + kLocMisc);
    const uint64_t cb = pack_mode(pc) ? key_constbits(a, pc) : 0ull;
    misc[125] = pc;
    misc[126] = uint32_t(cb);
    misc[127] = uint32_t(cb >> 32);
  }
  const bool pk = packed_rows(pc, a);
  switch (pack_mode(pc)) {
    case 0: local_phase<kLocalThreads, 0, true, false, 2, 0, true>(a, smem, 1u); break;
    case 1:
      if (pk) local_phase<kLocalThreads, 1, true, true, 2, 0, true>(a, smem, 1u);
      else local_phase<kLocalThreads, 1, true, false, 2, 0, true>(a, smem, 1u);
      break;
    default:
      if (pk) local_phase<kLocalThreads, 2, true, true, 2, 0, true>(a, smem, 1u);
      else local_phase<kLocalThreads, 2, true, false, 2, 0, true>(a, smem, 1u);
      break;
  }
  if (a.stamps && threadIdx.x == 0)  // (profiling: the last CTA's end, pass-6 slot unused here)
    atomicMax(reinterpret_cast<unsigned long long*>(a.stamps + 8), (unsigned long long)globaltimer());
  if (stamper) {
    a.stamps[kStamps - 2] = globaltimer();
    a.stamps[kStamps - 1] = 3;
  }
}

// The three-level local phase on its own kernel (the two-level kernel's code
// stays as tuned): runs of (d7, d6, d5) sub-sub-buckets out of keys_b.
__global__ void __launch_bounds__(kLocalWsThreads, 1024 / kLocalThreads) local3_kernel(SortArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_wait();  // the digit-5 pass
  pdl_launch_dependents();
  if (local_fallback(a)) return;  // LSD fallback (final before this launch)
  const uint32_t pc = __ldcg(a.flags + 6);
  if (threadIdx.x == 0) {
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + kLocMisc);
    const uint64_t cb = pack_mode(pc) ? key_constbits(a, pc) : 0ull;
    misc[125] = pc;
    misc[126] = uint32_t(cb);
    misc[127] = uint32_t(cb >> 32);
  }
  const bool pk = packed_rows(pc, a);
  switch (pack_mode(pc)) {
    case 0: local_phase<kLocalThreads, 0, true, false, 3, 0, true>(a, smem, 2u); break;
    case 1:
      if (pk) local_phase<kLocalThreads, 1, true, true, 3, 0, true>(a, smem, 2u);
      else local_phase<kLocalThreads, 1, true, false, 3, 0, true>(a, smem, 2u);
      break;
    default:
      if (pk) local_phase<kLocalThreads, 2, true, true, 3, 0, true>(a, smem, 2u);
      else local_phase<kLocalThreads, 2, true, false, 3, 0, true>(a, smem, 2u);
      break;
  }
}

// The local phase of a sort with carried columns (packed rows; the columns'
// bytes ride beside every row through the counting passes and are copied out
// of the run's payload window): its own kernel, so the plain sort's local
// kernels keep their code.
template <int LEVELS>
__global__ void __launch_bounds__(kLocalWsThreads, 1024 / kLocalThreads) local_carry_kernel(SortArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_wait();
  pdl_launch_dependents();
  if (local_fallback(a)) return;  // LSD fallback (final before this launch)
  const uint32_t pc = __ldcg(a.flags + 6);
  if (threadIdx.x == 0) {
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + kLocMisc);
    const uint64_t cb = pack_mode(pc) ? key_constbits(a, pc) : 0ull;
    misc[125] = pc;
    misc[126] = uint32_t(cb);
    misc[127] = uint32_t(cb >> 32);
  }
  constexpr uint32_t src = LEVELS == 3 ? 2u : 1u;
  if (!packed_rows(pc, a)) {  // idw (the counting passes declined anything else)
    switch (pack_mode(pc)) {
      case 0: local_phase<kLocalThreads, 0, true, false, LEVELS, 1, true>(a, smem, src); break;
      case 1: local_phase<kLocalThreads, 1, true, false, LEVELS, 1, true>(a, smem, src); break;
      default: local_phase<kLocalThreads, 2, true, false, LEVELS, 1, true>(a, smem, src); break;
    }
    return;
  }
  const bool m1 = pack_mode(pc) == 1;  // (packed rows: mode 1 or 2, checked by the counting passes)
  if (a.cw == 1) {
    if (m1) local_phase<kLocalThreads, 1, true, true, LEVELS, 1, true>(a, smem, src);
    else local_phase<kLocalThreads, 2, true, true, LEVELS, 1, true>(a, smem, src);
  } else {
    if (m1) local_phase<kLocalThreads, 1, true, true, LEVELS, 2, true>(a, smem, src);
    else local_phase<kLocalThreads, 2, true, true, LEVELS, 2, true>(a, smem, src);
  }
}

__global__ void __launch_bounds__(kThreads, RL_ONESWEEP_MIN_BLOCKS) sort_kernel(SortArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* bin_off = reinterpret_cast<uint32_t*>(smem + kPassSmemBytes);  // [kPasses][kBins], whole kernel
  uint32_t* plan = bin_off + kPasses * kBins;  // [0..7] active, [8] n_active, [9] hybrid, [10..17] hybrid passes, [18] their count, [19] low digits to count
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOffset);
  const int tid = threadIdx.x;
  uint32_t barrier_no = 0;
  const bool stamper = a.stamps && blockIdx.x == 0 && tid == 0;

  // ---- scatter hybrid: local_kernel sorted the sub-buckets already; this
  // launch only runs the LSD fallback
  pdl_wait();  // launched as a programmatic dependent of the histogram / local-phase kernel
  if (stamper && a.mode == kModeScatter) a.stamps[9] = globaltimer();  // (profiling: pass-7 slot unused here)
  if (a.mode == kModeScatter && *reinterpret_cast<volatile const uint32_t*>(a.flags) == 0) return;
  // ---- histograms come from hist_kernel (launched just before, on the same stream)
  if (stamper) a.stamps[1] = globaltimer();
  if (a.mode == kModeScatter) {  // LSD fallback: the look-back words were left out of the zeroed prefix
    const size_t words = size_t((a.n + kTile - 1) / kTile) * kBins;
    for (size_t i = size_t(blockIdx.x) * kThreads + tid; i < words; i += size_t(gridDim.x) * kThreads) a.status[i] = 0;
    grid_sync(a.grid_bar, ++barrier_no);
  }

  // ---- plan (every CTA for itself): global digit bases + active digits.
  // Raw int64 keys: the histogram kernel counted digits 6 and 7 and ORed
  // the varying bits; the other digits are counted here only on the LSD
  // path, and only if they vary.
  const bool raw = a.src_mode == kSrcInt64;
  auto scan_rows = [&](int p0, int p1) {  // bin_off rows [p0, p1) from the global histograms
    uint32_t* warp_sums = reinterpret_cast<uint32_t*>(smem);  // scratch
    for (int p = p0; p < p1; ++p) {
      const uint32_t c = ghist_at(a, p, tid);
      uint32_t total;
      bin_off[p * kBins + tid] = block_exclusive_scan<kThreads>(c, warp_sums, &total);
      __syncthreads();
    }
  };
  {
    uint32_t* warp_sums = reinterpret_cast<uint32_t*>(smem);  // scratch
    const uint64_t vary = raw ? __ldcg(reinterpret_cast<const unsigned long long*>(a.flags + 4)) : 0ull;
    uint32_t nz = 1, mx = 1;
    for (int p = raw && !a.count_all ? 6 : 0; p < kPasses; ++p) {
      const uint32_t c = ghist_at(a, p, tid);
      uint32_t total;
      bin_off[p * kBins + tid] = block_exclusive_scan<kThreads>(c, warp_sums, &total);
      const int full = __syncthreads_or(uint64_t(c) == uint64_t(a.n));
      if (p >= 6) {  // spread of the top two digits (the hybrid's pre-check)
        nz *= uint32_t(__syncthreads_count(c != 0));
        uint32_t m = c;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((tid & 31) == 0) warp_sums[16 + (tid >> 5)] = m;
        __syncthreads();
        m = 0;
        for (int w = 0; w < kWarps; ++w) m = max(m, warp_sums[16 + w]);
        const uint64_t est = uint64_t(mx) * m / uint64_t(a.n) + 1;  // largest sub-bucket if d6, d7 independent
        mx = p == 6 ? m : uint32_t(est > 0xFFFFFFFFull ? 0xFFFFFFFFull : est);
        __syncthreads();
      }
      if (tid == 0 && !raw) plan[p] = full ? 0u : 1u;
    }
    if (tid == 0) {
      if (raw)
        for (int p = 0; p < kPasses; ++p) plan[p] = ((vary >> (p * kBits)) & (kBins - 1)) ? 1u : 0u;
      uint32_t na = 0;
      for (int p = 0; p < kPasses; ++p) na += plan[p];
      plan[kPasses] = na;
      // hybrid: wide raw keys whose top two digits spread the rows into
      // sub-buckets that fit on chip (pigeonhole + independent-digit estimate)
      // and at least two passes to save
      const bool hyb = a.mode == kModeHybrid && na >= 4 && (plan[6] | plan[7]) &&
                       uint64_t(a.n) <= uint64_t(nz) * kLocalCap && mx <= uint32_t(kLocalCap) * 4 / 5;
      plan[kPasses + 1] = hyb ? 1u : 0u;
      for (int p = 0; p < kPasses; ++p) plan[kPasses + 2 + p] = p >= 6 ? plan[p] : 0u;
      plan[2 * kPasses + 2] = plan[6] + plan[7];
      uint32_t low = 0;
      for (int p = 0; p < 6; ++p) low |= plan[p] << p;
      // scatter fallback: the scatter path builds no digit-6/7 histograms, the LSD counts them
      if (a.mode == kModeScatter) low |= (plan[6] << 6) | (plan[7] << 7);
      plan[2 * kPasses + 3] = raw && !a.count_all ? low : 0u;  // digits the LSD path still has to count
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
    }
    __syncthreads();
  }
  // raw keys going LSD: count the varying low digits now (every CTA), then their bases
  auto count_low_digits = [&]() {
    const uint32_t low = plan[2 * kPasses + 3];
    if (!low) return;
    count_digits(a, smem, low);  // (digit-6/7 rows are still zero on a scatter fallback)
    grid_sync(a.grid_bar, ++barrier_no);
    scan_rows(0, (low >> 6) ? kPasses : 6);
  };
  if (!plan[kPasses + 1]) count_low_digits();

  PassState ps{0, 0};
  uint32_t src = 0;
  if (plan[kPasses + 1]) {
    // ---- hybrid: the two top-digit passes (stable by the top 16 bits); the
    // digit-7 pass also writes the sub-bucket starts. With digit 7 constant
    // (c7) the starts are digit 6's bases on row c7.
    if (!plan[7]) {
      uint32_t c7 = 0;
      for (int d = 0; d < kBins; ++d)
        if (bin_off[7 * kBins + d] == 0 && (d == kBins - 1 || bin_off[7 * kBins + d + 1] == uint32_t(a.n))) c7 = d;
      for (uint32_t b = blockIdx.x * kThreads + tid; b <= uint32_t(kSubBuckets); b += gridDim.x * kThreads) {
        const uint32_t d7 = b >> kBits;
        a.sub_off[b] = b == uint32_t(kSubBuckets) || d7 > c7 ? uint32_t(a.n) : d7 < c7 ? 0u : bin_off[6 * kBins + (b & 255u)];
      }
    }
    run_passes(a, smem, bin_off, plan + kPasses + 2, plan[2 * kPasses + 2], false, true, ps, 0u, a.tile_counter,
               a.grid_bar, barrier_no, src, stamper);
    {  // sub-buckets larger than the on-chip cap? (each CTA checks a slice)
      int over = 0;
      for (uint32_t b = blockIdx.x * kThreads + tid; b < uint32_t(kSubBuckets); b += gridDim.x * kThreads)
        over |= __ldcg(a.sub_off + b + 1) - __ldcg(a.sub_off + b) > uint32_t(kLocalCap);
      if (__syncthreads_or(over) && tid == 0) atomicExch(a.flags, 1u);
    }
    grid_sync(a.grid_bar, ++barrier_no);
    if (stamper) a.stamps[2] = globaltimer();  // (pass 0's slot: the hybrid's sub-bucket check)
    // every sub-bucket fits on chip: local_kernel (launched next) sorts them
    if (*reinterpret_cast<volatile uint32_t*>(a.flags) == 0) {
      if (blockIdx.x == 0 && tid == 0) a.flags[7] = 1u;  // the go signal (an LSD sort leaves it 0)
      return;
    }
    // a sub-bucket does not fit on chip: the LSD sort, fresh epochs and counters
    if (stamper)
      for (int p = 0; p < kPasses; ++p) a.stamps[2 + p] = 0;
    count_low_digits();
  }

  // ---- LSD: the active digit passes, least significant first
  const bool fb = plan[kPasses + 1] != 0;
  run_passes(a, smem, bin_off, plan, plan[kPasses], true, false, ps, fb ? kHybridEpoch : 0u,
             a.tile_counter + (fb ? kPasses : 0), a.grid_bar, barrier_no, src, stamper);

  // ---- no active digit (all keys equal, or n == 1): copy through
  if (plan[kPasses] == 0) {
    for (int64_t i = int64_t(blockIdx.x) * kThreads + tid; i < a.n; i += int64_t(gridDim.x) * kThreads) {
      const uint32_t row = a.perm_in ? a.perm_in[i] : uint32_t(i);
      a.out_vals[i] = row;
      if (a.out_keys) a.out_keys[i] = static_cast<const int64_t*>(a.col)[i];
      gather_fused(a.gather, row, uint64_t(i));
    }
  }
  if (stamper) {
    a.stamps[kStamps - 2] = globaltimer();
    a.stamps[kStamps - 1] = a.mode == kModeScatter ? 4 : plan[kPasses + 1] ? 2 : 0;
  }
}

// RL_SCATTER_MIN_ROWS overrides kScatterMinRows (tests: every hybrid shape through both paths)
static int64_t scatter_min_rows() {
  const char* v = getenv("RL_SCATTER_MIN_ROWS");
  const long long r = v && v[0] ? atoll(v) : 0;
  return r > 0 ? std::max<int64_t>(r, kHybridMinRows) : kScatterMinRows;
}

struct Layout {
  uint32_t* hist;
  uint32_t* tile_counter;
  uint32_t* grid_bar;
  uint32_t* flags;
  uint64_t* status;
  size_t zero_bytes;  // prefix [hist .. status] zeroed per call
  size_t head_bytes;  // prefix [hist .. cur16]: the scatter path zeroes only this (its LSD fallback clears status)
  uint32_t* sub_off;
  uint64_t* keys_a;
  uint64_t* keys_b;
  uint32_t* vals_a;
  uint32_t* vals_b;
  uint32_t* chunk_cnt;  // scatter hybrid only (n >= scatter_min_rows())
  uint32_t* cur7;
  uint32_t* cur16;
  uint32_t* d7rep;
  uint32_t* d7_base;
  uint32_t* items;
  uint32_t* meta;
  uint32_t* sub3_off;  // three-level scatter only (n >= kLevel3MinRows)
  uint32_t* cur24;
  uint32_t* tile3;
  uint32_t* tmap;
};

// Above this the (d7, d6) sub-buckets of uniform keys come close to kLocalCap:
// the scatter path splits them by digit 5 as well (three levels).
// Measured (uniform keys): 2e8 rows 8.5 ms vs 7.4 ms for the LSD passes (small
// sub-sub-buckets make short local runs), 1e9 rows 30.3 vs 36.5 ms: the third
// level starts at 3e8 rows; between ~65536 x kLocalCap x 0.85 and that, LSD.
constexpr int64_t kLevel3MinRows = 300000000;
// above this the two-level sub-buckets of uniform keys overflow kLocalCap (pigeonhole + spread): LSD instead
constexpr int64_t kTwoLevelMaxRows = int64_t(kSubBuckets) * kLocalCap * 85 / 100;

// RL_LEVEL3_MIN_ROWS overrides kLevel3MinRows (tests: the third level at small n)
static int64_t level3_min_rows() {
  const char* v = getenv("RL_LEVEL3_MIN_ROWS");
  const long long r = v && v[0] ? atoll(v) : 0;
  return r > 0 ? r : kLevel3MinRows;
}

template <typename C, typename T32, typename T64>
static void carve_all(C& c, int64_t n, T32 t32, T64 t64, Layout* L, bool force_scatter = false,
                      int force_levels = 0) {
  const size_t tiles = size_t((n + kTile - 1) / kTile);
  auto h = t32(c, size_t(kHistReps) * kPasses * kBins);
  auto tc = t32(c, 2 * kPasses);
  auto gb = t32(c, 2);
  auto fl = t32(c, 8);
  const bool scat = force_scatter || n >= scatter_min_rows();
  auto c7 = scat ? t32(c, size_t(kBins)) : nullptr;          // zeroed with the prefix
  auto c16 = scat ? t32(c, size_t(kSubBuckets)) : nullptr;
  auto d7r = scat ? t32(c, size_t(kD7Reps) * kBins) : nullptr;
  const size_t head = c.used;
  auto st = t64(c, tiles * kBins);
  const size_t zero = c.used;
  auto so = t32(c, kSubBuckets + 1);
  auto ka = t64(c, size_t(n));
  auto kb = t64(c, size_t(n));
  auto va = t32(c, size_t(n));
  auto vb = t32(c, size_t(n));
  auto cc = scat ? t32(c, size_t(kMaxChunks) * kScatWords) : nullptr;
  auto db = scat ? t32(c, size_t(kBins + 4)) : nullptr;
  auto it = scat ? t32(c, 4 * size_t(kBins + 2 + n / kPTile)) : nullptr;
  auto me = scat ? t32(c, 4) : nullptr;
  const bool lvl3 = scat && (force_levels ? force_levels == 3 : n >= level3_min_rows());
  auto s3 = lvl3 ? t32(c, size_t(kSub3) + 1) : nullptr;
  auto c24 = lvl3 ? t32(c, size_t(kSub3)) : nullptr;
  auto t3 = lvl3 ? t32(c, size_t(kSubBuckets) + 1) : nullptr;
  auto tm = lvl3 ? t32(c, 4 * (size_t(kSubBuckets) + size_t(n / kPTile) + 1)) : nullptr;  // <= one partial tile a sub-bucket
  if (L) *L = Layout{h, tc, gb, fl, st, zero, head, so, ka, kb, va, vb, cc, c7, c16, d7r, db, it, me, s3, c24, t3, tm};
}

size_t workspace_bytes(int64_t n) {
  if (n <= 0) return 256;
  CarveSize c;
  carve_all(c, n, [](CarveSize& c, size_t k) { c.take<uint32_t>(k); return (uint32_t*)nullptr; },
            [](CarveSize& c, size_t k) { c.take<uint64_t>(k); return (uint64_t*)nullptr; }, nullptr);
  return c.used + 256;
}

static bool carve_layout(Layout& L, void* ws, size_t ws_bytes, int64_t n) {
  Carve c{static_cast<char*>(ws), ws_bytes};
  carve_all(c, n, [](Carve& c, size_t k) { return c.take<uint32_t>(k); },
            [](Carve& c, size_t k) { return c.take<uint64_t>(k); }, &L);
  return c.ok;
}

__global__ void identity_kernel(const uint32_t* perm_in, int64_t n, uint32_t* out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = perm_in ? perm_in[i] : uint32_t(i);
}

// RL_NO_HYBRID=1 forces the LSD path, RL_NO_SCATTER=1 the onesweep-pass hybrid
// (A/B measurements and tests).
static bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && v[0] && v[0] != '0';
}
static bool getenv_flag_no_hybrid() { return getenv_flag("RL_NO_HYBRID"); }

constexpr size_t kHistSmem = size_t(kScatWords) * 4 + size_t(kScatThreads) * 4;

static bool scatter_kernels_ready() {
  static int ready[kMaxDevices] = {};  // per device: 1 = every opt-in took, -1 = refused
  return per_device(ready, [] {
           const bool ok =
               cudaFuncSetAttribute(sub_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kHistSmem)) ==
                   cudaSuccess &&
               cudaFuncSetAttribute(top_scatter_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPSmem)) ==
                   cudaSuccess &&
               cudaFuncSetAttribute(sub_scatter_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPSmem)) ==
                   cudaSuccess &&
               cudaFuncSetAttribute(local_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kLocalSmemBytes)) == cudaSuccess &&
               cudaFuncSetAttribute(local3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kLocalKernelSmem)) == cudaSuccess &&
               cudaFuncSetAttribute(local_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kLocalSmemBytes)) == cudaSuccess &&
               cudaFuncSetAttribute(local_carry_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kLocalSmemBytes)) == cudaSuccess &&
               cudaFuncSetAttribute(local_carry_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kLocalKernelSmem)) == cudaSuccess &&
               cudaFuncSetAttribute(sub3_scatter_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPSmem)) ==
                   cudaSuccess;
           if (!ok) cudaGetLastError();
#ifdef RL_CARVEOUT_MAX
           if (ok) {  // one L1/shared split for every kernel of the sort: no SM reconfiguration between them
             cudaFuncSetAttribute(sub_hist_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
             cudaFuncSetAttribute(top_scatter_kernel<0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
             cudaFuncSetAttribute(sub_scatter_kernel<0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
             cudaFuncSetAttribute(local_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
             cudaFuncSetAttribute(sort_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
           }
#endif
           return ok ? 1 : -1;
         }) > 0;
}

// The counting-pass instances that carry CW payload words: their shared
// memory opt-in, once per device.
template <int CW>
static bool carry_kernels_ready() {
  static int ready[kMaxDevices] = {};
  return per_device(ready, [] {
           const bool ok = cudaFuncSetAttribute(top_scatter_kernel<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                int(psmem_bytes(CW))) == cudaSuccess &&
                           cudaFuncSetAttribute(sub_scatter_kernel<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                int(psmem_bytes(CW))) == cudaSuccess &&
                           cudaFuncSetAttribute(sub3_scatter_kernel<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                int(psmem_bytes(CW))) == cudaSuccess;
           if (!ok) cudaGetLastError();
           return ok ? 1 : -1;
         }) > 0;
}

// Co-resident CTAs per SM of the counting passes (both have the same shape).
static int pass_ctas_per_sm() {
  static int cache[kMaxDevices] = {};
  return per_device(cache, [] {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, top_scatter_kernel<0>, kPThreads, kPSmem) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    return per_sm;
  });
}

// Largest co-resident grid of the cooperative sort kernel on this device
// (-1: the shared-memory opt-in or the occupancy query failed).
static int sort_grid_limit() {
  static int cache[kMaxDevices] = {};
  return per_device(cache, [] {
    if (cudaFuncSetAttribute(sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes)) !=
        cudaSuccess)
      return -1;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sort_kernel, kThreads, kSmemBytes) != cudaSuccess ||
        per_sm < 1)
      return -1;
    return per_sm * device_sm_count();
  });
}

#ifndef RL_HIST_CTAS_PER_SM
#define RL_HIST_CTAS_PER_SM 2
#endif
static int hist_grid(int64_t n) {  // one co-resident wave (2 CTAs of 512 threads per SM), >= 1 step each
  const int64_t per_cta = int64_t(kHistThreads) * kHistUnroll;
  return int(std::max<int64_t>(1, std::min<int64_t>((n + per_cta - 1) / per_cta,
                                                    int64_t(device_sm_count()) * RL_HIST_CTAS_PER_SM)));
}

// The cooperative sort kernel as a programmatic dependent of the kernel before
// it (scheduled while that one drains; it waits on the device), or a plain
// cooperative launch where the runtime refuses the combination.
static cudaError_t launch_sort_kernel(SortArgs& a, int grid, cudaStream_t stream, bool pdl) {
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, sort_kernel, a);
  if (e == cudaErrorNotSupported || e == cudaErrorInvalidValue) {
    cudaGetLastError();
    void* params[] = {&a};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(sort_kernel), dim3(grid), dim3(kThreads), params,
                                    kSmemBytes, stream);
  }
  return e;
}

// Histograms, then the cooperative kernel (LSD, or the wide-key hybrid
// with its in-kernel LSD fallback).
static int launch_sort(SortArgs a, const Layout& L, cudaStream_t stream, void* const* events, int max_ctas = 0) {
  int limit = sort_grid_limit();
  if (max_ctas > 0 && limit > max_ctas) limit = max_ctas;  // leave room for a concurrent sort
  // programmatic dependent launches between this sort's kernels — not when a
  // concurrent sort shares the device (early-scheduled dependents of one sort
  // hold SMs the other's kernels need: the join plan's two index sorts went
  // 0.75 -> 1.14 ms with them)
  const bool pdl = max_ctas <= 0 && !getenv_flag("RL_NO_PDL");
  if (limit < 1) {
    cudaError_t e = cudaGetLastError();
    return rl_cuda_status(e != cudaSuccess ? e : cudaErrorInvalidConfiguration);
  }
  const bool scatter = a.src_mode == kSrcInt64 && a.n >= kHybridMinRows && !getenv_flag_no_hybrid() && L.chunk_cnt &&
                       (a.n <= kTwoLevelMaxRows || L.sub3_off) && !getenv_flag("RL_NO_SCATTER") &&
                       scatter_kernels_ready();
  cudaError_t e = cudaMemsetAsync(L.hist, 0, scatter ? L.head_bytes : L.zero_bytes, stream);
  if (e != cudaSuccess) return rl_cuda_status(e);
  // enough CTAs for the tiles, at most all co-resident
  const int64_t tiles = (a.n + kTile - 1) / kTile;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(limit, tiles)));
  a.mode = a.src_mode == kSrcInt64 && a.n >= kHybridMinRows && !getenv_flag_no_hybrid() ? kModeHybrid : kModeLsd;
  // (pigeonhole: above 65536 * kLocalCap rows some sub-bucket overflows for sure)
  if (scatter) {
    // scatter hybrid: chunk counts, digit-7 pass, digit-6 pass, then the local phase
    a.mode = kModeScatter;
    a.count_all = 0;
    a.chunk_cnt = L.chunk_cnt;
    a.cur7 = L.cur7;
    a.cur16 = L.cur16;
    a.d7rep = L.d7rep;
    a.d7_base = L.d7_base;
    a.items = reinterpret_cast<uint4*>(L.items);
    a.meta = L.meta;
    int chunks = int(std::min<int64_t>(std::min(device_sm_count(), kMaxChunks),
                                       std::max<int64_t>(32, (a.n + kChunkMinRows - 1) / kChunkMinRows)));
    if (const char* e = getenv("RL_SCATTER_CHUNKS")) chunks = std::max(1, std::min(atoi(e), kMaxChunks));
    int pgrid = device_sm_count() * pass_ctas_per_sm();
    if (max_ctas > 0) {  // a concurrent sort shares the device: scale with the sort's cap (2 CTAs per SM)
      chunks = std::max(1, std::min(chunks, max_ctas / 2));
      pgrid = std::max(1, std::min(pgrid, max_ctas / 2 * pass_ctas_per_sm()));
    }
    a.chunks = chunks;
    a.allow_pk = getenv_flag("RL_NO_PACKED_ROWS") ? 0 : 1;
    a.levels = L.sub3_off ? 3 : 2;
    a.sub3_off = L.sub3_off;
    a.cur24 = L.cur24;
    a.tile3 = L.tile3;
    a.tmap = L.tmap;
    if (a.levels == 3 && (e = cudaMemsetAsync(L.cur24, 0, sizeof(uint32_t) * size_t(kSub3), stream)) != cudaSuccess)
      return rl_cuda_status(e);
    int lgrid = device_sm_count() * (1024 / kLocalThreads);
    if (max_ctas > 0) lgrid = std::max(1, std::min(lgrid, max_ctas));
    if (events) cudaEventRecord(static_cast<cudaEvent_t>(events[0]), stream);
    const bool dbg = getenv_flag("RL_SCATTER_DEBUG");
    auto chk = [&](const char* what) {
      if (!dbg) return;
      cudaError_t x = cudaStreamSynchronize(stream);
      uint32_t fl[8] = {0};
      cudaMemcpy(fl, L.flags, sizeof(fl), cudaMemcpyDeviceToHost);
      fprintf(stderr, "[scatter-debug] %s: %s flags=%u,%u,%u,%u\n", what, cudaGetErrorString(x), fl[0], fl[1], fl[2], fl[3]);
    };
    // the launches after the key sample may be scheduled early (programmatic
    // dependent launch); each waits on the device for its predecessor's results
    auto launch_dep = [&](auto kernel, int g, int threads, size_t smem) {
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(g);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = stream;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, kernel, a);
    };
    sub_hist_kernel<<<chunks, kScatThreads, kHistSmem, stream>>>(a);
    chk("sub_hist");
    int launched = 5;
    // the counting passes (with a sort's carried columns: the CW-word instances)
    auto passes = [&](auto cwc) -> cudaError_t {
      constexpr int CW = decltype(cwc)::value;
      const size_t sm = psmem_bytes(CW);
      cudaError_t x;
      if ((x = launch_dep(top_scatter_kernel<CW>, pgrid, kPThreads, sm)) != cudaSuccess) return x;
      chk("top_scatter");
      if ((x = launch_dep(sub_scatter_kernel<CW>, pgrid, kPThreads, sm)) != cudaSuccess) return x;
      chk("sub_scatter");
      if (a.levels == 3) {  // digit 5 inside every sub-bucket
        if ((x = launch_dep(count3_kernel, pgrid, kPThreads, size_t(0))) != cudaSuccess) return x;
        if ((x = launch_dep(tile_scan_kernel, 1, 1024, size_t(0))) != cudaSuccess) return x;
        if ((x = launch_dep(sub3_scatter_kernel<CW>, pgrid, kPThreads, sm)) != cudaSuccess) return x;
        chk("level 3");
        launched += 3;
      }
      return cudaSuccess;
    };
    if ((a.cw == 1 && !carry_kernels_ready<1>()) || (a.cw == 2 && !carry_kernels_ready<2>()))
      return rl_cuda_status(cudaErrorInvalidConfiguration);
    if (a.cw == 1) e = passes(std::integral_constant<int, 1>{});
    else if (a.cw == 2) e = passes(std::integral_constant<int, 2>{});
    else e = passes(std::integral_constant<int, 0>{});
    if (e != cudaSuccess) return rl_cuda_status(e);
    if (a.cw > 0 && a.levels == 3) e = launch_dep(local_carry_kernel<3>, lgrid, kLocalWsThreads, kLocalKernelSmem);
    else if (a.cw > 0) e = launch_dep(local_carry_kernel<2>, lgrid, kLocalWsThreads, kLocalSmemBytes);
    else if (a.levels == 3) e = launch_dep(local3_kernel, lgrid, kLocalWsThreads, kLocalKernelSmem);
    else e = launch_dep(local_ws_kernel, lgrid, kLocalWsThreads, kLocalSmemBytes);
    if (e != cudaSuccess) return rl_cuda_status(e);
    chk("local");
    if (events) cudaEventRecord(static_cast<cudaEvent_t>(events[1]), stream);
    e = launch_sort_kernel(a, grid, stream, pdl);  // returns at once unless the fallback flag is set
    if (events) cudaEventRecord(static_cast<cudaEvent_t>(events[2]), stream);
    count_launches(launched);
    return rl_cuda_status(e != cudaSuccess ? e : cudaGetLastError());
  }
  if (events) cudaEventRecord(static_cast<cudaEvent_t>(events[0]), stream);
  // small raw inputs (never worth the hybrid's skipped histograms): every digit in the histogram kernel
  a.count_all = a.src_mode == kSrcInt64 && a.n < kCountAllRows ? 1 : 0;
  if (a.src_mode == kSrcInt64 && a.count_all) hist_kernel<true, true><<<hist_grid(a.n), kHistThreads, 0, stream>>>(a);
  else if (a.src_mode == kSrcInt64) hist_kernel<true, false><<<hist_grid(a.n), kHistThreads, 0, stream>>>(a);
  else hist_kernel<false><<<hist_grid(a.n), kHistThreads, 0, stream>>>(a);
  if (events) cudaEventRecord(static_cast<cudaEvent_t>(events[1]), stream);
  e = launch_sort_kernel(a, grid, stream, pdl);
  int launched = 2;
  if (e == cudaSuccess && a.mode == kModeHybrid) {  // the local phase (returns at once after an LSD fallback)
    if (!scatter_kernels_ready()) return rl_cuda_status(cudaErrorInvalidConfiguration);
    int lgrid = device_sm_count() * (1024 / kLocalThreads);
    if (max_ctas > 0) lgrid = std::max(1, std::min(lgrid, max_ctas));
    local_kernel<<<lgrid, kLocalThreads, kLocalSmemBytes, stream>>>(a);
    e = cudaGetLastError();
    launched = 3;
  }
  if (events) cudaEventRecord(static_cast<cudaEvent_t>(events[2]), stream);
  count_launches(launched);
  return rl_cuda_status(e != cudaSuccess ? e : cudaGetLastError());
}

int sort_axis_capped(const void* col, int col_kind, int width, int word, int descending, const uint32_t* perm_in,
                     int64_t n, int64_t* sorted_keys_out, uint32_t* perm_out, void* ws, size_t ws_bytes,
                     cudaStream_t stream, void* const* events, unsigned long long* stamps, const rl_column* columns,
                     int n_columns, int max_ctas) {
  if (n_columns < 0 || n_columns > kMaxFusedColumns || (n_columns > 0 && columns == nullptr)) return RL_ERR_BAD_ARG;
  for (int i = 0; i < n_columns; ++i)
    if (columns[i].width < 0 || columns[i].side != RL_SIDE_LEFT ||
        (columns[i].width > 0 && (!columns[i].src || !columns[i].dst)))
      return RL_ERR_BAD_ARG;
  const bool zero_width = col_kind == RL_COL_BYTES && width == 0;  // no key bytes: col may be NULL
  if (n < 0 || (n > 0 && perm_out == nullptr) || (n > 0 && col == nullptr && !zero_width)) return RL_ERR_BAD_ARG;
  if (n > RL_MAX_ROWS) return RL_ERR_TOO_MANY_ROWS;
  if (col_kind == RL_COL_INT64) {
    if (width != 8 || word != 0) return RL_ERR_BAD_ARG;
  } else if (col_kind == RL_COL_BYTES) {
    if (width < 0 || word < 0 || (width > 0 && word >= (width + 7) / 8)) return RL_ERR_BAD_ARG;
    if (sorted_keys_out) return RL_ERR_BAD_ARG;
  } else {
    return RL_ERR_BAD_ARG;
  }
  if (sorted_keys_out && perm_in) return RL_ERR_BAD_ARG;
  // the digit passes stream int64 keys / row ids with 16-byte TMA bulk copies
  if (col_kind == RL_COL_INT64 && !perm_in && (reinterpret_cast<uintptr_t>(col) & 15)) return RL_ERR_BAD_ARG;
  if (reinterpret_cast<uintptr_t>(perm_in) & 15) return RL_ERR_BAD_ARG;
  if (n == 0) return RL_OK;
  if (zero_width && n_columns == 0) {  // tensorpath.py:218-219: identity order
    int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(device_sm_count()) * 8));
    identity_kernel<<<grid, 256, 0, stream>>>(perm_in, n, perm_out);
    count_launches(1);
    return rl_cuda_status(cudaGetLastError());
  }
  if (zero_width) return RL_ERR_BAD_ARG;  // fused gathers need a real key word
  if (reinterpret_cast<uintptr_t>(ws) % 256 != 0) return RL_ERR_WORKSPACE;
  Layout L;
  if (!carve_layout(L, ws, ws_bytes, n)) return RL_ERR_WORKSPACE;

  SortArgs a = {};
  a.col = col;
  a.perm_in = perm_in;
  a.n = n;
  a.width = width;
  a.word = word;
  a.desc = descending ? 1 : 0;
  a.keys_a = L.keys_a;
  a.keys_b = L.keys_b;
  a.vals_a = L.vals_a;
  a.vals_b = L.vals_b;
  a.out_vals = perm_out;
  a.ghist = L.hist;
  a.tile_counter = L.tile_counter;
  a.grid_bar = L.grid_bar;
  a.flags = L.flags;
  a.sub_off = L.sub_off;
  a.status = L.status;
  a.stamps = stamps;
  a.gather.n = n_columns;
  for (int i = 0; i < n_columns; ++i) a.gather.c[i] = columns[i];
  if (col_kind == RL_COL_INT64 && perm_in == nullptr) {
    a.src_mode = kSrcInt64;
    a.materialized = nullptr;
    a.key_mode = descending ? kRawDesc : kRawAsc;
    a.orig_keys = col;
    a.out_keys = sorted_keys_out;
  } else {
    a.src_mode = col_kind == RL_COL_INT64 ? kSrcInt64Gather : kSrcBytes;
    a.materialized = L.keys_b;  // read once by the first active pass, then reused as ping-pong B
    a.key_mode = kMaterialized;
    a.orig_keys = L.keys_b;
    a.out_keys = nullptr;
  }
  return launch_sort(a, L, stream, events, max_ctas);
}

// Co-resident CTAs of the cooperative sort kernel on this device (0 if unknown).
int sort_grid_capacity() { return std::max(0, sort_grid_limit()); }

// ---------------------------------------------------------------- carried columns
// A raw int64 ORDER BY whose other columns (<= 16 bytes a row, <= 4 columns)
// ride with the rows instead of being gathered by the permutation afterwards:
// on the scatter path with packed rows the counting passes carry their bytes
// beside every key and the local phase copies them out of each run's payload
// window; otherwise (small n, keys varying in more than 32 bits) the same call
// sorts and fuses the gathers into the final pass. Same outputs either way:
// dst row o = src row perm[o].
static int carry_layout(const rl_column* cols, int n, int* offs, int* words) {
  if (n < 1 || n > 4) return RL_ERR_BAD_ARG;
  int order[4] = {0, 1, 2, 3};
  for (int i = 0; i < n; ++i)
    if (!cols[i].src || !cols[i].dst || cols[i].width <= 0) return RL_ERR_BAD_ARG;
  std::sort(order, order + n, [&](int x, int y) { return cols[x].width > cols[y].width; });
  int at = 0;
  for (int k = 0; k < n; ++k) {
    const int w = cols[order[k]].width;
    const int al = (w % 8 == 0) ? 8 : (w % 4 == 0) ? 4 : 1;
    at = (at + al - 1) / al * al;
    offs[order[k]] = at;
    at += w;
  }
  *words = at <= 16 ? (at + 7) / 8 : 0;
  return RL_OK;
}

size_t carry_workspace_bytes(int64_t n, int words) {
  CarveSize c;
  c.take<uint8_t>(workspace_bytes(n));
  if (words > 0) {
    c.take<uint64_t>(size_t(std::max<int64_t>(n, 1)) * words);
    c.take<uint64_t>(size_t(std::max<int64_t>(n, 1)) * words);
  }
  return c.used + 256;
}

int sort_axis_carry(const int64_t* keys, int64_t n, int descending, int64_t* sorted_keys_out, uint32_t* perm_out,
                    const rl_column* columns, int n_columns, void* ws, size_t ws_bytes, cudaStream_t stream) {
  int offs[4] = {0, 0, 0, 0}, words = 0;
  if (n_columns < 1 || !columns) return RL_ERR_BAD_ARG;
  int st = carry_layout(columns, n_columns, offs, &words);
  if (st != RL_OK) return st;
  for (int i = 0; i < n_columns; ++i)
    if (columns[i].side != RL_SIDE_LEFT) return RL_ERR_BAD_ARG;
  const bool scatter = n >= scatter_min_rows() && n >= kHybridMinRows && !getenv_flag_no_hybrid() &&
                       !getenv_flag("RL_NO_SCATTER") && !getenv_flag("RL_NO_CARRY") &&
                       (n <= kTwoLevelMaxRows || n >= level3_min_rows()) && words > 0;
  if (!scatter)  // plain sort + the gathers fused into its final writes
    return sort_axis_capped(keys, RL_COL_INT64, 8, 0, descending, nullptr, n, sorted_keys_out, perm_out, ws, ws_bytes,
                            stream, nullptr, nullptr, columns, n_columns, 0);
  if (n < 0 || !keys || !perm_out || (reinterpret_cast<uintptr_t>(keys) & 15)) return RL_ERR_BAD_ARG;
  if (n > RL_MAX_ROWS) return RL_ERR_TOO_MANY_ROWS;
  if (reinterpret_cast<uintptr_t>(ws) % 256 != 0) return RL_ERR_WORKSPACE;
  Carve c{static_cast<char*>(ws), ws_bytes};
  char* inner = c.take<char>(workspace_bytes(n));
  uint64_t* pa = c.take<uint64_t>(size_t(n) * words);
  uint64_t* pb = c.take<uint64_t>(size_t(n) * words);
  if (!c.ok) return RL_ERR_WORKSPACE;
  Layout L;
  if (!carve_layout(L, inner, workspace_bytes(n), n)) return RL_ERR_WORKSPACE;
  SortArgs a = {};
  a.col = keys;
  a.n = n;
  a.width = 8;
  a.desc = descending ? 1 : 0;
  a.src_mode = kSrcInt64;
  a.key_mode = descending ? kRawDesc : kRawAsc;
  a.orig_keys = keys;
  a.out_keys = sorted_keys_out;
  a.out_vals = perm_out;
  a.keys_a = L.keys_a;
  a.keys_b = L.keys_b;
  a.vals_a = L.vals_a;
  a.vals_b = L.vals_b;
  a.ghist = L.hist;
  a.tile_counter = L.tile_counter;
  a.grid_bar = L.grid_bar;
  a.flags = L.flags;
  a.sub_off = L.sub_off;
  a.status = L.status;
  a.gather.n = n_columns;  // the LSD fallback's fused gathers
  for (int i = 0; i < n_columns; ++i) {
    a.gather.c[i] = columns[i];
    a.carry_src[i] = static_cast<const uint8_t*>(columns[i].src);
    a.carry_dst[i] = static_cast<uint8_t*>(columns[i].dst);
    a.carry_width[i] = columns[i].width;
    a.carry_off[i] = offs[i];
  }
  a.carry_n = n_columns;
  a.cw = words;
  int carried = 0;
  for (int i = 0; i < n_columns; ++i) carried += columns[i].width;
  a.idw = carried <= 4 && !getenv_flag("RL_NO_IDW") ? 1 : 0;
  a.pay_a = pa;
  a.pay_b = pb;
  return launch_sort(a, L, stream, nullptr, 0);
}

int sort_axis(const void* col, int col_kind, int width, int word, int descending, const uint32_t* perm_in,
              int64_t n, int64_t* sorted_keys_out, uint32_t* perm_out, void* ws, size_t ws_bytes,
              cudaStream_t stream, void* const* events, unsigned long long* stamps, const rl_column* columns,
              int n_columns) {
  return sort_axis_capped(col, col_kind, width, word, descending, perm_in, n, sorted_keys_out, perm_out, ws,
                          ws_bytes, stream, events, stamps, columns, n_columns, 0);
}

// ---------------------------------------------------------------- K8
// Stable hash partition: destination word d(i) = fmix64(u64(key) ^
// fmix64(seed)) % parts (hashing.py:54-61), then one stable counting pass
// (only digit 0 is active since parts <= 256) carries the row ids; the
// per-destination counts are the digit-0 histogram.
__global__ void dest_kernel(const int64_t* __restrict__ keys, int64_t n, uint32_t parts, uint64_t mixed_seed,
                            uint64_t* __restrict__ words) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    words[i] = fmix64(uint64_t(keys[i]) ^ mixed_seed) % parts;
}

__global__ void counts_kernel(const uint32_t* hist, int parts, int64_t* counts_out) {
  const int d = threadIdx.x;
  if (d < parts) {  // digit 0's count: the sum of the histogram replicas
    uint32_t c = 0;
    for (int r = 0; r < kHistReps; ++r) c += hist[r * kPasses * kBins + d];
    counts_out[d] = int64_t(c);
  }
}

size_t partition_workspace_bytes(int64_t n) {
  CarveSize c;
  c.take<uint64_t>(size_t(std::max<int64_t>(n, 1)));
  return c.used + 256 + workspace_bytes(n);
}

// Stable counting pass over destination words (< parts <= 256): row ids
// grouped by destination, input order kept within each destination.
static int partition_by_words(const uint64_t* words, int64_t n, int parts, uint32_t* perm_out, int64_t* counts_out,
                              const Layout& L, cudaStream_t stream) {
  SortArgs a = {};
  a.col = words;
  a.perm_in = nullptr;
  a.materialized = nullptr;
  a.n = n;
  a.width = 8;
  a.word = 0;
  a.desc = 0;
  a.src_mode = kSrcWords;
  a.key_mode = kMaterialized;
  a.orig_keys = words;
  a.keys_a = L.keys_a;
  a.keys_b = L.keys_b;
  a.vals_a = L.vals_a;
  a.vals_b = L.vals_b;
  a.out_keys = nullptr;
  a.out_vals = perm_out;
  a.ghist = L.hist;
  a.tile_counter = L.tile_counter;
  a.grid_bar = L.grid_bar;
  a.flags = L.flags;
  a.sub_off = L.sub_off;
  a.status = L.status;
  a.stamps = nullptr;
  a.gather.n = 0;
  int st = launch_sort(a, L, stream, nullptr);
  if (st != RL_OK) return st;
  counts_kernel<<<1, kBins, 0, stream>>>(L.hist, parts, counts_out);
  count_launches(1);
  return rl_cuda_status(cudaGetLastError());
}

static int partition_prologue(int64_t n, int parts, int64_t* counts_out, uint32_t* perm_out, void* ws,
                              size_t ws_bytes, cudaStream_t stream, uint64_t** words, Layout* L) {
  if (n < 0 || parts < 1 || parts > kBins || counts_out == nullptr || (n > 0 && perm_out == nullptr))
    return RL_ERR_BAD_ARG;
  if (n > RL_MAX_ROWS) return RL_ERR_TOO_MANY_ROWS;
  if (reinterpret_cast<uintptr_t>(ws) % 256 != 0) return RL_ERR_WORKSPACE;
  cudaError_t e = cudaMemsetAsync(counts_out, 0, sizeof(int64_t) * size_t(parts), stream);
  if (e != cudaSuccess) return rl_cuda_status(e);
  if (n == 0) return RL_OK;
  Carve c{static_cast<char*>(ws), ws_bytes};
  *words = c.take<uint64_t>(size_t(n));
  if (!c.ok) return RL_ERR_WORKSPACE;
  if (!carve_layout(*L, c.base + align_up(c.used, 256), ws_bytes - align_up(c.used, 256), n)) return RL_ERR_WORKSPACE;
  return RL_OK;
}

int hash_partition_perm(const int64_t* keys, int64_t n, int parts, uint64_t seed, uint32_t* perm_out,
                        int64_t* counts_out, void* ws, size_t ws_bytes, cudaStream_t stream) {
  if (n > 0 && keys == nullptr) return RL_ERR_BAD_ARG;
  uint64_t* words = nullptr;
  Layout L;
  int st = partition_prologue(n, parts, counts_out, perm_out, ws, ws_bytes, stream, &words, &L);
  if (st != RL_OK || n == 0) return st;
  const int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(device_sm_count()) * 8));
  dest_kernel<<<grid, 256, 0, stream>>>(keys, n, uint32_t(parts), fmix64(seed), words);
  count_launches(1);
  return partition_by_words(words, n, parts, perm_out, counts_out, L, stream);
}

// Range partition for the distributed sort: row i (global id gid_base + i)
// goes to the number of splitters strictly below (key, gid) in
// lexicographic order, so equal keys split by global row id and every
// rank's range is contiguous in the global (stable) order.
__global__ void range_dest_kernel(const int64_t* __restrict__ keys, int64_t n, int64_t gid_base,
                                  const int64_t* __restrict__ split_keys, const int64_t* __restrict__ split_gids,
                                  int nsplit, int desc, uint64_t* __restrict__ words) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = xform(uint64_t(keys[i]), desc);
    const int64_t g = gid_base + i;
    uint32_t d = 0;
    for (int s = 0; s < nsplit; ++s) {
      const uint64_t sk = xform(uint64_t(split_keys[s]), desc);
      d += (sk < k || (sk == k && split_gids[s] < g)) ? 1u : 0u;
    }
    words[i] = d;
  }
}

int range_partition_perm(const int64_t* keys, int64_t n, int64_t gid_base, const int64_t* split_keys,
                         const int64_t* split_gids, int nsplit, int descending, uint32_t* perm_out,
                         int64_t* counts_out, void* ws, size_t ws_bytes, cudaStream_t stream) {
  if ((n > 0 && keys == nullptr) || nsplit < 0 || (nsplit > 0 && (!split_keys || !split_gids))) return RL_ERR_BAD_ARG;
  uint64_t* words = nullptr;
  Layout L;
  const int parts = nsplit + 1;
  int st = partition_prologue(n, parts, counts_out, perm_out, ws, ws_bytes, stream, &words, &L);
  if (st != RL_OK || n == 0) return st;
  const int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(device_sm_count()) * 8));
  range_dest_kernel<<<grid, 256, 0, stream>>>(keys, n, gid_base, split_keys, split_gids, nsplit, descending ? 1 : 0,
                                              words);
  count_launches(1);
  return partition_by_words(words, n, parts, perm_out, counts_out, L, stream);
}

// ---------------------------------------------------------------- bucket join
static_assert(kBjCap == kLocalCap, "the sub-bucket overflow check guards the bucket join's capacity");
// bucket_join.cu partitions BOTH join sides into the same 65536 sub-buckets
// (top 16 bits of one joint key packing) with the scatter path's first three
// kernels in packed-row mode, then joins sub-bucket pairs on chip. Here: the
// joint pack code and the per-side launches.

// One CTA: the joint pack code from 512 strided samples of each side, the
// varying bits taken against the LEFT side's first key (every key of both
// sides is checked against it by the chunk counts). Packed rows need <= 32
// varying bits and n <= 2^32 per side; otherwise both sides are flagged to
// fall back (flags[0]) and every later kernel returns at once.
// Heavy keys are caught here too: if one sub-bucket holds >= 8 of a side's
// 512 samples (uniform keys: <= 3 almost surely) and its share of the side's
// rows would exceed twice the on-chip cap, the plan declines at once instead
// of after both sides' partition passes (BASELINE cfg3's Zipf keys).
__global__ void __launch_bounds__(1024) bj_pack_kernel(const long long* lk, int64_t nl, const long long* rk,
                                                       int64_t nr, uint32_t* flags_l, uint32_t* flags_r) {
  __shared__ unsigned long long red;
  __shared__ uint32_t code, heavy;
  __shared__ uint16_t sub[1024];
  const int tid = threadIdx.x;
  if (tid == 0) {
    red = 0;
    heavy = 0;
  }
  __syncthreads();
  const uint64_t k0 = xform(uint64_t(__ldg(lk)), 0);
  const long long* col = tid < 512 ? lk : rk;
  const int64_t n = tid < 512 ? nl : nr;
  const int j = tid & 511;
  uint64_t u = 0, v = 0;
  if (n > 0) {
    u = xform(uint64_t(__ldg(col + int64_t(j) * n / 512)), 0);
    v = u ^ k0;
  }
  const uint32_t vh = __reduce_or_sync(0xffffffffu, uint32_t(v >> 32));
  const uint32_t vl = __reduce_or_sync(0xffffffffu, uint32_t(v));
  if ((tid & 31) == 0 && (vh | vl)) atomicOr(&red, (uint64_t(vh) << 32) | vl);
  __syncthreads();
  if (tid == 0) {
    // all keys equal in the sample: pack one low bit so the code is valid (the
    // chunk counts catch any key that differs)
    const uint64_t vary = red ? red : 1ull;
    code = pack_code_of(vary);
  }
  __syncthreads();
  const uint32_t c = code;
  sub[tid] = uint16_t(pack_key(u, c) >> 48);
  __syncthreads();
  if (n > 0) {  // this sample's sub-bucket among its side's samples
    const uint16_t me = sub[tid];
    const int base = tid < 512 ? 0 : 512;
    uint32_t same = 0;
    for (int i = 0; i < 512; ++i) same += sub[base + i] == me ? 1u : 0u;
    if (same >= 8u && double(same - 2) / 512.0 * double(n) > 2.0 * kLocalCap) atomicOr(&heavy, 1u);
  }
  __syncthreads();
  if (tid == 0) {
    const bool ok = pack_mode(c) != 0 && (c >> 14 & 127) + (c & 127) <= 32u && nl <= (int64_t(1) << 32) &&
                    nr <= (int64_t(1) << 32) && !heavy;
    flags_l[6] = c;
    flags_r[6] = c;
    if (!ok) {
      flags_l[0] = 1u;
      flags_r[0] = 1u;
    }
  }
}

int bj_levels(int64_t nl, int64_t nr) {
  const char* v = getenv("RL_BJ_LEVELS");  // "3": the third level at any size (tests)
  if (v && v[0] == '3') return 3;
  return std::max(nl, nr) > kTwoLevelMaxRows ? 3 : 2;
}

size_t bj_side_workspace_bytes(int64_t n, int words, int levels) {
  CarveSize c;
  carve_all(c, std::max<int64_t>(n, 1), [](CarveSize& c, size_t k) { c.take<uint32_t>(k); return (uint32_t*)nullptr; },
            [](CarveSize& c, size_t k) { c.take<uint64_t>(k); return (uint64_t*)nullptr; }, nullptr, true, levels);
  if (words > 0) {  // carried payload, ping-pong
    c.take<uint64_t>(size_t(std::max<int64_t>(n, 1)) * words);
    c.take<uint64_t>(size_t(std::max<int64_t>(n, 1)) * words);
  }
  return c.used + 256;
}


static SortArgs bj_args(const int64_t* keys, int64_t n, const int64_t* k0_src, const Layout& L) {
  SortArgs a = {};
  a.col = keys;
  a.n = n;
  a.width = 8;
  a.src_mode = kSrcInt64;
  a.key_mode = kRawAsc;
  a.orig_keys = keys;
  a.keys_a = L.keys_a;
  a.keys_b = L.keys_b;
  a.vals_a = L.vals_a;
  a.vals_b = L.vals_b;
  a.ghist = L.hist;
  a.tile_counter = L.tile_counter;
  a.grid_bar = L.grid_bar;
  a.flags = L.flags;
  a.sub_off = L.sub_off;
  a.status = L.status;
  a.mode = kModeScatter;
  a.chunk_cnt = L.chunk_cnt;
  a.cur7 = L.cur7;
  a.cur16 = L.cur16;
  a.d7rep = L.d7rep;
  a.d7_base = L.d7_base;
  a.items = reinterpret_cast<uint4*>(L.items);
  a.meta = L.meta;
  a.allow_pk = 1;
  a.pack_given = 1;
  a.k0_src = reinterpret_cast<const long long*>(k0_src);
  a.bj = 1;
  return a;
}

// Both sides into their sub-buckets: packed rows (key | row id) end up in each
// side's rows_out array (the workspace's keys_a), grouped by the top 16 bits of
// the joint packing; sub_off[65536 + 1] holds the sub-bucket starts; flags[0]
// != 0 on either side means "fall back" (a sub-bucket above kLocalCap, keys not
// packable into 32 bits, a wrapped chunk counter). Nothing is synchronised.
int bj_partition(const int64_t* lkeys, int64_t nl, const int64_t* rkeys, int64_t nr, const BjCarry& lcarry,
                 const BjCarry& rcarry, void* ws_l, size_t ws_l_bytes, void* ws_r, size_t ws_r_bytes,
                 cudaStream_t stream, BjSide* left, BjSide* right) {
  if (nl < 1 || nr < 1 || !lkeys || !rkeys || !left || !right) return RL_ERR_BAD_ARG;
  if (nl > RL_MAX_ROWS || nr > RL_MAX_ROWS) return RL_ERR_TOO_MANY_ROWS;
  if ((reinterpret_cast<uintptr_t>(lkeys) | reinterpret_cast<uintptr_t>(rkeys)) & 15) return RL_ERR_BAD_ARG;
  if ((reinterpret_cast<uintptr_t>(ws_l) | reinterpret_cast<uintptr_t>(ws_r)) % 256 != 0) return RL_ERR_WORKSPACE;
  if (!scatter_kernels_ready() || !carry_kernels_ready<1>() || !carry_kernels_ready<2>())
    return rl_cuda_status(cudaErrorInvalidConfiguration);
  Layout L[2];
  uint64_t* pays[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  const int64_t ns[2] = {nl, nr};
  const int levels = bj_levels(nl, nr);  // both sides alike: equal keys meet in the same sub-bucket index
  const BjCarry* carries[2] = {&lcarry, &rcarry};
  void* wss[2] = {ws_l, ws_r};
  const size_t wsb[2] = {ws_l_bytes, ws_r_bytes};
  for (int i = 0; i < 2; ++i) {
    const BjCarry& cy = *carries[i];
    if (cy.words < 0 || cy.words > kBjMaxCarryWords || cy.n < 0 || cy.n > kBjMaxCarryCols || (cy.n > 0) != (cy.words > 0))
      return RL_ERR_BAD_ARG;
    for (int c = 0; c < cy.n; ++c)
      if (!cy.src[c] || cy.width[c] <= 0 || cy.off[c] < 0 || cy.off[c] + cy.width[c] > 8 * cy.words) return RL_ERR_BAD_ARG;
    Carve c{static_cast<char*>(wss[i]), wsb[i]};
    carve_all(c, ns[i], [](Carve& c, size_t k) { return c.take<uint32_t>(k); },
              [](Carve& c, size_t k) { return c.take<uint64_t>(k); }, &L[i], true, levels);
    if (cy.words > 0) {
      pays[i][0] = c.take<uint64_t>(size_t(ns[i]) * cy.words);
      pays[i][1] = c.take<uint64_t>(size_t(ns[i]) * cy.words);
    }
    if (!c.ok) return RL_ERR_WORKSPACE;
    cudaError_t e = cudaMemsetAsync(L[i].hist, 0, L[i].head_bytes, stream);
    if (e == cudaSuccess && levels == 3) e = cudaMemsetAsync(L[i].cur24, 0, sizeof(uint32_t) * size_t(kSub3), stream);
    if (e != cudaSuccess) return rl_cuda_status(e);
  }
  bj_pack_kernel<<<1, 1024, 0, stream>>>(reinterpret_cast<const long long*>(lkeys), nl,
                                          reinterpret_cast<const long long*>(rkeys), nr, L[0].flags, L[1].flags);
  int launched = 1;
  const int64_t* keys[2] = {lkeys, rkeys};
  BjSide* outs[2] = {left, right};
  for (int i = 0; i < 2; ++i) {
    SortArgs a = bj_args(keys[i], ns[i], lkeys, L[i]);
    a.chunks = int(std::min<int64_t>(std::min(device_sm_count(), kMaxChunks),
                                     std::max<int64_t>(32, (ns[i] + kChunkMinRows - 1) / kChunkMinRows)));
    const BjCarry& cy = *carries[i];
    a.carry_n = cy.n;
    for (int c = 0; c < cy.n; ++c) {
      a.carry_src[c] = cy.src[c];
      a.carry_width[c] = cy.width[c];
      a.carry_off[c] = cy.off[c];
    }
    a.pay_a = pays[i][0];
    a.pay_b = pays[i][1];
    a.levels = levels;
    a.sub3_off = L[i].sub3_off;
    a.cur24 = L[i].cur24;
    a.tile3 = L[i].tile3;
    a.tmap = L[i].tmap;
    const int pgrid = device_sm_count() * pass_ctas_per_sm();
    sub_hist_kernel<<<a.chunks, kScatThreads, kHistSmem, stream>>>(a);
    const size_t sm = psmem_bytes(cy.words);
    auto passes = [&](auto cwc) {
      constexpr int CW = decltype(cwc)::value;
      top_scatter_kernel<CW><<<pgrid, kPThreads, sm, stream>>>(a);
      sub_scatter_kernel<CW><<<pgrid, kPThreads, sm, stream>>>(a);
      if (levels == 3) {  // digit 5 inside every sub-bucket: keys_b / pay_b
        count3_kernel<<<pgrid, kPThreads, 0, stream>>>(a);
        tile_scan_kernel<<<1, 1024, 0, stream>>>(a);
        sub3_scatter_kernel<CW><<<pgrid, kPThreads, sm, stream>>>(a);
      }
    };
    if (cy.words == 0) passes(std::integral_constant<int, 0>{});
    else if (cy.words == 1) passes(std::integral_constant<int, 1>{});
    else passes(std::integral_constant<int, 2>{});
    launched += levels == 3 ? 6 : 3;
    // the last counting pass leaves rows + payload in keys_a / pay_a (two levels) or keys_b / pay_b
    outs[i]->pay = levels == 3 ? pays[i][1] : pays[i][0];
    outs[i]->words = cy.words;
    outs[i]->rows = levels == 3 ? L[i].keys_b : L[i].keys_a;
    outs[i]->levels = levels;
    outs[i]->sub_off = levels == 3 ? L[i].sub3_off : L[i].sub_off;
    outs[i]->flags = L[i].flags;
    outs[i]->n = ns[i];
  }
  count_launches(launched);
  return rl_cuda_status(cudaGetLastError());
}

}  // namespace radix
}  // namespace rl

#ifdef RL_PASS_PROFILE
extern "C" __attribute__((visibility("default"))) int rl_debug_pass_prof(unsigned long long* out16, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out16, rl::radix::g_pass_prof, sizeof(unsigned long long) * 32) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[32] = {};
    cudaMemcpyToSymbol(rl::radix::g_pass_prof, z, sizeof(z));
  }
  return 0;
}
#endif
static_assert(2 * (rl::radix::kLocalKernelSmem + 1024) <= 228 * 1024, "two local-phase CTAs an SM");
