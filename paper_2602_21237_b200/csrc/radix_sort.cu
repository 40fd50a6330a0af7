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
// Key transform (self-inverse): int64 ascending  u = x ^ 2^63;
// descending u = ~x ^ 2^63 (the reference's np.invert, tensorpath.py:215,
// keeps ties in ascending row order). Bytes words are built big-endian
// from (complemented when descending) bytes, zero padded
// (tensorpath.py:220-225).
#include <algorithm>

#include "common.cuh"

namespace rl {
namespace radix {

#ifndef RL_ONESWEEP_ITEMS
#define RL_ONESWEEP_ITEMS 12
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
#define RL_HIST_UNROLL 8
#endif
constexpr int kHistUnroll = RL_HIST_UNROLL;
constexpr int kStamps = 2 + kPasses + 1;  // per-phase globaltimer stamps (profiling)

static_assert(kThreads == kBins, "tile scan maps one digit per thread");
static_assert(kStamps == RL_SORT_STAMPS, "stamp layout is part of the ABI");

enum KeyMode : int { kRawAsc = 0, kRawDesc = 1, kMaterialized = 2 };
enum SrcMode : int { kSrcInt64 = 0, kSrcInt64Gather = 1, kSrcBytes = 2, kSrcWords = 3 };

__device__ __forceinline__ uint64_t xform(uint64_t x, int desc) {
  return (desc ? ~x : x) ^ 0x8000000000000000ull;
}

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
  // zeroed per call
  uint32_t* ghist;           // [kPasses][kBins]
  uint32_t* tile_counter;    // [kPasses]
  uint32_t* grid_bar;        // grid barrier arrivals
  uint64_t* status;          // [num_tiles][kBins] look-back words (epoch = pass + 1)
  unsigned long long* stamps;  // optional [kStamps] globaltimer ns (device)
  // columns gathered by the final permutation inside the last pass
  // (Relation.take fused into the sort: dst row o = src row perm[o])
  FusedColumns gather;
};

__device__ __forceinline__ uint64_t load_key(const SortArgs& a, int64_t i) {
  if (a.src_mode == kSrcInt64) return xform(uint64_t(__ldg(static_cast<const long long*>(a.col) + i)), a.desc);
  if (a.src_mode == kSrcWords) return __ldg(static_cast<const unsigned long long*>(a.col) + i);
  const uint64_t row = a.perm_in ? uint64_t(__ldg(a.perm_in + i)) : uint64_t(i);
  if (a.src_mode == kSrcInt64Gather) return xform(uint64_t(__ldg(static_cast<const long long*>(a.col) + row)), a.desc);
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
constexpr size_t kSmemBytes = kPassSmemBytes + size_t(kPasses) * kBins * 4 + 64;

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
template <int PASS>
__device__ __forceinline__ void run_pass(const SortArgs& a, uint8_t* smem, uint32_t src, uint32_t dst,
                                      const uint32_t* bin_off, PassState& ps) {
  constexpr int kShift = PASS * kBits;
  constexpr uint32_t kEpoch = PASS + 1;
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
    const uint32_t t = atomicAdd(&a.tile_counter[PASS], 1u);
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
      const uint32_t nt = atomicAdd(&a.tile_counter[PASS], 1u);
      misc[cb ^ 1] = nt;  // slot cb^1: its previous value was read before the last barrier
      if (nt < num_tiles) {
        fence_proxy_async_smem();
        prefetch_tile(a.n, kin, vin, nt, bufs + (cb ^ 1) * kBufBytes, &bars[cb ^ 1]);
      }
    }
    const int64_t tile_begin = int64_t(tile) * kTile;
    const int64_t left = a.n - tile_begin;
    const uint32_t count = left < kTile ? uint32_t(left) : uint32_t(kTile);
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
constexpr int kHistThreads = 512;
__global__ void __launch_bounds__(kHistThreads) hist_kernel(SortArgs a) {
  __shared__ uint32_t h[kPasses * kBins];
  const int tid = threadIdx.x;
  if (a.stamps && blockIdx.x == 0 && tid == 0) a.stamps[0] = globaltimer();
  for (int i = tid; i < kPasses * kBins; i += kHistThreads) h[i] = 0;
  __syncthreads();
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
#pragma unroll
      for (int p = 0; p < kPasses; ++p) atomicAdd(&h[p * kBins + ((k[u] >> (p * kBits)) & (kBins - 1))], 1u);
    }
  }
  __syncthreads();
  for (int i = tid; i < kPasses * kBins; i += kHistThreads) {
    const uint32_t c = h[i];
    if (c) atomicAdd(&a.ghist[i], c);
  }
}

// The whole sort after the histograms: plan, every active digit pass,
// copy-through — one cooperative launch.
__global__ void __launch_bounds__(kThreads, RL_ONESWEEP_MIN_BLOCKS) sort_kernel(SortArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* bin_off = reinterpret_cast<uint32_t*>(smem + kPassSmemBytes);  // [kPasses][kBins], whole kernel
  uint32_t* plan = bin_off + kPasses * kBins;                                // [0..7] active, [8] n_active
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOffset);
  const int tid = threadIdx.x;
  uint32_t barrier_no = 0;
  const bool stamper = a.stamps && blockIdx.x == 0 && tid == 0;

  // ---- histograms come from hist_kernel (launched just before, on the same stream)
  if (stamper) a.stamps[1] = globaltimer();

  // ---- plan (every CTA for itself): global digit bases + active digits
  {
    uint32_t* warp_sums = reinterpret_cast<uint32_t*>(smem);  // scratch
    for (int p = 0; p < kPasses; ++p) {
      const uint32_t c = __ldcg(a.ghist + p * kBins + tid);
      uint32_t total;
      bin_off[p * kBins + tid] = block_exclusive_scan<kThreads>(c, warp_sums, &total);
      const int full = __syncthreads_or(uint64_t(c) == uint64_t(a.n));
      if (tid == 0) plan[p] = full ? 0u : 1u;
    }
    if (tid == 0) {
      uint32_t na = 0;
      for (int p = 0; p < kPasses; ++p) na += plan[p];
      plan[kPasses] = na;
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
    }
    __syncthreads();
  }

  // ---- the active digit passes, least significant first
  const uint32_t n_active = plan[kPasses];
  PassState ps{0, 0};
  uint32_t src = 0, seen = 0;
  for (int p = 0; p < kPasses; ++p) {
    if (!plan[p]) continue;
    ++seen;
    const uint32_t dst = seen == n_active ? 3u : (src == 1 ? 2u : 1u);
    switch (p) {
      case 0: run_pass<0>(a, smem, src, dst, bin_off, ps); break;
      case 1: run_pass<1>(a, smem, src, dst, bin_off, ps); break;
      case 2: run_pass<2>(a, smem, src, dst, bin_off, ps); break;
      case 3: run_pass<3>(a, smem, src, dst, bin_off, ps); break;
      case 4: run_pass<4>(a, smem, src, dst, bin_off, ps); break;
      case 5: run_pass<5>(a, smem, src, dst, bin_off, ps); break;
      case 6: run_pass<6>(a, smem, src, dst, bin_off, ps); break;
      default: run_pass<7>(a, smem, src, dst, bin_off, ps); break;
    }
    src = dst;
    if (seen < n_active) grid_sync(a.grid_bar, ++barrier_no);  // the next pass reads what this one wrote
    if (stamper) a.stamps[2 + p] = globaltimer();
  }

  // ---- no active digit (all keys equal, or n == 1): copy through
  if (n_active == 0) {
    for (int64_t i = int64_t(blockIdx.x) * kThreads + tid; i < a.n; i += int64_t(gridDim.x) * kThreads) {
      const uint32_t row = a.perm_in ? a.perm_in[i] : uint32_t(i);
      a.out_vals[i] = row;
      if (a.out_keys) a.out_keys[i] = static_cast<const int64_t*>(a.col)[i];
      gather_fused(a.gather, row, uint64_t(i));
    }
  }
  if (stamper) a.stamps[kStamps - 1] = globaltimer();
}

struct Layout {
  uint32_t* hist;
  uint32_t* tile_counter;
  uint32_t* grid_bar;
  uint64_t* status;
  size_t zero_bytes;  // prefix [hist, counters, barrier, status] zeroed per call
  uint64_t* keys_a;
  uint64_t* keys_b;
  uint32_t* vals_a;
  uint32_t* vals_b;
};

template <typename C>
static void carve(C& c, int64_t n) {
  const size_t tiles = size_t((n + kTile - 1) / kTile);
  c.template take<uint32_t>(kPasses * kBins);
  c.template take<uint32_t>(kPasses);
  c.template take<uint32_t>(1);
  c.template take<uint64_t>(tiles * kBins);
  c.template take<uint64_t>(size_t(n));
  c.template take<uint64_t>(size_t(n));
  c.template take<uint32_t>(size_t(n));
  c.template take<uint32_t>(size_t(n));
}

size_t workspace_bytes(int64_t n) {
  if (n <= 0) return 256;
  CarveSize c;
  carve(c, n);
  return c.used + 256;
}

static bool carve_layout(Layout& L, void* ws, size_t ws_bytes, int64_t n) {
  Carve c{static_cast<char*>(ws), ws_bytes};
  const size_t tiles = size_t((n + kTile - 1) / kTile);
  L.hist = c.take<uint32_t>(kPasses * kBins);
  L.tile_counter = c.take<uint32_t>(kPasses);
  L.grid_bar = c.take<uint32_t>(1);
  L.status = c.take<uint64_t>(tiles * kBins);
  L.zero_bytes = c.used;
  L.keys_a = c.take<uint64_t>(size_t(n));
  L.keys_b = c.take<uint64_t>(size_t(n));
  L.vals_a = c.take<uint32_t>(size_t(n));
  L.vals_b = c.take<uint32_t>(size_t(n));
  return c.ok;
}

__global__ void identity_kernel(const uint32_t* perm_in, int64_t n, uint32_t* out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = perm_in ? perm_in[i] : uint32_t(i);
}

// Largest co-resident grid of the cooperative sort kernel on this device.
static int sort_grid_limit() {
  static int cached = 0;
  if (cached > 0) return cached;
  if (cudaFuncSetAttribute(sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes)) != cudaSuccess)
    return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sort_kernel, kThreads, kSmemBytes) != cudaSuccess ||
      per_sm < 1)
    return -1;
  cached = per_sm * device_sm_count();
  return cached;
}

static int launch_sort(SortArgs a, const Layout& L, cudaStream_t stream, void* const* events) {
  const int limit = sort_grid_limit();
  if (limit < 1) {
    cudaError_t e = cudaGetLastError();
    return rl_cuda_status(e != cudaSuccess ? e : cudaErrorInvalidConfiguration);
  }
  cudaError_t e = cudaMemsetAsync(L.hist, 0, L.zero_bytes, stream);
  if (e != cudaSuccess) return rl_cuda_status(e);
  // enough CTAs for the tiles (and ~8K keys each in the histogram phase), at most all co-resident
  const int64_t tiles = (a.n + kTile - 1) / kTile;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(limit, tiles)));
  if (events) cudaEventRecord(static_cast<cudaEvent_t>(events[0]), stream);
  {
    const int64_t per_cta = int64_t(kHistThreads) * kHistUnroll * 2;
    const int hgrid = int(std::max<int64_t>(1, std::min<int64_t>((a.n + per_cta - 1) / per_cta,
                                                                 int64_t(device_sm_count()) * 4)));
    hist_kernel<<<hgrid, kHistThreads, 0, stream>>>(a);
  }
  if (events) cudaEventRecord(static_cast<cudaEvent_t>(events[1]), stream);
  void* params[] = {&a};
  e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(sort_kernel), dim3(grid), dim3(kThreads), params,
                                  kSmemBytes, stream);
  if (events) cudaEventRecord(static_cast<cudaEvent_t>(events[2]), stream);
  count_launches(2);
  return rl_cuda_status(e != cudaSuccess ? e : cudaGetLastError());
}

int sort_axis(const void* col, int col_kind, int width, int word, int descending, const uint32_t* perm_in,
              int64_t n, int64_t* sorted_keys_out, uint32_t* perm_out, void* ws, size_t ws_bytes,
              cudaStream_t stream, void* const* events, unsigned long long* stamps, const rl_column* columns,
              int n_columns) {
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

  SortArgs a;
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
  return launch_sort(a, L, stream, events);
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
  if (d < parts) counts_out[d] = int64_t(hist[d]);
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
  SortArgs a;
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

}  // namespace radix
}  // namespace rl
