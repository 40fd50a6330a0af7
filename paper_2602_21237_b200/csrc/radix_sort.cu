// radix_sort.cu — K1 (upfront digit histograms) + K2 (onesweep digit pass).
//
// Stable LSD radix sort of 64-bit key words carrying uint32 row ids. It
// replaces the reference's stable argsorts:
//   _stable_key_order   /root/reference/pkg/src/relab/tensorpath.py:62-75
//   _stable_axis_order  /root/reference/pkg/src/relab/tensorpath.py:206-229
//
// Design (B200, HBM-bound integer work — no tensor cores):
//   * K1 reads the keys once and builds all eight 8-bit digit histograms in
//     shared memory (one global atomic per non-empty bin per CTA). For a
//     gathered key (a refinement step of a multi-key sort, or a Bytes word)
//     it also materialises the transformed 64-bit key words so the first
//     digit pass streams them contiguously.
//   * A one-CTA plan kernel scans the histograms into global digit bases
//     and marks passes whose digit is constant over the input as inactive.
//     The plan (active flags, ping-pong buffer choice, epochs) stays on the
//     device: the host launches all eight passes and inactive ones exit at
//     once, so a sort never synchronises the host.
//   * K2 is a onesweep pass: tiles of 4096 keys are claimed in launch order
//     by an atomic counter; each warp ranks its 512 keys with
//     __match_any_sync (stable: lanes in element order, items in order);
//     the tile publishes its per-digit counts, scatters keys+row ids into a
//     shared-memory staging buffer in digit order while the decoupled
//     look-back resolves its global digit offsets, and finally writes the
//     staged tile out in ascending local order, so every digit run is a
//     contiguous, coalesced burst.
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
#ifndef RL_RANK_BALLOT
#define RL_RANK_BALLOT 1
#endif
#ifndef RL_ONESWEEP_MIN_BLOCKS
#define RL_ONESWEEP_MIN_BLOCKS 2
#endif

constexpr int kBits = 8;
constexpr int kBins = 1 << kBits;
constexpr int kPasses = 64 / kBits;
constexpr int kThreads = 256;  // == kBins: one digit per thread in the tile scan
constexpr int kItems = RL_ONESWEEP_ITEMS;
constexpr int kTile = kThreads * kItems;
constexpr int kWarps = kThreads / 32;
#ifndef RL_LOOKBACK_WINDOW
#define RL_LOOKBACK_WINDOW 4
#endif
constexpr int kLookback = RL_LOOKBACK_WINDOW;
constexpr int kHistThreads = 512;
constexpr int kHistUnroll = 4;

static_assert(kThreads == kBins, "tile scan maps one digit per thread");

enum KeyMode : int { kRawAsc = 0, kRawDesc = 1, kMaterialized = 2 };
enum SrcMode : int { kSrcInt64 = 0, kSrcInt64Gather = 1, kSrcBytes = 2, kSrcWords = 3 };

struct Plan {
  uint32_t n_active;
  uint32_t active[kPasses];
  uint32_t src[kPasses];  // 0 original, 1 buffer A, 2 buffer B
  uint32_t dst[kPasses];  // 1 buffer A, 2 buffer B, 3 final outputs
};

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

struct HistArgs {
  const void* col;
  const uint32_t* perm_in;
  uint64_t* materialized;  // only for gather / bytes modes
  uint32_t* ghist;         // [kPasses][kBins]
  int64_t n;
  int width, word, desc, src_mode;
};

__device__ __forceinline__ uint64_t load_key(const HistArgs& a, int64_t i) {
  if (a.src_mode == kSrcInt64) {
    return xform(uint64_t(__ldg(static_cast<const long long*>(a.col) + i)), a.desc);
  }
  uint64_t row = a.perm_in ? uint64_t(__ldg(a.perm_in + i)) : uint64_t(i);
  if (a.src_mode == kSrcWords) return __ldg(static_cast<const unsigned long long*>(a.col) + i);
  if (a.src_mode == kSrcInt64Gather) {
    return xform(uint64_t(__ldg(static_cast<const long long*>(a.col) + row)), a.desc);
  }
  const uint8_t* base = static_cast<const uint8_t*>(a.col) + row * uint64_t(a.width);
  return bytes_word(base, a.width, a.word, a.desc);
}

// K1: all digit histograms in one read of the keys.
__global__ void __launch_bounds__(kHistThreads) hist_kernel(HistArgs a) {
  __shared__ uint32_t h[kPasses * kBins];
  for (int i = threadIdx.x; i < kPasses * kBins; i += kHistThreads) h[i] = 0;
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * kHistThreads * kHistUnroll;
  for (int64_t base = int64_t(blockIdx.x) * kHistThreads * kHistUnroll + threadIdx.x; base < a.n;
       base += stride) {
    uint64_t k[kHistUnroll];
    bool ok[kHistUnroll];
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      int64_t i = base + int64_t(u) * kHistThreads;
      ok[u] = i < a.n;
      k[u] = ok[u] ? load_key(a, i) : 0;
    }
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      if (!ok[u]) continue;
      if (a.materialized) a.materialized[base + int64_t(u) * kHistThreads] = k[u];
#pragma unroll
      for (int p = 0; p < kPasses; ++p) atomicAdd(&h[p * kBins + ((k[u] >> (p * kBits)) & (kBins - 1))], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kPasses * kBins; i += kHistThreads) {
    uint32_t c = h[i];
    if (c) atomicAdd(&a.ghist[i], c);
  }
}

// Global digit bases + the device-side pass plan.
__global__ void __launch_bounds__(kBins) plan_kernel(const uint32_t* ghist, uint32_t* bin_off, Plan* plan,
                                                     uint64_t n) {
  __shared__ uint32_t warp_sums[kBins / 32 + 1];
  __shared__ uint32_t active[kPasses];
  for (int p = 0; p < kPasses; ++p) {
    uint32_t c = ghist[p * kBins + threadIdx.x];
    uint32_t total;
    uint32_t excl = block_exclusive_scan<kBins>(c, warp_sums, &total);
    bin_off[p * kBins + threadIdx.x] = excl;
    int full = __syncthreads_or(uint64_t(c) == n);
    if (threadIdx.x == 0) active[p] = full ? 0u : 1u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t n_active = 0;
    for (int p = 0; p < kPasses; ++p) n_active += active[p];
    uint32_t seen = 0, cur = 0;
    for (int p = 0; p < kPasses; ++p) {
      plan->active[p] = active[p];
      plan->src[p] = 0;
      plan->dst[p] = 0;
      if (!active[p]) continue;
      plan->src[p] = cur;
      ++seen;
      uint32_t d = (seen == n_active) ? 3u : (cur == 1 ? 2u : 1u);
      plan->dst[p] = d;
      cur = d;
    }
    plan->n_active = n_active;
  }
}

struct PassArgs {
  const void* orig_keys;     // raw int64 (key_mode raw) or materialised u64
  const uint32_t* perm_in;   // values of the first pass (NULL = identity)
  uint64_t* keys_a;
  uint64_t* keys_b;
  uint32_t* vals_a;
  uint32_t* vals_b;
  int64_t* out_keys;         // final sorted int64 keys (optional)
  uint32_t* out_vals;        // final permutation
  const Plan* plan;
  const uint32_t* bin_off;
  uint32_t* tile_counter;    // [kPasses]
  uint64_t* status;          // [num_tiles][kBins]
  int64_t n;
  int key_mode;
};

#ifndef RL_RANK_MODE
#define RL_RANK_MODE 2  // 1: ballot match_any, 2: shared atomicOr match (fewest instructions)
#endif

// Shared memory of one persistent onesweep CTA: two tile buffers (one being
// processed — loaded by TMA, then reused as the digit-ordered staging area —
// and one being prefetched), per-warp digit counters and match masks.
constexpr size_t kBufBytes = size_t(kTile) * 12;  // keys (8 B) then row ids (4 B)
constexpr size_t kPassSmem = 2 * kBufBytes + size_t(kWarps) * kBins * 4 * 2 + size_t(kBins) * 4 * 2 + 64 * 4 + 64;

// Stable rank of every item of this warp within its digit, offset by the
// warp's base for that digit (wh[] holds the bases on entry). Warp-striped
// items: element order is (item, lane), so lanes of one item are ranked
// by peer mask and items by the in-order shared atomics on wh[].
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
__device__ __forceinline__ void prefetch_tile(const PassArgs& a, const uint64_t* kin, const uint32_t* vin,
                                              uint32_t tile, uint8_t* buf, uint64_t* bar) {
  const int64_t begin = int64_t(tile) * kTile;
  const int64_t left = a.n - begin;
  const uint32_t count = left < kTile ? uint32_t(left) : uint32_t(kTile);
  const uint32_t kbytes = (count * 8u) & ~15u;
  const uint32_t vbytes = vin ? ((count * 4u) & ~15u) : 0u;
  mbar_expect_tx(bar, kbytes + vbytes);
  if (kbytes) bulk_g2s(buf, kin + begin, kbytes, bar);
  if (vbytes) bulk_g2s(buf + size_t(kTile) * 8, vin + begin, vbytes, bar);
}

// K2: one stable 8-bit onesweep digit pass (PASS selects the digit).
// Persistent: each CTA claims tiles in increasing order from an atomic
// counter and prefetches tile i+1 with TMA while it ranks and scatters tile
// i, so HBM always has loads in flight. Progress: the smallest unfinished
// tile's predecessors are all finished, and it is either being processed
// or queued behind a smaller tile of the same CTA.
template <int PASS>
__global__ void __launch_bounds__(kThreads, RL_ONESWEEP_MIN_BLOCKS) onesweep_kernel(PassArgs a) {
  constexpr int kShift = PASS * kBits;
  constexpr uint32_t kEpoch = PASS + 1;
  const Plan* plan = a.plan;
  if (!plan->active[PASS]) return;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* bufs = smem;
  uint32_t* whist = reinterpret_cast<uint32_t*>(smem + 2 * kBufBytes);
  uint32_t* wmatch = whist + kWarps * kBins;
  uint32_t* local_start = wmatch + kWarps * kBins;
  uint32_t* gbase = local_start + kBins;
  uint32_t* misc = gbase + kBins;  // [0],[1] claimed tile ids (by iteration parity), [4..] scan scratch
  uint64_t* bars = reinterpret_cast<uint64_t*>(misc + 64);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t src = plan->src[PASS], dst = plan->dst[PASS];
  const uint32_t num_tiles = uint32_t((a.n + kTile - 1) / kTile);
  const uint64_t* kin = src == 1 ? a.keys_a : src == 2 ? a.keys_b : static_cast<const uint64_t*>(a.orig_keys);
  const uint32_t* vin = src == 1 ? a.vals_a : src == 2 ? a.vals_b : a.perm_in;
  const bool xf = src == 0 && a.key_mode != kMaterialized;
  const int desc_in = a.key_mode == kRawDesc;

  for (int i = tid; i < 2 * kWarps * kBins; i += kThreads) whist[i] = 0;  // whist + wmatch
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    const uint32_t t = atomicAdd(&a.tile_counter[PASS], 1u);
    misc[0] = t;
    if (t < num_tiles) prefetch_tile(a, kin, vin, t, bufs, &bars[0]);
  }
  __syncthreads();
  uint32_t tile = misc[0];
  uint32_t cb = 0, phase0 = 0, phase1 = 0;  // cb: buffer + claim slot of this iteration
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
        prefetch_tile(a, kin, vin, nt, bufs + (cb ^ 1) * kBufBytes, &bars[cb ^ 1]);
      }
    }
    const int64_t tile_begin = int64_t(tile) * kTile;
    const int64_t left = a.n - tile_begin;
    const uint32_t count = left < kTile ? uint32_t(left) : uint32_t(kTile);
    mbar_wait(&bars[cb], cb ? phase1 : phase0);
    if (cb) phase1 ^= 1; else phase0 ^= 1;
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
    uint32_t rank2[kItems / 2];  // two 16-bit tile-local digit ranks per register (rank < kTile)
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
    // inclusive prefix.
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
    gbase[tid] = a.bin_off[PASS * kBins + tid] + uint32_t(excl) - ls;
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
          __stcs(a.out_vals + o, svals[j]);
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

typedef void (*OnesweepFn)(PassArgs);
static const OnesweepFn kOnesweep[kPasses] = {onesweep_kernel<0>, onesweep_kernel<1>, onesweep_kernel<2>,
                                              onesweep_kernel<3>, onesweep_kernel<4>, onesweep_kernel<5>,
                                              onesweep_kernel<6>, onesweep_kernel<7>};

// No active pass (all keys share every digit, or n == 1): copy through.
__global__ void finalize_kernel(const Plan* plan, const int64_t* raw_keys, const uint32_t* perm_in,
                                int64_t n, int64_t* out_keys, uint32_t* out_vals) {
  if (plan != nullptr && plan->n_active != 0) return;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    out_vals[i] = perm_in ? perm_in[i] : uint32_t(i);
    if (out_keys) out_keys[i] = raw_keys[i];
  }
}

struct Layout {
  uint32_t* hist;
  uint32_t* tile_counter;
  uint64_t* status;
  size_t zero_bytes;  // prefix [hist, counters, status] zeroed per call
  uint32_t* bin_off;
  Plan* plan;
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
  c.template take<uint64_t>(tiles * kBins);
  c.template take<uint32_t>(kPasses * kBins);
  c.template take<Plan>(1);
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
  L.status = c.take<uint64_t>(tiles * kBins);
  L.zero_bytes = c.used;
  L.bin_off = c.take<uint32_t>(kPasses * kBins);
  L.plan = c.take<Plan>(1);
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

// Shared launcher: K1 → plan → 8 × K2 → finalize. `h` describes how K1
// reads keys; `orig_keys`/`key_mode` how the first active pass reads them.
static int launch_sort(HistArgs h, const void* orig_keys, int key_mode, const uint32_t* perm_in, int64_t n,
                       int64_t* sorted_keys_out, uint32_t* perm_out, const Layout& L, cudaStream_t stream,
                       void* const* events = nullptr) {
  const int sms = device_sm_count();
  auto mark = [&](int i) {
    if (events) cudaEventRecord(static_cast<cudaEvent_t>(events[i]), stream);
  };
  cudaError_t e = cudaMemsetAsync(L.hist, 0, L.zero_bytes, stream);
  if (e != cudaSuccess) return rl_cuda_status(e);
  {
    int64_t per_cta = int64_t(kHistThreads) * kHistUnroll * 4;
    int grid = int(std::min<int64_t>((n + per_cta - 1) / per_cta, int64_t(sms) * 4));
    mark(0);
    hist_kernel<<<std::max(grid, 1), kHistThreads, 0, stream>>>(h);
  }
  mark(1);
  plan_kernel<<<1, kBins, 0, stream>>>(L.hist, L.bin_off, L.plan, uint64_t(n));

  PassArgs p;
  p.orig_keys = orig_keys;
  p.perm_in = perm_in;
  p.keys_a = L.keys_a;
  p.keys_b = L.keys_b;
  p.vals_a = L.vals_a;
  p.vals_b = L.vals_b;
  p.out_keys = sorted_keys_out;
  p.out_vals = perm_out;
  p.plan = L.plan;
  p.bin_off = L.bin_off;
  p.tile_counter = L.tile_counter;
  p.status = L.status;
  p.n = n;
  p.key_mode = key_mode;
  static bool attr_set = false;  // idempotent; a racing duplicate call is harmless
  if (!attr_set) {
    for (int pass = 0; pass < kPasses; ++pass) {
      e = cudaFuncSetAttribute(kOnesweep[pass], cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPassSmem));
      if (e != cudaSuccess) return rl_cuda_status(e);
    }
    attr_set = true;
  }
  const int tiles = int((n + kTile - 1) / kTile);
  const int grid = std::min(tiles, sms * RL_ONESWEEP_MIN_BLOCKS);
  for (int pass = 0; pass < kPasses; ++pass) {
    mark(2 + pass);
    kOnesweep[pass]<<<grid, kThreads, kPassSmem, stream>>>(p);
  }
  {
    int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(sms) * 8));
    mark(2 + kPasses);
    finalize_kernel<<<grid, 256, 0, stream>>>(L.plan, static_cast<const int64_t*>(orig_keys), perm_in, n,
                                              key_mode == kMaterialized ? nullptr : sorted_keys_out, perm_out);
    mark(3 + kPasses);
  }
  count_launches(3 + kPasses);
  return rl_cuda_status(cudaGetLastError());
}

int sort_axis(const void* col, int col_kind, int width, int word, int descending, const uint32_t* perm_in,
              int64_t n, int64_t* sorted_keys_out, uint32_t* perm_out, void* ws, size_t ws_bytes,
              cudaStream_t stream, void* const* events) {
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
  if (col_kind == RL_COL_BYTES && width == 0) {  // tensorpath.py:218-219: identity order
    int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(device_sm_count()) * 8));
    identity_kernel<<<grid, 256, 0, stream>>>(perm_in, n, perm_out);
    count_launches(1);
    return rl_cuda_status(cudaGetLastError());
  }
  if (reinterpret_cast<uintptr_t>(ws) % 256 != 0) return RL_ERR_WORKSPACE;
  Layout L;
  if (!carve_layout(L, ws, ws_bytes, n)) return RL_ERR_WORKSPACE;

  HistArgs h;
  h.col = col;
  h.perm_in = perm_in;
  h.ghist = L.hist;
  h.n = n;
  h.width = width;
  h.word = word;
  h.desc = descending ? 1 : 0;
  if (col_kind == RL_COL_INT64 && perm_in == nullptr) {
    h.src_mode = kSrcInt64;
    h.materialized = nullptr;
    return launch_sort(h, col, descending ? kRawDesc : kRawAsc, nullptr, n, sorted_keys_out, perm_out, L, stream,
                       events);
  }
  h.src_mode = col_kind == RL_COL_INT64 ? kSrcInt64Gather : kSrcBytes;
  h.materialized = L.keys_b;  // read once by the first active pass, then reused as ping-pong B
  return launch_sort(h, L.keys_b, kMaterialized, perm_in, n, nullptr, perm_out, L, stream, events);
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

int hash_partition_perm(const int64_t* keys, int64_t n, int parts, uint64_t seed, uint32_t* perm_out,
                        int64_t* counts_out, void* ws, size_t ws_bytes, cudaStream_t stream) {
  if (n < 0 || parts < 1 || parts > kBins || counts_out == nullptr || (n > 0 && (keys == nullptr || perm_out == nullptr)))
    return RL_ERR_BAD_ARG;
  if (n > RL_MAX_ROWS) return RL_ERR_TOO_MANY_ROWS;
  if (reinterpret_cast<uintptr_t>(ws) % 256 != 0) return RL_ERR_WORKSPACE;
  cudaError_t e = cudaMemsetAsync(counts_out, 0, sizeof(int64_t) * size_t(parts), stream);
  if (e != cudaSuccess) return rl_cuda_status(e);
  if (n == 0) return RL_OK;
  Carve c{static_cast<char*>(ws), ws_bytes};
  uint64_t* words = c.take<uint64_t>(size_t(n));
  if (!c.ok) return RL_ERR_WORKSPACE;
  Layout L;
  if (!carve_layout(L, c.base + align_up(c.used, 256), ws_bytes - align_up(c.used, 256), n)) return RL_ERR_WORKSPACE;
  const int sms = device_sm_count();
  const int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(sms) * 8));
  dest_kernel<<<grid, 256, 0, stream>>>(keys, n, uint32_t(parts), fmix64(seed), words);
  count_launches(2);
  HistArgs h;
  h.col = words;
  h.perm_in = nullptr;
  h.ghist = L.hist;
  h.n = n;
  h.width = 8;
  h.word = 0;
  h.desc = 0;
  h.src_mode = kSrcWords;
  h.materialized = nullptr;
  int st = launch_sort(h, words, kMaterialized, nullptr, n, nullptr, perm_out, L, stream);
  if (st != RL_OK) return st;
  counts_kernel<<<1, kBins, 0, stream>>>(L.hist, parts, counts_out);
  return rl_cuda_status(cudaGetLastError());
}

}  // namespace radix
}  // namespace rl
