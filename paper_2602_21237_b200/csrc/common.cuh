// common.cuh — shared device helpers for the sm_100a tensor-path kernels.
//
// Decoupled look-back status words (Merrill & Garland single-pass scan;
// Adinets & Merrill onesweep) are packed into one 64-bit word so a
// reader sees flag, epoch and value atomically:
//
//   [63:62] flag   0 = not yet published, 1 = tile aggregate, 2 = inclusive
//   [61:56] epoch  which pass/launch wrote it (stale words are ignored)
//   [55:0]  value
//
// The status arrays are zeroed once per call (one cudaMemsetAsync); the
// epoch lets the eight radix passes of one sort share a single array.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/relab_b200.h"

namespace rl {

constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagIncl = 2ull << 62;
constexpr uint64_t kFlagMask = 3ull << 62;
constexpr uint64_t kValueMask = (1ull << 56) - 1;

__device__ __forceinline__ uint64_t pack_status(uint64_t flag, uint32_t epoch,
                                                uint64_t value) {
  return flag | (uint64_t(epoch & 63u) << 56) | (value & kValueMask);
}
__device__ __forceinline__ uint32_t status_epoch(uint64_t s) {
  return uint32_t(s >> 56) & 63u;
}

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Streaming stores: output columns are written once and not re-read by
// this kernel, so keep them from displacing the gathered inputs in L2.
__device__ __forceinline__ void st_stream(uint64_t* p, uint64_t v) { __stcs(reinterpret_cast<unsigned long long*>(p), v); }
__device__ __forceinline__ void st_stream(uint32_t* p, uint32_t v) { __stcs(p, v); }

// ---- TMA bulk copies (cp.async.bulk, global → shared) completed on an
// mbarrier. Sizes and addresses must be 16-byte multiples / aligned.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {  // release: prior accesses of this thread
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred done;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      " @!done bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// L2 prefetch of [p, p + bytes) by one bulk request (the span is widened to
// whole 16-byte units; a hint: no completion to wait for).
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, size_t bytes) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  if (a1 > a0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(uint32_t(a1 - a0)) : "memory");
}
// Order earlier generic-proxy accesses to shared memory before later
// async-proxy (TMA) writes into the same buffer.
// Programmatic dependent launch: the next kernel of the stream may be
// scheduled now (its CTAs take SMs as this kernel's CTAs exit) / wait until
// the previous kernel has completed and its writes are visible (a no-op for a
// kernel not launched as a programmatic dependent).
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Murmur3 fmix64 (hashing.py:32-40).
__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xFF51AFD7ED558CCDull;
  x ^= x >> 33;
  x *= 0xC4CEB9FE1A85EC53ull;
  x ^= x >> 33;
  return x;
}

// Block-wide exclusive scan of one value per thread (THREADS ≤ 1024).
// `warp_sums` must hold THREADS/32 entries. Returns the exclusive prefix;
// *total receives the block total.
template <int THREADS, typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* warp_sums, T* total) {
  constexpr int kWarps = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += n;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    T s = lane < kWarps ? warp_sums[lane] : T(0);
    T si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T n = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += n;
    }
    if (lane < kWarps) warp_sums[lane] = si - s;  // exclusive warp offsets
    if (lane == kWarps - 1) warp_sums[kWarps] = si;
  }
  __syncthreads();
  T out = warp_sums[warp] + incl - v;
  *total = warp_sums[kWarps];
  return out;
}

// Counters -> exclusive starts over hist[0, nbins) (nbins <= NBINS, a multiple
// of 4; hist 16-byte aligned). Warp w owns bins [w W, (w + 1) W) and reads them
// as uint4 by consecutive lanes — conflict-free, where a thread owning
// consecutive bins strides the banks. `warp_tot` holds THREADS / 32 words.
// Ends with the block synchronised.
// BAR > 0: the threads [0, THREADS) synchronise on named barrier BAR (a
// producer warp beside them does not take part), else the whole block.
template <int THREADS, int BAR>
__device__ __forceinline__ void threads_sync() {
  if constexpr (BAR > 0) asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(THREADS) : "memory");
  else __syncthreads();
}

template <int THREADS, int NBINS, int BAR = 0>
__device__ __forceinline__ void scan_counters(uint32_t* hist, uint32_t nbins, uint32_t* warp_tot) {
  constexpr int kWarps = THREADS / 32;
  constexpr uint32_t W = uint32_t(NBINS / kWarps), C = W / 128;
  static_assert(NBINS % (kWarps * 128) == 0, "uint4 counters, whole warps");
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint4* h4 = reinterpret_cast<uint4*>(hist) + warp * (W / 4);
  const uint32_t lo4 = warp * (W / 4);
  const uint32_t lim4 = nbins / 4 > lo4 ? nbins / 4 - lo4 : 0u;  // this warp's counters in use
  uint32_t wt = 0;
#pragma unroll
  for (uint32_t i = 0; i < C; ++i) {
    const uint32_t q = i * 32 + lane;
    if (q < lim4) {
      const uint4 c = h4[q];
      wt += c.x + c.y + c.z + c.w;
    }
  }
  wt = __reduce_add_sync(0xffffffffu, wt);
  if (lane == 0) warp_tot[warp] = wt;
  threads_sync<THREADS, BAR>();
  uint32_t start = 0;
  for (uint32_t w = 0; w < warp; ++w) start += warp_tot[w];
#pragma unroll
  for (uint32_t i = 0; i < C; ++i) {
    const uint32_t q = i * 32 + lane;
    const uint4 c = q < lim4 ? h4[q] : make_uint4(0, 0, 0, 0);
    const uint32_t sum = c.x + c.y + c.z + c.w;
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= uint32_t(o)) incl += x;
    }
    if (q < lim4) {
      uint4 o4;
      o4.x = start + incl - sum;
      o4.y = o4.x + c.x;
      o4.z = o4.y + c.y;
      o4.w = o4.z + c.z;
      h4[q] = o4;
    }
    start += __shfl_sync(0xffffffffu, incl, 31);
  }
  threads_sync<THREADS, BAR>();
}

// Single-value decoupled look-back: returns the exclusive prefix of tile
// `tile` and publishes its inclusive value. Called by one thread.
__device__ __forceinline__ uint64_t lookback_publish(uint64_t* status, uint32_t tile,
                                                     uint32_t epoch, uint64_t aggregate) {
  if (tile == 0) {
    st_relaxed(&status[0], pack_status(kFlagIncl, epoch, aggregate));
    return 0;
  }
  st_relaxed(&status[tile], pack_status(kFlagAgg, epoch, aggregate));
  uint64_t excl = 0;
  int64_t p = int64_t(tile) - 1;
  while (true) {
    uint64_t s = ld_relaxed(&status[p]);
    if ((s & kFlagMask) == 0 || status_epoch(s) != (epoch & 63u)) continue;
    excl += s & kValueMask;
    if ((s & kFlagMask) == kFlagIncl) break;
    --p;
  }
  st_relaxed(&status[tile], pack_status(kFlagIncl, epoch, excl + aggregate));
  return excl;
}

// Warp-parallel decoupled look-back (called by all 32 lanes of one warp):
// lane l inspects predecessor tile - 1 - l, a whole window per round trip.
// Single packed value per tile. Returns the exclusive prefix (all lanes).
__device__ __forceinline__ uint64_t warp_lookback(const uint64_t* status, uint32_t tile, uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  uint64_t excl = 0;
  int64_t base = int64_t(tile) - 1;
  while (true) {
    const int64_t p = base - lane;
    const uint64_t s = p >= 0 ? ld_relaxed(status + p) : (kFlagIncl | (uint64_t(epoch & 63u) << 56));
    const bool ready = (s & kFlagMask) != 0 && status_epoch(s) == (epoch & 63u);
    const uint32_t incl = __ballot_sync(0xffffffffu, ready && (s & kFlagMask) == kFlagIncl);
    const uint32_t notready = __ballot_sync(0xffffffffu, !ready);
    const int stop = incl ? __ffs(incl) - 1 : 31;  // nearest inclusive predecessor in the window
    const uint32_t need = stop == 31 ? 0xffffffffu : ((2u << stop) - 1u);
    if (notready & need) {
      __nanosleep(32);
      continue;
    }
    uint64_t v = lane <= stop ? (s & kValueMask) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (incl) return excl;
    base -= 32;
  }
}

inline int rl_cuda_status(cudaError_t e) { return e == cudaSuccess ? RL_OK : RL_ERR_CUDA + int(e); }

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Simple bump allocator over the caller's workspace.
struct Carve {
  char* base;
  size_t cap;
  size_t used = 0;
  bool ok = true;
  template <typename T>
  T* take(size_t count) {
    size_t off = align_up(used, 256);
    size_t bytes = count * sizeof(T);
    if (off + bytes > cap) {
      ok = false;
      return nullptr;
    }
    used = off + bytes;
    return reinterpret_cast<T*>(base + off);
  }
};

// Measuring pass of the same carve sequence (workspace queries).
struct CarveSize {
  size_t used = 0;
  template <typename T>
  void take(size_t count) {
    used = align_up(used, 256) + count * sizeof(T);
  }
};

// Output column descriptors travel by value in kernel parameters.
struct ColumnSet {
  rl_column c[RL_MAX_COLUMNS];
  int n;
};

// Copy one w-byte row (w = 8 / 4 / 16 fast paths; any width >= 0).
// A random row read (the gathers): ld.global.cg, cached in L2 only — a row
// read once gains nothing from an L1 allocation. Measured on the 1e8-row
// join's expansion against __ldg: 4.58 -> 4.51 ms, DRAM writes 5.49 -> 5.08 GB;
// its DRAM reads (19.6 GB for 217M requested 32-byte sectors, i.e. ~3x) and
// L2 sector reads did not change, so the amplification is not L1 line fills.
template <typename T>
__device__ __forceinline__ T ld_row(const T* p) {
#ifdef RL_GATHER_LDG
  return __ldg(p);
#else
  return __ldcg(p);
#endif
}

__device__ __forceinline__ void copy_row(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int w) {
  if (w == 8) {
    __stcs(reinterpret_cast<unsigned long long*>(dst), ld_row(reinterpret_cast<const unsigned long long*>(src)));
  } else if (w == 4) {
    __stcs(reinterpret_cast<unsigned int*>(dst), ld_row(reinterpret_cast<const unsigned int*>(src)));
  } else if (w == 16) {
    __stcs(reinterpret_cast<uint4*>(dst), ld_row(reinterpret_cast<const uint4*>(src)));
  } else if ((w & 7) == 0) {
    for (int b = 0; b < w; b += 8)
      *reinterpret_cast<uint64_t*>(dst + b) = ld_row(reinterpret_cast<const unsigned long long*>(src + b));
  } else if ((w & 3) == 0) {
    for (int b = 0; b < w; b += 4)
      *reinterpret_cast<uint32_t*>(dst + b) = ld_row(reinterpret_cast<const unsigned int*>(src + b));
  } else {
    for (int b = 0; b < w; ++b) dst[b] = src[b];
  }
}


int device_sm_count();
void count_launches(int k);

// Per-device host caches. Function attributes (dynamic shared memory opt-in)
// and occupancy belong to a device context, so a value cached for cuda:0
// must not be reused on cuda:1: each cache has one slot per device ordinal
// (0 = not computed yet). Benign races: every writer stores the same value.
constexpr int kMaxDevices = 64;
int current_device();  // cudaGetDevice(); -1 on error or past kMaxDevices (no caching)
template <typename F>
inline int per_device(int (&slot)[kMaxDevices], F compute) {
  const int d = current_device();
  if (d >= 0 && slot[d] != 0) return slot[d];
  const int v = compute();
  if (d >= 0) slot[d] = v;
  return v;
}

}  // namespace rl
