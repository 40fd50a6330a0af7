// keypack.cuh — order-preserving key transforms shared by the sort
// (radix_sort.cu) and the bucket join (bucket_join.cu).
#pragma once

#include <cstdint>

namespace rl {
namespace radix {

// Key transform (self-inverse): int64 ascending u = x ^ 2^63; descending
// u = ~x ^ 2^63 (the reference's np.invert, tensorpath.py:215).
__device__ __forceinline__ uint64_t xform(uint64_t x, int desc) {
  return (desc ? ~x : x) ^ 0x8000000000000000ull;
}

// Key normalisation of the scatter path: the key bits that do not vary
// (estimated from a sample at the start of the chunk counts, checked by them
// against every key) are squeezed out — the varying bits, up to two runs of
// them, are packed left-aligned, high run first — so the sub-buckets are the
// top 16 VARYING bits (row-id-like keys, composite keys with a constant
// middle, keys with constant low bits). Order is unchanged: every key shares
// the dropped bits. The local phase puts the bits back when it writes keys.
// Pack code: bit 28 valid, then (lo, len) of the high run and of the low run
// (len 0: one run), 7 bits each; 0 = keys used as they are.
__device__ __forceinline__ uint64_t low_mask(uint32_t len) { return len >= 64 ? ~0ull : (1ull << len) - 1; }
__device__ __forceinline__ uint32_t pack_code_of(uint64_t vv) {
  if (vv == 0) return 0u;
  const uint32_t hi1 = 63u - uint32_t(__clzll((long long)vv));
  const uint64_t z1 = ~vv & low_mask(hi1);  // zero bits below the top varying bit
  const uint32_t lo1 = z1 ? 64u - uint32_t(__clzll((long long)z1)) : 0u;
  const uint32_t len1 = hi1 - lo1 + 1;
  const uint64_t rest = vv & low_mask(lo1);
  uint32_t lo2 = 0, len2 = 0;
  if (rest) {
    const uint32_t hi2 = 63u - uint32_t(__clzll((long long)rest));
    const uint64_t z2 = ~rest & low_mask(hi2);
    lo2 = z2 ? 64u - uint32_t(__clzll((long long)z2)) : 0u;
    len2 = hi2 - lo2 + 1;
    if (rest & low_mask(lo2)) return 0u;  // three or more runs: keys used as they are
  }
  if (len1 + len2 >= 64) return 0u;       // every bit varies
  return (1u << 28) | (lo1 << 21) | (len1 << 14) | (lo2 << 7) | len2;
}
__device__ __forceinline__ uint64_t pack_mask(uint32_t c) {
  if (!(c >> 28)) return ~0ull;
  const uint32_t lo1 = c >> 21 & 127, len1 = c >> 14 & 127, lo2 = c >> 7 & 127, len2 = c & 127;
  return (low_mask(len1) << lo1) | (len2 ? low_mask(len2) << lo2 : 0ull);
}
__device__ __forceinline__ uint64_t pack_key(uint64_t u, uint32_t c) {
  if (!(c >> 28)) return u;
  const uint32_t lo1 = c >> 21 & 127, len1 = c >> 14 & 127, lo2 = c >> 7 & 127, len2 = c & 127;
  const uint64_t r = (((u >> lo1) & low_mask(len1)) << len2) | (len2 ? (u >> lo2) & low_mask(len2) : 0ull);
  return r << (64 - len1 - len2);
}
__device__ __forceinline__ uint64_t unpack_key(uint64_t v, uint32_t c, uint64_t constbits) {
  if (!(c >> 28)) return v;
  const uint32_t lo1 = c >> 21 & 127, len1 = c >> 14 & 127, lo2 = c >> 7 & 127, len2 = c & 127;
  const uint64_t r = v >> (64 - len1 - len2);
  return constbits | ((r >> len2) << lo1) | (len2 ? (r & low_mask(len2)) << lo2 : 0ull);
}
// 0: keys as they are; 1: one run ending at bit 0 — a plain left shift; 2: the general pack.
__device__ __forceinline__ int pack_mode(uint32_t c) {
  if (!(c >> 28)) return 0;
  return ((c & 127) == 0 && (c >> 21 & 127) == 0) ? 1 : 2;
}
__device__ __forceinline__ uint32_t pack_shift(uint32_t c) { return 64u - (c >> 14 & 127); }  // mode 1

}  // namespace radix
}  // namespace rl
