// bjoin.cuh — the interface between the sort's scatter path (radix_sort.cu)
// and the bucket join (bucket_join.cu): both join sides partitioned into the
// same 65536 sub-buckets of one joint key packing, rows as packed words.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace rl {
namespace radix {

constexpr int kBjSubBuckets = 1 << 16;  // sub-buckets: top 16 bits of the packed key
constexpr int kBjCap = 2560;            // rows of one side in one sub-bucket at most (kLocalCap)

constexpr int kBjMaxCarryCols = 4;
constexpr int kBjMaxCarryWords = 2;  // <= 16 payload bytes a row carried through the passes

// Columns of one side carried with its rows (packed at byte offsets into
// `words` u64 words per row), so the emit reads them beside the row instead
// of gathering them by row id.
struct BjCarry {
  int n = 0;
  const uint8_t* src[kBjMaxCarryCols] = {};
  int width[kBjMaxCarryCols] = {};
  int off[kBjMaxCarryCols] = {};
  int words = 0;
};

struct BjSide {
  const uint64_t* rows;     // [n] packed words (key bits << 32 | row id), grouped by sub-bucket
  const uint64_t* pay;      // [n * words] carried payload words, parallel to rows (words > 0)
  int words;
  const uint32_t* sub_off;  // sub-bucket starts: [2^16 + 1] (two levels) or [2^24 + 1] (three)
  uint32_t* flags;          // [0] != 0: fall back; [6] the joint pack code
  int64_t n;
  int levels;               // 2: sub-buckets = top 16 packed bits; 3: top 24
};

// Two levels up to ~0.85 x 65536 x kBjCap rows a side, three above (both sides alike).
int bj_levels(int64_t nl, int64_t nr);
size_t bj_side_workspace_bytes(int64_t n, int words, int levels);
int bj_partition(const int64_t* lkeys, int64_t nl, const int64_t* rkeys, int64_t nr, const BjCarry& lcarry,
                 const BjCarry& rcarry, void* ws_l, size_t ws_l_bytes, void* ws_r, size_t ws_r_bytes,
                 cudaStream_t stream, BjSide* left, BjSide* right);

}  // namespace radix
}  // namespace rl
