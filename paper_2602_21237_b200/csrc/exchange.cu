// exchange.cu — the multi-GPU exchange step fused with the partition gather.
//
// After a stable partition (rl_hash_partition / rl_range_partition: row ids
// grouped by destination, counts per destination) the rows of every
// destination d must land in d's receive buffer, after the rows the lower
// ranks send to d, in partition order — exactly what an NCCL all-to-all-v
// of the gathered columns delivers. Here one
// kernel does the gather and the transfer: each thread reads one
// partitioned row from local HBM and stores it straight into the
// destination's receive buffer through its peer pointer (NVLink / NVSwitch
// P2P stores into symmetric memory; the local buffer for the own rank),
// together with its local row id. No send staging buffer, no second pass.
//
// The host side (dist.PeerExchange) exchanges the P x P counts first, so
// each source knows its block offset in every destination, and brackets
// the push with symmetric-memory barriers.
#include <algorithm>

#include "common.cuh"

namespace rl {
namespace exchange {

constexpr int kThreads = 256;
constexpr int kMaxParts = 64;
constexpr int kMaxCols = 8;

struct PushArgs {
  const uint32_t* rows;  // [n] local row ids grouped by destination (partition order)
  int64_t n;
  int parts;
  int ncols;
  const void* src[kMaxCols];
  int width[kMaxCols];
  const uint64_t* dest_bases;    // [parts][ncols + 1] base address of every column region (+ row ids) per dest
  const int64_t* dest_starts;    // [parts + 1] partition boundaries (device)
  const int64_t* dest_offsets;   // [parts] this source's first row in every destination's buffer
};

__global__ void __launch_bounds__(kThreads) push_kernel(PushArgs a) {
  __shared__ int64_t starts[kMaxParts + 1];
  __shared__ int64_t offs[kMaxParts];
  __shared__ uint64_t bases[kMaxParts * (kMaxCols + 1)];
  const int tid = threadIdx.x;
  for (int i = tid; i <= a.parts; i += kThreads) starts[i] = a.dest_starts[i];
  for (int i = tid; i < a.parts; i += kThreads) offs[i] = a.dest_offsets[i];
  for (int i = tid; i < a.parts * (a.ncols + 1); i += kThreads) bases[i] = a.dest_bases[i];
  __syncthreads();
  for (int64_t i = int64_t(blockIdx.x) * kThreads + tid; i < a.n; i += int64_t(gridDim.x) * kThreads) {
    int d = 0;
    while (d + 1 < a.parts && starts[d + 1] <= i) ++d;  // parts <= 64, rows of one d are contiguous
    const uint32_t row = __ldg(a.rows + i);
    const uint64_t o = uint64_t(offs[d] + (i - starts[d]));
    const uint64_t* b = bases + d * (a.ncols + 1);
    for (int c = 0; c < a.ncols; ++c) {
      const int w = a.width[c];
      copy_row(static_cast<const uint8_t*>(a.src[c]) + uint64_t(row) * w, reinterpret_cast<uint8_t*>(b[c]) + o * w, w);
    }
    reinterpret_cast<uint32_t*>(b[a.ncols])[o] = row;
  }
}

int push_rows(const uint32_t* rows, int64_t n, int parts, const int64_t* dest_starts, const rl_column* columns,
              int n_columns, const uint64_t* dest_bases, const int64_t* dest_offsets, cudaStream_t stream) {
  if (n < 0 || parts < 1 || parts > kMaxParts || n_columns < 0 || n_columns > kMaxCols) return RL_ERR_BAD_ARG;
  if (n > 0 && (!rows || !dest_starts || !dest_bases || !dest_offsets)) return RL_ERR_BAD_ARG;
  if (n_columns > 0 && !columns) return RL_ERR_BAD_ARG;
  if (n > RL_MAX_ROWS) return RL_ERR_TOO_MANY_ROWS;
  if (n == 0) return RL_OK;
  PushArgs a;
  a.rows = rows;
  a.n = n;
  a.parts = parts;
  a.ncols = n_columns;
  for (int c = 0; c < n_columns; ++c) {
    if (columns[c].width <= 0 || !columns[c].src) return RL_ERR_BAD_ARG;
    a.src[c] = columns[c].src;
    a.width[c] = columns[c].width;
  }
  a.dest_bases = dest_bases;
  a.dest_starts = dest_starts;
  a.dest_offsets = dest_offsets;
  const int grid = int(std::min<int64_t>((n + kThreads - 1) / kThreads, int64_t(device_sm_count()) * 8));
  push_kernel<<<grid, kThreads, 0, stream>>>(a);
  count_launches(1);
  return rl_cuda_status(cudaGetLastError());
}

}  // namespace exchange
}  // namespace rl

extern "C" {

RL_API int rl_push_rows(const uint32_t* rows, int64_t n, int32_t parts, const int64_t* dest_starts,
                        const rl_column* columns, int32_t n_columns, const uint64_t* dest_bases,
                        const int64_t* dest_offsets, void* stream) {
  return rl::exchange::push_rows(rows, n, parts, dest_starts, columns, n_columns, dest_bases, dest_offsets,
                                 static_cast<cudaStream_t>(stream));
}

}  // extern "C"
