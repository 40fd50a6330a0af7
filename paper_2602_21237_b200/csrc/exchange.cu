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
constexpr int kMaxParts = RL_PUSH_MAX_PARTS;
constexpr int kMaxCols = RL_PUSH_MAX_COLUMNS;

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
  int64_t gid_base;              // this rank's first global row id (GID mode)
};

template <bool GID>  // GID: the last region receives int64 global row ids (gid_base + row), else u32 rows
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
    if constexpr (GID) reinterpret_cast<int64_t*>(b[a.ncols])[o] = a.gid_base + int64_t(row);
    else reinterpret_cast<uint32_t*>(b[a.ncols])[o] = row;
  }
}

int push_rows(const uint32_t* rows, int64_t n, int parts, const int64_t* dest_starts, const rl_column* columns,
              int n_columns, const uint64_t* dest_bases, const int64_t* dest_offsets, cudaStream_t stream,
              bool gid = false, int64_t gid_base = 0) {
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
  a.gid_base = gid_base;
  const int grid = int(std::min<int64_t>((n + kThreads - 1) / kThreads, int64_t(device_sm_count()) * 8));
  if (gid) push_kernel<true><<<grid, kThreads, 0, stream>>>(a);
  else push_kernel<false><<<grid, kThreads, 0, stream>>>(a);
  count_launches(1);
  return rl_cuda_status(cudaGetLastError());
}

// ---------------------------------------------------------------- splitters
// Regular samples of this rank's keys, packed as the all-gather expects:
// [0][i] key in sort order (complemented when descending), [1][i] global row
// id, [2][i] 1 = a real sample (ranks with fewer rows than samples pad).
__global__ void sample_kernel(const int64_t* keys, int64_t n, int per_rank, int64_t gid_base, int descending,
                              int64_t* pack) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= per_rank) return;
  const int64_t m = n < per_rank ? n : per_rank;
  int64_t idx = (int64_t(i) * (n > 0 ? n : 1)) / (m > 0 ? m : 1);
  if (idx > n - 1) idx = n > 0 ? n - 1 : 0;
  const int64_t k = n > 0 ? keys[idx] : 0;
  pack[i] = descending ? ~k : k;
  pack[per_rank + i] = idx + gid_base;
  pack[2 * per_rank + i] = i < m ? 1 : 0;
}

// All ranks' samples (P blocks of [3][per_rank]) → the P-1 splitters: every
// sample's rank in the composite (real first, key, global id) order is counted
// in shared memory (S <= 2048), and the samples of rank j * cnt / P are kept.
constexpr int kSplitThreads = 1024;
constexpr int kMaxSamples = 2048;  // P x per_rank (static shared memory)
__global__ void __launch_bounds__(kSplitThreads) pick_kernel(const int64_t* all, int parts, int per_rank,
                                                             int descending, int64_t* out_keys, int64_t* out_gids) {
  __shared__ int64_t sk[kMaxSamples];
  __shared__ int64_t sg[kMaxSamples];
  __shared__ uint8_t sv[kMaxSamples];
  __shared__ int cnt_s;
  const int S = parts * per_rank, tid = threadIdx.x;
  if (tid == 0) cnt_s = 0;
  __syncthreads();
  int mine = 0;
  for (int i = tid; i < S; i += kSplitThreads) {
    const int r = i / per_rank, j = i % per_rank;
    const int64_t* blk = all + int64_t(r) * 3 * per_rank;
    sk[i] = blk[j];
    sg[i] = blk[per_rank + j];
    sv[i] = blk[2 * per_rank + j] != 0;
    mine += sv[i];
  }
  atomicAdd(&cnt_s, mine);
  __syncthreads();
  const int cnt = cnt_s;
  auto less = [&](int a, int b) {  // composite order: real samples first, then (key, gid)
    if (sv[a] != sv[b]) return sv[a] > sv[b];
    if (sk[a] != sk[b]) return sk[a] < sk[b];
    return sg[a] < sg[b];
  };
  for (int i = tid; i < S; i += kSplitThreads) {
    int rank = 0;
    for (int o = 0; o < S; ++o) rank += less(o, i) ? 1 : 0;
    for (int j = 1; j < parts; ++j) {
      int64_t pick = int64_t(j) * cnt / parts;
      if (pick > cnt - 1) pick = cnt > 0 ? cnt - 1 : 0;
      if (rank == pick) {
        out_keys[j - 1] = descending ? ~sk[i] : sk[i];
        out_gids[j - 1] = sg[i];
      }
    }
  }
}

// Global row ids of received rows: sender's base + its local row id (u32).
struct GidArgs {
  int64_t starts[kMaxParts + 1];
  int64_t bases[kMaxParts];
  int parts;
};
__global__ void gid_kernel(const uint32_t* rows, int64_t total, GidArgs g, int64_t* out) {
  for (int64_t i = int64_t(blockIdx.x) * kThreads + threadIdx.x; i < total; i += int64_t(gridDim.x) * kThreads) {
    int d = 0;
    while (d + 1 < g.parts && g.starts[d + 1] <= i) ++d;
    out[i] = g.bases[d] + int64_t(rows[i]);
  }
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

RL_API int rl_push_rows_gid(const uint32_t* rows, int64_t n, int32_t parts, const int64_t* dest_starts,
                            const rl_column* columns, int32_t n_columns, const uint64_t* dest_bases,
                            const int64_t* dest_offsets, int64_t gid_base, void* stream) {
  return rl::exchange::push_rows(rows, n, parts, dest_starts, columns, n_columns, dest_bases, dest_offsets,
                                 static_cast<cudaStream_t>(stream), true, gid_base);
}

RL_API int rl_sample_keys(const int64_t* keys, int64_t n, int32_t per_rank, int64_t gid_base, int32_t descending,
                          int64_t* pack, void* stream) {
  if (n < 0 || per_rank < 1 || !pack || (n > 0 && !keys)) return RL_ERR_BAD_ARG;
  rl::exchange::sample_kernel<<<(per_rank + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      keys, n, per_rank, gid_base, descending, pack);
  rl::count_launches(1);
  return rl::rl_cuda_status(cudaGetLastError());
}

RL_API int rl_pick_splitters(const int64_t* gathered, int32_t parts, int32_t per_rank, int32_t descending,
                             int64_t* split_keys, int64_t* split_gids, void* stream) {
  if (parts < 1 || per_rank < 1 || int64_t(parts) * per_rank > rl::exchange::kMaxSamples || !gathered)
    return RL_ERR_BAD_ARG;
  if (parts == 1) return RL_OK;
  if (!split_keys || !split_gids) return RL_ERR_BAD_ARG;
  rl::exchange::pick_kernel<<<1, rl::exchange::kSplitThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      gathered, parts, per_rank, descending, split_keys, split_gids);
  rl::count_launches(1);
  return rl::rl_cuda_status(cudaGetLastError());
}

RL_API int rl_global_ids(const uint32_t* rows, int64_t total, int32_t parts, const int64_t* recv_counts,
                         const int64_t* bases, int64_t* out, void* stream) {
  if (total < 0 || parts < 1 || parts > rl::exchange::kMaxParts || !recv_counts || !bases) return RL_ERR_BAD_ARG;
  if (total == 0) return RL_OK;
  if (!rows || !out) return RL_ERR_BAD_ARG;
  rl::exchange::GidArgs g;
  g.parts = parts;
  g.starts[0] = 0;
  for (int d = 0; d < parts; ++d) {
    g.starts[d + 1] = g.starts[d] + recv_counts[d];
    g.bases[d] = bases[d];
  }
  if (g.starts[parts] != total) return RL_ERR_BAD_ARG;
  const int grid = int(std::min<int64_t>((total + rl::exchange::kThreads - 1) / rl::exchange::kThreads,
                                         int64_t(rl::device_sm_count()) * 8));
  rl::exchange::gid_kernel<<<grid, rl::exchange::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(rows, total, g, out);
  rl::count_launches(1);
  return rl::rl_cuda_status(cudaGetLastError());
}

}  // extern "C"
