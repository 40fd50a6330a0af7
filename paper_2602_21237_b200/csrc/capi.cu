// capi.cu — extern "C" entry points of librelab_b200.so (include/relab_b200.h).
// Thin argument plumbing only; the kernels live in radix_sort.cu,
// key_axis.cu and expand.cu.
#include <atomic>
#include <cstdio>

#include "common.cuh"

namespace rl {
namespace radix {
size_t workspace_bytes(int64_t n);
size_t carry_workspace_bytes(int64_t n, int words);
int sort_axis_carry(const int64_t* keys, int64_t n, int descending, int64_t* sorted_keys_out, uint32_t* perm_out,
                    const rl_column* columns, int n_columns, void* ws, size_t ws_bytes, cudaStream_t stream);
int sort_axis(const void* col, int col_kind, int width, int word, int descending, const uint32_t* perm_in,
              int64_t n, int64_t* sorted_keys_out, uint32_t* perm_out, void* ws, size_t ws_bytes,
              cudaStream_t stream, void* const* events, unsigned long long* stamps, const rl_column* columns,
              int n_columns);
size_t partition_workspace_bytes(int64_t n);
int hash_partition_perm(const int64_t* keys, int64_t n, int parts, uint64_t seed, uint32_t* perm_out,
                        int64_t* counts_out, void* ws, size_t ws_bytes, cudaStream_t stream);
int range_partition_perm(const int64_t* keys, int64_t n, int64_t gid_base, const int64_t* split_keys,
                         const int64_t* split_gids, int nsplit, int descending, uint32_t* perm_out,
                         int64_t* counts_out, void* ws, size_t ws_bytes, cudaStream_t stream);
}  // namespace radix
namespace keyaxis {
size_t run_bounds_workspace_bytes(int64_t n);
int run_bounds(const int64_t* sk, int64_t n, int64_t* key_values, uint32_t* offsets, int64_t* d_out, void* ws,
               size_t ws_bytes, cudaStream_t stream);
size_t align_workspace_bytes(int64_t cap);
int key_axis_align(const int64_t* lkeys, const uint32_t* loff, const int64_t* d_left, int64_t cap,
                   const int64_t* rkeys, const uint32_t* roff, const int64_t* d_right, int64_t* matched_keys,
                   uint32_t* ls, uint32_t* lc, uint32_t* rs, uint32_t* rc, uint64_t* pair_offsets,
                   int64_t* m_out, uint64_t* total_out, void* ws, size_t ws_bytes, cudaStream_t stream);
}  // namespace keyaxis
namespace expand {
int join_expand(const int64_t* matched_keys, const uint32_t* ls, const uint32_t* rs, const uint32_t* rc,
                const uint64_t* offs, int64_t m, const uint32_t* lpos, const uint32_t* rpos, uint64_t out_begin,
                uint64_t out_end, uint32_t* lrows_out, uint32_t* rrows_out, const rl_column* columns,
                int n_columns, cudaStream_t stream);
int pair_checksum(const uint32_t* ls, const uint32_t* rs, const uint32_t* rc, const uint64_t* offs, int64_t m,
                  const uint32_t* lpos, const uint32_t* rpos, uint64_t out_begin, uint64_t out_end,
                  uint64_t* sum_out, cudaStream_t stream);
int gather_rows(const uint32_t* rows, int64_t m, const rl_column* columns, int n_columns, cudaStream_t stream);
int widen_u32(const uint32_t* src, int64_t n, int64_t* dst, cudaStream_t stream);
int gather_split16(const uint32_t* rows, int64_t m, const void* src, void* lo, void* hi, cudaStream_t stream);
}  // namespace expand

static std::atomic<int64_t> g_launches{0};
void count_launches(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return dev >= 0 && dev < kMaxDevices ? dev : -1;
}

int device_sm_count() {
  static int cache[kMaxDevices] = {};
  return per_device(cache, [] {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
      cudaGetLastError();
      return 148;
    }
    return sms;
  });
}

}  // namespace rl

static inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" {

int rl_abi_version(void) { return RL_ABI_VERSION; }

const char* rl_strerror(int status) {
  switch (status) {
    case RL_OK: return "ok";
    case RL_ERR_BAD_ARG: return "invalid argument";
    case RL_ERR_OUTPUT_TOO_LARGE: return "join output exceeds the row cap";
    case RL_ERR_WORKSPACE: return "workspace too small or misaligned";
    case RL_ERR_TOO_MANY_ROWS: return "more rows than uint32 row ids can address";
    case RL_ERR_IO: return "file read or write failed";
    default: break;
  }
  if (status >= RL_ERR_CUDA) return cudaGetErrorString(static_cast<cudaError_t>(status - RL_ERR_CUDA));
  return "unknown status";
}

int rl_device_sm_count(void) { return rl::device_sm_count(); }

int64_t rl_launch_count(void) { return rl::g_launches.load(std::memory_order_relaxed); }

size_t rl_sort_workspace_bytes(int64_t n) { return rl::radix::workspace_bytes(n); }

int rl_sort_axis(const void* col, int32_t col_kind, int32_t width, int32_t word, int32_t descending,
                 const uint32_t* perm_in, int64_t n, int64_t* sorted_keys_out, uint32_t* perm_out, void* ws,
                 size_t ws_bytes, void* stream) {
  return rl::radix::sort_axis(col, col_kind, width, word, descending, perm_in, n, sorted_keys_out, perm_out, ws,
                              ws_bytes, as_stream(stream), nullptr, nullptr, nullptr, 0);
}

int rl_sort_axis_gather(const void* col, int32_t col_kind, int32_t width, int32_t word, int32_t descending,
                        const uint32_t* perm_in, int64_t n, int64_t* sorted_keys_out, uint32_t* perm_out,
                        const rl_column* columns, int32_t n_columns, void* ws, size_t ws_bytes, void* stream) {
  return rl::radix::sort_axis(col, col_kind, width, word, descending, perm_in, n, sorted_keys_out, perm_out, ws,
                              ws_bytes, as_stream(stream), nullptr, nullptr, columns, n_columns);
}

int rl_sort_axis_profiled(const void* col, int32_t col_kind, int32_t width, int32_t word, int32_t descending,
                          const uint32_t* perm_in, int64_t n, int64_t* sorted_keys_out, uint32_t* perm_out,
                          const rl_column* columns, int32_t n_columns, void* ws, size_t ws_bytes, void* stream,
                          void* const* events, unsigned long long* stamps_dev) {
  if (events == nullptr) return RL_ERR_BAD_ARG;
  return rl::radix::sort_axis(col, col_kind, width, word, descending, perm_in, n, sorted_keys_out, perm_out, ws,
                              ws_bytes, as_stream(stream), events, stamps_dev, columns, n_columns);
}

size_t rl_sort_carry_workspace_bytes(int64_t n, int32_t carry_bytes) {
  return rl::radix::carry_workspace_bytes(n, carry_bytes > 0 && carry_bytes <= 16 ? (carry_bytes + 7) / 8 : 0);
}

int rl_sort_axis_carry(const int64_t* keys, int64_t n, int32_t descending, int64_t* sorted_keys_out,
                       uint32_t* perm_out, const rl_column* columns, int32_t n_columns, void* ws, size_t ws_bytes,
                       void* stream) {
  return rl::radix::sort_axis_carry(keys, n, descending, sorted_keys_out, perm_out, columns, n_columns, ws, ws_bytes,
                                    as_stream(stream));
}

size_t rl_run_bounds_workspace_bytes(int64_t n) { return rl::keyaxis::run_bounds_workspace_bytes(n); }

int rl_run_bounds(const int64_t* sorted_keys, int64_t n, int64_t* key_values, uint32_t* offsets, int64_t* d_out,
                  void* ws, size_t ws_bytes, void* stream) {
  return rl::keyaxis::run_bounds(sorted_keys, n, key_values, offsets, d_out, ws, ws_bytes, as_stream(stream));
}

size_t rl_align_workspace_bytes(int64_t d_left_cap) { return rl::keyaxis::align_workspace_bytes(d_left_cap); }

int rl_key_axis_align(const int64_t* left_keys, const uint32_t* left_offsets, const int64_t* d_left,
                      int64_t d_left_cap, const int64_t* right_keys, const uint32_t* right_offsets,
                      const int64_t* d_right, int64_t* matched_keys, uint32_t* left_starts, uint32_t* left_counts,
                      uint32_t* right_starts, uint32_t* right_counts, uint64_t* pair_offsets, int64_t* m_out,
                      uint64_t* total_out, void* ws, size_t ws_bytes, void* stream) {
  return rl::keyaxis::key_axis_align(left_keys, left_offsets, d_left, d_left_cap, right_keys, right_offsets,
                                     d_right, matched_keys, left_starts, left_counts, right_starts, right_counts,
                                     pair_offsets, m_out, total_out, ws, ws_bytes, as_stream(stream));
}

int rl_join_expand(const int64_t* matched_keys, const uint32_t* left_starts, const uint32_t* right_starts,
                   const uint32_t* right_counts, const uint64_t* pair_offsets, int64_t m,
                   const uint32_t* left_positions, const uint32_t* right_positions, uint64_t out_begin,
                   uint64_t out_end, uint32_t* left_rows_out, uint32_t* right_rows_out, const rl_column* columns,
                   int32_t n_columns, void* stream) {
  return rl::expand::join_expand(matched_keys, left_starts, right_starts, right_counts, pair_offsets, m,
                                 left_positions, right_positions, out_begin, out_end, left_rows_out,
                                 right_rows_out, columns, n_columns, as_stream(stream));
}

int rl_join_pair_checksum(const uint32_t* left_starts, const uint32_t* right_starts, const uint32_t* right_counts,
                          const uint64_t* pair_offsets, int64_t m, const uint32_t* left_positions,
                          const uint32_t* right_positions, uint64_t out_begin, uint64_t out_end, uint64_t* sum_out,
                          void* stream) {
  return rl::expand::pair_checksum(left_starts, right_starts, right_counts, pair_offsets, m, left_positions,
                                   right_positions, out_begin, out_end, sum_out, as_stream(stream));
}

int rl_gather_rows(const uint32_t* rows, int64_t m, const rl_column* columns, int32_t n_columns, void* stream) {
  return rl::expand::gather_rows(rows, m, columns, n_columns, as_stream(stream));
}

int rl_gather_rows_split16(const uint32_t* rows, int64_t m, const void* src, void* dst_lo, void* dst_hi,
                           void* stream) {
  return rl::expand::gather_split16(rows, m, src, dst_lo, dst_hi, as_stream(stream));
}

int rl_widen_u32(const uint32_t* src, int64_t n, int64_t* dst, void* stream) {
  return rl::expand::widen_u32(src, n, dst, as_stream(stream));
}

size_t rl_partition_workspace_bytes(int64_t n, int32_t parts) {
  (void)parts;
  return rl::radix::partition_workspace_bytes(n);
}

int rl_hash_partition(const int64_t* keys, int64_t n, int32_t parts, uint64_t seed, const rl_column* columns,
                      int32_t n_columns, uint32_t* row_ids_out, int64_t* counts_out, void* ws, size_t ws_bytes,
                      void* stream) {
  int st = rl::radix::hash_partition_perm(keys, n, parts, seed, row_ids_out, counts_out, ws, ws_bytes,
                                          as_stream(stream));
  if (st != RL_OK) return st;
  return rl::expand::gather_rows(row_ids_out, n, columns, n_columns, as_stream(stream));
}

int rl_range_partition(const int64_t* keys, int64_t n, int64_t gid_base, const int64_t* split_keys,
                       const int64_t* split_gids, int32_t n_splitters, int32_t descending, const rl_column* columns,
                       int32_t n_columns, uint32_t* row_ids_out, int64_t* counts_out, void* ws, size_t ws_bytes,
                       void* stream) {
  int st = rl::radix::range_partition_perm(keys, n, gid_base, split_keys, split_gids, n_splitters, descending,
                                           row_ids_out, counts_out, ws, ws_bytes, as_stream(stream));
  if (st != RL_OK) return st;
  return rl::expand::gather_rows(row_ids_out, n, columns, n_columns, as_stream(stream));
}

}  // extern "C"
