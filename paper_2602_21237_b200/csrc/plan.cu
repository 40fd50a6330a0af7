// plan.cu — one entry point for everything a join needs before its output
// size is known: index both key columns (K1+K2+K3) and align them (K4+K5).
//
// This is tensorpath.py:78-93 (to_tensor) twice + tensorpath.py:109-161
// (key_axis_align + sizing) as ONE C call over ONE caller workspace: the
// host issues a handful of launches back to back and allocates nothing, so
// a 1M x 1M join is not paced by per-launch host work. The plan arrays stay
// in the workspace for rl_join_expand.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace rl {
namespace radix {
size_t workspace_bytes(int64_t n);
int sort_axis(const void* col, int col_kind, int width, int word, int descending, const uint32_t* perm_in,
              int64_t n, int64_t* sorted_keys_out, uint32_t* perm_out, void* ws, size_t ws_bytes,
              cudaStream_t stream, void* const* events, unsigned long long* stamps, const rl_column* columns,
              int n_columns);
int sort_axis_capped(const void* col, int col_kind, int width, int word, int descending, const uint32_t* perm_in,
                     int64_t n, int64_t* sorted_keys_out, uint32_t* perm_out, void* ws, size_t ws_bytes,
                     cudaStream_t stream, void* const* events, unsigned long long* stamps, const rl_column* columns,
                     int n_columns, int max_ctas);
int sort_grid_capacity();
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
namespace plan {

// The key axes of both sides (kept for the expansion).
template <typename C>
static void carve_plan(C& c, int64_t nl, int64_t nr, rl_join_plan* p) {
  auto take64 = [&](size_t k) { return c.template take<int64_t>(k); };
  auto take32 = [&](size_t k) { return c.template take<uint32_t>(k); };
  p->scalars = take64(4);
  p->left_positions = take32(size_t(std::max<int64_t>(nl, 1)));
  p->left_key_values = take64(size_t(std::max<int64_t>(nl, 1)));
  p->left_offsets = take32(size_t(nl + 1));
  p->right_positions = take32(size_t(std::max<int64_t>(nr, 1)));
  p->right_key_values = take64(size_t(std::max<int64_t>(nr, 1)));
  p->right_offsets = take32(size_t(nr + 1));
}

// The alignment arrays (min(nl, nr) capacity, 32 bytes a matched key): carved
// in the scratch the index sorts used — free once both axes exist — so the
// plan's footprint at 1e9 x 1e9 is the axes + the larger of the two scratches
// (~65 GB), not their sum (~97 GB).
template <typename C>
static void carve_alignment(C& c, int64_t nl, int64_t nr, rl_join_plan* p) {
  const int64_t alloc = std::max<int64_t>(std::min(nl, nr), 1);
  auto take64 = [&](size_t k) { return c.template take<int64_t>(k); };
  auto take32 = [&](size_t k) { return c.template take<uint32_t>(k); };
  p->matched_keys = take64(size_t(alloc));
  p->left_starts = take32(size_t(alloc));
  p->left_counts = take32(size_t(alloc));
  p->right_starts = take32(size_t(alloc));
  p->right_counts = take32(size_t(alloc));
  p->pair_offsets = reinterpret_cast<uint64_t*>(take64(size_t(alloc + 1)));
}

struct Sizer {  // CarveSize with the pointer-returning interface of Carve
  size_t used = 0;
  template <typename T>
  T* take(size_t count) {
    used = align_up(used, 256) + count * sizeof(T);
    return nullptr;
  }
};

// Both sides are indexed concurrently (two streams, each sort on half the
// co-resident grid) when they are small enough to be latency-bound; each
// side then needs its own scratch.
constexpr int64_t kConcurrentMaxRows = int64_t(16) << 20;
static bool concurrent_sides(int64_t nl, int64_t nr) {
  static const bool serial = [] {  // RL_PLAN_SERIAL=1: one side after the other (A/B measurements)
    const char* v = getenv("RL_PLAN_SERIAL");
    return v && v[0] && v[0] != '0';
  }();
  return !serial && nl > 0 && nr > 0 && std::max(nl, nr) <= kConcurrentMaxRows;
}

static size_t side_scratch_bytes(int64_t n) {
  size_t s = align_up(size_t(std::max<int64_t>(n, 1)) * 8, 256);  // sorted keys
  size_t inner = std::max(radix::workspace_bytes(n), keyaxis::run_bounds_workspace_bytes(n));
  return s + align_up(inner, 256) + 256;
}

static size_t alignment_bytes(int64_t nl, int64_t nr) {
  Sizer z;
  rl_join_plan p;
  carve_alignment(z, nl, nr, &p);
  return align_up(z.used, 256);
}

static size_t scratch_bytes(int64_t nl, int64_t nr) {
  const int64_t n = std::max(nl, nr);
  const size_t sides = concurrent_sides(nl, nr) ? 2 * side_scratch_bytes(n) : side_scratch_bytes(n);
  const size_t align = alignment_bytes(nl, nr) + align_up(keyaxis::align_workspace_bytes(nl), 256) + 256;
  return std::max(sides, align);
}

size_t workspace_bytes(int64_t nl, int64_t nr) {
  Sizer z;
  rl_join_plan p;
  carve_plan(z, nl, nr, &p);
  return align_up(z.used, 256) + scratch_bytes(nl, nr) + 256;
}

// Per-host-thread auxiliary stream + fork/join events (created once).
struct Aux {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  int device = -1;
};
static Aux* aux_for_current_device() {
  thread_local Aux aux;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  if (aux.device != dev) {
    if (cudaStreamCreateWithFlags(&aux.stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&aux.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&aux.join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    aux.device = dev;
  }
  return &aux;
}

int build(const int64_t* lkeys, int64_t nl, const int64_t* rkeys, int64_t nr, void* ws, size_t ws_bytes,
          rl_join_plan* p, cudaStream_t stream) {
  if (nl < 0 || nr < 0 || !p || (nl > 0 && !lkeys) || (nr > 0 && !rkeys)) return RL_ERR_BAD_ARG;
  if (reinterpret_cast<uintptr_t>(ws) % 256 != 0) return RL_ERR_WORKSPACE;
  if (ws_bytes < workspace_bytes(nl, nr)) return RL_ERR_WORKSPACE;
  Carve c{static_cast<char*>(ws), ws_bytes};
  carve_plan(c, nl, nr, p);
  if (!c.ok) return RL_ERR_WORKSPACE;
  char* scratch = c.base + align_up(c.used, 256);
  const size_t scratch_cap = ws_bytes - align_up(c.used, 256);
  Aux* aux = concurrent_sides(nl, nr) ? aux_for_current_device() : nullptr;
  const int half = aux ? std::max(1, radix::sort_grid_capacity() / 2) : 0;
  const size_t per_side = aux ? scratch_cap / 2 / 256 * 256 : scratch_cap;

  struct Side {
    const int64_t* keys;
    int64_t n;
    uint32_t* pos;
    int64_t* kv;
    uint32_t* off;
    int64_t* d;
  } sides[2] = {{lkeys, nl, p->left_positions, p->left_key_values, p->left_offsets, p->scalars + 0},
                {rkeys, nr, p->right_positions, p->right_key_values, p->right_offsets, p->scalars + 1}};
  if (aux) {  // right side on the auxiliary stream, after everything already queued on `stream`
    cudaError_t e = cudaEventRecord(aux->fork, stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(aux->stream, aux->fork, 0);
    if (e != cudaSuccess) return rl_cuda_status(e);
  }
  for (int i = 0; i < 2; ++i) {
    const Side& sd = sides[i];
    cudaStream_t st_i = (aux && i == 1) ? aux->stream : stream;
    char* base = scratch + (aux ? i * per_side : 0);
    int64_t* sorted = reinterpret_cast<int64_t*>(base);
    const size_t sorted_bytes = align_up(size_t(std::max(std::max<int64_t>(nl, nr), int64_t(1))) * 8, 256);
    void* inner = base + sorted_bytes;
    const size_t inner_cap = per_side - sorted_bytes;
    if (sd.n > 0) {
      int st = radix::sort_axis_capped(sd.keys, RL_COL_INT64, 8, 0, 0, nullptr, sd.n, sorted, sd.pos, inner, inner_cap,
                                       st_i, nullptr, nullptr, nullptr, 0, half);
      if (st != RL_OK) return st;
    }
    int st = keyaxis::run_bounds(sd.n > 0 ? sorted : sd.keys, sd.n, sd.kv, sd.off, sd.d, inner, inner_cap, st_i);
    if (st != RL_OK) return st;
  }
  // the alignment arrays and the alignment's workspace reuse the scratch (both sides are done with it)
  Carve ca{scratch, scratch_cap};
  carve_alignment(ca, nl, nr, p);
  if (!ca.ok) return RL_ERR_WORKSPACE;
  void* inner = scratch + align_up(ca.used, 256);
  const size_t inner_cap = scratch_cap - align_up(ca.used, 256);
  if (aux) {  // join: the alignment waits for the right side
    cudaError_t e = cudaEventRecord(aux->join, aux->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, aux->join, 0);
    if (e != cudaSuccess) return rl_cuda_status(e);
  }
  const int64_t cap = std::min(nl, nr) > 0 ? nl : 0;
  return keyaxis::key_axis_align(p->left_key_values, p->left_offsets, p->scalars + 0, cap, p->right_key_values,
                                 p->right_offsets, p->scalars + 1, p->matched_keys, p->left_starts, p->left_counts,
                                 p->right_starts, p->right_counts, p->pair_offsets, p->scalars + 2,
                                 reinterpret_cast<uint64_t*>(p->scalars + 3), inner, inner_cap, stream);
}

}  // namespace plan
}  // namespace rl

extern "C" {

RL_API size_t rl_join_plan_workspace_bytes(int64_t n_left, int64_t n_right) {
  return rl::plan::workspace_bytes(n_left, n_right);
}

RL_API int rl_join_plan_build(const int64_t* left_keys, int64_t n_left, const int64_t* right_keys, int64_t n_right,
                              void* ws, size_t ws_bytes, rl_join_plan* plan, void* stream) {
  return rl::plan::build(left_keys, n_left, right_keys, n_right, ws, ws_bytes, plan,
                         static_cast<cudaStream_t>(stream));
}

}  // extern "C"
