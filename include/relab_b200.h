/*
 * relab_b200.h — C ABI of the B200 tensor path (sm_100a).
 *
 * This is the drop-in boundary for the reference's tensor path
 * (/root/reference/pkg/src/relab/tensorpath.py). The reference is pure
 * Python + numpy, so its "FFI" for this path is the Python call into
 * numpy primitives; every entry point below replaces one group of those
 * primitives and is bound from Python with ctypes
 * (paper_2602_21237_b200/_capi.py).
 *
 * Conventions
 *   - All data pointers are DEVICE pointers unless a parameter says "host".
 *   - Buffers are caller-allocated; the library never allocates or frees
 *     caller memory and keeps no global mutable state. Scratch space comes
 *     from the caller through (ws, ws_bytes); size it with the matching
 *     *_workspace_bytes() query. ws must be 256-byte aligned.
 *   - `stream` is a cudaStream_t passed as void*. Every call is
 *     asynchronous on that stream; nothing synchronises the host.
 *   - Row indices (positions, permutations, starts, counts, row ids) are
 *     uint32: one call handles at most RL_MAX_ROWS rows per side. The
 *     Python layer widens them to int64 when it hands numpy arrays back,
 *     matching the reference dtypes.
 *   - Counts that the host does not need before the next launch (distinct
 *     keys D, matched keys M, total output pairs) are written to device
 *     scalars, so a join runs with exactly one device→host sync (the output
 *     size, needed to allocate the output columns).
 *   - Return value: RL_OK or an RL_ERR_* status; rl_strerror() names it.
 */
#ifndef RELAB_B200_H
#define RELAB_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define RL_API __attribute__((visibility("default")))
#else
#define RL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define RL_ABI_VERSION 1

#define RL_OK 0
#define RL_ERR_BAD_ARG 1          /* ValueError on the Python side            */
#define RL_ERR_OUTPUT_TOO_LARGE 2 /* relab.errors.OutputTooLarge               */
#define RL_ERR_WORKSPACE 3        /* workspace too small / misaligned          */
#define RL_ERR_TOO_MANY_ROWS 4    /* n > RL_MAX_ROWS                           */
#define RL_ERR_IO 5               /* file read/write failed (OSError)          */
#define RL_ERR_CUDA 1000          /* RL_ERR_CUDA + cudaError_t                 */

#define RL_MAX_ROWS 4294967295LL  /* uint32 row ids */

/* Column kinds (relation.py:23-40: Int64, Bytes(w)). */
#define RL_COL_INT64 0
#define RL_COL_BYTES 1

/* Which row a gathered output column reads (tensorpath.py:174-185). */
#define RL_SIDE_LEFT 0   /* source row = left row id of the pair          */
#define RL_SIDE_RIGHT 1  /* source row = right row id of the pair         */
#define RL_SIDE_KEY 2    /* the matched key itself (int64, src ignored)    */

#define RL_MAX_COLUMNS 32

typedef struct rl_column {
  const void* src; /* device: n_src rows × width bytes, row-major          */
  void* dst;       /* device: out rows × width bytes                       */
  int32_t width;   /* bytes per row: 8 for Int64, w for Bytes(w) (w >= 0)  */
  int32_t side;    /* RL_SIDE_*                                            */
} rl_column;

RL_API int rl_abi_version(void);
RL_API const char* rl_strerror(int status);
/* Number of SMs of the current device (grid sizing; 148 on B200). */
RL_API int rl_device_sm_count(void);
/* Process-wide count of kernels this library has launched (a statistic for
 * the benchmark's gpu_launches claim; monotone, never reset). */
RL_API int64_t rl_launch_count(void);

/* ---------------------------------------------------------------------
 * K1+K2  Stable LSD radix sort of one key word, carrying row ids.
 *
 * Replaces  _stable_key_order      tensorpath.py:62-75
 *           _stable_axis_order     tensorpath.py:206-229
 *           one refinement step    tensorpath.py:244-246
 *             perm = perm[_stable_axis_order(axis[perm], direction)]
 *
 * The key of output slot i is word `word` of row r = perm_in[i] (or r = i
 * when perm_in is NULL) of column `col`:
 *   RL_COL_INT64 (width 8, word 0): the int64 value, ordered as signed;
 *       descending uses the bitwise complement (tensorpath.py:215).
 *   RL_COL_BYTES (width w, word j < ceil(w/8)): bytes [8j, 8j+8) of the
 *       row, complemented first when descending, zero-padded, read
 *       big-endian (tensorpath.py:220-225).
 * Output: perm_out[i] = the row at sorted position i; ties keep input
 * order (stable). sorted_keys_out (optional, INT64 without perm_in only)
 * receives the sorted int64 key values (tensorpath.py:84 `sk`).
 * A sort is two launches: the digit histograms, then ONE cooperative
 * kernel running the plan and every digit pass separated by grid barriers;
 * passes whose 8-bit digit is constant over the input are skipped on the
 * device (no host sync, no launch). Wide INT64 keys without perm_in
 * (n >= 2^18, top 16 bits spread so every one of the 65536 sub-buckets fits
 * on chip) take a hybrid: the rows reach their sub-bucket — by two onesweep
 * passes on the top two digits inside the cooperative kernel (n < 2^22), or
 * (n >= 2^22) by exact per-chunk sub-bucket counts and two non-stable
 * counting passes (three launches ahead of it) — then an on-chip sort of
 * each sub-bucket by (key, row id) is written straight to the outputs (the
 * cooperative kernel, or its own 512-thread launch on the scatter path). On
 * the scatter path keys whose bits do not all vary are packed first (up to
 * two runs of varying bits, estimated from a sample and checked against every
 * key), so narrow and composite keys get sub-buckets too. A sub-bucket over
 * the on-chip cap switches to the LSD passes on the device. Results are
 * identical on every path. An INT64 `col` read without perm_in, and perm_in,
 * must be 16-byte aligned (they are streamed with TMA bulk copies);
 * RL_ERR_BAD_ARG otherwise.
 * --------------------------------------------------------------------- */
RL_API size_t rl_sort_workspace_bytes(int64_t n);
RL_API int rl_sort_axis(const void* col, int32_t col_kind, int32_t width,
                 int32_t word, int32_t descending, const uint32_t* perm_in,
                 int64_t n, int64_t* sorted_keys_out, uint32_t* perm_out,
                 void* ws, size_t ws_bytes, void* stream);

/* rl_sort_axis + Relation.take fused into the final digit pass
 * (tensorpath.py:247): for every column c (side RL_SIDE_LEFT, at most 8),
 * c.dst row o = c.src row perm_out[o], written while the permutation is
 * written — no separate gather launch, no re-read of the permutation. */
RL_API int rl_sort_axis_gather(const void* col, int32_t col_kind, int32_t width,
                 int32_t word, int32_t descending, const uint32_t* perm_in,
                 int64_t n, int64_t* sorted_keys_out, uint32_t* perm_out,
                 const rl_column* columns, int32_t n_columns,
                 void* ws, size_t ws_bytes, void* stream);
#define RL_SORT_MAX_FUSED_COLUMNS 8

/* Same as rl_sort_axis_gather, for measurement: events[0..2] (cudaEvent_t
 * created by the caller with timing enabled) are recorded on `stream`
 * before the histogram kernel, between it and the cooperative pass kernel,
 * and after the pass kernel (scatter path: before the chunk counts, before
 * the local-phase kernel, after the cooperative kernel); if stamps_dev
 * (device, RL_SORT_STAMPS x uint64) is not NULL, CTA 0 writes %globaltimer
 * (ns) there: [0] histogram start, [1] pass kernel start, [2+p] after digit
 * pass p (0 for skipped passes; in the hybrid [2] = sub-bucket check done;
 * scatter path: [2] digit-7 pass start, [3] digit-6 pass start, [1] local
 * phase start), [10] end, and [11] the path taken: 0 LSD, 1 hybrid, 2
 * hybrid that fell back to LSD, 3 scatter hybrid, 4 scatter hybrid that
 * fell back to LSD. */
#define RL_SORT_EVENTS 3
#define RL_SORT_STAMPS 12
RL_API int rl_sort_axis_profiled(const void* col, int32_t col_kind, int32_t width,
                 int32_t word, int32_t descending, const uint32_t* perm_in,
                 int64_t n, int64_t* sorted_keys_out, uint32_t* perm_out,
                 const rl_column* columns, int32_t n_columns,
                 void* ws, size_t ws_bytes, void* stream,
                 void* const* events, unsigned long long* stamps_dev);

/* ---------------------------------------------------------------------
 * K3  Run bounds of sorted keys: distinct keys + CSR offsets.
 *
 * Replaces tensorpath.py:84-92
 *   bounds = flatnonzero(concat([True], sk[1:] != sk[:-1]))
 *   key_values = sk[bounds]; offsets = concat([bounds, [n]])
 * key_values and offsets need capacity n and n+1. *d_out (device int64)
 * receives D; offsets[D] = n. n == 0 gives D = 0, offsets = [0].
 * --------------------------------------------------------------------- */
RL_API size_t rl_run_bounds_workspace_bytes(int64_t n);
RL_API int rl_run_bounds(const int64_t* sorted_keys, int64_t n, int64_t* key_values,
                  uint32_t* offsets, int64_t* d_out, void* ws,
                  size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------
 * K4+K5  Key-axis alignment and join sizing.
 *
 * Replaces key_axis_align  tensorpath.py:109-128 (searchsorted + mask +
 * compaction) and the sizing of tensor_join tensorpath.py:149-161
 * (per_key = lc*rc, cumsum). Every left distinct key is searched in the
 * right distinct keys (vectorised searchsorted, lower bound); matches are
 * compacted in left-key order. D_left / D_right are read from device
 * scalars (rl_run_bounds' d_out); d_left_cap bounds the grid.
 * Outputs (capacity d_left_cap, pair_offsets d_left_cap+1):
 *   matched_keys[M]; left_starts/left_counts/right_starts/right_counts[M];
 *   pair_offsets[0..M] = exclusive prefix of lc*rc (uint64),
 *   pair_offsets[M] = total; *m_out = M; *total_out = total.
 * --------------------------------------------------------------------- */
RL_API size_t rl_align_workspace_bytes(int64_t d_left_cap);
RL_API int rl_key_axis_align(const int64_t* left_keys, const uint32_t* left_offsets,
                      const int64_t* d_left, int64_t d_left_cap,
                      const int64_t* right_keys,
                      const uint32_t* right_offsets, const int64_t* d_right,
                      int64_t* matched_keys, uint32_t* left_starts,
                      uint32_t* left_counts, uint32_t* right_starts,
                      uint32_t* right_counts, uint64_t* pair_offsets,
                      int64_t* m_out, uint64_t* total_out, void* ws,
                      size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------
 * Join plan: K1-K5 for both sides in ONE call over ONE workspace.
 * tensorpath.py:78-93 (to_tensor) x 2 + 109-161 (key_axis_align + sizing).
 * Fills *plan with device pointers into ws (valid while ws lives); the
 * device scalars are [0] D_left, [1] D_right, [2] M, [3] total pairs.
 * Feed the plan arrays to rl_join_expand / rl_join_pair_checksum.
 * --------------------------------------------------------------------- */
typedef struct rl_join_plan {
  int64_t* scalars;
  uint32_t* left_positions;
  int64_t* left_key_values;
  uint32_t* left_offsets;
  uint32_t* right_positions;
  int64_t* right_key_values;
  uint32_t* right_offsets;
  int64_t* matched_keys;
  uint32_t* left_starts;
  uint32_t* left_counts;
  uint32_t* right_starts;
  uint32_t* right_counts;
  uint64_t* pair_offsets;
} rl_join_plan;
RL_API size_t rl_join_plan_workspace_bytes(int64_t n_left, int64_t n_right);
RL_API int rl_join_plan_build(const int64_t* left_keys, int64_t n_left,
                              const int64_t* right_keys, int64_t n_right, void* ws,
                              size_t ws_bytes, rl_join_plan* plan, void* stream);

/* ---------------------------------------------------------------------
 * ORDER BY on a raw int64 key with the other columns carried (the sort +
 * Relation.take of tensorpath.py:232-252 in one call): dst row o of every
 * column = src row perm[o], as rl_sort_axis_gather. When the key varies in
 * <= 32 bits and n reaches the scatter path, the columns' bytes (<= 16 a row
 * after natural alignment, <= 4 columns) ride beside every packed row through
 * the counting passes and leave from each on-chip run — no gather by row id;
 * otherwise the gathers are fused into the sort's final pass. Workspace:
 * rl_sort_carry_workspace_bytes(n, the columns' total width in bytes).
 * --------------------------------------------------------------------- */
RL_API size_t rl_sort_carry_workspace_bytes(int64_t n, int32_t carry_bytes);
RL_API int rl_sort_axis_carry(const int64_t* keys, int64_t n, int32_t descending,
                              int64_t* sorted_keys_out, uint32_t* perm_out,
                              const rl_column* columns, int32_t n_columns, void* ws,
                              size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------
 * Bucket join: the join plan for keys with <= 32 varying bits (both sides
 * together), without sorted key axes. Replaces tensorpath.py:78-93 (x2),
 * 109-128 and the sizing of 131-161: one joint key packing; every row of
 * both sides as one packed word (key bits << 32 | row id) in the same 65536
 * sub-buckets (top 16 key bits; the sort's chunk counts + two counting
 * passes); per run of sub-buckets (<= 2560 rows a side) the pairs counted on
 * chip; an exclusive scan of the run counts. Device scalars[0] = total
 * pairs, scalars[1] = 1 if the plan applies — 0 (keys need more than 32
 * bits, a sub-bucket holds more than 2560 rows of a side, n > 2^32): use
 * rl_join_plan_build instead. Nothing is synchronised; read the two scalars
 * with one D2H. n_left, n_right >= 1; keys 16-byte aligned.
 * rl_bjoin_expand then writes output pairs [out_begin, out_end) exactly as
 * rl_join_expand does (same rows, same order, same columns; the key column
 * from RL_SIDE_KEY, other columns gathered by row id): each run's rows of
 * both sides are sorted on chip by (key, row id) and matched in their bins.
 * --------------------------------------------------------------------- */
typedef struct rl_bjoin_plan {
  const uint64_t* rows_left;
  const uint64_t* rows_right;
  const uint32_t* sub_off_left;
  const uint32_t* sub_off_right;
  uint32_t* flags_left;
  uint32_t* flags_right;
  uint32_t* counts;        /* pairs per (group, run) */
  uint64_t* offsets;       /* first output row per group */
  int64_t* scalars;
  const int64_t* left_keys;
  int32_t levels;          /* 2: sub-buckets = top 16 key bits; 3 (above ~142M rows a side): top 24 */
  /* carried payload (written by rl_bjoin_plan_build, read by rl_bjoin_expand) */
  const uint64_t* pay_left;
  const uint64_t* pay_right;
  int32_t words_left, words_right;
  int32_t carry_cols_left, carry_cols_right;
  const void* carry_src_left[4];
  const void* carry_src_right[4];
  int32_t carry_width_left[4];
  int32_t carry_width_right[4];
  int32_t carry_off_left[4];
  int32_t carry_off_right[4];
  /* selective runs' matches listed by the plan (two levels; null when off):
   * rl_bjoin_expand writes a listed run from these instead of re-binning it */
  const void* sel_pairs;
  const uint32_t* sel_idx;
  const uint32_t* run_sel;
} rl_bjoin_plan;
/* Payload words (8 B) a row of this side carries through the plan's passes
 * for these columns (0: none; at most 16 bytes / 4 columns, else 0 — they
 * are then gathered by row id); -1 on a bad argument. */
RL_API int rl_bjoin_carry_words(const rl_column* columns, int32_t n_columns);
RL_API size_t rl_bjoin_workspace_bytes(int64_t n_left, int64_t n_right, int32_t left_words,
                                       int32_t right_words);
/* left_carry / right_carry (src + width; optional): the output columns of each
 * side to carry with its rows — rl_bjoin_expand reads a carried column (same
 * src pointer and width) from beside the row instead of gathering it by row id. */
RL_API int rl_bjoin_plan_build(const int64_t* left_keys, int64_t n_left,
                               const int64_t* right_keys, int64_t n_right,
                               const rl_column* left_carry, int32_t n_left_carry,
                               const rl_column* right_carry, int32_t n_right_carry, void* ws,
                               size_t ws_bytes, rl_bjoin_plan* plan, void* stream);
RL_API int rl_bjoin_expand(const rl_bjoin_plan* plan, uint64_t out_begin,
                           uint64_t out_end, uint32_t* left_rows_out,
                           uint32_t* right_rows_out, const rl_column* columns,
                           int32_t n_columns, void* stream);
/* rl_bjoin_expand with a destination row stride per column (bytes; 0 = the
 * width): columns of width 8 or 16 may be written row-interleaved into one
 * buffer (stride a multiple of the width, dst aligned to the width). */
RL_API int rl_bjoin_expand_strided(const rl_bjoin_plan* plan, uint64_t out_begin,
                                   uint64_t out_end, uint32_t* left_rows_out,
                                   uint32_t* right_rows_out, const rl_column* columns,
                                   int32_t n_columns, const int32_t* dst_strides, void* stream);
/* rl_join_pair_checksum on a bucket-join plan: sum of fmix64((left_row << 32)
 * | right_row) over pairs [out_begin, out_end), added into *sum_out. */
RL_API int rl_bjoin_pair_checksum(const rl_bjoin_plan* plan, uint64_t out_begin,
                                  uint64_t out_end, uint64_t* sum_out, void* stream);

/* ---------------------------------------------------------------------
 * K6+K7  Run expansion fused with the column gathers.
 *
 * Replaces tensorpath.py:157-185: output pair t (global index in
 * [out_begin, out_end)) belongs to matched key g with
 * pair_offsets[g] <= t < pair_offsets[g+1]; local = t - pair_offsets[g];
 * (li, ri) = divmod(local, right_counts[g]);
 * left row  = left_positions[left_starts[g] + li],
 * right row = right_positions[right_starts[g] + ri].
 * Emits rows in (key, left row, right row) order — byte-identical to the
 * reference. Optional outputs (NULL to skip): left_rows/right_rows
 * (uint32, index t - out_begin; each 16-byte aligned — the pairs-only
 * path stores four row ids at a time — else RL_ERR_BAD_ARG) and up to
 * RL_MAX_COLUMNS gathered columns (rl_column, host array; dst indexed by
 * t - out_begin). m (number of matched keys) is passed from the host.
 * --------------------------------------------------------------------- */
RL_API int rl_join_expand(const int64_t* matched_keys, const uint32_t* left_starts,
                   const uint32_t* right_starts, const uint32_t* right_counts,
                   const uint64_t* pair_offsets, int64_t m,
                   const uint32_t* left_positions,
                   const uint32_t* right_positions, uint64_t out_begin,
                   uint64_t out_end, uint32_t* left_rows_out,
                   uint32_t* right_rows_out, const rl_column* columns,
                   int32_t n_columns, void* stream);

/* Order-independent checksum of the pairs in [out_begin, out_end):
 * sum over pairs of fmix64((left_row << 32) | right_row), into *sum_out
 * (device uint64, accumulated: zero it first). For joins too large to
 * materialise (BASELINE cfg3: 2.29e12 pairs). */
RL_API int rl_join_pair_checksum(const uint32_t* left_starts,
                          const uint32_t* right_starts,
                          const uint32_t* right_counts,
                          const uint64_t* pair_offsets, int64_t m,
                          const uint32_t* left_positions,
                          const uint32_t* right_positions, uint64_t out_begin,
                          uint64_t out_end, uint64_t* sum_out, void* stream);

/* ---------------------------------------------------------------------
 * K7  Row gather by a uint32 index vector (Relation.take,
 * relation.py:133-136, as used by tensor_sort tensorpath.py:247).
 * out row t of every column = src row rows[t]; side must be RL_SIDE_LEFT.
 * --------------------------------------------------------------------- */
RL_API int rl_gather_rows(const uint32_t* rows, int64_t m, const rl_column* columns,
                   int32_t n_columns, void* stream);

/* Relation.take of two 8-byte columns stored row-interleaved: src is m_src
 * rows of 16 bytes (16-byte aligned); dst_lo[t] / dst_hi[t] = the first /
 * last 8 bytes of src row rows[t]. One random 16-byte load a row (the fused
 * join -> ORDER BY pipeline writes the join's other two columns this way). */
RL_API int rl_gather_rows_split16(const uint32_t* rows, int64_t m, const void* src, void* dst_lo,
                                  void* dst_hi, void* stream);

/* Widen uint32 → int64 (positions/offsets handed back as numpy int64). */
RL_API int rl_widen_u32(const uint32_t* src, int64_t n, int64_t* dst, void* stream);

/* ---------------------------------------------------------------------
 * K8  Hash partitioning for the multi-GPU join (no reference
 * counterpart; the hash is hash_i64, hashing.py:54-61:
 * h(k) = fmix64(u64(k) ^ fmix64(seed)), destination = h(k) mod P).
 * Stable within each destination: rows keep input order.
 * counts_out[P] (device int64) receives per-destination row counts;
 * the packed outputs are grouped by destination in rank order.
 * --------------------------------------------------------------------- */
RL_API size_t rl_partition_workspace_bytes(int64_t n, int32_t parts);
RL_API int rl_hash_partition(const int64_t* keys, int64_t n, int32_t parts,
                      uint64_t seed, const rl_column* columns,
                      int32_t n_columns, uint32_t* row_ids_out,
                      int64_t* counts_out, void* ws, size_t ws_bytes,
                      void* stream);

/* Range partition for the distributed ORDER BY: row i (global row id
 * gid_base + i) goes to destination = number of splitters (split_keys[s],
 * split_gids[s]) strictly below (key, gid) in (key order, gid) order —
 * descending keys compare by complement like rl_sort_axis. n_splitters
 * <= 255 (destinations = n_splitters + 1). Stable within a destination;
 * counts_out[n_splitters + 1]; columns gathered like rl_hash_partition. */
RL_API int rl_range_partition(const int64_t* keys, int64_t n, int64_t gid_base,
                              const int64_t* split_keys, const int64_t* split_gids,
                              int32_t n_splitters, int32_t descending,
                              const rl_column* columns, int32_t n_columns,
                              uint32_t* row_ids_out, int64_t* counts_out, void* ws,
                              size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------
 * Multi-GPU exchange fused with the partition gather.
 * After rl_hash_partition / rl_range_partition (row ids grouped by
 * destination; dest_starts[parts + 1] = device prefix of the counts), every
 * partitioned row i of destination d is stored straight into d's receive
 * buffer — through d's peer pointer (NVLink P2P into symmetric memory; the
 * own rank's local buffer) — at row dest_offsets[d] + (i - dest_starts[d]):
 * each column c (src = local column, width bytes) into the region at
 * dest_bases[d * (n_columns + 1) + c], the local row id (uint32) into the
 * region at dest_bases[d * (n_columns + 1) + n_columns]. Replaces the
 * per-column gather + NCCL all-to-all-v; receive order = source rank order,
 * partition order within a source, as the all-to-all. parts <=
 * RL_PUSH_MAX_PARTS, n_columns <= RL_PUSH_MAX_COLUMNS (else RL_ERR_BAD_ARG;
 * wider exchanges go through NCCL). The caller brackets the call with
 * barriers.
 * --------------------------------------------------------------------- */
#define RL_PUSH_MAX_PARTS 64
#define RL_PUSH_MAX_COLUMNS 8
RL_API int rl_push_rows(const uint32_t* rows, int64_t n, int32_t parts,
                 const int64_t* dest_starts, const rl_column* columns,
                 int32_t n_columns, const uint64_t* dest_bases,
                 const int64_t* dest_offsets, void* stream);

/* rl_push_rows, but the last region of every destination receives int64
 * GLOBAL row ids (gid_base + local row id, 8 bytes per row) instead of u32
 * local row ids: the receiver needs no per-source bases. */
RL_API int rl_push_rows_gid(const uint32_t* rows, int64_t n, int32_t parts,
                 const int64_t* dest_starts, const rl_column* columns,
                 int32_t n_columns, const uint64_t* dest_bases,
                 const int64_t* dest_offsets, int64_t gid_base, void* stream);

/* Splitters of the multi-GPU ORDER BY (dist.choose_splitters_device; the
 * sample-sort step of SURVEY §8(e), ranges chosen on the composite
 * (key, global row id) order so stability survives duplicate-heavy keys).
 * rl_sample_keys writes this rank's [3][per_rank] int64 sample pack (key in
 * sort order — complemented when descending —, global row id, 1 = real
 * sample) for an all-gather; rl_pick_splitters takes the gathered
 * [parts][3][per_rank] packs (parts * per_rank <= RL_MAX_SPLIT_SAMPLES) and
 * writes the parts-1 splitter keys and global row ids (one CTA, no host
 * round trip). rl_global_ids turns received u32 local row ids into int64
 * global ids: out[i] = bases[s] + rows[i] for the rows of source s
 * (recv_counts[s] rows each, host arrays, parts <= 64). */
#define RL_MAX_SPLIT_SAMPLES 2048
RL_API int rl_sample_keys(const int64_t* keys, int64_t n, int32_t per_rank,
                 int64_t gid_base, int32_t descending, int64_t* pack, void* stream);
RL_API int rl_pick_splitters(const int64_t* gathered, int32_t parts, int32_t per_rank,
                 int32_t descending, int64_t* split_keys, int64_t* split_gids,
                 void* stream);
RL_API int rl_global_ids(const uint32_t* rows, int64_t total, int32_t parts,
                 const int64_t* recv_counts, const int64_t* bases, int64_t* out,
                 void* stream);

/* ---------------------------------------------------------------------
 * The reference's 128-bit multiset result digest (relation.py:319-330,
 * hashing.py:64-109), bit-exact, computed on the device from the columns
 * (src, width; schema order; Int64 width 8) of n rows without serialising
 * them. out2[0] = lane 0 (high 64 bits), out2[1] = lane 1 (low 64 bits);
 * n == 0 gives 0. Row width <= 512 bytes.
 * --------------------------------------------------------------------- */
RL_API int rl_multiset_digest(const rl_column* columns, int32_t n_columns,
                              int64_t n, uint64_t* out2, void* stream);

/* ---------------------------------------------------------------------
 * Host→device staging (the drop-in boundary's inputs are pageable numpy
 * columns). A stager owns a pinned ring of `slots` chunks, a copy stream
 * and `threads` native copy threads; rl_stager_h2d copies chunk c into the
 * ring in parallel while the copy engine DMAs chunk c-1, then makes
 * `stream` wait for the finished upload (no host sync on the data path).
 * ready_event (cudaEvent_t or NULL): the copy stream first waits for it —
 * record it on the allocating stream right after allocating dst, so the
 * upload cannot overtake earlier work on recycled memory while kernels
 * enqueued later still overlap the upload.
 * One stager serves one upload at a time (calls are serialised).
 * --------------------------------------------------------------------- */
RL_API void* rl_stager_create(int32_t threads, size_t chunk_bytes, int32_t slots);
RL_API void rl_stager_destroy(void* stager);
RL_API int rl_stager_h2d(void* stager, void* dst_dev, const void* src_host,
                         size_t bytes, void* stream, void* ready_event);

/* RELCOL01 relation files straight to / from HBM (relation.py:364-419).
 * rl_stager_file_h2d: `bytes` at `file_offset` of the open file `fd` are
 * pread() by the stager's threads into its pinned ring while the copy
 * engine DMAs the previous chunk to dst_dev on the stager's copy stream;
 * `stream` waits for the upload, ready_event (optional) orders it after
 * earlier work. rl_stager_file_d2h: device bytes -> file section through the
 * ring (DMA of chunk c+1 overlaps the pwrite of chunk c); synchronous.
 * RL_ERR_IO on a short read / failed write. */
RL_API int rl_stager_file_h2d(void* stager, void* dst_dev, int32_t fd,
                 uint64_t file_offset, size_t bytes, void* stream,
                 void* ready_event);
RL_API int rl_stager_file_d2h(void* stager, const void* src_dev, int32_t fd,
                 uint64_t file_offset, size_t bytes, void* stream);
/* File section -> host memory (page-locked columns), parallel pread(). */
RL_API int rl_stager_file_read(void* stager, void* dst_host, int32_t fd,
                 uint64_t file_offset, size_t bytes);
/* Long-lived inputs (a relation reused across repetitions) are page-locked
 * once and then uploaded with one direct DMA each (no staging copy). */
RL_API int rl_host_register(void* host, size_t bytes);
RL_API int rl_host_unregister(void* host);
RL_API int rl_host_is_pinned(const void* host);
RL_API int rl_stager_h2d_pinned(void* stager, void* dst_dev, const void* src_host,
                                size_t bytes, void* stream, void* ready_event);
/* Block until every upload issued through this stager has read its host
 * memory (call before unregistering or freeing a source buffer). */
RL_API int rl_stager_drain(void* stager);

#ifdef __cplusplus
}
#endif

#endif /* RELAB_B200_H */
