/*
 * rowblock_b200 — C ABI of the B200-native 1-SA → VBR → SpMM hot path.
 *
 * Drop-in boundary for the reference package rowblock v0.1.0
 * (/root/reference/pkg/src/rowblock).  The reference is pure Python, so its
 * "FFI" is its Python API; each entry point below replaces one reference
 * function and the Python host layer (paper_2202_05868_b200/) binds them with
 * ctypes under the reference's own names and signatures:
 *
 *   rb_block_1sa          replaces  block_1sa          blocking.py:283-306
 *   rb_vbr_plan/emit      replace   vbr_from_grouping  vbr.py:88-125
 *   rb_spmm_plan_create/  replace   spmm_vbr           multiply.py:72-97
 *     rb_spmm_execute
 *
 * Conventions
 *   - Plain C: integers, sizes and raw DEVICE pointers (CUDA global memory);
 *     `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Inputs are never written.  Outputs go to caller-allocated device buffers
 *     whose sizes are stated per argument (worst case, so no size query is
 *     needed first) or come from a *_workspace_size query.
 *   - Calls are stream-ordered.  Calls that must return a data-dependent count
 *     to the host (n_groups, n_blocks) synchronise `stream` before returning.
 *   - Return value: RB_OK, or an error code; rb_last_error_string() gives a
 *     thread-local message.  The Python layer maps RB_EINVAL → ValueError,
 *     RB_ENOMEM → MemoryError, everything else → RuntimeError (the reference
 *     raises ValueError for bad shapes/partitions/τ: vbr.py:96-97,
 *     multiply.py:76-77, blocking.py:80-84).
 *   - Deterministic: identical inputs give bit-identical outputs; C rows are
 *     written by exactly one CTA with a fixed accumulation order (no atomics).
 */
#ifndef ROWBLOCK_B200_H_
#define ROWBLOCK_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RB_OK 0
#define RB_EINVAL 1
#define RB_ECUDA 2
#define RB_ENOMEM 3
#define RB_EUNSUPPORTED 4

/* element types of tiles / B */
#define RB_F32 0
#define RB_BF16 1
#define RB_F16 2
#define RB_F64 3

/* similarity kinds (MergePolicy.similarity, blocking.py:75) */
#define RB_JACCARD 0
#define RB_COSINE 1

const char* rb_last_error_string(void);
int rb_abi_version(void);

/* ------------------------------------------------------------------ block_1sa
 * Replaces block_1sa(A, partition, policy, use_compression) (blocking.py:283-306):
 * quotient bitsets (blocking.py:118-136), exact-pattern compression in first-occurrence
 * order (295-301), the one-pass greedy scan (209-266) and grouping assembly (269-280).
 *
 * Inputs (device): CSR pattern row_ptr[n_rows+1], col_idx[nnz] (int64, columns strictly
 * increasing per row), column partition boundaries[n_seg+1] (int64, 0 .. n_cols).
 * Policy: tau in [0,1], similarity RB_JACCARD/RB_COSINE, bounded, pattern_update.
 * Outputs (device, caller-allocated):
 *   group_of[n_rows]       RowGrouping.group_of
 *   row_perm[n_rows]       concatenation of the groups' rows (= VbrMatrix.row_perm)
 *   group_ptr[n_rows+1]    row extents of each group inside row_perm (first n_groups+1 used)
 *   seed_size[n_rows]      RowGroup.seed_size (first n_groups used)
 *   pattern_ptr[n_rows+1], pattern_idx[max(nnz,1)]   RowGroup.pattern (sorted segment ids)
 *   *n_groups (HOST)       number of groups H
 */
int rb_block_1sa_workspace_size(int64_t n_rows, int64_t nnz, int64_t n_seg, int use_compression,
                                size_t* bytes);
int rb_block_1sa(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr, const int64_t* col_idx,
                 const int64_t* boundaries, int64_t n_seg, double tau, int similarity, int bounded,
                 int pattern_update, int use_compression, void* workspace, size_t workspace_bytes,
                 int64_t* group_of, int64_t* row_perm, int64_t* group_ptr, int64_t* seed_size,
                 int64_t* pattern_ptr, int64_t* pattern_idx, int64_t* n_groups, void* stream);

/* ------------------------------------------------------------------ vbr_from_grouping
 * Replaces vbr_from_grouping(A, grouping, partition) (vbr.py:88-125) in two stream-ordered
 * phases sharing one workspace (keep it alive from rb_vbr_plan to rb_vbr_emit):
 *
 * rb_vbr_plan: stored block columns of each block row recomputed from the data
 *   (vbr.py:106-112), tile layout.  Inputs: CSR pattern, boundaries, the grouping as
 *   row_perm[n_rows] / row_partition[H+1] (int64, device).  Outputs (device):
 *   perm32[n_rows], rpart32[H+1], blk_ptr[H+1] (int32), grp_tile_row[H] (int64: first tile
 *   row of each block row), bounds32[n_seg+1]; HOST: *n_blocks, *total_tile_rows.
 *   Tile layout: block t of block row g is an hp(g) x dp row-major tile starting at tile row
 *   grp_tile_row[g] + t*hp(g), hp(h) = 16 / next pow2 (h <= 128) or roundup(h,128).
 * rb_vbr_emit: blk_col[n_blocks] (int32, ascending per block row) and the zero-padded
 *   tiles[total_tile_rows x dp] of tile_dtype (RB_BF16/RB_F16/RB_F32/RB_F64) scattered
 *   from values[nnz] (float64, device) — vbr.py:113-123.  dp >= max segment width; dp must
 *   be a multiple of 64 for RB_BF16/RB_F16 (tensor-core path).
 */
int rb_vbr_workspace_size(int64_t n_rows, int64_t n_groups, int64_t n_seg, size_t* bytes);
int rb_vbr_plan(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_idx,
                const int64_t* boundaries, int64_t n_seg, const int64_t* row_perm, const int64_t* row_partition,
                int64_t n_groups, void* workspace, size_t workspace_bytes, int32_t* perm32, int32_t* rpart32,
                int32_t* blk_ptr, int64_t* grp_tile_row, int32_t* bounds32, int64_t* n_blocks,
                int64_t* total_tile_rows, void* stream);
/* Compact payloads of skinny block rows (h <= h_max): cmp_ptr[n_rows+1] (device, int64, by permuted
 * row: counts of rows of block rows with h <= h_max, 0 elsewhere, prefix-summed) and *total (HOST);
 * then per such row its nonzeros as int32 global columns and values rounded to tile_dtype held in
 * float — a block row's payload in block-column order without the segment padding (vbr.py:113-123).
 * perm32 / rpart32 are rb_vbr_plan outputs.                                                       */
int rb_vbr_compact_count(int64_t n_rows, const int64_t* row_ptr, const int32_t* perm32, const int32_t* rpart32,
                         int64_t n_groups, int32_t h_max, int64_t* cmp_ptr, int64_t* total, void* stream);
int rb_vbr_compact_emit(int64_t n_rows, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                        const int32_t* perm32, const int64_t* cmp_ptr, int32_t tile_dtype, int32_t* cmp_col,
                        float* cmp_val, void* stream);
int rb_vbr_emit(int64_t n_rows, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                const int64_t* boundaries, int64_t n_seg, int64_t n_groups, void* workspace, size_t workspace_bytes,
                const int32_t* perm32, const int32_t* rpart32, const int32_t* blk_ptr, const int64_t* grp_tile_row,
                int32_t* blk_col, void* tiles, int32_t tile_dtype, int32_t dp, int64_t total_tile_rows,
                void* stream);

/* ------------------------------------------------------------------ spmm_vbr
 * Replaces spmm_vbr(V, B, threads) (multiply.py:72-97): C = A·B with C rows written at
 * row_perm positions (un-permute, multiply.py:90); rows of empty block rows are written
 * as exact zeros (multiply.py:85-86).  C is float32 [n_rows x N] (row stride ldc);
 * B is [n_cols x N] row-major (row stride ldb, elements), RB_BF16 / RB_F16 (tcgen05
 * tensor-core path, fp32 accumulate in TMEM) or RB_F32 (fp32 check path, FFMA).
 * A plan owns its work list (device memory it allocates and frees in _destroy).
 * Sharding: shard k of n_shards takes a contiguous, work-balanced range of the work list
 * (whole block-row M-tiles); each C row is produced by exactly one shard.
 * Concurrency: rb_spmm_execute may be called on one plan from several host threads and streams.
 * A plan holds device work counters and split-K partials that its kernels reset, so executions of
 * ONE plan are serialised: each waits (cudaStreamWaitEvent, no host blocking) for the previous
 * execution of the same plan when it is issued on a different stream.  Products meant to run
 * concurrently need one plan each.                                                       */
typedef struct rb_vbr_device {
  int64_t n_rows;
  int64_t n_cols;
  int64_t n_block_rows;          /* H */
  int64_t n_blocks;              /* nb */
  int64_t n_seg;
  int64_t total_tile_rows;
  int32_t dp;                    /* padded segment width of a tile row */
  int32_t tile_dtype;            /* RB_BF16 / RB_F16 / RB_F32 */
  const int32_t* row_partition;  /* [H+1] */
  const int32_t* row_perm;       /* [n_rows] */
  const int32_t* blk_ptr;        /* [H+1] */
  const int32_t* blk_col;        /* [nb] */
  const int64_t* grp_tile_row;   /* [H] */
  const int32_t* col_bounds;     /* [n_seg+1] */
  const void* tiles;             /* [total_tile_rows x dp] */
  /* optional compact payloads of skinny block rows (rb_vbr_compact_*; NULL = none): block rows of
   * h <= cmp_h rows are multiplied from these instead of their tiles */
  const int64_t* cmp_ptr;        /* [n_rows+1] by permuted row */
  const int32_t* cmp_col;        /* [cmp_ptr[n_rows]] global columns */
  const float* cmp_val;          /* values rounded to tile_dtype */
  int32_t cmp_h;
} rb_vbr_device;

typedef struct rb_spmm_plan rb_spmm_plan;

typedef struct rb_spmm_info {
  int64_t n_items_tall;      /* (block row, 128-row M-tile, 256-col N-chunk) work items */
  int64_t n_items_short;     /* (block row, 256-col N-chunk) swap-AB work items (+ sweep steps) */
  int64_t n_items_simt;      /* fp32 check-path work items */
  double executed_flops;     /* 2 * sum over tiles of hp * dp * N_pad (MMA-padded work) */
  double vbr_flops;          /* 2 * stored_area * N (VBR-padded work) */
  int64_t row_begin_perm;    /* first permuted row covered by this shard (or -1 if empty) */
  int64_t n_items_skinny;    /* (block row, C-column slab) CUDA-core items for block rows with h <= 8 */
  int64_t n_launches;        /* kernel launches per rb_spmm_execute */
  double core_vbr_flops;     /* part of vbr_flops run on the CUDA cores (skinny / fp32 kernels) */
  int64_t n_sweep_steps;     /* block steps of the multi-slot sweep kernel (0: not used) */
  int64_t sweep_slots;       /* block rows resident in TMEM per CTA on the sweep kernel */
} rb_spmm_info;

int rb_spmm_plan_create(const rb_vbr_device* vbr, int64_t n_dense_cols, int32_t b_dtype, int32_t shard,
                        int32_t n_shards, rb_spmm_plan** plan, void* stream);
/* As rb_spmm_plan_create; work_shards (>= n_shards) = how many GPUs share the whole product when
 * `vbr` is itself one rank's sub-matrix (dist.shard_vbr): it sizes the parts that split hub rows. */
int rb_spmm_plan_create_ex(const rb_vbr_device* vbr, int64_t n_dense_cols, int32_t b_dtype, int32_t shard,
                           int32_t n_shards, int32_t work_shards, rb_spmm_plan** plan, void* stream);
int rb_spmm_plan_info(const rb_spmm_plan* plan, rb_spmm_info* info);
int rb_spmm_execute(const rb_spmm_plan* plan, const void* B, int64_t ldb, float* C, int64_t ldc, void* stream);
/* float64 path (plan made with b_dtype RB_F64 over RB_F64 tiles): C float64.  Every block row runs
 * on a CUDA-core FP64 kernel that multiplies the dense block payloads over exactly their segment
 * width, zeros included, as multiply.py:89 does — results within float64 rounding of the reference
 * and the same NaN / Inf propagation. */
int rb_spmm_execute_f64(const rb_spmm_plan* plan, const double* B, int64_t ldb, double* C, int64_t ldc,
                        void* stream);
/* Fused all-gather of C (north_star's optional collective): as rb_spmm_execute, and
 * every C element the kernels store is also stored, at the same offset, into peers[0..n_peers) —
 * the other ranks' full-size float32 C buffers mapped into this process over NVLink (P2P /
 * symmetric memory; any device pointers of C's layout work, e.g. several buffers on one GPU).  The
 * copies are written by the SpMM epilogues themselves, so the gather overlaps the math tile by tile
 * and needs no separate collective or un-permute pass.  c_rows (device int32 [plan n_rows], NULL =
 * the plan's row_perm) maps the plan's permuted row p to the output row c_rows[p]: a rank's
 * sub-matrix plan (dist.shard_vbr) passes the global source rows of its shard, so every buffer
 * receives the rank's rows exactly where multiply.py:90 puts them.  C, peers and ldc as in
 * rb_spmm_execute; with n_peers > 0 every pointer must be 16-byte aligned.  n_peers <= 7; not for
 * RB_F64 plans.  The caller orders the peers' reads after the writes (a barrier across ranks). */
int rb_spmm_execute_fanout(const rb_spmm_plan* plan, const void* B, int64_t ldb, float* C, int64_t ldc,
                           float* const* peers, int32_t n_peers, const int32_t* c_rows, void* stream);
int rb_spmm_plan_destroy(rb_spmm_plan* plan);
/* 2:4 sparse tensor-core form of the tall block rows (sparse24.cu): stage = 128 logical K of a
 * block row's padded block sequence; 64 compressed values + 4 TMEM metadata words per tile row and
 * stage; groups of 4 with more than two nonzeros spill into a residual CSR over permuted rows.
 *   rb_sparse24_layout       HOST sp_tile_row[H] (-1: not tall), total compressed rows, tall count
 *   rb_sparse24_workspace_size / rb_sparse24_emit   residual counts (res_ptr, device) and, given
 *                            buffers, the compressed tiles [total x 64], metadata [total x 8] u32,
 *                            residual columns (global) / values (float)
 *   rb_spmm_plan_attach_sparse24   switches a bf16/fp16 plan's tall rows to tcgen05.mma.sp plus the
 *                            residual pass (C += R·B).                                          */
typedef struct rb_sparse24_device {
  const void* sp_tiles;
  const uint32_t* sp_meta;
  const int64_t* sp_tile_row;   /* [H] device */
  int64_t total_sp_rows;
  const int64_t* res_ptr;       /* [n_rows + 1] device, permuted rows */
  const int32_t* res_col;
  const float* res_val;
  int64_t n_residuals;
} rb_sparse24_device;
int rb_sparse24_layout(const rb_vbr_device* vbr, int64_t* sp_tile_row_host, int64_t* total_sp_rows, int64_t* n_tall,
                       void* stream);
int rb_sparse24_workspace_size(int64_t n_rows, int64_t total_sp_rows, size_t* bytes);
int rb_sparse24_emit(const rb_vbr_device* vbr, const int64_t* sp_tile_row, const int32_t* tall_g,
                     const int64_t* thread_base, int32_t n_tall, int64_t total_threads, int64_t total_sp_rows,
                     void* workspace, size_t workspace_bytes, void* sp_tiles, uint32_t* sp_meta, int64_t* res_ptr,
                     int32_t* res_col, float* res_val, int64_t res_capacity, int64_t* n_residuals, void* stream);
int rb_spmm_plan_attach_sparse24(rb_spmm_plan* plan, const rb_sparse24_device* sp, void* stream);

/* Host-only shard planner (no device access): the contiguous range [*row_begin, *row_end) of
 * PERMUTED row positions owned by `shard`, given HOST copies of row_partition / blk_ptr.
 * rb_spmm_plan_create(..., shard, n_shards, ...) uses exactly this range; C rows
 * row_perm[row_begin:row_end] are produced by that shard and by no other.            */
int rb_spmm_shard_range(const int32_t* row_partition, const int32_t* blk_ptr, int64_t n_block_rows,
                        int32_t b_dtype, int32_t dp, int32_t shard, int32_t n_shards, int64_t* row_begin,
                        int64_t* row_end);

/* ------------------------------------------------------------------ spmm_csr
 * GPU comparator for spmm_csr(A, B, threads) (multiply.py:51-69): C = A·B straight from the
 * reference's CSR arrays (row_ptr/col_idx int64, values float64, device), C float32 [n_rows x N]
 * in row order (rows without nonzeros are exact zeros).  B as for rb_spmm_execute (RB_BF16/RB_F16/
 * RB_F32).  The plan (work list from a host copy of row_ptr) is reusable across B.            */
typedef struct rb_csr_plan rb_csr_plan;
int rb_csr_plan_create(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, int64_t n_dense_cols,
                       int32_t b_dtype, rb_csr_plan** plan, void* stream);
int rb_csr_execute(const rb_csr_plan* plan, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                   const void* B, int64_t ldb, float* C, int64_t ldc, void* stream);
int rb_csr_plan_destroy(rb_csr_plan* plan);

/* ------------------------------------------------------------------ blocking_stats / verify_density_bound
 * Replace blocking_stats (metrics.py:59-95) and verify_density_bound (metrics.py:178-216) for a
 * grouping in device memory (row_perm[n_rows] / group_ptr[H+1] as returned by rb_block_1sa,
 * pattern_ptr[H+1] / pattern_idx = RowGroup.pattern).  Per group g (device outputs, [H]):
 *   stored_cols[g]  = sum of the pattern's segment widths
 *   element_nnz[g]  = sum of the member rows' nnz
 *   quotient_nnz[g] = sum of the member rows' distinct segment counts
 *   ok[g]           = bit0 element_ok, bit1 quotient_ok, the reference's exact rational tests
 *                     k_elem/(h*stored_cols) >= tau/(2*max_width), k_quot/(h*lambda) >= tau/2
 *                     (empty patterns pass).
 * HOST totals: stored area, stored blocks, sum over blocks of the block height, violations.
 * Workspace: rb_group_stats_workspace_size.                                              */
int rb_group_stats_workspace_size(int64_t n_seg, size_t* bytes);
int rb_group_stats(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_idx,
                   const int64_t* boundaries, int64_t n_seg, const int64_t* row_perm, const int64_t* group_ptr,
                   const int64_t* pattern_ptr, const int64_t* pattern_idx, int64_t n_groups, double tau,
                   void* workspace, size_t workspace_bytes, int64_t* stored_cols, int64_t* element_nnz,
                   int64_t* quotient_nnz, uint8_t* ok, int64_t* stored_area, int64_t* n_blocks,
                   int64_t* height_sum, int64_t* n_violations, void* stream);

/* ------------------------------------------------------------------ helpers
 * Element conversion used by the drop-in path (DenseMatrix is float64, matrix.py:107-111):
 * dst[r, c] (row stride ldd, dtype dst_dtype) = src[r, c] (float64, row stride lds).   */
int rb_convert_f64(const double* src, int64_t rows, int64_t cols, int64_t lds, void* dst, int32_t dst_dtype,
                   int64_t ldd, void* stream);
/* rb_convert_f64 that also reports non-finite input: *nonfinite (device int32, caller-zeroed) is set
 * to 1 if any element of src is NaN or +-Inf.  The drop-in spmm_vbr raises ValueError on that
 * instead of returning the reference's NaN/Inf pattern (multiply.py:89 multiplies the dense block
 * payloads, zeros included, while the kernels skip zero tile entries and pad tiles to 64 columns). */
int rb_convert_f64_checked(const double* src, int64_t rows, int64_t cols, int64_t lds, void* dst, int32_t dst_dtype,
                           int64_t ldd, int32_t* nonfinite, void* stream);
/* float32 C → float64 (for DenseMatrix returns). */
int rb_widen_f32(const float* src, int64_t rows, int64_t cols, int64_t lds, double* dst, int64_t ldd,
                 void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ROWBLOCK_B200_H_ */
