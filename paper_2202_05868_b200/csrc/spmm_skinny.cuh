// Skinny block rows (h <= 8): VBR SpMM on the CUDA cores, skipping the tiles' zero columns.
// See spmm_skinny.cu.
#pragma once
#include <cstdint>
#include <vector>

#include "common.cuh"

#include <cuda_runtime.h>

namespace rb {

// One unit of skinny work: blocks [bb, be) of block row g, C columns [n0, n0 + cols).  A block row
// with many blocks (power-law hubs) is cut into `nparts` parts; part p parks its h x cols fp32
// partial at ws + (wsoff + p * h_class * cols / 128) * 128 floats and the last-arriving part sums
// all partials in part order (deterministic) into C.  nparts == 1: C is written directly.
struct SkinnyItem {
  int32_t g, n0, bb, be;
  int32_t part, nparts, slot, wsoff;
};

struct SkinnyArgs {
  const int32_t* row_partition;
  const int32_t* row_perm;
  const int32_t* blk_ptr;
  const int32_t* blk_col;
  const int64_t* grp_tile_row;
  const int32_t* col_bounds;
  const SkinnyItem* items;
  int64_t n_items;
  const void* tiles;
  int32_t dp;
  const void* B;
  int64_t ldb;
  float* C;
  int64_t ldc;
  int32_t N;
  float* ws;      // split-row partials
  int32_t* cnt;   // split-row arrival counters (zero between launches)
  int32_t accumulate;  // 1: C += result (2:4 residual pass), 0: C = result
  CFan fan;            // further copies of every C store (fused all-gather); fan.n = 0: none
};

// CSR operand of the comparator kernel (spmm_csr): the reference's CsrMatrix arrays on the device.
struct CsrArgs {
  const int64_t* row_ptr;
  const int64_t* col_idx;
  const double* values;
  const int32_t* col32;  // alternative operand (2:4 residuals): int32 columns, float values
  const float* val32;
  int32_t chunk;  // items claimed per atomic (csr_claim_chunk; 0 / 1 = one at a time)
};

// Items per claim for a CSR work list: 2 when the list is uniform (no split rows, longest item at
// most twice the mean), else 1.  Pairs hold consecutive items, i.e. the C-column slabs of one row.
// A compile-time chunk for every list (profiles/r02/chunk_ab/) cost config 3 2.4x at 4 and 1.3x
// at 2: its split hub rows' parts are consecutive items, and one group then runs them serially.
// Config 1 has fewer items than resident groups and lost too.  The bench configs' lists all hold
// split rows, so they run at chunk 1.
int csr_claim_chunk(const std::vector<SkinnyItem>& items);

// Height classes: block rows with h <= 1, 2, 4, 8 run the instance with H = 1, 2, 4, 8.
constexpr int SKINNY_CLASSES = 4;
constexpr int SKINNY_PART_BLOCKS = 256;  // blocks per part of a split block row
inline int skinny_class(int h) { return h <= 1 ? 0 : h <= 2 ? 1 : h <= 4 ? 2 : 3; }
inline int skinny_class_h(int cls) { return 1 << cls; }

// C columns covered by one item: 16-byte loads of B per lane, 32 (or 16 when N is small) lanes.
int skinny_cols(int32_t b_dtype, int64_t N);

// Appends the items of block row g (h rows, nb blocks starting at blk_begin) for every C-column
// slab; rows with more than SKINNY_PART_BLOCKS blocks are split (slot / workspace bookkeeping in
// n_slots and ws_units, in 128-float units).
void skinny_items_for_row(int32_t g, int h, int32_t blk_begin, int nb, int64_t N, int cols,
                          std::vector<SkinnyItem>& out, int64_t& n_slots, int64_t& ws_units,
                          int part_blocks = SKINNY_PART_BLOCKS);

// Launches the class-`cls` kernel over a.items[0 .. a.n_items) (persistent grid; `sched` = two
// zero-initialised device counters owned by the plan, reset by the kernel itself on exit).
int launch_skinny(const SkinnyArgs& a, int32_t b_dtype, int cls, unsigned long long* sched, cudaStream_t stream);

// CSR comparator: items are (row, C-column slab, nonzero range relative to row_ptr[row]); a.row_perm
// must be null (C rows = A rows).
int launch_csr(const SkinnyArgs& a, const CsrArgs& c, int32_t b_dtype, unsigned long long* sched,
               cudaStream_t stream);

}  // namespace rb
