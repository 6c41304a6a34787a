// Column-segment lookup shared by the 1-SA and VBR kernels.
//   segment_of(c) = searchsorted(boundaries, c, 'right') - 1        (matrix.py:164-166)
// Uniform partitions (ColumnPartition.uniform, matrix.py:144-150) use c / delta.
#pragma once
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace rb {

struct SegMap {
  const int32_t* bounds;  // [n_seg + 1] int32 (device)
  int32_t n_seg;
  int32_t delta;          // > 0: uniform width delta (last segment may be narrower); 0: binary search

  __device__ __forceinline__ int32_t operator()(int32_t c) const {
    if (delta > 0) return c / delta;
    int32_t lo = 0, hi = n_seg + 1;  // first index with bounds[i] > c
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (__ldg(bounds + mid) > c) hi = mid;
      else lo = mid + 1;
    }
    return lo - 1;
  }
};

// Copies the (small) boundaries array to the host to validate it and detect a uniform width.
// Returns RB_OK / error; fills delta (0 if not uniform) and max_width.
int inspect_boundaries(const int64_t* d_bounds, int64_t n_seg, int64_t n_cols, int32_t* delta, int32_t* max_width,
                       std::vector<int64_t>* host, cudaStream_t stream);

// int64 -> int32 boundaries on device.
int narrow_bounds(const int64_t* d_bounds, int64_t n_seg, int32_t* d_out, cudaStream_t stream);

}  // namespace rb
