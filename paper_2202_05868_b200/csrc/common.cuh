// Shared definitions for the rowblock B200 kernels.
#pragma once
#include <cstdint>
#include <cstdio>
#include <string>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/rowblock_b200.h"

namespace rb {

constexpr int kNumSMs = 148;

// Padded block-row height used by the device tile layout:
//   short block rows (h <= 128) are multiplied in swap-AB orientation, MMA N = hp,
//   padded to a power of two in [16, 128];
//   tall block rows (h > 128) are multiplied in M-tiles of 128 rows, hp = roundup(h, 128).
__host__ __device__ inline int32_t hp_of(int32_t h) {
  if (h <= 16) return 16;
  if (h <= 128) {
    int32_t p = 16;
    while (p < h) p <<= 1;
    return p;
  }
  return (h + 127) / 128 * 128;
}
__host__ __device__ inline bool is_short_row(int32_t h) { return h <= 128; }
// Row pitch of a block row's tiles in the tile array: block rows of h <= 8 rows (CUDA-core skinny
// kernels; config 3 / 2b are almost all h = 1) store exactly h rows per tile instead of hp = 16, so
// their tiles are 16x smaller and contiguous.  The swap-AB tensor-core kernel, when it does take
// such a block row, reads hp rows from the pitch-spaced start: rows h..hp-1 then belong to the next
// tiles (or are TMA zero fill) and only feed accumulator rows the epilogue never stores.
__host__ __device__ inline int32_t tile_pitch(int32_t h) { return h <= 8 ? h : hp_of(h); }

// NVTX range over one C-ABI call (1-SA, VBR build, SpMM, ...): named stages on an nsys / ncu timeline;
// header-only NVTX v3, a no-op unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Fused all-gather of C (rb_spmm_execute_fanout): every C store of the SpMM kernels is repeated
// into up to RB_MAX_FAN further buffers of C's layout at the same element offset.  The buffers are
// the other ranks' full-size C, mapped into this process (NVLink P2P / symmetric memory), so a rank
// writes its rows, already in source row order, straight into every peer's C: the all-gather and
// the un-permute of multiply.py:90 ride on the epilogue's own stores.  n = 0: plain stores.
constexpr int RB_MAX_FAN = 7;
struct CFan {
  float* p[RB_MAX_FAN];
  int32_t n;
};

// Thread-local error string for rb_last_error_string().
void set_error(const std::string& s);
int fail(int code, const std::string& s);

}  // namespace rb

#define RB_CUDA_TRY(expr)                                                                      \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess)                                                                     \
      return ::rb::fail(_e == cudaErrorMemoryAllocation ? RB_ENOMEM : RB_ECUDA,                \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));                   \
  } while (0)
