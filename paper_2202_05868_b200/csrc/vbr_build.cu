// VBR build on the device (K4): replaces vbr_from_grouping (vbr.py:88-125).
//
//   rb_vbr_plan : row -> (block row, local row) maps, per-block-row segment bitsets recomputed
//                 from the data (vbr.py:106-112), block counts, blk_ptr, tile row offsets.
//   rb_vbr_emit : blk_col (ascending per block row) and the zero-padded dense tiles, one pass
//                 over the nonzeros (vbr.py:113-123), converted to the tile dtype.
#include <cub/device/device_scan.cuh>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <vector>

#include "common.cuh"
#include "segments.cuh"

namespace rb {

namespace {

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct VbrWs {
  int32_t* group_of_row;  // [n]
  int32_t* pos_of_row;    // [n]
  unsigned long long* gbits;  // [H*W]
  unsigned long long* rbits;  // [n*W] per-row segment bits
  int32_t* wprefix;       // [H*W]
  int32_t* blk_cnt;       // [H+1]
  int64_t* tile_cnt;      // [H+1]
  int32_t* err;           // [4]
  int32_t* b32;           // [n_seg+1] narrowed boundaries
  void* cub_tmp;
  size_t cub_bytes;
  size_t total;
};

size_t cub_scan_bytes(int64_t n) {
  size_t a = 0, b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, (int)std::max<int64_t>(n, 1));
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int)std::max<int64_t>(n, 1));
  return std::max(a, b);
}

VbrWs carve(void* base, int64_t n, int64_t H, int64_t W, int64_t n_seg) {
  VbrWs w;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    void* p = base ? static_cast<char*>(base) + off : nullptr;
    off += align256(bytes);
    return p;
  };
  w.group_of_row = (int32_t*)take(sizeof(int32_t) * std::max<int64_t>(n, 1));
  w.pos_of_row = (int32_t*)take(sizeof(int32_t) * std::max<int64_t>(n, 1));
  w.gbits = (unsigned long long*)take(sizeof(uint64_t) * std::max<int64_t>(H * W, 1));
  w.rbits = (unsigned long long*)take(sizeof(uint64_t) * std::max<int64_t>(n * W, 1));
  w.wprefix = (int32_t*)take(sizeof(int32_t) * std::max<int64_t>(H * W, 1));
  w.blk_cnt = (int32_t*)take(sizeof(int32_t) * (H + 1));
  w.tile_cnt = (int64_t*)take(sizeof(int64_t) * (H + 1));
  w.err = (int32_t*)take(sizeof(int32_t) * 4);
  w.b32 = (int32_t*)take(sizeof(int32_t) * (n_seg + 1));
  w.cub_bytes = cub_scan_bytes(H + 1);
  w.cub_tmp = take(w.cub_bytes);
  w.total = off;
  return w;
}

inline int64_t words_of(int64_t n_seg) { return n_seg > 0 ? (n_seg + 63) / 64 : 1; }

// position p of the permutation -> (row, group); validates the permutation.
__global__ void positions_kernel(const int64_t* __restrict__ row_perm, const int64_t* __restrict__ row_partition,
                                 int64_t n, int64_t H, int32_t* group_of_row, int32_t* pos_of_row, int32_t* perm32,
                                 int32_t* err) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = H + 1;  // first index with row_partition[i] > p
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (row_partition[mid] > p) hi = mid;
      else lo = mid + 1;
    }
    const int64_t g = lo - 1;
    const int64_t r = row_perm[p];
    if (r < 0 || r >= n || g < 0 || g >= H) {
      atomicExch(err, 1);
      continue;
    }
    const int old = atomicExch(pos_of_row + r, (int32_t)p);
    if (old != -1) atomicExch(err, 2);
    group_of_row[r] = (int32_t)g;
    perm32[p] = (int32_t)r;
  }
}

__global__ void rpart_kernel(const int64_t* __restrict__ row_partition, int64_t H, int32_t* rpart32, int32_t* err,
                             int64_t n) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g <= H; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = row_partition[g];
    rpart32[g] = (int32_t)v;
    if ((g == 0 && v != 0) || (g == H && v != n) || (g > 0 && v <= row_partition[g - 1])) atomicExch(err, 3);
  }
}

// Stored block columns of a block row (vbr.py:108-112) = OR of its rows' segment bitsets.
// Pass 1 (row_bits_kernel): warp per row, segment bits of that row (atomics only within the row).
// Pass 2 (group_or_kernel): warp per chunk of 256 permuted positions; lane w ORs word w of the
// chunk's rows in registers and flushes one atomicOr per (block row, word) it touched, so a single
// huge block row (config 2: 32768 rows in one group) does not serialise on 8 words.
__global__ void row_bits_kernel(const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col_idx, int64_t n,
                                SegMap seg, int64_t W, unsigned long long* rbits) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const int64_t s0 = row_ptr[r], s1 = row_ptr[r + 1];
    unsigned long long* rb = rbits + r * W;
    for (int64_t j = s0 + lane; j < s1; j += 32) {
      const int32_t s = seg((int32_t)col_idx[j]);
      // columns strictly increase, so segments are non-decreasing: OR once per segment run
      if (j == s0 || seg((int32_t)col_idx[j - 1]) != s) atomicOr(rb + (s >> 6), 1ull << (s & 63));
    }
  }
}

constexpr int kOrChunk = 256;
__global__ void group_or_kernel(const unsigned long long* __restrict__ rbits, const int32_t* __restrict__ perm32,
                                const int32_t* __restrict__ group_of_row, int64_t n, int64_t W,
                                unsigned long long* gbits) {
  const int lane = threadIdx.x & 31;
  const int64_t n_chunks = (n + kOrChunk - 1) / kOrChunk;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); c < n_chunks; c += warps) {
    const int64_t p0 = c * kOrChunk, p1 = min(n, p0 + kOrChunk);
    for (int64_t w0 = 0; w0 < W; w0 += 32) {
      const int64_t w = w0 + lane;
      unsigned long long acc = 0;
      int32_t g_cur = group_of_row[perm32[p0]];
      for (int64_t p = p0; p < p1; ++p) {
        const int32_t r = perm32[p];
        const int32_t g = group_of_row[r];
        if (g != g_cur) {
          if (w < W && acc) atomicOr(gbits + (int64_t)g_cur * W + w, acc);
          acc = 0;
          g_cur = g;
        }
        if (w < W) acc |= rbits[(int64_t)r * W + w];
      }
      if (w < W && acc) atomicOr(gbits + (int64_t)g_cur * W + w, acc);
    }
  }
}

// warp per block row: block count and exclusive per-word popcount prefix
__global__ void count_kernel(const unsigned long long* __restrict__ gbits, int64_t H, int64_t W,
                             const int64_t* __restrict__ row_partition, int32_t* wprefix, int32_t* blk_cnt,
                             int64_t* tile_cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); g < H; g += warps) {
    int32_t running = 0;
    for (int64_t w0 = 0; w0 < W; w0 += 32) {
      const int64_t w = w0 + lane;
      const int c = w < W ? __popcll(gbits[g * W + w]) : 0;
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (w < W) wprefix[g * W + w] = running + incl - c;
      running += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      blk_cnt[g] = running;
      const int32_t h = (int32_t)(row_partition[g + 1] - row_partition[g]);
      tile_cnt[g] = (int64_t)running * tile_pitch(h);
    }
  }
}

__global__ void blkcol_kernel(const unsigned long long* __restrict__ gbits, const int32_t* __restrict__ wprefix,
                              const int32_t* __restrict__ blk_ptr, int64_t H, int64_t W, int32_t* blk_col) {
  const int64_t total = H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = i / W, w = i - g * W;
    unsigned long long x = gbits[i];
    int32_t k = blk_ptr[g] + wprefix[i];
    while (x) {
      const int b = __ffsll((long long)x) - 1;
      blk_col[k++] = (int32_t)(w * 64 + b);
      x &= x - 1;
    }
  }
}

template <typename T>
__device__ __forceinline__ T cvt(double v);
template <>
__device__ __forceinline__ float cvt<float>(double v) { return (float)v; }
template <>
__device__ __forceinline__ double cvt<double>(double v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(double v) { return __double2bfloat16(v); }
template <>
__device__ __forceinline__ __half cvt<__half>(double v) { return __double2half(v); }

// warp per row: scatter values into tiles (vbr.py:117-123)
template <typename T>
__global__ void scatter_kernel(const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col_idx,
                               const double* __restrict__ values, int64_t n, SegMap seg,
                               const int32_t* __restrict__ group_of_row, const int32_t* __restrict__ pos_of_row,
                               const int32_t* __restrict__ rpart, const unsigned long long* __restrict__ gbits,
                               const int32_t* __restrict__ wprefix, const int64_t* __restrict__ grp_tile_row,
                               int64_t W, int32_t dp, T* tiles) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const int64_t s0 = row_ptr[r], s1 = row_ptr[r + 1];
    if (s1 == s0) continue;
    const int32_t g = group_of_row[r];
    const int32_t local = pos_of_row[r] - rpart[g];
    const int32_t hp = tile_pitch(rpart[g + 1] - rpart[g]);  // row pitch of this block row's tiles
    const int64_t base = grp_tile_row[g];
    const unsigned long long* gb = gbits + (int64_t)g * W;
    const int32_t* wp = wprefix + (int64_t)g * W;
    for (int64_t j = s0 + lane; j < s1; j += 32) {
      const int32_t c = (int32_t)col_idx[j];
      const int32_t s = seg(c);
      const int32_t rank = wp[s >> 6] + __popcll(gb[s >> 6] & ((1ull << (s & 63)) - 1ull));
      const int32_t c0 = seg.delta > 0 ? s * seg.delta : __ldg(seg.bounds + s);
      tiles[(base + (int64_t)rank * hp + local) * dp + (c - c0)] = cvt<T>(values[j]);
    }
  }
}

inline unsigned grid_for(int64_t work, int per_block) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + per_block - 1) / per_block, 148 * 16));
}

}  // namespace
}  // namespace rb

using namespace rb;

extern "C" int rb_vbr_workspace_size(int64_t n_rows, int64_t n_groups, int64_t n_seg, size_t* bytes) {
  if (!bytes || n_rows < 0 || n_groups < 0 || n_seg < 0) return fail(RB_EINVAL, "bad arguments");
  *bytes = carve(nullptr, n_rows, n_groups, words_of(n_seg), n_seg).total;
  return RB_OK;
}

extern "C" int rb_vbr_plan(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_idx,
                           const int64_t* boundaries, int64_t n_seg, const int64_t* row_perm,
                           const int64_t* row_partition, int64_t H, void* workspace, size_t ws_bytes, int32_t* perm32,
                           int32_t* rpart32, int32_t* blk_ptr, int64_t* grp_tile_row, int32_t* bounds32,
                           int64_t* n_blocks, int64_t* total_tile_rows, void* stream_) {
  rb::NvtxRange nvtx_range_("rb_vbr_plan");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (n_rows < 0 || H < 0 || !n_blocks || !total_tile_rows) return fail(RB_EINVAL, "bad arguments");
  if (n_rows >= (int64_t(1) << 31)) return fail(RB_EUNSUPPORTED, "n_rows must be < 2^31");
  if (H > n_rows || (n_rows > 0 && H == 0)) return fail(RB_EINVAL, "grouping/partition inconsistent with matrix dimensions");
  const int64_t W = words_of(n_seg);
  VbrWs ws = carve(workspace, n_rows, H, W, n_seg);
  if (ws_bytes < ws.total) return fail(RB_EINVAL, "workspace too small");
  int32_t delta = 0, maxw = 0;
  int rc = inspect_boundaries(boundaries, n_seg, n_cols, &delta, &maxw, nullptr, stream);
  if (rc) return rc;
  rc = narrow_bounds(boundaries, n_seg, bounds32, stream);
  if (rc) return rc;
  SegMap seg{bounds32, (int32_t)n_seg, delta};

  RB_CUDA_TRY(cudaMemsetAsync(ws.err, 0, sizeof(int32_t) * 4, stream));
  RB_CUDA_TRY(cudaMemsetAsync(ws.pos_of_row, 0xFF, sizeof(int32_t) * std::max<int64_t>(n_rows, 1), stream));
  RB_CUDA_TRY(cudaMemsetAsync(ws.gbits, 0, sizeof(uint64_t) * std::max<int64_t>(H * W, 1), stream));
  rpart_kernel<<<grid_for(H + 1, 256), 256, 0, stream>>>(row_partition, H, rpart32, ws.err, n_rows);
  if (n_rows > 0) {
    positions_kernel<<<grid_for(n_rows, 256), 256, 0, stream>>>(row_perm, row_partition, n_rows, H, ws.group_of_row,
                                                                ws.pos_of_row, perm32, ws.err);
    RB_CUDA_TRY(cudaMemsetAsync(ws.rbits, 0, sizeof(uint64_t) * n_rows * W, stream));
    row_bits_kernel<<<grid_for(n_rows, 8), 256, 0, stream>>>(row_ptr, col_idx, n_rows, seg, W, ws.rbits);
    group_or_kernel<<<grid_for((n_rows + kOrChunk - 1) / kOrChunk, 8), 256, 0, stream>>>(
        ws.rbits, perm32, ws.group_of_row, n_rows, W, ws.gbits);
  }
  if (H > 0)
    count_kernel<<<grid_for(H, 8), 256, 0, stream>>>(ws.gbits, H, W, row_partition, ws.wprefix, ws.blk_cnt,
                                                     ws.tile_cnt);
  RB_CUDA_TRY(cudaGetLastError());
  // exclusive scans over H+1 entries (last entry counts 0 -> total)
  RB_CUDA_TRY(cudaMemsetAsync(ws.blk_cnt + H, 0, sizeof(int32_t), stream));
  RB_CUDA_TRY(cudaMemsetAsync(ws.tile_cnt + H, 0, sizeof(int64_t), stream));
  size_t tb = ws.cub_bytes;
  RB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws.cub_tmp, tb, ws.blk_cnt, blk_ptr, (int)(H + 1), stream));
  tb = ws.cub_bytes;
  int64_t* scan_out = ws.tile_cnt;  // in-place exclusive scan (cub supports d_in == d_out)
  RB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws.cub_tmp, tb, ws.tile_cnt, scan_out, (int)(H + 1), stream));
  if (H > 0) RB_CUDA_TRY(cudaMemcpyAsync(grp_tile_row, scan_out, sizeof(int64_t) * H, cudaMemcpyDeviceToDevice, stream));
  int32_t err[4];
  int32_t nb32 = 0;
  int64_t rows64 = 0;
  RB_CUDA_TRY(cudaMemcpyAsync(err, ws.err, sizeof(err), cudaMemcpyDeviceToHost, stream));
  RB_CUDA_TRY(cudaMemcpyAsync(&nb32, blk_ptr + H, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
  RB_CUDA_TRY(cudaMemcpyAsync(&rows64, scan_out + H, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  RB_CUDA_TRY(cudaStreamSynchronize(stream));
  if (err[0] == 3) return fail(RB_EINVAL, "row_partition must be strictly increasing from 0 to n_rows");
  if (err[0] != 0) return fail(RB_EINVAL, "row_perm is not a permutation consistent with row_partition");
  *n_blocks = nb32;
  *total_tile_rows = rows64;
  return RB_OK;
}

extern "C" int rb_vbr_emit(int64_t n_rows, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                           const int64_t* boundaries, int64_t n_seg, int64_t H, void* workspace, size_t ws_bytes,
                           const int32_t* perm32, const int32_t* rpart32, const int32_t* blk_ptr,
                           const int64_t* grp_tile_row, int32_t* blk_col, void* tiles, int32_t tile_dtype, int32_t dp,
                           int64_t total_tile_rows, void* stream_) {
  rb::NvtxRange nvtx_range_("rb_vbr_emit");
  (void)perm32;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const int64_t W = words_of(n_seg);
  VbrWs ws = carve(workspace, n_rows, H, W, n_seg);
  if (ws_bytes < ws.total) return fail(RB_EINVAL, "workspace too small");
  int32_t delta = 0, maxw = 0;
  int rc = inspect_boundaries(boundaries, n_seg, /*n_cols: from boundaries*/ -1, &delta, &maxw, nullptr, stream);
  if (rc) return rc;
  if (dp < maxw) return fail(RB_EINVAL, "dp smaller than the widest segment");
  if ((tile_dtype == RB_BF16 || tile_dtype == RB_F16) && dp % 64 != 0)
    return fail(RB_EINVAL, "dp must be a multiple of 64 for 16-bit tiles");
  if (H > 0)
    blkcol_kernel<<<grid_for(H * W, 256), 256, 0, stream>>>(ws.gbits, ws.wprefix, blk_ptr, H, W, blk_col);
  RB_CUDA_TRY(cudaGetLastError());
  if (!tiles || total_tile_rows <= 0) return RB_OK;
  size_t esz = tile_dtype == RB_F64 ? 8 : tile_dtype == RB_F32 ? 4 : 2;
  RB_CUDA_TRY(cudaMemsetAsync(tiles, 0, esz * (size_t)total_tile_rows * dp, stream));
  if (n_rows == 0) return RB_OK;
  rc = narrow_bounds(boundaries, n_seg, ws.b32, stream);
  if (rc) return rc;
  SegMap seg{ws.b32, (int32_t)n_seg, delta};
  const unsigned grid = grid_for(n_rows, 8);
  switch (tile_dtype) {
    case RB_BF16:
      scatter_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(row_ptr, col_idx, values, n_rows, seg, ws.group_of_row,
                                                              ws.pos_of_row, rpart32, ws.gbits, ws.wprefix, grp_tile_row,
                                                              W, dp, (__nv_bfloat16*)tiles);
      break;
    case RB_F16:
      scatter_kernel<__half><<<grid, 256, 0, stream>>>(row_ptr, col_idx, values, n_rows, seg, ws.group_of_row,
                                                       ws.pos_of_row, rpart32, ws.gbits, ws.wprefix, grp_tile_row, W,
                                                       dp, (__half*)tiles);
      break;
    case RB_F32:
      scatter_kernel<float><<<grid, 256, 0, stream>>>(row_ptr, col_idx, values, n_rows, seg, ws.group_of_row,
                                                      ws.pos_of_row, rpart32, ws.gbits, ws.wprefix, grp_tile_row, W,
                                                      dp, (float*)tiles);
      break;
    case RB_F64:
      scatter_kernel<double><<<grid, 256, 0, stream>>>(row_ptr, col_idx, values, n_rows, seg, ws.group_of_row,
                                                       ws.pos_of_row, rpart32, ws.gbits, ws.wprefix, grp_tile_row, W,
                                                       dp, (double*)tiles);
      break;
    default:
      return fail(RB_EINVAL, "bad tile dtype");
  }
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}

// ------------------------------------------------------------------------------------------
// Compact payloads of skinny block rows.  A block row of h <= h_max rows (config 3 / 2b: almost
// all h = 1) stores tiles that are mostly the zero padding of its blocks' segments: config 3 holds
// 1.2 nonzeros per 32-wide block.  Beside the tiles, K4 emits the same payload without the padding:
// for every permuted row p of such a block row, its nonzeros (global column int32, value rounded to
// the tile dtype and held in a float) in cmp_ptr[p] .. cmp_ptr[p+1] — the block payloads in
// block-column order, zeros dropped.  The SpMM multiplies these block rows by gathering only those
// B rows (the CSR engine of spmm_skinny.cu), reading ~8 B of A per nonzero instead of a 16-byte
// tile row segment per block.
namespace rb {
namespace {

__global__ void compact_count_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ perm32,
                                     const int32_t* __restrict__ rpart32, int64_t H, int32_t h_max,
                                     int64_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; g < H;
       g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t lo = rpart32[g], hi = rpart32[g + 1];
    const bool take = hi - lo <= h_max;
    for (int32_t p = lo + lane; p < hi; p += 32) {
      const int32_t r = perm32[p];
      cnt[p] = take ? row_ptr[r + 1] - row_ptr[r] : 0;
    }
  }
}

template <typename T>
__global__ void compact_emit_kernel(const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col_idx,
                                    const double* __restrict__ values, const int32_t* __restrict__ perm32, int64_t n,
                                    const int64_t* __restrict__ cmp_ptr, int32_t* __restrict__ cmp_col,
                                    float* __restrict__ cmp_val) {
  const int lane = threadIdx.x & 31;
  for (int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; p < n;
       p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t o = cmp_ptr[p], c = cmp_ptr[p + 1] - o;
    if (c == 0) continue;
    const int64_t s = row_ptr[perm32[p]];
    for (int64_t j = lane; j < c; j += 32) {
      cmp_col[o + j] = (int32_t)col_idx[s + j];
      cmp_val[o + j] = (float)cvt<T>(values[s + j]);
    }
  }
}

}  // namespace
}  // namespace rb

extern "C" int rb_vbr_compact_count(int64_t n_rows, const int64_t* row_ptr, const int32_t* perm32,
                                    const int32_t* rpart32, int64_t n_groups, int32_t h_max, int64_t* cmp_ptr,
                                    int64_t* total, void* stream_) {
  rb::NvtxRange nvtx_range_("rb_vbr_compact_count");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (n_rows < 0 || n_groups < 0 || !cmp_ptr || !total) return fail(RB_EINVAL, "bad arguments");
  RB_CUDA_TRY(cudaMemsetAsync(cmp_ptr, 0, sizeof(int64_t) * (n_rows + 1), stream));
  if (n_rows > 0 && n_groups > 0) {
    const unsigned grid = (unsigned)std::min<int64_t>((n_groups + 7) / 8, 148 * 32);
    rb::compact_count_kernel<<<grid, 256, 0, stream>>>(row_ptr, perm32, rpart32, n_groups, h_max, cmp_ptr + 1);
    RB_CUDA_TRY(cudaGetLastError());
    size_t tb = 0;
    RB_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tb, cmp_ptr + 1, cmp_ptr + 1, (int)n_rows, stream));
    void* tmp = nullptr;
    RB_CUDA_TRY(cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), stream));
    const cudaError_t e = cub::DeviceScan::InclusiveSum(tmp, tb, cmp_ptr + 1, cmp_ptr + 1, (int)n_rows, stream);
    RB_CUDA_TRY(cudaFreeAsync(tmp, stream));
    RB_CUDA_TRY(e);
  }
  RB_CUDA_TRY(cudaMemcpyAsync(total, cmp_ptr + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  RB_CUDA_TRY(cudaStreamSynchronize(stream));
  return RB_OK;
}

extern "C" int rb_vbr_compact_emit(int64_t n_rows, const int64_t* row_ptr, const int64_t* col_idx,
                                   const double* values, const int32_t* perm32, const int64_t* cmp_ptr,
                                   int32_t tile_dtype, int32_t* cmp_col, float* cmp_val, void* stream_) {
  rb::NvtxRange nvtx_range_("rb_vbr_compact_emit");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (n_rows < 0 || !cmp_ptr) return fail(RB_EINVAL, "bad arguments");
  if (n_rows == 0) return RB_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((n_rows + 7) / 8, 148 * 32);
  switch (tile_dtype) {
    case RB_BF16:
      rb::compact_emit_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(row_ptr, col_idx, values, perm32, n_rows,
                                                                       cmp_ptr, cmp_col, cmp_val);
      break;
    case RB_F16:
      rb::compact_emit_kernel<__half><<<grid, 256, 0, stream>>>(row_ptr, col_idx, values, perm32, n_rows, cmp_ptr,
                                                                cmp_col, cmp_val);
      break;
    case RB_F32:
      rb::compact_emit_kernel<float><<<grid, 256, 0, stream>>>(row_ptr, col_idx, values, perm32, n_rows, cmp_ptr,
                                                               cmp_col, cmp_val);
      break;
    default: return fail(RB_EINVAL, "compact payloads need a bf16 / f16 / f32 tile dtype");
  }
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}
