// 2:4-structured form of the tall VBR tiles for the sparse tensor-core path (tcgen05.mma.sp).
//
// A tall block row (h > 128) is multiplied as a sequence of "stages" of 128 logical K columns of
// its padded block sequence (block t, column c  <->  logical k = t*dp + c).  Per stage and tile row
// every group of 4 logical columns keeps its first two nonzeros (2:4) in a compressed row of 64
// values (128 B, one SW128 TMA row); groups with more than two nonzeros (rare on the inputs 1-SA
// leaves to the tall kernel: 6e-4 of the groups of config 2) spill the rest into a residual CSR
// over permuted rows that a CUDA-core pass adds to C after the tensor-core pass.
//
// Layout (per tall block row g, hs = roundup(h, 256) rows, S_g = ceil(nb_g * dp / 128) stages):
//   sp_tiles [sp_tile_row[g] + s*hs + r][64]   compressed values (bf16/fp16), rows >= h are zero
//   sp_meta  [(sp_tile_row[g] + s*hs + 128*q + L) * 8 + 4*(j/2) + j%2]  uint32 (words 2,3,6,7 zero):
//            the TMEM metadata word of lane L (of the 128-row group q) for the j-th K=32 MMA of the
//            stage.  Two 16-byte planes per row, one tcgen05.cp 128x128b each; the MMA reads its word
//            at a 4-column-aligned TMEM address with idesc sparse_id2 = j%2 (tools/sp_probe).
//            Word layout (f16 sparse, verified by tools/sp_probe): lane L = m0 + 8*k1 + 16*m2 holds rows
//            m = m0 + 8*m1 + 16*m2 (m1 = 0, 1) at bits 16*m1 + k0 for logical k = 16*k1 + k0;
//            each 4-bit nibble = (i1 << 2) | i0, the kept positions of a group of 4.
//   res_ptr [n_rows + 1] (permuted rows), res_col (global column), res_val (float).
#include <cub/device/device_scan.cuh>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <vector>

#include "common.cuh"

namespace rb {
namespace {

constexpr int SP_STAGE_K = 128;  // logical K per stage
constexpr int SP_PHYS = 64;      // compressed values per stage row

struct SpArgs {
  const int32_t* rpart;
  const int32_t* perm;
  const int32_t* blk_ptr;
  const int32_t* blk_col;
  const int64_t* grp_tile_row;
  const int32_t* col_bounds;
  const int64_t* sp_tile_row;  // [H], -1 if not tall
  const int32_t* tall_g;       // [n_tall] block rows with h > 128
  int32_t n_tall;
  int32_t dp;
};

template <typename T>
__device__ __forceinline__ uint16_t bits_of(T v) {
  uint16_t b;
  memcpy(&b, &v, 2);
  return b;
}

// One thread per (tall block row, tile row r < hs).  MODE 0: count residuals of the row into
// res_cnt[perm position].  MODE 1: write compressed rows, nibbles (tmp, 4 words per stage row,
// chunk order) and residuals at res_ptr.
template <typename T, int MODE>
__global__ void __launch_bounds__(256) sp24_rows_kernel(SpArgs a, const T* __restrict__ tiles, T* sp_tiles,
                                                        uint32_t* nib_tmp, int64_t* res_cnt, const int64_t* res_ptr,
                                                        int32_t* res_col, float* res_val, int64_t total_threads,
                                                        const int64_t* thread_base) {
  for (int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; tid < total_threads;
       tid += (int64_t)gridDim.x * blockDim.x) {
    // locate (tall index i, row r) by binary search over thread_base[n_tall + 1]
    int lo = 0, hi = a.n_tall;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (thread_base[mid] <= tid) lo = mid;
      else hi = mid;
    }
    const int g = a.tall_g[lo];
    const int r = (int)(tid - thread_base[lo]);
    const int p0 = a.rpart[g], h = a.rpart[g + 1] - p0;
    const int hs = (h + 255) / 256 * 256;
    const int hp = hp_of(h);
    const int b0 = a.blk_ptr[g], nb = a.blk_ptr[g + 1] - b0;
    const int dp = a.dp;
    const int S = (nb * dp + SP_STAGE_K - 1) / SP_STAGE_K;
    const int64_t tbase = a.grp_tile_row[g];
    const bool live = r < h;
    int64_t out = MODE == 1 && live ? res_ptr[p0 + r] : 0;
    int64_t cnt = 0;
    for (int s = 0; s < S; ++s) {
      T vals[SP_STAGE_K];
      uint32_t words[4] = {0u, 0u, 0u, 0u};
      T comp[SP_PHYS];
#pragma unroll 4
      for (int q = 0; q < SP_STAGE_K; q += 8) {  // 8 logical columns (16 B) at a time
        const int k = s * SP_STAGE_K + q;
        const int t = k / dp, c = k - t * dp;
        uint4 u = make_uint4(0u, 0u, 0u, 0u);
        if (live && t < nb) u = *reinterpret_cast<const uint4*>(tiles + (tbase + (int64_t)t * hp + r) * dp + c);
        memcpy(&vals[q], &u, 16);
      }
      for (int ch = 0; ch < SP_STAGE_K / 4; ++ch) {
        int pos[4], np = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (bits_of(vals[4 * ch + i]) & 0x7fffu) pos[np++] = i;
        int i0, i1;
        if (np == 0) {
          i0 = 0;
          i1 = 1;
        } else if (np == 1) {
          i0 = pos[0] < 3 ? pos[0] : 2;
          i1 = i0 + 1;
        } else {
          i0 = pos[0];
          i1 = pos[1];
        }
        if (MODE == 1) {
          comp[2 * ch] = vals[4 * ch + i0];
          comp[2 * ch + 1] = vals[4 * ch + i1];
          words[ch >> 3] |= (uint32_t)((i1 << 2) | i0) << (4 * (ch & 7));
        }
        for (int e = 2; e < np; ++e) {
          if (MODE == 1) {
            const int k = s * SP_STAGE_K + 4 * ch + pos[e];
            const int t = k / dp, c = k - t * dp;
            res_col[out] = a.col_bounds[a.blk_col[b0 + t]] + c;
            res_val[out] = (float)vals[4 * ch + pos[e]];
            ++out;
          }
          ++cnt;
        }
      }
      if (MODE == 1) {
        const int64_t row = a.sp_tile_row[g] + (int64_t)s * hs + r;
        uint4* dst = reinterpret_cast<uint4*>(sp_tiles + row * SP_PHYS);
#pragma unroll
        for (int v = 0; v < SP_PHYS / 8; ++v) {
          uint4 u;
          memcpy(&u, &comp[8 * v], 16);
          dst[v] = u;
        }
        reinterpret_cast<uint4*>(nib_tmp)[row] = make_uint4(words[0], words[1], words[2], words[3]);
      }
    }
    if (MODE == 0 && live) res_cnt[p0 + r] = cnt;
  }
}

// Transpose chunk-ordered nibbles into TMEM lane words (see the layout note at the top).
__global__ void sp24_meta_kernel(const uint32_t* __restrict__ nib_tmp, int64_t total_rows, uint32_t* sp_meta) {
  const int64_t n = total_rows * 4;  // (row-of-lane, j); output words 8 per row
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lane_row = i >> 2;
    const int j = (int)(i & 3);
    const int64_t base = lane_row & ~int64_t(127);
    const int L = (int)(lane_row & 127);
    const int m0 = L & 7, k1 = (L >> 3) & 1, m2 = L >> 4;
    uint32_t w = 0;
#pragma unroll
    for (int m1 = 0; m1 < 2; ++m1) {
      const int64_t row = base + m0 + 8 * m1 + 16 * m2;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int chunk = 8 * j + 4 * k1 + c;  // logical k = 32 j + 16 k1 + 4 c
        const uint32_t nibble = (nib_tmp[row * 4 + (chunk >> 3)] >> (4 * (chunk & 7))) & 0xFu;
        w |= nibble << (4 * c + 16 * m1);
      }
    }
    sp_meta[lane_row * 8 + 4 * (j >> 1) + (j & 1)] = w;
  }
}

inline unsigned grid_of(int64_t work) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 16));
}

}  // namespace
}  // namespace rb

using namespace rb;

// Host-side layout of the sparse form (no device work beyond copying row_partition / blk_ptr).
extern "C" int rb_sparse24_layout(const rb_vbr_device* v, int64_t* sp_tile_row_host, int64_t* total_sp_rows,
                                  int64_t* n_tall, void* stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (!v || !sp_tile_row_host || !total_sp_rows || !n_tall) return fail(RB_EINVAL, "null argument");
  if (v->tile_dtype != RB_BF16 && v->tile_dtype != RB_F16) return fail(RB_EUNSUPPORTED, "2:4 form needs 16-bit tiles");
  if (v->dp % 64 != 0) return fail(RB_EINVAL, "dp must be a multiple of 64");
  const int64_t H = v->n_block_rows;
  std::vector<int32_t> rp(H + 1), bp(H + 1);
  if (H > 0) {
    RB_CUDA_TRY(cudaMemcpyAsync(rp.data(), v->row_partition, 4 * (H + 1), cudaMemcpyDeviceToHost, stream));
    RB_CUDA_TRY(cudaMemcpyAsync(bp.data(), v->blk_ptr, 4 * (H + 1), cudaMemcpyDeviceToHost, stream));
    RB_CUDA_TRY(cudaStreamSynchronize(stream));
  }
  int64_t run = 0, nt = 0;
  for (int64_t g = 0; g < H; ++g) {
    const int64_t h = rp[g + 1] - rp[g], nb = bp[g + 1] - bp[g];
    if (is_short_row((int32_t)h) || nb == 0) {
      sp_tile_row_host[g] = -1;
      continue;
    }
    sp_tile_row_host[g] = run;
    run += (nb * v->dp + 127) / 128 * ((h + 255) / 256 * 256);
    ++nt;
  }
  *total_sp_rows = run;
  *n_tall = nt;
  return RB_OK;
}

// Residual counts + scan: res_ptr[n_rows+1] (device, permuted rows); *n_residuals (host).
// Emission: compressed tiles, metadata words, residual CSR.  tall_g / thread_base are small device
// arrays built by the caller from the layout (block rows with sp_tile_row >= 0, cumulative hs).
extern "C" int rb_sparse24_emit(const rb_vbr_device* v, const int64_t* sp_tile_row, const int32_t* tall_g,
                                const int64_t* thread_base, int32_t n_tall, int64_t total_threads,
                                int64_t total_sp_rows, void* workspace, size_t workspace_bytes, void* sp_tiles,
                                uint32_t* sp_meta, int64_t* res_ptr, int32_t* res_col, float* res_val,
                                int64_t res_capacity, int64_t* n_residuals, void* stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (!v || !n_residuals) return fail(RB_EINVAL, "null argument");
  const int64_t n = v->n_rows;
  // workspace: nib_tmp [total_sp_rows * 4] u32, res_cnt [n] i64, cub temp
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n + 1));
  const size_t need = 16 * (size_t)std::max<int64_t>(total_sp_rows, 1) + 8 * (size_t)(n + 1) + cub_bytes + 512;
  if (!workspace || workspace_bytes < need) return fail(RB_EINVAL, "workspace too small");
  char* w = static_cast<char*>(workspace);
  uint32_t* nib_tmp = reinterpret_cast<uint32_t*>(w);
  int64_t* res_cnt = reinterpret_cast<int64_t*>(w + ((16 * (size_t)std::max<int64_t>(total_sp_rows, 1) + 255) & ~255ull));
  void* cub_tmp = reinterpret_cast<char*>(res_cnt) + ((8 * (size_t)(n + 1) + 255) & ~255ull);
  SpArgs a{v->row_partition, v->row_perm, v->blk_ptr, v->blk_col, v->grp_tile_row, v->col_bounds,
           sp_tile_row, tall_g, n_tall, v->dp};
  RB_CUDA_TRY(cudaMemsetAsync(res_cnt, 0, 8 * (n + 1), stream));
  const bool bf = v->tile_dtype == RB_BF16;
  if (total_threads > 0) {
    if (bf)
      sp24_rows_kernel<__nv_bfloat16, 0><<<grid_of(total_threads), 256, 0, stream>>>(
          a, (const __nv_bfloat16*)v->tiles, nullptr, nullptr, res_cnt, nullptr, nullptr, nullptr, total_threads,
          thread_base);
    else
      sp24_rows_kernel<__half, 0><<<grid_of(total_threads), 256, 0, stream>>>(
          a, (const __half*)v->tiles, nullptr, nullptr, res_cnt, nullptr, nullptr, nullptr, total_threads,
          thread_base);
    RB_CUDA_TRY(cudaGetLastError());
  }
  RB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, res_cnt, res_ptr, (int)(n + 1), stream));
  int64_t total_res = 0;
  RB_CUDA_TRY(cudaMemcpyAsync(&total_res, res_ptr + n, 8, cudaMemcpyDeviceToHost, stream));
  RB_CUDA_TRY(cudaStreamSynchronize(stream));
  *n_residuals = total_res;
  if (!sp_tiles || !sp_meta) return RB_OK;  // count-only call
  if (total_res > res_capacity) return fail(RB_EINVAL, "residual capacity too small");
  if (total_threads > 0) {
    if (bf)
      sp24_rows_kernel<__nv_bfloat16, 1><<<grid_of(total_threads), 256, 0, stream>>>(
          a, (const __nv_bfloat16*)v->tiles, (__nv_bfloat16*)sp_tiles, nib_tmp, nullptr, res_ptr, res_col, res_val,
          total_threads, thread_base);
    else
      sp24_rows_kernel<__half, 1><<<grid_of(total_threads), 256, 0, stream>>>(
          a, (const __half*)v->tiles, (__half*)sp_tiles, nib_tmp, nullptr, res_ptr, res_col, res_val, total_threads,
          thread_base);
    RB_CUDA_TRY(cudaGetLastError());
    RB_CUDA_TRY(cudaMemsetAsync(sp_meta, 0, 32 * (size_t)total_sp_rows, stream));
    sp24_meta_kernel<<<grid_of(total_sp_rows * 4), 256, 0, stream>>>(nib_tmp, total_sp_rows, sp_meta);
    RB_CUDA_TRY(cudaGetLastError());
  }
  return RB_OK;
}

extern "C" int rb_sparse24_workspace_size(int64_t n_rows, int64_t total_sp_rows, size_t* bytes) {
  if (!bytes) return fail(RB_EINVAL, "null argument");
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_rows + 1));
  *bytes = ((16 * (size_t)std::max<int64_t>(total_sp_rows, 1) + 255) & ~255ull) + ((8 * (size_t)(n_rows + 1) + 255) & ~255ull) +
           cub_bytes + 512;
  return RB_OK;
}
