// VBR x dense SpMM on sm_100a: TMA -> SMEM -> tcgen05.mma (bf16/fp16 in, fp32 accumulate in
// TMEM) -> tcgen05.ld -> un-permuted C rows.  Replaces spmm_vbr (multiply.py:72-97).
//
// Both tensor-core kernels are persistent and warp specialised (192 threads):
//   warp 0 lane 0  TMA producer (mbarrier ring of SMEM stages)
//   warp 1         TMEM allocator; lane 0 issues tcgen05.mma (leader CTA only for 2-CTA)
//   warps 2..5     epilogue: tcgen05.ld (32 lanes x 32b) -> C rows at row_perm positions
// with two TMEM accumulators (2 x 256 columns) so the epilogue of work item i overlaps the
// MMAs of item i+1.
//
//   spmm_tall2_kernel   block rows with h > 128, CTA pair (cta_group::2): D = 256 rows x 256
//                       cols; each CTA stages its 128 A-tile rows (K-major, SW128) and its
//                       128-column half of the B panel (MN-major, SW128); the leader issues
//                       tcgen05.mma.cta_group::2 M=256 N=256 K=16.
//   spmm_short2_kernel  block rows with h <= 128 (swap-AB): D^T = Bpanel^T (MN-major, M = 128 C
//                       columns, two M-tiles per item) x tile^T (K-major, N = hp rows).
// The K loop of an item runs over the block row's stored blocks (ascending bcol) and their 64-wide
// K chunks; the B panel of block (g, bcol) is rows col_bounds[bcol] .. +64.  Tile columns past the
// segment width are zero, so neighbouring-segment B rows (or TMA zero fill past n_cols) add 0.
//
// spmm_simt_f32_kernel is the fp32 check path (tcgen05 has no fp32-exact MMA).
#include <algorithm>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <queue>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"
#include "spmm_skinny.cuh"

namespace rb {

constexpr int KCH = 64;                      // K elements per pipeline stage (one SW128 row)
constexpr int kAuxStreams = 3;               // extra streams for concurrent launches of one SpMM
constexpr int TC_THREADS = 192;
constexpr uint32_t BOX_BYTES = 64 * 64 * 2;  // one [64 k x 64 n] B box (8 KB)
constexpr int ACC_COLS = 256;                // TMEM columns per accumulator (x2 buffers)

// tall (2-CTA)
constexpr int PAIR_BM = 256;                 // rows of a tall work item (2 CTAs x 128)
constexpr int TALL_BN = 256;
constexpr int T_STAGES = 6;
constexpr uint32_t T_A_BYTES = 128 * KCH * 2;           // 16 KB: this CTA's 128 A rows
constexpr uint32_t T_B_BYTES = 2 * BOX_BYTES;           // 16 KB: this CTA's 128 B columns
constexpr uint32_t T_STAGE = T_A_BYTES + T_B_BYTES;     // 32 KB
constexpr uint32_t SMEM_TALL = T_STAGES * T_STAGE + 1024 + 256;

// short (swap-AB, 1 CTA)
constexpr int SHORT_NS = 256;                // C columns per item (2 x M=128)
constexpr int S_STAGES = 4;
constexpr uint32_t S_A_SLOT = 128 * KCH * 2;            // up to 128 tile rows
constexpr uint32_t S_B_BYTES = 4 * BOX_BYTES;           // 64 k x 256 n
constexpr uint32_t S_STAGE = S_A_SLOT + S_B_BYTES;      // 48 KB
constexpr uint32_t SMEM_SHORT = S_STAGES * S_STAGE + 1024 + 256;

constexpr int SIMT_ROWS = 8;
constexpr int SIMT_COLS = 128;
constexpr int CMP_PART_NNZ = 2048;  // nonzeros per part of a split row on the compact-payload path

struct SpmmArgs {
  const int32_t* row_partition;
  const int32_t* row_perm;
  const int32_t* blk_ptr;
  const int32_t* blk_col;
  const int64_t* grp_tile_row;
  const int32_t* col_bounds;
  const int4* items;
  int32_t n_items;
  int32_t dp_chunks;
  float* C;
  int64_t ldc;
  int32_t N;
  uint32_t ab_fmt;      // 0 = f16, 1 = bf16
  uint32_t a_evict_first;  // L2 policy of A-tile loads: 1 = evict_first, 0 = evict_normal
  uint32_t b_policy;       // short kernel B loads: 0 = evict_last, 1 = evict_normal, 2 = evict_first
  uint32_t c_evict_first;  // short kernel C stores: 1 = L2 evict_first
  const int32_t* cta_ptr;  // short kernel: items of CTA b are [cta_ptr[b], cta_ptr[b+1]) (null = round robin)
  int32_t short_ns;        // C columns per short item: 128 or 256
  float* ws;               // split-K partials of tall units: [slot][split][8 warps][8 chunks][32 cols][32 lanes]
  int32_t* cnt;            // split-K arrival counters: [slot][8 warps] (zero between launches)
  const uint32_t* sp_meta;     // 2:4 path: TMEM metadata words (sparse24.cu layout)
  const int64_t* sp_tile_row;  // 2:4 path: first compressed row of each tall block row
  CFan fan;                    // further copies of every C store (fused all-gather); fan.n = 0: none
};

// Tall work unit = two int4: (g, m, n0, k0) and (k1, split, n_splits, slot).  Units with
// n_splits > 1 cover the K range [k0, k1) of a split item; their partial accumulators meet in
// `ws` ([slot][split][warp][chunk][8][lane] float4), and the epilogue warp that arrives last
// sums them in split order (deterministic: the sum order does not depend on arrival order).
constexpr int MAX_SPLIT = 4;
constexpr int WARP_PART = 8 * 32 * 32;  // floats of one epilogue warp's partial (32 rows x 256 cols)

// Item range of this CTA: a precomputed per-CTA list (cta_ptr) or plain round robin.
__device__ __forceinline__ int item_begin(const SpmmArgs& a) { return a.cta_ptr ? a.cta_ptr[blockIdx.x] : blockIdx.x; }
__device__ __forceinline__ int item_end(const SpmmArgs& a) { return a.cta_ptr ? a.cta_ptr[blockIdx.x + 1] : a.n_items; }
__device__ __forceinline__ int item_step(const SpmmArgs& a) { return a.cta_ptr ? 1 : (int)gridDim.x; }

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void store_row_chunk(float* dst, const uint32_t (&r)[32], int ncols, bool vec) {
  if (vec && ncols >= 32) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      float4 v = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                             __uint_as_float(r[j + 3]));
      *reinterpret_cast<float4*>(dst + j) = v;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < ncols) dst[j] = __uint_as_float(r[j]);
  }
}

// store_row_chunk into C and every fan-out copy (same element offset in each buffer)
__device__ __forceinline__ void store_row_chunk_fan(const CFan& fan, const float* C, float* dst,
                                                    const uint32_t (&r)[32], int ncols, bool vec) {
  store_row_chunk(dst, r, ncols, vec);
  const int64_t off = dst - C;
  for (int f = 0; f < fan.n; ++f) store_row_chunk(fan.p[f] + off, r, ncols, vec);
}

__device__ __forceinline__ void st_fan(const CFan& fan, float* C, int64_t off, float v) {
  C[off] = v;
  for (int f = 0; f < fan.n; ++f) fan.p[f][off] = v;
}

struct PipeState {
  int s = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void advance(int stages) {
    if (++s == stages) {
      s = 0;
      ph ^= 1;
    }
  }
};

// ------------------------------------------------------------------------------------------
// tall block rows, CTA pair.  Item = (g, 256-row pair tile m, n0).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    spmm_tall2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      SpmmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + T_STAGES * T_STAGE);
  uint64_t* empty = full + T_STAGES;
  uint64_t* tfull = empty + T_STAGES;  // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < T_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);  // 4 epilogue warps x 2 CTAs
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised before any remote arrive / complete_tx
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs; bytes land on the leader's full barrier)
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      const uint64_t pol_a = a.a_evict_first ? policy_evict_first() : policy_evict_normal();
      const uint64_t pol_b = policy_evict_last();
      PipeState ps;
      for (int i = pair; i < a.n_items; i += n_pairs) {
        const int4 it = a.items[2 * i], iu = a.items[2 * i + 1];
        const int g = it.x, m = it.y, n0 = it.z;
        const int h = a.row_partition[g + 1] - a.row_partition[g];
        const int hp = hp_of(h);
        const int b_begin = a.blk_ptr[g];
        const int64_t row0 = a.grp_tile_row[g] + (int64_t)m * PAIR_BM + rank * 128;
        for (int k = it.w; k < iu.x; ++k) {
          mbar_wait(&empty[ps.s], ps.ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[ps.s], 2 * T_STAGE);
          const int t = k / a.dp_chunks, kc = k - t * a.dp_chunks;
          const int bcol = a.blk_col[b_begin + t];
          uint8_t* sA = smem + ps.s * T_STAGE;
          uint8_t* sB = sA + T_A_BYTES;
          tma_load_2d_2sm(sA, &tmA, &full[ps.s], kc * KCH, (int32_t)(row0 + (int64_t)t * hp), pol_a);
          const int krow = a.col_bounds[bcol] + kc * KCH;
          const int nb0 = n0 + (int)rank * 128;
          tma_load_2d_2sm(sB, &tmB, &full[ps.s], nb0, krow, pol_b);
          tma_load_2d_2sm(sB + BOX_BYTES, &tmB, &full[ps.s], nb0 + 64, krow, pol_b);
          ps.advance(T_STAGES);
        }
      }
      // drain: every stage's last MMA commit has landed before teardown
      for (int k = 0; k < T_STAGES; ++k) {
        mbar_wait(&empty[ps.s], ps.ph ^ 1);
        ps.advance(T_STAGES);
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ---------------- MMA issuer (leader CTA, one thread)
      const uint32_t idesc = idesc_f16(256, TALL_BN, a.ab_fmt, /*a_mn=*/0, /*b_mn=*/1);
      PipeState ps;
      int acc = 0;
      uint32_t aph = 0;
      for (int i = pair; i < a.n_items; i += n_pairs) {
        const int k0 = a.items[2 * i].w, k1 = a.items[2 * i + 1].x;
        if (k1 <= k0) continue;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * ACC_COLS;
        for (int k = k0; k < k1; ++k) {
          mbar_wait(&full[ps.s], ps.ph);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + ps.s * T_STAGE);
          const uint32_t b_base = a_base + T_A_BYTES;
#pragma unroll
          for (int kk = 0; kk < KCH / 16; ++kk) {
            const uint64_t ad = sdesc_sw128(a_base + kk * 32, 16, 1024);            // K-major: +16 elems
            const uint64_t bd = sdesc_sw128(b_base + kk * 2048, BOX_BYTES, 1024);   // MN-major: +16 rows
            umma_f16_2sm(d, ad, bd, idesc, (k != k0) || kk != 0);
          }
          umma_commit_2sm_mc(&empty[ps.s], 0x3);
          ps.advance(T_STAGES);
        }
        umma_commit_2sm_mc(&tfull[acc], 0x3);
        acc ^= 1;
        if (acc == 0) aph ^= 1;
      }
    }
  } else {
    // ---------------- epilogue (both CTAs): TMEM lane = row rank*128 + 32q + lane of the pair tile
    const int q = warp & 3;
    const bool vec = ((a.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.C) & 15) == 0);
    int acc = 0;
    uint32_t aph = 0;
    for (int i = pair; i < a.n_items; i += n_pairs) {
      const int4 it = a.items[2 * i], iu = a.items[2 * i + 1];
      const int g = it.x, m = it.y, n0 = it.z;
      const int p0 = a.row_partition[g];
      const int h = a.row_partition[g + 1] - p0;
      const int nk = iu.x - it.w;
      const int row_local = m * PAIR_BM + (int)rank * 128 + q * 32 + lane;
      const bool valid = row_local < h;
      const int64_t crow = valid ? (int64_t)a.row_perm[p0 + row_local] : 0;
      float* dst = a.C + crow * a.ldc + n0;
      const int ncol = min(TALL_BN, a.N - n0);
      if (nk > 0) {
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
      }
      if (iu.z > 1) {
        // split-K unit: park the partial (lane-contiguous, coalesced), release the accumulator,
        // and let the last-arriving split of this warp's 32 rows reduce all partials in split order
        const int wslot = (int)rank * 4 + q;
        float* part = a.ws + ((size_t)iu.w * MAX_SPLIT + iu.y) * 8 * WARP_PART + (size_t)wslot * WARP_PART;
        float4* part4 = reinterpret_cast<float4*>(part);
        for (int c = 0; c < ncol; c += 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem + acc * ACC_COLS + ((uint32_t)(q * 32) << 16) + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j)  // [chunk][j][lane] float4: 512 contiguous bytes per instruction
            __stcg(part4 + (c >> 5) * 256 + j * 32 + lane,
                   make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                               __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) aph ^= 1;
        __threadfence();
        __syncwarp();
        int old = 0;
        int* ctr = a.cnt + iu.w * 8 + wslot;
        if (lane == 0) old = atomicAdd(ctr, 1);
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old == iu.z - 1) {
          __threadfence();
          const float4* base4 =
              reinterpret_cast<const float4*>(a.ws + (size_t)iu.w * MAX_SPLIT * 8 * WARP_PART + (size_t)wslot * WARP_PART);
          constexpr int SPLIT_STRIDE4 = 8 * WARP_PART / 4;
          for (int c = 0; c < ncol; c += 32) {
            // all splits' loads of this chunk in flight at once, then summed in split order
            float4 v[MAX_SPLIT][8];
#pragma unroll
            for (int sp = 0; sp < MAX_SPLIT; ++sp)
#pragma unroll
              for (int j = 0; j < 8; ++j)
                v[sp][j] = sp < iu.z ? __ldcg(base4 + sp * SPLIT_STRIDE4 + (c >> 5) * 256 + j * 32 + lane)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
            uint32_t r[32];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 t = v[0][j];
#pragma unroll
              for (int sp = 1; sp < MAX_SPLIT; ++sp)
                if (sp < iu.z) {
                  t.x += v[sp][j].x;
                  t.y += v[sp][j].y;
                  t.z += v[sp][j].z;
                  t.w += v[sp][j].w;
                }
              r[4 * j] = __float_as_uint(t.x);
              r[4 * j + 1] = __float_as_uint(t.y);
              r[4 * j + 2] = __float_as_uint(t.z);
              r[4 * j + 3] = __float_as_uint(t.w);
            }
            if (valid) store_row_chunk_fan(a.fan, a.C, dst + c, r, ncol - c, vec);
          }
          if (lane == 0) *ctr = 0;  // ready for the next launch (stream ordered)
        }
        continue;
      }
      for (int c = 0; c < ncol; c += 32) {
        uint32_t r[32];
        if (nk > 0) {
          tmem_ld_32x32b_x32(tmem + acc * ACC_COLS + ((uint32_t)(q * 32) << 16) + c, r);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = 0u;
        }
        if (valid) store_row_chunk_fan(a.fan, a.C, dst + c, r, ncol - c, vec);
      }
      if (nk > 0) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) aph ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc_2sm<512>(tmem);
}

// ------------------------------------------------------------------------------------------
// tall block rows on the 2:4 sparse tensor cores (tcgen05.mma.sp, cta_group::2, M=256 N=256 K=32
// logical per MMA).  A stage = 128 logical K of the block row's padded block sequence: this CTA's
// 128 compressed A rows (64 values, one SW128 TMA box of the sparse24.cu layout), the 128 x 128 B
// panel half (four 64x64 boxes: K sub-ranges of 64 each inside one block) and this CTA's metadata
// (two 2 KB planes: 128 lanes x 16 B).  The MMA thread moves the metadata to TMEM with two
// tcgen05.cp 128x128b (ordered before its MMAs in the tensor pipe) and points MMA j at the
// 4-column-aligned plane j/2 with idesc sparse_id2 = j%2 (tools/sp_probe).  Single 256-column
// accumulator (TMEM also holds the metadata ring); epilogue as the dense kernel.  Groups' extra
// nonzeros (more than 2 of 4) are added by the residual pass after this kernel.
constexpr int SP_STAGES = 4;
constexpr int SP_THREADS = 192;  // warp 0 TMA, 1 MMA, 2-5 epilogue
constexpr uint32_t SP_A_BYTES = 128 * 128;
constexpr uint32_t SP_B_BYTES = 4 * BOX_BYTES;
constexpr uint32_t SP_E_PLANE = 128 * 16;
constexpr uint32_t SP_STAGE_BYTES = SP_A_BYTES + SP_B_BYTES + 2 * SP_E_PLANE;  // 52 KB
constexpr uint32_t SMEM_SP = SP_STAGES * SP_STAGE_BYTES + 1024 + 256;
constexpr uint32_t SP_META_COL = 256;  // TMEM metadata ring: + 8 * stage + 4 * plane

__device__ __forceinline__ void umma_sp_2sm(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t e_tmem,
                                            uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%5], %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(e_tmem)
      : "memory");
}
// 128 lanes x 128 bits from shared memory (128 rows of 16 B, no swizzle) into 4 TMEM columns of both CTAs
__device__ __forceinline__ void tmem_cp_128x128b_2sm(uint32_t taddr, uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // LBO 16 B (single core matrix along K)
  d |= (uint64_t)(128 >> 4) << 32;   // SBO: 8-row core matrices 128 B apart
  d |= (uint64_t)1 << 46;            // version
  asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(taddr), "l"(d) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(SP_THREADS, 1)
    spmm_tall2_sp_kernel(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmE, SpmmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SP_STAGES * SP_STAGE_BYTES);
  uint64_t* empty = full + SP_STAGES;
  uint64_t* tfull = empty + SP_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < SP_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 8);  // 4 epilogue warps x 2 CTAs
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: compressed A rows + metadata planes + B panel half, both CTAs
      tma_prefetch_desc(&tmS);
      tma_prefetch_desc(&tmB);
      tma_prefetch_desc(&tmE);
      const uint64_t pol_a = policy_evict_normal();  // compressed A is re-read by the next N chunk
      const uint64_t pol_b = policy_evict_last();
      PipeState ps;
      for (int i = pair; i < a.n_items; i += n_pairs) {
        const int4 it = a.items[2 * i], iu = a.items[2 * i + 1];
        const int g = it.x, m = it.y, n0 = it.z;
        const int h = a.row_partition[g + 1] - a.row_partition[g];
        const int hs = (h + 255) / 256 * 256;
        const int b_begin = a.blk_ptr[g];
        const int nb = a.blk_ptr[g + 1] - b_begin;
        const int64_t row0 = a.sp_tile_row[g] + (int64_t)m * PAIR_BM + rank * 128;
        const int dp = a.dp_chunks * KCH;
        for (int s = it.w; s < iu.x; ++s) {
          mbar_wait(&empty[ps.s], ps.ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[ps.s], 2 * SP_STAGE_BYTES);
          uint8_t* sA = smem + ps.s * SP_STAGE_BYTES;
          uint8_t* sB = sA + SP_A_BYTES;
          uint8_t* sE = sB + SP_B_BYTES;
          const int32_t r = (int32_t)(row0 + (int64_t)s * hs);
          tma_load_2d_2sm(sA, &tmS, &full[ps.s], 0, r, pol_a);
          tma_load_2d_2sm(sE, &tmE, &full[ps.s], 0, r, pol_a);
          tma_load_2d_2sm(sE + SP_E_PLANE, &tmE, &full[ps.s], 4, r, pol_a);
          const int nb0 = n0 + (int)rank * 128;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int k = s * 128 + 64 * u;
            const int t = k / dp, c = k - t * dp;
            const int krow = t < nb ? a.col_bounds[a.blk_col[b_begin + t]] + c : 0;  // past the end: A is 0
            tma_load_2d_2sm(sB + u * 2 * BOX_BYTES, &tmB, &full[ps.s], nb0, krow, pol_b);
            tma_load_2d_2sm(sB + u * 2 * BOX_BYTES + BOX_BYTES, &tmB, &full[ps.s], nb0 + 64, krow, pol_b);
          }
          ps.advance(SP_STAGES);
        }
      }
      for (int k = 0; k < SP_STAGES; ++k) {
        mbar_wait(&empty[ps.s], ps.ph ^ 1);
        ps.advance(SP_STAGES);
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ---------------- metadata copies + sparse MMAs (one thread, in tensor-pipe order)
      const uint32_t idesc = idesc_f16(256, TALL_BN, a.ab_fmt, /*a_mn=*/0, /*b_mn=*/1) | (1u << 2);
      PipeState ps;
      uint32_t aph = 0;
      for (int i = pair; i < a.n_items; i += n_pairs) {
        const int k0 = a.items[2 * i].w, k1 = a.items[2 * i + 1].x;
        if (k1 <= k0) continue;
        mbar_wait(tempty, aph ^ 1);
        tc_fence_after();
        for (int s = k0; s < k1; ++s) {
          mbar_wait(&full[ps.s], ps.ph);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + ps.s * SP_STAGE_BYTES);
          const uint32_t b_base = a_base + SP_A_BYTES;
          const uint32_t e_base = b_base + SP_B_BYTES;
          const uint32_t e_tmem = tmem + SP_META_COL + 8 * ps.s;
          tmem_cp_128x128b_2sm(e_tmem, e_base);
          tmem_cp_128x128b_2sm(e_tmem + 4, e_base + SP_E_PLANE);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t ad = sdesc_sw128(a_base + j * 32, 16, 1024);  // 16 compressed values
            const uint64_t bd = sdesc_sw128(b_base + (j >> 1) * 2 * BOX_BYTES + (j & 1) * 4096, BOX_BYTES, 1024);
            umma_sp_2sm(tmem, ad, bd, idesc | (uint32_t)(j & 1), e_tmem + 4 * (j >> 1), (s != k0) || j != 0);
          }
          umma_commit_2sm_mc(&empty[ps.s], 0x3);
          ps.advance(SP_STAGES);
        }
        umma_commit_2sm_mc(tfull, 0x3);
        aph ^= 1;
      }
    }
  } else {
    // ---------------- epilogue (both CTAs), single accumulator
    const int q = warp & 3;
    const bool vec = ((a.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.C) & 15) == 0);
    uint32_t aph = 0;
    for (int i = pair; i < a.n_items; i += n_pairs) {
      const int4 it = a.items[2 * i], iu = a.items[2 * i + 1];
      const int g = it.x, m = it.y, n0 = it.z;
      const int p0 = a.row_partition[g];
      const int h = a.row_partition[g + 1] - p0;
      const int nk = iu.x - it.w;
      const int row_local = m * PAIR_BM + (int)rank * 128 + q * 32 + lane;
      const bool valid = row_local < h;
      const int64_t crow = valid ? (int64_t)a.row_perm[p0 + row_local] : 0;
      float* dst = a.C + crow * a.ldc + n0;
      const int ncol = min(TALL_BN, a.N - n0);
      if (nk <= 0) continue;
      mbar_wait(tfull, aph);
      tc_fence_after();
      if (iu.z > 1) {
        const int wslot = (int)rank * 4 + q;
        float* part = a.ws + ((size_t)iu.w * MAX_SPLIT + iu.y) * 8 * WARP_PART + (size_t)wslot * WARP_PART;
        float4* part4 = reinterpret_cast<float4*>(part);
        for (int c = 0; c < ncol; c += 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            __stcg(part4 + (c >> 5) * 256 + j * 32 + lane,
                   make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                               __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(tempty);
        aph ^= 1;
        __threadfence();
        __syncwarp();
        int old = 0;
        int* ctr = a.cnt + iu.w * 8 + wslot;
        if (lane == 0) old = atomicAdd(ctr, 1);
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old == iu.z - 1) {
          __threadfence();
          const float4* base4 = reinterpret_cast<const float4*>(a.ws + (size_t)iu.w * MAX_SPLIT * 8 * WARP_PART +
                                                                (size_t)wslot * WARP_PART);
          constexpr int SPLIT_STRIDE4 = 8 * WARP_PART / 4;
          for (int c = 0; c < ncol; c += 32) {
            float4 v[MAX_SPLIT][8];
#pragma unroll
            for (int sp = 0; sp < MAX_SPLIT; ++sp)
#pragma unroll
              for (int j = 0; j < 8; ++j)
                v[sp][j] = sp < iu.z ? __ldcg(base4 + sp * SPLIT_STRIDE4 + (c >> 5) * 256 + j * 32 + lane)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
            uint32_t r[32];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 t = v[0][j];
#pragma unroll
              for (int sp = 1; sp < MAX_SPLIT; ++sp)
                if (sp < iu.z) {
                  t.x += v[sp][j].x;
                  t.y += v[sp][j].y;
                  t.z += v[sp][j].z;
                  t.w += v[sp][j].w;
                }
              r[4 * j] = __float_as_uint(t.x);
              r[4 * j + 1] = __float_as_uint(t.y);
              r[4 * j + 2] = __float_as_uint(t.z);
              r[4 * j + 3] = __float_as_uint(t.w);
            }
            if (valid) store_row_chunk_fan(a.fan, a.C, dst + c, r, ncol - c, vec);
          }
          if (lane == 0) *ctr = 0;
        }
        continue;
      }
      for (int c = 0; c < ncol; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + c, r);
        tmem_ld_wait();
        if (valid) store_row_chunk_fan(a.fan, a.C, dst + c, r, ncol - c, vec);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(tempty);
      aph ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc_2sm<512>(tmem);
}

// ------------------------------------------------------------------------------------------
// short block rows (swap-AB), one CTA.  Item = (g, hp, n0).  D_mt^T[128 C cols x hp rows] at TMEM
// columns acc*256 + mt*hp.
__global__ void __launch_bounds__(TC_THREADS, 1)
    spmm_short2_kernel(const __grid_constant__ CUtensorMap tmA16, const __grid_constant__ CUtensorMap tmA32,
                       const __grid_constant__ CUtensorMap tmA64, const __grid_constant__ CUtensorMap tmA128,
                       const __grid_constant__ CUtensorMap tmB, SpmmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S_STAGES * S_STAGE);
  uint64_t* empty = full + S_STAGES;
  uint64_t* tfull = empty + S_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmB);
      const uint64_t pol_a = a.a_evict_first ? policy_evict_first() : policy_evict_normal();
      const uint64_t pol_b = a.b_policy == 0 ? policy_evict_last()
                             : a.b_policy == 1 ? policy_evict_normal() : policy_evict_first();
      PipeState ps;
      for (int i = item_begin(a); i < item_end(a); i += item_step(a)) {
        const int4 it = a.items[i];
        const int g = it.x, hp = it.y, n0 = it.z;
        const CUtensorMap* tmA = hp == 16 ? &tmA16 : hp == 32 ? &tmA32 : hp == 64 ? &tmA64 : &tmA128;
        const int b_begin = a.blk_ptr[g];
        const int nk = (a.blk_ptr[g + 1] - b_begin) * a.dp_chunks;
        const int64_t row0 = a.grp_tile_row[g];
        const int pitch = tile_pitch(a.row_partition[g + 1] - a.row_partition[g]);
        const int n_boxes = min(a.short_ns / 64, (a.N - n0 + 63) / 64);
        const uint32_t tx = (uint32_t)hp * KCH * 2 + n_boxes * BOX_BYTES;
        for (int k = 0; k < nk; ++k) {
          mbar_wait(&empty[ps.s], ps.ph ^ 1);
          mbar_arrive_expect_tx(&full[ps.s], tx);
          const int t = k / a.dp_chunks, kc = k - t * a.dp_chunks;
          const int bcol = a.blk_col[b_begin + t];
          uint8_t* sA = smem + ps.s * S_STAGE;
          uint8_t* sB = sA + S_A_SLOT;
          tma_load_2d_hint(sA, tmA, &full[ps.s], kc * KCH, (int32_t)(row0 + (int64_t)t * pitch), pol_a);
          const int krow = a.col_bounds[bcol] + kc * KCH;
          for (int bx = 0; bx < n_boxes; ++bx)
            tma_load_2d_hint(sB + bx * BOX_BYTES, &tmB, &full[ps.s], n0 + 64 * bx, krow, pol_b);
          ps.advance(S_STAGES);
        }
      }
      for (int k = 0; k < S_STAGES; ++k) {
        mbar_wait(&empty[ps.s], ps.ph ^ 1);
        ps.advance(S_STAGES);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      PipeState ps;
      int acc = 0;
      uint32_t aph = 0;
      for (int i = item_begin(a); i < item_end(a); i += item_step(a)) {
        const int4 it = a.items[i];
        const int g = it.x, hp = it.y, n0 = it.z;
        const int nk = (a.blk_ptr[g + 1] - a.blk_ptr[g]) * a.dp_chunks;
        if (nk == 0) continue;
        const int n_mt = min(a.short_ns / 128, (a.N - n0 + 127) / 128);
        const uint32_t idesc = idesc_f16(128, hp, a.ab_fmt, /*a_mn=*/1, /*b_mn=*/0);
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * ACC_COLS;
        for (int k = 0; k < nk; ++k) {
          mbar_wait(&full[ps.s], ps.ph);
          tc_fence_after();
          const uint32_t t_base = smem_u32(smem + ps.s * S_STAGE);  // tile rows (K-major)
          const uint32_t b_base = t_base + S_A_SLOT;                 // B panel (MN-major)
          for (int mt = 0; mt < n_mt; ++mt) {
#pragma unroll
            for (int kk = 0; kk < KCH / 16; ++kk) {
              const uint64_t ad = sdesc_sw128(b_base + mt * 2 * BOX_BYTES + kk * 2048, BOX_BYTES, 1024);
              const uint64_t bd = sdesc_sw128(t_base + kk * 32, 16, 1024);
              umma_f16(d + mt * hp, ad, bd, idesc, (k | kk) != 0);
            }
          }
          umma_commit(&empty[ps.s]);
          ps.advance(S_STAGES);
        }
        umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) aph ^= 1;
      }
    }
  } else {
    // epilogue: TMEM lane = C column, column = block-row row; a warp stores 32 consecutive floats
    // (128 B) of one C row per instruction
    const int q = warp & 3;
    const uint64_t pol_c = policy_evict_first();
    int acc = 0;
    uint32_t aph = 0;
    for (int i = item_begin(a); i < item_end(a); i += item_step(a)) {
      const int4 it = a.items[i];
      const int g = it.x, hp = it.y, n0 = it.z;
      const int p0 = a.row_partition[g];
      const int h = a.row_partition[g + 1] - p0;
      const int nk = (a.blk_ptr[g + 1] - a.blk_ptr[g]) * a.dp_chunks;
      const int n_mt = min(a.short_ns / 128, (a.N - n0 + 127) / 128);
      if (nk > 0) {
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
      }
      for (int mt = 0; mt < n_mt; ++mt) {
        const int n = n0 + mt * 128 + q * 32 + lane;
        const bool nvalid = n < a.N;
        for (int j0 = 0; j0 < h; j0 += 16) {
          uint32_t r[16];
          if (nk > 0) {
            tmem_ld_32x32b_x16(tmem + acc * ACC_COLS + ((uint32_t)(q * 32) << 16) + mt * hp + j0, r);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) r[j] = 0u;
          }
          if (nvalid) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (j0 + j < h) {
                const int64_t off = (int64_t)a.row_perm[p0 + j0 + j] * a.ldc + n;
                if (a.c_evict_first)
                  st_global_hint(a.C + off, __uint_as_float(r[j]), pol_c);
                else
                  a.C[off] = __uint_as_float(r[j]);
                for (int f = 0; f < a.fan.n; ++f) a.fan.p[f][off] = __uint_as_float(r[j]);
              }
            }
          }
        }
      }
      if (nk > 0) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) aph ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------------------------------
// short block rows of one height class on a static multi-slot sweep (swap-AB, one CTA).
//
// Config 5 (4,096 block rows of h = 64, each ~41 blocks spread uniformly over 4,096 block columns,
// N = 1024) has no B reuse inside a CTA: every B panel an SM fetches is used by one block row.
// Reuse can only come from L2, across the block rows that are resident on the chip at the same
// time.  Round 1 ran one (block row, 256-column slab) item per CTA at a time, each sweeping its
// blocks from block column 0: 148 rows in flight at random phases, so the L2 working set was the
// whole 134 MB slab of B (> the ~90 MB hot L2) and 48 % of the B panel bytes came from DRAM.
// Here each CTA keeps `n_slots` block rows resident in TMEM (slot s = columns s*2*hp .. +2*hp: two
// M-tiles of 128 C columns x hp rows; 4 slots at hp = 64 fill the 512 columns) and walks a
// plan-time step list that merges the slots' blocks in CIRCULAR block-column order: a block row
// that enters a freed slot starts at the CTA's current block column and wraps around.  All CTAs
// therefore sweep B in near lockstep with 4x more rows in flight, the live B window is a small
// arc of the slab, and every B panel fetched from DRAM serves ~6 block rows (tools/l2sim.py,
// calibrated on the round-1 schedule: 16.0 -> 10.6 GB of A + B misses per step).
// The per-row accumulation order is fixed by the plan (rotated ascending block columns), so C is
// run-to-run deterministic.  Slot handshakes: the MMA thread commits sdone[s] after a row's last
// block; the epilogue drains slot s and the 4 epilogue warps arrive on sfree[s]; the MMA waits on
// sfree[s] before the first block of the next row in slot s (the plan leaves `delay` steps of
// other slots' work between the two so the drain overlaps MMAs).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}" : "=r"(pred));
  return pred != 0;
}

constexpr int MAX_SLOTS = 16;
// MMA-issuing warps (slots alternate between them).  Two issuers were meant to hide one issuer's
// per-stage wait + commit (~100+ cycles against an M=128 N=64 MMA of ~48): with 2-stage rings each
// they measured 2.69 ms against 2.34 ms for one issuer with the 4-stage ring on config 5, so one.
constexpr int SW_MMA_WARPS = 1;
constexpr int SW_THREADS = (1 + SW_MMA_WARPS + 4) * 32;
constexpr int SW64_THREADS = (1 + SW_MMA_WARPS + 8) * 32;  // M64 form: 8 epilogue warps
#ifdef RB_DBG_NOEPI  // developer experiment: no epilogue (C is not written)
constexpr bool NOEPI_DBG = true;
#else
constexpr bool NOEPI_DBG = false;
#endif
// Idle epilogue warps probe their slot barrier with one lane and sleep between probes.
#ifndef SW_EPI_SLEEP_NS
#define SW_EPI_SLEEP_NS 256
#endif
// Each MMA warp has its own ring of S_STAGES / SW_MMA_WARPS stages (one consumer per ring): with a
// shared ring a warp that skips the other's steps can run two phases ahead of a stage's barrier,
// where a parity wait no longer tells the phases apart (it deadlocked).
// Stage ring: 4 x 48 KB (16 KB of tile rows for hp up to 128 + the 32 KB B panel slab of 256
// columns), or 5 x 40 KB for hp <= 64 (RB_SWEEP_BIG=0).
constexpr int SW_STAGES_BIG = 4, SW_STAGES_SMALL = 5;
constexpr uint32_t SW_ASLOT_BIG = 128 * KCH * 2, SW_ASLOT_SMALL = 64 * KCH * 2;
constexpr uint32_t sweep_smem(int st, uint32_t aslot) { return st * (aslot + S_B_BYTES) + 1024 + 512; }
constexpr uint32_t SW64_EPI_BYTES = 8 * 16 * 36 * 4;  // M64 epilogue staging: 16 x 36 floats per warp
constexpr uint32_t sweep64_smem(int st, uint32_t aslot) { return st * (aslot + S_B_BYTES) + 1024 + 1024 + SW64_EPI_BYTES; }

struct SweepArgs {
  const int4* steps;        // (A tile row, first B row, n0, slot | first << 8 | last << 9)
  const int32_t* step_ptr;  // CTA b's steps are [step_ptr[b], step_ptr[b+1])
  const int4* done;         // row completions in commit order: (g, n0, slot, -)
  const int32_t* done_ptr;
  int32_t hp;
};

// PAIR: the full barrier of an even stage covers it and the next one (2 arrivals per phase), so the
// MMA warp waits once per two stages (16 MMAs) instead of once per stage.
// Step list reader for the producer / MMA warps: the warp loads 32 steps at a time (one per lane,
// coalesced) one batch ahead and hands step i to every lane with __shfl_sync.  A per-step load
// issued one step ahead left its L2/DRAM latency (~1 us under this kernel's memory load) on the
// issue path of every step.
struct StepReader {
  const int4* p;
  int end, base, lane;
  int4 cur, nxt;
  __device__ __forceinline__ int4 load(int idx) const { return idx < end ? __ldg(p + idx) : make_int4(0, 0, 0, 0); }
  __device__ __forceinline__ void init(const int4* steps, int b, int e, int ln) {
    p = steps;
    end = e;
    base = b;
    lane = ln;
    cur = load(b + ln);
    nxt = load(b + 32 + ln);
  }
  __device__ __forceinline__ int4 get(int i) {  // i = base, base + 1, ... in order
    if (i - base == 32) {
      base += 32;
      cur = nxt;
      nxt = load(base + 32 + lane);
    }
    const int k = i - base;
    return make_int4(__shfl_sync(0xffffffffu, cur.x, k), __shfl_sync(0xffffffffu, cur.y, k),
                     __shfl_sync(0xffffffffu, cur.z, k), __shfl_sync(0xffffffffu, cur.w, k));
  }
};

// M64: block rows of exactly hp = 64 on NON-swapped MMAs, D[64 rows x 256 C columns] =
// tile[64 x K] (K-major) x Bpanel[K x 256] (MN-major), one tcgen05.mma M=64 N=256 K=16 per K16.  An
// M=64 accumulator fills one lane half of TMEM (rows 16q..16q+15 at lanes 32q + 16*half + 0..15;
// tools/mma_probe/m64_layout.cu), so slot s sits at lane half s & 1, columns (s >> 1) * 256: the
// same 4 slots of 64 rows x 256 columns as the swapped form, with half as many MMAs per block and
// each one 128 cycles long — the per-stage wait / commit no longer starves the tensor pipe, as the
// 48-cycle swapped N=64 MMAs did.  Eight epilogue warps (two per lane quadrant, one per 128-column
// half) each copy 16 rows x 128 columns to registers, release the slot, then store.
template <int ST, uint32_t ASLOT, bool PAIR, bool M64 = false>
__global__ void __launch_bounds__(M64 ? SW64_THREADS : SW_THREADS, 1)
    spmm_sweep_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, SpmmArgs a,
                      SweepArgs w) {
  extern __shared__ uint8_t smem_raw[];
#ifdef RB_PROF_SWEEP
  long long k_t0 = clock64();
  unsigned long long k_g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(k_g0));
#endif
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * (ASLOT + S_B_BYTES));
  uint64_t* empty = full + ST;
  uint64_t* sdone = empty + ST;
  uint64_t* sfree = sdone + MAX_SLOTS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfree + MAX_SLOTS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hp = w.hp;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], PAIR ? 2 : 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < MAX_SLOTS; ++s) {
      mbar_init(&sdone[s], 1);
      mbar_init(&sfree[s], M64 ? 8 : 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int s_begin = w.step_ptr[blockIdx.x], s_end = w.step_ptr[blockIdx.x + 1];

  // Producer and MMA warps run converged: per-step values are loaded by every lane (the next step's
  // ahead of time), broadcast with __shfl_sync so the compiler keeps them warp-uniform, and one
  // elected lane issues the TMA / tcgen05 instructions.  (A lone lane-0 loop made ptxas wrap every
  // UTCHMMA in an ELECT / R2UR.BROADCAST waterfall and left a dependent global load in front of
  // each step: ~165 cycles per M=128 N=64 MMA against the 48-cycle issue floor measured by
  // tools/mma_probe.)
  if (warp == 0) {
#ifdef RB_DBG_MMAONLY  // developer experiment: MMA issue loop alone (no producer, no stage barriers)
    if (true) {
    } else
#endif
    {
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmA);
    const uint64_t pol_a = policy_evict_first();
    const uint64_t pol_b = policy_evict_last();
    PipeState rings[SW_MMA_WARPS];
    StepReader rd;
    rd.init(w.steps, s_begin, s_end, lane);
    for (int i = s_begin; i < s_end; ++i) {
      const int4 st = rd.get(i);
      const int row0 = st.x, krow0 = st.y, n0 = st.z, fl = st.w;
      const int r = (fl & 0xff) % SW_MMA_WARPS;  // the ring of the MMA warp that owns the step's slot
      const int n_boxes = min(a.short_ns / 64, (a.N - n0 + 63) / 64);
      const uint32_t tx = (uint32_t)hp * KCH * 2 + n_boxes * BOX_BYTES;
      for (int kc = 0; kc < a.dp_chunks; ++kc) {
        const int sg = r * (ST / SW_MMA_WARPS) + rings[r].s;
        uint64_t* fb = &full[PAIR ? (sg & ~1) : sg];
        if (elect_one()) {
          mbar_wait(&empty[sg], rings[r].ph ^ 1);
#ifdef RB_DBG_NOLOAD  // developer experiment: MMA + barrier pipeline without any operand traffic
          mbar_arrive(fb);
#else
          mbar_arrive_expect_tx(fb, tx);
          uint8_t* sA = smem + sg * (ASLOT + S_B_BYTES);
          uint8_t* sB = sA + ASLOT;
          tma_load_2d_hint(sA, &tmA, fb, kc * KCH, row0, pol_a);
          for (int bx = 0; bx < n_boxes; ++bx)
            tma_load_2d_hint(sB + bx * BOX_BYTES, &tmB, fb, n0 + 64 * bx, krow0 + kc * KCH, pol_b);
#endif
        }
        __syncwarp();
        rings[r].advance((ST / SW_MMA_WARPS));
      }
    }
    if (PAIR)  // a pair left half-filled: complete its phase (the MMA warp waits on it)
      for (int r = 0; r < SW_MMA_WARPS; ++r)
        if (rings[r].s & 1) {
          if (elect_one()) mbar_arrive(&full[r * (ST / SW_MMA_WARPS) + rings[r].s - 1]);
          __syncwarp();
        }
    for (int r = 0; r < SW_MMA_WARPS; ++r)
      for (int k = 0; k < (ST / SW_MMA_WARPS); ++k) {
        mbar_wait(&empty[r * (ST / SW_MMA_WARPS) + rings[r].s], rings[r].ph ^ 1);
        rings[r].advance((ST / SW_MMA_WARPS));
      }
    }
  } else if (warp <= SW_MMA_WARPS) {
    const int mw = warp - 1;  // this MMA warp issues the steps of slots with slot % SW_MMA_WARPS == mw
    PipeState ps;
#ifdef RB_PROF_SWEEP
    long long prof_free = 0, prof_full = 0;
    const long long prof_t0 = clock64();
#endif
    uint32_t use_ph = 0;  // bit s: parity of slot s's next sfree wait (flipped per row)
    const uint32_t idesc = M64 ? idesc_f16(64, 256, a.ab_fmt, /*a_mn=*/0, /*b_mn=*/1)
                               : idesc_f16(128, hp, a.ab_fmt, /*a_mn=*/1, /*b_mn=*/0);
    const uint64_t adesc0 = sdesc_sw128(smem_u32(smem) + ASLOT, BOX_BYTES, 1024);  // B panel (MN-major)
    const uint64_t bdesc0 = sdesc_sw128(smem_u32(smem), 16, 1024);                    // tile rows (K-major)
    StepReader rd;
    rd.init(w.steps, s_begin, s_end, lane);
    for (int i = s_begin; i < s_end; ++i) {
      const int4 st = rd.get(i);
      const int n0 = st.z, fl = st.w;
      const int slot = fl & 0xff;
      if (slot % SW_MMA_WARPS != mw) continue;  // the other MMA warp's step (its own ring)
      const bool first = (fl >> 8) & 1, last = (fl >> 9) & 1;
      const int n_mt = min(a.short_ns / 128, (a.N - n0 + 127) / 128);
      if (first) {
#ifdef RB_PROF_SWEEP
        const long long t0 = clock64();
#endif
#ifndef RB_DBG_NOEPI
        mbar_wait(&sfree[slot], ((use_ph >> slot) & 1) ^ 1);
#endif
#ifdef RB_PROF_SWEEP
        prof_free += clock64() - t0;
#endif
        use_ph ^= 1u << slot;
        tc_fence_after();
      }
      const uint32_t d = M64 ? tmem + ((uint32_t)(slot & 1) << 20) + (uint32_t)((slot >> 1) * 256)
                             : tmem + (uint32_t)(slot * 2 * hp);
      for (int kc = 0; kc < a.dp_chunks; ++kc) {
        // descriptors = stage-0 descriptor + (byte offset >> 4): one add per operand (SMEM < 256 KB,
        // so the 14-bit address field never carries)
        const int sg = mw * (ST / SW_MMA_WARPS) + ps.s;  // this warp's ring
        const uint64_t soff = (uint64_t)((sg * (ASLOT + S_B_BYTES)) >> 4);
        if (elect_one()) {  // one lane waits and issues (a SYNCS wait by the whole warp costs more)
#ifdef RB_PROF_SWEEP
          const long long t1 = clock64();
#endif
#ifndef RB_DBG_MMAONLY
          if (!PAIR || (sg & 1) == 0) mbar_wait(&full[PAIR ? (sg & ~1) : sg], ps.ph);
#endif
#ifdef RB_PROF_SWEEP
          prof_full += clock64() - t1;
#endif
          tc_fence_after();
          if (M64) {  // tile (K-major) x B panel (MN-major, 4 boxes of 64 columns): M=64 N=256
#pragma unroll
            for (int kk = 0; kk < KCH / 16; ++kk)
              umma_f16(d, bdesc0 + soff + kk * 2, adesc0 + soff + ((kk * 2048) >> 4), idesc,
                       !(first && kc == 0 && kk == 0));
          } else if (n_mt == 2) {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
              for (int kk = 0; kk < KCH / 16; ++kk)
                umma_f16(d + mt * hp, adesc0 + soff + ((mt * 2 * BOX_BYTES + kk * 2048) >> 4), bdesc0 + soff + kk * 2,
                         idesc, !(first && kc == 0 && kk == 0));
          } else {
#pragma unroll
            for (int kk = 0; kk < KCH / 16; ++kk)
              umma_f16(d, adesc0 + soff + ((kk * 2048) >> 4), bdesc0 + soff + kk * 2, idesc,
                       !(first && kc == 0 && kk == 0));
          }
#ifndef RB_DBG_MMAONLY
          umma_commit(&empty[sg]);
#endif
          if (last && kc + 1 == a.dp_chunks) umma_commit(&sdone[slot]);
        }
        __syncwarp();
        ps.advance((ST / SW_MMA_WARPS));
      }
    }
#ifdef RB_PROF_SWEEP
    if (blockIdx.x % 8 == 0 && lane == 0)
      printf("sweep cta %d mma: total %lld wait_free %lld wait_full %lld steps %d\n", blockIdx.x, clock64() - prof_t0,
             prof_free, prof_full, s_end - s_begin);
#endif
  } else if (NOEPI_DBG) {
  } else if (M64) {
    // epilogue (M64): warp quadrant q = warp & 3 holds rows 16q..16q+15 of both lane halves; this
    // warp drains 128 of the slot's 256 columns (half ch).  A lane of the slot's half owns one row.
    const int q = warp & 3, ch = (warp - 1 - SW_MMA_WARPS) >> 2;
    float* epi_buf = reinterpret_cast<float*>(smem + ST * (ASLOT + S_B_BYTES) + 1024) +
                     (warp - 1 - SW_MMA_WARPS) * 16 * 36;  // 16 x 33 used
    uint32_t done_ph = 0;
    for (int j = w.done_ptr[blockIdx.x]; j < w.done_ptr[blockIdx.x + 1]; ++j) {
      const int4 c = w.done[j];
      const int g = c.x, n0 = c.y, slot = c.z;
      const int p0 = a.row_partition[g];
      const int h = a.row_partition[g + 1] - p0;
      const int row = 16 * q + (lane & 15);
      const bool mine = (lane >> 4) == (slot & 1) && row < h;
      const int crow = mine ? a.row_perm[p0 + row] : 0;
      if (lane == 0) mbar_wait_backoff(&sdone[slot], (done_ph >> slot) & 1, SW_EPI_SLEEP_NS);
      __syncwarp();
      done_ph ^= 1u << slot;
      tc_fence_after();
      uint32_t r[4][32];
      const uint32_t t0 = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((slot >> 1) * 256 + ch * 128);
#pragma unroll
      for (int k = 0; k < 4; ++k) tmem_ld_32x32b_x32(t0 + k * 32, r[k]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfree[slot]);
#ifdef RB_DBG_NOSTORE  // developer experiment: drain TMEM but do not store C
      if (mine && r[0][0] == 0x7f7f7f7fu) a.C[crow] = 0.f;
      continue;
#endif
      // A lane holds 32 consecutive columns of ITS row per chunk: stores straight from registers
      // would be 16 rows x 16 B per instruction, and that L1 traffic measurably slows the tensor
      // core's SMEM operand reads (config 5: 0.59 -> 0.83 kcycles per step).  Each chunk goes
      // through a 16 x 32 float SMEM tile instead (row stride 33 floats: conflict-free scalar writes
      // and reads) and leaves as 16 coalesced 128-byte row stores.
      const int nb = n0 + ch * 128;
      const int slab_rows = min(16, h - 16 * q);
      const int my_row = __shfl_sync(0xffffffffu, crow, (lane & 15) + 16 * (slot & 1));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if ((lane >> 4) == (slot & 1)) {  // row stride 33: lane i writes bank (i + t) % 32, no conflicts
          float* srow = epi_buf + (lane & 15) * 33;
#pragma unroll
          for (int t = 0; t < 32; ++t) srow[t] = __uint_as_float(r[k][t]);
        }
        __syncwarp();
        const int n = nb + k * 32 + lane;
        if (a.fan.n == 0) {  // the plain store loop (a fan-out test inside it cost config 5 ~10 %)
          for (int i = 0; i < slab_rows; ++i) {
            const int cr = __shfl_sync(0xffffffffu, my_row, i);
            if (n < a.N) a.C[(int64_t)cr * a.ldc + n] = epi_buf[i * 33 + lane];
          }
        } else {
          for (int i = 0; i < slab_rows; ++i) {
            const int cr = __shfl_sync(0xffffffffu, my_row, i);
            if (n < a.N) st_fan(a.fan, a.C, (int64_t)cr * a.ldc + n, epi_buf[i * 33 + lane]);
          }
        }
        __syncwarp();
      }
      (void)mine;
    }
  } else {
    // epilogue: drain finished slots in commit order; TMEM lane = C column, a warp stores 32
    // consecutive floats (128 B) of one C row per instruction
    const int q = warp & 3;
    uint32_t done_ph = 0;
#ifdef RB_PROF_SWEEP
    long long prof_wait = 0, prof_drain = 0, prof_max = 0, prof_ld = 0;
#endif
    for (int j = w.done_ptr[blockIdx.x]; j < w.done_ptr[blockIdx.x + 1]; ++j) {
      const int4 c = w.done[j];
      const int g = c.x, n0 = c.y, slot = c.z;
      const int p0 = a.row_partition[g];
      const int h = a.row_partition[g + 1] - p0;
      const int n_mt = min(a.short_ns / 128, (a.N - n0 + 127) / 128);
#ifdef RB_PROF_SWEEP
      const long long e0 = clock64();
#endif
      if (lane == 0) mbar_wait_backoff(&sdone[slot], (done_ph >> slot) & 1, SW_EPI_SLEEP_NS);
      __syncwarp();
#ifdef RB_PROF_SWEEP
      const long long e1 = clock64();
      prof_wait += e1 - e0;
#endif
      done_ph ^= 1u << slot;
      tc_fence_after();
      const uint32_t t0 = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(slot * 2 * hp);
      // the row's C row indices, one per lane (two registers cover h <= 64), fetched once: a load
      // per store would put 64 dependent global loads on the drain's critical path
      const int rp_lo = lane < h ? a.row_perm[p0 + lane] : 0;
      const int rp_hi = lane + 32 < h ? a.row_perm[p0 + 32 + lane] : 0;
      if (hp <= 64) {
        // Copy the whole slot (<= 2 M-tiles x 64 rows) to registers, hand the slot back to the MMA
        // warp, then store: the slot's reuse waits only for the TMEM reads, not for the C stores.
        uint32_t r[2][64];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          if (mt < n_mt) {
            const uint32_t ta = t0 + (uint32_t)(mt * hp);
            if (hp == 16) {
              tmem_ld_32x32b_x16(ta, *reinterpret_cast<uint32_t(*)[16]>(r[mt]));
            } else {
              tmem_ld_32x32b_x32(ta, *reinterpret_cast<uint32_t(*)[32]>(r[mt]));
              if (hp == 64) tmem_ld_32x32b_x32(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(r[mt] + 32));
            }
          }
        }
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sfree[slot]);
#ifdef RB_PROF_SWEEP
        prof_ld += clock64() - e1;
#endif
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int n = n0 + mt * 128 + q * 32 + lane;
          const bool nvalid = mt < n_mt && n < a.N;
          if (a.fan.n == 0) {
#pragma unroll
            for (int jj = 0; jj < 64; ++jj) {
              const int row = __shfl_sync(0xffffffffu, jj < 32 ? rp_lo : rp_hi, jj & 31);
              if (nvalid && jj < h) a.C[(int64_t)row * a.ldc + n] = __uint_as_float(r[mt][jj]);
            }
          } else {
#pragma unroll
            for (int jj = 0; jj < 64; ++jj) {
              const int row = __shfl_sync(0xffffffffu, jj < 32 ? rp_lo : rp_hi, jj & 31);
              if (nvalid && jj < h) st_fan(a.fan, a.C, (int64_t)row * a.ldc + n, __uint_as_float(r[mt][jj]));
            }
          }
        }
      } else {
        for (int mt = 0; mt < n_mt; ++mt) {
          const int n = n0 + mt * 128 + q * 32 + lane;
          const bool nvalid = n < a.N;
          for (int j0 = 0; j0 < h; j0 += 64) {  // up to 64 rows per TMEM round trip
            uint32_t r[64];
            const uint32_t ta = t0 + (uint32_t)(mt * hp + j0);
            tmem_ld_32x32b_x32(ta, *reinterpret_cast<uint32_t(*)[32]>(r));
            tmem_ld_32x32b_x32(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
            tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 64; ++jj) {
              const int row = j0 == 0 ? __shfl_sync(0xffffffffu, jj < 32 ? rp_lo : rp_hi, jj & 31)
                                      : a.row_perm[p0 + j0 + jj];
              if (nvalid && j0 + jj < h) st_fan(a.fan, a.C, (int64_t)row * a.ldc + n, __uint_as_float(r[jj]));
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sfree[slot]);
      }
#ifdef RB_PROF_SWEEP
      const long long e2 = clock64();
      prof_drain += e2 - e1;
      prof_max = max(prof_max, e2 - e1);
#endif
    }
#ifdef RB_PROF_SWEEP
    if (blockIdx.x % 37 == 0 && lane == 0)
      printf("sweep cta %d epi warp %d: wait %lld drain %lld (tmem->regs %lld) max_drain %lld rows %d\n", blockIdx.x,
             warp, prof_wait, prof_drain, prof_ld, prof_max, w.done_ptr[blockIdx.x + 1] - w.done_ptr[blockIdx.x]);
#endif
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
#ifdef RB_PROF_SWEEP
  if (threadIdx.x == 0 && blockIdx.x % 8 == 0) {
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    printf("sweep cta %d kernel: cycles %lld ns %llu start_ns %llu\n", blockIdx.x, clock64() - k_t0, g1 - k_g0, k_g0);
  }
#endif
}

// ------------------------------------------------------------------------------------------
// fp32 check path: CTA = (g, 8-row chunk r0, 128-col chunk n0); thread = one C column.
// Per row the accumulation order is blocks ascending, then k ascending (fixed, deterministic).
// T = float: the fp32 check path for h > 8.  T = double: the fp64 path (every block row), which
// multiplies exactly the segment width with the zeros of the dense block payload included, so it
// reproduces the reference's float64 arithmetic and its NaN / Inf propagation (multiply.py:89).
template <typename T>
__global__ void __launch_bounds__(SIMT_COLS) spmm_simt_kernel(SpmmArgs a, const T* __restrict__ tiles, int32_t dp,
                                                              const T* __restrict__ B, int64_t ldb, T* C) {
  const int4 it = a.items[blockIdx.x];
  const int g = it.x, r0 = it.y, n0 = it.z;
  const int p0 = a.row_partition[g];
  const int h = a.row_partition[g + 1] - p0;
  const int hp = tile_pitch(h);  // tile row pitch
  const int rows = min(SIMT_ROWS, h - r0);
  const int n = n0 + threadIdx.x;
  const bool nv = n < a.N;
  T acc[SIMT_ROWS];
#pragma unroll
  for (int r = 0; r < SIMT_ROWS; ++r) acc[r] = T(0);
  const int b0 = a.blk_ptr[g], b1 = a.blk_ptr[g + 1];
  const int64_t base = a.grp_tile_row[g];
  for (int b = b0; b < b1; ++b) {
    const int s = a.blk_col[b];
    const int k0 = a.col_bounds[s], w = a.col_bounds[s + 1] - k0;
    const T* t = tiles + (base + (int64_t)(b - b0) * hp + r0) * dp;
    const T* bp = B + (int64_t)k0 * ldb + n;
    if (rows == 1) {  // most short block rows have h = 1 (config 1): no wasted FMAs on padding rows
      for (int k = 0; k < w; ++k) {
        const T bv = nv ? __ldg(bp + (int64_t)k * ldb) : T(0);
        acc[0] = fma(__ldg(t + k), bv, acc[0]);
      }
    } else {
      for (int k = 0; k < w; ++k) {
        const T bv = nv ? __ldg(bp + (int64_t)k * ldb) : T(0);
#pragma unroll
        for (int r = 0; r < SIMT_ROWS; ++r)
          if (r < rows) acc[r] = fma(__ldg(t + r * dp + k), bv, acc[r]);
      }
    }
  }
  if (nv) {
    for (int r = 0; r < rows; ++r) {
      const int64_t off = (int64_t)a.row_perm[p0 + r0 + r] * a.ldc + n;
      C[off] = acc[r];
      if constexpr (sizeof(T) == sizeof(float))  // fan-out is float32 C only (the host refuses fp64)
        for (int f = 0; f < a.fan.n; ++f) a.fan.p[f][off] = acc[r];
    }
  }
}

// ------------------------------------------------------------------------------------------
// Rows of block rows without stored blocks: C[row_perm[pos], 0:N] = 0 with float4 stores
// (multiply.py:85-86 leaves them exactly 0).  A warp takes 32 rows at a time: each lane resolves
// one row's offset (one coalesced pos[] load and one row_perm gather for all 32), then the warp
// zeroes the rows one after another.  One dependent-load chain per 32 rows instead of per row keeps
// the kernel store-bound.
__global__ void __launch_bounds__(256) zero_rows_kernel(const int32_t* __restrict__ pos, int64_t n,
                                                        const int32_t* __restrict__ row_perm, float* C, int64_t ldc,
                                                        int32_t N, CFan fan) {
  const int lane = threadIdx.x & 31;
  const bool vec = ((ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
  const int n4 = N >> 2;
  const int64_t n_batches = (n + 31) >> 5;
  for (int64_t bt = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; bt < n_batches;
       bt += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t r0 = bt << 5;
    const int cnt = n - r0 < 32 ? (int)(n - r0) : 32;
    const int64_t my_off = lane < cnt ? (int64_t)row_perm[pos[r0 + lane]] * ldc : 0;
    for (int j = 0; j < cnt; ++j) {
      const int64_t off = __shfl_sync(0xffffffffu, my_off, j);
      for (int f = -1; f < fan.n; ++f) {  // C, then every fan-out copy
        float* dst = (f < 0 ? C : fan.p[f]) + off;
        if (vec) {
          for (int c = lane; c < n4; c += 32) reinterpret_cast<float4*>(dst)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int c = (n4 << 2) + lane; c < N; c += 32) dst[c] = 0.f;
        } else {
          for (int c = lane; c < N; c += 32) dst[c] = 0.f;
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// host side

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static int make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, uint64_t inner, uint64_t outer,
                        uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                        CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) return fail(RB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  {  // a driver-API call: make the device's primary context current in this host thread (a thread
     // whose first CUDA call this is has none yet -> CUDA_ERROR_INVALID_CONTEXT)
    int dev = 0;
    RB_CUDA_TRY(cudaGetDevice(&dev));
    RB_CUDA_TRY(cudaSetDevice(dev));
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return fail(RB_EINVAL, "TMA base must be 16-byte aligned");
  if (row_bytes % 16 != 0) return fail(RB_EINVAL, "TMA row stride must be a multiple of 16 bytes");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(RB_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return RB_OK;
}

// Work unit of the shard planner: rows of one tall pair tile (256), a whole short block row, or an
// 8-row chunk on the fp32 path.
static int unit_rows(bool tc, int h) { return !tc ? SIMT_ROWS : is_short_row(h) ? h : PAIR_BM; }

// Shard = contiguous range of permuted rows, cut at work-unit boundaries so that every C row (and
// every work item) belongs to exactly one shard.  Weight = padded MMA work (K chunks + 1) x rows;
// a unit goes to the shard owning its weight midpoint.
int shard_range(const int32_t* rp, const int32_t* bp, int64_t H, int32_t b_dtype, int32_t dp, int32_t shard,
                int32_t n_shards, int64_t* row_lo, int64_t* row_hi) {
  if (n_shards < 1 || shard < 0 || shard >= n_shards) return fail(RB_EINVAL, "bad shard");
  const bool tc = (b_dtype == RB_BF16 || b_dtype == RB_F16);
  const int dpc = tc ? std::max(1, dp / KCH) : 1;
  struct Unit {
    int64_t r0, r1;
    double w;
  };
  std::vector<Unit> units;
  units.reserve(H);
  double total = 0;
  for (int64_t g = 0; g < H; ++g) {
    const int h = rp[g + 1] - rp[g];
    const int nb = bp[g + 1] - bp[g];
    if (h <= 0) continue;
    const int step = unit_rows(tc, h);
    for (int r = 0; r < h; r += step) {
      const int rows = std::min(step, h - r);
      const double w = (nb * (double)dpc + 1.0) * (tc ? (is_short_row(h) ? hp_of(h) : PAIR_BM) : rows);
      units.push_back({rp[g] + r, rp[g] + r + rows, w});
      total += w;
    }
  }
  const double lo = total * shard / n_shards, hi = total * (shard + 1) / n_shards;
  double acc = 0;
  int64_t first = -1, last = -1, before = 0;
  for (auto& u : units) {
    const double mid = acc + 0.5 * u.w;
    acc += u.w;
    if (mid < lo) before = u.r1;
    const bool mine = mid >= lo && (mid < hi || shard == n_shards - 1);
    if (mine) {
      if (first < 0) first = u.r0;
      last = u.r1;
    }
  }
  if (first < 0) first = last = before;  // empty shard: empty range after the previous shards
  *row_lo = first;
  *row_hi = last;
  return RB_OK;
}

}  // namespace rb

struct rb_spmm_plan {
  rb_vbr_device v;
  int64_t N;
  int32_t b_dtype;
  int4* d_items = nullptr;  // tall units (2 x int4 each), then short items, then simt items
  float* d_ws = nullptr;    // split-K partials of the tall tail
  int32_t* d_cnt = nullptr;
  int64_t n_split_slots = 0;
  int32_t short_ns = rb::SHORT_NS;
  int64_t n_tall = 0, n_short = 0, n_simt = 0;
  rb::SkinnyItem* d_skinny = nullptr;  // skinny items, grouped by height class
  int32_t* d_zero = nullptr;            // permuted positions of rows in block rows without blocks
  int32_t* d_short_ptr = nullptr;       // per-CTA ranges of the short items (short_schedule)
  int32_t short_ctas = 0;
  int64_t n_zero = 0;
  std::vector<int4> tall_items;         // (g, m, n0, -) before K splitting (for the 2:4 re-plan)
  int64_t shard_lo = 0, shard_hi = 0;
  // 2:4 sparse path (rb_spmm_plan_attach_sparse24)
  bool use_sp = false;
  rb_sparse24_device sp{};
  CUtensorMap tmSP, tmSPE;
  int4* d_sp_units = nullptr;
  int64_t n_sp_units = 0;
  float* d_sp_ws = nullptr;
  int32_t* d_sp_cnt = nullptr;
  rb::SkinnyItem* d_res_items = nullptr;
  int64_t n_res_items = 0;
  unsigned long long* d_res_sched = nullptr;
  // Executions of one plan are serialised: the work counters, split partials and schedules above
  // are per-plan device state that every launch resets itself, so two executions must never
  // overlap.  `mu` makes rb_spmm_execute safe from several host threads; `done` (recorded at the
  // end of every execution) is waited on by the next execution when it comes on another stream.
  mutable std::mutex mu;
  mutable cudaEvent_t done = nullptr;
  mutable cudaStream_t done_stream = nullptr;
  mutable bool done_valid = false;
  // fork/join streams of rb_spmm_execute (created on first use)
  mutable bool aux_ready = false;
  mutable cudaStream_t aux[rb::kAuxStreams] = {};
  mutable cudaEvent_t ev[rb::kAuxStreams + 1] = {};
  float* d_skinny_ws = nullptr;     // partials of split skinny block rows
  int32_t* d_skinny_cnt = nullptr;
  unsigned long long* d_sched = nullptr;  // 2 work counters per skinny height class
  int64_t skinny_off[rb::SKINNY_CLASSES + 1] = {0, 0, 0, 0, 0};
  rb::SkinnyItem* d_cmp_items = nullptr;  // compact-payload rows (CSR engine over permuted rows)
  int64_t n_cmp_items = 0;
  int32_t cmp_chunk = 1;  // items per claim in the CSR engine (csr_claim_chunk)
  unsigned long long* d_cmp_sched = nullptr;
  CUtensorMap tmA16, tmA32, tmA64, tmA128;
  // multi-slot sweep (spmm_sweep_kernel) for the dominant short height class
  int4* d_sw_steps = nullptr;
  int32_t* d_sw_step_ptr = nullptr;
  int4* d_sw_done = nullptr;
  int32_t* d_sw_done_ptr = nullptr;
  int32_t sw_hp = 0, sw_ctas = 0, sw_slots = 0;
  int64_t n_sw_steps = 0;
  rb_spmm_info info;
};

using namespace rb;

namespace {

// Static round-robin makespan (the persistent kernel hands unit i to pair i % P) in K steps; each
// split unit pays `split_cost` extra steps for parking and re-reading its partial.
double rr_makespan(const std::vector<int>& len, const std::vector<int>& nsplit, int P, double split_cost) {
  std::vector<double> t(P, 0.0);
  for (size_t i = 0; i < len.size(); ++i) t[i % P] += len[i] + (nsplit[i] > 1 ? split_cost : 0.0);
  return *std::max_element(t.begin(), t.end());
}

// Tall items (g, m, n0, L = K steps), LPT-sorted, become units.  The last partial wave is the
// tail: keep every full wave whole and, when the tail leaves more than half of the P pairs idle,
// split each tail item into s equal K ranges (r*s <= P, units >= 64 K steps), choosing the s with
// the smallest static makespan.  Measured on B200 (tools/split_probe.py, tools/shard_sim.py): a
// split costs far more than its partial bytes suggest (the parked partials and the final reduce
// sit on the critical path at the very end), so a 3/4-full tail (config 4: 54 of 74 pairs) is
// left alone; config 2 (34 of 74) splits in two (0.674 -> 0.632 ms), and small shards (config 4
// at 8 ranks: 16 items for 74 pairs) split in four.  A split item's units are adjacent so they
// run concurrently on neighbouring pairs.
void split_tail(const std::vector<int4>& items, int P, std::vector<int4>& units, int64_t& n_slots) {
  const int n = (int)items.size();
  const int full = P > 0 ? n / P : n;
  int best_s = 1;
  const char* env = std::getenv("RB_TALL_SPLIT");
  const int max_s = env ? std::max(1, std::min(MAX_SPLIT, std::atoi(env))) : MAX_SPLIT;
  const int r = n - full * P;
  if (P > 0 && r > 0 && 2 * r <= P && max_s > 1) {  // only a tail wave that leaves most pairs idle
    auto eval = [&](int s) {
      std::vector<int> len, ns;
      for (int i = 0; i < n; ++i) {
        const int L = items[i].w;
        const int si = (i >= full * P && L >= 64 * s) ? s : 1;
        for (int j = 0; j < si; ++j) {
          len.push_back(L * (j + 1) / si - L * j / si);
          ns.push_back(si);
        }
      }
      return rr_makespan(len, ns, P, 8.0);
    };
    double best = eval(1);
    for (int s = 2; s <= max_s && r * s <= P; ++s) {
      const double t = eval(s);
      if (t < best * 0.95) {
        best = t;
        best_s = s;
      }
    }
  }
  const int best_f = full;
  n_slots = 0;
  for (int i = 0; i < n; ++i) {
    const int4 it = items[i];
    const int L = it.w;
    const int si = (i >= best_f * P && best_s > 1 && L >= 64 * best_s) ? best_s : 1;
    const int slot = si > 1 ? (int)n_slots++ : -1;
    for (int j = 0; j < si; ++j) {
      units.push_back(make_int4(it.x, it.y, it.z, L * j / si));
      units.push_back(make_int4(L * (j + 1) / si, j, si, slot));
    }
  }
}

}  // namespace

extern "C" int rb_spmm_shard_range(const int32_t* row_partition, const int32_t* blk_ptr, int64_t n_block_rows,
                                   int32_t b_dtype, int32_t dp, int32_t shard, int32_t n_shards, int64_t* row_begin,
                                   int64_t* row_end) {
  if (!row_partition || !blk_ptr || !row_begin || !row_end || n_block_rows < 0) return fail(RB_EINVAL, "bad arguments");
  return shard_range(row_partition, blk_ptr, n_block_rows, b_dtype, dp, shard, n_shards, row_begin, row_end);
}

// Static balanced schedule of the short items: list scheduling, in the given order, onto `ctas`
// CTAs (each item goes to the CTA that frees up first under a bytes-per-K-step cost model); the
// items are then regrouped CTA-contiguously and cta_ptr[b] .. cta_ptr[b+1] is CTA b's sequence.
// Within one column slab the block rows go longest first, so the slab-major order that keeps the
// B slab hot in L2 is kept while the partial last wave of every rank's shard is filled evenly.
static void short_schedule(std::vector<int4>& items, int ctas, int dpc, bool slab_major,
                           std::vector<int32_t>& cta_ptr) {
  if (slab_major)
    std::stable_sort(items.begin(), items.end(), [](const int4& x, const int4& y) {
      return x.z != y.z ? x.z < y.z : x.w > y.w;
    });
  // cost in 8 KB units: per K step 4 B boxes + the hp x 64 tile; per item ~2 units of setup
  std::vector<double> fin(ctas, 0.0);
  std::vector<int32_t> owner(items.size());
  using E = std::pair<double, int>;
  std::priority_queue<E, std::vector<E>, std::greater<E>> heap;
  for (int c = 0; c < ctas; ++c) heap.push({0.0, c});
  std::vector<int32_t> count(ctas, 0);
  for (size_t i = 0; i < items.size(); ++i) {
    const int4& it = items[i];
    const double cost = (double)it.w * dpc * (4.0 + it.y / 64.0) + 2.0;
    E top = heap.top();
    heap.pop();
    owner[i] = top.second;
    ++count[top.second];
    heap.push({top.first + cost, top.second});
  }
  cta_ptr.assign(ctas + 1, 0);
  for (int c = 0; c < ctas; ++c) cta_ptr[c + 1] = cta_ptr[c] + count[c];
  std::vector<int4> out(items.size());
  std::vector<int32_t> pos(cta_ptr.begin(), cta_ptr.end() - 1);
  for (size_t i = 0; i < items.size(); ++i) out[pos[owner[i]]++] = items[i];
  items.swap(out);
}

// Static multi-slot sweep schedule (spmm_sweep_kernel).  Block rows are assigned to CTAs by LPT on
// their block counts (the same rows for every slab); CTA c's queue is its rows for slab 0, then for
// slab 1, ...  A CTA holds n_slots rows at a time and repeatedly takes, among the resident rows
// whose slot is usable, the one whose next block column is the nearest ahead of the CTA's current
// block column (circular), so it sweeps block columns 0..nbc-1 over and over with all its rows
// merged.  A row entering a slot starts at the first of its blocks at or after the current block
// column (rotation) and wraps around.  A freed slot becomes usable `delay` steps after its row's
// last step (time for the epilogue to drain it while the other slots keep the MMA busy).
static void sweep_schedule(const std::vector<int32_t>& rows, const std::vector<int32_t>& slabs,
                           const std::vector<int32_t>& rp, const std::vector<int32_t>& bp,
                           const std::vector<int32_t>& bcol, const std::vector<int64_t>& tile_row,
                           const std::vector<int32_t>& col_bounds, int64_t n_seg, int ctas, int n_slots, int delay,
                           int dpc, std::vector<int4>& steps, std::vector<int32_t>& step_ptr, std::vector<int4>& done,
                           std::vector<int32_t>& done_ptr) {
  // LPT over (block row, slab) items rather than whole block rows: with few rows per CTA (a rank's
  // shard at 8 GPUs: 512 block rows for 148 CTAs) whole-row assignment leaves a 4-vs-3-rows
  // imbalance; items balance to within one item.  Each CTA then walks its items slab by slab.
  std::vector<std::vector<int2>> mine(ctas);  // (g, slab index)
  {
    // slab by slab (longest rows first within a slab) onto one running heap: every CTA gets about
    // the same work in every slab, so the CTAs leave a slab together and the live B window stays
    // within one slab, while the totals still balance to one item
    std::vector<int32_t> by_len(rows);
    std::stable_sort(by_len.begin(), by_len.end(),
                     [&](int32_t x, int32_t y) { return bp[x + 1] - bp[x] > bp[y + 1] - bp[y]; });
    std::vector<int2> order;
    order.reserve(rows.size() * slabs.size());
    for (int32_t si = 0; si < (int32_t)slabs.size(); ++si)
      for (int32_t g : by_len) order.push_back(make_int2(g, si));
    using E = std::pair<double, int>;
    std::priority_queue<E, std::vector<E>, std::greater<E>> heap;
    for (int c = 0; c < ctas; ++c) heap.push({0.0, c});
    for (const int2& it : order) {
      E top = heap.top();
      heap.pop();
      mine[top.second].push_back(it);
      heap.push({top.first + (bp[it.x + 1] - bp[it.x]) * (double)dpc + 2.0, top.second});
    }
    for (auto& m : mine)
      std::stable_sort(m.begin(), m.end(), [](const int2& x, const int2& y) { return x.y < y.y; });
  }
  steps.clear();
  done.clear();
  step_ptr.assign(1, 0);
  done_ptr.assign(1, 0);
  struct Slot {
    int32_t g = -1, n0 = 0, nb = 0, start = 0, count = 0;
    bool started = false;
    int64_t usable = 0;
    int32_t first_phase = -1;  // start column of the slot's first row (staggered); -1 afterwards
  };
  for (int c = 0; c < ctas; ++c) {
    std::vector<int2> queue;  // (g, n0)
    for (const int2& it : mine[c]) queue.push_back(make_int2(it.x, slabs[it.y]));
    size_t qi = 0;
    // A row ends where it started (it wraps around once), so rows that start together also finish
    // together and their drains would queue behind each other while the MMA waits for a slot.  The
    // slots' first rows therefore start at evenly spaced block columns; every later row starts
    // where its slot's previous row ended, so completions stay spread over the revolution.
    std::vector<Slot> slot(n_slots);
    for (int s = 0; s < n_slots; ++s) slot[s].first_phase = (int32_t)((int64_t)s * n_seg / n_slots);
    int32_t phase = 0;
    int64_t k = 0;
    int active = 0;
    for (;;) {
      for (int s = 0; s < n_slots; ++s)
        if (slot[s].g < 0 && qi < queue.size()) {
          slot[s].g = queue[qi].x;
          slot[s].n0 = queue[qi].y;
          slot[s].nb = bp[slot[s].g + 1] - bp[slot[s].g];
          slot[s].count = 0;
          slot[s].started = false;
          ++qi;
          ++active;
        }
      if (active == 0) break;
      int best = -1;
      int64_t best_key = 0;
      for (int s = 0; s < n_slots; ++s) {
        Slot& r = slot[s];
        if (r.g < 0) continue;
        const int32_t* cols = bcol.data() + bp[r.g];
        if (!r.started && r.usable <= k) {  // rotation: first block at or after the current column
          const int32_t at = r.first_phase >= 0 ? r.first_phase : phase;
          r.first_phase = -1;
          r.start = (int32_t)(std::lower_bound(cols, cols + r.nb, at) - cols);
          if (r.start == r.nb) r.start = 0;
          r.started = true;
        }
        int64_t key;
        if (!r.started) {
          key = (int64_t)1 << 40 | r.usable;  // not usable yet: only if nothing else is
        } else {
          const int32_t b = cols[(r.start + r.count) % r.nb];
          key = ((int64_t)(b - phase) + (b < phase ? (int64_t)1 << 30 : 0));
        }
        if (best < 0 || key < best_key) {
          best = s;
          best_key = key;
        }
      }
      Slot& r = slot[best];
      if (!r.started) {  // every resident row waits for its slot: start it now (the MMA stalls)
        const int32_t* cols = bcol.data() + bp[r.g];
        r.start = (int32_t)(std::lower_bound(cols, cols + r.nb, phase) - cols);
        if (r.start == r.nb) r.start = 0;
        r.started = true;
      }
      const int32_t t = (r.start + r.count) % r.nb;
      const int32_t blk = bp[r.g] + t;
      const bool first = r.count == 0, last = r.count + 1 == r.nb;
      // the kernel's step: A tile row, first B row of the block's segment, n0, slot | first | last
      const int64_t trow = tile_row[r.g] + (int64_t)t * tile_pitch(rp[r.g + 1] - rp[r.g]);
      steps.push_back(make_int4((int32_t)trow, col_bounds[bcol[blk]], r.n0,
                                best | (first ? 1 << 8 : 0) | (last ? 1 << 9 : 0)));
      phase = bcol[blk];
      ++k;
      if (++r.count == r.nb) {
        done.push_back(make_int4(r.g, r.n0, best, 0));
        r.g = -1;
        r.usable = k + delay;
        --active;
      }
    }
    step_ptr.push_back((int32_t)steps.size());
    done_ptr.push_back((int32_t)done.size());
  }
}

extern "C" int rb_spmm_plan_create_ex(const rb_vbr_device* vbr, int64_t N, int32_t b_dtype, int32_t shard,
                                      int32_t n_shards, int32_t work_shards, rb_spmm_plan** out, void* stream_);

extern "C" int rb_spmm_plan_create(const rb_vbr_device* vbr, int64_t N, int32_t b_dtype, int32_t shard,
                                   int32_t n_shards, rb_spmm_plan** out, void* stream_) {
  return rb_spmm_plan_create_ex(vbr, N, b_dtype, shard, n_shards, n_shards, out, stream_);
}

extern "C" int rb_spmm_plan_create_ex(const rb_vbr_device* vbr, int64_t N, int32_t b_dtype, int32_t shard,
                                      int32_t n_shards, int32_t work_shards, rb_spmm_plan** out, void* stream_) {
  rb::NvtxRange nvtx_range_("rb_spmm_plan_create");
  if (work_shards < n_shards) work_shards = n_shards;
  if (!vbr || !out) return fail(RB_EINVAL, "null argument");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const bool tc = (b_dtype == RB_BF16 || b_dtype == RB_F16);
  const bool f64 = b_dtype == RB_F64;
  if (!tc && !f64 && b_dtype != RB_F32) return fail(RB_EUNSUPPORTED, "B dtype must be bf16, f16, f32 or f64");
  if (tc && vbr->tile_dtype != b_dtype) return fail(RB_EINVAL, "tile dtype must equal B dtype");
  if (!tc && !f64 && vbr->tile_dtype != RB_F32) return fail(RB_EINVAL, "fp32 path needs fp32 tiles");
  if (f64 && vbr->tile_dtype != RB_F64) return fail(RB_EINVAL, "fp64 path needs fp64 tiles");
  if (tc && (vbr->dp <= 0 || vbr->dp % 64 != 0)) return fail(RB_EINVAL, "dp must be a positive multiple of 64");
  if (N <= 0 || N > (1ll << 30)) return fail(RB_EINVAL, "bad n_dense_cols");
  if (n_shards < 1 || shard < 0 || shard >= n_shards) return fail(RB_EINVAL, "bad shard");
  const int64_t H = vbr->n_block_rows;
  std::vector<int32_t> rp(H + 1), bp(H + 1);
  if (H > 0) {
    RB_CUDA_TRY(cudaMemcpyAsync(rp.data(), vbr->row_partition, sizeof(int32_t) * (H + 1), cudaMemcpyDeviceToHost,
                                stream));
    RB_CUDA_TRY(cudaMemcpyAsync(bp.data(), vbr->blk_ptr, sizeof(int32_t) * (H + 1), cudaMemcpyDeviceToHost, stream));
    RB_CUDA_TRY(cudaStreamSynchronize(stream));
  }
  int64_t row_lo = 0, row_hi = 0;
  {
    int rc = shard_range(rp.data(), bp.data(), H, b_dtype, vbr->dp, shard, n_shards, &row_lo, &row_hi);
    if (rc) return rc;
  }
  std::vector<int4> tall, shrt, simt;
  double exec_flops = 0, vbr_flops = 0, core_vbr_flops = 0;
  const int dpc = tc ? vbr->dp / KCH : 1;
  // short items: item order n-chunk-major keeps one 256-column B slab hot in L2 while A tiles stream
  // (RB_SHORT_ORDER=g switches to block-row-major)
  const char* order_env = std::getenv("RB_SHORT_ORDER");
  const bool short_g_major = order_env && order_env[0] == 'g';
  // column chunk of the short items: 256 (two M-tiles; each A tile is read N/256 times).  Measured on
  // config 5 (B slab per chunk 134 MB > L2): 128 halves B misses but doubles A reads and is 1.5x
  // slower, so 256 is the default.  RB_SHORT_NS=128 overrides.
  int32_t short_ns = rb::SHORT_NS;
  if (const char* ns_env = std::getenv("RB_SHORT_NS")) short_ns = std::atoi(ns_env) >= 256 ? 256 : 128;
  // block rows with h <= skinny_h run on the CUDA cores (spmm_skinny.cu): a tensor-core tile would
  // be >= 15/16 padding rows.  fp32 path: h <= 8; tensor path: h <= 4 (RB_SKINNY_H overrides, 0..8).
  int skinny_h = tc ? 4 : 8;
  if (const char* sk = std::getenv("RB_SKINNY_H")) skinny_h = std::max(0, std::min(8, std::atoi(sk)));
  if (f64) skinny_h = 0;  // fp64: every block row on the float64 SIMT kernel
  const int sk_cols = skinny_cols(b_dtype, N);
  std::vector<SkinnyItem> skinny[SKINNY_CLASSES];
  std::vector<int32_t> zero_rows;  // permuted positions of the rows of empty block rows
  int64_t sk_slots = 0, sk_units = 0;
  std::vector<int32_t> short_rows;
  std::vector<int2> skinny_rows;  // (g, nb), turned into items once the class totals are known
  // compact payloads (rb_vbr_compact_*): skinny block rows of h <= cmp_h are multiplied from their
  // nonzeros (CSR engine over permuted rows) rather than from their padded tiles
  const bool use_cmp = vbr->cmp_ptr && vbr->cmp_col && vbr->cmp_val && vbr->cmp_h > 0 && b_dtype != RB_F64;
  std::vector<int64_t> cmp;
  if (use_cmp) {
    cmp.resize(vbr->n_rows + 1);
    RB_CUDA_TRY(cudaMemcpyAsync(cmp.data(), vbr->cmp_ptr, sizeof(int64_t) * (vbr->n_rows + 1),
                                cudaMemcpyDeviceToHost, stream));
    RB_CUDA_TRY(cudaStreamSynchronize(stream));
  }
  std::vector<SkinnyItem> cmp_items;
  for (int64_t g = 0; g < H; ++g) {
    const int h = rp[g + 1] - rp[g];
    const int nb = bp[g + 1] - bp[g];
    if (h <= 0 || rp[g + 1] <= row_lo || rp[g] >= row_hi) continue;
    if (nb == 0) {  // no stored blocks: C rows are exact zeros (multiply.py:85-86), one coalesced pass
      for (int64_t i = std::max<int64_t>(rp[g], row_lo); i < std::min<int64_t>(rp[g + 1], row_hi); ++i)
        zero_rows.push_back((int32_t)i);
      continue;
    }
    if (h <= skinny_h && use_cmp && h <= vbr->cmp_h) {
      // one CSR item per row and C-column slab; hub rows split into CSR_PART_NNZ parts reduced in
      // part order by the last-arriving part (same workspace as the skinny split rows)
      for (int64_t pos = std::max<int64_t>(rp[g], row_lo); pos < std::min<int64_t>(rp[g + 1], row_hi); ++pos) {
        const int64_t nz = cmp[pos + 1] - cmp[pos];
        if (nz <= 0) continue;  // an empty row inside a non-empty block row: written below as zeros
        const int nparts = nz > CMP_PART_NNZ ? (int)((nz + CMP_PART_NNZ - 1) / CMP_PART_NNZ) : 1;
        for (int64_t n0 = 0; n0 < N; n0 += sk_cols) {
          if (nparts == 1) {
            cmp_items.push_back(SkinnyItem{(int32_t)pos, (int32_t)n0, 0, (int32_t)nz, 0, 1, -1, 0});
            continue;
          }
          const int32_t slot = (int32_t)sk_slots++, wsoff = (int32_t)sk_units;
          sk_units += (int64_t)nparts * (sk_cols / 128);
          for (int q = 0; q < nparts; ++q)
            cmp_items.push_back(SkinnyItem{(int32_t)pos, (int32_t)n0, (int32_t)(nz * q / nparts),
                                           (int32_t)(nz * (q + 1) / nparts), q, nparts, slot, wsoff});
        }
      }
      for (int64_t pos = std::max<int64_t>(rp[g], row_lo); pos < std::min<int64_t>(rp[g + 1], row_hi); ++pos)
        if (cmp[pos + 1] == cmp[pos]) zero_rows.push_back((int32_t)pos);
      exec_flops += 2.0 * (double)(cmp[rp[g + 1]] - cmp[rp[g]]) * N;
      vbr_flops += 2.0 * nb * h * (double)vbr->dp * N;
      core_vbr_flops += 2.0 * nb * h * (double)vbr->dp * N;
    } else if (h <= skinny_h) {
      skinny_rows.push_back(make_int2((int)g, nb));
      exec_flops += 2.0 * nb * h * (double)vbr->dp * N;
      vbr_flops += 2.0 * nb * h * (double)vbr->dp * N;
      core_vbr_flops += 2.0 * nb * h * (double)vbr->dp * N;
    } else if (!tc) {
      for (int r0 = 0; r0 < h; r0 += SIMT_ROWS) {
        if (rp[g] + r0 < row_lo || rp[g] + r0 >= row_hi) continue;
        for (int64_t n0 = 0; n0 < N; n0 += SIMT_COLS) simt.push_back(make_int4((int)g, r0, (int)n0, nb));
        exec_flops += 2.0 * nb * std::min(SIMT_ROWS, h - r0) * (double)vbr->dp * N;
        vbr_flops += 2.0 * nb * std::min(SIMT_ROWS, h - r0) * (double)vbr->dp * N;
        core_vbr_flops += 2.0 * nb * std::min(SIMT_ROWS, h - r0) * (double)vbr->dp * N;
      }
    } else if (is_short_row(h)) {
      short_rows.push_back((int32_t)g);
      exec_flops += 2.0 * nb * dpc * KCH * hp_of(h) * (double)((N + 127) / 128 * 128);  // M tiles of 128
      vbr_flops += 2.0 * nb * h * (double)vbr->dp * N;
    } else {
      for (int m = 0; m < (h + PAIR_BM - 1) / PAIR_BM; ++m) {
        if (rp[g] + m * PAIR_BM < row_lo || rp[g] + m * PAIR_BM >= row_hi) continue;
        for (int64_t n0 = 0; n0 < N; n0 += TALL_BN) tall.push_back(make_int4((int)g, m, (int)n0, nb * dpc));
        exec_flops += 2.0 * nb * dpc * KCH * PAIR_BM * (double)((N + TALL_BN - 1) / TALL_BN * TALL_BN);
        vbr_flops += 2.0 * nb * std::min(PAIR_BM, h - m * PAIR_BM) * (double)vbr->dp * N;
      }
    }
  }
  {
    // Part size per height class: hub rows are always cut at SKINNY_PART_BLOCKS; a class with little
    // work (config 1's few 4..8-row block rows) is cut finer so that ~8 units per SM exist — a part
    // is a serial chain of staged batches, and one group working through a 30-block row alone is
    // the whole step's latency.
    int64_t cls_blocks[SKINNY_CLASSES] = {0, 0, 0, 0};
    for (const int2& r : skinny_rows) cls_blocks[skinny_class(rp[r.x + 1] - rp[r.x])] += r.y;
    int dev_ = 0, sms_ = kNumSMs;
    RB_CUDA_TRY(cudaGetDevice(&dev_));
    RB_CUDA_TRY(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev_));
    const int64_t target = 8LL * sms_;
    int part[SKINNY_CLASSES];
    for (int c = 0; c < SKINNY_CLASSES; ++c) {
      const int nb_batch = std::max(2, 32 / skinny_class_h(c));  // blocks per staged batch (LPR / H)
      const int64_t want = (cls_blocks[c] + target - 1) / std::max<int64_t>(target, 1);
      int min_batches = 1;
      if (const char* e = std::getenv("RB_SKINNY_MIN_BATCHES")) min_batches = std::max(1, std::atoi(e));
      // A shard holds 1/n_shards of the work but still a whole hub row: R-MAT hub rows are ~20x denser
      // per block than the average skinny row, so at 4+ ranks their 256-block parts become the
      // critical path (config 3, 8 ranks: 0.76 -> 0.48 ms with 64-block parts).  One GPU keeps 256
      // (smaller parts cost more reduction than they save there).
      int part_max = work_shards >= 8 ? SKINNY_PART_BLOCKS / 4
                     : work_shards >= 4 ? SKINNY_PART_BLOCKS / 2 : SKINNY_PART_BLOCKS;
      if (const char* e = std::getenv("RB_SKINNY_PART_MAX")) part_max = std::max(1, std::atoi(e));
      part[c] = (int)std::min<int64_t>(part_max, std::max<int64_t>(min_batches * nb_batch, want));
    }
    for (const int2& r : skinny_rows) {
      const int h = rp[r.x + 1] - rp[r.x];
      const int c = skinny_class(h);
      skinny_items_for_row(r.x, h, bp[r.x], r.y, N, sk_cols, skinny[c], sk_slots, sk_units, part[c]);
    }
  }
  // Multi-slot sweep for the short height class with the most work, when it fills every CTA's slots
  // at least once (RB_SWEEP=0 turns it off, RB_SWEEP=2 forces it; RB_SWEEP_DELAY = slot reuse delay in
  // steps).
  std::vector<int32_t> sw_rows;
  int sw_hp = 0, sw_slots = 0;
  {
    const char* e = std::getenv("RB_SWEEP");
    bool on = tc && !(e && e[0] == '0') && !short_g_major;
    double work[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    auto cls = [](int hp) { return hp == 16 ? 0 : hp == 32 ? 1 : hp == 64 ? 2 : 3; };
    for (int32_t g : short_rows) {
      const int hp = hp_of(rp[g + 1] - rp[g]);
      work[cls(hp)] += (double)(bp[g + 1] - bp[g]) * hp;
      ++cnt[cls(hp)];
    }
    int best = 0;
    for (int c = 1; c < 4; ++c)
      if (work[c] > work[best]) best = c;
    const int hp = 16 << best;
    const int slots = std::min(MAX_SLOTS, 512 / (2 * hp));
    int dev_ = 0, sms_ = kNumSMs;
    RB_CUDA_TRY(cudaGetDevice(&dev_));
    RB_CUDA_TRY(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev_));
    const int64_t n_slabs = (N + short_ns - 1) / short_ns;
    const bool force = e && e[0] == '2';  // tests: sweep even a class that cannot fill the slots
    if (vbr->total_tile_rows >= (1ll << 31) || vbr->n_cols >= (1ll << 31)) on = false;  // int32 step fields
    if (on && work[best] > 0 && (force || cnt[best] * n_slabs >= (int64_t)sms_ * slots)) {
      sw_hp = hp;
      sw_slots = slots;
      std::vector<int32_t> rest;
      for (int32_t g : short_rows) (hp_of(rp[g + 1] - rp[g]) == hp ? sw_rows : rest).push_back(g);
      short_rows.swap(rest);
    }
  }
  if (short_g_major) {
    for (int32_t g : short_rows)
      for (int64_t n0 = 0; n0 < N; n0 += short_ns)
        shrt.push_back(make_int4(g, hp_of(rp[g + 1] - rp[g]), (int)n0, bp[g + 1] - bp[g]));
  } else {
    for (int64_t n0 = 0; n0 < N; n0 += short_ns)
      for (int32_t g : short_rows) shrt.push_back(make_int4(g, hp_of(rp[g + 1] - rp[g]), (int)n0, bp[g + 1] - bp[g]));
  }
  // Longest-first (LPT against the tail) for the tall items, stable so the N chunks of one pair tile
  // stay adjacent (they run concurrently and share the A tile through L2).
  std::stable_sort(tall.begin(), tall.end(), [](const int4& x, const int4& y) { return x.w > y.w; });
  int dev = 0, sms = kNumSMs;
  RB_CUDA_TRY(cudaGetDevice(&dev));
  RB_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  std::vector<int4> tall_units;
  int64_t n_slots = 0;
  split_tail(tall, sms / 2, tall_units, n_slots);
  std::vector<int32_t> short_ptr;
  const int short_ctas = (int)std::min<int64_t>(sms, (int64_t)shrt.size());
  if (short_ctas > 0) short_schedule(shrt, short_ctas, dpc, !short_g_major, short_ptr);

  auto* p = new rb_spmm_plan();
  p->v = *vbr;
  p->N = N;
  p->b_dtype = b_dtype;
  p->short_ns = short_ns;
  p->n_tall = (int64_t)tall_units.size() / 2;
  p->tall_items = tall;
  p->shard_lo = row_lo;
  p->shard_hi = row_hi;
  p->n_split_slots = n_slots;
  p->n_short = (int64_t)shrt.size();
  p->n_simt = (int64_t)simt.size();
  // longest first: groups pull items dynamically, so LPT order keeps the tail short
  for (int c = 0; c < SKINNY_CLASSES; ++c)
    std::stable_sort(skinny[c].begin(), skinny[c].end(),
                     [](const SkinnyItem& x, const SkinnyItem& y) { return x.be - x.bb > y.be - y.bb; });
  for (int c = 0; c < SKINNY_CLASSES; ++c) p->skinny_off[c + 1] = p->skinny_off[c] + (int64_t)skinny[c].size();
  if (p->skinny_off[SKINNY_CLASSES] > 0) {
    std::vector<SkinnyItem> all;
    all.reserve(p->skinny_off[SKINNY_CLASSES]);
    for (int c = 0; c < SKINNY_CLASSES; ++c) all.insert(all.end(), skinny[c].begin(), skinny[c].end());
    cudaError_t e = cudaMalloc(&p->d_skinny, sizeof(SkinnyItem) * all.size());
    if (e == cudaSuccess) e = cudaMalloc(&p->d_sched, sizeof(unsigned long long) * 2 * SKINNY_CLASSES);
    if (e == cudaSuccess) e = cudaMemsetAsync(p->d_sched, 0, sizeof(unsigned long long) * 2 * SKINNY_CLASSES, stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(p->d_skinny, all.data(), sizeof(SkinnyItem) * all.size(), cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
      rb_spmm_plan_destroy(p);
      return fail(e == cudaErrorMemoryAllocation ? RB_ENOMEM : RB_ECUDA, "skinny work list");
    }
  }
  if (!cmp_items.empty()) {  // longest first (items are pulled dynamically)
    std::stable_sort(cmp_items.begin(), cmp_items.end(),
                     [](const SkinnyItem& x, const SkinnyItem& y) { return x.be - x.bb > y.be - y.bb; });
    p->n_cmp_items = (int64_t)cmp_items.size();
    p->cmp_chunk = csr_claim_chunk(cmp_items);
    cudaError_t e = cudaMalloc(&p->d_cmp_items, sizeof(SkinnyItem) * cmp_items.size());
    if (e == cudaSuccess) e = cudaMalloc(&p->d_cmp_sched, 2 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemsetAsync(p->d_cmp_sched, 0, 2 * sizeof(unsigned long long), stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(p->d_cmp_items, cmp_items.data(), sizeof(SkinnyItem) * cmp_items.size(),
                          cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
      rb_spmm_plan_destroy(p);
      return fail(e == cudaErrorMemoryAllocation ? RB_ENOMEM : RB_ECUDA, "compact work list");
    }
  }
  if (sk_slots > 0) {  // split-row partials and arrival counters (skinny and compact items)
    cudaError_t e = cudaMalloc(&p->d_skinny_ws, sizeof(float) * 128 * (size_t)sk_units);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_skinny_cnt, sizeof(int32_t) * (size_t)sk_slots);
    if (e == cudaSuccess) e = cudaMemsetAsync(p->d_skinny_cnt, 0, sizeof(int32_t) * sk_slots, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
      rb_spmm_plan_destroy(p);
      return fail(e == cudaErrorMemoryAllocation ? RB_ENOMEM : RB_ECUDA, "split-row workspace");
    }
  }
  const int64_t n_items = 2 * p->n_tall + p->n_short + p->n_simt;
  if (n_slots > 0) {
    cudaError_t e = cudaMalloc(&p->d_ws, sizeof(float) * (size_t)n_slots * MAX_SPLIT * 8 * WARP_PART);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_cnt, sizeof(int32_t) * 8 * n_slots);
    if (e == cudaSuccess) e = cudaMemsetAsync(p->d_cnt, 0, sizeof(int32_t) * 8 * n_slots, stream);
    if (e != cudaSuccess) {
      rb_spmm_plan_destroy(p);
      return fail(RB_ENOMEM, "cudaMalloc split-K workspace");
    }
  }
  if (n_items > 0) {
    cudaError_t e = cudaMalloc(&p->d_items, sizeof(int4) * n_items);
    if (e != cudaSuccess) {
      rb_spmm_plan_destroy(p);
      return fail(RB_ENOMEM, "cudaMalloc work list");
    }
    std::vector<int4> all;
    all.reserve(n_items);
    all.insert(all.end(), tall_units.begin(), tall_units.end());
    all.insert(all.end(), shrt.begin(), shrt.end());
    all.insert(all.end(), simt.begin(), simt.end());
    e = cudaMemcpyAsync(p->d_items, all.data(), sizeof(int4) * n_items, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
      rb_spmm_plan_destroy(p);
      return fail(RB_ECUDA, cudaGetErrorString(e));
    }
  }
  if (tc && vbr->n_blocks > 0) {
    if (!vbr->tiles || vbr->total_tile_rows <= 0) {
      rb_spmm_plan_destroy(p);
      return fail(RB_EINVAL, "tiles missing");
    }
    const CUtensorMapDataType dt = b_dtype == RB_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    const uint64_t rows = (uint64_t)vbr->total_tile_rows, rb = (uint64_t)vbr->dp * 2;
    int rc = make_tmap_2d(&p->tmA16, vbr->tiles, dt, vbr->dp, rows, rb, 64, 16);
    if (!rc) rc = make_tmap_2d(&p->tmA32, vbr->tiles, dt, vbr->dp, rows, rb, 64, 32);
    if (!rc) rc = make_tmap_2d(&p->tmA64, vbr->tiles, dt, vbr->dp, rows, rb, 64, 64);
    if (!rc) rc = make_tmap_2d(&p->tmA128, vbr->tiles, dt, vbr->dp, rows, rb, 64, 128);
    if (rc) {
      rb_spmm_plan_destroy(p);
      return rc;
    }
  }
  if (short_ctas > 0) {
    p->short_ctas = short_ctas;
    cudaError_t e = cudaMalloc(&p->d_short_ptr, sizeof(int32_t) * short_ptr.size());
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(p->d_short_ptr, short_ptr.data(), sizeof(int32_t) * short_ptr.size(),
                          cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
      rb_spmm_plan_destroy(p);
      return fail(e == cudaErrorMemoryAllocation ? RB_ENOMEM : RB_ECUDA, "short schedule");
    }
  }
  if (!zero_rows.empty()) {
    p->n_zero = (int64_t)zero_rows.size();
    cudaError_t e = cudaMalloc(&p->d_zero, sizeof(int32_t) * zero_rows.size());
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(p->d_zero, zero_rows.data(), sizeof(int32_t) * zero_rows.size(), cudaMemcpyHostToDevice,
                          stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
      rb_spmm_plan_destroy(p);
      return fail(e == cudaErrorMemoryAllocation ? RB_ENOMEM : RB_ECUDA, "zero-row list");
    }
  }
  if (!sw_rows.empty()) {
    std::vector<int32_t> bcol(vbr->n_blocks), cb(vbr->n_seg + 1);
    std::vector<int64_t> trow(H);
    cudaError_t e = cudaMemcpyAsync(bcol.data(), vbr->blk_col, sizeof(int32_t) * vbr->n_blocks, cudaMemcpyDeviceToHost,
                                    stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(trow.data(), vbr->grp_tile_row, sizeof(int64_t) * H, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(cb.data(), vbr->col_bounds, sizeof(int32_t) * (vbr->n_seg + 1), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
      rb_spmm_plan_destroy(p);
      return fail(RB_ECUDA, cudaGetErrorString(e));
    }
    std::vector<int32_t> slabs;
    for (int64_t n0 = 0; n0 < N; n0 += short_ns) slabs.push_back((int32_t)n0);
    int dev_ = 0, sms_ = kNumSMs;
    RB_CUDA_TRY(cudaGetDevice(&dev_));
    RB_CUDA_TRY(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev_));
    // slot reuse delay: the epilogue copies a finished slot to registers (~400 cycles) and hands it
    // back before storing C, so a short delay suffices (config 5: 4 -> 2.32 ms, 8 -> 2.35, 32 -> 2.67)
    int delay = 4;
    if (const char* d = std::getenv("RB_SWEEP_DELAY")) delay = std::max(0, std::atoi(d));
    const int ctas = (int)std::min<int64_t>(sms_, (int64_t)sw_rows.size() * (int64_t)slabs.size());
    std::vector<int4> steps, done;
    std::vector<int32_t> step_ptr, done_ptr;
    sweep_schedule(sw_rows, slabs, rp, bp, bcol, trow, cb, vbr->n_seg, ctas, sw_slots, delay, dpc, steps, step_ptr, done,
                   done_ptr);
    e = cudaMalloc(&p->d_sw_steps, sizeof(int4) * steps.size());
    if (e == cudaSuccess) e = cudaMalloc(&p->d_sw_done, sizeof(int4) * done.size());
    if (e == cudaSuccess) e = cudaMalloc(&p->d_sw_step_ptr, sizeof(int32_t) * step_ptr.size());
    if (e == cudaSuccess) e = cudaMalloc(&p->d_sw_done_ptr, sizeof(int32_t) * done_ptr.size());
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(p->d_sw_steps, steps.data(), sizeof(int4) * steps.size(), cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(p->d_sw_done, done.data(), sizeof(int4) * done.size(), cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(p->d_sw_step_ptr, step_ptr.data(), sizeof(int32_t) * step_ptr.size(), cudaMemcpyHostToDevice,
                          stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(p->d_sw_done_ptr, done_ptr.data(), sizeof(int32_t) * done_ptr.size(), cudaMemcpyHostToDevice,
                          stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
      rb_spmm_plan_destroy(p);
      return fail(e == cudaErrorMemoryAllocation ? RB_ENOMEM : RB_ECUDA, "sweep schedule");
    }
    p->sw_hp = sw_hp;
    p->sw_slots = sw_slots;
    p->sw_ctas = ctas;
    p->n_sw_steps = (int64_t)steps.size();
  }
  p->info.n_items_tall = p->n_tall;
  p->info.n_items_short = p->n_short + p->n_sw_steps;
  p->info.n_sweep_steps = p->n_sw_steps;
  p->info.sweep_slots = p->sw_slots;
  p->info.n_items_simt = p->n_simt;
  p->info.n_items_skinny = p->skinny_off[SKINNY_CLASSES] + p->n_cmp_items;
  p->info.core_vbr_flops = core_vbr_flops;
  p->info.n_launches = (p->n_tall > 0) + (p->n_short > 0) + (p->n_simt > 0) + (p->n_zero > 0) + (p->n_sw_steps > 0) +
                       (p->n_cmp_items > 0);
  for (int c = 0; c < SKINNY_CLASSES; ++c) p->info.n_launches += p->skinny_off[c + 1] > p->skinny_off[c];
  p->info.executed_flops = exec_flops;
  p->info.vbr_flops = vbr_flops;
  p->info.row_begin_perm = row_lo < row_hi ? row_lo : -1;
  *out = p;
  return RB_OK;
}

// Switch the plan's tall block rows to the 2:4 sparse tensor-core kernel over the compressed form
// built by rb_sparse24_emit, plus the residual pass (C += residuals x B) for the groups that keep
// more than two nonzeros.  Work units are re-planned in stages of 128 logical K.
extern "C" int rb_spmm_plan_attach_sparse24(rb_spmm_plan* p, const rb_sparse24_device* sp, void* stream_) {
  if (!p || !sp) return fail(RB_EINVAL, "null argument");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (p->b_dtype != RB_BF16 && p->b_dtype != RB_F16) return fail(RB_EUNSUPPORTED, "2:4 path needs bf16/fp16");
  const int64_t H = p->v.n_block_rows, n = p->v.n_rows;
  std::vector<int32_t> rp(H + 1), bp(H + 1);
  std::vector<int64_t> spr(std::max<int64_t>(H, 1)), res(n + 1);
  if (H > 0) {
    RB_CUDA_TRY(cudaMemcpyAsync(rp.data(), p->v.row_partition, 4 * (H + 1), cudaMemcpyDeviceToHost, stream));
    RB_CUDA_TRY(cudaMemcpyAsync(bp.data(), p->v.blk_ptr, 4 * (H + 1), cudaMemcpyDeviceToHost, stream));
    RB_CUDA_TRY(cudaMemcpyAsync(spr.data(), sp->sp_tile_row, 8 * H, cudaMemcpyDeviceToHost, stream));
  }
  if (sp->n_residuals > 0)
    RB_CUDA_TRY(cudaMemcpyAsync(res.data(), sp->res_ptr, 8 * (n + 1), cudaMemcpyDeviceToHost, stream));
  RB_CUDA_TRY(cudaStreamSynchronize(stream));
  std::vector<int4> items;
  for (const int4& it : p->tall_items) {
    const int g = it.x;
    if (spr[g] < 0) return fail(RB_EINVAL, "sparse form does not cover a tall block row");
    const int64_t S = ((int64_t)(bp[g + 1] - bp[g]) * p->v.dp + 127) / 128;
    items.push_back(make_int4(g, it.y, it.z, (int)S));
  }
  std::stable_sort(items.begin(), items.end(), [](const int4& x, const int4& y) { return x.w > y.w; });
  int dev = 0, sms = kNumSMs;
  RB_CUDA_TRY(cudaGetDevice(&dev));
  RB_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  std::vector<int4> units;
  int64_t n_slots = 0;
  split_tail(items, sms / 2, units, n_slots);
  // residual rows of this shard's tall block rows
  const int cols = skinny_cols(p->b_dtype, p->N);
  std::vector<SkinnyItem> ritems;
  if (sp->n_residuals > 0)
    for (const int4& it : p->tall_items) {
      const int g = it.x;
      if (it.z != 0) continue;  // one pass per pair tile: rows m*256 .. +256
      for (int r = it.y * PAIR_BM; r < std::min(rp[g + 1] - rp[g], (it.y + 1) * PAIR_BM); ++r) {
        const int64_t pos = rp[g] + r;
        const int64_t c = res[pos + 1] - res[pos];
        if (c <= 0) continue;
        for (int64_t n0 = 0; n0 < p->N; n0 += cols)
          ritems.push_back(SkinnyItem{(int32_t)pos, (int32_t)n0, 0, (int32_t)c, 0, 1, -1, 0});
      }
    }
  cudaError_t e = cudaSuccess;
  if (p->d_sp_units) cudaFree(p->d_sp_units);
  p->d_sp_units = nullptr;
  if (!units.empty()) e = cudaMalloc(&p->d_sp_units, sizeof(int4) * units.size());
  if (e == cudaSuccess && !units.empty())
    e = cudaMemcpyAsync(p->d_sp_units, units.data(), sizeof(int4) * units.size(), cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess && n_slots > 0 && !p->d_sp_ws)
    e = cudaMalloc(&p->d_sp_ws, sizeof(float) * (size_t)n_slots * MAX_SPLIT * 8 * WARP_PART);
  if (e == cudaSuccess && n_slots > 0 && !p->d_sp_cnt) e = cudaMalloc(&p->d_sp_cnt, sizeof(int32_t) * 8 * n_slots);
  if (e == cudaSuccess && n_slots > 0) e = cudaMemsetAsync(p->d_sp_cnt, 0, sizeof(int32_t) * 8 * n_slots, stream);
  if (e == cudaSuccess && !ritems.empty()) e = cudaMalloc(&p->d_res_items, sizeof(SkinnyItem) * ritems.size());
  if (e == cudaSuccess && !ritems.empty())
    e = cudaMemcpyAsync(p->d_res_items, ritems.data(), sizeof(SkinnyItem) * ritems.size(), cudaMemcpyHostToDevice,
                        stream);
  if (e == cudaSuccess && !p->d_res_sched) e = cudaMalloc(&p->d_res_sched, 2 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemsetAsync(p->d_res_sched, 0, 2 * sizeof(unsigned long long), stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return fail(e == cudaErrorMemoryAllocation ? RB_ENOMEM : RB_ECUDA, cudaGetErrorString(e));
  if (sp->total_sp_rows > 0) {
    const CUtensorMapDataType dt =
        p->b_dtype == RB_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    int rc = make_tmap_2d(&p->tmSP, sp->sp_tiles, dt, 64, (uint64_t)sp->total_sp_rows, 128, 64, 128);
    if (!rc)
      rc = make_tmap_2d(&p->tmSPE, sp->sp_meta, CU_TENSOR_MAP_DATA_TYPE_UINT32, 8, (uint64_t)sp->total_sp_rows, 32, 4,
                        128, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
  }
  p->sp = *sp;
  p->n_sp_units = (int64_t)units.size() / 2;
  p->n_res_items = (int64_t)ritems.size();
  p->use_sp = true;
  p->info.n_launches = (p->n_tall > 0) + (p->n_short > 0) + (p->n_simt > 0) + (p->n_zero > 0) +
                       (p->n_res_items > 0) + (p->n_sw_steps > 0) + (p->n_cmp_items > 0);
  for (int c = 0; c < SKINNY_CLASSES; ++c) p->info.n_launches += p->skinny_off[c + 1] > p->skinny_off[c];
  return RB_OK;
}

extern "C" int rb_spmm_plan_info(const rb_spmm_plan* p, rb_spmm_info* info) {
  if (!p || !info) return fail(RB_EINVAL, "null argument");
  *info = p->info;
  return RB_OK;
}

extern "C" int rb_spmm_plan_destroy(rb_spmm_plan* p) {
  if (!p) return RB_OK;
  if (p->d_items) cudaFree(p->d_items);
  if (p->d_ws) cudaFree(p->d_ws);
  if (p->d_cnt) cudaFree(p->d_cnt);
  if (p->d_skinny) cudaFree(p->d_skinny);
  if (p->d_skinny_ws) cudaFree(p->d_skinny_ws);
  if (p->d_skinny_cnt) cudaFree(p->d_skinny_cnt);
  if (p->d_sched) cudaFree(p->d_sched);
  if (p->d_zero) cudaFree(p->d_zero);
  if (p->d_short_ptr) cudaFree(p->d_short_ptr);
  if (p->d_sw_steps) cudaFree(p->d_sw_steps);
  if (p->d_cmp_items) cudaFree(p->d_cmp_items);
  if (p->d_cmp_sched) cudaFree(p->d_cmp_sched);
  if (p->d_sw_done) cudaFree(p->d_sw_done);
  if (p->d_sw_step_ptr) cudaFree(p->d_sw_step_ptr);
  if (p->d_sw_done_ptr) cudaFree(p->d_sw_done_ptr);
  if (p->d_sp_units) cudaFree(p->d_sp_units);
  if (p->d_sp_ws) cudaFree(p->d_sp_ws);
  if (p->d_sp_cnt) cudaFree(p->d_sp_cnt);
  if (p->d_res_items) cudaFree(p->d_res_items);
  if (p->d_res_sched) cudaFree(p->d_res_sched);
  if (p->aux_ready) {
    for (int l = 0; l < kAuxStreams; ++l) cudaStreamDestroy(p->aux[l]);
    for (int l = 0; l <= kAuxStreams; ++l) cudaEventDestroy(p->ev[l]);
  }
  if (p->done) cudaEventDestroy(p->done);
  delete p;
  return RB_OK;
}

// Kernel attributes are per device: set them once per device ordinal (thread-safe).
static int ensure_kernel_attributes() {
  static std::mutex m;
  static bool done[64] = {};
  int dev = 0;
  RB_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(m);
  if (dev >= 0 && dev < 64 && done[dev]) return RB_OK;
  RB_CUDA_TRY(cudaFuncSetAttribute(spmm_tall2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TALL));
  RB_CUDA_TRY(cudaFuncSetAttribute(spmm_short2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_SHORT));
  RB_CUDA_TRY(cudaFuncSetAttribute(spmm_tall2_sp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_SP));
  RB_CUDA_TRY(cudaFuncSetAttribute(spmm_sweep_kernel<SW_STAGES_BIG, SW_ASLOT_BIG, false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, sweep_smem(SW_STAGES_BIG, SW_ASLOT_BIG)));
  RB_CUDA_TRY(cudaFuncSetAttribute(spmm_sweep_kernel<SW_STAGES_BIG, SW_ASLOT_BIG, false, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   sweep64_smem(SW_STAGES_BIG, SW_ASLOT_BIG)));
  RB_CUDA_TRY(cudaFuncSetAttribute(spmm_sweep_kernel<SW_STAGES_SMALL, SW_ASLOT_SMALL, false, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   sweep64_smem(SW_STAGES_SMALL, SW_ASLOT_SMALL)));
  RB_CUDA_TRY(cudaFuncSetAttribute(spmm_sweep_kernel<SW_STAGES_BIG, SW_ASLOT_BIG, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, sweep_smem(SW_STAGES_BIG, SW_ASLOT_BIG)));
  RB_CUDA_TRY(cudaFuncSetAttribute(spmm_sweep_kernel<SW_STAGES_SMALL, SW_ASLOT_SMALL, false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   sweep_smem(SW_STAGES_SMALL, SW_ASLOT_SMALL)));
  if (dev >= 0 && dev < 64) done[dev] = true;
  return RB_OK;
}

static int spmm_execute_locked(const rb_spmm_plan* p, const void* B, int64_t ldb, float* C, int64_t ldc,
                               cudaStream_t stream, const CFan& fan, const int32_t* c_rows);

static int spmm_execute_entry(const rb_spmm_plan* p, const void* B, int64_t ldb, float* C, int64_t ldc,
                              void* stream_, const CFan* fan = nullptr, const int32_t* c_rows = nullptr);

extern "C" int rb_spmm_execute(const rb_spmm_plan* p, const void* B, int64_t ldb, float* C, int64_t ldc,
                               void* stream_) {
  rb::NvtxRange nvtx_range_("rb_spmm_execute");
  if (p && p->b_dtype == RB_F64) return fail(RB_EINVAL, "fp64 plan: use rb_spmm_execute_f64");
  return spmm_execute_entry(p, B, ldb, C, ldc, stream_);
}

extern "C" int rb_spmm_execute_f64(const rb_spmm_plan* p, const double* B, int64_t ldb, double* C, int64_t ldc,
                                   void* stream_) {
  rb::NvtxRange nvtx_range_("rb_spmm_execute_f64");
  if (p && p->b_dtype != RB_F64) return fail(RB_EINVAL, "rb_spmm_execute_f64 needs a plan made for RB_F64");
  return spmm_execute_entry(p, B, ldb, reinterpret_cast<float*>(C), ldc, stream_);
}

extern "C" int rb_spmm_execute_fanout(const rb_spmm_plan* p, const void* B, int64_t ldb, float* C, int64_t ldc,
                                      float* const* peers, int32_t n_peers, const int32_t* c_rows, void* stream_) {
  rb::NvtxRange nvtx_range_("rb_spmm_execute_fanout");
  if (!p) return fail(RB_EINVAL, "null plan");
  if (p->b_dtype == RB_F64) return fail(RB_EINVAL, "fan-out needs a float32-C plan (not RB_F64)");
  if (n_peers < 0 || n_peers > RB_MAX_FAN) return fail(RB_EINVAL, "n_peers must be in [0, 7]");
  if (n_peers > 0 && !peers) return fail(RB_EINVAL, "null peers");
  CFan fan{};
  fan.n = n_peers;
  for (int i = 0; i < n_peers; ++i) {
    if (!peers[i] && p->v.n_rows > 0) return fail(RB_EINVAL, "null peer buffer");
    if ((reinterpret_cast<uintptr_t>(peers[i]) & 15) || (reinterpret_cast<uintptr_t>(C) & 15) || (ldc & 3))
      return fail(RB_EINVAL, "fan-out buffers must be 16-byte aligned (ldc a multiple of 4)");
    fan.p[i] = peers[i];
  }
  return spmm_execute_entry(p, B, ldb, C, ldc, stream_, &fan, c_rows);
}

static int spmm_execute_entry(const rb_spmm_plan* p, const void* B, int64_t ldb, float* C, int64_t ldc,
                              void* stream_, const CFan* fan, const int32_t* c_rows) {
  if (!p) return fail(RB_EINVAL, "null plan");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  std::lock_guard<std::mutex> lk(p->mu);
  if (!p->done) RB_CUDA_TRY(cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming));
  if (p->done_valid && p->done_stream != stream) RB_CUDA_TRY(cudaStreamWaitEvent(stream, p->done, 0));
  static const CFan no_fan{};
  const int rc = spmm_execute_locked(p, B, ldb, C, ldc, stream, fan ? *fan : no_fan, c_rows);
  if (rc) return rc;
  RB_CUDA_TRY(cudaEventRecord(p->done, stream));
  p->done_stream = stream;
  p->done_valid = true;
  return RB_OK;
}

static int spmm_execute_locked(const rb_spmm_plan* p, const void* B, int64_t ldb, float* C, int64_t ldc,
                               cudaStream_t stream, const CFan& fan, const int32_t* c_rows) {
  // output row of permuted row p: the plan's row_perm, or the caller's map (fan-out shards)
  const int32_t* out_rows = c_rows ? c_rows : p->v.row_perm;
  if (ldc < p->N || ldb < p->N) return fail(RB_EINVAL, "leading dimension smaller than N");
  if (!C && p->v.n_rows > 0) return fail(RB_EINVAL, "null C");
  SpmmArgs a;
  a.row_partition = p->v.row_partition;
  a.row_perm = out_rows;
  a.blk_ptr = p->v.blk_ptr;
  a.blk_col = p->v.blk_col;
  a.grp_tile_row = p->v.grp_tile_row;
  a.col_bounds = p->v.col_bounds;
  a.dp_chunks = p->v.dp / KCH;
  a.C = C;
  a.ldc = ldc;
  a.N = (int32_t)p->N;
  a.ab_fmt = p->b_dtype == RB_BF16 ? 1u : 0u;
  a.a_evict_first = 0;
  a.b_policy = 0;
  a.c_evict_first = 0;
  a.cta_ptr = nullptr;
  a.short_ns = p->short_ns;
  a.ws = p->d_ws;
  a.cnt = p->d_cnt;
  a.sp_meta = nullptr;
  a.sp_tile_row = nullptr;
  a.fan = fan;
  // Independent launches (disjoint C rows): zero rows, each skinny height class, the fp32 SIMT
  // kernel, the tall and the short tensor-core kernels.  With more than one, they are forked over
  // the caller's stream and up to three auxiliary streams and joined back (small latency-bound
  // classes overlap the large kernels instead of queueing behind them).
  std::vector<std::function<int(cudaStream_t)>> tasks;
  if (p->n_zero > 0)
    tasks.push_back([&](cudaStream_t st) {
      const unsigned grid = (unsigned)std::min<int64_t>((p->n_zero + 255) / 256, 148 * 16);  // 8 warps x 32 rows
      // fp64 C: a row of N doubles is 2N zero floats
      const int w = p->b_dtype == RB_F64 ? 2 : 1;
      zero_rows_kernel<<<grid, 256, 0, st>>>(p->d_zero, p->n_zero, out_rows, C, ldc * w, (int32_t)p->N * w, fan);
      RB_CUDA_TRY(cudaGetLastError());
      return RB_OK;
    });
  SkinnyArgs k{};
  k.row_partition = p->v.row_partition;
  k.row_perm = out_rows;
  k.blk_ptr = p->v.blk_ptr;
  k.blk_col = p->v.blk_col;
  k.grp_tile_row = p->v.grp_tile_row;
  k.col_bounds = p->v.col_bounds;
  k.tiles = p->v.tiles;
  k.dp = p->v.dp;
  k.B = B;
  k.ldb = ldb;
  k.C = C;
  k.ldc = ldc;
  k.N = (int32_t)p->N;
  k.ws = p->d_skinny_ws;
  k.cnt = p->d_skinny_cnt;
  k.fan = fan;
  for (int c = 0; c < SKINNY_CLASSES; ++c) {
    if (p->skinny_off[c + 1] == p->skinny_off[c]) continue;
    tasks.push_back([&, c](cudaStream_t st) {
      SkinnyArgs kc = k;
      kc.items = p->d_skinny + p->skinny_off[c];
      kc.n_items = p->skinny_off[c + 1] - p->skinny_off[c];
      return launch_skinny(kc, p->b_dtype, c, p->d_sched + 2 * c, st);
    });
  }
  if (p->n_cmp_items > 0)
    tasks.push_back([&](cudaStream_t st) {
      SkinnyArgs kc = k;
      kc.items = p->d_cmp_items;
      kc.n_items = p->n_cmp_items;
      const CsrArgs cr{p->v.cmp_ptr, nullptr, nullptr, p->v.cmp_col, p->v.cmp_val, p->cmp_chunk};
      return launch_csr(kc, cr, p->b_dtype, p->d_cmp_sched, st);
    });
  if ((p->b_dtype == RB_F32 || p->b_dtype == RB_F64) && p->n_simt > 0)
    tasks.push_back([&](cudaStream_t st) {
      SpmmArgs s = a;
      s.items = p->d_items + 2 * p->n_tall + p->n_short;
      s.n_items = (int32_t)p->n_simt;
      s.dp_chunks = 1;
      if (p->b_dtype == RB_F64)
        spmm_simt_kernel<double><<<(unsigned)p->n_simt, SIMT_COLS, 0, st>>>(
            s, static_cast<const double*>(p->v.tiles), p->v.dp, static_cast<const double*>(B), ldb,
            reinterpret_cast<double*>(C));
      else
        spmm_simt_kernel<float><<<(unsigned)p->n_simt, SIMT_COLS, 0, st>>>(
            s, static_cast<const float*>(p->v.tiles), p->v.dp, static_cast<const float*>(B), ldb, C);
      RB_CUDA_TRY(cudaGetLastError());
      return RB_OK;
    });
  CUtensorMap tmB;
  memset(&tmB, 0, sizeof(tmB));
  int sms = kNumSMs;
  const bool tc = p->b_dtype == RB_BF16 || p->b_dtype == RB_F16;
  if (tc && (p->n_tall > 0 || p->n_short > 0 || p->n_sw_steps > 0)) {
    if (int rc = ensure_kernel_attributes()) return rc;
    const CUtensorMapDataType dt =
        p->b_dtype == RB_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    int rc = make_tmap_2d(&tmB, B, dt, (uint64_t)p->N, (uint64_t)p->v.n_cols, (uint64_t)ldb * 2, 64, 64);
    if (rc) return rc;
    int dev = 0;
    RB_CUDA_TRY(cudaGetDevice(&dev));
    RB_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  if (tc && p->n_tall > 0)
    tasks.push_back([&](cudaStream_t st) {
      if (p->use_sp) {
        SpmmArgs s = a;
        s.items = p->d_sp_units;
        s.n_items = (int32_t)p->n_sp_units;
        s.ws = p->d_sp_ws;
        s.cnt = p->d_sp_cnt;
        s.sp_meta = p->sp.sp_meta;
        s.sp_tile_row = p->sp.sp_tile_row;
        const int pairs = (int)std::min<int64_t>(sms / 2, p->n_sp_units);
        if (pairs > 0) {
          spmm_tall2_sp_kernel<<<(unsigned)(2 * pairs), SP_THREADS, SMEM_SP, st>>>(p->tmSP, tmB, p->tmSPE, s);
          RB_CUDA_TRY(cudaGetLastError());
        }
        if (p->n_res_items > 0) {  // C += residuals x B (groups of 4 with more than two nonzeros), same stream
          SkinnyArgs kr{};
          kr.row_perm = out_rows;
          kr.fan = fan;
          kr.items = p->d_res_items;
          kr.n_items = p->n_res_items;
          kr.B = B;
          kr.ldb = ldb;
          kr.C = C;
          kr.ldc = ldc;
          kr.N = (int32_t)p->N;
          kr.accumulate = 1;
          CsrArgs cr{p->sp.res_ptr, nullptr, nullptr, p->sp.res_col, p->sp.res_val, 1};
          return launch_csr(kr, cr, p->b_dtype, p->d_res_sched, st);
        }
        return (int)RB_OK;
      }
      SpmmArgs s = a;
      s.items = p->d_items;
      s.n_items = (int32_t)p->n_tall;
      const int pairs = (int)std::min<int64_t>(sms / 2, p->n_tall);
      spmm_tall2_kernel<<<(unsigned)(2 * pairs), TC_THREADS, SMEM_TALL, st>>>(p->tmA128, tmB, s);
      RB_CUDA_TRY(cudaGetLastError());
      return (int)RB_OK;
    });
  if (tc && p->n_short > 0)
    tasks.push_back([&](cudaStream_t st) {
      SpmmArgs s = a;
      s.items = p->d_items + 2 * p->n_tall;
      s.n_items = (int32_t)p->n_short;
      s.a_evict_first = 1;
      if (const char* e = std::getenv("RB_SHORT_CACHE")) {  // experiment knob: "<a><b><c>" digits
        if (e[0]) s.a_evict_first = e[0] == '1';
        if (e[0] && e[1]) s.b_policy = (uint32_t)(e[1] - '0') % 3;
        if (e[0] && e[1] && e[2]) s.c_evict_first = e[2] == '1';
      }
      s.cta_ptr = p->d_short_ptr;
      const int ctas = p->short_ctas;
      spmm_short2_kernel<<<(unsigned)ctas, TC_THREADS, SMEM_SHORT, st>>>(p->tmA16, p->tmA32, p->tmA64, p->tmA128,
                                                                        tmB, s);
      RB_CUDA_TRY(cudaGetLastError());
      return (int)RB_OK;
    });
  if (tc && p->n_sw_steps > 0)
    tasks.push_back([&](cudaStream_t st) {
      SpmmArgs s = a;
      SweepArgs w{p->d_sw_steps, p->d_sw_step_ptr, p->d_sw_done, p->d_sw_done_ptr, p->sw_hp};
      const CUtensorMap& tA = p->sw_hp == 16 ? p->tmA16 : p->sw_hp == 32 ? p->tmA32 : p->sw_hp == 64 ? p->tmA64 : p->tmA128;
      // 4 x 48 KB measured 2.26 ms against 2.30 ms for 5 x 40 KB on config 5 (3 runs each): the
      // ring is not the limit, so the 4-stage layout is the default (RB_SWEEP_BIG=0: the 5-stage one)
      static const bool big_env = [] {
        const char* e = std::getenv("RB_SWEEP_BIG");
        return !(e && e[0] == '0');
      }();
      static const bool pair_env = [] {
        const char* e = std::getenv("RB_SWEEP_PAIR");
        return e && e[0] == '1';
      }();
      static const bool m64_env = [] {
        const char* e = std::getenv("RB_SWEEP_M64");
        return !(e && e[0] == '0');
      }();
      if (p->sw_hp == 64 && m64_env && !big_env)  // RB_SWEEP_BIG=0: the 5 x 40 KB ring
        spmm_sweep_kernel<SW_STAGES_SMALL, SW_ASLOT_SMALL, false, true>
            <<<(unsigned)p->sw_ctas, SW64_THREADS, sweep64_smem(SW_STAGES_SMALL, SW_ASLOT_SMALL), st>>>(tA, tmB, s, w);
      else if (p->sw_hp == 64 && m64_env)
        spmm_sweep_kernel<SW_STAGES_BIG, SW_ASLOT_BIG, false, true>
            <<<(unsigned)p->sw_ctas, SW64_THREADS, sweep64_smem(SW_STAGES_BIG, SW_ASLOT_BIG), st>>>(tA, tmB, s, w);
      else if (pair_env)
        spmm_sweep_kernel<SW_STAGES_BIG, SW_ASLOT_BIG, true>
            <<<(unsigned)p->sw_ctas, SW_THREADS, sweep_smem(SW_STAGES_BIG, SW_ASLOT_BIG), st>>>(tA, tmB, s, w);
      else if (p->sw_hp > 64 || big_env)
        spmm_sweep_kernel<SW_STAGES_BIG, SW_ASLOT_BIG, false>
            <<<(unsigned)p->sw_ctas, SW_THREADS, sweep_smem(SW_STAGES_BIG, SW_ASLOT_BIG), st>>>(tA, tmB, s, w);
      else
        spmm_sweep_kernel<SW_STAGES_SMALL, SW_ASLOT_SMALL, false>
            <<<(unsigned)p->sw_ctas, SW_THREADS, sweep_smem(SW_STAGES_SMALL, SW_ASLOT_SMALL), st>>>(tA, tmB, s, w);
      RB_CUDA_TRY(cudaGetLastError());
      return (int)RB_OK;
    });
  if (tasks.size() <= 1) return tasks.empty() ? (int)RB_OK : tasks[0](stream);
  // fork / join over auxiliary streams (created once per plan); the largest task stays on `stream`
  if (!p->aux_ready) {
    for (int l = 0; l < kAuxStreams; ++l) RB_CUDA_TRY(cudaStreamCreateWithFlags(&p->aux[l], cudaStreamNonBlocking));
    for (int l = 0; l <= kAuxStreams; ++l) RB_CUDA_TRY(cudaEventCreateWithFlags(&p->ev[l], cudaEventDisableTiming));
    p->aux_ready = true;
  }
  RB_CUDA_TRY(cudaEventRecord(p->ev[kAuxStreams], stream));
  const int lanes = (int)std::min<size_t>(tasks.size(), kAuxStreams + 1);
  for (int l = 1; l < lanes; ++l) RB_CUDA_TRY(cudaStreamWaitEvent(p->aux[l - 1], p->ev[kAuxStreams], 0));
  for (size_t i = 0; i < tasks.size(); ++i) {
    const int l = (int)(i % lanes);
    int rc = tasks[i](l == 0 ? stream : p->aux[l - 1]);
    if (rc) return rc;
  }
  for (int l = 1; l < lanes; ++l) {
    RB_CUDA_TRY(cudaEventRecord(p->ev[l - 1], p->aux[l - 1]));
    RB_CUDA_TRY(cudaStreamWaitEvent(stream, p->ev[l - 1], 0));
  }
  return RB_OK;
}
