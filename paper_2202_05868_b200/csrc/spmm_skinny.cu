// Skinny block rows (h <= 8) of the VBR SpMM on the CUDA cores (replaces spmm_vbr's per-block
// `data @ B[bounds]` for the block rows where a tensor-core tile would be >= 94 % padding,
// multiply.py:84-89).
//
// 1-SA leaves most rows of sparse inputs (configs 1, 2b, 3) in block rows of one or two rows: an
// MMA tile of 16 x 64 would then multiply >= 15 padding rows and every zero column of the tile,
// and fetch the whole 64-row B panel per block.  Here a lane group (32 lanes, or 16 when N <= 128)
// owns one block row (or one part of a long one) and a slab of C columns (16-byte B loads per
// lane), reads the stored tiles and gathers only the B rows of tile columns that hold a nonzero.
// Groups pull items from a self-resetting work counter (persistent grid), items are ordered
// longest first, and block rows with > 256 stored blocks are cut into parts whose partials are
// summed in part order by the last-arriving part.
//
// Accumulation order per C element is fixed — blocks ascending, k ascending (parts in order) — so
// C is deterministic, and on the fp32 path identical to the dense-tile order (skipped terms are
// exact zeros: fma(0, b, acc) == acc for finite b).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "spmm_skinny.cuh"

namespace rb {
namespace {

template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}
template <>
__device__ __forceinline__ float to_f<__half>(__half x) {
  return __half2float(x);
}
template <>
__device__ __forceinline__ float to_f<float>(float x) {
  return x;
}

// 16 bytes of one B row (VEC = 16 / sizeof(T) elements from column n), kept raw until the FMA so
// eight gathers in flight cost 32 registers.  Columns >= N read as 0.
template <typename T, bool ALIGNED>
__device__ __forceinline__ uint4 load_b_raw(const T* p, int n, int N) {
  constexpr int VEC = 16 / sizeof(T);
  if (ALIGNED && n + VEC <= N) return __ldg(reinterpret_cast<const uint4*>(p));
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (n + e < N) w[e] = __float_as_uint(__ldg(reinterpret_cast<const float*>(p) + e));
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (n + e < N) w[e >> 1] |= (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(p) + e) << (16 * (e & 1));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// float64 -> operand dtype (round to nearest even, as the VBR tile emission does) -> float
template <typename T>
__device__ __forceinline__ float round_to(double v);
template <>
__device__ __forceinline__ float round_to<__nv_bfloat16>(double v) {
  return __bfloat162float(__double2bfloat16(v));
}
template <>
__device__ __forceinline__ float round_to<__half>(double v) {
  return __half2float(__double2half(v));
}
template <>
__device__ __forceinline__ float round_to<float>(double v) {
  return (float)v;
}

template <typename T>
__device__ __forceinline__ float elem(const uint4& u, int e) {
  if constexpr (sizeof(T) == 4) {
    return __uint_as_float(e == 0 ? u.x : e == 1 ? u.y : e == 2 ? u.z : u.w);
  } else {
    const uint32_t x = (e >> 1) == 0 ? u.x : (e >> 1) == 1 ? u.y : (e >> 1) == 2 ? u.z : u.w;
    const uint16_t b = (uint16_t)((e & 1) ? (x >> 16) : (x & 0xffffu));
    T t;
    memcpy(&t, &b, 2);
    return to_f(t);
  }
}

template <typename T>
__device__ __forceinline__ void fma_row(float (&acc)[16 / sizeof(T)], float a, const uint4& u) {
#pragma unroll
  for (int e = 0; e < (int)(16 / sizeof(T)); ++e) acc[e] = __fmaf_rn(a, elem<T>(u, e), acc[e]);
}

template <int VEC, bool ALIGNED>
__device__ __forceinline__ void store_c(float* dst, int n, int N, const float (&v)[VEC], bool accumulate = false) {
  if (ALIGNED && n + VEC <= N) {
#pragma unroll
    for (int e = 0; e < VEC; e += 4) {
      float4 o = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
      if (accumulate) {
        const float4 c = *reinterpret_cast<const float4*>(dst + e);
        o = make_float4(c.x + o.x, c.y + o.y, c.z + o.z, c.w + o.w);
      }
      *reinterpret_cast<float4*>(dst + e) = o;
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e)
      if (n + e < N) dst[e] = accumulate ? dst[e] + v[e] : v[e];
  }
}

// Epilogue shared by both kernels: direct store, or (split block row) park the partial and let the
// last-arriving part sum every part's partial in part order.
template <int H, int VEC, int LPR, bool ALIGNED>
__device__ __forceinline__ void skinny_finish(const SkinnyArgs& a, const SkinnyItem& it, int cols, int h, int p0,
                                              int n, int gl, unsigned gmask, float (&acc)[H][VEC]) {
  if (it.nparts > 1) {
    float* mine = a.ws + ((size_t)it.wsoff + (size_t)it.part * H * (cols / 128)) * 128;
#pragma unroll
    for (int r = 0; r < H; ++r)
#pragma unroll
      for (int e = 0; e < VEC; e += 4)
        __stcg(reinterpret_cast<float4*>(mine + r * cols + gl * VEC + e),
               make_float4(acc[r][e], acc[r][e + 1], acc[r][e + 2], acc[r][e + 3]));
    __threadfence();
    __syncwarp(gmask);
    int old = 0;
    if (gl == 0) old = atomicAdd(a.cnt + it.slot, 1);
    old = __shfl_sync(gmask, old, 0, LPR);
    if (old != it.nparts - 1) return;
    __threadfence();
    const float* base = a.ws + (size_t)it.wsoff * 128 + gl * VEC;
    const size_t pstride = (size_t)H * cols;
#pragma unroll
    for (int r = 0; r < H; ++r)
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[r][e] = 0.f;
#pragma unroll
    for (int r = 0; r < H; ++r) {
      for (int q = 0; q < it.nparts; q += 4) {  // four parts' loads in flight, summed in part order
        float4 v[4][VEC / 4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (q + u < it.nparts)
#pragma unroll
            for (int e = 0; e < VEC / 4; ++e)
              v[u][e] = __ldcg(reinterpret_cast<const float4*>(base + (q + u) * pstride + r * cols) + e);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (q + u < it.nparts)
#pragma unroll
            for (int e = 0; e < VEC / 4; ++e) {
              acc[r][4 * e] += v[u][e].x;
              acc[r][4 * e + 1] += v[u][e].y;
              acc[r][4 * e + 2] += v[u][e].z;
              acc[r][4 * e + 3] += v[u][e].w;
            }
      }
    }
    if (gl == 0) a.cnt[it.slot] = 0;  // ready for the next launch (stream ordered)
  }
  if (n >= a.N) return;
#pragma unroll
  for (int r = 0; r < H; ++r)
    if (r < h) {
      const int64_t crow = a.row_perm ? (int64_t)a.row_perm[p0 + r] : (int64_t)p0 + r;  // CSR: identity
      store_c<VEC, ALIGNED>(a.C + crow * a.ldc + n, n, a.N, acc[r], a.accumulate != 0);
      for (int f = 0; f < a.fan.n; ++f)  // fused all-gather: the same row into every peer's C
        store_c<VEC, ALIGNED>(a.fan.p[f] + crow * a.ldc + n, n, a.N, acc[r], a.accumulate != 0);
    }
}

__device__ __forceinline__ SkinnyItem load_item(const SkinnyItem* p) {
  const int4 x = __ldg(reinterpret_cast<const int4*>(p)), y = __ldg(reinterpret_cast<const int4*>(p) + 1);
  return SkinnyItem{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
}

// Persistent scheduling: lane 0 of a group pulls the next item index; every group overshoots the
// counter exactly once, and the last group to leave resets both counters for the next launch.
template <int LPR>
__device__ __forceinline__ int64_t next_item(unsigned long long* sched, int gl, unsigned gmask) {
  unsigned long long i = 0;
  if (gl == 0) i = atomicAdd(sched, 1ull);
  return (int64_t)__shfl_sync(gmask, i, 0, LPR);
}
template <int LPR>
__device__ __forceinline__ void leave(unsigned long long* sched, int gl, unsigned long long total_groups) {
  if (gl == 0) {
    __threadfence();
    if (atomicAdd(sched + 1, 1ull) == total_groups - 1) {
      sched[0] = 0ull;
      sched[1] = 0ull;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Staged kernel (tiles at most 64 columns wide, every height class), see staged_item below.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(pred ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// h = 1 class: B gathers in flight per lane and resident CTAs per SM (developer overrides)
#ifndef RB_SK1_DEPTH
#define RB_SK1_DEPTH 6
#endif
#ifndef RB_SK1_MINB
#define RB_SK1_MINB 5
#endif
constexpr int STAGED_WARPS = 4;  // 128-thread CTAs: 5 resident per SM (registers <= 102, 41 KB smem each)

template <typename T, int LPR>
struct SkinnySmem {
  static constexpr int KC = 64;                          // tile columns staged per block (dp <= 64)
  static constexpr int PPB = KC * (int)sizeof(T) / 16;   // 16-byte pieces per staged row
  static constexpr int ROW = KC * (int)sizeof(T) + 16;   // padded row stride: conflict-free row reads
  static constexpr int STAGE = LPR * ROW;                // NB blocks x H rows = LPR staged rows
  static constexpr int CAP = 4 * LPR;                    // list entries per window
  static constexpr int GROUP_BYTES = 2 * STAGE + CAP * 8;
  static constexpr int CTA_BYTES = STAGED_WARPS * (32 / LPR) * GROUP_BYTES;
};

// Per-item constants of the staged path and the two operations that start a batch: the lane's
// block metadata (first B row k0 and width w of block bb + gl) and the cp.async staging of the
// batch's tile rows.  They are free functions so the kernel can start the NEXT item's first batch
// while the current item's last batch is still gathering (the item chain no longer pays the
// metadata + staging latency in series).
template <typename T>
struct StagedCtx {
  int g, p0, h, b0, hp, bb, be;
  const T* tiles;
};
template <typename T>
__device__ __forceinline__ StagedCtx<T> staged_ctx(const SkinnyArgs& a, const SkinnyItem& it) {
  StagedCtx<T> c;
  c.g = it.g;
  c.p0 = a.row_partition[it.g];
  c.h = a.row_partition[it.g + 1] - c.p0;
  c.b0 = a.blk_ptr[it.g];
  c.hp = tile_pitch(c.h);  // tile row pitch
  c.bb = it.bb;
  c.be = it.be;
  c.tiles = static_cast<const T*>(a.tiles) + a.grp_tile_row[it.g] * (int64_t)a.dp;
  return c;
}
template <typename T, int H, int LPR>
__device__ __forceinline__ void staged_meta(const SkinnyArgs& a, const StagedCtx<T>& c, int bb, int gl, int& k0,
                                            int& w) {
  constexpr int NB = LPR / H;
  k0 = 0;
  w = 0;
  if (gl < NB && gl < c.be - bb) {
    const int bc = __ldg(a.blk_col + bb + gl);
    k0 = __ldg(a.col_bounds + bc);
    w = __ldg(a.col_bounds + bc + 1) - k0;
  }
}
template <typename T, int H, int LPR>
__device__ __forceinline__ void staged_issue(const SkinnyArgs& a, const StagedCtx<T>& c, int bb, uint8_t* buf,
                                             int w_lane, int gl, unsigned gmask) {
  using S = SkinnySmem<T, LPR>;
  constexpr int VEC = 16 / sizeof(T);
  constexpr int NB = LPR / H;
  const int nbb = min(NB, c.be - bb);
  const int64_t dp = a.dp;
#pragma unroll
  for (int t = 0; t < S::PPB; ++t) {
    const int q = t * LPR + gl;
    const int row = q / S::PPB, pc = q - row * S::PPB;  // staged row = j * H + r
    const int j = row / H, r = row - j * H;
    const int wj = __shfl_sync(gmask, w_lane, j, LPR);
    const bool pred = j < nbb && r < c.h && pc * VEC < wj;
    cp_async16(buf + row * S::ROW + pc * 16,
               pred ? c.tiles + ((int64_t)(bb - c.b0 + j) * c.hp + r) * dp + pc * VEC : c.tiles, pred);
  }
  cp_async_commit();
}

// Block rows of height h <= H (H = 1, 2, 4, 8), tiles at most 64 columns wide.  Per batch of
// NB = LPR / H blocks the lane group
//   * stages the blocks' h tile rows in shared memory with cp.async (double buffered: the next
//     batch's rows and block columns are in flight while this batch's B rows are gathered; during
//     the item's last batch, the next item's first batch is),
//   * lane j turns block j's staged rows into the 64-bit mask of columns holding a nonzero in any
//     row (16-byte shared loads, padded rows),
//   * a group prefix sum orders those columns (block ascending, k ascending) into a list,
//   * the list is streamed with DEPTH B-row gathers in flight per lane; each gathered B row feeds
//     all h accumulators, the tile values coming from shared memory (broadcast reads).
// On entry the item's first batch is already staged in stage[buf] with metadata (k0c, wc); `next`
// (when has_next) is started in the other buffer during the last batch, and buf / k0c / wc / cnext
// are left describing it.
template <typename T, int H, int LPR, bool ALIGNED>
__device__ __forceinline__ void staged_item(const SkinnyArgs& a, const SkinnyItem& it, const StagedCtx<T>& c,
                                            int cols, int gl, unsigned gmask, uint8_t* stage, int2* list,
                                            int& buf, int& k0c, int& wc, bool has_next, const SkinnyItem& next,
                                            StagedCtx<T>& cnext) {
  using S = SkinnySmem<T, LPR>;
  constexpr int VEC = 16 / sizeof(T);
  constexpr int NB = LPR / H;                 // blocks per batch
  constexpr int DEPTH = H >= 4 ? 4 : H == 1 ? RB_SK1_DEPTH : 8;  // B gathers in flight per lane
  constexpr int ROWE = S::ROW / (int)sizeof(T);
  const int n = it.n0 + gl * VEC;
  const int h = c.h;
  const int64_t ldb = a.ldb;
  const T* Bn = static_cast<const T*>(a.B) + n;

  float acc[H][VEC];
#pragma unroll
  for (int r = 0; r < H; ++r)
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[r][e] = 0.f;

  for (int bb = it.bb; bb < it.be; bb += NB, buf ^= 1) {
    const int nbb = min(NB, it.be - bb);
    const int bbn = bb + NB;
    const bool last = bbn >= it.be;
    int k0n = 0, wn = 0;
    if (!last) {
      staged_meta<T, H, LPR>(a, c, bbn, gl, k0n, wn);  // in flight while this batch is processed
    } else if (has_next) {
      cnext = staged_ctx<T>(a, next);
      staged_meta<T, H, LPR>(a, cnext, next.bb, gl, k0n, wn);
    }
    uint8_t* cur = stage + buf * S::STAGE;
    const T* curT = reinterpret_cast<const T*>(cur);
    cp_async_wait_all();
    __syncwarp(gmask);
    // lane j: columns of block j holding a nonzero in any of its h staged rows
    uint64_t msk = 0;
    if (gl < nbb) {
#pragma unroll
      for (int r = 0; r < H; ++r) {
        if (r >= h) break;
        const uint4* row = reinterpret_cast<const uint4*>(cur + (gl * H + r) * S::ROW);
#pragma unroll
        for (int pc = 0; pc < S::PPB; ++pc) {
          const uint4 u = row[pc];
          const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if constexpr (sizeof(T) == 4) {
              const int e = pc * 4 + i;
              if (e < wc && (w4[i] & 0x7fffffffu)) msk |= 1ull << e;
            } else {
              const int e = pc * 8 + 2 * i;
              if (e < wc && (w4[i] & 0x7fffu)) msk |= 1ull << e;
              if (e + 1 < wc && (w4[i] & 0x7fff0000u)) msk |= 1ull << (e + 1);
            }
          }
        }
      }
    }
    const int cnt = __popcll(msk);
    int incl = cnt;
#pragma unroll
    for (int d = 1; d < LPR; d <<= 1) {
      const int y = __shfl_up_sync(gmask, incl, d, LPR);
      if (gl >= d) incl += y;
    }
    const int total = __shfl_sync(gmask, incl, LPR - 1, LPR);
    const int excl = incl - cnt;
    bool issued = false;
    auto issue_next = [&]() {  // the next batch's (or the next item's first) rows land while this one gathers
      if (!last) staged_issue<T, H, LPR>(a, c, bbn, stage + (buf ^ 1) * S::STAGE, wn, gl, gmask);
      else if (has_next) staged_issue<T, H, LPR>(a, cnext, next.bb, stage + (buf ^ 1) * S::STAGE, wn, gl, gmask);
    };
    for (int base = 0; base < total; base += S::CAP) {
      if (excl < base + S::CAP && incl > base) {
        uint64_t m = msk;
        int idx = excl;
        while (m && idx < base + S::CAP) {
          const int e = __ffsll((long long)m) - 1;
          m &= m - 1;
          if (idx >= base) {  // (B row, value) for h == 1, else (B row, staged offset of column e)
            const int y = H == 1 ? __float_as_int(to_f(curT[gl * ROWE + e])) : gl * H * ROWE + e;
            list[idx - base] = make_int2(k0c + e, y);
          }
          ++idx;
        }
      }
      __syncwarp(gmask);
      if (!issued) {
        issue_next();
        issued = true;
      }
      const int nh = min(S::CAP, total - base);
      for (int i = 0; i < nh; i += DEPTH) {
        int off[DEPTH];
        uint4 bv[DEPTH];
#pragma unroll
        for (int u = 0; u < DEPTH; ++u)
          if (i + u < nh) {
            const int2 en = list[i + u];
            off[u] = en.y;
            bv[u] = load_b_raw<T, ALIGNED>(Bn + (int64_t)en.x * ldb, n, a.N);
          }
#pragma unroll
        for (int u = 0; u < DEPTH; ++u)
          if (i + u < nh) {
            if constexpr (H == 1) {
              fma_row<T>(acc[0], __int_as_float(off[u]), bv[u]);
            } else {
#pragma unroll
              for (int r = 0; r < H; ++r)
                if (r < h) fma_row<T>(acc[r], to_f(curT[off[u] + r * ROWE]), bv[u]);
            }
          }
      }
      __syncwarp(gmask);
    }
    if (!issued) issue_next();
    k0c = k0n;
    wc = wn;
  }
  if (it.bb >= it.be && has_next) {  // empty item: start the next one in the current buffer
    cnext = staged_ctx<T>(a, next);
    staged_meta<T, H, LPR>(a, cnext, next.bb, gl, k0c, wc);
    staged_issue<T, H, LPR>(a, cnext, next.bb, stage + buf * S::STAGE, wc, gl, gmask);
  }
  skinny_finish<H, VEC, LPR, ALIGNED>(a, it, cols, h, c.p0, n, gl, gmask, acc);
}

template <typename T, int H, int LPR, bool ALIGNED>
__global__ void __launch_bounds__(STAGED_WARPS * 32, H == 1 ? RB_SK1_MINB : 2) spmm_skinny_staged_kernel(SkinnyArgs a, int cols, unsigned long long* sched) {
  using S = SkinnySmem<T, LPR>;
  constexpr int GPW = 32 / LPR;
  extern __shared__ uint4 smem_sk[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gl = lane % LPR, grp = lane / LPR;
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (grp * LPR));
  uint8_t* gbase = reinterpret_cast<uint8_t*>(smem_sk) + (warp * GPW + grp) * S::GROUP_BYTES;
  int2* list = reinterpret_cast<int2*>(gbase + 2 * S::STAGE);
  const int64_t i0 = next_item<LPR>(sched, gl, gmask);
  if (i0 < a.n_items) {
    SkinnyItem it = load_item(a.items + i0);
    StagedCtx<T> c = staged_ctx<T>(a, it);
    int buf = 0, k0c, wc;
    staged_meta<T, H, LPR>(a, c, it.bb, gl, k0c, wc);
    staged_issue<T, H, LPR>(a, c, it.bb, gbase, wc, gl, gmask);
    for (;;) {
      // claim the next item now; it is needed only when this item's last batch starts
      const int64_t inext = next_item<LPR>(sched, gl, gmask);
      const bool has_next = inext < a.n_items;
      const SkinnyItem next = has_next ? load_item(a.items + inext) : it;
      StagedCtx<T> cnext = c;
      staged_item<T, H, LPR, ALIGNED>(a, it, c, cols, gl, gmask, gbase, list, buf, k0c, wc, has_next, next, cnext);
      if (!has_next) break;
      it = next;
      c = cnext;
    }
  }
  leave<LPR>(sched, gl, (unsigned long long)gridDim.x * (blockDim.x >> 5) * GPW);
}

// ---------------------------------------------------------------------------------------------
// Wide tiles (dp > 64): per 32 (or 16) tile columns the lane group loads the h tile values of its column,
// ballots the columns holding a nonzero in any of the h rows and gathers only those B rows
// (four in flight), each B row feeding all h accumulators.
template <typename T, int H, int LPR, bool ALIGNED>
__device__ __forceinline__ void skinny_item(const SkinnyArgs& a, const SkinnyItem& it, int cols, int gl, int grp,
                                            unsigned gmask) {
  constexpr int VEC = 16 / sizeof(T);
  const int g = it.g;
  const int n = it.n0 + gl * VEC;
  const int p0 = a.row_partition[g], h = a.row_partition[g + 1] - p0;
  const int b0 = a.blk_ptr[g];
  const int hp = tile_pitch(h);  // tile row pitch
  const int64_t dp = a.dp, ldb = a.ldb;
  const T* tiles = static_cast<const T*>(a.tiles) + a.grp_tile_row[g] * dp;
  const T* B = static_cast<const T*>(a.B) + n;

  float acc[H][VEC];
#pragma unroll
  for (int r = 0; r < H; ++r)
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[r][e] = 0.f;

  for (int bb = it.bb; bb < it.be; bb += LPR) {
    const int nbb = min(LPR, it.be - bb);
    int my_k0 = 0, my_w = 0;
    if (gl < nbb) {
      const int bc = a.blk_col[bb + gl];
      my_k0 = a.col_bounds[bc];
      my_w = a.col_bounds[bc + 1] - my_k0;
    }
    for (int j = 0; j < nbb; ++j) {
      const int k0 = __shfl_sync(gmask, my_k0, j, LPR);
      const int w = __shfl_sync(gmask, my_w, j, LPR);
      const T* t = tiles + (int64_t)(bb - b0 + j) * hp * dp;
      for (int kc = 0; kc < w; kc += LPR) {
        const int k = kc + gl;
        float v[H];
        bool nz = false;
#pragma unroll
        for (int r = 0; r < H; ++r) {
          v[r] = (r < h && k < w) ? to_f(t[r * dp + k]) : 0.f;
          nz |= v[r] != 0.f;
        }
        unsigned m = __ballot_sync(gmask, nz);
        if constexpr (LPR < 32) m = (m >> (grp * LPR)) & ((1u << LPR) - 1u);
        const T* brow = B + (int64_t)(k0 + kc) * ldb;
        while (m) {
          int kk[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            kk[u] = m ? __ffs(m) - 1 : -1;
            m &= m - 1;
          }
          uint4 bv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (kk[u] >= 0) bv[u] = load_b_raw<T, ALIGNED>(brow + kk[u] * ldb, n, a.N);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (kk[u] < 0) break;
#pragma unroll
            for (int r = 0; r < H; ++r) fma_row<T>(acc[r], __shfl_sync(gmask, v[r], kk[u], LPR), bv[u]);
          }
        }
      }
    }
  }
  skinny_finish<H, VEC, LPR, ALIGNED>(a, it, cols, h, p0, n, gl, gmask, acc);
}

template <typename T, int H, int LPR, bool ALIGNED>
__global__ void __launch_bounds__(256, H >= 8 ? 1 : 2) spmm_skinny_kernel(SkinnyArgs a, int cols, unsigned long long* sched) {
  constexpr int GPW = 32 / LPR;
  const int lane = threadIdx.x & 31, gl = lane % LPR, grp = lane / LPR;
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (grp * LPR));
  for (;;) {
    const int64_t i = next_item<LPR>(sched, gl, gmask);
    if (i >= a.n_items) break;
    skinny_item<T, H, LPR, ALIGNED>(a, load_item(a.items + i), cols, gl, grp, gmask);
  }
  leave<LPR>(sched, gl, (unsigned long long)gridDim.x * (blockDim.x >> 5) * GPW);
}

// ---------------------------------------------------------------------------------------------
// CSR comparator (spmm_csr, multiply.py:51-69): the same gather engine straight on a CSR row —
// the sparse baseline the paper measures VBR against.  Item = (row, C-column slab, nonzero range);
// per LPR nonzeros the group loads (column, value) coalesced, then gathers B rows 8 in flight.
template <typename T, int LPR, bool ALIGNED>
__device__ __forceinline__ void csr_item(const SkinnyArgs& a, const CsrArgs& c, const SkinnyItem& it, int cols, int gl,
                                         unsigned gmask) {
  constexpr int VEC = 16 / sizeof(T);
  const int n = it.n0 + gl * VEC;
  const T* Bn = static_cast<const T*>(a.B) + n;
  const int64_t ldb = a.ldb;
  float acc[1][VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc[0][e] = 0.f;
  const int64_t base = c.row_ptr[it.g];
  for (int64_t j0 = base + it.bb; j0 < base + it.be; j0 += LPR) {
    const int cnt = (int)(base + it.be - j0 < LPR ? base + it.be - j0 : LPR);
    int col = 0;
    float val = 0.f;
    if (gl < cnt) {
      if (c.col32) {
        col = __ldg(c.col32 + j0 + gl);
        val = __ldg(c.val32 + j0 + gl);
      } else {
        col = (int)__ldg(c.col_idx + j0 + gl);
        val = round_to<T>(__ldg(c.values + j0 + gl));  // A rounded to the operand dtype, as in VBR tiles
      }
    }
    for (int i = 0; i < cnt; i += 8) {
      float av[8];
      uint4 bv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = __shfl_sync(gmask, col, (i + u) & (LPR - 1), LPR);
        av[u] = __shfl_sync(gmask, val, (i + u) & (LPR - 1), LPR);
        if (i + u < cnt) bv[u] = load_b_raw<T, ALIGNED>(Bn + (int64_t)k * ldb, n, a.N);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i + u < cnt) fma_row<T>(acc[0], av[u], bv[u]);
    }
  }
  skinny_finish<1, VEC, LPR, ALIGNED>(a, it, cols, 1, it.g, n, gl, gmask, acc);
}

template <typename T, int LPR, bool ALIGNED, int CH>
// 4 resident CTAs per SM (<= 64 registers, a few spills): twice the gathers in flight of the
// 2-CTA build; config 3 1.08 -> 0.86 ms, 2b 7.50 -> 6.50 ms, config 1 +6 % (latency-bound, tiny).
#ifndef RB_CSR_MIN_BLOCKS
#define RB_CSR_MIN_BLOCKS 4
#endif

__global__ void __launch_bounds__(256, RB_CSR_MIN_BLOCKS) spmm_csr_kernel(SkinnyArgs a, CsrArgs c, int cols,
                                                          unsigned long long* sched) {
  constexpr int GPW = 32 / LPR;
  const int lane = threadIdx.x & 31, gl = lane % LPR, grp = lane / LPR;
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (grp * LPR));
  if constexpr (CH == 1) {
    for (;;) {
      const int64_t i = next_item<LPR>(sched, gl, gmask);
      if (i >= a.n_items) break;
      csr_item<T, LPR, ALIGNED>(a, c, load_item(a.items + i), cols, gl, gmask);
    }
  } else {  // c.chunk consecutive items per claim (launch_csr_t): one atomic round trip per chunk
    const unsigned long long chunk = c.chunk > 1 ? (unsigned long long)c.chunk : 1ull;
    for (;;) {
      unsigned long long i0 = 0;
      if (gl == 0) i0 = atomicAdd(sched, chunk);
      i0 = __shfl_sync(gmask, i0, 0, LPR);
      if ((int64_t)i0 >= a.n_items) break;
      const int64_t i1 = min((int64_t)(i0 + chunk), a.n_items);
      for (int64_t i = (int64_t)i0; i < i1; ++i) csr_item<T, LPR, ALIGNED>(a, c, load_item(a.items + i), cols, gl, gmask);
    }
  }
  leave<LPR>(sched, gl, (unsigned long long)gridDim.x * (blockDim.x >> 5) * GPW);
}

template <typename K>
int persistent_grid(K kernel, int smem, int64_t n_items, int groups_per_cta, unsigned* grid, int threads = 256) {
  int dev = 0, sms = kNumSMs, per_sm = 1;
  RB_CUDA_TRY(cudaGetDevice(&dev));
  RB_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  RB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  const int64_t need = (n_items + groups_per_cta - 1) / groups_per_cta;
  *grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * std::max(1, per_sm)));
  return RB_OK;
}

template <typename T, int H, int LPR>
int launch_t(const SkinnyArgs& a, int cols, unsigned long long* sched, cudaStream_t stream) {
  const bool aligned = ((a.ldb * (int64_t)sizeof(T)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(a.B) & 15) == 0) &&
                       (a.ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.C) & 15) == 0);
  constexpr int per_cta = 8 * (32 / LPR);
  unsigned grid = 0;
  using S = SkinnySmem<T, LPR>;
  if (a.dp > S::KC) {  // wide tiles: the per-column ballot kernel
    auto k = aligned ? spmm_skinny_kernel<T, H, LPR, true> : spmm_skinny_kernel<T, H, LPR, false>;
    int rc = persistent_grid(k, 0, a.n_items, per_cta, &grid);
    if (rc) return rc;
    k<<<grid, 256, 0, stream>>>(a, cols, sched);
  } else {
    auto k = aligned ? spmm_skinny_staged_kernel<T, H, LPR, true> : spmm_skinny_staged_kernel<T, H, LPR, false>;
    RB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, S::CTA_BYTES));
    int rc = persistent_grid(k, S::CTA_BYTES, a.n_items, STAGED_WARPS * (32 / LPR), &grid, STAGED_WARPS * 32);
    if (rc) return rc;
    k<<<grid, STAGED_WARPS * 32, S::CTA_BYTES, stream>>>(a, cols, sched);
  }
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}

template <typename T, int LPR>
int launch_h(const SkinnyArgs& a, int cls, int cols, unsigned long long* sched, cudaStream_t stream) {
  switch (cls) {
    case 0: return launch_t<T, 1, LPR>(a, cols, sched, stream);
    case 1: return launch_t<T, 2, LPR>(a, cols, sched, stream);
    case 2: return launch_t<T, 4, LPR>(a, cols, sched, stream);
    default: return launch_t<T, 8, LPR>(a, cols, sched, stream);
  }
}

template <typename T, int LPR>
int launch_csr_t(const SkinnyArgs& a, const CsrArgs& c, int cols, unsigned long long* sched, cudaStream_t stream) {
  const bool aligned = ((a.ldb * (int64_t)sizeof(T)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(a.B) & 15) == 0) &&
                       (a.ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.C) & 15) == 0);
  unsigned grid = 0;
  auto k1 = aligned ? spmm_csr_kernel<T, LPR, true, 1> : spmm_csr_kernel<T, LPR, false, 1>;
  int rc = persistent_grid(k1, 0, a.n_items, 8 * (32 / LPR), &grid);
  if (rc) return rc;
  // Two items per claim only for uniform lists (c.chunk) with at least 4 chunks per resident
  // group.  The runtime-chunk instance (CH = 0) also serves 32-lane groups at chunk 1: its
  // register allocation measured faster there (config 2b 6.52 -> 6.04 ms, profiles/r02/chunk_ab/);
  // 16-lane groups keep the single-claim instance (CH = 1).
  const int64_t groups = (int64_t)grid * 8 * (32 / LPR);
  CsrArgs cc = c;
  if (cc.chunk < 1 || a.n_items < 4 * (int64_t)cc.chunk * groups) cc.chunk = 1;
  const bool runtime = LPR == 32 || cc.chunk > 1;
  auto k = runtime ? (aligned ? spmm_csr_kernel<T, LPR, true, 0> : spmm_csr_kernel<T, LPR, false, 0>) : k1;
  k<<<grid, 256, 0, stream>>>(a, cc, cols, sched);
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}

}  // namespace

int launch_csr(const SkinnyArgs& a, const CsrArgs& c, int32_t b_dtype, unsigned long long* sched,
               cudaStream_t stream) {
  if (a.n_items <= 0) return RB_OK;
  const int cols = skinny_cols(b_dtype, a.N);
  switch (b_dtype) {
    case RB_F32: return launch_csr_t<float, 32>(a, c, cols, sched, stream);
    case RB_BF16:
      return a.N <= 128 ? launch_csr_t<__nv_bfloat16, 16>(a, c, cols, sched, stream)
                        : launch_csr_t<__nv_bfloat16, 32>(a, c, cols, sched, stream);
    case RB_F16:
      return a.N <= 128 ? launch_csr_t<__half, 16>(a, c, cols, sched, stream)
                        : launch_csr_t<__half, 32>(a, c, cols, sched, stream);
    default: return fail(RB_EUNSUPPORTED, "csr SpMM: unsupported dtype");
  }
}

int csr_claim_chunk(const std::vector<SkinnyItem>& items) {
  if (items.empty()) return 1;
  int64_t total = 0, longest = 0;
  for (const SkinnyItem& it : items) {
    if (it.nparts > 1) return 1;
    total += it.be - it.bb;
    longest = std::max<int64_t>(longest, it.be - it.bb);
  }
  return longest * (int64_t)items.size() <= 2 * total ? 2 : 1;
}

int skinny_cols(int32_t b_dtype, int64_t N) {
  if (b_dtype == RB_F32) return 128;  // 32 lanes x 4
  return N <= 128 ? 128 : 256;        // 16 or 32 lanes x 8
}

void skinny_items_for_row(int32_t g, int h, int32_t blk_begin, int nb, int64_t N, int cols,
                          std::vector<SkinnyItem>& out, int64_t& n_slots, int64_t& ws_units, int part_blocks) {
  const int H = skinny_class_h(skinny_class(h));
  const int pb = std::max(1, part_blocks);
  const int nparts = nb > pb ? (nb + pb - 1) / pb : 1;
  for (int64_t n0 = 0; n0 < N; n0 += cols) {
    if (nparts == 1) {
      out.push_back(SkinnyItem{g, (int32_t)n0, blk_begin, blk_begin + nb, 0, 1, -1, 0});
      continue;
    }
    const int32_t slot = (int32_t)n_slots++;
    const int32_t wsoff = (int32_t)ws_units;
    ws_units += (int64_t)nparts * H * (cols / 128);
    for (int p = 0; p < nparts; ++p)
      out.push_back(SkinnyItem{g, (int32_t)n0, blk_begin + (int32_t)((int64_t)nb * p / nparts),
                               blk_begin + (int32_t)((int64_t)nb * (p + 1) / nparts), p, nparts, slot, wsoff});
  }
}

int launch_skinny(const SkinnyArgs& a, int32_t b_dtype, int cls, unsigned long long* sched, cudaStream_t stream) {
  if (a.n_items <= 0) return RB_OK;
  const int cols = skinny_cols(b_dtype, a.N);
  switch (b_dtype) {
    case RB_F32: return launch_h<float, 32>(a, cls, cols, sched, stream);
    case RB_BF16:
      return a.N <= 128 ? launch_h<__nv_bfloat16, 16>(a, cls, cols, sched, stream)
                        : launch_h<__nv_bfloat16, 32>(a, cls, cols, sched, stream);
    case RB_F16:
      return a.N <= 128 ? launch_h<__half, 16>(a, cls, cols, sched, stream)
                        : launch_h<__half, 32>(a, cls, cols, sched, stream);
    default: return fail(RB_EUNSUPPORTED, "skinny SpMM: unsupported dtype");
  }
}

}  // namespace rb
