// 1-SA row reordering on the device: replaces block_1sa (blocking.py:283-306).
//
//   K1 quotient_kernel   per-row segment bitsets + sizes         (blocking.py:118-136)
//   K2 compression       64-bit pattern hash, stable radix sort, exact word compare inside
//                        equal-hash runs, classes numbered by their smallest row
//                        (first-occurrence order, blocking.py:295-301)
//   K3 greedy_kernel     the one-pass greedy scan (blocking.py:209-266) as ONE persistent
//                        cooperative kernel: every round evaluates the whole unassigned suffix
//                        in parallel against the current pattern, reduces the first growing hit
//                        (argmin) and the first rejection, and applies them after a grid barrier;
//                        verdicts are bit-exact (IEEE double products, sqrt and division exactly
//                        as numpy evaluates blocking.py:239-248).
//   assembly             rows ordered by (group, item, row) (blocking.py:269-280), group
//                        extents, seed sizes, group patterns = OR of member bitsets.
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "segments.cuh"

namespace rb {
namespace {

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
inline int64_t words_of(int64_t n_seg) { return n_seg > 0 ? (n_seg + 63) / 64 : 1; }
constexpr int kMaxTesters = 4096;  // speculative seeds per batch of the dense greedy (one per warp)
inline unsigned grid_for(int64_t work, int per_block) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + per_block - 1) / per_block, 148 * 16));
}

struct MaxOp {
  __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

struct Ws {
  unsigned long long* bits;       // [n*W]   (reused as group bits after the gather)
  int32_t* sizes;                 // [n]
  unsigned long long* item_bits;  // [n*W]
  int32_t* item_sizes;            // [n]
  int32_t* item_of_row;           // [n]
  int32_t* reps;                  // [n]
  int32_t* group_of_item;         // [n]
  int32_t* seed_item;             // [n]
  uint8_t* ok;                    // [n]
  int32_t* ctrl;                  // [16]
  unsigned long long* keys_a;     // [n]
  unsigned long long* keys_b;     // [n]
  int32_t* vals_a;                // [n]
  int32_t* vals_b;                // [n]
  int32_t* t0;                    // [n+1]
  int32_t* t1;                    // [n+1]
  int64_t* pcnt;                  // [n+1]
  int32_t* b32;                   // [n_seg+1]
  void* cub_tmp;
  size_t cub_bytes;
  size_t total;
};

size_t cub_bytes_for(int64_t n) {
  const int nn = (int)std::max<int64_t>(n + 1, 2);
  size_t a = 0, b = 0, c = 0, d = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, nn);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int32_t*)nullptr, (int32_t*)nullptr, nn);
  cub::DeviceScan::ExclusiveSum(nullptr, c, (int64_t*)nullptr, (int64_t*)nullptr, nn);
  cub::DeviceScan::InclusiveScan(nullptr, d, (int32_t*)nullptr, (int32_t*)nullptr, MaxOp(), nn);
  return std::max(std::max(a, b), std::max(c, d));
}

Ws carve(void* base, int64_t n, int64_t W, int64_t n_seg) {
  Ws w;
  size_t off = 0;
  const int64_t n1 = std::max<int64_t>(n, 1);
  auto take = [&](size_t bytes) {
    void* p = base ? static_cast<char*>(base) + off : nullptr;
    off += align256(bytes);
    return p;
  };
  w.bits = (unsigned long long*)take(sizeof(uint64_t) * n1 * W);
  w.sizes = (int32_t*)take(sizeof(int32_t) * n1);
  w.item_bits = (unsigned long long*)take(sizeof(uint64_t) * n1 * W);
  w.item_sizes = (int32_t*)take(sizeof(int32_t) * n1);
  w.item_of_row = (int32_t*)take(sizeof(int32_t) * n1);
  w.reps = (int32_t*)take(sizeof(int32_t) * n1);
  w.group_of_item = (int32_t*)take(sizeof(int32_t) * n1);
  w.seed_item = (int32_t*)take(sizeof(int32_t) * n1);
  w.ok = (uint8_t*)take(n1);
  w.ctrl = (int32_t*)take(sizeof(int32_t) * (16 + 2 * kMaxTesters));
  w.keys_a = (unsigned long long*)take(sizeof(uint64_t) * n1);
  w.keys_b = (unsigned long long*)take(sizeof(uint64_t) * n1);
  w.vals_a = (int32_t*)take(sizeof(int32_t) * n1);
  w.vals_b = (int32_t*)take(sizeof(int32_t) * n1);
  w.t0 = (int32_t*)take(sizeof(int32_t) * (n1 + 1));
  w.t1 = (int32_t*)take(sizeof(int32_t) * (n1 + 1));
  w.pcnt = (int64_t*)take(sizeof(int64_t) * (n1 + 1));
  w.b32 = (int32_t*)take(sizeof(int32_t) * (n_seg + 1));
  w.cub_bytes = cub_bytes_for(n);
  w.cub_tmp = take(w.cub_bytes);
  w.total = off;
  return w;
}

// ---------------------------------------------------------------- K1: quotient bitsets
__global__ void quotient_kernel(const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col_idx, int64_t n,
                                SegMap seg, int64_t W, unsigned long long* bits, int32_t* sizes) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const int64_t s0 = row_ptr[r], s1 = row_ptr[r + 1];
    unsigned long long* row = bits + r * W;
    int cnt = 0;
    for (int64_t j = s0 + lane; j < s1; j += 32) {
      const int32_t s = seg((int32_t)col_idx[j]);
      if (j == s0 || seg((int32_t)col_idx[j - 1]) != s) {  // first column of a segment run
        atomicOr(row + (s >> 6), 1ull << (s & 63));
        ++cnt;
      }
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) sizes[r] = cnt;
  }
}

// ---------------------------------------------------------------- K2: compression
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

__global__ void hash_kernel(const unsigned long long* __restrict__ bits, int64_t n, int64_t W,
                            unsigned long long* keys, int32_t* vals) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long h = 0x9E3779B97F4A7C15ull;
    const unsigned long long* row = bits + r * W;
    for (int64_t w = 0; w < W; ++w) h = mix64(h ^ (row[w] + 0x632BE59BD9B4E019ull * (unsigned long long)(w + 1)));
    keys[r] = h;
    vals[r] = (int32_t)r;
  }
}

__global__ void run_head_kernel(const unsigned long long* __restrict__ keys, int64_t n, int32_t* head) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    head[p] = (p == 0 || keys[p] != keys[p - 1]) ? (int32_t)p : 0;
}

__device__ __forceinline__ bool words_equal(const unsigned long long* a, const unsigned long long* b, int64_t W) {
  for (int64_t w = 0; w < W; ++w)
    if (a[w] != b[w]) return false;
  return true;
}

// rep(row) = smallest row with identical bits: the first equal row of its equal-hash run (rows are
// ascending inside a run because the radix sort is stable).
__global__ void rep_kernel(const unsigned long long* __restrict__ bits, const int32_t* __restrict__ rows_sorted,
                           const int32_t* __restrict__ run_start, int64_t n, int64_t W, int32_t* rep_of_row) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows_sorted[p];
    int32_t rep = r;
    for (int64_t q = run_start[p]; q < p; ++q) {
      const int32_t c = rows_sorted[q];
      if (words_equal(bits + (int64_t)c * W, bits + (int64_t)r * W, W)) {
        rep = c;
        break;
      }
    }
    rep_of_row[r] = rep;
  }
}

__global__ void is_rep_kernel(const int32_t* __restrict__ rep_of_row, int64_t n, int32_t* flag) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    flag[r] = rep_of_row[r] == (int32_t)r ? 1 : 0;
}

__global__ void items_kernel(const int32_t* __restrict__ rep_of_row, const int32_t* __restrict__ idx, int64_t n,
                             int32_t* item_of_row, int32_t* reps) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t rep = rep_of_row[r];
    item_of_row[r] = idx[rep];
    if (rep == (int32_t)r) reps[idx[r]] = (int32_t)r;
  }
}

__global__ void identity_items_kernel(int64_t n, int32_t* item_of_row, int32_t* reps) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    item_of_row[r] = (int32_t)r;
    reps[r] = (int32_t)r;
  }
}

__global__ void gather_items_kernel(const unsigned long long* __restrict__ bits, const int32_t* __restrict__ sizes,
                                    const int32_t* __restrict__ reps, int64_t m, int64_t W,
                                    unsigned long long* item_bits, int32_t* item_sizes, int32_t* group_of_item) {
  const int64_t total = m * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i / W, w = i - j * W;
    const int32_t r = reps[j];
    item_bits[i] = bits[(int64_t)r * W + w];
    if (w == 0) {
      item_sizes[j] = sizes[r];
      group_of_item[j] = -1;
    }
  }
}

// ---------------------------------------------------------------- K3: greedy scan
struct GreedyArgs {
  int32_t m;
  int32_t W;
  const unsigned long long* bits;  // item bitsets [m*W]
  const int32_t* sizes;            // item sizes [m]
  double tau;
  int32_t cosine, bounded, update;
  int32_t* group_of_item;  // [m], -1 = unassigned
  uint8_t* ok;             // [m] verdict of the latest evaluation
  int32_t* seed_item;      // [H]
  int32_t* ctrl;           // [0..2] first growing hit, [3..5] first rejection, [6] H, [8] count, [9] gen,
                           // [10..12] ok counts, [16..16+2*kMaxTesters) speculative flags (two batches)
  int32_t batching;        // speculative singleton batching enabled
};

// Merge predicate (blocking.py:239-248 == merge_condition 184-203), IEEE double, no contraction.
__device__ __forceinline__ bool accept_dev(int64_t inter, int64_t psize, int64_t size, double tau, int cosine,
                                           int bounded, double cap) {
  const int64_t uni = psize + size - inter;
  bool ok;
  if (!cosine) {
    ok = (double)inter >= __dmul_rn(tau, (double)uni);
  } else {
    ok = (double)inter >= __dmul_rn(tau, __dsqrt_rn((double)(psize * size)));
    if (tau > 0.0) ok = ok && ((size == 0) == (psize == 0));
  }
  if (ok && bounded) ok = (double)uni <= cap;
  return ok;
}

__device__ __forceinline__ void grid_barrier(int32_t* count, int32_t* gen) {
  __syncthreads();
  if (gridDim.x == 1) return;
  if (threadIdx.x == 0) {
    volatile int32_t* vgen = gen;
    const int32_t my = *vgen;
    __threadfence();
    if (atomicAdd(count, 1) == (int32_t)gridDim.x - 1) {
      atomicExch(count, 0);
      __threadfence();
      atomicAdd(gen, 1);
    } else {
      while (*vgen == my) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// The greedy scan (blocking.py:209-266) with speculative singleton batching (exact):
//  GROUP round: all CTAs evaluate every unassigned item >= pos against the pattern; the first
//         growing hit grows the pattern, a complete group seeds the next one at its first rejection.
//  BATCH: after a singleton group (one round, nothing accepted) every warp takes one of the next K
//         unassigned items as a speculative seed and tests whether ANY later unassigned item passes
//         the merge test against it.  Seeds before the first one with a hit are singleton groups in
//         the sequential scan too (a singleton assigns only itself, never a candidate of a later
//         seed), so they are committed in order at once; the first seed with a hit starts a GROUP.
//         A batch whose first seed has a hit backs off (2^k later groups skip batching).
template <bool kWarpPerItem>
__global__ void __launch_bounds__(512) greedy_kernel(GreedyArgs a) {
  extern __shared__ unsigned long long sP[];  // current pattern, W words
  __shared__ int32_t s_js, s_rj, s_ok;
  __shared__ int32_t s_pos, s_g, s_first_rej, s_acc_lo, s_acc_hi, s_acc_g, s_finishing;
  __shared__ int32_t s_mode, s_grounds, s_cursor, s_batch, s_backoff, s_skip, s_len, s_f;
  __shared__ long long s_psize;
  __shared__ double s_cap;
  __shared__ int32_t s_inter;
  __shared__ int32_t s_list[kMaxTesters];

  const int32_t m = a.m, W = a.W;
  const double tau = a.tau;
  const double cap_den = __dsub_rn(1.0, __dmul_rn(0.5, tau));
  if (threadIdx.x == 0) {
    s_g = 0;
    s_pos = 1;
    s_first_rej = INT_MAX;
    s_acc_lo = s_acc_hi = 0;
    s_acc_g = 0;
    s_finishing = 0;
    s_mode = 0;
    s_grounds = 0;
    s_batch = 0;
    s_backoff = 0;
    s_skip = 0;
    s_psize = a.sizes[0];
    s_cap = __ddiv_rn((double)a.sizes[0], cap_den);
    if (blockIdx.x == 0) {
      a.group_of_item[0] = 0;
      a.seed_item[0] = 0;
    }
  }
  for (int w = threadIdx.x; w < W; w += blockDim.x) sP[w] = a.bits[w];
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int32_t K = min((int32_t)(gridDim.x * nwarps), (int32_t)kMaxTesters);
  for (int r = 0;;) {
    if (s_mode == 1) {
      // ============================ BATCH: speculative singleton seeds, one per warp
      if (warp == 0) {
        int32_t cnt = 0;
        for (int32_t j0 = s_cursor; j0 < m && cnt < K; j0 += 32) {
          const int32_t j = j0 + lane;
          const bool un = j < m && __ldcg(a.group_of_item + j) < 0;
          const unsigned b = __ballot_sync(0xffffffffu, un);
          const int32_t rk = __popc(b & ((1u << lane) - 1u));
          if (un && cnt + rk < K) s_list[cnt + rk] = j;
          cnt += __popc(b);
        }
        if (lane == 0) s_len = min(cnt, K);
      }
      __syncthreads();
      const int32_t len = s_len, batch = s_batch;
      if (len == 0) break;  // every item is assigned
      int32_t* flags = a.ctrl + 16 + (batch & 1) * kMaxTesters;
      const int32_t t = (int32_t)blockIdx.x * nwarps + warp;
      if (t < len) {
        const int32_t seed = s_list[t];
        const unsigned long long* bs = a.bits + (int64_t)seed * W;
        const int64_t ps = a.sizes[seed];
        const double cap = __ddiv_rn((double)ps, cap_den);
        bool hit = false;
        for (int32_t j0 = seed + 1; j0 < m && !hit; j0 += 32) {
          const int32_t j = j0 + lane;
          bool v = false;
          if (j < m && __ldcg(a.group_of_item + j) < 0) {
            const unsigned long long* bj = a.bits + (int64_t)j * W;
            int64_t inter = 0;
            for (int w = 0; w < W; ++w) inter += __popcll(__ldg(bj + w) & __ldg(bs + w));
            v = accept_dev(inter, ps, a.sizes[j], tau, a.cosine, a.bounded, cap);
          }
          hit = __any_sync(0xffffffffu, v);
        }
        if (lane == 0) flags[t] = hit ? 1 : 0;
      }
      grid_barrier(a.ctrl + 8, a.ctrl + 9);
      if (warp == 0) {
        int32_t f = len;
        for (int32_t k0 = 0; k0 < len; k0 += 32) {
          const int32_t k = k0 + lane;
          const bool hit = k < len && *((volatile const int32_t*)(flags + k)) != 0;
          const unsigned b = __ballot_sync(0xffffffffu, hit);
          if (b) {
            f = k0 + __ffs(b) - 1;
            break;
          }
        }
        if (lane == 0) s_f = f;
      }
      __syncthreads();
      const int32_t f = s_f, g0 = s_g;
      if (blockIdx.x == 0)  // singletons before the first hit, in order
        for (int32_t k = threadIdx.x; k < f; k += blockDim.x) {
          a.group_of_item[s_list[k]] = g0 + 1 + k;
          a.seed_item[g0 + 1 + k] = s_list[k];
        }
      if (f == len) {
        __syncthreads();
        if (threadIdx.x == 0) {
          s_g = g0 + len;
          s_cursor = s_list[len - 1] + 1;
          s_batch = batch + 1;
          s_backoff = 0;
        }
        __syncthreads();
        continue;
      }
      const int32_t seed = s_list[f], gid = g0 + 1 + f;
      __syncthreads();
      if (threadIdx.x == 0) {
        if (blockIdx.x == 0) {
          a.group_of_item[seed] = gid;
          a.seed_item[gid] = seed;
        }
        s_g = gid;
        s_pos = seed + 1;
        s_first_rej = INT_MAX;
        s_acc_lo = s_acc_hi = 0;
        s_psize = a.sizes[seed];
        s_cap = __ddiv_rn((double)a.sizes[seed], cap_den);
        s_grounds = 0;
        s_batch = batch + 1;
        if (f == 0) {  // wasted batch: back off
          s_backoff = min(s_backoff + 1, 12);
          s_skip = 1 << s_backoff;
        } else {
          s_backoff = 0;
        }
        s_mode = 0;
      }
      for (int w = threadIdx.x; w < W; w += blockDim.x) sP[w] = a.bits[(int64_t)seed * W + w];
      __syncthreads();
      continue;
    }

    // ============================ GROUP round
    const int slot = r % 3;
    ++r;
    if (threadIdx.x == 0) {
      s_js = INT_MAX;
      s_rj = INT_MAX;
      s_ok = 0;
    }
    __syncthreads();
    const int32_t pos = s_pos, acc_lo = s_acc_lo, acc_hi = s_acc_hi, acc_g = s_acc_g, g = s_g;
    const long long psize = s_psize;
    const double cap = s_cap;
    const int32_t lo = acc_lo < acc_hi ? min(acc_lo, pos) : pos;
    int32_t my_js = INT_MAX, my_rj = INT_MAX, my_ok = 0;
    if (kWarpPerItem) {
      const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
      const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
      for (int64_t j = lo + wid; j < m; j += nw) {
        // group_of_item / ok are written by other CTAs between phases: read through L2 (ld.cg)
        int32_t gi = __ldcg(a.group_of_item + j);
        if (gi < 0 && j >= acc_lo && j < acc_hi && __ldcg(a.ok + j)) {
          gi = acc_g;
          if (lane == 0) a.group_of_item[j] = acc_g;
        }
        if (j >= pos && gi < 0) {
          const unsigned long long* bj = a.bits + j * W;
          int c = 0;
          for (int w = lane; w < W; w += 32) c += __popcll(bj[w] & sP[w]);
          const int64_t inter = __reduce_add_sync(0xffffffffu, c);
          const int64_t sz = a.sizes[j];
          const bool v = accept_dev(inter, psize, sz, tau, a.cosine, a.bounded, cap);
          if (lane == 0) {
            a.ok[j] = v;
            my_ok += v;
            if (v && a.update && inter < sz) my_js = min(my_js, (int32_t)j);
            if (!v) my_rj = min(my_rj, (int32_t)j);
          }
        }
      }
    } else {
      const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
      const int64_t nt = (int64_t)gridDim.x * blockDim.x;
      for (int64_t j = lo + tid; j < m; j += nt) {
        int32_t gi = __ldcg(a.group_of_item + j);
        if (gi < 0 && j >= acc_lo && j < acc_hi && __ldcg(a.ok + j)) {
          gi = acc_g;
          a.group_of_item[j] = acc_g;
        }
        if (j >= pos && gi < 0) {
          const unsigned long long* bj = a.bits + j * W;
          int64_t inter = 0;
          for (int w = 0; w < W; ++w) inter += __popcll(bj[w] & sP[w]);
          const int64_t sz = a.sizes[j];
          const bool v = accept_dev(inter, psize, sz, tau, a.cosine, a.bounded, cap);
          a.ok[j] = v;
          my_ok += v;
          if (v && a.update && inter < sz) my_js = min(my_js, (int32_t)j);
          if (!v) my_rj = min(my_rj, (int32_t)j);
        }
      }
    }
    my_js = __reduce_min_sync(0xffffffffu, my_js);
    my_rj = __reduce_min_sync(0xffffffffu, my_rj);
    my_ok = __reduce_add_sync(0xffffffffu, my_ok);
    if (lane == 0) {
      if (my_js != INT_MAX) atomicMin(&s_js, my_js);
      if (my_rj != INT_MAX) atomicMin(&s_rj, my_rj);
      if (my_ok) atomicAdd(&s_ok, my_ok);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_js != INT_MAX) atomicMin(a.ctrl + slot, s_js);
      if (s_rj != INT_MAX) atomicMin(a.ctrl + 3 + slot, s_rj);
      if (s_ok) atomicAdd(a.ctrl + 10 + slot, s_ok);
    }
    grid_barrier(a.ctrl + 8, a.ctrl + 9);
    if (s_finishing) break;  // the final acceptance has been applied
    const int32_t js = *((volatile int32_t*)(a.ctrl + slot));
    const int32_t rj = *((volatile int32_t*)(a.ctrl + 3 + slot));
    const int32_t okc = *((volatile int32_t*)(a.ctrl + 10 + slot));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.ctrl[(slot + 2) % 3] = INT_MAX;
      a.ctrl[3 + (slot + 2) % 3] = INT_MAX;
      a.ctrl[10 + (slot + 2) % 3] = 0;
    }
    if (js < m) {
      // growth at js: accept ok items in [pos, js] (next phase), OR js's bits into the pattern
      if (threadIdx.x < 32) {
        int c = 0;
        for (int w = lane; w < W; w += 32) c += __popcll(a.bits[(int64_t)js * W + w] & sP[w]);
        c = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0) s_inter = c;
      }
      __syncthreads();
      for (int w = threadIdx.x; w < W; w += blockDim.x) sP[w] |= a.bits[(int64_t)js * W + w];
      if (threadIdx.x == 0) {
        s_acc_lo = pos;
        s_acc_hi = js + 1;
        s_acc_g = g;
        if (rj < js) s_first_rej = min(s_first_rej, rj);
        s_psize = psize + a.sizes[js] - s_inter;
        s_pos = js + 1;
        s_grounds += 1;
      }
    } else {
      // the group is complete: accept ok items in [pos, m); the first rejected item seeds the next group
      const int32_t fr = min(s_first_rej, rj);
      const bool singleton = s_grounds == 0 && okc == 0;
      const bool to_batch = a.batching && singleton && fr < m && s_skip == 0;
      __syncthreads();
      if (threadIdx.x == 0) {
        s_acc_lo = pos;
        s_acc_hi = m;
        s_acc_g = g;
        if (s_skip > 0) --s_skip;
        if (fr >= m) {
          s_finishing = 1;
          s_pos = m;
        } else if (to_batch) {
          s_acc_lo = s_acc_hi = 0;  // nothing was accepted
          s_cursor = fr;
          s_mode = 1;
        } else {
          s_g = g + 1;
          s_first_rej = INT_MAX;
          s_psize = a.sizes[fr];
          s_cap = __ddiv_rn((double)a.sizes[fr], cap_den);
          s_pos = fr + 1;
          s_grounds = 0;
          if (blockIdx.x == 0) {
            a.group_of_item[fr] = g + 1;
            a.seed_item[g + 1] = fr;
          }
        }
      }
      if (fr < m && !to_batch)
        for (int w = threadIdx.x; w < W; w += blockDim.x) sP[w] = a.bits[(int64_t)fr * W + w];
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.ctrl[6] = s_g + 1;
}

// ---------------------------------------------------------------- assembly
__global__ void assembly_keys_kernel(const int32_t* __restrict__ item_of_row, const int32_t* __restrict__ group_of_item,
                                     int64_t n, int64_t m, unsigned long long* keys, int32_t* vals) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t it = item_of_row[r];
    keys[r] = (unsigned long long)group_of_item[it] * (unsigned long long)m + (unsigned long long)it;
    vals[r] = (int32_t)r;
  }
}

__global__ void assembly_out_kernel(const int32_t* __restrict__ rows_sorted, const unsigned long long* __restrict__ keys,
                                    int64_t n, int64_t m, int64_t H, int64_t* row_perm, int64_t* group_of,
                                    int64_t* group_ptr) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows_sorted[p];
    const int64_t g = (int64_t)(keys[p] / (unsigned long long)m);
    row_perm[p] = r;
    group_of[r] = g;
    if (p == 0 || (int64_t)(keys[p - 1] / (unsigned long long)m) != g) group_ptr[g] = p;
    if (p == 0) group_ptr[H] = n;
  }
}

__global__ void seed_size_kernel(const int32_t* __restrict__ seed_item, const int32_t* __restrict__ item_sizes,
                                 int64_t H, int64_t* seed_size) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < H; g += (int64_t)gridDim.x * blockDim.x)
    seed_size[g] = item_sizes[seed_item[g]];
}

__global__ void group_or_kernel(const unsigned long long* __restrict__ item_bits,
                                const int32_t* __restrict__ group_of_item, int64_t m, int64_t W,
                                unsigned long long* gbits) {
  const int64_t total = m * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long x = item_bits[i];
    if (x) {
      const int64_t j = i / W, w = i - j * W;
      atomicOr(gbits + (int64_t)group_of_item[j] * W + w, x);
    }
  }
}

// warp per group: popcount (pass 0) or extraction into pattern_idx (pass 1)
__global__ void pattern_kernel(const unsigned long long* __restrict__ gbits, int64_t H, int64_t W, int pass,
                               int64_t* pcnt, const int64_t* __restrict__ pattern_ptr, int64_t* pattern_idx) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); g < H; g += warps) {
    int64_t running = pass ? pattern_ptr[g] : 0;
    for (int64_t w0 = 0; w0 < W; w0 += 32) {
      const int64_t w = w0 + lane;
      const unsigned long long x = w < W ? gbits[g * W + w] : 0ull;
      const int c = __popcll(x);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (pass) {
        int64_t k = running + incl - c;
        unsigned long long y = x;
        while (y) {
          const int b = __ffsll((long long)y) - 1;
          pattern_idx[k++] = w * 64 + b;
          y &= y - 1;
        }
      }
      running += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (!pass && lane == 0) pcnt[g] = running;
  }
}


// =============================================================================================
// Sparse pipeline (large W, e.g. config 3: 32768 segments): segment LISTS instead of bitsets and an
// inverted index (segment -> items ascending).  The greedy kernel enumerates, per round, only the
// candidates that share a segment with a PREFIX of the current pattern: every acceptable candidate
// shares >= t = ceil(fl(tau*psize)) segments with P (jaccard; cosine: tau^2*psize, conservative),
// so it must hit any psize - t + 1 of P's segments (exact).  The prefix is every
// segment whose postings length falls in the log2-length buckets that first reach psize - t + 1
// segments (a superset of the rarest ones, hence still exact).  t == 0 (tau == 0) scans all
// unassigned items; an empty pattern (tau > 0) only the empty items.

constexpr int64_t kDenseMaxWords = 64;

bool use_sparse_path(int64_t W) {
  const char* m = std::getenv("RB_1SA_MODE");
  if (m && m[0] == 's') return true;
  if (m && m[0] == 'd') return false;
  return W > kDenseMaxWords;
}

struct SWs {
  int32_t* sizes;          // [n]
  int64_t* rs_ptr;         // [n+1]
  int32_t* rs;             // [nnz]   row segment lists
  unsigned long long* keys_a;  // [max(n, nnz)]
  unsigned long long* keys_b;  // [max(n, nnz)]
  int32_t* vals_a;         // [n]
  int32_t* vals_b;         // [n]
  int32_t* t0;             // [n+1]
  int32_t* t1;             // [n+1]
  int32_t* item_of_row;    // [n]
  int32_t* reps;           // [n]
  int32_t* item_size;      // [n]
  int64_t* item_ptr;       // [n+1]
  int32_t* item_seg;       // [nnz]
  int64_t* post_ptr;       // [n_seg+1]
  int32_t* post_item;      // [nnz]
  int32_t* seg_cnt;        // [n_seg+1]
  int32_t* empties;        // [n]
  int32_t* n_empty;        // [1]
  int32_t* group_of_item;  // [n]
  int32_t* stamp;          // [n]
  int32_t* sstamp;         // [n] speculative-test dedupe stamps
  int32_t* cand_j;         // [3*n]
  uint8_t* cand_ok;        // [3*n]
  int32_t* seed_item;      // [n]
  int32_t* ctrl;           // [16 + 4*blocks]
  int64_t* htotal;         // [blocks] candidate-set sizes of the punted seeds of a batch
  unsigned long long* stats;  // [8]
  int32_t* scratch;        // [blocks * 3 * (n_seg+1)]
  int64_t* pcnt;           // [n+1]
  int32_t* b32;            // [n_seg+1]
  void* cub_tmp;
  size_t cub_bytes;
  size_t total;
};

constexpr int kSparseBlocks = 148;
constexpr int kSparseThreads = 512;

size_t sparse_cub_bytes(int64_t n, int64_t nnz, int64_t n_seg) {
  const int nn = (int)std::max<int64_t>(n + 1, 2), ee = (int)std::max<int64_t>(nnz + 1, 2);
  size_t a = 0, b = 0, c = 0, d = 0, e = 0, f = 0, g = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, nn);
  cub::DeviceRadixSort::SortKeys(nullptr, b, (unsigned long long*)nullptr, (unsigned long long*)nullptr, ee);
  cub::DeviceScan::ExclusiveSum(nullptr, c, (int32_t*)nullptr, (int32_t*)nullptr, nn);
  cub::DeviceScan::ExclusiveSum(nullptr, d, (int64_t*)nullptr, (int64_t*)nullptr, std::max(nn, (int)(n_seg + 2)));
  cub::DeviceScan::InclusiveScan(nullptr, e, (int32_t*)nullptr, (int32_t*)nullptr, MaxOp(), nn);
  cub::DeviceSelect::Unique(nullptr, f, (unsigned long long*)nullptr, (unsigned long long*)nullptr, (int*)nullptr, ee);
  cub::DeviceScan::ExclusiveSum(nullptr, g, (int32_t*)nullptr, (int64_t*)nullptr, std::max(nn, (int)(n_seg + 2)));
  return std::max({a, b, c, d, e, f, g});
}

SWs carve_sparse(void* base, int64_t n, int64_t nnz, int64_t n_seg) {
  SWs w;
  size_t off = 0;
  const int64_t n1 = std::max<int64_t>(n, 1), e1 = std::max<int64_t>(nnz, 1), s1 = n_seg + 1;
  auto take = [&](size_t bytes) {
    void* p = base ? static_cast<char*>(base) + off : nullptr;
    off += align256(bytes);
    return p;
  };
  w.sizes = (int32_t*)take(4 * n1);
  w.rs_ptr = (int64_t*)take(8 * (n1 + 1));
  w.rs = (int32_t*)take(4 * e1);
  w.keys_a = (unsigned long long*)take(8 * std::max(n1, e1));
  w.keys_b = (unsigned long long*)take(8 * std::max(n1, e1));
  w.vals_a = (int32_t*)take(4 * (n1 + 1));
  w.vals_b = (int32_t*)take(4 * (n1 + 1));
  w.t0 = (int32_t*)take(4 * (n1 + 1));
  w.t1 = (int32_t*)take(4 * (n1 + 1));
  w.item_of_row = (int32_t*)take(4 * n1);
  w.reps = (int32_t*)take(4 * n1);
  w.item_size = (int32_t*)take(4 * (n1 + 1));
  w.item_ptr = (int64_t*)take(8 * (n1 + 1));
  w.item_seg = (int32_t*)take(4 * e1);
  w.post_ptr = (int64_t*)take(8 * (s1 + 1));
  w.post_item = (int32_t*)take(4 * e1);
  w.seg_cnt = (int32_t*)take(4 * (s1 + 1));
  w.empties = (int32_t*)take(4 * n1);
  w.n_empty = (int32_t*)take(16);
  w.group_of_item = (int32_t*)take(4 * n1);
  w.stamp = (int32_t*)take(4 * n1);
  w.sstamp = (int32_t*)take(4 * n1);
  w.cand_j = (int32_t*)take(4 * 3 * n1);
  w.cand_ok = (uint8_t*)take(3 * n1);
  w.seed_item = (int32_t*)take(4 * n1);
  w.ctrl = (int32_t*)take(4 * (16 + 4 * kSparseBlocks));
  w.htotal = (int64_t*)take(8 * kSparseBlocks);
  w.stats = (unsigned long long*)take(8 * 24);
  w.scratch = (int32_t*)take(4 * (size_t)kSparseBlocks * 3 * (s1 + 1));
  w.pcnt = (int64_t*)take(8 * (n1 + 1));
  w.b32 = (int32_t*)take(4 * s1);
  w.cub_bytes = sparse_cub_bytes(n, nnz, n_seg);
  w.cub_tmp = take(w.cub_bytes);
  w.total = off;
  return w;
}

// warp per row: number of segment runs (= quotient pattern size, blocking.py:135)
__global__ void seg_count_kernel(const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col_idx, int64_t n,
                                 SegMap seg, int32_t* sizes) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const int64_t s0 = row_ptr[r], s1 = row_ptr[r + 1];
    int cnt = 0;
    for (int64_t j = s0 + lane; j < s1; j += 32)
      cnt += (j == s0 || seg((int32_t)col_idx[j - 1]) != seg((int32_t)col_idx[j])) ? 1 : 0;
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) sizes[r] = cnt;
  }
}

// warp per row: ascending unique segment list of the row (the quotient row, blocking.py:118-136)
__global__ void seg_write_kernel(const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col_idx, int64_t n,
                                 SegMap seg, const int64_t* __restrict__ rs_ptr, int32_t* rs) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const int64_t s0 = row_ptr[r], s1 = row_ptr[r + 1];
    int64_t out = rs_ptr[r];
    for (int64_t j0 = s0; j0 < s1; j0 += 32) {
      const int64_t j = j0 + lane;
      int32_t sg = 0;
      bool flag = false;
      if (j < s1) {
        sg = seg((int32_t)col_idx[j]);
        flag = (j == s0) || seg((int32_t)col_idx[j - 1]) != sg;
      }
      const unsigned b = __ballot_sync(0xffffffffu, flag);
      if (flag) rs[out + __popc(b & ((1u << lane) - 1u))] = sg;
      out += __popc(b);
    }
  }
}

__global__ void list_hash_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ lst, int64_t n,
                                 unsigned long long* keys, int32_t* vals) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long h = 0x9E3779B97F4A7C15ull ^ (unsigned long long)(ptr[r + 1] - ptr[r]);
    for (int64_t p = ptr[r]; p < ptr[r + 1]; ++p) h = mix64(h ^ (0x632BE59BD9B4E019ull * (unsigned long long)(lst[p] + 1)));
    keys[r] = h;
    vals[r] = (int32_t)r;
  }
}

__device__ __forceinline__ bool lists_equal(const int64_t* ptr, const int32_t* lst, int32_t a, int32_t b) {
  const int64_t la = ptr[a + 1] - ptr[a];
  if (la != ptr[b + 1] - ptr[b]) return false;
  for (int64_t k = 0; k < la; ++k)
    if (lst[ptr[a] + k] != lst[ptr[b] + k]) return false;
  return true;
}

__global__ void list_rep_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ lst,
                                const int32_t* __restrict__ rows_sorted, const int32_t* __restrict__ run_start,
                                int64_t n, int32_t* rep_of_row) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows_sorted[p];
    int32_t rep = r;
    for (int64_t q = run_start[p]; q < p; ++q) {
      const int32_t c = rows_sorted[q];
      if (lists_equal(ptr, lst, c, r)) {
        rep = c;
        break;
      }
    }
    rep_of_row[r] = rep;
  }
}

__global__ void item_size_kernel(const int32_t* __restrict__ reps, const int32_t* __restrict__ sizes, int64_t m,
                                 int32_t* item_size, int32_t* group_of_item, int32_t* stamp) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    item_size[j] = sizes[reps[j]];
    group_of_item[j] = -1;
    stamp[j] = -1;
  }
}

// warp per item: copy the representative row's segment list; histogram segment frequencies
__global__ void item_lists_kernel(const int32_t* __restrict__ reps, const int64_t* __restrict__ rs_ptr,
                                  const int32_t* __restrict__ rs, const int64_t* __restrict__ item_ptr, int64_t m,
                                  int32_t* item_seg, int32_t* seg_cnt, unsigned long long* pkeys) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); j < m; j += warps) {
    const int32_t r = reps[j];
    const int64_t src = rs_ptr[r], len = rs_ptr[r + 1] - src, dst = item_ptr[j];
    for (int64_t k = lane; k < len; k += 32) {
      const int32_t s = rs[src + k];
      item_seg[dst + k] = s;
      atomicAdd(seg_cnt + s, 1);
      pkeys[dst + k] = ((unsigned long long)s << 32) | (unsigned long long)(uint32_t)j;  // postings sort key
    }
  }
}

__global__ void postings_kernel(const unsigned long long* __restrict__ pkeys_sorted, int64_t E, int32_t* post_item) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    post_item[e] = (int32_t)(pkeys_sorted[e] & 0xffffffffull);
}

__global__ void empties_kernel(const int32_t* __restrict__ item_size, int64_t m, int32_t* empties, int32_t* n_empty) {
  // single block: ascending list of empty items (blocking.py: an empty pattern accepts only empty rows)
  __shared__ int32_t base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t j0 = 0; j0 < m; j0 += blockDim.x) {
    const int64_t j = j0 + threadIdx.x;
    const bool e = j < m && item_size[j] == 0;
    const unsigned b = __ballot_sync(0xffffffffu, e);
    __shared__ int32_t wcnt[32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) wcnt[w] = __popc(b);
    __syncthreads();
    int off = base;
    for (int k = 0; k < w; ++k) off += wcnt[k];
    if (e) empties[off + __popc(b & ((1u << lane) - 1u))] = (int32_t)j;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) tot += wcnt[k];
      base += tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_empty = base;
}

struct SGreedyArgs {
  int32_t m, n_seg, W;
  const int64_t* item_ptr;
  const int32_t* item_seg;
  const int32_t* item_size;
  const int64_t* post_ptr;
  const int32_t* post_item;
  const int32_t* empties;
  const int32_t* n_empty;
  double tau;
  int32_t cosine, bounded, update;
  int32_t* group_of_item;
  int32_t* stamp;
  int32_t* sstamp;   // [m] speculative tests: id of the last (batch, seed) test that claimed the item
  int32_t* cand_j;   // [3][m]
  uint8_t* cand_ok;  // [3][m]
  int32_t* seed_item;
  int32_t* ctrl;     // [0..2] first growing hit, [3..5] candidate counts, [6] H, [8] count, [9] gen,
                     // [10..12] accepted-candidate counts, [16..16+2*kSparseBlocks) speculative flags,
                     // [16+2*kSparseBlocks..16+4*kSparseBlocks) HEAVY verdicts of punted seeds
  int32_t* scratch;  // per block: overflow of the pattern list arrays, 3 x (n_seg+1)
  unsigned long long* stats;  // [8] counters (block 0): batches, batch seeds, singletons, rounds, accepts,
                              //     cycles in BATCH, cycles in GROUP, HEAVY passes
  int64_t batch_max_enum;
  int64_t* htotal;   // [kSparseBlocks] candidate-set size of each punted seed of the current batch
  int32_t heavy;     // resolve punted seeds with all CTAs in one pass (HEAVY phase)
  int64_t heavy_max_enum;  // entries one HEAVY pass may enumerate (the punted seeds that fit, in order)
};

constexpr int kPlistSmem = 4096;
// A speculative CTA enumerates at most batch_max_enum candidate entries (SGreedyArgs); larger
// candidate sets go to the all-CTA GROUP round.  24 x 512 measured best on config 3 (R-MAT 2^20):
// tau 0.7 3.60 -> 2.08 s, 0.3 6.51 -> 5.95 s vs 4 x 512 (RB_1SA_BATCH_ENUM overrides).
constexpr int64_t kBatchMaxEnumDefault = 24 * kSparseThreads;
// A HEAVY pass resolves, in batch order, the punted seeds whose candidate sets fit this many entries
// in total (the rest still go to GROUP rounds).  A hit on seed k stops the work on every later seed.
constexpr int64_t kHeavyMaxEnumDefault = 2 << 20;

// The pattern's segment list and its prefix-enumeration arrays (start, exclusive-scan of lengths).
struct PList {
  int32_t* sm;  // [3][kPlistSmem]
  int32_t* gm;  // [3][n1]
  int32_t n1;
  __device__ __forceinline__ int32_t& seg(int32_t q) { return q < kPlistSmem ? sm[q] : gm[q]; }
  __device__ __forceinline__ int32_t& scan(int32_t q) { return q < kPlistSmem ? sm[kPlistSmem + q] : gm[n1 + q]; }
  __device__ __forceinline__ int32_t& start(int32_t q) {
    return q < kPlistSmem ? sm[2 * kPlistSmem + q] : gm[2 * n1 + q];
  }
};

// block-wide exclusive scan of pl.scan(0..n), returns the total
__device__ int32_t block_scan_plist(PList& pl, int32_t n, int32_t* smem_w /*[32]*/, int32_t* smem_carry) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) *smem_carry = 0;
  __syncthreads();
  for (int32_t base = 0; base < n; base += blockDim.x) {
    const int32_t i = base + threadIdx.x;
    const int32_t x = i < n ? pl.scan(i) : 0;
    int32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) smem_w[w] = incl;
    __syncthreads();
    if (w == 0) {
      int32_t t = lane < nw ? smem_w[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      if (lane < nw) smem_w[lane] = t;
    }
    __syncthreads();
    const int32_t carry = *smem_carry;
    if (i < n) pl.scan(i) = carry + (w > 0 ? smem_w[w - 1] : 0) + incl - x;
    __syncthreads();
    if (threadIdx.x == 0) *smem_carry = carry + smem_w[nw - 1];
    __syncthreads();
  }
  return *smem_carry;
}

struct BlockShared {
  int32_t w[32], carry, hist[33], bstar, T, flag;
};

// Replace the block's pattern (bits in sP + list in pl) by item `it`'s segments; returns its size.
__device__ int32_t load_pattern(const SGreedyArgs& a, unsigned long long* sP, PList& pl, int32_t old_psize,
                                int32_t it) {
  for (int32_t q = threadIdx.x; q < old_psize; q += blockDim.x) {
    const int32_t sg = pl.seg(q);
    atomicAnd(&sP[sg >> 6], ~(1ull << (sg & 63)));
  }
  __syncthreads();
  const int64_t p0 = a.item_ptr[it];
  const int32_t len = (int32_t)(a.item_ptr[it + 1] - p0);
  for (int32_t k = threadIdx.x; k < len; k += blockDim.x) {
    const int32_t sg = a.item_seg[p0 + k];
    pl.seg(k) = sg;
    atomicOr(&sP[sg >> 6], 1ull << (sg & 63));
  }
  __syncthreads();
  return len;
}

// Enumeration set of one round: 0 = prefix postings, 1 = empty items, 2 = all items >= pos.
// For mode 0 fills pl.start / pl.scan and returns the number of enumerated postings entries.
__device__ int64_t prepare_round(const SGreedyArgs& a, PList& pl, BlockShared& bs, int32_t psize, int32_t pos,
                                 int* mode_out, int32_t* emp_lo_out) {
  const double tau = a.tau;
  int32_t t;
  if (!a.cosine) t = (int32_t)ceil(__dmul_rn(tau, (double)psize));
  else t = (int32_t)ceil(__dmul_rn(__dmul_rn(__dmul_rn(tau, tau), (double)psize), 1.0 - 1e-12));
  const int mode = (t >= 1 && psize > 0) ? 0 : (psize == 0 && tau > 0.0) ? 1 : 2;
  *mode_out = mode;
  *emp_lo_out = 0;
  if (mode == 2) return a.m - pos;
  if (mode == 1) {
    int32_t lo = 0, hi = __ldg(a.n_empty);
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (a.empties[mid] < pos) lo = mid + 1;
      else hi = mid;
    }
    *emp_lo_out = lo;
    return __ldg(a.n_empty) - lo;
  }
  if (threadIdx.x < 33) bs.hist[threadIdx.x] = 0;
  __syncthreads();
  for (int32_t q = threadIdx.x; q < psize; q += blockDim.x) {
    const int32_t sg = pl.seg(q);
    const int64_t len = a.post_ptr[sg + 1] - a.post_ptr[sg];
    atomicAdd(&bs.hist[63 - __clzll((long long)(len > 1 ? len : 1))], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int32_t npre = psize - t + 1;
    int32_t cum = 0, b = 0;
    for (; b < 33; ++b) {
      cum += bs.hist[b];
      if (cum >= npre) break;
    }
    bs.bstar = b;
  }
  __syncthreads();
  const int32_t bstar = bs.bstar;
  for (int32_t q = threadIdx.x; q < psize; q += blockDim.x) {  // thread per pattern segment
    const int32_t sg = pl.seg(q);
    const int64_t lo0 = a.post_ptr[sg], hi0 = a.post_ptr[sg + 1];
    int32_t rem = 0, st = 0;
    if (63 - __clzll((long long)((hi0 - lo0) > 1 ? (hi0 - lo0) : 1)) <= bstar) {
      int64_t lo = lo0, hi = hi0;  // first posting >= pos
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(a.post_item + mid) < pos) lo = mid + 1;
        else hi = mid;
      }
      st = (int32_t)lo;
      rem = (int32_t)(hi0 - lo);
    }
    pl.start(q) = st;
    pl.scan(q) = rem;
  }
  __syncthreads();
  const int32_t T = block_scan_plist(pl, psize, bs.w, &bs.carry);
  if (threadIdx.x == 0) bs.T = T;
  __syncthreads();
  return bs.T;
}

__device__ __forceinline__ int32_t entry_item(const SGreedyArgs& a, PList& pl, int mode, int32_t psize, int64_t e,
                                              int32_t pos, int32_t emp_lo) {
  if (mode == 0) {
    int32_t lo = 0, hi = psize;  // last q with scan(q) <= e
    while (hi - lo > 1) {
      const int32_t mid = (lo + hi) >> 1;
      if (pl.scan(mid) <= e) lo = mid;
      else hi = mid;
    }
    return a.post_item[pl.start(lo) + (e - pl.scan(lo))];
  }
  if (mode == 1) return a.empties[emp_lo + e];
  return pos + (int32_t)e;
}

// |P ∩ segs(j)| with the pattern bits in shared memory; loads issued 8 at a time.
__device__ __forceinline__ int64_t item_inter(const SGreedyArgs& a, const unsigned long long* sP, int64_t p0,
                                              int64_t p1) {
  int64_t inter = 0;
  int64_t p = p0;
  for (; p + 8 <= p1; p += 8) {
    int32_t sg[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) sg[k] = __ldg(a.item_seg + p + k);
#pragma unroll
    for (int k = 0; k < 8; ++k) inter += (sP[sg[k] >> 6] >> (sg[k] & 63)) & 1ull;
  }
  for (; p < p1; ++p) {
    const int32_t sg = __ldg(a.item_seg + p);
    inter += (sP[sg >> 6] >> (sg & 63)) & 1ull;
  }
  return inter;
}

// Candidates with more segments than this are intersected by a whole warp (deferred through a
// shared queue), so one thread never walks a hub item's long list alone while the block (and, in a
// GROUP round, the grid barrier) waits for it.
constexpr int64_t kWarpItem = 32;

// warp-cooperative |P ∩ segs(j)| (all lanes return the total)
__device__ __forceinline__ int64_t warp_item_inter(const SGreedyArgs& a, const unsigned long long* sP, int64_t p0,
                                                   int64_t p1) {
  const int lane = threadIdx.x & 31;
  int cnt = 0;
  for (int64_t p = p0 + lane; p < p1; p += 32) {
    const int32_t sg = __ldg(a.item_seg + p);
    cnt += (int)((sP[sg >> 6] >> (sg & 63)) & 1ull);
  }
  return (int64_t)__reduce_add_sync(0xffffffffu, cnt);
}

// Merge verdict for candidate j.  accept_dev is non-decreasing in inter and inter <= min(psize, size),
// so a candidate that fails even with inter = min(psize, size) is rejected without reading its list.
// Returns 1 = accepted, 0 = rejected, -1 = deferred (passes the size pre-check and has more than
// kWarpItem segments: the caller queues it for warp_eval).
__device__ __forceinline__ int eval_candidate(const SGreedyArgs& a, const unsigned long long* sP, int32_t j,
                                              int64_t psize, double cap, bool* grows) {
  const int64_t p0 = __ldg(a.item_ptr + j), p1 = __ldg(a.item_ptr + j + 1);
  const int64_t sz = p1 - p0;
  *grows = false;
  if (!accept_dev(min(psize, sz), psize, sz, a.tau, a.cosine, a.bounded, cap)) return 0;
  if (sz > kWarpItem) return -1;
  const int64_t inter = item_inter(a, sP, p0, p1);
  const bool ok = accept_dev(inter, psize, sz, a.tau, a.cosine, a.bounded, cap);
  *grows = ok && a.update && inter < sz;
  return ok ? 1 : 0;
}

// Warp verdict for a deferred candidate (all lanes get the same answer).
__device__ __forceinline__ bool warp_eval(const SGreedyArgs& a, const unsigned long long* sP, int32_t j,
                                          int64_t psize, double cap, bool* grows) {
  const int64_t p0 = __ldg(a.item_ptr + j), p1 = __ldg(a.item_ptr + j + 1);
  const int64_t sz = p1 - p0;
  const int64_t inter = warp_item_inter(a, sP, p0, p1);
  const bool ok = accept_dev(inter, psize, sz, a.tau, a.cosine, a.bounded, cap);
  *grows = ok && a.update && inter < sz;
  return ok;
}

// Speculative test of a seed over its enumeration entries [e_lo, e_hi): bs.flag becomes 1 at the
// first accepted candidate (bs.flag must be 0 on entry).  `stop` (optional) is polled every
// iteration: another CTA already found a hit for this seed.
// Returns true iff this CTA itself found an accepted candidate.
__device__ bool spec_enumerate(const SGreedyArgs& a, const unsigned long long* sP, PList& pl, BlockShared& bs,
                               int mode, int32_t psize, int32_t pos, int32_t emp_lo, double cap, int64_t e_lo,
                               int64_t e_hi, int32_t* s_defer, int32_t* s_ndefer, int32_t sid,
                               const int32_t* stop, const int32_t* stop_min = nullptr, int32_t my_k = 0) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) *s_ndefer = 0;
  __syncthreads();
  for (int64_t e0 = e_lo; e0 < e_hi; e0 += blockDim.x) {
    const int64_t e = e0 + threadIdx.x;
    if (e < e_hi) {
      const int32_t j = entry_item(a, pl, mode, psize, e, pos, emp_lo);
      // an item listed under several prefix segments is tested once per (batch, seed): `sid`
      if (__ldcg(a.group_of_item + j) < 0 && (mode == 2 || atomicExch(a.sstamp + j, sid) != sid)) {
        bool grows;
        const int v = eval_candidate(a, sP, j, psize, cap, &grows);
        if (v > 0) bs.flag = 1;
        else if (v < 0) s_defer[atomicAdd(s_ndefer, 1)] = j;
      }
    }
    __syncthreads();
    const int32_t nd = *s_ndefer;
    const bool hit = bs.flag != 0;
    __syncthreads();  // the reads above complete before the warp verdicts below may set the flag
    if (!hit && nd > 0) {
      for (int32_t k = threadIdx.x >> 5; k < nd; k += blockDim.x >> 5) {
        bool grows;
        if (warp_eval(a, sP, s_defer[k], psize, cap, &grows) && lane == 0) atomicExch(&bs.flag, 1);
      }
    }
    // stop early (flag 3, not a hit of ours): another CTA found a hit for this seed or an earlier one.
    // CAS so that a hit (1) set concurrently by a warp verdict above is never overwritten.
    if (threadIdx.x == 0 && !hit && stop &&
        (*((volatile const int32_t*)stop) || (stop_min && *((volatile const int32_t*)stop_min) < my_k)))
      atomicCAS(&bs.flag, 0, 3);
    __syncthreads();
    const int32_t f = bs.flag;  // every thread reads the flag of this iteration ...
    if (threadIdx.x == 0) *s_ndefer = 0;
    __syncthreads();  // ... before any thread can set it again in the next one (racecheck hazard)
    if (f) break;     // uniform
  }
  __syncthreads();
  const bool found = bs.flag == 1;
  __syncthreads();
  return found;
}

// The greedy scan with speculative singleton batching (exact):
//  BATCH: every CTA b takes the b-th unassigned item >= next as a speculative seed and tests whether
//         ANY later unassigned item passes the merge test against it.  Seeds before the first one that
//         has a hit are singleton groups in the sequential scan too (a singleton assigns only itself,
//         which is not a candidate of any later seed), so they are committed in order at once.
//  GROUP: the first seed with a hit runs the round protocol with all CTAs: enumerate + evaluate the
//         candidates, reduce the first growing hit, accept the ok items before it, grow, repeat.
__global__ void __launch_bounds__(kSparseThreads) sparse_greedy_kernel(SGreedyArgs a) {
  extern __shared__ unsigned long long smem_dyn[];
  unsigned long long* sP = smem_dyn;                                     // W words
  int32_t* pl_sm = reinterpret_cast<int32_t*>(smem_dyn + a.W);           // 3 * kPlistSmem
  __shared__ BlockShared bs;
  __shared__ int32_t s_list[kSparseBlocks];
  __shared__ int32_t s_list_len, s_f, s_js;
  __shared__ int32_t s_mode, s_next, s_gnext, s_seed, s_g, s_pos, s_psize, s_rid, s_batch;
  __shared__ int32_t s_acc_list, s_acc_cnt, s_acc_limit, s_acc_g;
  __shared__ int32_t s_defer[kSparseThreads], s_ndefer;  // large candidates for warp_eval
  __shared__ int64_t s_pre[kSparseBlocks + 1];            // HEAVY: prefix of the punted totals
  __shared__ int32_t s_f1, s_fh;  // first definite hit of the batch; end of the HEAVY-resolved prefix
  __shared__ int32_t s_bpos, s_blen, s_grounds;  // batch cursor / length, rounds of the current group
  __shared__ double s_cap;

  PList pl{pl_sm, a.scratch + (size_t)blockIdx.x * 3 * (a.n_seg + 1), a.n_seg + 1};
  const int32_t m = a.m;
  const double tau = a.tau;
  const double cap_den = __dsub_rn(1.0, __dmul_rn(0.5, tau));
  const int lane = threadIdx.x & 31;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;

  for (int w = threadIdx.x; w < a.W; w += blockDim.x) sP[w] = 0ull;
  if (threadIdx.x == 0) {
    s_mode = 0;
    s_next = 0;
    s_gnext = 0;
    s_psize = 0;
    s_rid = 0;
    s_batch = 0;
    s_acc_cnt = 0;
    s_bpos = 0;
    s_blen = 0;
    s_grounds = 0;
  }
  __syncthreads();

  long long t_phase = clock64();
  for (;;) {
    if (s_mode == 0) {
      // ============================ BATCH phase
      t_phase = clock64();
      if (threadIdx.x < 32) {
        int32_t cnt = 0;
        for (int32_t j0 = s_next; j0 < m && cnt < (int32_t)gridDim.x; j0 += 32) {
          const int32_t j = j0 + lane;
          const bool un = j < m && __ldcg(a.group_of_item + j) < 0;
          const unsigned b = __ballot_sync(0xffffffffu, un);
          const int32_t r = __popc(b & ((1u << lane) - 1u));
          if (un && cnt + r < (int32_t)gridDim.x) s_list[cnt + r] = j;
          cnt += __popc(b);
        }
        if (lane == 0) s_list_len = min(cnt, (int32_t)gridDim.x);
      }
      __syncthreads();
      const int32_t len = s_list_len;
      if (len == 0) break;
      const int32_t batch = s_batch;
      int32_t* flags = a.ctrl + 16 + (batch & 1) * kSparseBlocks;
      int32_t* hres = a.ctrl + 16 + (2 + (batch & 1)) * kSparseBlocks;
      int32_t* hmin = a.ctrl + 13 + (batch & 1);  // earliest seed index with a HEAVY hit
      if (blockIdx.x == 0 && threadIdx.x == 0) *hmin = INT_MAX;
      const int32_t my = (int32_t)blockIdx.x < len ? s_list[blockIdx.x] : -1;
      if (my >= 0) {
#ifdef RB_PROF_1SA
        const long long c0 = clock64();
#endif
        const int32_t psize = load_pattern(a, sP, pl, s_psize, my);
        if (threadIdx.x == 0) {
          s_psize = psize;
          bs.flag = 0;
        }
        __syncthreads();
#ifdef RB_PROF_1SA
        const long long c1 = clock64();
#endif
        const double cap = __ddiv_rn((double)psize, cap_den);
        int mode;
        int32_t emp_lo;
        const int64_t total = prepare_round(a, pl, bs, psize, my + 1, &mode, &emp_lo);
#ifdef RB_PROF_1SA
        const long long c2 = clock64();
#endif
        // a seed with a large candidate set is not tested by one CTA: it is punted (flag 2) and, if it
        // precedes the batch's first definite hit, resolved by the HEAVY pass below with all CTAs
        if (total > a.batch_max_enum) {
          if (threadIdx.x == 0) {
            a.htotal[blockIdx.x] = total;
            hres[blockIdx.x] = 0;
            flags[blockIdx.x] = 2;
          }
        } else {
          spec_enumerate(a, sP, pl, bs, mode, psize, my + 1, emp_lo, cap, 0, total, s_defer, &s_ndefer,
                         batch * kSparseBlocks + (int32_t)blockIdx.x + 1, nullptr);
          if (threadIdx.x == 0) flags[blockIdx.x] = bs.flag;
        }
#ifdef RB_PROF_1SA
        if (threadIdx.x == 0) {
          const long long c3 = clock64();
          atomicAdd(a.stats + 8, (unsigned long long)(c1 - c0));
          atomicAdd(a.stats + 9, (unsigned long long)(c2 - c1));
          atomicAdd(a.stats + 10, (unsigned long long)(c3 - c2));
          atomicAdd(a.stats + 11, (unsigned long long)total);
          atomicMax(a.stats + 12 + (batch & 1), (unsigned long long)(c3 - t_phase));
          atomicMax(a.stats + 16 + (batch & 1), (unsigned long long)psize);
          if (total > a.batch_max_enum) atomicAdd(a.stats + 15, 1ull);
        }
#endif
      }
#ifdef RB_PROF_1SA
      const long long cb = clock64();
#endif
      grid_barrier(a.ctrl + 8, a.ctrl + 9);
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.stats[0] += 1;
        a.stats[1] += len;
        a.stats[5] += clock64() - t_phase;
#ifdef RB_PROF_1SA
        a.stats[14] += a.stats[12 + (batch & 1)];
        a.stats[12 + (batch & 1)] = 0;
        a.stats[18] += clock64() - cb;
        a.stats[19] += a.stats[16 + (batch & 1)];
        a.stats[16 + (batch & 1)] = 0;
#endif
      }
      // ============================ HEAVY: the punted seeds before the first definite hit, all
      // candidate sets concatenated and cut evenly over the CTAs (one pass, one barrier)
      if (threadIdx.x == 0) s_f1 = len;
      __syncthreads();
      for (int32_t k = threadIdx.x; k < len; k += blockDim.x)
        if (*((volatile const int32_t*)(flags + k)) == 1) atomicMin(&s_f1, k);
      __syncthreads();
      const int32_t f1 = s_f1;
      {
        // s_pre[k] = exclusive prefix of the punted totals (k < f1), s_pre[len] = total
        for (int32_t k = threadIdx.x; k < kSparseBlocks + 1; k += blockDim.x) s_pre[k] = 0;
        __syncthreads();
        if (a.heavy)
          for (int32_t k = threadIdx.x; k < f1; k += blockDim.x)
            if (*((volatile const int32_t*)(flags + k)) == 2) s_pre[k + 1] = __ldcg(a.htotal + k);
        __syncthreads();
        if (threadIdx.x == 0) {  // include punted seeds in order while the pass stays within budget
          int32_t fh = f1;
          for (int32_t k = 1; k <= len; ++k) {
            if (k - 1 >= fh || s_pre[k - 1] + s_pre[k] > a.heavy_max_enum) {
              if (k - 1 < fh && s_pre[k] > 0) fh = k - 1;
              s_pre[k] = s_pre[k - 1];
            } else {
              s_pre[k] += s_pre[k - 1];
            }
          }
          s_fh = fh;
        }
        __syncthreads();
      }
      const int64_t T_all = s_pre[len];
      if (T_all > 0) {
        const int64_t c_lo = T_all * blockIdx.x / gridDim.x, c_hi = T_all * (blockIdx.x + 1) / gridDim.x;
        for (int32_t k = 0; k < s_fh; ++k) {  // block-uniform
          const int64_t k_lo = s_pre[k], k_hi = s_pre[k + 1];
          if (k_hi <= k_lo || k_hi <= c_lo || k_lo >= c_hi) continue;
          // another CTA may set hres[k] at any time: one thread reads it, the block follows
          if (threadIdx.x == 0)
            bs.flag = *((volatile const int32_t*)(hres + k)) || *((volatile const int32_t*)hmin) < k;
          __syncthreads();
          const bool done = bs.flag != 0;
          __syncthreads();
          if (done) continue;
          const int32_t seed = s_list[k];
          const int32_t psize = load_pattern(a, sP, pl, s_psize, seed);
          if (threadIdx.x == 0) {
            s_psize = psize;
            bs.flag = 0;
          }
          __syncthreads();
          const double cap = __ddiv_rn((double)psize, cap_den);
          int mode;
          int32_t emp_lo;
          prepare_round(a, pl, bs, psize, seed + 1, &mode, &emp_lo);
          if (threadIdx.x == 0) bs.flag = 0;
          __syncthreads();
          const bool found = spec_enumerate(a, sP, pl, bs, mode, psize, seed + 1, emp_lo, cap,
                                            max(c_lo, k_lo) - k_lo, min(c_hi, k_hi) - k_lo, s_defer, &s_ndefer,
                                            batch * kSparseBlocks + k + 1, hres + k, hmin, k);
          if (threadIdx.x == 0 && found) {
            hres[k] = 1;
            atomicMin(hmin, k);
          }
        }
        grid_barrier(a.ctrl + 8, a.ctrl + 9);
        if (blockIdx.x == 0 && threadIdx.x == 0) a.stats[7] += 1;
        // the earliest resolved hit ends the resolved prefix: seeds after it may have been cut short
        if (threadIdx.x == 0) {
          const int32_t hm = *((volatile const int32_t*)hmin);
          if (hm != INT_MAX) s_fh = min(s_fh, hm + 1);
        }
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        s_bpos = 0;
        s_blen = len;
        s_batch = batch + 1;
        s_mode = 2;
      }
      __syncthreads();
    }
    if (s_mode == 2) {
      // ============================ consume the batch verdicts from s_bpos (no barrier needed: every
      // CTA reads the same flags and commits nothing that any CTA reads again)
      const int32_t len = s_blen, bpos = s_bpos;
      const int32_t* flags = a.ctrl + 16 + ((s_batch - 1) & 1) * kSparseBlocks;
      const int32_t* hres = a.ctrl + 16 + (2 + ((s_batch - 1) & 1)) * kSparseBlocks;
      const int32_t f1 = s_fh;  // punted seeds before this index were resolved by the HEAVY pass
      if (threadIdx.x < 32) {
        int32_t f = len;
        for (int32_t k0 = bpos; k0 < len; k0 += 32) {
          const int32_t k = k0 + lane;
          int32_t v = k < len ? *((volatile const int32_t*)(flags + k)) : 0;
          // a punted seed before the first definite hit was resolved by the HEAVY pass (if enabled)
          if (v == 2 && a.heavy && k < f1) v = *((volatile const int32_t*)(hres + k));
          const bool hit = v != 0;
          const unsigned b = __ballot_sync(0xffffffffu, hit);
          if (b) {
            f = k0 + __ffs(b) - 1;
            break;
          }
        }
        if (lane == 0) s_f = f;
      }
      __syncthreads();
      const int32_t f = s_f, g0 = s_gnext;
      if (blockIdx.x == 0) {  // singletons before the first hit (nobody reads items < the next seed again)
        for (int32_t k = bpos + threadIdx.x; k < f; k += blockDim.x) {
          a.group_of_item[s_list[k]] = g0 + (k - bpos);
          a.seed_item[g0 + (k - bpos)] = s_list[k];
        }
        if (threadIdx.x == 0) a.stats[2] += f - bpos;
      }
      __syncthreads();
      if (f == len) {
        if (threadIdx.x == 0) {
          s_gnext = g0 + (f - bpos);
          s_next = s_list[len - 1] + 1;
          s_mode = 0;
        }
        __syncthreads();
        continue;
      }
      // the seed with a hit (or too large to test speculatively) starts a GROUP on all CTAs
      const int32_t seed = s_list[f];
      const int32_t gid = g0 + (f - bpos);
      const int32_t psize = load_pattern(a, sP, pl, s_psize, seed);
      if (threadIdx.x == 0) {
        if (blockIdx.x == 0) {
          a.group_of_item[seed] = gid;
          a.seed_item[gid] = seed;
        }
        s_seed = seed;
        s_g = gid;
        s_gnext = gid + 1;
        s_psize = psize;
        s_cap = __ddiv_rn((double)psize, cap_den);
        s_pos = seed + 1;
        s_acc_cnt = 0;
        s_bpos = f + 1;
        s_grounds = 0;
        s_mode = 1;
      }
      __syncthreads();
      continue;
    }

    // ============================ GROUP: EVAL round (+ acceptance of the previous round)
    t_phase = clock64();
    const int32_t rid = s_rid + 1;
    const int slot = rid % 3;
    const int32_t psize = s_psize, pos = s_pos, g = s_g;
    const double cap = s_cap;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.ctrl[3 + (rid + 1) % 3] = 0;   // candidate list of 2 rounds ago is free again
      a.ctrl[10 + (rid + 1) % 3] = 0;
    }
    if (s_acc_cnt > 0) {
      const int32_t* cj = a.cand_j + (size_t)s_acc_list * m;
      const uint8_t* co = a.cand_ok + (size_t)s_acc_list * m;
      const int32_t lim = s_acc_limit, ag = s_acc_g, cnt = s_acc_cnt;
      for (int64_t i = gtid; i < cnt; i += gthreads) {
        const int32_t j = __ldcg(cj + i);
        if (__ldcg(co + i) && j <= lim) a.group_of_item[j] = ag;
      }
    }
    if (threadIdx.x == 0) s_js = INT_MAX;
    __syncthreads();
    int mode;
    int32_t emp_lo;
    const int64_t total = prepare_round(a, pl, bs, psize, pos, &mode, &emp_lo);
    int32_t my_js = INT_MAX, my_ok = 0;
    {
      int32_t* cj = a.cand_j + (size_t)slot * m;
      uint8_t* co = a.cand_ok + (size_t)slot * m;
      if (threadIdx.x == 0) s_ndefer = 0;
      __syncthreads();
      for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x; e0 < total; e0 += gthreads) {  // uniform per block
        const int64_t e = e0 + threadIdx.x;
        bool has = false, ok = false;
        int32_t j = -1;
        if (e < total) {
          j = entry_item(a, pl, mode, psize, e, pos, emp_lo);
          if (__ldcg(a.group_of_item + j) < 0 && (mode == 2 || atomicExch(a.stamp + j, rid) != rid)) {
            bool grows;
            const int v = eval_candidate(a, sP, j, psize, cap, &grows);
            if (v < 0) {
              s_defer[atomicAdd(&s_ndefer, 1)] = j;
            } else {
              has = true;
              ok = v > 0;
              my_ok += ok ? 1 : 0;
              if (grows) my_js = min(my_js, j);
            }
          }
        }
        const unsigned ball = __ballot_sync(0xffffffffu, has);
        if (ball) {
          int32_t base = 0;
          if (lane == 0) base = atomicAdd(a.ctrl + 3 + slot, __popc(ball));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (has) {
            const int32_t idx = base + __popc(ball & ((1u << lane) - 1u));
            cj[idx] = j;
            co[idx] = ok ? 1 : 0;
          }
        }
        __syncthreads();
        const int32_t nd = s_ndefer;
        for (int32_t k = threadIdx.x >> 5; k < nd; k += blockDim.x >> 5) {  // warp per large candidate
          const int32_t jd = s_defer[k];
          bool grows;
          const bool okd = warp_eval(a, sP, jd, psize, cap, &grows);
          if (lane == 0) {
            const int32_t idx = atomicAdd(a.ctrl + 3 + slot, 1);
            cj[idx] = jd;
            co[idx] = okd ? 1 : 0;
            my_ok += okd ? 1 : 0;
            if (grows) my_js = min(my_js, jd);
          }
        }
        __syncthreads();
        if (threadIdx.x == 0) s_ndefer = 0;
      }
    }
    my_js = __reduce_min_sync(0xffffffffu, my_js);
    my_ok = __reduce_add_sync(0xffffffffu, my_ok);
    if (lane == 0) {
      if (my_js != INT_MAX) atomicMin(&s_js, my_js);
      if (my_ok) atomicAdd(a.ctrl + 10 + slot, my_ok);
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_js != INT_MAX) atomicMin(a.ctrl + slot, s_js);
    grid_barrier(a.ctrl + 8, a.ctrl + 9);

    const int32_t js = *((volatile int32_t*)(a.ctrl + slot));
    const int32_t ccnt = *((volatile int32_t*)(a.ctrl + 3 + slot));
    const int32_t okcnt = *((volatile int32_t*)(a.ctrl + 10 + slot));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.stats[3] += 1;
      a.stats[4] += (js >= m && okcnt > 0) ? 1 : 0;
      a.stats[6] += clock64() - t_phase;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.ctrl[(rid + 2) % 3] = INT_MAX;
    if (threadIdx.x == 0) {
      s_rid = rid;
      s_acc_list = slot;
      s_acc_cnt = ccnt;
      s_acc_g = g;
      s_grounds += 1;
    }
    if (js < m) {
      // growth at js: OR its segments into P, appending new ones to the list in list order
      if (threadIdx.x == 0) {
        const int64_t p0 = a.item_ptr[js], p1 = a.item_ptr[js + 1];
        int32_t ps = psize;
        for (int64_t p = p0; p < p1; ++p) {
          const int32_t sg = a.item_seg[p];
          const unsigned long long bit = 1ull << (sg & 63);
          if (!(sP[sg >> 6] & bit)) {
            sP[sg >> 6] |= bit;
            pl.seg(ps++) = sg;
          }
        }
        s_psize = ps;
        s_pos = js + 1;
        s_acc_limit = js;
      }
      __syncthreads();
      continue;
    }
    // group complete: accept the ok candidates of the last round (only if there are any)
    if (okcnt > 0) {
      const int32_t* cj = a.cand_j + (size_t)slot * m;
      const uint8_t* co = a.cand_ok + (size_t)slot * m;
      for (int64_t i = gtid; i < ccnt; i += gthreads) {
        const int32_t j = __ldcg(cj + i);
        if (__ldcg(co + i)) a.group_of_item[j] = g;
      }
      grid_barrier(a.ctrl + 8, a.ctrl + 9);
    }
    if (threadIdx.x == 0) {
      s_acc_cnt = 0;
      // a singleton group (one round, nothing accepted) leaves the batch's later verdicts valid
      if (s_grounds == 1 && okcnt == 0 && s_bpos < s_blen) {
        s_mode = 2;
      } else {
        s_mode = 0;
        s_next = s_seed + 1;
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.ctrl[6] = s_gnext;
}

// patterns of the sparse path: unique (group, segment) pairs of all member items
__global__ void pattern_pairs_kernel(const int32_t* __restrict__ group_of_item, const int64_t* __restrict__ item_ptr,
                                     const int32_t* __restrict__ item_seg, int64_t m, int64_t n_seg,
                                     unsigned long long* keys) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); j < m; j += warps) {
    const unsigned long long g = (unsigned long long)group_of_item[j];
    for (int64_t p = item_ptr[j] + lane; p < item_ptr[j + 1]; p += 32)
      keys[p] = g * (unsigned long long)n_seg + (unsigned long long)item_seg[p];
  }
}

__global__ void pattern_emit_kernel(const unsigned long long* __restrict__ ukeys, const int* __restrict__ n_unique,
                                    int64_t n_seg, int64_t* pattern_idx, int32_t* gcnt) {
  const int64_t U = *n_unique;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < U; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = ukeys[i];
    pattern_idx[i] = (int64_t)(k % (unsigned long long)n_seg);
    atomicAdd(gcnt + (int64_t)(k / (unsigned long long)n_seg), 1);
  }
}


__global__ void widen_i32_kernel(const int32_t* __restrict__ in, int64_t n, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

int block_1sa_sparse(int64_t n, int64_t nnz, const int64_t* row_ptr, const int64_t* col_idx, const int64_t* boundaries,
                     int64_t n_seg, int32_t delta, double tau, int similarity, int bounded, int pattern_update,
                     int use_compression, void* workspace, size_t ws_bytes, int64_t* group_of, int64_t* row_perm,
                     int64_t* group_ptr, int64_t* seed_size, int64_t* pattern_ptr, int64_t* pattern_idx,
                     int64_t* n_groups, cudaStream_t stream) {
  SWs ws = carve_sparse(workspace, n, nnz, n_seg);
  if (ws_bytes < ws.total) return fail(RB_EINVAL, "workspace too small");
  const int64_t W = words_of(n_seg);
  int rc = narrow_bounds(boundaries, n_seg, ws.b32, stream);
  if (rc) return rc;
  SegMap seg{ws.b32, (int32_t)n_seg, delta};
  const unsigned g1 = grid_for(n, 256);
  size_t tb;
  // ---- K1: row segment lists
  seg_count_kernel<<<grid_for(n, 8), 256, 0, stream>>>(row_ptr, col_idx, n, seg, ws.sizes);
  widen_i32_kernel<<<g1, 256, 0, stream>>>(ws.sizes, n, ws.pcnt);
  RB_CUDA_TRY(cudaMemsetAsync(ws.pcnt + n, 0, sizeof(int64_t), stream));
  tb = ws.cub_bytes;
  RB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws.cub_tmp, tb, ws.pcnt, ws.rs_ptr, (int)(n + 1), stream));
  seg_write_kernel<<<grid_for(n, 8), 256, 0, stream>>>(row_ptr, col_idx, n, seg, ws.rs_ptr, ws.rs);
  RB_CUDA_TRY(cudaGetLastError());
  // ---- K2: compression on the exact lists
  int32_t m = (int32_t)n;
  if (use_compression) {
    list_hash_kernel<<<g1, 256, 0, stream>>>(ws.rs_ptr, ws.rs, n, ws.keys_a, ws.vals_a);
    tb = ws.cub_bytes;
    RB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(ws.cub_tmp, tb, ws.keys_a, ws.keys_b, ws.vals_a, ws.vals_b, (int)n, 0,
                                                64, stream));
    run_head_kernel<<<g1, 256, 0, stream>>>(ws.keys_b, n, ws.t0);
    tb = ws.cub_bytes;
    RB_CUDA_TRY(cub::DeviceScan::InclusiveScan(ws.cub_tmp, tb, ws.t0, ws.t1, MaxOp(), (int)n, stream));
    list_rep_kernel<<<g1, 256, 0, stream>>>(ws.rs_ptr, ws.rs, ws.vals_b, ws.t1, n, ws.t0);
    is_rep_kernel<<<g1, 256, 0, stream>>>(ws.t0, n, ws.t1);
    RB_CUDA_TRY(cudaMemsetAsync(ws.t1 + n, 0, sizeof(int32_t), stream));
    tb = ws.cub_bytes;
    RB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws.cub_tmp, tb, ws.t1, ws.vals_a, (int)(n + 1), stream));
    items_kernel<<<g1, 256, 0, stream>>>(ws.t0, ws.vals_a, n, ws.item_of_row, ws.reps);
    RB_CUDA_TRY(cudaMemcpyAsync(&m, ws.vals_a + n, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    RB_CUDA_TRY(cudaStreamSynchronize(stream));
  } else {
    identity_items_kernel<<<g1, 256, 0, stream>>>(n, ws.item_of_row, ws.reps);
  }
  // ---- item lists + inverted index
  const unsigned gm = grid_for(m, 256);
  item_size_kernel<<<gm, 256, 0, stream>>>(ws.reps, ws.sizes, m, ws.item_size, ws.group_of_item, ws.stamp);
  widen_i32_kernel<<<gm, 256, 0, stream>>>(ws.item_size, m, ws.pcnt);
  RB_CUDA_TRY(cudaMemsetAsync(ws.pcnt + m, 0, sizeof(int64_t), stream));
  tb = ws.cub_bytes;
  RB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws.cub_tmp, tb, ws.pcnt, ws.item_ptr, (int)(m + 1), stream));
  RB_CUDA_TRY(cudaMemsetAsync(ws.seg_cnt, 0, sizeof(int32_t) * (n_seg + 1), stream));
  item_lists_kernel<<<grid_for(m, 8), 256, 0, stream>>>(ws.reps, ws.rs_ptr, ws.rs, ws.item_ptr, m, ws.item_seg,
                                                        ws.seg_cnt, ws.keys_a);
  int64_t E = 0;
  RB_CUDA_TRY(cudaMemcpyAsync(&E, ws.item_ptr + m, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  RB_CUDA_TRY(cudaStreamSynchronize(stream));
  widen_i32_kernel<<<grid_for(n_seg + 1, 256), 256, 0, stream>>>(ws.seg_cnt, n_seg + 1, ws.pcnt);
  tb = ws.cub_bytes;
  RB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws.cub_tmp, tb, ws.pcnt, ws.post_ptr, (int)(n_seg + 1), stream));
  if (E > 0) {
    int end_bit = 32;
    while (end_bit < 64 && ((unsigned long long)n_seg >> (end_bit - 32)) != 0) ++end_bit;
    tb = ws.cub_bytes;
    RB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(ws.cub_tmp, tb, ws.keys_a, ws.keys_b, (int)E, 0, end_bit, stream));
    postings_kernel<<<grid_for(E, 256), 256, 0, stream>>>(ws.keys_b, E, ws.post_item);
  }
  empties_kernel<<<1, 1024, 0, stream>>>(ws.item_size, m, ws.empties, ws.n_empty);
  RB_CUDA_TRY(cudaGetLastError());
  // ---- K3: pruned greedy scan
  {
    std::vector<int32_t> ctrl0(16 + 4 * kSparseBlocks, 0);
    for (int i = 0; i < 3; ++i) ctrl0[i] = INT_MAX;
    RB_CUDA_TRY(cudaMemcpyAsync(ws.ctrl, ctrl0.data(), sizeof(int32_t) * ctrl0.size(), cudaMemcpyHostToDevice, stream));
    SGreedyArgs ga;
    ga.m = m;
    ga.n_seg = (int32_t)n_seg;
    ga.W = (int32_t)W;
    ga.item_ptr = ws.item_ptr;
    ga.item_seg = ws.item_seg;
    ga.item_size = ws.item_size;
    ga.post_ptr = ws.post_ptr;
    ga.post_item = ws.post_item;
    ga.empties = ws.empties;
    ga.n_empty = ws.n_empty;
    ga.tau = tau;
    ga.cosine = similarity == RB_COSINE;
    ga.bounded = bounded != 0;
    ga.update = pattern_update != 0;
    ga.group_of_item = ws.group_of_item;
    ga.stamp = ws.stamp;
    ga.sstamp = ws.sstamp;
    RB_CUDA_TRY(cudaMemsetAsync(ws.sstamp, 0, sizeof(int32_t) * std::max<int64_t>(m, 1), stream));
    ga.cand_j = ws.cand_j;
    ga.cand_ok = ws.cand_ok;
    ga.seed_item = ws.seed_item;
    ga.ctrl = ws.ctrl;
    ga.scratch = ws.scratch;
    ga.stats = ws.stats;
    ga.batch_max_enum = kBatchMaxEnumDefault;
    ga.htotal = ws.htotal;
    ga.heavy = 1;
    if (const char* e = std::getenv("RB_1SA_HEAVY")) ga.heavy = e[0] != '0';
    ga.heavy_max_enum = kHeavyMaxEnumDefault;
    if (const char* e = std::getenv("RB_1SA_HEAVY_ENUM")) ga.heavy_max_enum = std::max<int64_t>(0, std::atoll(e));
    if (const char* e = std::getenv("RB_1SA_BATCH_ENUM")) ga.batch_max_enum = std::max<int64_t>(0, std::atoll(e));
    RB_CUDA_TRY(cudaMemsetAsync(ws.stats, 0, 8 * 24, stream));
    const size_t shm = sizeof(uint64_t) * W + sizeof(int32_t) * 3 * kPlistSmem;
    if (shm > 200 * 1024) return fail(RB_EUNSUPPORTED, "too many segments for the pattern bitset in shared memory");
    void* fn = (void*)sparse_greedy_kernel;
    if (shm > 48 * 1024) RB_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    int blocks = 1;
    if ((int64_t)m * 8 > 64 * 1024 || E > 256 * 1024) {
      int dev = 0, per_sm = 0, sms = 0;
      RB_CUDA_TRY(cudaGetDevice(&dev));
      RB_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      RB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kSparseThreads, shm));
      if (per_sm < 1) return fail(RB_ECUDA, "sparse greedy kernel cannot be resident");
      blocks = std::min(sms, kSparseBlocks);
    }
    if (const char* b = std::getenv("RB_1SA_BLOCKS")) blocks = std::max(1, std::min(std::atoi(b), kSparseBlocks));
    void* args[] = {&ga};
    RB_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kSparseThreads), args, shm, stream));
  }
  int32_t H32 = 0;
  RB_CUDA_TRY(cudaMemcpyAsync(&H32, ws.ctrl + 6, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
  RB_CUDA_TRY(cudaStreamSynchronize(stream));
  const int64_t H = H32;
  if (std::getenv("RB_1SA_STATS")) {
    unsigned long long st[8];
    RB_CUDA_TRY(cudaMemcpy(st, ws.stats, sizeof(st), cudaMemcpyDeviceToHost));
    fprintf(stderr, "[rb 1sa sparse] m=%d H=%lld batches=%llu seeds=%llu singletons=%llu rounds=%llu accepts=%llu "
            "batch_Mcyc=%.1f group_Mcyc=%.1f heavy_passes=%llu\n", m, (long long)H, st[0], st[1], st[2], st[3], st[4],
            st[5] / 1e6, st[6] / 1e6, st[7]);
#ifdef RB_PROF_1SA
    unsigned long long pf[24];
    RB_CUDA_TRY(cudaMemcpy(pf, ws.stats, sizeof(pf), cudaMemcpyDeviceToHost));
    const double seeds = std::max(1.0, (double)pf[1]), batches = std::max(1.0, (double)pf[0]);
    fprintf(stderr, "[rb 1sa prof] per seed: load %.0f prep %.0f enum %.0f cyc, entries %.0f; per batch: max CTA "
            "%.0f cyc, block0 barrier wait %.0f cyc, max psize %.0f; punted seeds %llu\n", pf[8] / seeds,
            pf[9] / seeds, pf[10] / seeds, pf[11] / seeds, pf[14] / batches, pf[18] / batches, pf[19] / batches,
            pf[15]);
#endif
  }
  // ---- assembly (as the dense path)
  assembly_keys_kernel<<<g1, 256, 0, stream>>>(ws.item_of_row, ws.group_of_item, n, m, ws.keys_a, ws.vals_a);
  {
    int end_bit = 1;
    while (end_bit < 64 && ((unsigned long long)H * (unsigned long long)m) > (1ull << end_bit)) ++end_bit;
    tb = ws.cub_bytes;
    RB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(ws.cub_tmp, tb, ws.keys_a, ws.keys_b, ws.vals_a, ws.vals_b, (int)n, 0,
                                                end_bit, stream));
  }
  assembly_out_kernel<<<g1, 256, 0, stream>>>(ws.vals_b, ws.keys_b, n, m, H, row_perm, group_of, group_ptr);
  seed_size_kernel<<<grid_for(H, 256), 256, 0, stream>>>(ws.seed_item, ws.item_size, H, seed_size);
  // ---- patterns: sorted unique (group, segment) pairs
  RB_CUDA_TRY(cudaMemsetAsync(ws.t1, 0, sizeof(int32_t) * (H + 1), stream));
  if (E > 0) {
    pattern_pairs_kernel<<<grid_for(m, 8), 256, 0, stream>>>(ws.group_of_item, ws.item_ptr, ws.item_seg, m, n_seg,
                                                             ws.keys_a);
    int end_bit = 1;
    while (end_bit < 64 && ((unsigned long long)H * (unsigned long long)n_seg) > (1ull << end_bit)) ++end_bit;
    tb = ws.cub_bytes;
    RB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(ws.cub_tmp, tb, ws.keys_a, ws.keys_b, (int)E, 0, end_bit, stream));
    tb = ws.cub_bytes;
    RB_CUDA_TRY(cub::DeviceSelect::Unique(ws.cub_tmp, tb, ws.keys_b, ws.keys_a, (int*)ws.t0, (int)E, stream));
    pattern_emit_kernel<<<grid_for(E, 256), 256, 0, stream>>>(ws.keys_a, (const int*)ws.t0, n_seg, pattern_idx, ws.t1);
  }
  widen_i32_kernel<<<grid_for(H + 1, 256), 256, 0, stream>>>(ws.t1, H + 1, ws.pcnt);
  tb = ws.cub_bytes;
  RB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws.cub_tmp, tb, ws.pcnt, pattern_ptr, (int)(H + 1), stream));
  RB_CUDA_TRY(cudaGetLastError());
  *n_groups = H;
  return RB_OK;
}
}  // namespace
}  // namespace rb

using namespace rb;

extern "C" int rb_block_1sa_workspace_size(int64_t n_rows, int64_t nnz, int64_t n_seg, int use_compression,
                                           size_t* bytes) {
  (void)use_compression;
  if (!bytes || n_rows < 0 || n_seg < 0 || nnz < 0) return fail(RB_EINVAL, "bad arguments");
  *bytes = use_sparse_path(words_of(n_seg)) ? carve_sparse(nullptr, n_rows, nnz, n_seg).total
                                            : carve(nullptr, n_rows, words_of(n_seg), n_seg).total;
  return RB_OK;
}

extern "C" int rb_block_1sa(int64_t n, int64_t n_cols, int64_t nnz, const int64_t* row_ptr, const int64_t* col_idx,
                            const int64_t* boundaries, int64_t n_seg, double tau, int similarity, int bounded,
                            int pattern_update, int use_compression, void* workspace, size_t ws_bytes,
                            int64_t* group_of, int64_t* row_perm, int64_t* group_ptr, int64_t* seed_size,
                            int64_t* pattern_ptr, int64_t* pattern_idx, int64_t* n_groups, void* stream_) {
  rb::NvtxRange nvtx_range_("rb_block_1sa");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  // MergePolicy validation (blocking.py:80-84)
  if (similarity != RB_JACCARD && similarity != RB_COSINE) return fail(RB_EINVAL, "unknown similarity");
  if (!(tau >= 0.0 && tau <= 1.0)) return fail(RB_EINVAL, "tau must be in [0, 1]");
  if (n < 0 || !n_groups) return fail(RB_EINVAL, "bad arguments");
  if (n >= (int64_t(1) << 31)) return fail(RB_EUNSUPPORTED, "n_rows must be < 2^31");
  const int64_t W = words_of(n_seg);
  int32_t delta = 0, maxw = 0;
  int rc = inspect_boundaries(boundaries, n_seg, n_cols, &delta, &maxw, nullptr, stream);
  if (rc) return rc;
  if (n == 0) {
    *n_groups = 0;
    RB_CUDA_TRY(cudaMemsetAsync(group_ptr, 0, sizeof(int64_t), stream));
    RB_CUDA_TRY(cudaMemsetAsync(pattern_ptr, 0, sizeof(int64_t), stream));
    return RB_OK;
  }
  if (use_sparse_path(W))
    return block_1sa_sparse(n, nnz, row_ptr, col_idx, boundaries, n_seg, delta, tau, similarity, bounded,
                            pattern_update, use_compression, workspace, ws_bytes, group_of, row_perm, group_ptr,
                            seed_size, pattern_ptr, pattern_idx, n_groups, stream);
  Ws ws = carve(workspace, n, W, n_seg);
  if (ws_bytes < ws.total) return fail(RB_EINVAL, "workspace too small");
  rc = narrow_bounds(boundaries, n_seg, ws.b32, stream);
  if (rc) return rc;
  SegMap seg{ws.b32, (int32_t)n_seg, delta};

  // ---- K1
  RB_CUDA_TRY(cudaMemsetAsync(ws.bits, 0, sizeof(uint64_t) * n * W, stream));
  if (n_seg > 0)
    quotient_kernel<<<grid_for(n, 8), 256, 0, stream>>>(row_ptr, col_idx, n, seg, W, ws.bits, ws.sizes);
  else
    RB_CUDA_TRY(cudaMemsetAsync(ws.sizes, 0, sizeof(int32_t) * n, stream));
  RB_CUDA_TRY(cudaGetLastError());

  // ---- K2
  int32_t m = (int32_t)n;
  const unsigned g1 = grid_for(n, 256);
  if (use_compression) {
    hash_kernel<<<g1, 256, 0, stream>>>(ws.bits, n, W, ws.keys_a, ws.vals_a);
    size_t tb = ws.cub_bytes;
    RB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(ws.cub_tmp, tb, ws.keys_a, ws.keys_b, ws.vals_a, ws.vals_b, (int)n, 0,
                                                64, stream));
    run_head_kernel<<<g1, 256, 0, stream>>>(ws.keys_b, n, ws.t0);
    tb = ws.cub_bytes;
    RB_CUDA_TRY(cub::DeviceScan::InclusiveScan(ws.cub_tmp, tb, ws.t0, ws.t1, MaxOp(), (int)n, stream));
    rep_kernel<<<g1, 256, 0, stream>>>(ws.bits, ws.vals_b, ws.t1, n, W, ws.t0);  // t0 = rep_of_row
    is_rep_kernel<<<g1, 256, 0, stream>>>(ws.t0, n, ws.t1);                     // t1 = flag
    RB_CUDA_TRY(cudaMemsetAsync(ws.t1 + n, 0, sizeof(int32_t), stream));
    tb = ws.cub_bytes;
    RB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws.cub_tmp, tb, ws.t1, ws.vals_a, (int)(n + 1), stream));  // idx
    items_kernel<<<g1, 256, 0, stream>>>(ws.t0, ws.vals_a, n, ws.item_of_row, ws.reps);
    RB_CUDA_TRY(cudaMemcpyAsync(&m, ws.vals_a + n, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    RB_CUDA_TRY(cudaStreamSynchronize(stream));
  } else {
    identity_items_kernel<<<g1, 256, 0, stream>>>(n, ws.item_of_row, ws.reps);
  }
  gather_items_kernel<<<grid_for((int64_t)m * W, 256), 256, 0, stream>>>(ws.bits, ws.sizes, ws.reps, m, W, ws.item_bits,
                                                                         ws.item_sizes, ws.group_of_item);
  RB_CUDA_TRY(cudaGetLastError());

  // ---- K3
  {
    int32_t ctrl0[16];
    for (int i = 0; i < 16; ++i) ctrl0[i] = 0;
    for (int i = 0; i < 6; ++i) ctrl0[i] = INT_MAX;
    RB_CUDA_TRY(cudaMemcpyAsync(ws.ctrl, ctrl0, sizeof(ctrl0), cudaMemcpyHostToDevice, stream));
    RB_CUDA_TRY(cudaMemsetAsync(ws.ctrl + 16, 0, sizeof(int32_t) * 2 * kMaxTesters, stream));
    GreedyArgs ga;
    ga.m = m;
    ga.W = (int32_t)W;
    ga.bits = ws.item_bits;
    ga.sizes = ws.item_sizes;
    ga.tau = tau;
    ga.cosine = similarity == RB_COSINE;
    ga.bounded = bounded != 0;
    ga.update = pattern_update != 0;
    ga.group_of_item = ws.group_of_item;
    ga.ok = ws.ok;
    ga.seed_item = ws.seed_item;
    ga.ctrl = ws.ctrl;
    ga.batching = 1;
    if (const char* e = std::getenv("RB_1SA_BATCH")) ga.batching = std::atoi(e) != 0;
    const bool warp_item = W > 4;
    const size_t shm = sizeof(uint64_t) * W;
    if (shm > 200 * 1024) return fail(RB_EUNSUPPORTED, "too many segments for the dense-bitset scan");
    void* fn = warp_item ? (void*)greedy_kernel<true> : (void*)greedy_kernel<false>;
    if (shm > 48 * 1024) RB_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    // small problems: one CTA (barrier = __syncthreads); large: one CTA per SM, cooperative
    const int64_t work = (int64_t)m * W;
    int blocks = 1;
    if (work > 64 * 1024) {
      int dev = 0, per_sm = 0, sms = 0;
      RB_CUDA_TRY(cudaGetDevice(&dev));
      RB_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      RB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 512, shm));
      if (per_sm < 1) return fail(RB_ECUDA, "greedy kernel cannot be resident");
      blocks = sms;
    }
    void* args[] = {&ga};
    RB_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(512), args, shm, stream));
  }
  int32_t H32 = 0;
  RB_CUDA_TRY(cudaMemcpyAsync(&H32, ws.ctrl + 6, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
  RB_CUDA_TRY(cudaStreamSynchronize(stream));
  const int64_t H = H32;

  // ---- assembly
  assembly_keys_kernel<<<g1, 256, 0, stream>>>(ws.item_of_row, ws.group_of_item, n, m, ws.keys_a, ws.vals_a);
  {
    int end_bit = 1;
    while (end_bit < 64 && ((unsigned long long)H * (unsigned long long)m) > (1ull << end_bit)) ++end_bit;
    size_t tb = ws.cub_bytes;
    RB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(ws.cub_tmp, tb, ws.keys_a, ws.keys_b, ws.vals_a, ws.vals_b, (int)n, 0,
                                                end_bit, stream));
  }
  assembly_out_kernel<<<g1, 256, 0, stream>>>(ws.vals_b, ws.keys_b, n, m, H, row_perm, group_of, group_ptr);
  seed_size_kernel<<<grid_for(H, 256), 256, 0, stream>>>(ws.seed_item, ws.item_sizes, H, seed_size);
  // patterns: OR of member item bitsets (bits buffer reused for the group bitsets)
  RB_CUDA_TRY(cudaMemsetAsync(ws.bits, 0, sizeof(uint64_t) * H * W, stream));
  group_or_kernel<<<grid_for((int64_t)m * W, 256), 256, 0, stream>>>(ws.item_bits, ws.group_of_item, m, W, ws.bits);
  pattern_kernel<<<grid_for(H, 8), 256, 0, stream>>>(ws.bits, H, W, 0, ws.pcnt, nullptr, nullptr);
  RB_CUDA_TRY(cudaMemsetAsync(ws.pcnt + H, 0, sizeof(int64_t), stream));
  {
    size_t tb = ws.cub_bytes;
    RB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws.cub_tmp, tb, ws.pcnt, pattern_ptr, (int)(H + 1), stream));
  }
  pattern_kernel<<<grid_for(H, 8), 256, 0, stream>>>(ws.bits, H, W, 1, nullptr, pattern_ptr, pattern_idx);
  RB_CUDA_TRY(cudaGetLastError());
  *n_groups = H;
  return RB_OK;
}
