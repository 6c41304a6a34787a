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

#include <climits>
#include <vector>

#include "common.cuh"
#include "segments.cuh"

namespace rb {
namespace {

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
inline int64_t words_of(int64_t n_seg) { return n_seg > 0 ? (n_seg + 63) / 64 : 1; }
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
  w.ctrl = (int32_t*)take(sizeof(int32_t) * 16);
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
  int32_t* ctrl;           // [0..2] first growing hit, [3..5] first rejection, [6] H, [8] count, [9] gen
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

template <bool kWarpPerItem>
__global__ void __launch_bounds__(512) greedy_kernel(GreedyArgs a) {
  extern __shared__ unsigned long long sP[];  // current pattern, W words
  __shared__ int32_t s_js, s_rj;
  __shared__ int32_t s_pos, s_g, s_first_rej, s_acc_lo, s_acc_hi, s_acc_g, s_finishing;
  __shared__ long long s_psize;
  __shared__ double s_cap;
  __shared__ int32_t s_inter;

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
    s_psize = a.sizes[0];
    s_cap = __ddiv_rn((double)a.sizes[0], cap_den);
    if (blockIdx.x == 0) {
      a.group_of_item[0] = 0;
      a.seed_item[0] = 0;
    }
  }
  for (int w = threadIdx.x; w < W; w += blockDim.x) sP[w] = a.bits[w];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  for (int r = 0;; ++r) {
    const int slot = r % 3;
    if (threadIdx.x == 0) {
      s_js = INT_MAX;
      s_rj = INT_MAX;
    }
    __syncthreads();
    const int32_t pos = s_pos, acc_lo = s_acc_lo, acc_hi = s_acc_hi, acc_g = s_acc_g, g = s_g;
    const long long psize = s_psize;
    const double cap = s_cap;
    const int32_t lo = acc_lo < acc_hi ? min(acc_lo, pos) : pos;
    int32_t my_js = INT_MAX, my_rj = INT_MAX;
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
          if (v && a.update && inter < sz) my_js = min(my_js, (int32_t)j);
          if (!v) my_rj = min(my_rj, (int32_t)j);
        }
      }
    }
    my_js = __reduce_min_sync(0xffffffffu, my_js);
    my_rj = __reduce_min_sync(0xffffffffu, my_rj);
    if (lane == 0) {
      if (my_js != INT_MAX) atomicMin(&s_js, my_js);
      if (my_rj != INT_MAX) atomicMin(&s_rj, my_rj);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_js != INT_MAX) atomicMin(a.ctrl + slot, s_js);
      if (s_rj != INT_MAX) atomicMin(a.ctrl + 3 + slot, s_rj);
    }
    grid_barrier(a.ctrl + 8, a.ctrl + 9);
    if (s_finishing) break;  // the final acceptance has been applied
    const int32_t js = *((volatile int32_t*)(a.ctrl + slot));
    const int32_t rj = *((volatile int32_t*)(a.ctrl + 3 + slot));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.ctrl[(r + 2) % 3] = INT_MAX;
      a.ctrl[3 + (r + 2) % 3] = INT_MAX;
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
      }
    } else {
      // the group is complete: accept ok items in [pos, m); the first rejected item seeds the next group
      const int32_t fr = min(s_first_rej, rj);
      __syncthreads();
      if (threadIdx.x == 0) {
        s_acc_lo = pos;
        s_acc_hi = m;
        s_acc_g = g;
        if (fr >= m) {
          s_finishing = 1;
          s_pos = m;
        } else {
          s_g = g + 1;
          s_first_rej = INT_MAX;
          s_psize = a.sizes[fr];
          s_cap = __ddiv_rn((double)a.sizes[fr], cap_den);
          s_pos = fr + 1;
          if (blockIdx.x == 0) {
            a.group_of_item[fr] = g + 1;
            a.seed_item[g + 1] = fr;
          }
        }
      }
      if (fr < m)
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

}  // namespace
}  // namespace rb

using namespace rb;

extern "C" int rb_block_1sa_workspace_size(int64_t n_rows, int64_t nnz, int64_t n_seg, int use_compression,
                                           size_t* bytes) {
  (void)nnz;
  (void)use_compression;
  if (!bytes || n_rows < 0 || n_seg < 0) return fail(RB_EINVAL, "bad arguments");
  *bytes = carve(nullptr, n_rows, words_of(n_seg), n_seg).total;
  return RB_OK;
}

extern "C" int rb_block_1sa(int64_t n, int64_t n_cols, int64_t nnz, const int64_t* row_ptr, const int64_t* col_idx,
                            const int64_t* boundaries, int64_t n_seg, double tau, int similarity, int bounded,
                            int pattern_update, int use_compression, void* workspace, size_t ws_bytes,
                            int64_t* group_of, int64_t* row_perm, int64_t* group_ptr, int64_t* seed_size,
                            int64_t* pattern_ptr, int64_t* pattern_idx, int64_t* n_groups, void* stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  (void)nnz;
  // MergePolicy validation (blocking.py:80-84)
  if (similarity != RB_JACCARD && similarity != RB_COSINE) return fail(RB_EINVAL, "unknown similarity");
  if (!(tau >= 0.0 && tau <= 1.0)) return fail(RB_EINVAL, "tau must be in [0, 1]");
  if (n < 0 || !n_groups) return fail(RB_EINVAL, "bad arguments");
  if (n >= (int64_t(1) << 31)) return fail(RB_EUNSUPPORTED, "n_rows must be < 2^31");
  const int64_t W = words_of(n_seg);
  Ws ws = carve(workspace, n, W, n_seg);
  if (ws_bytes < ws.total) return fail(RB_EINVAL, "workspace too small");
  int32_t delta = 0, maxw = 0;
  int rc = inspect_boundaries(boundaries, n_seg, n_cols, &delta, &maxw, nullptr, stream);
  if (rc) return rc;
  if (n == 0) {
    *n_groups = 0;
    RB_CUDA_TRY(cudaMemsetAsync(group_ptr, 0, sizeof(int64_t), stream));
    RB_CUDA_TRY(cudaMemsetAsync(pattern_ptr, 0, sizeof(int64_t), stream));
    return RB_OK;
  }
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
