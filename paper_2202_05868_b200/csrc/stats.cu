// Blocking-quality statistics on the device: replaces blocking_stats (metrics.py:59-95) and
// verify_density_bound (metrics.py:178-216) for groupings that live in HBM.
//
// One CTA per group: stored columns = sum of the pattern's segment widths, element nnz = sum of
// the member rows' nnz, quotient nnz = sum of the member rows' distinct segment counts (columns
// are sorted, so a row's segments are non-decreasing and distinct ones are counted at changes).
// The density verdicts use the reference's exact rational comparisons
// (Fraction(k, h*w) >= Fraction(float(tau)) / (2*max_w)), evaluated exactly in 128-bit integers
// from tau's binary64 value.
#include <cub/block/block_reduce.cuh>

#include "common.cuh"
#include "segments.cuh"

namespace rb {
namespace {

constexpr int STATS_THREADS = 256;

// lhs >= tau * x, exactly (tau in [0, 1] as a binary64 value, lhs, x >= 0).
__device__ bool ge_tau_times(unsigned long long lhs, unsigned long long x, double tau) {
  if (tau == 0.0 || x == 0ull) return true;
  if (lhs == 0ull) return false;
  int E = 0;
  const double f = frexp(tau, &E);                            // tau = f * 2^E, f in [0.5, 1)
  const unsigned long long mant = (unsigned long long)ldexp(f, 53);  // exact
  const int s = 53 - E;                                        // tau = mant / 2^s, s >= 52
  const unsigned __int128 rhs = (unsigned __int128)mant * x;   // < 2^117
  const int lbits = 64 - __clzll((long long)lhs);
  if (lbits + s > 118) return true;                            // lhs * 2^s >= 2^117 > rhs
  return ((unsigned __int128)lhs << s) >= rhs;
}

__global__ void __launch_bounds__(STATS_THREADS) group_stats_kernel(
    const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col_idx, SegMap seg,
    const int32_t* __restrict__ bounds, const int64_t* __restrict__ row_perm, const int64_t* __restrict__ group_ptr,
    const int64_t* __restrict__ pattern_ptr, const int64_t* __restrict__ pattern_idx, int32_t max_w, double tau,
    int64_t* stored_cols, int64_t* element_nnz, int64_t* quotient_nnz, uint8_t* ok, unsigned long long* totals) {
  using Reduce = cub::BlockReduce<long long, STATS_THREADS>;
  __shared__ typename Reduce::TempStorage tmp;
  const int64_t g = blockIdx.x;
  const int64_t r0 = group_ptr[g], r1 = group_ptr[g + 1];
  const int64_t p0 = pattern_ptr[g], p1 = pattern_ptr[g + 1];
  long long sc = 0, ke = 0, kq = 0;
  for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    const int64_t s = pattern_idx[p];
    sc += bounds[s + 1] - bounds[s];
  }
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    const int64_t r = row_perm[i];
    const int64_t a = row_ptr[r], b = row_ptr[r + 1];
    ke += b - a;
    int32_t prev = -1;
    for (int64_t j = a; j < b; ++j) {
      const int32_t sg = seg((int32_t)col_idx[j]);
      kq += sg != prev;
      prev = sg;
    }
  }
  sc = Reduce(tmp).Sum(sc);
  __syncthreads();
  ke = Reduce(tmp).Sum(ke);
  __syncthreads();
  kq = Reduce(tmp).Sum(kq);
  if (threadIdx.x == 0) {
    const unsigned long long h = (unsigned long long)(r1 - r0), lam = (unsigned long long)(p1 - p0);
    stored_cols[g] = sc;
    element_nnz[g] = ke;
    quotient_nnz[g] = kq;
    bool e_ok = true, q_ok = true;
    if (lam > 0) {  // empty patterns pass vacuously (metrics.py:197-199)
      e_ok = ge_tau_times((unsigned long long)ke * 2ull * (unsigned long long)max_w, h * (unsigned long long)sc, tau);
      q_ok = ge_tau_times((unsigned long long)kq * 2ull, h * lam, tau);
    }
    ok[g] = (uint8_t)((e_ok ? 1 : 0) | (q_ok ? 2 : 0));
    atomicAdd(totals + 0, h * (unsigned long long)sc);  // stored area
    atomicAdd(totals + 1, lam);                          // stored blocks
    atomicAdd(totals + 2, h * lam);                      // height sum over blocks
    if (!(e_ok && q_ok)) atomicAdd(totals + 3, 1ull);    // violations
  }
}

}  // namespace
}  // namespace rb

using namespace rb;

extern "C" int rb_group_stats(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_idx,
                              const int64_t* boundaries, int64_t n_seg, const int64_t* row_perm,
                              const int64_t* group_ptr, const int64_t* pattern_ptr, const int64_t* pattern_idx,
                              int64_t n_groups, double tau, void* workspace, size_t workspace_bytes,
                              int64_t* stored_cols, int64_t* element_nnz, int64_t* quotient_nnz, uint8_t* ok,
                              int64_t* stored_area, int64_t* n_blocks, int64_t* height_sum, int64_t* n_violations,
                              void* stream_) {
  rb::NvtxRange nvtx_range_("rb_group_stats");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (n_rows < 0 || n_groups < 0 || !(tau >= 0.0 && tau <= 1.0)) return fail(RB_EINVAL, "bad arguments");
  if (!stored_area || !n_blocks || !height_sum || !n_violations) return fail(RB_EINVAL, "null total");
  size_t need = 0;
  rb_group_stats_workspace_size(n_seg, &need);
  if (workspace_bytes < need || !workspace) return fail(RB_EINVAL, "workspace too small");
  int32_t delta = 0, max_w = 0;
  {
    int rc = inspect_boundaries(boundaries, n_seg, n_cols, &delta, &max_w, nullptr, stream);
    if (rc) return rc;
  }
  unsigned long long* totals = static_cast<unsigned long long*>(workspace);
  int32_t* b32 = reinterpret_cast<int32_t*>(static_cast<char*>(workspace) + 256);
  RB_CUDA_TRY(cudaMemsetAsync(totals, 0, 4 * sizeof(unsigned long long), stream));
  {
    int rc = narrow_bounds(boundaries, n_seg, b32, stream);
    if (rc) return rc;
  }
  if (n_groups > 0) {
    SegMap seg{b32, (int32_t)n_seg, delta};
    group_stats_kernel<<<(unsigned)n_groups, STATS_THREADS, 0, stream>>>(
        row_ptr, col_idx, seg, b32, row_perm, group_ptr, pattern_ptr, pattern_idx, max_w > 0 ? max_w : 1, tau,
        stored_cols, element_nnz, quotient_nnz, ok, totals);
    RB_CUDA_TRY(cudaGetLastError());
  }
  unsigned long long h[4];
  RB_CUDA_TRY(cudaMemcpyAsync(h, totals, sizeof(h), cudaMemcpyDeviceToHost, stream));
  RB_CUDA_TRY(cudaStreamSynchronize(stream));
  *stored_area = (int64_t)h[0];
  *n_blocks = (int64_t)h[1];
  *height_sum = (int64_t)h[2];
  *n_violations = (int64_t)h[3];
  return RB_OK;
}

extern "C" int rb_group_stats_workspace_size(int64_t n_seg, size_t* bytes) {
  if (!bytes || n_seg < 0) return fail(RB_EINVAL, "bad arguments");
  *bytes = 256 + sizeof(int32_t) * (size_t)(n_seg + 1);
  return RB_OK;
}
