// GPU comparator for spmm_csr (multiply.py:51-69): C = A·B straight from the CSR arrays, on the
// CUDA-core gather engine of spmm_skinny.cu.  This is the sparse baseline of the paper's VBR vs CSR
// comparison, measured on the same B200 as the VBR kernels.
#include <algorithm>
#include <vector>

#include <mutex>

#include "common.cuh"
#include "spmm_skinny.cuh"

namespace rb {
constexpr int CSR_PART_NNZ = 2048;  // nonzeros per part of a split (hub) row
}

struct rb_csr_plan {
  int64_t n_rows, n_cols, N;
  int32_t b_dtype;
  rb::SkinnyItem* d_items = nullptr;
  int64_t n_items = 0;
  int32_t chunk = 1;  // items per claim (csr_claim_chunk)
  float* d_ws = nullptr;
  int32_t* d_cnt = nullptr;
  unsigned long long* d_sched = nullptr;
  // executions of one plan are serialised (its work counters and split partials are reset by the
  // kernels themselves): host threads through `mu`, streams through the `done` event
  mutable std::mutex mu;
  mutable cudaEvent_t done = nullptr;
  mutable cudaStream_t done_stream = nullptr;
  mutable bool done_valid = false;
};

using namespace rb;

extern "C" int rb_csr_plan_destroy(rb_csr_plan* p) {
  if (!p) return RB_OK;
  if (p->d_items) cudaFree(p->d_items);
  if (p->d_ws) cudaFree(p->d_ws);
  if (p->d_cnt) cudaFree(p->d_cnt);
  if (p->d_sched) cudaFree(p->d_sched);
  if (p->done) cudaEventDestroy(p->done);
  delete p;
  return RB_OK;
}

extern "C" int rb_csr_plan_create(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, int64_t N, int32_t b_dtype,
                                  rb_csr_plan** out, void* stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (!out || n_rows < 0 || n_cols < 0 || (n_rows > 0 && !row_ptr)) return fail(RB_EINVAL, "bad arguments");
  if (N <= 0 || N > (1ll << 30)) return fail(RB_EINVAL, "bad n_dense_cols");
  if (b_dtype != RB_BF16 && b_dtype != RB_F16 && b_dtype != RB_F32) return fail(RB_EUNSUPPORTED, "bad B dtype");
  if (n_rows >= (1ll << 31) || n_cols >= (1ll << 31)) return fail(RB_EUNSUPPORTED, "dimensions must be < 2^31");
  std::vector<int64_t> rp(n_rows + 1, 0);
  if (n_rows > 0) {
    RB_CUDA_TRY(cudaMemcpyAsync(rp.data(), row_ptr, sizeof(int64_t) * (n_rows + 1), cudaMemcpyDeviceToHost, stream));
    RB_CUDA_TRY(cudaStreamSynchronize(stream));
  }
  const int cols = skinny_cols(b_dtype, N);
  std::vector<SkinnyItem> items;
  items.reserve((size_t)n_rows * ((N + cols - 1) / cols));
  int64_t n_slots = 0, ws_units = 0;
  for (int64_t r = 0; r < n_rows; ++r) {
    const int64_t nnz = rp[r + 1] - rp[r];
    if (nnz < 0) return fail(RB_EINVAL, "row_ptr must be non-decreasing");
    if (nnz >= (1ll << 31)) return fail(RB_EUNSUPPORTED, "row too long");
    const int nparts = nnz > CSR_PART_NNZ ? (int)((nnz + CSR_PART_NNZ - 1) / CSR_PART_NNZ) : 1;
    for (int64_t n0 = 0; n0 < N; n0 += cols) {
      if (nparts == 1) {
        items.push_back(SkinnyItem{(int32_t)r, (int32_t)n0, 0, (int32_t)nnz, 0, 1, -1, 0});
        continue;
      }
      const int32_t slot = (int32_t)n_slots++, wsoff = (int32_t)ws_units;
      ws_units += (int64_t)nparts * (cols / 128);
      for (int p = 0; p < nparts; ++p)
        items.push_back(SkinnyItem{(int32_t)r, (int32_t)n0, (int32_t)(nnz * p / nparts),
                                   (int32_t)(nnz * (p + 1) / nparts), p, nparts, slot, wsoff});
    }
  }
  std::stable_sort(items.begin(), items.end(),
                   [](const SkinnyItem& x, const SkinnyItem& y) { return x.be - x.bb > y.be - y.bb; });
  auto* p = new rb_csr_plan();
  p->n_rows = n_rows;
  p->n_cols = n_cols;
  p->N = N;
  p->b_dtype = b_dtype;
  p->n_items = (int64_t)items.size();
  p->chunk = csr_claim_chunk(items);
  cudaError_t e = cudaSuccess;
  if (p->n_items > 0) e = cudaMalloc(&p->d_items, sizeof(SkinnyItem) * items.size());
  if (e == cudaSuccess) e = cudaMalloc(&p->d_sched, 2 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemsetAsync(p->d_sched, 0, 2 * sizeof(unsigned long long), stream);
  if (e == cudaSuccess && n_slots > 0) e = cudaMalloc(&p->d_ws, sizeof(float) * 128 * (size_t)ws_units);
  if (e == cudaSuccess && n_slots > 0) e = cudaMalloc(&p->d_cnt, sizeof(int32_t) * (size_t)n_slots);
  if (e == cudaSuccess && n_slots > 0) e = cudaMemsetAsync(p->d_cnt, 0, sizeof(int32_t) * n_slots, stream);
  if (e == cudaSuccess && p->n_items > 0)
    e = cudaMemcpyAsync(p->d_items, items.data(), sizeof(SkinnyItem) * items.size(), cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) {
    rb_csr_plan_destroy(p);
    return fail(e == cudaErrorMemoryAllocation ? RB_ENOMEM : RB_ECUDA, cudaGetErrorString(e));
  }
  *out = p;
  return RB_OK;
}

extern "C" int rb_csr_execute(const rb_csr_plan* p, const int64_t* row_ptr, const int64_t* col_idx,
                              const double* values, const void* B, int64_t ldb, float* C, int64_t ldc, void* stream_) {
  rb::NvtxRange nvtx_range_("rb_csr_execute");
  if (!p) return fail(RB_EINVAL, "null plan");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (ldb < p->N || ldc < p->N) return fail(RB_EINVAL, "leading dimension smaller than N");
  if (p->n_items == 0) return RB_OK;
  if (!C || !B || !row_ptr) return fail(RB_EINVAL, "null operand");
  SkinnyArgs a{};
  a.row_partition = nullptr;
  a.row_perm = nullptr;
  a.items = p->d_items;
  a.n_items = p->n_items;
  a.B = B;
  a.ldb = ldb;
  a.C = C;
  a.ldc = ldc;
  a.N = (int32_t)p->N;
  a.ws = p->d_ws;
  a.cnt = p->d_cnt;
  CsrArgs c{row_ptr, col_idx, values, nullptr, nullptr, p->chunk};
  std::lock_guard<std::mutex> lk(p->mu);
  if (!p->done) RB_CUDA_TRY(cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming));
  if (p->done_valid && p->done_stream != stream) RB_CUDA_TRY(cudaStreamWaitEvent(stream, p->done, 0));
  if (int rc = launch_csr(a, c, p->b_dtype, p->d_sched, stream)) return rc;
  RB_CUDA_TRY(cudaEventRecord(p->done, stream));
  p->done_stream = stream;
  p->done_valid = true;
  return RB_OK;
}
