// C-ABI plumbing: error reporting, boundary inspection, dtype conversion kernels.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <string>
#include <vector>

#include "common.cuh"
#include "segments.cuh"

namespace rb {

static thread_local std::string g_last_error;

void set_error(const std::string& s) { g_last_error = s; }
int fail(int code, const std::string& s) {
  g_last_error = s;
  return code;
}

int inspect_boundaries(const int64_t* d_bounds, int64_t n_seg, int64_t n_cols, int32_t* delta, int32_t* max_width,
                       std::vector<int64_t>* host, cudaStream_t stream) {
  if (n_seg < 0) return fail(RB_EINVAL, "n_seg must be >= 0");
  if (n_cols >= (int64_t(1) << 31)) return fail(RB_EUNSUPPORTED, "n_cols must be < 2^31");
  std::vector<int64_t> b(n_seg + 1);
  if (!d_bounds) return fail(RB_EINVAL, "null boundaries");
  RB_CUDA_TRY(cudaMemcpyAsync(b.data(), d_bounds, sizeof(int64_t) * (n_seg + 1), cudaMemcpyDeviceToHost, stream));
  RB_CUDA_TRY(cudaStreamSynchronize(stream));
  // ColumnPartition invariants (matrix.py:136-142)
  if (n_cols < 0) n_cols = b[n_seg];
  if (b[0] != 0 || b[n_seg] != n_cols) return fail(RB_EINVAL, "boundaries must start at 0 and end at n_cols");
  int64_t mw = 0;
  for (int64_t i = 0; i < n_seg; ++i) {
    if (b[i + 1] <= b[i]) return fail(RB_EINVAL, "boundaries must be strictly increasing");
    mw = std::max<int64_t>(mw, b[i + 1] - b[i]);
  }
  int64_t d = n_seg > 0 ? b[1] - b[0] : 0;
  bool uni = n_seg > 0;
  for (int64_t i = 0; i < n_seg && uni; ++i) uni = (b[i] == i * d);
  *delta = uni ? (int32_t)d : 0;
  *max_width = (int32_t)mw;
  if (host) host->swap(b);
  return RB_OK;
}

__global__ void narrow_kernel(const int64_t* in, int64_t n, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}

int narrow_bounds(const int64_t* d_bounds, int64_t n_seg, int32_t* d_out, cudaStream_t stream) {
  const int64_t n = n_seg + 1;
  narrow_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, stream>>>(d_bounds, n, d_out);
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}

template <typename T>
__device__ __forceinline__ T from_f64(double v);
template <>
__device__ __forceinline__ float from_f64<float>(double v) { return (float)v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f64<__nv_bfloat16>(double v) { return __double2bfloat16(v); }
template <>
__device__ __forceinline__ __half from_f64<__half>(double v) { return __double2half(v); }
template <>
__device__ __forceinline__ double from_f64<double>(double v) { return v; }

// float64 -> kernel dtype; with `nonfinite`, any NaN / Inf in src sets *nonfinite = 1 (all writers
// store the same value, so the race is benign).
template <typename T>
__global__ void convert_kernel(const double* __restrict__ src, int64_t rows, int64_t cols, int64_t lds, T* dst,
                               int64_t ldd, int32_t* nonfinite) {
  const int64_t total = rows * cols;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const double v = src[r * lds + c];
    bad |= !isfinite(v);
    dst[r * ldd + c] = from_f64<T>(v);
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *nonfinite = 1;
}

__global__ void widen_kernel(const float* __restrict__ src, int64_t rows, int64_t cols, int64_t lds, double* dst,
                             int64_t ldd) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    dst[r * ldd + c] = (double)src[r * lds + c];
  }
}

}  // namespace rb

using namespace rb;

extern "C" const char* rb_last_error_string(void) { return g_last_error.c_str(); }
extern "C" int rb_abi_version(void) { return 1; }

extern "C" int rb_convert_f64_checked(const double* src, int64_t rows, int64_t cols, int64_t lds, void* dst,
                                      int32_t dst_dtype, int64_t ldd, int32_t* nonfinite, void* stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (rows < 0 || cols < 0 || lds < cols || ldd < cols) return fail(RB_EINVAL, "bad convert shape");
  if (rows * cols == 0) return RB_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((rows * cols + 255) / 256, 148 * 32);
  int32_t* f = nonfinite;
  switch (dst_dtype) {
    case RB_F32: convert_kernel<<<grid, 256, 0, stream>>>(src, rows, cols, lds, (float*)dst, ldd, f); break;
    case RB_BF16: convert_kernel<<<grid, 256, 0, stream>>>(src, rows, cols, lds, (__nv_bfloat16*)dst, ldd, f); break;
    case RB_F16: convert_kernel<<<grid, 256, 0, stream>>>(src, rows, cols, lds, (__half*)dst, ldd, f); break;
    case RB_F64: convert_kernel<<<grid, 256, 0, stream>>>(src, rows, cols, lds, (double*)dst, ldd, f); break;
    default: return fail(RB_EINVAL, "bad dtype");
  }
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}

extern "C" int rb_convert_f64(const double* src, int64_t rows, int64_t cols, int64_t lds, void* dst,
                              int32_t dst_dtype, int64_t ldd, void* stream_) {
  return rb_convert_f64_checked(src, rows, cols, lds, dst, dst_dtype, ldd, nullptr, stream_);
}

extern "C" int rb_widen_f32(const float* src, int64_t rows, int64_t cols, int64_t lds, double* dst, int64_t ldd,
                            void* stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (rows < 0 || cols < 0 || lds < cols || ldd < cols) return fail(RB_EINVAL, "bad widen shape");
  if (rows * cols == 0) return RB_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((rows * cols + 255) / 256, 148 * 32);
  widen_kernel<<<grid, 256, 0, stream>>>(src, rows, cols, lds, dst, ldd);
  RB_CUDA_TRY(cudaGetLastError());
  return RB_OK;
}
