// Where does a cta_group::1 M=64 tcgen05.mma accumulator land in TMEM, and can a second one be
// placed at a lane offset?  A = 64 x 16 (K-major) with A[r][k] = (k == 0 ? r + 1 : 0), B = 16 x N
// (MN-major) with B[k][n] = (k == 0 ? n + 1 : 0), so D[r][n] = (r + 1) * (n + 1).  The MMA writes
// D at TMEM (lane offset L, column 0); four warps then dump all 128 lanes x N columns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2202_05868_b200/csrc tools/mma_probe/m64_layout.cu
#include <cstdio>
#include <cuda.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
using namespace rb;

constexpr int N = 64;

__global__ void __launch_bounds__(128) probe(float* out, int lane_off) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // A: 64 rows x 64 K (one SW128 row of 128 B per matrix row), K-major, 16-byte chunks XOR-swizzled
  // by (row & 7).  Only k = 0 is non-zero: byte 0..1 of chunk 0 of each row.
  __nv_bfloat16* a = reinterpret_cast<__nv_bfloat16*>(sm);
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) a[i] = __float2bfloat16(0.f);
  // B: MN-major, [k][n] rows of 64 n (128 B) per SW128 box; only k = 0 non-zero.
  __nv_bfloat16* b = reinterpret_cast<__nv_bfloat16*>(sm + 16384);
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) b[i] = __float2bfloat16(0.f);
  __syncthreads();
  if (threadIdx.x < 64) {  // A[r][0] at row r, chunk 0 -> swizzled chunk (0 ^ (r & 7))
    const int r = threadIdx.x;
    a[r * 64 + ((0 ^ (r & 7)) * 8)] = __float2bfloat16((float)(r + 1));
  }
  if (threadIdx.x < N) {  // B[0][n]: row k = 0 (chunk of 8 n per 16 B), swizzle by (k & 7) = 0
    const int n = threadIdx.x;
    b[n] = __float2bfloat16((float)(n + 1));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  {  // zero all 512 columns of this warp's 32 lanes (TMEM keeps stale data across kernels)
    for (int c0 = 0; c0 < 512; c0 += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};"
                   ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + c0), "r"(0u) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16(64, N, 1, /*a_mn=*/0, /*b_mn=*/1);
    const uint64_t ad = sdesc_sw128(smem_u32(a), 16, 1024);
    const uint64_t bd = sdesc_sw128(smem_u32(b), 8192, 1024);
    umma_f16(tmem + ((uint32_t)lane_off << 16), ad, bd, idesc, 0);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * N * 4);
  float h[128 * N];
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int off : {0, 16, 32, 64}) {
    cudaMemset(d, 0, 128 * N * 4);
    probe<<<1, 128, 64 * 1024>>>(d, off);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("lane offset %d (%s):\n", off, cudaGetErrorString(e));
    for (int l = 0; l < 128; ++l) {
      // print lanes with data: the value at column 0 and 1 -> (r+1)*(n+1) identifies row r, col n
      bool any = false;
      for (int c = 0; c < N; ++c) any |= h[l * N + c] != 0.f;
      if (any) printf("  lane %3d: row %3.0f  (c1 %4.0f, c%d %5.0f)\n", l, h[l * N] - 1, h[l * N + 1], N - 1,
                      h[l * N + N - 1]);
    }
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
