// L2 -> SM read bandwidth probe.  (1) every thread streams 16-byte ld.global.cg loads, 8 in flight;
// (2) every CTA streams 32 KB cp.async.bulk (TMA bulk) copies into a 4-stage SMEM ring.  Working
// sets below the L2 size measure L2 hit bandwidth, above it HBM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void rd(const int4* __restrict__ p, size_t n, int reps, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x + (size_t)r * 7919 * 64) % n;
    for (size_t c = 0; c < n; c += 8 * stride) {
      int4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        size_t j = (i + u * stride) % n;
        asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + j));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; }
      i = (i + 8 * stride) % n;
    }
  }
  if (acc.x == 0x12345 && acc.y == 7) sink[0] = acc;
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
constexpr int CH = 32768, ST = 4;
__global__ void __launch_bounds__(32) bulk(const char* __restrict__ p, size_t nchunks, int reps, int* sink) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) uint64_t bar[ST];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < ST; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  uint32_t ph[ST] = {0, 0, 0, 0};
  long k = 0;
  const size_t total = nchunks * reps;
  for (size_t c = blockIdx.x; c < total; c += gridDim.x, ++k) {
    const int s = k % ST;
    if (k >= ST) {
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                     : "=r"(done) : "r"(su32(&bar[s])), "r"(ph[s]));
      ph[s] ^= 1;
    }
    const char* src = p + (c % nchunks) * CH;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(CH));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(sm + s * CH)), "l"(src), "r"(CH), "r"(su32(&bar[s])) : "memory");
  }
  for (long j = (k > ST ? k - ST : 0); j < k; ++j) {
    const int s = j % ST;
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                   : "=r"(done) : "r"(su32(&bar[s])), "r"(ph[s]));
    ph[s] ^= 1;
  }
  if (sm[5] == 123 && sm[7] == 45) sink[0] = 1;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t sizes_mb[] = {16, 32, 48, 64, 80, 96, 128, 256, 1024};
  char* buf; cudaMalloc(&buf, (size_t)1024 << 20); cudaMemset(buf, 1, (size_t)1024 << 20);
  int4* sink; cudaMalloc(&sink, 64);
  cudaFuncSetAttribute(bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * ST);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (size_t mb : sizes_mb) {
    size_t n = (mb << 20) / 16;
    int reps = (int)(4096 / mb); if (reps < 2) reps = 2;
    for (int occ : {4, 8}) {
      rd<<<sms * occ, 256>>>((const int4*)buf, n, 1, sink);
      cudaEventRecord(a);
      rd<<<sms * occ, 256>>>((const int4*)buf, n, reps, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("ldg  W=%5zu MB occ=%d  %8.1f GB/s\n", mb, occ, (double)n * 16 * reps / (ms * 1e-3) / 1e9);
    }
    size_t nch = (mb << 20) / CH;
    for (int per : {1, 2}) {
      bulk<<<sms * per, 32, CH * ST>>>(buf, nch, 1, (int*)sink);
      cudaEventRecord(a);
      bulk<<<sms * per, 32, CH * ST>>>(buf, nch, reps, (int*)sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("bulk W=%5zu MB ctas/sm=%d  %8.1f GB/s  (%s)\n", mb, per, (double)nch * CH * reps / (ms * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
