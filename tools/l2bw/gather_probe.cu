// Random-row gather bandwidth: the access pattern of the CSR gather engine (spmm_csr_kernel), where
// every nonzero pulls one B row segment of R bytes from a random row.  (1) ldg: groups of R/16
// lanes load one row each, 16 B per lane, 8 rows in flight per group (the engine's depth),
// 256-thread CTAs at 4 per SM.  (2) bulk: one thread per CTA issues R-byte cp.async.bulk copies of
// random rows into a DEPTH-deep SMEM ring (TMA gathers).  Working sets below L2 measure L2-hit
// gather bandwidth; the 256 MB set (config 3's B is 268 MB) mixes in HBM misses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2bw/gather_probe tools/l2bw/gather_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

template <int R>
__global__ void __launch_bounds__(256, 4) gather_ldg(const int4* __restrict__ p, uint32_t rows, int per_group,
                                                     int4* sink) {
  constexpr int LPR = R / 16;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const int gl = (int)(t % LPR);  // a 1 KB row spans two warps
  const uint32_t grp = t / LPR;
  int4 acc = make_int4(0, 0, 0, 0);
  for (int i = 0; i < per_group; i += 8) {
    int4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t r = hash32(grp * 2654435761u + (uint32_t)(i + u)) % rows;
      v[u] = __ldg(p + (size_t)r * LPR + gl);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc.x ^= v[u].x;
      acc.y += v[u].y;
    }
  }
  if (acc.x == 0x12345 && acc.y == 7) sink[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int R, int DEPTH>
__global__ void __launch_bounds__(32) gather_bulk(const char* __restrict__ p, uint32_t rows, int per_cta, int* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[DEPTH];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < DEPTH; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  uint32_t ph = 0;  // DEPTH slots complete in order, one phase bit per ring revolution
  for (int k = 0; k < per_cta; ++k) {
    const int s = k % DEPTH;
    if (k >= DEPTH) {
      uint32_t done = 0;
      const uint32_t par = ((k / DEPTH) - 1) & 1;
      while (!done)
        asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                     : "=r"(done) : "r"(su32(&bar[s])), "r"(par));
    }
    const uint32_t r = hash32(blockIdx.x * 2654435761u + (uint32_t)k) % rows;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(R));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(sm + s * R)), "l"(p + (size_t)r * R), "r"(R), "r"(su32(&bar[s])) : "memory");
  }
  for (int k = per_cta > DEPTH ? per_cta - DEPTH : 0; k < per_cta; ++k) {
    const int s = k % DEPTH;
    uint32_t done = 0;
    const uint32_t par = (k / DEPTH) & 1;
    while (!done)
      asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                   : "=r"(done) : "r"(su32(&bar[s])), "r"(par));
  }
  (void)ph;
  if (sm[5] == 123 && sm[7] == 45) sink[0] = 1;
}

template <int R>
void run(int sms, char* buf, int4* sink, size_t mb) {
  const uint32_t rows = (uint32_t)((mb << 20) / R);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  {
    const int per_group = 512;
    const unsigned grid = sms * 4;
    const double bytes = (double)grid * 256 / (R / 16) * per_group * R;
    gather_ldg<R><<<grid, 256>>>((const int4*)buf, rows, per_group, sink);
    cudaEventRecord(a);
    gather_ldg<R><<<grid, 256>>>((const int4*)buf, rows, per_group, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("ldg  row=%4d B W=%5zu MB  %8.1f GB/s  (%s)\n", R, mb, bytes / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int per_sm : {2, 4, 8}) {
    constexpr int DEPTH = 32;
    const int per_cta = 4096;
    cudaFuncSetAttribute(gather_bulk<R, DEPTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, R * DEPTH);
    const unsigned grid = sms * per_sm;
    gather_bulk<R, DEPTH><<<grid, 32, R * DEPTH>>>(buf, rows, per_cta, (int*)sink);
    cudaEventRecord(a);
    gather_bulk<R, DEPTH><<<grid, 32, R * DEPTH>>>(buf, rows, per_cta, (int*)sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("bulk row=%4d B W=%5zu MB ctas/sm=%d depth=%d  %8.1f GB/s  (%s)\n", R, mb, per_sm, DEPTH,
           (double)grid * per_cta * R / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  char* buf;
  cudaMalloc(&buf, (size_t)512 << 20);
  cudaMemset(buf, 1, (size_t)512 << 20);
  int4* sink;
  cudaMalloc(&sink, 64);
  for (size_t mb : {64, 256}) {
    run<256>(sms, buf, sink, mb);
    run<512>(sms, buf, sink, mb);
    run<1024>(sms, buf, sink, mb);
  }
  return 0;
}
