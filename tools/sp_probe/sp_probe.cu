// Probe of tcgen05.mma.sp (2:4 sparse A, kind::f16, cta_group::1, M=128, K=32 logical) on sm_100a:
// checks an assumed metadata layout/encoding against a host reference.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2202_05868_b200/csrc tools/sp_probe/sp_probe.cu -o /tmp/sp_probe
//   /tmp/sp_probe <variant>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ptx.cuh"

using namespace rb;

constexpr int M = 128, N = 64, KL = 32, KP = 16;  // logical / physical K

__device__ __forceinline__ void tmem_st_32x32b_x1(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void umma_sp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t e_tmem,
                                        uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(e_tmem)
      : "memory");
}

// A_c: [128][16] bf16 compressed (row-major), B: [32][64] bf16 (k rows, n contiguous), E: [128] u32 per lane
__global__ void probe(const __nv_bfloat16* Ac, const __nv_bfloat16* B, const uint32_t* E, float* C, uint32_t idesc,
                      int e_col, int mode) {
  __shared__ __align__(1024) uint32_t sE[128 * 4];  // 128 lanes x 16 B, row-contiguous (cp source)
  __shared__ __align__(1024) uint8_t sA[128 * 128];  // SW128 K-major: 128 rows x 128 B (only first 32 B used)
  __shared__ __align__(1024) uint8_t sB[32 * 128];   // SW128 MN-major: 32 k-rows x 128 B (64 n)
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  // fill smem with the 128B swizzle: 16-byte chunk c of row r lands at chunk c ^ (r & 7)
  for (int i = t; i < 128 * 8; i += blockDim.x) {
    const int r = i >> 3, c = i & 7;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (c < 2) v = reinterpret_cast<const uint4*>(Ac + r * KP)[c];
    *reinterpret_cast<uint4*>(sA + r * 128 + ((c ^ (r & 7)) << 4)) = v;
  }
  for (int i = t; i < 32 * 8; i += blockDim.x) {
    const int r = i >> 3, c = i & 7;
    const uint4 v = reinterpret_cast<const uint4*>(B + r * N)[c];
    *reinterpret_cast<uint4*>(sB + r * 128 + ((c ^ (r & 7)) << 4)) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<128>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  // metadata: each warp writes its 32 lanes of column e_col (mode 0), or tcgen05.cp 128x128b
  if (mode == 0) {
    tmem_st_32x32b_x1(tmem + ((uint32_t)(warp * 32) << 16) + e_col, E[t]);
    tmem_st_wait();
  } else {
    const int w = mode >= 2 ? mode - 2 : 0;  // word slot of this MMA's metadata (selected by idesc id2)
    for (int j = 0; j < 4; ++j) sE[t * 4 + j] = j == w ? E[t] : 0xFFFFFFFFu;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    const uint64_t ad = sdesc_sw128(smem_u32(sA), 16, 1024);
    const uint64_t bd = sdesc_sw128(smem_u32(sB), 8192, 1024);
    if (mode != 0) {
      // no-swizzle K-major descriptor: 8-row core matrices of 16 B rows, SBO = 128 B between them
      uint64_t ed = 0;
      ed |= (uint64_t)((smem_u32(sE) >> 4) & 0x3FFF);
      ed |= (uint64_t)((16 >> 4) & 0x3FFF) << 16;
      ed |= (uint64_t)((128 >> 4) & 0x3FFF) << 32;
      ed |= (uint64_t)1 << 46;
      asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tmem + e_col), "l"(ed) : "memory");
    }
    umma_sp(tmem, ad, bd, idesc, tmem + e_col, 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[32];
  for (int c = 0; c < N; c += 32) {
    tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) C[t * N + c + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tmem);
}


__device__ __forceinline__ void umma_sp_2sm(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t e_tmem,
                                            uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%5], %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(e_tmem)
      : "memory");
}

// 2-CTA: CTA rank r holds A rows [128r, 128r+128) (compressed) and B columns [64r, 64r+64); M=256, N=128
__global__ void __cluster_dims__(2, 1, 1) probe2(const __nv_bfloat16* Ac, const __nv_bfloat16* B, const uint32_t* E,
                                                 float* C, uint32_t idesc, int e_col) {
  __shared__ __align__(1024) uint8_t sA[128 * 128];
  __shared__ __align__(1024) uint8_t sB[32 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t rank = cluster_ctarank();
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * 8; i += blockDim.x) {
    const int r = i >> 3, c = i & 7;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (c < 2) v = reinterpret_cast<const uint4*>(Ac + (rank * 128 + r) * KP)[c];
    *reinterpret_cast<uint4*>(sA + r * 128 + ((c ^ (r & 7)) << 4)) = v;
  }
  for (int i = t; i < 32 * 8; i += blockDim.x) {
    const int r = i >> 3, c = i & 7;
    const uint4 v = reinterpret_cast<const uint4*>(B + r * 128 + rank * 64)[c];
    *reinterpret_cast<uint4*>(sB + r * 128 + ((c ^ (r & 7)) << 4)) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_2sm<128>(&tslot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tslot;
  tmem_st_32x32b_x1(tmem + ((uint32_t)(warp * 32) << 16) + e_col, E[rank * 128 + t]);
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (rank == 0 && t == 0) {
    const uint64_t ad = sdesc_sw128(smem_u32(sA), 16, 1024);
    const uint64_t bd = sdesc_sw128(smem_u32(sB), 8192, 1024);
    umma_sp_2sm(tmem, ad, bd, idesc, tmem + e_col, 0);
    umma_commit_2sm_mc(&bar, 0x3);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[32];
  for (int c = 0; c < 128; c += 32) {
    tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) C[(rank * 128 + t) * 128 + c + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc_2sm<128>(tmem);
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }


int main2() {
  const int M2 = 256, N2 = 128;
  srand(11);
  std::vector<float> Al(M2 * KL, 0.f);
  std::vector<__nv_bfloat16> Ac(M2 * KP);
  std::vector<uint32_t> E(256, 0);
  const int pairs[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  for (int m = 0; m < M2; ++m)
    for (int c = 0; c < 8; ++c) {
      const int p = rand() % 6, i0 = pairs[p][0], i1 = pairs[p][1];
      const float v0 = bf((rand() % 17 - 8) / 8.f), v1 = bf((rand() % 17 - 8) / 8.f);
      Al[m * KL + 4 * c + i0] = v0;
      Al[m * KL + 4 * c + i1] = v1;
      Ac[m * KP + 2 * c] = __float2bfloat16(v0);
      Ac[m * KP + 2 * c + 1] = __float2bfloat16(v1);
      const int ml = m & 127, k = 4 * c;
      const int m0 = ml & 7, m1 = (ml >> 3) & 1, m2 = ml >> 4, k0 = k & 15, k1 = k >> 4;
      E[(m >> 7) * 128 + m0 + 8 * k1 + 16 * m2] |= (uint32_t)((i1 << 2) | i0) << (k0 + 16 * m1);
    }
  std::vector<__nv_bfloat16> Bh(KL * N2);
  std::vector<float> Bf(KL * N2);
  for (int i = 0; i < KL * N2; ++i) {
    Bf[i] = bf((rand() % 9 - 4) / 4.f);
    Bh[i] = __float2bfloat16(Bf[i]);
  }
  __nv_bfloat16 *dA, *dB;
  uint32_t* dE;
  float* dC;
  cudaMalloc(&dA, Ac.size() * 2);
  cudaMalloc(&dB, Bh.size() * 2);
  cudaMalloc(&dE, 1024);
  cudaMalloc(&dC, M2 * N2 * 4);
  cudaMemcpy(dA, Ac.data(), Ac.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bh.data(), Bh.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dE, E.data(), 1024, cudaMemcpyHostToDevice);
  const uint32_t idesc = idesc_f16(M2, N2, 1, 0, 1) | (1u << 2);
  probe2<<<2, 128>>>(dA, dB, dE, dC, idesc, 96);
  cudaError_t err = cudaDeviceSynchronize();
  printf("2sm: %s\n", cudaGetErrorString(err));
  if (err) return 1;
  std::vector<float> C(M2 * N2);
  cudaMemcpy(C.data(), dC, M2 * N2 * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < M2; ++m)
    for (int n = 0; n < N2; ++n) {
      float s = 0;
      for (int k = 0; k < KL; ++k) s += Al[m * KL + k] * Bf[k * N2 + n];
      if (fabs(C[m * N2 + n] - s) > 1e-3) {
        if (bad < 6) printf("  m=%d n=%d got %f want %f\n", m, n, C[m * N2 + n], s);
        ++bad;
      }
    }
  printf("2sm: %d / %d mismatches\n", bad, M2 * N2);
  return bad != 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == '2') return main2();
  const int variant = argc > 1 ? atoi(argv[1]) : 0;
  srand(7);
  // logical A: each chunk of 4 keeps 2 positions (i0 < i1)
  std::vector<float> Al(M * KL, 0.f);
  std::vector<__nv_bfloat16> Ac(M * KP);
  std::vector<uint8_t> nib(M * 8);  // per row, per chunk: (i1 << 2) | i0
  const int pairs[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  for (int m = 0; m < M; ++m)
    for (int c = 0; c < 8; ++c) {
      const int p = rand() % 6;
      const int i0 = pairs[p][0], i1 = pairs[p][1];
      const float v0 = bf((rand() % 17 - 8) / 8.f), v1 = bf((rand() % 17 - 8) / 8.f);
      Al[m * KL + 4 * c + i0] = v0;
      Al[m * KL + 4 * c + i1] = v1;
      Ac[m * KP + 2 * c] = __float2bfloat16(v0);
      Ac[m * KP + 2 * c + 1] = __float2bfloat16(v1);
      nib[m * 8 + c] = (uint8_t)((i1 << 2) | i0);
    }
  std::vector<__nv_bfloat16> Bh(KL * N);
  std::vector<float> Bf(KL * N);
  for (int i = 0; i < KL * N; ++i) {
    Bf[i] = bf((rand() % 9 - 4) / 4.f);
    Bh[i] = __float2bfloat16(Bf[i]);
  }
  // metadata words per TMEM lane (32 bits), hypothesis from CUTLASS tmem_e_frg (f16):
  //   lane = m0 + 8*k1 + 16*m2, bit = k0 + 16*m1 with m = m0 + 8 m1 + 16 m2, k = k0 + 16 k1,
  //   nibble of chunk (k0/4) at bits 4*(k0/4) + 16*m1
  std::vector<uint32_t> E(128, 0);
  for (int m = 0; m < M; ++m)
    for (int c = 0; c < 8; ++c) {
      const int k = 4 * c;
      uint32_t lane, bit;
      if (variant != 1) {
        const int m0 = m & 7, m1 = (m >> 3) & 1, m2 = m >> 4, k0 = k & 15, k1 = k >> 4;
        lane = m0 + 8 * k1 + 16 * m2;
        bit = k0 + 16 * m1;
      } else {  // variant 1: lane = row, nibbles in k order
        lane = m;
        bit = k;
      }
      E[lane] |= (uint32_t)nib[m * 8 + c] << bit;
    }
  std::vector<float> Cref(M * N, 0.f);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float s = 0;
      for (int k = 0; k < KL; ++k) s += Al[m * KL + k] * Bf[k * N + n];
      Cref[m * N + n] = s;
    }
  __nv_bfloat16 *dA, *dB;
  uint32_t* dE;
  float* dC;
  cudaMalloc(&dA, Ac.size() * 2);
  cudaMalloc(&dB, Bh.size() * 2);
  cudaMalloc(&dE, 512);
  cudaMalloc(&dC, M * N * 4);
  cudaMemcpy(dA, Ac.data(), Ac.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bh.data(), Bh.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dE, E.data(), 512, cudaMemcpyHostToDevice);
  const uint32_t idesc = idesc_f16(M, N, 1, 0, 1) | (1u << 2);  // sparse flag
  int mode = variant >= 3 ? 1 : 0;
  int ecol = variant == 4 ? 97 : variant == 5 ? 98 : 96;
  uint32_t id = idesc;
  if (variant >= 6) {  // metadata in word (variant - 6) of the 128-bit cp, selected by sparse_id2
    mode = 2 + (variant - 6);
    id = idesc | (uint32_t)(variant - 6);
  }
  probe<<<1, 128>>>(dA, dB, dE, dC, id, ecol, variant == 4 ? 0 : mode);
  cudaError_t err = cudaDeviceSynchronize();
  printf("variant %d: %s\n", variant, cudaGetErrorString(err));
  if (err) return 1;
  std::vector<float> C(M * N);
  cudaMemcpy(C.data(), dC, M * N * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  double maxe = 0;
  for (int i = 0; i < M * N; ++i) {
    const double e = fabs(C[i] - Cref[i]);
    maxe = e > maxe ? e : maxe;
    if (e > 1e-3) {
      if (bad < 6) printf("  m=%d n=%d got %f want %f\n", i / N, i % N, C[i], Cref[i]);
      ++bad;
    }
  }
  printf("variant %d: %d / %d mismatches, max err %g\n", variant, bad, M * N, maxe);
  // dense reference of the compressed values placed at k = 2c, 2c+1 (diagnostic)
  return bad != 0;
}
