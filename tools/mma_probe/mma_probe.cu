// tcgen05.mma (kind::f16, cta_group::1, both operands in SMEM, SW128) issue-to-completion throughput
// per shape and operand major-ness.  One CTA per SM, thread 0 issues `reps` x 4 (K = 64) MMAs into
// one TMEM accumulator and waits on a commit; cycles per MMA are reported for CTA 0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2202_05868_b200/csrc tools/mma_probe/mma_probe.cu
#include <cstdio>
#include <cuda.h>
#include "ptx.cuh"
using namespace rb;

// MODE bits: 1 = commit to an mbarrier after every 8 MMAs; 2 = warps 2-3 spin on an mbarrier that
// never completes while the MMAs run; 4 = wait on an already completed mbarrier + fence per 8 MMAs;
// 8 = two accumulators alternate (d, d + N) as the swap-AB M-tiles do; 16 = warps 2-3 stream
// tcgen05.ld from TMEM columns 256.. meanwhile (epilogue drains); 32 = operands rotate over four
// 48 KB SMEM stages (the kernels' ring) instead of one fixed address.
// 64 = warp 2 streams 40 KB of TMA bulk copies (global -> SMEM) per 8 MMAs into the stage being
// consumed, as the producer does (SMEM write bandwidth shared with the tensor core's operand reads?).
__device__ int g_random_fill = 0;
template <int M, int N, int AMN, int BMN, int MODE = 0>
__global__ void __launch_bounds__(128) probe(long long* out, int reps, const uint8_t* gsrc = nullptr) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bar2, spin;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 196 * 1024 / 16; i += blockDim.x) {
    uint32_t x = g_random_fill ? (uint32_t)(i * 2654435761u + blockIdx.x * 40503u) : 0u;
    // random bf16 in [0.5, 1): sign 0, exponent 126, random mantissa (no NaN / Inf)
    const uint32_t lo = 0x3F00u | ((x >> 3) & 0x7F), hi = 0x3F00u | ((x >> 13) & 0x7F);
    const uint32_t w = g_random_fill ? (lo | (hi << 16)) : 0u;
    reinterpret_cast<int4*>(sm)[i] = make_int4(w, w ^ 0x00010001u, w, w ^ 0x00030003u);
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    mbar_init(&spin, 1);
    stop = 0;
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16(M, N, 1, AMN, BMN);
    if (MODE & 4) mbar_arrive(&bar2);  // completes phase 0: later waits on parity 0 return at once
    uint32_t ready_next = 1;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t st = (MODE & 32) ? (((MODE & 1024) ? (r >> 2) & 1 : (r >> 1) & 3)) * ((MODE & 1024) ? 98304 : 49152) : 0;
      const uint32_t a_base = smem_u32(sm) + st + 16384 + ((MODE & 32) ? (r & 1) * 16384 : 0), b_base = smem_u32(sm) + st;
      const int per = (MODE & 1024) ? 3 : 1;
      if ((MODE & 4) && (r & per) == 0 && !(MODE & 512)) {
        mbar_wait(&bar2, 0);
        if (!(MODE & 128)) tc_fence_after();
      }
      if ((MODE & 512) && (r & 1) == 0) {  // software-pipelined: use the probe issued one stage earlier
        if (!ready_next) mbar_wait(&bar2, 0);
        asm volatile("{ .reg .pred P; mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                     : "=r"(ready_next) : "r"(smem_u32(&bar2)), "r"(0u));
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        // K-major: rows of 128 B (64 K), +32 B per K16; MN-major: [k][64-wide chunk] boxes of 8 KB, +2 KB per K16
        uint64_t ad = AMN ? sdesc_sw128(a_base + kk * 2048, 8192, 1024) : sdesc_sw128(a_base + kk * 32, 16, 1024);
        uint64_t bd = BMN ? sdesc_sw128(b_base + kk * 2048, 8192, 1024) : sdesc_sw128(b_base + kk * 32, 16, 1024);
        if (MODE & 256) {  // descriptors as base + (offset >> 4): one add each
          const uint32_t off = st + ((MODE & 32) ? (r & 1) * 16384 : 0);
          ad = (AMN ? sdesc_sw128(smem_u32(sm) + 16384 + kk * 2048, 8192, 1024)
                    : sdesc_sw128(smem_u32(sm) + 16384 + kk * 32, 16, 1024)) + (off >> 4);
          bd = (BMN ? sdesc_sw128(smem_u32(sm) + kk * 2048, 8192, 1024) : sdesc_sw128(smem_u32(sm) + kk * 32, 16, 1024)) +
               (st >> 4);
        }
        uint32_t d = (MODE & 8) ? tmem + (uint32_t)((r & 1) * N) : tmem;
        if (MODE & 2048) {  // 4 accumulators cycling every 8 MMAs (the sweep kernel's slots)
          const int sl = (r >> 1) & 3;
          d = M == 64 ? tmem + ((uint32_t)(sl & 1) << 20) + (uint32_t)((sl >> 1) * 256)
                      : tmem + (uint32_t)(sl * 2 * N) + (uint32_t)((r & 1) * N);
        }
        umma_f16(d, ad, bd, idesc, (r | kk) != 0);
      }
      if ((MODE & 1) && (r & per) == per) umma_commit(&spin);  // never waited on
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
    stop = 1;
  } else if ((MODE & 64) && warp == 2) {
    if ((threadIdx.x & 31) == 0) {
      __shared__ uint64_t tbar[2];
      mbar_init(&tbar[0], 1);
      mbar_init(&tbar[1], 1);
      fence_mbar_init();
      uint32_t ph[2] = {0, 0};
      for (int r = 0; !stop; ++r) {
        const int b = r & 1;
        const uint32_t dst = smem_u32(sm) + (uint32_t)((r & 3) * 49152);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&tbar[b])), "r"(40960));
        for (int c = 0; c < 5; ++c)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(dst + c * 8192), "l"(gsrc + ((size_t)(r * 5 + c) % 4096) * 8192), "r"(8192),
                       "r"(smem_u32(&tbar[b])) : "memory");
        if (r >= 1) {
          mbar_wait(&tbar[b ^ 1], ph[b ^ 1]);
          ph[b ^ 1] ^= 1;
        }
      }
    }
  } else if ((MODE & 16) && warp >= 2) {
    while (!stop) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + 256, v);
      tmem_ld_wait();
      if (v[3] == 12345u) stop = 2;
    }
  } else if ((MODE & 2) && warp >= 2) {
    // spin like idle epilogue warps: try_wait on a barrier phase that does not complete
    while (!stop) {
      uint32_t ok;
      asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                   : "=r"(ok) : "r"(smem_u32(&bar2)), "r"(1u) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <int M, int N, int AMN, int BMN, int MODE = 0>
void run(const char* name, long long* d_out, int sms) {
  const int reps = 4096;
  static uint8_t* gsrc = nullptr;
  if (!gsrc) cudaMalloc(&gsrc, 32 << 20);
  cudaFuncSetAttribute(probe<M, N, AMN, BMN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  probe<M, N, AMN, BMN, MODE><<<sms, 128, 200 * 1024>>>(d_out, 16, gsrc);
  probe<M, N, AMN, BMN, MODE><<<sms, 128, 200 * 1024>>>(d_out, reps, gsrc);
  long long cyc = 0;
  cudaError_t e = cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  const double per = (double)cyc / (reps * 4);
  const double flops = 2.0 * M * N * 16;
  printf("%-34s M=%3d N=%3d A%s B%s: %7.1f cyc/MMA  %6.0f flop/cyc/SM  (%s)\n", name, M, N, AMN ? "mn" : "k ",
         BMN ? "mn" : "k ", per, flops / per, cudaGetErrorString(e));
}


__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}" : "=r"(pred));
  return pred != 0;
}

// Issue pattern of the SpMM kernels: per step of 2 M-tiles x 4 K16 MMAs, the slot (TMEM offset)
// and first-flag come from a step list in global memory and the stage index rotates.
// STYLE 0: lane 0 of warp 0 alone (divergent; ptxas waterfalls every operand into uniform regs).
// STYLE 1: the whole warp walks the list, values broadcast with __shfl_sync, MMAs under elect.sync.
template <int STYLE>
__global__ void __launch_bounds__(128) issue_probe(const int4* steps, long long* out, int n) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 196 * 1024 / 16; i += blockDim.x) reinterpret_cast<int4*>(sm)[i] = make_int4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t idesc = idesc_f16(128, 64, 1, 1, 0);
  if (STYLE == 0 && threadIdx.x == 0) {
    const long long t0 = clock64();
    int stage = 0;
    for (int i = 0; i < n; ++i) {
      const int4 st = steps[i];
      const uint32_t base = smem_u32(sm) + stage * 40960;
      const uint32_t d = tmem + st.x * 128;
      for (int mt = 0; mt < st.y; ++mt)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_f16(d + mt * 64, sdesc_sw128(base + 8192 + mt * 16384 + kk * 2048, 8192, 1024),
                   sdesc_sw128(base + kk * 32, 16, 1024), idesc, !(st.z && kk == 0));
      stage = stage == 3 ? 0 : stage + 1;
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0) out[0] = clock64() - t0;
  } else if (STYLE == 1 && warp == 0) {
    const long long t0 = clock64();
    int stage = 0;
    for (int i = 0; i < n; ++i) {
      int4 st = steps[i];
      st.x = __shfl_sync(0xffffffffu, st.x, 0);
      st.y = __shfl_sync(0xffffffffu, st.y, 0);
      st.z = __shfl_sync(0xffffffffu, st.z, 0);
      const uint32_t base = smem_u32(sm) + stage * 40960;
      const uint32_t d = tmem + st.x * 128;
      if (elect_one()) {
        for (int mt = 0; mt < st.y; ++mt)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_f16(d + mt * 64, sdesc_sw128(base + 8192 + mt * 16384 + kk * 2048, 8192, 1024),
                     sdesc_sw128(base + kk * 32, 16, 1024), idesc, !(st.z && kk == 0));
      }
      __syncwarp();
      stage = stage == 3 ? 0 : stage + 1;
    }
    if (elect_one()) umma_commit(&bar);
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <int STYLE>
void run_issue(const char* name, const int4* d_steps, int n, long long* d_out, int sms) {
  cudaFuncSetAttribute(issue_probe<STYLE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  issue_probe<STYLE><<<sms, 128, 200 * 1024>>>(d_steps, d_out, 64);
  issue_probe<STYLE><<<sms, 128, 200 * 1024>>>(d_steps, d_out, n);
  long long cyc = 0;
  cudaError_t e = cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  printf("%-44s %7.1f cyc/MMA  (%s)\n", name, (double)cyc / (n * 8), cudaGetErrorString(e));
}

// cta_group::2: the leader CTA of a 2-CTA cluster issues M=2*128 x N MMAs (each CTA holds its 128
// A rows and half of B's N rows).  ROT: operands rotate over 4 SMEM stages, with a wait/fence
// per 8 MMAs and a multicast commit (the kernels' per-stage pattern).
template <int N, int AMN, int BMN, int ROT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) probe2(long long* out, int reps) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bar2, spin;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 196 * 1024 / 16; i += blockDim.x) {
    uint32_t x = g_random_fill ? (uint32_t)(i * 2654435761u + blockIdx.x * 40503u) : 0u;
    // random bf16 in [0.5, 1): sign 0, exponent 126, random mantissa (no NaN / Inf)
    const uint32_t lo = 0x3F00u | ((x >> 3) & 0x7F), hi = 0x3F00u | ((x >> 13) & 0x7F);
    const uint32_t w = g_random_fill ? (lo | (hi << 16)) : 0u;
    reinterpret_cast<int4*>(sm)[i] = make_int4(w, w ^ 0x00010001u, w, w ^ 0x00030003u);
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    mbar_init(&spin, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_2sm<512>(&tslot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const bool leader = cluster_ctarank() == 0;
  if (threadIdx.x == 0 && leader) {
    const uint32_t idesc = idesc_f16(256, N, 1, AMN, BMN);
    if (ROT) mbar_arrive(&bar2);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t st = ROT ? ((r >> 1) & 3) * 49152 : 0;
      const uint32_t a_base = smem_u32(sm) + st + 16384, b_base = smem_u32(sm) + st;
      if (ROT && (r & 1) == 0) {
        mbar_wait(&bar2, 0);
        tc_fence_after();
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = AMN ? sdesc_sw128(a_base + kk * 2048, 8192, 1024) : sdesc_sw128(a_base + kk * 32, 16, 1024);
        const uint64_t bd = BMN ? sdesc_sw128(b_base + kk * 2048, 8192, 1024) : sdesc_sw128(b_base + kk * 32, 16, 1024);
        umma_f16_2sm(tmem, ad, bd, idesc, (r | kk) != 0);
      }
      if (ROT && (r & 1) == 1) umma_commit_2sm_mc(&spin, 3);
    }
    umma_commit_2sm_mc(&bar, 3);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  } else if (threadIdx.x == 0) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) tmem_dealloc_2sm<512>(tmem);
}

template <int N, int AMN, int BMN, int ROT>
void run2(const char* name, long long* d_out, int sms) {
  const int reps = 4096;
  cudaFuncSetAttribute(probe2<N, AMN, BMN, ROT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  probe2<N, AMN, BMN, ROT><<<sms, 128, 200 * 1024>>>(d_out, 16);
  probe2<N, AMN, BMN, ROT><<<sms, 128, 200 * 1024>>>(d_out, reps);
  long long cyc = 0;
  cudaError_t e = cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  const double per = (double)cyc / (reps * 4);
  printf("%-34s M=256 N=%3d (2-CTA): %7.1f cyc/MMA  %6.0f flop/cyc/SM  (%s)\n", name, N, per,
         2.0 * 128 * N * 16 / per, cudaGetErrorString(e));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d_out;
  cudaMalloc(&d_out, 64);
  for (int rf = 0; rf < 2; ++rf) {
  cudaMemcpyToSymbol(g_random_fill, &rf, sizeof(int));
  printf("---- SMEM operands: %s\n", rf ? "random bf16 in [0.5, 1)" : "zeros");
  run<128, 64, 1, 0>("swap-AB (short kernel today)", d_out, sms);
  run<64, 256, 0, 1>("rows-as-M M=64 (tile K, B mn)", d_out, sms);
  run<128, 256, 0, 1>("tall-like 1-CTA (A K, B mn)", d_out, sms);
  run<128, 64, 1, 0, 63 + 128 + 256>("swap everything, no fence, desc add", d_out, sms);
  run<64, 256, 0, 1, 63 + 128 + 256>("M=64 everything, no fence, desc add", d_out, sms);
  run<64, 256, 0, 1, 63 + 128 + 256 + 2048>("M=64 everything + 4 slots", d_out, sms);
  run<128, 64, 1, 0, 63 + 128 + 256 + 2048>("swap everything + 4 slots", d_out, sms);
  run<64, 256, 0, 1, 2048>("M=64 only 4 slots", d_out, sms);
  run<128, 64, 1, 0, 2048>("swap only 4 slots", d_out, sms);
  }
  run<128, 64, 1, 0>("swap-AB (short kernel today)", d_out, sms);
  run<128, 64, 0, 0>("swap-AB, both K-major", d_out, sms);
  run<128, 128, 1, 0>("swap-AB N=128", d_out, sms);
  run<128, 256, 1, 0>("swap-AB N=256", d_out, sms);
  run<128, 32, 1, 0>("swap-AB N=32", d_out, sms);
  run<128, 16, 1, 0>("swap-AB N=16", d_out, sms);
  run<64, 256, 0, 1>("rows-as-M M=64 (tile K, B mn)", d_out, sms);
  run<64, 128, 0, 1>("rows-as-M M=64 N=128", d_out, sms);
  run<128, 256, 0, 1>("tall-like 1-CTA (A K, B mn)", d_out, sms);
  run<128, 128, 0, 1>("tall-like N=128", d_out, sms);
  run<128, 64, 0, 1>("tall-like N=64", d_out, sms);
  run<128, 64, 1, 0, 1>("swap +commit/8", d_out, sms);
  run<128, 64, 1, 0, 2>("swap +spinning warps", d_out, sms);
  run<128, 64, 1, 0, 4>("swap +wait/fence per 8", d_out, sms);
  run<128, 64, 1, 0, 8>("swap +2 accumulators", d_out, sms);
  run<128, 64, 1, 0, 15>("swap all of the above", d_out, sms);
  run<128, 64, 1, 0, 16>("swap +concurrent tcgen05.ld", d_out, sms);
  run<128, 64, 1, 0, 32>("swap +4 rotating SMEM stages", d_out, sms);
  run<128, 64, 1, 0, 40>("swap +4 stages +2 accumulators", d_out, sms);
  run<128, 64, 1, 0, 63>("swap everything", d_out, sms);
  run<128, 64, 1, 0, 4 + 128>("swap +wait per 8, no fence", d_out, sms);
  run<128, 64, 1, 0, 32 + 256>("swap +4 stages, desc by add", d_out, sms);
  run<128, 64, 1, 0, 63 + 128 + 256>("swap everything, no fence, desc add", d_out, sms);
  run<128, 64, 1, 0, 4 + 512>("swap +test_wait per 8", d_out, sms);
  run<128, 64, 1, 0, 63 + 256 + 1024>("swap everything, syncs per 16, desc add", d_out, sms);
  run<128, 64, 1, 0, 5 + 1024>("swap wait+commit per 16", d_out, sms);
  run<128, 64, 1, 0, 1 + 4 + 512 + 32 + 256 + 128>("swap pipelined test_wait+commit+stages(add)", d_out, sms);
  run<128, 64, 1, 0, 1 + 4 + 32 + 256 + 128>("swap blocking wait+commit+stages(add)", d_out, sms);
  run<128, 256, 0, 1, 32>("tall-like N=256 +4 stages", d_out, sms);
  run<128, 64, 1, 0, 64>("swap +TMA writes 40KB/8 MMA", d_out, sms);
  run<128, 64, 1, 0, 96>("swap +TMA writes +4 stages", d_out, sms);
  run<128, 256, 0, 1, 96>("tall-like N=256 +TMA +4 stages", d_out, sms);
  run<128, 256, 0, 1, 15>("tall-like N=256 all of the above", d_out, sms);
  run2<64, 1, 0, 0>("2-CTA swap N=64", d_out, sms);
  run2<64, 1, 0, 1>("2-CTA swap N=64 +rot/wait/commit", d_out, sms);
  run2<128, 1, 0, 0>("2-CTA swap N=128", d_out, sms);
  run2<256, 0, 1, 1>("2-CTA tall N=256 +rot", d_out, sms);
  const int n = 4096;
  int4* h = new int4[n];
  for (int i = 0; i < n; ++i) h[i] = make_int4(i % 4, 2, (i % 41) == 0, 0);
  int4* d_steps;
  cudaMalloc(&d_steps, sizeof(int4) * n);
  cudaMemcpy(d_steps, h, sizeof(int4) * n, cudaMemcpyHostToDevice);
  run_issue<0>("issue from lane 0 (kernel style today)", d_steps, n, d_out, sms);
  run_issue<1>("issue from converged warp + shfl + elect", d_steps, n, d_out, sms);
  return 0;
}
