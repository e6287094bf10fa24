// Probe (diagnostics only): semantics of tcgen05.mma.cta_group::2 (two SMs of a
// cluster computing one M = 256 tile) as the next fused-forward design would
// use it.  D[256 x N] = A[256 x K] * B[N x K]^T, bf16 in, fp32 out.
//   CTA c of the pair holds A rows [128c, 128c + 128) in its SMEM (K-major,
//   canonical no-swizzle) and, depending on MODE, B rows [c*N/2, (c+1)*N/2)
//   (MODE 0: B split by N) or the whole B (MODE 1); the leader (rank 0) issues
//   the MMAs; a multicast commit signals both CTAs; each CTA reads its 128
//   TMEM lanes x N columns.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/umma2sm_probe tools/umma2sm_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include "../paper_2211_03578_b200/csrc/tc_ptx.cuh"

constexpr int K = 64;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe(const float* A, const float* B, float* D, int N, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tptr;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t rank = cta_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sb = tc::smem_u32(smem);
  const uint32_t a_off = 0, b_off = 128 * K * 2;
  // A rows of this CTA
  for (int e = threadIdx.x; e < 128 * K; e += 128) {
    const int r = e / K, k = e % K;
    *reinterpret_cast<__nv_bfloat16*>(smem + a_off + tc::canon_off(r, k, K)) =
        __float2bfloat16_rn(A[(128 * rank + r) * K + k]);
  }
  const int nb = mode == 0 ? N / 2 : N;   // B rows held by this CTA
  const int b0 = mode == 0 ? rank * (N / 2) : 0;
  for (int e = threadIdx.x; e < nb * K; e += 128) {
    const int r = e / K, k = e % K;
    *reinterpret_cast<__nv_bfloat16*>(smem + b_off + tc::canon_off(r, k, K)) =
        __float2bfloat16_rn(B[(b0 + r) * K + k]);
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(tc::smem_u32(&bar), 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tptr)),
                 "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = tptr;
  if (rank == 0 && threadIdx.x == 0) {
    // M = 256 (cta_group::2): idesc M field = 256 >> 4
    const uint32_t idesc = tc::idesc_bf16(256, N);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t ad = tc::smem_desc(sb + a_off + ks * 2 * 128, 128, K * 16);
      const uint64_t bd = tc::smem_desc(sb + b_off + ks * 2 * 128, 128, K * 16);
      const uint32_t en = ks > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(en)
          : "memory");
    }
    const uint16_t mask = 0x3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            tc::smem_u32(&bar)),
        "h"(mask)
        : "memory");
  }
  tc::mbar_wait(tc::smem_u32(&bar), 0);
  tc::tc_fence_after();
  for (int c = 0; c < N; c += 32) {
    float v[32];
    tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + c, v);
    tc::tmem_wait_ld();
    for (int i = 0; i < 32; ++i) D[(128 * rank + 32 * warp + lane) * N + c + i] = v[i];
  }
  tc::tc_fence_before();
  cluster_sync();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
}

// timing: the leader issues `iters` back-to-back MMAs (M = 256, N, K = 16 each)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
rate(int N, int iters, long long* out, int a_tmem) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tptr;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t rank = cta_rank();
  const int warp = threadIdx.x >> 5;
  const uint32_t sb = tc::smem_u32(smem);
  for (int e = threadIdx.x; e < (128 * K * 2 + 128 * K * 2) / 16; e += 128)
    reinterpret_cast<uint4*>(smem)[e] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  if (threadIdx.x == 0) { tc::mbar_init(tc::smem_u32(&bar), 1); tc::fence_barrier_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tptr)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = tptr;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t idesc = tc::idesc_bf16(256, N);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int ks = i & 3;
      const uint64_t bd = tc::smem_desc(sb + 128 * K * 2 + ks * 2 * 128, 128, K * 16);
      if (a_tmem) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256),
                     "r"(tmem + 384 + ks * 8), "l"(bd), "r"(idesc), "r"((uint32_t)(i > 0)) : "memory");
      } else {
        const uint64_t ad = tc::smem_desc(sb + ks * 2 * 128, 128, K * 16);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(i > 0)) : "memory");
      }
    }
    const uint16_t mask = 0x3;
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(tc::smem_u32(&bar)), "h"(mask) : "memory");
    tc::mbar_wait(tc::smem_u32(&bar), 0);
    out[blockIdx.x / 2] = clock64() - t0;
  } else {
    tc::mbar_wait(tc::smem_u32(&bar), 0);
  }
  tc::tc_fence_before();
  cluster_sync();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

int main() {
  {
    long long* out;
    cudaMalloc(&out, 148 * sizeof(long long));
    const int smem = 128 * K * 2 * 2;
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int a_tmem : {0, 1})
      for (int N : {96, 128, 192, 256}) {
        const int iters = 4096;
        rate<<<148, 128, smem>>>(N, iters, out, a_tmem);
        rate<<<148, 128, smem>>>(N, iters, out, a_tmem);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[74];
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 74; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("cta_group::2 A=%s N=%3d: %.1f cycles per M=256 MMA (= %.1f per SM-tile of 128 rows) %s\n",
               a_tmem ? "tmem" : "smem", N, (double)mx / iters, (double)mx / iters / 2, cudaGetErrorString(e));
      }
  }
  for (int mode : {0, 1})
    for (int N : {64, 128, 256}) {
      std::vector<float> hA(256 * K), hB(N * K), hD(256 * N, -1.f);
      srand(1);
      for (auto& x : hA) x = (float)(rand() % 17 - 8) / 8.f;
      for (auto& x : hB) x = (float)(rand() % 17 - 8) / 8.f;
      float *A, *B, *D;
      cudaMalloc(&A, hA.size() * 4); cudaMalloc(&B, hB.size() * 4); cudaMalloc(&D, hD.size() * 4);
      cudaMemcpy(A, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice);
      cudaMemcpy(B, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice);
      cudaMemset(D, 0, hD.size() * 4);
      const int smem = 128 * K * 2 + N * K * 2;
      cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      probe<<<2, 128, smem>>>(A, B, D, N, mode);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(hD.data(), D, hD.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0, mx = 0;
      for (int m = 0; m < 256; ++m)
        for (int n = 0; n < N; ++n) {
          double ref = 0;
          for (int k = 0; k < K; ++k) ref += (double)hA[m * K + k] * hB[n * K + k];
          err = fmax(err, fabs(ref - hD[m * N + n]));
          mx = fmax(mx, fabs(ref));
        }
      printf("mode %d (B %s) N=%3d: max |err| %.3g (max |ref| %.3g) %s\n", mode,
             mode == 0 ? "split by N" : "whole in each CTA", N, err, mx, cudaGetErrorString(e));
      cudaFree(A); cudaFree(B); cudaFree(D);
      if (e != cudaSuccess) return 1;
    }
  return 0;
}
