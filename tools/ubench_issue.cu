// Issue-rate probe for tcgen05.mma (M = 128, K = 16 bf16) from ONE thread:
// does the ~108-cycle-per-MMA floor measured by ubench_umma.cu at N <= 192
// depend on (a) the shared-memory layout mode of the operands (SWIZZLE_NONE
// canonical vs SWIZZLE_128B), (b) the issue loop (a per-MMA elect.sync +
// __syncwarp vs one lane issuing a fully unrolled run), (c) N.
// Operand values are constant (bf16 1.0), so the layout only affects timing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_issue tools/ubench_issue.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_bf16.h>
#include "../paper_2211_03578_b200/csrc/tc_ptx.cuh"

__device__ __forceinline__ uint64_t with_layout(uint64_t d, int swz) {
  if (!swz) return d;
  // SWIZZLE_128B (layout type 2 in [61,64)), SBO = 1024 (8 rows x 128 B), LBO unused (1)
  d &= ~(((uint64_t)0x3FFF << 16) | ((uint64_t)0x3FFF << 32));
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int MODE>  // 0: whole warp, elect per MMA; 1: lane 0 issues 16 unrolled MMAs
__global__ void __launch_bounds__(128, 1) issue_bench(int N, int a_tmem, int swz, int iters, int nacc,
                                                      long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tptr;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t sb = (tc::smem_u32(smem) + 1023u) & ~1023u;
  uint8_t* sm = smem + (sb - tc::smem_u32(smem));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 48 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
  if (threadIdx.x == 0) {
    tc::mbar_init(tc::smem_u32(&bar), 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc(tc::smem_u32(&tptr), 512);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tptr;
  if (warp == 1) {
    const uint32_t idesc = tc::idesc_bf16(128, N);
    // A: 128 x 64 tile at sb, B: N x 64 at sb + 16 KB
    const uint64_t a0 = with_layout(tc::smem_desc(sb, 128, 64 * 16), swz);
    const uint64_t b0 = with_layout(tc::smem_desc(sb + 16384, 128, 64 * 16), swz);
    // K step of 16 elements: +256 B (2 core matrices) unswizzled, +32 B inside the 128-B row swizzled
    const uint64_t kstep = swz ? (32 >> 4) : (256 >> 4);
    __syncwarp();
    const long long t0 = clock64();
    if (MODE == 0) {
      for (int i = 0; i < iters; i += 16) {
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
          const uint64_t kk = (uint64_t)(ks & 3) * kstep;
          const uint32_t d = tmem + (nacc == 1 ? 0u : (uint32_t)((ks % 2) * 256));
          uint32_t pred = 0;
          asm volatile("{\n\t.reg .pred px;\n\telect.sync _|px, 0xffffffff;\n\tselp.u32 %0, 1, 0, px;\n\t}"
                       : "=r"(pred));
          if (pred) {
            if (a_tmem) tc::mma_bf16_ta(d, tmem + 256 + ks * 8, b0 + kk, idesc, 1);
            else tc::mma_bf16(d, a0 + kk, b0 + kk, idesc, 1);
          }
          __syncwarp();
        }
      }
    } else if (lane == 0) {
      for (int i = 0; i < iters; i += 16) {
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
          const uint64_t kk = (uint64_t)(ks & 3) * kstep;
          const uint32_t d = tmem + (nacc == 1 ? 0u : (uint32_t)((ks % 2) * 256));
          if (a_tmem) tc::mma_bf16_ta(d, tmem + 256 + ks * 8, b0 + kk, idesc, 1);
          else tc::mma_bf16(d, a0 + kk, b0 + kk, idesc, 1);
        }
      }
    }
    if (lane == 0) tc::mma_commit(tc::smem_u32(&bar));
    __syncwarp();
    tc::mbar_wait(tc::smem_u32(&bar), 0);
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

int main() {
  long long* out;
  cudaMalloc(&out, 148 * sizeof(long long));
  const int iters = 4096, smem = 1024 + 48 * 1024;
  auto run = [&](auto kern, const char* mode) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int swz : {0, 1})
      for (int a_tmem : {0, 1})
        for (int nacc : {1, 2})
          for (int N : {64, 96, 128, 192, 256}) {
            if (nacc == 2 && N > 256) continue;
            kern<<<148, 128, smem>>>(N, a_tmem, swz, iters, nacc, out);
            kern<<<148, 128, smem>>>(N, a_tmem, swz, iters, nacc, out);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<long long> h(148);
            cudaMemcpy(h.data(), out, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (long long v : h) mx = v > mx ? v : mx;
            printf("%s swz=%d A=%s nacc=%d N=%3d: %6.1f cyc/MMA (floor %3.0f) %s\n", mode, swz,
                   a_tmem ? "tmem" : "smem", nacc, N, (double)mx / iters, 128.0 * N / 256.0,
                   cudaGetErrorString(e));
          }
  };
  run(issue_bench<0>, "elect ");
  run(issue_bench<1>, "lane0 ");
  return 0;
}
