// Microbenchmark (diagnostics only): tcgen05.mma kind::f16 M=128 issue rate as
// the fused forward uses it -- A from shared memory (canonical no-swizzle,
// Kt = 256) or from TMEM, B = N x 64 canonical chunks -- with and without a
// concurrent 1-D bulk-TMA stream into another shared-memory region.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_umma tools/ubench_umma.cu -lcuda
#include <cstdio>
#include <vector>
#include <cstdint>
#include <cuda_bf16.h>
#include "../paper_2211_03578_b200/csrc/tc_ptx.cuh"

constexpr uint32_t kA = 0, kB = 65536, kRing = 65536 + 16384, kBar = kRing + 16384;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\t"
      "elect.sync rx|px, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, px;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__global__ void __launch_bounds__(128, 1) umma_bench(int N, int a_tmem, int tma, int iters, int nacc,
                                                     const uint8_t* gsrc, long long* out, int nis, int ncols) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tptr;
  const uint32_t sb = tc::smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (int)(kRing / 16); i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 10; ++i) tc::mbar_init(sb + kBar + 8 * i, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc(tc::smem_u32(&tptr), ncols);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tptr;
  volatile int* stop = reinterpret_cast<volatile int*>(smem + kBar + 64);
  if (threadIdx.x == 0) *stop = 0;
  __syncthreads();
  if (warp < nis) {  // whole warp runs the issue loop (warp-uniform values), one elected lane issues
    const uint32_t idesc = tc::idesc_bf16(128, N);
    const uint64_t a0 = tc::smem_desc(sb + kA, 128, 256 * 16);
    const uint64_t b0 = tc::smem_desc(sb + kB, 128, 64 * 16);
    __syncwarp();
    const long long t0 = clock64();
    for (int i = 0; i < iters; i += 16) {
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) {
        const uint64_t bd = b0 + (uint64_t)(((ks & 3) * 2 * 128) >> 4);
        const uint32_t d = tmem + (uint32_t)(warp * (ncols / nis)) + (nacc == 1 ? 0u : (uint32_t)((ks % 2) * 256));
        if (elect_one()) {
          if (a_tmem)
            tc::mma_bf16_ta(d, tmem + (ncols - 128) + ks * 8, bd, idesc, (i + ks) >= nacc);
          else
            tc::mma_bf16(d, a0 + (uint64_t)((ks * 2 * 128) >> 4), bd, idesc, (i + ks) >= nacc);
        }
        __syncwarp();
      }
    }
    if (elect_one()) tc::mma_commit(sb + kBar + 40 + 8 * warp);
    __syncwarp();
    tc::mbar_wait(sb + kBar + 40 + 8 * warp, 0);
    const long long t1 = clock64();
    if (lane == 0) {
      out[blockIdx.x * 4 + warp] = t1 - t0;
      *stop = 1;
    }
  } else if (warp == 3 && lane == 0 && tma) {
    uint32_t cnt[4] = {0, 0, 0, 0};
    long long bytes = 0;
    for (int i = 0; !*stop; ++i) {
      const int st = i & 3;
      if (cnt[st]) tc::mbar_wait(sb + kBar + 8 * st, (cnt[st] - 1) & 1);
      tc::mbar_arrive_expect_tx(sb + kBar + 8 * st, 16384);
      tc::bulk_g2s(sb + kRing + st * 16384, gsrc + (size_t)(i & 63) * 16384, 16384, sb + kBar + 8 * st);
      ++cnt[st];
      bytes += 16384;
    }
    for (int st = 0; st < 4; ++st)
      if (cnt[st]) tc::mbar_wait(sb + kBar + 8 * st, (cnt[st] - 1) & 1);
    out[gridDim.x + blockIdx.x] = bytes;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}

int main() {
  long long* out;
  uint8_t* src;
  cudaMalloc(&out, 8 * 4 * 148 * sizeof(long long));
  cudaMalloc(&src, 64 * 16384);
  cudaMemset(src, 0, 64 * 16384);
  const int iters = 4096;
  // (ctas per SM, issuers per CTA)
  const int cfgs[4][2] = {{1, 1}, {1, 2}, {2, 1}, {1, 4}};
  for (auto& cf : cfgs) {
    const int cps = cf[0], nis = cf[1];
    const int smem = cps == 1 ? 160 * 1024 : 100 * 1024;
    cudaFuncSetAttribute(umma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int ncols = cps == 1 ? 512 : 256;
    for (int a_tmem : {0, 1})
      for (int N : {64, 96, 128, 256}) {
        if (N * nis + (a_tmem ? 128 : 0) > ncols) continue;
        const int grid = 148 * cps;
        umma_bench<<<grid, 128, smem>>>(N, a_tmem, 0, iters, 1, src, out, nis, ncols);
        umma_bench<<<grid, 128, smem>>>(N, a_tmem, 0, iters, 1, src, out, nis, ncols);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<long long> h(grid * 4);
        cudaMemcpy(h.data(), out, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int b = 0; b < grid; ++b)
          for (int w = 0; w < nis; ++w) mx = h[b * 4 + w] > mx ? h[b * 4 + w] : mx;
        const double per_sm = (double)mx / (iters * (double)nis * cps);  // cycles per MMA per SM
        printf("ctas/SM=%d issuers=%d A=%s N=%3d: %.1f cyc per MMA per SM (floor %.0f)  %s\n", cps, nis,
               a_tmem ? "tmem" : "smem", N, per_sm, 128.0 * N / 256.0, cudaGetErrorString(e));
      }
  }
  return 0;
}
