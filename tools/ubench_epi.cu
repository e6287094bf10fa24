// Microbenchmarks for the fused forward's epilogue design (diagnostics only):
//   1. tcgen05.ld (32x32b.x32) throughput per SM with W warps (W/4 per lane quarter)
//   2. mma.sync m16n8k16 bf16 throughput per SM with W warps
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench tools/ubench_epi.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include "../paper_2211_03578_b200/csrc/tc_ptx.cuh"

__global__ void tmem_ld_bench(int iters, int ncols_per_ld2, long long* cyc, float* sink) {
  __shared__ uint32_t tptr;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc(tc::smem_u32(&tptr), 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tl = tptr + ((32u * (warp & 3)) << 16);
  const uint32_t col0 = 64u * ((warp >> 2) & 7);
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    float v0[32], v1[32];
    tc::tmem_ld32(tl + col0, v0);
    tc::tmem_ld32(tl + col0 + 32, v1);
    tc::tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 32; ++j) acc += v0[j] + v1[j];
  }
  long long t1 = clock64();
  __syncthreads();
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tptr, 512);
}

__global__ void hmma_bench(int iters, long long* cyc, float* sink) {
  const int warp = threadIdx.x >> 5;
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  float d[4][4] = {};
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) tc::mma16816(d[j], a, a[j & 1] + i, a[2 + (j & 1)]);
  }
  long long t1 = clock64();
  __syncthreads();
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  float s = 0.f;
  for (int j = 0; j < 4; ++j) for (int k = 0; k < 4; ++k) s += d[j][k];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  long long* cyc; float* sink;
  cudaMalloc(&cyc, 148 * 32 * sizeof(long long));
  cudaMalloc(&sink, 148 * 1024 * sizeof(float));
  long long h[32];
  const int iters = 4096;
  for (int W : {4, 8, 16}) {
    tmem_ld_bench<<<148, 32 * W>>>(iters, 64, cyc, sink);
    tmem_ld_bench<<<148, 32 * W>>>(iters, 64, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int w = 0; w < W; ++w) mx = h[w] > mx ? h[w] : mx;
    const double bytes = (double)W * iters * 64 * 32 * 4;
    printf("tmem ld  W=%2d: %lld cyc, %.1f B/cyc/SM, %.1f cyc per 64-col ld pair per warp (%s)\n", W, mx,
           bytes / mx, (double)mx / iters, cudaGetErrorString(e));
  }
  for (int W : {4, 8, 16}) {
    hmma_bench<<<148, 32 * W>>>(iters, cyc, sink);
    hmma_bench<<<148, 32 * W>>>(iters, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int w = 0; w < W; ++w) mx = h[w] > mx ? h[w] : mx;
    const double flops = (double)W * iters * 4 * 16 * 8 * 16 * 2;
    printf("mma.sync W=%2d: %lld cyc, %.0f flop/cyc/SM, %.2f cyc per HMMA per SMSP (%s)\n", W, mx,
           flops / mx, (double)mx / (iters * 4.0 * W / 4), cudaGetErrorString(e));
  }
  return 0;
}
