// Probe: which UMMA descriptor encoding makes an MN-major (transposed) B operand
// work for kind::f16 and kind::tf32 (no swizzle).  Standalone diagnostic.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include "../paper_2211_03578_b200/csrc/tc_ptx.cuh"

__device__ __forceinline__ void mma_f16_(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}

// elem: 2 (bf16) or 4 (tf32).  A: [128][K] K-major.  B given as Bt[K][N] (MN-major).
// variant 0: LBO = K-group stride, SBO = MN-group stride; variant 1: swapped.
__global__ void probe(const float* A, const float* Bt, float* D, int N, int K, int elem, int variant,
                      int layout_kgroup_outer) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t sb = tc::smem_u32(sm);
  const int T = 16 / elem;  // elements per 16B
  const uint32_t offB = 128 * K * elem;
  // A K-major canonical: (r,k) -> (r/8)*(K*16/T... ) use generic: core = 8 rows x 16B
  for (int e = threadIdx.x; e < 128 * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    uint32_t off = (r / 8) * (K / T) * 128 + (k / T) * 128 + (r % 8) * 16 + (k % T) * elem;
    if (elem == 2) *reinterpret_cast<__nv_bfloat16*>(sm + off) = __float2bfloat16_rn(A[e]);
    else *reinterpret_cast<float*>(sm + off) = A[e];
  }
  // B MN-major canonical: element (n,k): core = 8 K-rows x 16B (T MN elems)
  const int ngroups = N / T, kgroups = K / 8;
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    int k = e / N, n = e % N;  // Bt[k][n]
    uint32_t off;
    if (layout_kgroup_outer) off = (k / 8) * (ngroups * 128) + (n / T) * 128 + (k % 8) * 16 + (n % T) * elem;
    else off = (n / T) * (kgroups * 128) + (k / 8) * 128 + (k % 8) * 16 + (n % T) * elem;
    if (elem == 2) *reinterpret_cast<__nv_bfloat16*>(sm + offB + off) = __float2bfloat16_rn(Bt[e]);
    else *reinterpret_cast<float*>(sm + offB + off) = Bt[e];
  }
  const uint32_t offBar = offB + N * K * elem, offT = offBar + 8;
  uint32_t* tp = reinterpret_cast<uint32_t*>(sm + offT);
  if (threadIdx.x == 0) { tc::mbar_init(sb + offBar, 1); tc::fence_barrier_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(tc::smem_u32(tp), 256);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = *tp;
  if (threadIdx.x == 0) {
    const uint32_t fmt = elem == 2 ? 1u : 2u;
    const uint32_t id = (1u << 4) | (fmt << 7) | (fmt << 10) | (0u << 15) | (1u << 16) | ((N >> 3) << 17) | ((128 >> 4) << 24);
    const int kstep = 32 / elem;
    uint32_t kgs = layout_kgroup_outer ? ngroups * 128 : 128;     // K-group stride
    uint32_t mgs = layout_kgroup_outer ? 128 : kgroups * 128;     // MN-group stride
    for (int ks = 0; ks < K; ks += kstep) {
      uint64_t ad = tc::smem_desc(sb + (ks / T) * 128, 128, (K / T) * 128);
      uint32_t bstart = sb + offB + (ks / 8) * kgs;
      uint64_t bd = variant == 0 ? tc::smem_desc(bstart, kgs, mgs) : tc::smem_desc(bstart, mgs, kgs);
      if (elem == 2) mma_f16_(tm, ad, bd, id, ks > 0);
      else tc::mma_tf32(tm, ad, bd, id, ks > 0);
    }
    tc::mma_commit(sb + offBar);
  }
  tc::mbar_wait(sb + offBar, 0);
  tc::tc_fence_after();
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  for (int c = 0; c < N; c += 32) {
    float v[32];
    tc::tmem_ld32(tm + ((32 * w) << 16) + c, v);
    tc::tmem_wait_ld();
    for (int i = 0; i < 32 && c + i < N; ++i) D[(32 * w + ln) * N + c + i] = v[i];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc::tc_fence_after(); tc::tmem_dealloc(tm, 256); }
}

int main(int argc, char** argv) {
  const int N = 64;
  const int elem = atoi(argv[1]), K = atoi(argv[2]), lay0 = atoi(argv[3]), var0 = atoi(argv[4]);
  {
    {
      std::vector<float> A(128 * K), Bt(K * N), ref(128 * N);
      for (auto& x : A) x = (rand() % 9 - 4) * 0.25f;
      for (auto& x : Bt) x = (rand() % 9 - 4) * 0.25f;
      for (int i = 0; i < 128; ++i)
        for (int j = 0; j < N; ++j) {
          double s = 0;
          for (int k = 0; k < K; ++k) s += A[i * K + k] * Bt[k * N + j];
          ref[i * N + j] = (float)s;
        }
      float *dA, *dB, *dD;
      cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, Bt.size() * 4); cudaMalloc(&dD, 128 * N * 4);
      cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
      cudaMemcpy(dB, Bt.data(), Bt.size() * 4, cudaMemcpyHostToDevice);
      const size_t smem = 128 * K * elem + N * K * elem + 64;
      cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int lay = lay0; lay <= lay0; ++lay)
        for (int var = var0; var <= var0; ++var) {
          cudaMemset(dD, 0, 128 * N * 4);
          probe<<<1, 128, smem>>>(dA, dB, dD, N, K, elem, var, lay);
          cudaError_t e = cudaDeviceSynchronize();
          std::vector<float> D(128 * N);
          cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
          double err = 0, mx = 0;
          for (int i = 0; i < 128 * N; ++i) { err = fmax(err, fabs(D[i] - ref[i])); mx = fmax(mx, fabs(ref[i])); }
          printf("elem=%d K=%d layout_kgroup_outer=%d variant=%d  err=%s  maxerr=%.4g (max %.3g) D00=%g ref00=%g\n",
                 elem, K, lay, var, cudaGetErrorString(e), err, mx, D[0], ref[0]);
        }
      cudaFree(dA); cudaFree(dB); cudaFree(dD);
    }
  }
  return 0;
}
