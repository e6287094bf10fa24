// Probe: kind::tf32 / kind::f16 tcgen05.mma with BOTH operands MN-major in the
// SWIZZLE_128B canonical layout (the layout a 2-D TMA box of [32 rows x 128 B]
// with 128B swizzle produces).  Standalone diagnostic for the wgrad kernel:
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tf32_sw128_probe tools/tf32_sw128_probe.cu
//   tools/tf32_sw128_probe <elem 2|4> <lbo> <sbo> <ltype>
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

// At[K][128], Bt[K][N] row-major fp32 in global; D[128][N]
__global__ void probe(const float* At, const float* Bt, float* D, int N, int K, int elem, uint32_t lbo,
                      uint32_t sbo, uint32_t ltype) {
  extern __shared__ uint8_t raw[];
  const uint32_t r0 = tc::smem_u32(raw);
  uint8_t* sm = raw + (((r0 + 1023) & ~1023u) - r0);
  const uint32_t sb = tc::smem_u32(sm);
  const int T = 128 / elem;  // elements per 128-byte swizzle row
  // MN-major SW128: element (mn, k) -> atom column mn / T (stride LBO_layout),
  // k group k / 8 (stride 1024), row k % 8 (128 B), 16-byte chunk ((mn % T) / (16/elem)) ^ (k % 8)
  const int kgroups = K / 8;
  // ltype 1 (SWIZZLE_128B_BASE32B): 32-byte chunks XOR (k % 4) -- what a TMA box
  // with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B writes
  auto off = [&](int mn, int k) {
    const int col = mn / T, w = mn % T;
    if (ltype == 1) {
      const int byte = w * elem, ch = byte >> 5;
      return (uint32_t)(col * kgroups * 1024 + k * 128 + ((ch ^ (k % 4)) << 5) + (byte & 31));
    }
    const int ch = w / (16 / elem), e = w % (16 / elem);
    return (uint32_t)(col * kgroups * 1024 + (k / 8) * 1024 + (k % 8) * 128 + ((ch ^ (k % 8)) << 4) + e * elem);
  };
  const uint32_t offB = 128 * K * elem;
  for (int i = threadIdx.x; i < 128 * K; i += blockDim.x) {
    const int k = i / 128, mn = i % 128;
    if (elem == 2) *reinterpret_cast<__nv_bfloat16*>(sm + off(mn, k)) = __float2bfloat16_rn(At[i]);
    else *reinterpret_cast<float*>(sm + off(mn, k)) = At[i];
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int k = i / N, mn = i % N;
    if (elem == 2) *reinterpret_cast<__nv_bfloat16*>(sm + offB + off(mn, k)) = __float2bfloat16_rn(Bt[i]);
    else *reinterpret_cast<float*>(sm + offB + off(mn, k)) = Bt[i];
  }
  const uint32_t offBar = offB + N * K * elem + 1024;
  uint32_t* tp = reinterpret_cast<uint32_t*>(sm + offBar + 64);
  if (threadIdx.x == 0) { tc::mbar_init(sb + offBar, 1); tc::fence_barrier_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(tc::smem_u32(tp), 256);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = *tp;
  if (threadIdx.x == 0) {
    const uint32_t fmt = elem == 2 ? 1u : 2u;
    const uint32_t id = (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 15) | (1u << 16) | ((N >> 3) << 17) |
                        ((128 >> 4) << 24);
    const int kstep = 32 / elem;
    for (int ks = 0; ks < K; ks += kstep) {
      const uint32_t ko = (ks / 8) * 1024 + (ks % 8) * 128;
      uint64_t ad = tc::smem_desc(sb + ko, lbo, sbo) | ((uint64_t)ltype << 61);
      uint64_t bd = tc::smem_desc(sb + offB + ko, lbo, sbo) | ((uint64_t)ltype << 61);
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
  const int elem = atoi(argv[1]);
  const uint32_t lbo = atoi(argv[2]), sbo = atoi(argv[3]), ltype = atoi(argv[4]);
  const int N = 64, K = 32;
  std::vector<float> At(K * 128), Bt(K * N), D(128 * N);
  srand(1);
  for (auto& x : At) x = (float)(rand() % 17 - 8) / 8.f;
  for (auto& x : Bt) x = (float)(rand() % 17 - 8) / 8.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, At.size() * 4); cudaMalloc(&dB, Bt.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, At.data(), At.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bt.data(), Bt.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  const int smem = 128 * K * 4 + N * K * 4 + 4096;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dA, dB, dD, N, K, elem, lbo, sbo, ltype);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double mx = 0, mref = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0;
      for (int k = 0; k < K; ++k) r += (double)At[k * 128 + m] * Bt[k * N + n];
      mx = fmax(mx, fabs(r - D[m * N + n]));
      mref = fmax(mref, fabs(r));
    }
  printf("elem %d lbo %u sbo %u ltype %u: %s max err %.3g (ref %.3g) D[0..3] %.3f %.3f %.3f\n", elem, lbo, sbo, ltype,
         cudaGetErrorString(e), mx, mref, D[0], D[1], D[2]);
  return 0;
}
