// Generic tcgen05 GEMM (kind::f16, bf16 operands, fp32 accumulate) for the
// training path of TLP_PREC_BF16 contexts: every dense layer of the forward,
// every dgrad and every wgrad of the backward ("the loss is
// back-propagated to update the weights").
//
//   C[M,N] = epi( op(A)[M,K] * op(B)[K,N] )      fp32 in HBM, bf16 on the tensor core
//
// op(A) = A (row-major [M][K] -> K-major UMMA operand) or A^T (A stored [K][M]
// -> MN-major operand); op(B) likewise (B stored [K][N] -> MN-major, B^T
// stored [N][K] -> K-major).  Operands are read as fp32 (float4 when aligned),
// rounded to bf16 (RN, R28) in registers and stored into the UMMA no-swizzle
// canonical layouts of a 2-stage smem ring as hi + lo pairs ("bf16x3": three
// MMAs per k-step recover fp32-class accuracy); one thread issues tcgen05.mma
// (M=128, N=128, K=16) into a 128-column TMEM accumulator and tcgen05.commit
// frees each stage; global loads for k-block i+2 are in flight while the
// tensor core works on block i.  (kind::tf32 cannot take an MN-major operand
// in the no-swizzle layout -- tools/mn_major_probe.cu -- hence bf16.)
// Epilogue: TMEM -> registers -> smem transpose -> coalesced fp32 row stores
// with bias / residual / ReLU / ReLU-mask / accumulate.  blockIdx.z splits K into fixed slices (wgrad over
// the 204,800 rows of a step); the caller reduces the partials in a fixed
// order, so training stays deterministic.
#include "tlp_internal.cuh"
#include "tc_ptx.cuh"

#include <algorithm>

namespace {

constexpr int BM = 128, BN = 128, BK = 32, STAGES = 2, THREADS = 256;
constexpr uint32_t TILE_BYTES = BM * BK * 2;                 // 8 KB (A) == BN*BK*2 (B)
// stage = [A_hi][B_hi][A_lo][B_lo]: "bf16x3" split precision, x = hi + lo with
// hi = bf16(x), lo = bf16(x - hi); A.B ~= Ah.Bh + Ah.Bl + Al.Bh (error ~2^-16,
// i.e. fp32-class gradients from the bf16 tensor core; R28 rounding per term)
constexpr uint32_t STAGE_BYTES = 4 * TILE_BYTES;
constexpr uint32_t SMEM_BYTES = STAGES * STAGE_BYTES + 128;  // + barriers / tmem ptr
constexpr int CHUNKS = BM * BK / 4 / THREADS;                // float4 chunks per thread per tile (4)

struct Epi {
  const float* bias;
  const float* resid;
  int64_t ldr;
  const float* mask;
  int64_t ldm;
  int relu;
  int accumulate;
  int mask_after;  // mask the accumulated value (C + result) instead of the result
};

struct Src {
  const float* p;
  int64_t ld;
  int64_t rows;   // extent along the M (or N) dimension
  int64_t r0;
  bool vec;       // float4 loads allowed (16-byte aligned rows)
};

// Which 4 elements (r, k..k+3 for K-major; r..r+3, k for MN-major) thread
// `tid` moves in iteration `it`: every warp store covers two whole 8 x 16-byte
// core matrices (256 contiguous bytes: bank-conflict free), and every warp load
// reads 8 rows x 64 contiguous bytes.
template <bool KMAJOR, int ROWS = BM>
__device__ __forceinline__ void chunk_rk(int it, int& r, int& k) {
  const int w = threadIdx.x >> 5, t = threadIdx.x & 31;
  const int task = it * (THREADS / 32) + w;
  if (KMAJOR) {  // task = (row group, pair of K groups)
    r = (task >> 1) * 8 + ((t >> 1) & 7);
    k = (2 * (task & 1) + (t >> 4)) * 8 + 4 * (t & 1);
  } else {       // task = (K group, pair of row groups)
    constexpr int RP = ROWS / 16;  // row-group pairs per K group
    k = (task / RP) * 8 + ((t >> 1) & 7);
    r = (2 * (task % RP) + (t >> 4)) * 8 + 4 * (t & 1);
  }
}

// One 128 x 32 (rows x K) operand tile: fp32 global -> registers.
//  KMAJOR: source [rows][K], chunk = (r, k..k+3);  !KMAJOR: source [K][rows], chunk = (r..r+3, k)
template <bool KMAJOR, int ROWS = BM>
__device__ __forceinline__ void load_regs(const Src& s, int64_t k0, int64_t kend,
                                          float4 (&v)[ROWS * BK / 4 / THREADS]) {
#pragma unroll
  for (int it = 0; it < ROWS * BK / 4 / THREADS; ++it) {
    int r, k;
    chunk_rk<KMAJOR, ROWS>(it, r, k);
    const int64_t gr = s.r0 + r, gk = k0 + k;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (KMAJOR) {
      if (gr < s.rows) {
        const float* p = s.p + gr * s.ld + gk;
        if (s.vec && gk + 3 < kend) x = __ldg(reinterpret_cast<const float4*>(p));
        else {
          if (gk < kend) x.x = __ldg(p);
          if (gk + 1 < kend) x.y = __ldg(p + 1);
          if (gk + 2 < kend) x.z = __ldg(p + 2);
          if (gk + 3 < kend) x.w = __ldg(p + 3);
        }
      }
    } else {
      if (gk < kend) {
        const float* p = s.p + gk * s.ld + gr;
        if (s.vec && gr + 3 < s.rows) x = __ldg(reinterpret_cast<const float4*>(p));
        else {
          if (gr < s.rows) x.x = __ldg(p);
          if (gr + 1 < s.rows) x.y = __ldg(p + 1);
          if (gr + 2 < s.rows) x.z = __ldg(p + 2);
          if (gr + 3 < s.rows) x.w = __ldg(p + 3);
        }
      }
    }
    v[it] = x;
  }
}

// registers -> bf16 hi / lo canonical layouts (8-byte stores)
//  KMAJOR: (r,k) -> (r/8)*512 + (k/8)*128 + (r%8)*16 + (k%8)*2      (SBO 512, LBO 128)
//  !KMAJOR: (r,k) -> (k/8)*2048 + (r/8)*128 + (k%8)*16 + (r%8)*2    (LBO 2048, SBO 128)
template <bool KMAJOR, int ROWS = BM>
__device__ __forceinline__ void store_smem(uint8_t* dst, uint8_t* dst_lo,
                                           const float4 (&v)[ROWS * BK / 4 / THREADS]) {
#pragma unroll
  for (int it = 0; it < ROWS * BK / 4 / THREADS; ++it) {
    int r, k;
    chunk_rk<KMAJOR, ROWS>(it, r, k);
    uint32_t off;
    if (KMAJOR) off = (r >> 3) * 512 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
    else off = (k >> 3) * (ROWS * 16) + (r >> 3) * 128 + (k & 7) * 16 + (r & 7) * 2;
    // hi = x truncated to its upper 16 bits (one PRMT per pair), lo = RN_bf16(x - hi)
    // (x - hi is exact in fp32): |x - hi - lo| <= 2^-8 |x - hi| < 2^-15 |x|
    const uint32_t x0 = __float_as_uint(v[it].x), x1 = __float_as_uint(v[it].y);
    const uint32_t x2 = __float_as_uint(v[it].z), x3 = __float_as_uint(v[it].w);
    const uint32_t h0 = __byte_perm(x0, x1, 0x7632), h1 = __byte_perm(x2, x3, 0x7632);
    const uint32_t l0 = tc::pack_bf16(v[it].x - __uint_as_float(x0 & 0xffff0000u),
                                      v[it].y - __uint_as_float(x1 & 0xffff0000u));
    const uint32_t l1 = tc::pack_bf16(v[it].z - __uint_as_float(x2 & 0xffff0000u),
                                      v[it].w - __uint_as_float(x3 & 0xffff0000u));
    *reinterpret_cast<uint2*>(dst + off) = make_uint2(h0, h1);
    *reinterpret_cast<uint2*>(dst_lo + off) = make_uint2(l0, l1);
  }
}

// Epilogue stores of one 64-column slab staged in smem ([128][ld] fp32): warp w
// handles rows w, w+8, ..; lane l columns 2l, 2l+1 (8-byte accesses, coalesced
// rows).  Four rows per round with every global read (bias, residual, mask,
// accumulate) issued before the stores, so the slab streams at memory-level
// parallelism 4 per warp instead of one dependent round trip per row.
__device__ __forceinline__ void epi_store_slab(const float* stage, int ld, int64_t m0, int64_t M,
                                               int64_t col0, int64_t N, float* __restrict__ Cz,
                                               int64_t ldc, const Epi& ep, bool partial) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cc = 2 * lane;
  const int64_t gj = col0 + cc;
  const bool c0 = gj < N, c1 = gj + 1 < N;
  const float* __restrict__ bias = ep.bias;
  const float* __restrict__ resid = ep.resid;
  const float* __restrict__ mask = ep.mask;
  float2 b = make_float2(0.f, 0.f);
  if (!partial && bias) {
    if (c0) b.x = __ldg(bias + gj);
    if (c1) b.y = __ldg(bias + gj + 1);
  }
  const uintptr_t al = reinterpret_cast<uintptr_t>(Cz) | reinterpret_cast<uintptr_t>(resid) |
                       reinterpret_cast<uintptr_t>(mask);
  const bool vec = c1 && (al & 7) == 0 && ((ldc | (resid ? ep.ldr : 0) | (mask ? ep.ldm : 0)) % 2 == 0);
  for (int r0 = warp; r0 < BM; r0 += 4 * (THREADS / 32)) {
    float2 x[4], rv[4], mv[4], cv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int rr = r0 + u * (THREADS / 32);
      const int64_t gi = m0 + rr;
      x[u] = *reinterpret_cast<const float2*>(stage + rr * ld + cc);
      rv[u] = mv[u] = cv[u] = make_float2(0.f, 0.f);
      if (partial || gi >= M || !c0) continue;
      if (vec) {
        if (resid) rv[u] = __ldg(reinterpret_cast<const float2*>(resid + gi * ep.ldr + gj));
        if (mask) mv[u] = __ldg(reinterpret_cast<const float2*>(mask + gi * ep.ldm + gj));
        if (ep.accumulate) cv[u] = *reinterpret_cast<const float2*>(Cz + gi * ldc + gj);
      } else {
        if (resid) { rv[u].x = resid[gi * ep.ldr + gj]; if (c1) rv[u].y = resid[gi * ep.ldr + gj + 1]; }
        if (mask) { mv[u].x = mask[gi * ep.ldm + gj]; if (c1) mv[u].y = mask[gi * ep.ldm + gj + 1]; }
        if (ep.accumulate) { cv[u].x = Cz[gi * ldc + gj]; if (c1) cv[u].y = Cz[gi * ldc + gj + 1]; }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int rr = r0 + u * (THREADS / 32);
      const int64_t gi = m0 + rr;
      if (gi >= M || !c0) continue;
      float2 y = x[u];
      if (!partial) {
        y.x += b.x; y.y += b.y;
        y.x += rv[u].x; y.y += rv[u].y;
        if (ep.relu) { y.x = fmaxf(y.x, 0.f); y.y = fmaxf(y.y, 0.f); }
        if (mask && !ep.mask_after) { y.x = mv[u].x > 0.f ? y.x : 0.f; y.y = mv[u].y > 0.f ? y.y : 0.f; }
        y.x += cv[u].x; y.y += cv[u].y;
        if (mask && ep.mask_after) { y.x = mv[u].x > 0.f ? y.x : 0.f; y.y = mv[u].y > 0.f ? y.y : 0.f; }
      }
      if (vec) *reinterpret_cast<float2*>(Cz + gi * ldc + gj) = y;
      else {
        Cz[gi * ldc + gj] = y.x;
        if (c1) Cz[gi * ldc + gj + 1] = y.y;
      }
    }
  }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(THREADS, 3) tc_gemm_kernel(int64_t M, int64_t N, int64_t K,
                                                          const float* __restrict__ A, int64_t lda,
                                                          const float* __restrict__ B, int64_t ldb,
                                                          float* __restrict__ C, int64_t ldc,
                                                          Epi ep, int64_t kslice, int avec, int bvec) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sb = tc::smem_u32(smem);
  const uint32_t bar = sb + STAGES * STAGE_BYTES;  // STAGES mbarriers
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + STAGES * STAGE_BYTES + 64);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t kb = (int64_t)blockIdx.z * kslice;
  const int64_t ke = std::min<int64_t>(K, kb + kslice);
  const int nk = ke > kb ? (int)((ke - kb + BK - 1) / BK) : 0;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) tc::mbar_init(bar + 8 * s, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc(tc::smem_u32(tptr), BN);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tptr;
  constexpr bool A_K = !TA;   // A stored [M][K] -> K-major
  constexpr bool B_K = TB;    // B stored [N][K] -> K-major
  const uint32_t idesc = tc::idesc_bf16(BM, BN) | ((A_K ? 0u : 1u) << 15) | ((B_K ? 0u : 1u) << 16);
  const Src sa{A, lda, M, m0, avec != 0};
  const Src sbb{B, ldb, N, n0, bvec != 0};

  float4 ra[CHUNKS], rb[CHUNKS];
  if (nk > 0) {
    load_regs<A_K>(sa, kb, ke, ra);
    load_regs<B_K>(sbb, kb, ke, rb);
    store_smem<A_K>(smem, smem + 2 * TILE_BYTES, ra);
    store_smem<B_K>(smem + TILE_BYTES, smem + 3 * TILE_BYTES, rb);
    if (nk > 1) {
      load_regs<A_K>(sa, kb + BK, ke, ra);
      load_regs<B_K>(sbb, kb + BK, ke, rb);
    }
  }
  for (int it = 0; it < nk; ++it) {
    const int s = it % STAGES;
    tc::fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc::tc_fence_after();
      const uint32_t a0 = sb + s * STAGE_BYTES, b0 = a0 + TILE_BYTES;
      const uint32_t al = a0 + 2 * TILE_BYTES, bl = a0 + 3 * TILE_BYTES;
      auto da = [&](uint32_t base, int ks) {
        return A_K ? tc::smem_desc(base + ks * 256, 128, 512) : tc::smem_desc(base + ks * 4096, 2048, 128);
      };
      auto db = [&](uint32_t base, int ks) {
        return B_K ? tc::smem_desc(base + ks * 256, 128, 512) : tc::smem_desc(base + ks * 4096, 2048, 128);
      };
#pragma unroll
      for (int ks = 0; ks < BK / 16; ++ks) {
        tc::mma_bf16(tmem, da(al, ks), db(b0, ks), idesc, (it > 0 || ks > 0) ? 1u : 0u);  // Al.Bh
        tc::mma_bf16(tmem, da(a0, ks), db(bl, ks), idesc, 1u);                          // Ah.Bl
        tc::mma_bf16(tmem, da(a0, ks), db(b0, ks), idesc, 1u);                          // Ah.Bh
      }
      tc::mma_commit(bar + 8 * s);
    }
    if (it + 1 < nk) {
      const int ns = (it + 1) % STAGES;
      if (it + 1 >= STAGES)  // stage ns last used by k-block it+1-STAGES
        tc::mbar_wait(bar + 8 * ns, (uint32_t)(((it + 1 - STAGES) / STAGES) & 1));
      uint8_t* st = smem + ns * STAGE_BYTES;
      store_smem<A_K>(st, st + 2 * TILE_BYTES, ra);
      store_smem<B_K>(st + TILE_BYTES, st + 3 * TILE_BYTES, rb);
      if (it + 2 < nk) {
        load_regs<A_K>(sa, kb + (int64_t)(it + 2) * BK, ke, ra);
        load_regs<B_K>(sbb, kb + (int64_t)(it + 2) * BK, ke, rb);
      }
    }
  }
  if (nk > 0) {
    const int ls = (nk - 1) % STAGES;
    tc::mbar_wait(bar + 8 * ls, (uint32_t)(((nk - 1) / STAGES) & 1));
  }
  tc::tc_fence_after();
  __syncthreads();  // every thread is past its last smem store: the ring is free
  // ---- epilogue: TMEM (thread = row) -> smem transpose -> coalesced row stores
  float* Cz = C + (int64_t)blockIdx.z * M * ldc;
  const bool partial = gridDim.z > 1;
  float* stage = reinterpret_cast<float*>(smem);       // [128][EPI_LD]
  constexpr int EPI_COLS = 64, EPI_LD = 68;
  const int q = warp & 3, hh = warp >> 2;  // TMEM lane quarter, column half
  for (int p = 0; p < BN / EPI_COLS; ++p) {
    if (n0 + p * EPI_COLS >= N) break;
    {
      float v[32];
      if (nk > 0) {
        tc::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + p * EPI_COLS + 32 * hh, v);
        tc::tmem_wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      float* dst = stage + (q * 32 + lane) * EPI_LD + 32 * hh;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        reinterpret_cast<float4*>(dst)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
    __syncthreads();
    epi_store_slab(stage, EPI_LD, m0, M, n0 + p * EPI_COLS, N, Cz, ldc, ep, partial);
    __syncthreads();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, BN);
  }
}

// ---------------------------------------------------------------- B-image variant
// For the N in (128, 256] layers with a row-major activation A (every dense
// forward layer and every dgrad of the bf16-context training path): the weight
// operand op(B) is split into bf16 hi / lo ONCE per call into a K-major
// canonical image [K/32 blocks][hi 16 KB | lo 16 KB] (bimg_kernel), and each
// stage receives its 32 KB block by one 1-D bulk copy (no LSU traffic, no
// per-CTA re-splitting); A (read from HBM exactly once: one 128 x 256 tile per
// row block) keeps the conflict-free register-staged split.
constexpr int BNI = 256;
constexpr uint32_t IMG_HALF = BNI * BK * 2;                       // 16 KB
constexpr uint32_t ISTAGE = 2 * (BM * BK * 2) + 2 * IMG_HALF;     // A hi | A lo | B hi | B lo = 48 KB
constexpr uint32_t ISMEM = STAGES * ISTAGE + 128;

// blockIdx.x = k-block, blockIdx.y = 32-row group of n (8 per 256-wide column
// block nb = blockIdx.y / 8, whose image is [nb][K/32 blocks]): 8x the CTAs of
// one block per k-block (the image is launch-latency bound)
}  // namespace
// The next weight image's half of ws_bimg (alternating; grown to the largest
// image so far, the halves at fixed offsets).
// An image launched after an earlier one of the SAME call (its TMA GEMM did not
// apply) goes without PDL: a plain launch waits for that image, which waits
// for the GEMM still reading this half.
#define BIMG_LAUNCH(grid, block, smem, stream, ...)                                  \
  do {                                                                              \
    if (img_launched) {                                                             \
      bimg_kernel<<<grid, block, smem, stream>>>(__VA_ARGS__);                      \
    } else {                                                                        \
      TLP_LAUNCH_PDL(bimg_kernel, grid, block, smem, stream, __VA_ARGS__);          \
    }                                                                               \
    img_launched = true;                                                            \
  } while (0)
static uint8_t* bimg_buffer(tlp_ctx* ctx, size_t bytes, cudaError_t* err) {
  bytes = (bytes + 255) & ~(size_t)255;
  if (bytes > ctx->bimg_half) ctx->bimg_half = bytes;
  *err = ctx->ws_bimg.ensure(2 * ctx->bimg_half);
  ctx->bimg_flip ^= 1;
  return ctx->ws_bimg.as<uint8_t>() + (ctx->bimg_flip ? ctx->bimg_half : 0);
}
namespace {
__global__ void bimg_kernel(const float* __restrict__ B, int64_t ldb, int tb, int64_t N, int64_t K,
                            uint8_t* __restrict__ img) {
  // Programmatic dependent launch: the image goes to the half of the buffer
  // the previous GEMM does not read (bimg_buffer) and depends only on weights
  // final since the step began (P, or Wcat / the head concatenation packed at
  // its start), so it is built while the previous kernel still runs; the wait
  // at the END keeps the chain -- this grid completes only after its
  // predecessor did, so the GEMM that follows still sees every earlier result.
  pdl_trigger();
  const int64_t kb = blockIdx.x, nb = blockIdx.y / (BNI / 32);
  uint8_t* dst = img + (nb * gridDim.x + kb) * 2 * IMG_HALF;
  for (int e = threadIdx.x; e < 32 * BK; e += blockDim.x) {
    const int nl = 32 * (int)(blockIdx.y % (BNI / 32)) + e / BK, k = e % BK;
    const int64_t n = nb * BNI + nl;
    const int64_t gk = kb * BK + k;
    float x = 0.f;
    if (n < N && gk < K) x = tb ? B[(int64_t)n * ldb + gk] : B[gk * ldb + n];
    const uint32_t off = (nl >> 3) * 512 + (k >> 3) * 128 + (nl & 7) * 16 + (k & 7) * 2;
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    *reinterpret_cast<__nv_bfloat16*>(dst + off) = h;
    *reinterpret_cast<__nv_bfloat16*>(dst + IMG_HALF + off) = __float2bfloat16_rn(x - __bfloat162float(h));
  }
  pdl_wait();
}

__global__ void __launch_bounds__(THREADS, 2) tc_gemm_bimg_kernel(int64_t M, int64_t N, int64_t K,
                                                                   const float* __restrict__ A, int64_t lda,
                                                                   const uint8_t* __restrict__ img,
                                                                   float* __restrict__ C, int64_t ldc,
                                                                   Epi ep, int avec) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sb = tc::smem_u32(smem);
  const uint32_t bar = sb + STAGES * ISTAGE;   // [STAGES] MMA done
  const uint32_t bfull = bar + 8 * STAGES;     // [STAGES] B block landed
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + STAGES * ISTAGE + 64);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int nk = K > 0 ? (int)((K + BK - 1) / BK) : 0;
  constexpr uint32_t AB = BM * BK * 2;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(bar + 8 * s, 1);
      tc::mbar_init(bfull + 8 * s, 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc(tc::smem_u32(tptr), BNI);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tptr;
  const uint32_t idesc = tc::idesc_bf16(BM, BNI);
  const Src sa{A, lda, M, m0, avec != 0};
  auto copy_b = [&](int kblk, int st) {
    tc::mbar_arrive_expect_tx(bfull + 8 * st, 2 * IMG_HALF);
    tc::bulk_g2s(sb + st * ISTAGE + 2 * AB, img + (size_t)kblk * 2 * IMG_HALF, 2 * IMG_HALF, bfull + 8 * st);
  };

  float4 ra[CHUNKS];
  if (nk > 0) {
    if (tid == 0) {
      copy_b(0, 0);
      if (nk > 1) copy_b(1, 1);
    }
    load_regs<true>(sa, 0, K, ra);
    store_smem<true>(smem, smem + AB, ra);
    if (nk > 1) load_regs<true>(sa, BK, K, ra);
  }
  for (int it = 0; it < nk; ++it) {
    const int s = it % STAGES;
    tc::fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc::mbar_wait(bfull + 8 * s, (uint32_t)((it / STAGES) & 1));
      tc::tc_fence_after();
      const uint32_t a0 = sb + s * ISTAGE, al = a0 + AB, b0 = a0 + 2 * AB, bl = b0 + IMG_HALF;
#pragma unroll
      for (int ks = 0; ks < BK / 16; ++ks) {
        const uint64_t dah = tc::smem_desc(a0 + ks * 256, 128, 512), dal = tc::smem_desc(al + ks * 256, 128, 512);
        const uint64_t dbh = tc::smem_desc(b0 + ks * 256, 128, 512), dbl = tc::smem_desc(bl + ks * 256, 128, 512);
        tc::mma_bf16(tmem, dal, dbh, idesc, (it > 0 || ks > 0) ? 1u : 0u);  // Al.Bh
        tc::mma_bf16(tmem, dah, dbl, idesc, 1u);                          // Ah.Bl
        tc::mma_bf16(tmem, dah, dbh, idesc, 1u);                          // Ah.Bh
      }
      tc::mma_commit(bar + 8 * s);
    }
    if (it + 1 < nk) {
      const int ns = (it + 1) % STAGES;
      if (it + 1 >= STAGES) {  // stage ns last used by k-block it+1-STAGES
        tc::mbar_wait(bar + 8 * ns, (uint32_t)(((it + 1 - STAGES) / STAGES) & 1));
        if (tid == 0) copy_b(it + 1, ns);
      }
      uint8_t* st = smem + ns * ISTAGE;
      store_smem<true>(st, st + AB, ra);
      if (it + 2 < nk) load_regs<true>(sa, (int64_t)(it + 2) * BK, K, ra);
    }
  }
  if (nk > 0) {
    const int ls = (nk - 1) % STAGES;
    tc::mbar_wait(bar + 8 * ls, (uint32_t)(((nk - 1) / STAGES) & 1));
  }
  tc::tc_fence_after();
  __syncthreads();
  // ---- epilogue (as tc_gemm_kernel): TMEM -> smem transpose -> coalesced row stores
  float* stage = reinterpret_cast<float*>(smem);
  constexpr int EPI_COLS = 64, EPI_LD = 68;
  const int q = warp & 3, hh = warp >> 2;
  for (int p = 0; p < BNI / EPI_COLS; ++p) {
    if (p * EPI_COLS >= N) break;
    {
      float v[32];
      if (nk > 0) {
        tc::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + p * EPI_COLS + 32 * hh, v);
        tc::tmem_wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      float* dst = stage + (q * 32 + lane) * EPI_LD + 32 * hh;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        reinterpret_cast<float4*>(dst)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
    __syncthreads();
    epi_store_slab(stage, EPI_LD, m0, M, p * EPI_COLS, N, C, ldc, ep, false);
    __syncthreads();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, BNI);
  }
}

// ---------------------------------------------------------------- wgrad variant
// dW[M<=256, N<=256] = A^T B over a slice of the K = 204,800 rows (A = X
// [rows][M], B = dY [rows][N], both MN-major operands): ONE CTA per slice owns
// the whole 256 x 256 output (two M=128 accumulators, 512 TMEM columns), so X
// and dY are each read from HBM exactly once (the 128 x 128 tiling read both
// twice).  Partials [Z][M][N] are reduced in a fixed order by the caller.
constexpr int WROWS = 256;
constexpr uint32_t WT = WROWS * BK * 2;                  // one 256 x 32 bf16 operand tile (16 KB)
constexpr uint32_t WSTAGE = 4 * WT;                      // A hi | A lo | B hi | B lo = 64 KB
constexpr uint32_t WSMEM = STAGES * WSTAGE + 128;
constexpr int WCH = WROWS * BK / 4 / THREADS;            // float4 chunks per operand per thread (8)

__global__ void __launch_bounds__(THREADS, 1) tc_wgrad_kernel(int64_t M, int64_t N, int64_t K,
                                                               const float* __restrict__ A, int64_t lda,
                                                               const float* __restrict__ B, int64_t ldb,
                                                               float* __restrict__ part, int64_t ldc,
                                                               int64_t kslice, int avec, int bvec,
                                                               int colsum, int64_t bjs, int64_t pjs) {
  extern __shared__ __align__(128) uint8_t smem[];
  // blockIdx.y = j of J products sharing A (B_j = B + j bjs, partials + j pjs):
  // the J CTAs of one slice are adjacent in launch order, so A's slice comes
  // from HBM once and from L2 for the other J - 1
  B += blockIdx.y * bjs;
  part += blockIdx.y * pjs;
  const uint32_t sb = tc::smem_u32(smem);
  const uint32_t bar = sb + STAGES * WSTAGE;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + STAGES * WSTAGE + 64);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t kb = (int64_t)blockIdx.z * kslice;
  const int64_t ke = std::min<int64_t>(K, kb + kslice);
  const int nk = ke > kb ? (int)((ke - kb + BK - 1) / BK) : 0;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) tc::mbar_init(bar + 8 * s, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc(tc::smem_u32(tptr), 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tptr;
  // both operands MN-major: a_major = b_major = 1; M = 128 per MMA, N = 256
  const uint32_t idesc = tc::idesc_bf16(BM, WROWS) | (1u << 15) | (1u << 16);
  const Src sa{A, lda, M, 0, avec != 0};
  const Src sbb{B, ldb, N, 0, bvec != 0};
  float4 ra[WCH], rb[WCH];
  // colsum: the bias gradient 1^T B of this slice rides along -- every thread
  // always moves the same columns (chunk_rk), so it sums its chunks over the
  // K tiles in order, then a fixed-order reduction over the 32 tile rows
  float4 cs[WCH];
#pragma unroll
  for (int i = 0; i < WCH; ++i) cs[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  auto col_acc = [&]() {
    if (colsum) {
#pragma unroll
      for (int i = 0; i < WCH; ++i) {
        cs[i].x += rb[i].x; cs[i].y += rb[i].y; cs[i].z += rb[i].z; cs[i].w += rb[i].w;
      }
    }
  };
  if (nk > 0) {
    load_regs<false, WROWS>(sa, kb, ke, ra);
    load_regs<false, WROWS>(sbb, kb, ke, rb);
    col_acc();
    store_smem<false, WROWS>(smem, smem + WT, ra);
    store_smem<false, WROWS>(smem + 2 * WT, smem + 3 * WT, rb);
    if (nk > 1) {
      load_regs<false, WROWS>(sa, kb + BK, ke, ra);
      load_regs<false, WROWS>(sbb, kb + BK, ke, rb);
    }
  }
  for (int it = 0; it < nk; ++it) {
    const int s = it % STAGES;
    tc::fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc::tc_fence_after();
      const uint32_t ah = sb + s * WSTAGE, al = ah + WT, bh = ah + 2 * WT, bl = ah + 3 * WT;
      // MN-major 256-row tile: K group stride (LBO) = 256 * 16, 8-row group stride (SBO) = 128;
      // the second M half starts 16 row groups (2 KB) in
#pragma unroll
      for (int ks = 0; ks < BK / 16; ++ks) {
        const uint32_t ko = ks * 2 * WROWS * 16;
        const uint64_t dbh = tc::smem_desc(bh + ko, WROWS * 16, 128), dbl = tc::smem_desc(bl + ko, WROWS * 16, 128);
#pragma unroll
        for (int mh = 0; mh < 2; ++mh) {
          const uint32_t mo = ko + mh * 2048;
          const uint64_t dah = tc::smem_desc(ah + mo, WROWS * 16, 128), dal = tc::smem_desc(al + mo, WROWS * 16, 128);
          const uint32_t d = tmem + 256 * mh;
          tc::mma_bf16(d, dal, dbh, idesc, (it > 0 || ks > 0) ? 1u : 0u);  // Al.Bh
          tc::mma_bf16(d, dah, dbl, idesc, 1u);                          // Ah.Bl
          tc::mma_bf16(d, dah, dbh, idesc, 1u);                          // Ah.Bh
        }
      }
      tc::mma_commit(bar + 8 * s);
    }
    if (it + 1 < nk) {
      const int ns = (it + 1) % STAGES;
      if (it + 1 >= STAGES) tc::mbar_wait(bar + 8 * ns, (uint32_t)(((it + 1 - STAGES) / STAGES) & 1));
      uint8_t* st = smem + ns * WSTAGE;
      col_acc();
      store_smem<false, WROWS>(st, st + WT, ra);
      store_smem<false, WROWS>(st + 2 * WT, st + 3 * WT, rb);
      if (it + 2 < nk) {
        load_regs<false, WROWS>(sa, kb + (int64_t)(it + 2) * BK, ke, ra);
        load_regs<false, WROWS>(sbb, kb + (int64_t)(it + 2) * BK, ke, rb);
      }
    }
  }
  if (nk > 0) {
    const int ls = (nk - 1) % STAGES;
    tc::mbar_wait(bar + 8 * ls, (uint32_t)(((nk - 1) / STAGES) & 1));
  }
  tc::tc_fence_after();
  __syncthreads();
  // epilogue: raw partial sums, TMEM -> smem transpose -> coalesced rows of part[z]
  // (with colsum, part[z] has M + 1 rows: row M is the slice's column sum)
  float* Pz = part + (int64_t)blockIdx.z * (M + (colsum ? 1 : 0)) * ldc;
  float* stage = reinterpret_cast<float*>(smem);
  constexpr int EPI_COLS = 64, EPI_LD = 68;
  const int q = warp & 3, hh = warp >> 2;
  Epi none{nullptr, nullptr, 0, nullptr, 0, 0, 0};
  for (int mh = 0; mh < 2; ++mh) {
    if (mh * BM >= M) break;
    for (int p = 0; p < WROWS / EPI_COLS; ++p) {
      if (p * EPI_COLS >= N) break;
      {
        float v[32];
        if (nk > 0) {
          tc::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + 256 * mh + p * EPI_COLS + 32 * hh, v);
          tc::tmem_wait_ld();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        float* dst = stage + (q * 32 + lane) * EPI_LD + 32 * hh;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          reinterpret_cast<float4*>(dst)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
      __syncthreads();
      epi_store_slab(stage, EPI_LD, mh * BM, M, p * EPI_COLS, N, Pz, ldc, none, true);
      __syncthreads();
    }
  }
  if (colsum) {
    float* red = reinterpret_cast<float*>(smem);  // [32 tile rows][WROWS columns]
#pragma unroll
    for (int i = 0; i < WCH; ++i) {
      int r, k;
      chunk_rk<false, WROWS>(i, r, k);
      *reinterpret_cast<float4*>(red + k * WROWS + r) = cs[i];
    }
    __syncthreads();
    for (int c = tid; c < N; c += THREADS) {
      float sum = 0.f;
      for (int k = 0; k < BK; ++k) sum += red[k * WROWS + c];  // fixed order
      Pz[M * ldc + c] = sum;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

tlp_status tc_gemm(tlp_ctx* ctx, bool ta, bool tb, int64_t M, int64_t N, int64_t K,
                   const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                   int64_t ldc, const EpiParams& e, int splits, int64_t kslice, cudaStream_t s) {
  bool img_launched = false;  // BIMG_LAUNCH
  TLP_SMEM_ATTR((tc_gemm_kernel<false, false>), SMEM_BYTES);
  TLP_SMEM_ATTR((tc_gemm_kernel<false, true>), SMEM_BYTES);
  TLP_SMEM_ATTR((tc_gemm_kernel<true, false>), SMEM_BYTES);
  TLP_SMEM_ATTR((tc_gemm_kernel<true, true>), SMEM_BYTES);
  Epi ep{e.bias, e.resid, e.ldr, e.mask, e.ldm, e.relu ? 1 : 0, e.accumulate ? 1 : 0, e.mask_after ? 1 : 0};
  if (ta && !tb && splits > 1 && M > BM && M <= WROWS && N > BN && N <= WROWS) {
    TLP_SMEM_ATTR(tc_wgrad_kernel, WSMEM);
    const int av = aligned16(A) && lda % 4 == 0, bv = aligned16(B) && ldb % 4 == 0;
    tc_wgrad_kernel<<<dim3(1, 1, (unsigned)splits), THREADS, WSMEM, s>>>(M, N, K, A, lda, B, ldb, C,
                                                                         ldc, kslice, av, bv, 0, 0, 0);
    TLP_LAUNCH_CHECK();
    return TLP_OK;
  }
  // 64 < N <= 128, row-major A: the TMA kernel (N padded to its 256-wide tile
  // in the weight image: zero columns on a memory-bound kernel) when it applies
  if (!ta && splits == 1 && N > 64 && N <= BN && N % 16 == 0 && K > 0 && M >= 4096) {
    const int64_t nkb = cdiv(K, BK);
    cudaError_t be;
    uint8_t* img = bimg_buffer(ctx, (size_t)nkb * 2 * IMG_HALF, &be);
    TLP_CUDA_TRY(be);
    BIMG_LAUNCH( dim3((unsigned)nkb, BNI / 32), 256, 0, s, B, ldb, tb ? 1 : 0, N, K, img);
    TLP_LAUNCH_CHECK();
    const tlp_status ts = tc_gemm_tma(ctx, M, N, K, A, lda, img, C, ldc, e, s);
    if (ts != TLP_ERR_UNSUPPORTED) return ts;
  }
  // N a multiple of 256 above it (the fused Q/K/V projection, the LSTM gate
  // GEMMs): one launch over [row block x 256-wide column block] tiles
  if (!ta && splits == 1 && N > BNI && N % BNI == 0 && K > 0 && M >= 4096) {
    const int64_t nkb = cdiv(K, BK), ntn = N / BNI;
    cudaError_t be;
    uint8_t* img = bimg_buffer(ctx, (size_t)ntn * nkb * 2 * IMG_HALF, &be);
    TLP_CUDA_TRY(be);
    BIMG_LAUNCH( dim3((unsigned)nkb, (unsigned)(ntn * BNI / 32)), 256, 0, s, B, ldb, tb ? 1 : 0, N, K, img);
    TLP_LAUNCH_CHECK();
    const tlp_status ts = tc_gemm_tma(ctx, M, N, K, A, lda, img, C, ldc, e, s);
    if (ts != TLP_ERR_UNSUPPORTED) return ts;
  }
  if (!ta && splits == 1 && N > BN && N <= BNI && K > 0) {
    TLP_SMEM_ATTR(tc_gemm_bimg_kernel, ISMEM);
    const int64_t nkb = cdiv(K, BK);
    cudaError_t be;
    uint8_t* img = bimg_buffer(ctx, (size_t)nkb * 2 * IMG_HALF, &be);
    TLP_CUDA_TRY(be);
    BIMG_LAUNCH( dim3((unsigned)nkb, BNI / 32), 256, 0, s, B, ldb, tb ? 1 : 0, N, K, img);
    TLP_LAUNCH_CHECK();
    // the TMA-fed persistent kernel (k_tc_tma.cu) when the operands allow it
    const tlp_status ts = tc_gemm_tma(ctx, M, N, K, A, lda, img, C, ldc, e, s);
    if (ts != TLP_ERR_UNSUPPORTED) return ts;
    const int av = aligned16(A) && lda % 4 == 0;
    tc_gemm_bimg_kernel<<<dim3(1, (unsigned)cdiv(M, BM), 1), THREADS, ISMEM, s>>>(M, N, K, A, lda, img, C,
                                                                                ldc, ep, av);
    TLP_LAUNCH_CHECK();
    return TLP_OK;
  }
  dim3 grid((unsigned)cdiv(N, BN), (unsigned)cdiv(M, BM), (unsigned)splits);
  if (splits == 1) kslice = K > 0 ? K : 1;
  const int av = aligned16(A) && lda % 4 == 0, bv = aligned16(B) && ldb % 4 == 0;
  if (!ta && !tb) tc_gemm_kernel<false, false><<<grid, THREADS, SMEM_BYTES, s>>>(M, N, K, A, lda, B, ldb, C, ldc, ep, kslice, av, bv);
  else if (!ta && tb) tc_gemm_kernel<false, true><<<grid, THREADS, SMEM_BYTES, s>>>(M, N, K, A, lda, B, ldb, C, ldc, ep, kslice, av, bv);
  else if (ta && !tb) tc_gemm_kernel<true, false><<<grid, THREADS, SMEM_BYTES, s>>>(M, N, K, A, lda, B, ldb, C, ldc, ep, kslice, av, bv);
  else tc_gemm_kernel<true, true><<<grid, THREADS, SMEM_BYTES, s>>>(M, N, K, A, lda, B, ldb, C, ldc, ep, kslice, av, bv);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

// dW partials + bias-gradient partials in one pass (the fused path of
// sgemm_wgrad_bias): part [splits][M + 1][N], row M = column sums of B's
// slice.  Returns false (nothing launched) if the shape is not the wgrad
// kernel's.
bool tc_wgrad_bias(tlp_ctx* ctx, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                   const float* B, int64_t ldb, float* part, int splits, int64_t kslice,
                   cudaStream_t s, tlp_status* st, int J, int64_t bjs, int64_t pjs) {
  // 64 < M, N <= 256: also the head (256 x 128) and second upsample (128 x 256)
  // layers, whose bias sums then ride along instead of a separate colsum pass
  // (the unused part of the 256 x 256 tile computes zeros)
  if (!(splits > 1 && M > 64 && M <= WROWS && N > 64 && N <= WROWS)) return false;
  if (J > 1 && (bjs % 4 != 0)) return false;
  TLP_SMEM_ATTR(tc_wgrad_kernel, WSMEM);
  const int av = aligned16(A) && lda % 4 == 0, bv = aligned16(B) && ldb % 4 == 0;
  tc_wgrad_kernel<<<dim3(1, (unsigned)J, (unsigned)splits), THREADS, WSMEM, s>>>(M, N, K, A, lda, B, ldb,
                                                                                part, N, kslice, av, bv, 1,
                                                                                bjs, pjs);
  ctx->launches++;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    ctx->last_error = std::string("CUDA launch: ") + cudaGetErrorString(e);
    *st = TLP_ERR_CUDA;
  } else {
    *st = TLP_OK;
  }
  return true;
}

// ---------------------------------------------------------------- test hook
extern "C" tlp_status tlp_debug_gemm(tlp_ctx* ctx, int32_t ta, int32_t tb, int64_t M, int64_t N,
                                     int64_t K, const float* A, int64_t lda, const float* B,
                                     int64_t ldb, float* C, int64_t ldc, int32_t splits,
                                     void* stream) {
  if (!ctx || !A || !B || !C || M < 1 || N < 1 || K < 0 || splits < 1) return TLP_ERR_ARG;
  EpiParams none;
  const int64_t kslice = splits > 1 ? cdiv(cdiv(K, splits), 32) * 32 : K;
  return tc_gemm(ctx, ta != 0, tb != 0, M, N, K, A, lda, B, ldb, C, ldc, none, splits, kslice,
                 reinterpret_cast<cudaStream_t>(stream));
}
