// Attention core of the TRAINING path of TLP_PREC_BF16 contexts on the tensor
// cores: warp-level mma.sync m16n8k8 tf32 (fp32 accumulate), one warp per
// (candidate, head), d_h = 32, L <= 32 (padded to 32).  Same contract as the
// fp32 SIMT kernels of k_simt.cu (P:295 / SURVEY §8(a) a4; R14 scale 1/sqrt(d_h);
// R42 optional padding-key mask); the fp32 context keeps the SIMT kernels (the
// 1e-5 path).  Operands are split "3xTF32" (x = hi + lo, both tf32; A.B ~=
// Ah.Bh + Ah.Bl + Al.Bh, ~2^-21 relative): plain tf32 is NOT enough here --
// dS = A (dA - rowdot) cancels to ~1e-3 of |dA| at the paper's initial scale and
// the Wq / Wk gradients are ~1e-3 of the Wv one (measured: 53% error on Wk).
//
// forward:  one warp per (candidate, head): S = Q K^T (32 MMAs), masked softmax
//           in registers, A (probabilities, fp32) saved for the backward,
//           O = A V (32 MMAs; A re-read from smem in the A-fragment layout)
// backward: dA = dO V^T, rowdot = sum_m dA A, dS = A (dA - rowdot);
//           dQ = dS K / sqrt(d_h), dK = dS^T Q / sqrt(d_h), dV = A^T dO
//           (transposed operands are read from smem by index)
// backward: one (candidate, head) per block of 4 warps, one 16 x 16 quadrant
// each (a 4-warp forward measured slower: 344 vs 291 us per step).
// Operands staged in smem as fp32 [32][LD] (LD = 36 or 40 per access pattern,
// below).
#include "tlp_internal.cuh"

namespace {

// Row strides of the staged fp32 [32][LD] matrices: an operand read with rows
// on the lane's group id g and columns on its thread-in-group t (X[g][t]) is
// bank-conflict free at LD = 36 (36 g + t distinct mod 32), one read
// transposed (X[t][g]) at LD = 40 (40 t + g distinct): the forward's V (read
// transposed by O = P V) and the backward's Q, K (read transposed only) and A
// (transposed by dV = A^T dO) are staged at LD = 40.  (Transposed copies of
// dS, A and dO as well measured slower: 25% fewer conflicts but a lower
// occupancy and the extra transposes.)
constexpr int DH = 32, LP = 32, LD = 36, LDT = 40;
constexpr int MAT = LP * LD;    // floats per staged matrix
constexpr int MATT = LP * LDT;  // ... read transposed

__device__ __forceinline__ uint32_t tf32(float x) {
  uint32_t r;
  asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));  // one F2FP (cvt.rna: four instructions)
  return r;
}

// x = hi + lo with hi = tf32(x), lo = tf32(x - hi)  ("3xTF32")
__device__ __forceinline__ void split(float x, uint32_t& hi, uint32_t& lo) {
  hi = tf32(x);
  lo = tf32(x - __uint_as_float(hi));
}

// D (+)= A B: m16n8k8, A row-major tf32, B col-major tf32, fp32 accumulate
__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// One (candidate, head) per 4-warp block: warp w owns the 16 x 16 quadrant
// (rows 16 (w & 1), columns 16 (w >> 1)) of every 32 x 32 product, so each
// warp's dependent MMA chain is a quarter of the single-warp version's and
// four times as many warps share an SM (ncu: the one-warp-per-pair kernels ran
// at 12% / 24% occupancy, latency-bound).  Row reductions that span the two
// column halves (softmax max / sum, the backward's rowdot) go through shared
// memory in a fixed order (deterministic).
// C[16 x 16 quadrant] = op(X) op(Y), k over 32: 3xTF32 (SPLIT) or plain tf32
template <bool TA, bool TB, bool SPLIT = true, int LX = LD, int LY = LD>
__device__ __forceinline__ void gemm_q(const float* X, const float* Y, float (&c)[2][4], int mt, int nh,
                                       int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[nt][i] = 0.f;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int k0 = 8 * ks + t, k1 = k0 + 4;
    const int r0 = 16 * mt + g, r1 = r0 + 8;
    uint32_t ah[4], al[4];
    const float x0 = TA ? X[k0 * LX + r0] : X[r0 * LX + k0], x1 = TA ? X[k0 * LX + r1] : X[r1 * LX + k0];
    const float x2 = TA ? X[k1 * LX + r0] : X[r0 * LX + k1], x3 = TA ? X[k1 * LX + r1] : X[r1 * LX + k1];
    if (SPLIT) {
      split(x0, ah[0], al[0]); split(x1, ah[1], al[1]); split(x2, ah[2], al[2]); split(x3, ah[3], al[3]);
    } else {
      ah[0] = tf32(x0); ah[1] = tf32(x1); ah[2] = tf32(x2); ah[3] = tf32(x3);
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int jj = 16 * nh + 8 * nt + g;
      const float y0 = TB ? Y[jj * LY + k0] : Y[k0 * LY + jj], y1 = TB ? Y[jj * LY + k1] : Y[k1 * LY + jj];
      if (SPLIT) {
        uint32_t bh0, bl0, bh1, bl1;
        split(y0, bh0, bl0);
        split(y1, bh1, bl1);
        mma_tf32(c[nt], al[0], al[1], al[2], al[3], bh0, bh1);
        mma_tf32(c[nt], ah[0], ah[1], ah[2], ah[3], bl0, bl1);
        mma_tf32(c[nt], ah[0], ah[1], ah[2], ah[3], bh0, bh1);
      } else {
        mma_tf32(c[nt], ah[0], ah[1], ah[2], ah[3], tf32(y0), tf32(y1));
      }
    }
  }
}

// stage rows [0, L) of a [*, ld] fp32 matrix slice (32 columns), zero pad, with
// the block's 128 threads (16-byte cp.async)
template <int LS = LD>
__device__ __forceinline__ void stage128(float* dst, const float* src, int64_t ld, int L, int tid) {
#pragma unroll
  for (int i = 0; i < LP * DH / 4 / 128; ++i) {
    const int e = tid + 128 * i, m = e >> 3, c = (e & 7) * 4;
    const float* g = src + (int64_t)(m < L ? m : 0) * ld + c;
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(dst + m * LS + c));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(g), "r"(m < L ? 16 : 0)
                 : "memory");
  }
}

// C[32 x 32] = op(X) op(Y): for every (m-tile, n-tile) of 16 x 8, k over 32.
//   A element (row i, k) = TA ? X[k][i] : X[i][k];  B element (k, col j) = TB ? Y[j][k] : Y[k][j]
template <bool TA, bool TB, int LX = LD, int LY = LD>
__device__ __forceinline__ void gemm32(const float* X, const float* Y, float (&c)[2][4][4], int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) c[mt][nt][i] = 0.f;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int k0 = 8 * ks + t, k1 = k0 + 4;
    uint32_t ah[2][4], al[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r0 = 16 * mt + g, r1 = r0 + 8;
      split(TA ? X[k0 * LX + r0] : X[r0 * LX + k0], ah[mt][0], al[mt][0]);
      split(TA ? X[k0 * LX + r1] : X[r1 * LX + k0], ah[mt][1], al[mt][1]);
      split(TA ? X[k1 * LX + r0] : X[r0 * LX + k1], ah[mt][2], al[mt][2]);
      split(TA ? X[k1 * LX + r1] : X[r1 * LX + k1], ah[mt][3], al[mt][3]);
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int j = 8 * nt + g;
      uint32_t bh0, bl0, bh1, bl1;
      split(TB ? Y[j * LY + k0] : Y[k0 * LY + j], bh0, bl0);
      split(TB ? Y[j * LY + k1] : Y[k1 * LY + j], bh1, bl1);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        mma_tf32(c[mt][nt], al[mt][0], al[mt][1], al[mt][2], al[mt][3], bh0, bh1);
        mma_tf32(c[mt][nt], ah[mt][0], ah[mt][1], ah[mt][2], ah[mt][3], bl0, bl1);
        mma_tf32(c[mt][nt], ah[mt][0], ah[mt][1], ah[mt][2], ah[mt][3], bh0, bh1);
      }
    }
  }
}

// stage rows [0, L) of a [*, ld] fp32 matrix slice (32 columns), zero pad:
// 16-byte cp.async (all eight chunks of every row in flight at once; rows of
// the QKV / dO buffers are 16-byte aligned), zero-fill for the pad rows
template <int LS = LD>
__device__ __forceinline__ void stage(float* dst, const float* src, int64_t ld, int L, int lane) {
#pragma unroll
  for (int i = 0; i < LP * DH / 4 / 32; ++i) {
    const int e = lane + 32 * i, m = e >> 3, c = (e & 7) * 4;
    const float* g = src + (int64_t)(m < L ? m : 0) * ld + c;
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(dst + m * LS + c));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(g), "r"(m < L ? 16 : 0)
                 : "memory");
  }
}
__device__ __forceinline__ void stage_wait() {
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();
}

__global__ void __launch_bounds__(128) attn_fwd_tc_kernel(const float* __restrict__ QKV, int L, int H,
                                                          int nh, int64_t pairs, float* __restrict__ O,
                                                          float* __restrict__ Asave,
                                                          const float* __restrict__ kvalid) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  extern __shared__ float sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pair = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
  if (pair >= pairs) return;
  float* Qs = sm + w * (2 * MAT + MATT);
  float* Ks = Qs + MAT;  // reused for P after S
  float* Vs = Ks + MAT;  // read transposed by O = P V: LDT
  const int64_t n = pair / nh;
  const int hd = (int)(pair % nh);
  const int64_t row0 = n * L, ld = 3 * (int64_t)H;
  stage(Qs, QKV + row0 * ld + hd * DH, ld, L, lane);
  stage(Ks, QKV + row0 * ld + H + hd * DH, ld, L, lane);
  stage<LDT>(Vs, QKV + row0 * ld + 2 * H + hd * DH, ld, L, lane);
  stage_wait();
  float c[2][4][4];
  gemm32<false, true>(Qs, Ks, c, lane);  // S = Q K^T
  const int g = lane >> 2, t = lane & 3;
  const float scale = 1.0f / sqrtf((float)DH);
  // key validity for this thread's 8 key columns (2 per n-tile)
  bool kv[4][2];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int m = 8 * nt + 2 * t + e;
      kv[nt][e] = m < L && (!kvalid || kvalid[row0 + m] != 0.f);
    }
  float* Ps = Ks;  // K no longer needed: A [32][36] goes here (rows l, cols m)
  __syncwarp();
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int l = 16 * mt + g + 8 * half;
      float mx = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (kv[nt][e]) mx = fmaxf(mx, c[mt][nt][2 * half + e] * scale);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const bool none = mx == -INFINITY;  // no valid key (not produced by tlp_encode): uniform
      float sum = 0.f;
      float p[4][2];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int m = 8 * nt + 2 * t + e;
          p[nt][e] = none ? (m < L ? 1.f : 0.f)
                          : (kv[nt][e] ? expf(c[mt][nt][2 * half + e] * scale - mx) : 0.f);
          sum += p[nt][e];
        }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      const float inv = __frcp_rn(sum);  // == 1.0f / sum bitwise (correctly rounded)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int m = 8 * nt + 2 * t + e;
          const float a = l < L ? p[nt][e] * inv : 0.f;
          Ps[l * LD + m] = a;
          if (Asave && l < L && m < L) Asave[((n * nh + hd) * L + l) * (int64_t)L + m] = a;
        }
    }
  __syncwarp();
  gemm32<false, false, LD, LDT>(Ps, Vs, c, lane);  // O = A V
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int l = 16 * mt + g + 8 * half;
      if (l >= L) continue;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
        *reinterpret_cast<float2*>(O + (row0 + l) * H + hd * DH + 8 * nt + 2 * t) =
            make_float2(c[mt][nt][2 * half], c[mt][nt][2 * half + 1]);
    }
}

__global__ void __launch_bounds__(128) attn_bwd_tc_kernel(const float* __restrict__ QKV,
                                                          const float* __restrict__ Asave,
                                                          const float* __restrict__ dO, int L, int H,
                                                          int nh, float* __restrict__ dQKV) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  extern __shared__ float sm[];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int mt = w & 1, nhf = w >> 1;
  // Q, K (read transposed only: LDT), V, dO, A (LDT: read transposed by dV);
  // dS overwrites V once every
  // warp is past dA = dO V^T (the rowdot barrier) -- 24 KB per block, 9
  // blocks (36 warps) per SM
  float* Qs = sm;
  float* Ks = Qs + MATT;
  float* Vs = Ks + MATT;
  float* dOs = Vs + MAT;
  float* As = dOs + MAT;
  float* dSs = Vs;
  float* red = As + MATT;  // [2 column halves][32 rows] partial rowdot
  const int64_t pair = blockIdx.x;
  const int64_t n = pair / nh;
  const int hd = (int)(pair % nh);
  const int64_t row0 = n * L, ld = 3 * (int64_t)H;
  stage128<LDT>(Qs, QKV + row0 * ld + hd * DH, ld, L, tid);
  stage128<LDT>(Ks, QKV + row0 * ld + H + hd * DH, ld, L, tid);
  stage128(Vs, QKV + row0 * ld + 2 * H + hd * DH, ld, L, tid);
  stage128(dOs, dO + row0 * H + hd * DH, H, L, tid);
  const float* Ab = Asave + (n * nh + hd) * (int64_t)L * L;
  for (int e = tid; e < LP * LP; e += 128) {
    const int l = e / LP, m = e % LP;
    As[l * LDT + m] = (l < L && m < L) ? Ab[l * L + m] : 0.f;  // LDT: read transposed by dV
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const int g = lane >> 2, t = lane & 3;
  float c[2][4];
  gemm_q<false, true>(dOs, Vs, c, mt, nhf, lane);  // dA = dO V^T (quadrant: rows l, keys m)
  // rowdot_l = sum_m dA[l,m] A[l,m]: this warp's 16 keys, then both halves in a fixed order
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int l = 16 * mt + g + 8 * half;
    float rd = 0.f;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) rd += c[nt][2 * half + e] * As[l * LDT + 16 * nhf + 8 * nt + 2 * t + e];
    rd += __shfl_xor_sync(0xffffffffu, rd, 1);
    rd += __shfl_xor_sync(0xffffffffu, rd, 2);
    if (t == 0) red[nhf * 32 + l] = rd;
  }
  __syncthreads();
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int l = 16 * mt + g + 8 * half;
    const float rd = red[l] + red[32 + l];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int m = 16 * nhf + 8 * nt + 2 * t;
      const float2 a2 = *reinterpret_cast<const float2*>(As + l * LDT + m);
      *reinterpret_cast<float2*>(dSs + l * LD + m) =
          make_float2(a2.x * (c[nt][2 * half] - rd), a2.y * (c[nt][2 * half + 1] - rd));  // dS = A (dA - rowdot)
    }
  }
  __syncthreads();
  const float scale = 1.0f / sqrtf((float)DH);
  auto store = [&](const float (&cc)[2][4], int64_t col, float f) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int r = 16 * mt + g + 8 * half;
      if (r >= L) continue;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
        *reinterpret_cast<float2*>(dQKV + (row0 + r) * ld + col + 16 * nhf + 8 * nt + 2 * t) =
            make_float2(cc[nt][2 * half] * f, cc[nt][2 * half + 1] * f);
    }
  };
  // dQ, dK, dV in plain tf32 (R53): no cancellation downstream of dS, and their
  // weight gradients are tf32 products anyway (R52); only dA keeps 3xTF32
  gemm_q<false, false, false, LD, LDT>(dSs, Ks, c, mt, nhf, lane);  // dQ = dS K
  store(c, hd * DH, scale);
  gemm_q<true, false, false, LD, LDT>(dSs, Qs, c, mt, nhf, lane);   // dK = dS^T Q
  store(c, H + hd * DH, scale);
  gemm_q<true, false, false, LDT, LD>(As, dOs, c, mt, nhf, lane);   // dV = A^T dO
  store(c, 2 * H + hd * DH, 1.f);
}

}  // namespace

bool attn_tc_ok(const tlp_ctx* ctx) {
  return ctx->cfg.precision == TLP_PREC_BF16 && ctx->cfg.hidden / ctx->cfg.attn_heads == DH &&
         ctx->cfg.L <= LP;
}

tlp_status attn_fwd_tc(tlp_ctx* ctx, const float* qkv, int64_t N, float* O, float* A,
                       const float* kvalid, cudaStream_t s) {
  const tlp_config& c = ctx->cfg;
  const int64_t pairs = N * c.attn_heads;
  const int warps = 4;
  const size_t smem = (size_t)warps * (2 * MAT + MATT) * sizeof(float);
  TLP_SMEM_ATTR(attn_fwd_tc_kernel, smem);
  TLP_LAUNCH_PDL(attn_fwd_tc_kernel, (unsigned)cdiv(pairs, warps), warps * 32, smem, s, qkv, c.L, c.hidden,
                                                                           c.attn_heads, pairs, O, A, kvalid);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

tlp_status attn_bwd_tc(tlp_ctx* ctx, const float* qkv, const float* A, const float* dO, int64_t N,
                       float* dqkv, cudaStream_t s) {
  const tlp_config& c = ctx->cfg;
  const int64_t pairs = N * c.attn_heads;
  if (pairs == 0) return TLP_OK;
  const size_t smem = (3 * MATT + 2 * MAT + 64) * sizeof(float);
  TLP_SMEM_ATTR(attn_bwd_tc_kernel, smem);
  TLP_LAUNCH_PDL(attn_bwd_tc_kernel, (unsigned)pairs, 128, smem, s, qkv, A, dO, c.L, c.hidden, c.attn_heads, dqkv);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}
