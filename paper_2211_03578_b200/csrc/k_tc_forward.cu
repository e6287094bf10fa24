// bf16 tcgen05 fused forward of the TLP network (the scoring hot path).
//
// One persistent CTA per SM walks tiles of 5 candidates = 125 rows (+3 pad
// rows) = one M=128 UMMA tile, and runs the WHOLE network on chip for the tile
// (readings R8-R14, R28 in DESIGN.md):
//   X (fp32 [5,25,22] from HBM) -> bf16 smem
//   h = relu(relu(X W1 + b1) W2 + b2)                          2 GEMMs
//   per attention layer, per head j (8 heads, d_h = 32):
//     [Q_j|K_j|V_j] = h W_qkv_j + b                             GEMM N=96
//     S_j = Q_j K_j^T  (block-diagonal: 5 candidates x 32 padded keys) GEMM N=160
//     P_j = softmax(S_j / sqrt(32)) over the candidate's 25 keys (fp32, epilogue)
//     O_j = P_j V_j                                             GEMM N=32, K=160
//     acc += O_j Wo[32j:32j+32, :]                              GEMM (accumulated in TMEM)
//   h = h + acc + bo
//   per residual block: h = h + relu(h Wa + a) Wb + b           4 GEMMs (N-split halves)
//   per task t: s_t = sum_l relu(h_l W1_t + c1_t) . w2_t + 25 c2_t   GEMM + row dot + ordered sum
// Only X (2,200 B/candidate) is read and n_tasks floats written per candidate;
// all activations stay in SMEM/TMEM.  Weights (bf16, pre-packed in UMMA
// canonical layout in consumption order) stream from L2 through a 3-stage
// ring of 16 KB stages filled by 1-D bulk TMA (cp.async.bulk).
//
// Warp roles: warp 0 = TMA producer (one lane), warp 1 = tcgen05.mma issuer
// (one lane) and TMEM owner, warps 2..5 = epilogue (thread = tile row = TMEM
// lane).  MMA -> epilogue: tcgen05.commit on `acc_bar`; epilogue -> MMA:
// 128 arrivals on `opnd_bar` after fence.proxy.async.
//
// Batch invariance: a candidate's keys sit at K positions 32*slot..32*slot+24
// (zero padded to 32), so the PV accumulation grouping is identical for every
// slot; every other step is row-local and the final 25-row sum runs in a fixed
// order.  Scores therefore do not depend on the batch size or tile placement.
#include "tlp_internal.cuh"
#include "tc_ptx.cuh"

#include <algorithm>
#include <array>
#include <cmath>
#include <vector>

namespace {

constexpr int kL = 25, kE = 22, kH = 256, kHeads = 8, kDH = 32, kHD = 128;
constexpr int kCand = 5;            // candidates per tile
constexpr int kKX = 32;             // padded K of the first GEMM (22 -> 32)
constexpr int kKP = 160;            // padded key positions (5 x 32)
constexpr int kStages = 3;
constexpr uint32_t kStageBytes = 16384;
constexpr int kThreads = 192;

// shared memory map (bytes)
constexpr uint32_t OFF_H = 0;                              // h        [128 x 256] bf16, Kt=256
constexpr uint32_t OFF_R = OFF_H + 65536;                  // X / U1 / r-half [128 x <=128]
constexpr uint32_t OFF_Q = OFF_R + 32768;                  // Q_j      [128 x 32]
constexpr uint32_t OFF_K = OFF_Q + 8192;                   // K_j      [160 x 32]  (B operand)
constexpr uint32_t OFF_V = OFF_K + 10240;                  // V_j^T    [32 x 160]  (B operand)
constexpr uint32_t OFF_P = OFF_V + 10240;                  // P_j      [128 x 160]
constexpr uint32_t OFF_O = OFF_P + 40960;                  // O_j      [128 x 32]
constexpr uint32_t OFF_RING = OFF_O + 8192;                // 3 x 16 KB weight stages
constexpr uint32_t OFF_DOT = OFF_RING + kStages * kStageBytes;  // 128 fp32 row dots
constexpr uint32_t OFF_BAR = OFF_DOT + 512;                // 2*kStages + 2 mbarriers
constexpr uint32_t OFF_TPTR = OFF_BAR + 8 * (2 * kStages + 2);
constexpr uint32_t SMEM_BYTES = OFF_TPTR + 16;
static_assert(SMEM_BYTES <= 232448, "smem budget");

// TMEM column map (512 allocated)
constexpr uint32_t T_A = 0;    // 256: up / oproj / residual-block / output accumulators
constexpr uint32_t T_B = 256;  // 160: QKV_j, then S_j; resblock halves; head
constexpr uint32_t T_O = 416;  // 32:  O_j

struct ChunkRef {
  uint32_t off16;  // byte offset / 16 into the weight stream
  uint32_t bytes;
};

struct TcArgs {
  const float* X;
  float* scores;
  int64_t N;
  int64_t ntile;
  const uint8_t* wstream;
  const ChunkRef* chunks;
  int nchunks;
  const float* P;  // fp32 parameters (biases / w2 / c2 read by the epilogue)
  int64_t up_b0, up_b1;
  int64_t bq[TLP_MAX_ATTN], bk[TLP_MAX_ATTN], bv[TLP_MAX_ATTN], bo[TLP_MAX_ATTN];
  int64_t ra[TLP_MAX_RES], rb[TLP_MAX_RES];
  int64_t c1[TLP_MAX_TASKS], w2[TLP_MAX_TASKS], c2[TLP_MAX_TASKS];
  int n_attn, n_res, n_tasks;
};

// ---------------------------------------------------------------- epilogue helpers
__device__ __forceinline__ void store_row32(uint8_t* smem, uint32_t base, uint32_t r, uint32_t k0,
                                            uint32_t Kt, const uint32_t (&pk)[16]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 v = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
    *reinterpret_cast<uint4*>(smem + base + tc::canon_off(r, k0 + 8 * i, Kt)) = v;
  }
}

__device__ __forceinline__ void load_bias32(const float* __restrict__ b, float (&o)[32]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(b) + i);
    o[4 * i] = v.x; o[4 * i + 1] = v.y; o[4 * i + 2] = v.z; o[4 * i + 3] = v.w;
  }
}

// relu(acc[c0..c0+ncol) + bias) -> bf16 operand (row r, k = c0..)
__device__ __forceinline__ void epi_bias_relu(uint8_t* smem, uint32_t tl, uint32_t tcol,
                                              int ncol, const float* bias, uint32_t dst,
                                              uint32_t Kt, uint32_t r) {
  for (int c = 0; c < ncol; c += 32) {
    float v[32], b[32];
    tc::tmem_ld32(tl + tcol + c, v);
    load_bias32(bias + c, b);
    tc::tmem_wait_ld();
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      pk[i] = tc::pack_bf16(fmaxf(v[2 * i] + b[2 * i], 0.f), fmaxf(v[2 * i + 1] + b[2 * i + 1], 0.f));
    store_row32(smem, dst, r, c, Kt, pk);
  }
}

// h[r, :] = bf16(h[r, :] + acc[r, :] + bias)   (R10 / R12 residual)
__device__ __forceinline__ void epi_residual(uint8_t* smem, uint32_t tl, const float* bias,
                                             uint32_t r) {
  for (int c = 0; c < kH; c += 32) {
    float v[32], b[32];
    tc::tmem_ld32(tl + T_A + c, v);
    load_bias32(bias + c, b);
    uint4 old[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      old[i] = *reinterpret_cast<const uint4*>(smem + OFF_H + tc::canon_off(r, c + 8 * i, kH));
    tc::tmem_wait_ld();
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t w = (&old[i >> 2].x)[i & 3];
      __nv_bfloat162 hb = *reinterpret_cast<const __nv_bfloat162*>(&w);
      const float2 hf = __bfloat1622float2(hb);
      pk[i] = tc::pack_bf16(hf.x + (v[2 * i] + b[2 * i]), hf.y + (v[2 * i + 1] + b[2 * i + 1]));
    }
    store_row32(smem, OFF_H, r, c, kH, pk);
  }
}

__global__ void __launch_bounds__(kThreads, 1) tc_forward_kernel(const TcArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sbase = tc::smem_u32(smem);
  const uint32_t bar_full = sbase + OFF_BAR;               // kStages
  const uint32_t bar_empty = bar_full + 8 * kStages;       // kStages
  const uint32_t bar_acc = bar_empty + 8 * kStages;
  const uint32_t bar_opnd = bar_acc + 8;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + OFF_TPTR);

  // zero the attention operand buffers once: their pad entries must stay 0
  for (uint32_t o = OFF_K + threadIdx.x * 16; o < OFF_O; o += kThreads * 16)
    *reinterpret_cast<uint4*>(smem + o) = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(bar_full + 8 * s, 1);
      tc::mbar_init(bar_empty + 8 * s, 1);
    }
    tc::mbar_init(bar_acc, 1);
    tc::mbar_init(bar_opnd, 128);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tc::smem_u32(tptr), 512);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tptr;
  const int NA = a.n_attn, NR = a.n_res, NT = a.n_tasks;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < a.ntile; tile += gridDim.x) {
        for (int c = 0; c < a.nchunks; ++c) {
          tc::mbar_wait(bar_empty + 8 * stage, phase ^ 1);
          const ChunkRef ch = a.chunks[c];
          tc::mbar_arrive_expect_tx(bar_full + 8 * stage, ch.bytes);
          tc::bulk_g2s(sbase + OFF_RING + stage * kStageBytes, a.wstream + (size_t)ch.off16 * 16,
                       ch.bytes, bar_full + 8 * stage);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, op_phase = 0;
      auto wait_opnd = [&]() {
        tc::mbar_wait(bar_opnd, op_phase);
        op_phase ^= 1;
        tc::tc_fence_after();
      };
      // D (+)= A[smem, Kt=a_kt] x (ring chunks of N x Kc)^T over K
      auto gemm_w = [&](uint32_t a_off, uint32_t a_kt, uint32_t d_col, uint32_t N, int K, int Kc,
                        bool acc) {
        const uint32_t idesc = tc::idesc_bf16(128, N);
        for (int kc = 0; kc < K; kc += Kc) {
          tc::mbar_wait(bar_full + 8 * stage, phase);
          tc::tc_fence_after();
          const uint32_t b = sbase + OFF_RING + stage * kStageBytes;
#pragma unroll 4
          for (int ks = 0; ks < Kc; ks += 16) {
            const uint64_t ad = tc::smem_desc(sbase + a_off + ((kc + ks) >> 3) * 128, 128, a_kt * 16);
            const uint64_t bd = tc::smem_desc(b + (ks >> 3) * 128, 128, Kc * 16);
            tc::mma_bf16(tmem + d_col, ad, bd, idesc, (acc || kc + ks > 0) ? 1u : 0u);
          }
          tc::mma_commit(bar_empty + 8 * stage);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      };
      // D = A[smem] x B[smem]^T (both operands produced on chip)
      auto gemm_s = [&](uint32_t a_off, uint32_t a_kt, uint32_t b_off, uint32_t b_kt,
                        uint32_t d_col, uint32_t N, int K) {
        const uint32_t idesc = tc::idesc_bf16(128, N);
        for (int ks = 0; ks < K; ks += 16) {
          const uint64_t ad = tc::smem_desc(sbase + a_off + (ks >> 3) * 128, 128, a_kt * 16);
          const uint64_t bd = tc::smem_desc(sbase + b_off + (ks >> 3) * 128, 128, b_kt * 16);
          tc::mma_bf16(tmem + d_col, ad, bd, idesc, ks > 0 ? 1u : 0u);
        }
      };
      auto done = [&]() { tc::mma_commit(bar_acc); };
      for (int64_t tile = blockIdx.x; tile < a.ntile; tile += gridDim.x) {
        wait_opnd();                                             // X
        gemm_w(OFF_R, kKX, T_A, 128, kKX, 32, false); done();    // upsample 0
        wait_opnd();                                             // U1
        gemm_w(OFF_R, 128, T_A, kH, 128, 32, false); done();     // upsample 1
        wait_opnd();                                             // h
        for (int l = 0; l < NA; ++l) {
          for (int j = 0; j < kHeads; ++j) {
            if (j > 0) gemm_w(OFF_O, kDH, T_A, kH, kDH, 32, j > 1);   // oproj_{j-1}
            gemm_w(OFF_H, kH, T_B, 96, kH, 64, false); done();        // QKV_j
            wait_opnd();
            gemm_s(OFF_Q, kDH, OFF_K, kDH, T_B, kKP, kDH); done();    // S_j
            wait_opnd();
            gemm_s(OFF_P, kKP, OFF_V, kKP, T_O, kDH, kKP); done();    // O_j = P_j V_j
            wait_opnd();
          }
          gemm_w(OFF_O, kDH, T_A, kH, kDH, 32, true); done();         // oproj_7
          wait_opnd();                                                // h += ...
        }
        for (int r = 0; r < NR; ++r) {
          gemm_w(OFF_H, kH, T_B, 128, kH, 64, false); done();         // G1 half 0
          wait_opnd();
          gemm_w(OFF_R, 128, T_A, kH, 128, 32, false);                // G2 part 0
          gemm_w(OFF_H, kH, T_B, 128, kH, 64, false); done();         // G1 half 1
          wait_opnd();
          gemm_w(OFF_R, 128, T_A, kH, 128, 32, true); done();         // G2 part 1
          wait_opnd();                                                // h += ...
        }
        for (int t = 0; t < NT; ++t) {
          gemm_w(OFF_H, kH, T_B, kHD, kH, 64, false); done();         // head t
          if (t < NT - 1) wait_opnd();
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (128 threads)
    const uint32_t q = warp & 3;
    const uint32_t r = 32 * q + lane;                  // tile row == TMEM lane
    const uint32_t tl = tmem + ((32 * q) << 16);       // this warp's lane quarter
    const float* P = a.P;
    float* rowdot = reinterpret_cast<float*>(smem + OFF_DOT);
    uint32_t acc_phase = 0;
    auto wait_acc = [&]() {
      tc::mbar_wait(bar_acc, acc_phase);
      acc_phase ^= 1;
      tc::tc_fence_after();
    };
    auto signal = [&]() {
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      tc::mbar_arrive(bar_opnd);
    };
    const uint32_t slot = r / kL;                      // candidate slot (5 = pad rows)
    const uint32_t kk = r - slot * kL;
    const bool real = r < kCand * kL;
    const uint32_t s_lo = (32 * q) / kL;
    const float sm_scale = 1.4426950408889634f / sqrtf((float)kDH);  // log2(e)/sqrt(d_h)
    for (int64_t tile = blockIdx.x; tile < a.ntile; tile += gridDim.x) {
      const int64_t n = tile * kCand + slot;
      // E0: X rows -> bf16 [128 x 32]
      {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = 0;
        if (real && n < a.N) {
          const float2* src = reinterpret_cast<const float2*>(a.X + (tile * kCand * kL + r) * kE);
#pragma unroll
          for (int i = 0; i < kE / 2; ++i) {
            const float2 x = __ldg(src + i);
            pk[i] = tc::pack_bf16(x.x, x.y);
          }
        }
        store_row32(smem, OFF_R, r, 0, kKX, pk);
        signal();
      }
      wait_acc(); epi_bias_relu(smem, tl, T_A, 128, P + a.up_b0, OFF_R, 128, r); signal();
      wait_acc(); epi_bias_relu(smem, tl, T_A, kH, P + a.up_b1, OFF_H, kH, r); signal();
      for (int l = 0; l < NA; ++l) {
        for (int j = 0; j < kHeads; ++j) {
          // ---- Q_j, K_j, V_j -> operand layouts
          wait_acc();
          {
            float v[32], b[32];
            uint32_t pk[16];
            tc::tmem_ld32(tl + T_B + 0, v);
            load_bias32(P + a.bq[l] + kDH * j, b);
            tc::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = tc::pack_bf16(v[2 * i] + b[2 * i], v[2 * i + 1] + b[2 * i + 1]);
            store_row32(smem, OFF_Q, r, 0, kDH, pk);
            tc::tmem_ld32(tl + T_B + 32, v);
            load_bias32(P + a.bk[l] + kDH * j, b);
            tc::tmem_wait_ld();
            if (real) {
#pragma unroll
              for (int i = 0; i < 16; ++i) pk[i] = tc::pack_bf16(v[2 * i] + b[2 * i], v[2 * i + 1] + b[2 * i + 1]);
              store_row32(smem, OFF_K, 32 * slot + kk, 0, kDH, pk);
            }
            tc::tmem_ld32(tl + T_B + 64, v);
            load_bias32(P + a.bv[l] + kDH * j, b);
            tc::tmem_wait_ld();
            if (real) {
              const uint32_t kpos = 32 * slot + kk;
#pragma unroll
              for (int d = 0; d < kDH; ++d) {
                __nv_bfloat16 hv = __float2bfloat16_rn(v[d] + b[d]);
                *reinterpret_cast<__nv_bfloat16*>(smem + OFF_V + tc::canon_off(d, kpos, kKP)) = hv;
              }
            }
          }
          signal();
          // ---- softmax over the candidate's 25 keys -> P_j
          wait_acc();
          {
            float va[32], vb[32];
            tc::tmem_ld32(tl + T_B + 32 * s_lo, va);
            tc::tmem_ld32(tl + T_B + 32 * s_lo + 32, vb);
            tc::tmem_wait_ld();
            if (real) {
              const bool hi = slot != s_lo;
              float x[kL];
              float mx = -INFINITY;
#pragma unroll
              for (int c = 0; c < kL; ++c) {
                x[c] = (hi ? vb[c] : va[c]) * sm_scale;
                mx = fmaxf(mx, x[c]);
              }
              float sum = 0.f;
#pragma unroll
              for (int c = 0; c < kL; ++c) { x[c] = exp2f(x[c] - mx); sum += x[c]; }
              const float inv = 1.0f / sum;
              uint32_t pk[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float p0 = (2 * i < kL) ? x[(2 * i) % kL] * inv : 0.f;
                const float p1 = (2 * i + 1 < kL) ? x[(2 * i + 1) % kL] * inv : 0.f;
                pk[i] = tc::pack_bf16(p0, p1);
              }
              store_row32(smem, OFF_P, r, 32 * slot, kKP, pk);
            }
          }
          signal();
          // ---- O_j -> bf16 operand
          wait_acc();
          {
            float v[32];
            tc::tmem_ld32(tl + T_O, v);
            tc::tmem_wait_ld();
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = tc::pack_bf16(v[2 * i], v[2 * i + 1]);
            store_row32(smem, OFF_O, r, 0, kDH, pk);
          }
          signal();
        }
        wait_acc(); epi_residual(smem, tl, P + a.bo[l], r); signal();
      }
      for (int rb = 0; rb < NR; ++rb) {
        wait_acc(); epi_bias_relu(smem, tl, T_B, 128, P + a.ra[rb], OFF_R, 128, r); signal();
        wait_acc(); epi_bias_relu(smem, tl, T_B, 128, P + a.ra[rb] + 128, OFF_R, 128, r); signal();
        wait_acc(); epi_residual(smem, tl, P + a.rb[rb], r); signal();
      }
      for (int t = 0; t < NT; ++t) {
        wait_acc();
        float dot = 0.f;
        for (int c = 0; c < kHD; c += 32) {
          float v[32], b[32], w[32];
          tc::tmem_ld32(tl + T_B + c, v);
          load_bias32(P + a.c1[t] + c, b);
          load_bias32(P + a.w2[t] + c, w);
          tc::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) dot = fmaf(fmaxf(v[i] + b[i], 0.f), w[i], dot);
        }
        rowdot[r] = dot;
        tc::tc_fence_before();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (r < kCand) {
          const int64_t nn = tile * kCand + r;
          if (nn < a.N) {
            float s = 0.f;
            for (int l2 = 0; l2 < kL; ++l2) s += rowdot[r * kL + l2];  // fixed order (batch invariance)
            a.scores[nn * NT + t] = s + (float)kL * __ldg(P + a.c2[t]);
          }
        }
        if (t < NT - 1) signal();
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- weight packing
struct PackChunk {
  uint32_t dst;  // byte offset
  int N, Kc, k0, Kreal, nseg;
  int seg_row[3];
  int64_t seg_src[3];
  int seg_ld[3];
  int seg_col[3];
};

__global__ void pack_kernel(const PackChunk* __restrict__ pcs, const float* __restrict__ P,
                            uint8_t* __restrict__ out) {
  const PackChunk c = pcs[blockIdx.x];
  for (int e = threadIdx.x; e < c.N * c.Kc; e += blockDim.x) {
    const int n = e / c.Kc, k = e % c.Kc;
    int s = 0;
    for (int i = 1; i < c.nseg; ++i)
      if (n >= c.seg_row[i]) s = i;
    const int gk = c.k0 + k;
    float v = 0.f;
    if (gk < c.Kreal) v = P[c.seg_src[s] + (int64_t)gk * c.seg_ld[s] + c.seg_col[s] + (n - c.seg_row[s])];
    *reinterpret_cast<__nv_bfloat16*>(out + c.dst + tc::canon_off(n, k, c.Kc)) = __float2bfloat16_rn(v);
  }
}

}  // namespace

struct TcWeights {
  uint8_t* wstream = nullptr;
  ChunkRef* chunks = nullptr;
  PackChunk* pack = nullptr;
  int nchunks = 0;
  size_t bytes = 0;
  std::vector<PackChunk> host;
  // epilogue vectors (biases, w2, c2) copied to 16-byte aligned slots so the
  // epilogue can use float4 loads (flat R24 offsets are not all aligned)
  float* vec = nullptr;
  std::vector<std::array<int64_t, 3>> vec_copies;  // {src flat offset, dst offset, n}
  TcArgs slots{};                                  // offsets into `vec`
};

bool tc_supported(const tlp_config& c) {
  return c.L == kL && c.E == kE && c.T == 11 && c.hidden == kH && c.n_up == 2 &&
         c.up_dims[0] == 128 && c.up_dims[1] == kH && c.attn_heads == kHeads &&
         c.head_dim == kHD && c.n_tasks <= TLP_MAX_TASKS;
}

static std::vector<PackChunk> build_schedule(const tlp_ctx* ctx) {
  const tlp_config& c = ctx->cfg;
  const ParamOffsets& o = ctx->off;
  std::vector<PackChunk> v;
  uint32_t dst = 0;
  auto add = [&](int N, int Kc, int k0, int Kreal, std::vector<std::array<int64_t, 4>> segs) {
    PackChunk p{};
    p.dst = dst;
    p.N = N; p.Kc = Kc; p.k0 = k0; p.Kreal = Kreal; p.nseg = (int)segs.size();
    for (int i = 0; i < p.nseg; ++i) {
      p.seg_row[i] = (int)segs[i][0]; p.seg_src[i] = segs[i][1];
      p.seg_ld[i] = (int)segs[i][2]; p.seg_col[i] = (int)segs[i][3];
    }
    dst += (uint32_t)(N * Kc * 2);
    v.push_back(p);
  };
  add(128, 32, 0, kE, {{0, o.up_W[0], 128, 0}});
  for (int k0 = 0; k0 < 128; k0 += 32) add(256, 32, k0, 128, {{0, o.up_W[1], 256, 0}});
  for (int l = 0; l < c.n_attn; ++l)
    for (int j = 0; j < kHeads; ++j) {
      for (int k0 = 0; k0 < kH; k0 += 64)
        add(96, 64, k0, kH, {{0, o.Wq[l], kH, kDH * j}, {32, o.Wk[l], kH, kDH * j}, {64, o.Wv[l], kH, kDH * j}});
      add(256, 32, kDH * j, kH, {{0, o.Wo[l], kH, 0}});
    }
  for (int r = 0; r < c.n_res; ++r) {
    for (int k0 = 0; k0 < kH; k0 += 64) add(128, 64, k0, kH, {{0, o.Wa[r], kH, 0}});
    for (int k0 = 0; k0 < 128; k0 += 32) add(256, 32, k0, kH, {{0, o.Wb[r], kH, 0}});
    for (int k0 = 0; k0 < kH; k0 += 64) add(128, 64, k0, kH, {{0, o.Wa[r], kH, 128}});
    for (int k0 = 128; k0 < kH; k0 += 32) add(256, 32, k0, kH, {{0, o.Wb[r], kH, 0}});
  }
  for (int t = 0; t < c.n_tasks; ++t)
    for (int k0 = 0; k0 < kH; k0 += 64) add(kHD, 64, k0, kH, {{0, o.W1[t], kHD, 0}});
  return v;
}

tlp_status tc_prepare(tlp_ctx* ctx, cudaStream_t s) {
  if (!ctx->tc) {
    ctx->tc = new TcWeights();
    ctx->tc->host = build_schedule(ctx);
    TcWeights& w = *ctx->tc;
    w.nchunks = (int)w.host.size();
    w.bytes = w.host.back().dst + (size_t)w.host.back().N * w.host.back().Kc * 2;
    std::vector<ChunkRef> refs(w.nchunks);
    for (int i = 0; i < w.nchunks; ++i) {
      refs[i].off16 = w.host[i].dst / 16;
      refs[i].bytes = (uint32_t)(w.host[i].N * w.host[i].Kc * 2);
      if (refs[i].bytes > kStageBytes || w.host[i].dst % 16) {
        ctx->last_error = "tc schedule: chunk exceeds a ring stage";
        return TLP_ERR_STATE;
      }
    }
    TLP_CUDA_TRY(cudaMalloc(&w.wstream, w.bytes));
    TLP_CUDA_TRY(cudaMalloc(&w.chunks, w.nchunks * sizeof(ChunkRef)));
    TLP_CUDA_TRY(cudaMalloc(&w.pack, w.nchunks * sizeof(PackChunk)));
    TLP_CUDA_TRY(cudaMemcpy(w.chunks, refs.data(), w.nchunks * sizeof(ChunkRef), cudaMemcpyHostToDevice));
    TLP_CUDA_TRY(cudaMemcpy(w.pack, w.host.data(), w.nchunks * sizeof(PackChunk), cudaMemcpyHostToDevice));
    TLP_CUDA_TRY(cudaFuncSetAttribute(tc_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)SMEM_BYTES));
  }
  TcWeights& w = *ctx->tc;
  if (!w.vec) {
    const tlp_config& c = ctx->cfg;
    const ParamOffsets& o = ctx->off;
    int64_t dst = 0;
    auto slot = [&](int64_t src, int64_t n) {
      const int64_t d = dst;
      w.vec_copies.push_back({src, d, n});
      dst += (n + 3) / 4 * 4;
      return d;
    };
    TcArgs& t = w.slots;
    t.up_b0 = slot(o.up_b[0], 128);
    t.up_b1 = slot(o.up_b[1], kH);
    for (int l = 0; l < c.n_attn; ++l) {
      t.bq[l] = slot(o.bq[l], kH); t.bk[l] = slot(o.bk[l], kH);
      t.bv[l] = slot(o.bv[l], kH); t.bo[l] = slot(o.bo[l], kH);
    }
    for (int r = 0; r < c.n_res; ++r) { t.ra[r] = slot(o.a[r], kH); t.rb[r] = slot(o.b[r], kH); }
    for (int k = 0; k < c.n_tasks; ++k) {
      t.c1[k] = slot(o.c1[k], kHD); t.w2[k] = slot(o.w2[k], kHD); t.c2[k] = slot(o.c2[k], 1);
    }
    TLP_CUDA_TRY(cudaMalloc(&w.vec, dst * sizeof(float)));
    TLP_CUDA_TRY(cudaMemset(w.vec, 0, dst * sizeof(float)));
  }
  for (const auto& cp : w.vec_copies)
    TLP_CUDA_TRY(cudaMemcpyAsync(w.vec + cp[1], ctx->d_params + cp[0], cp[2] * sizeof(float),
                                 cudaMemcpyDeviceToDevice, s));
  pack_kernel<<<w.nchunks, 256, 0, s>>>(w.pack, ctx->d_params, w.wstream);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

tlp_status tc_forward(tlp_ctx* ctx, const float* feats, int64_t N, float* scores, cudaStream_t s) {
  const tlp_config& c = ctx->cfg;
  const ParamOffsets& o = ctx->off;
  TcWeights& w = *ctx->tc;
  TcArgs a = w.slots;  // epilogue vector offsets into w.vec
  a.X = feats; a.scores = scores; a.N = N; a.ntile = cdiv(N, kCand);
  a.wstream = w.wstream; a.chunks = w.chunks; a.nchunks = w.nchunks; a.P = w.vec;
  (void)o;
  a.n_attn = c.n_attn; a.n_res = c.n_res; a.n_tasks = c.n_tasks;
  const int grid = (int)std::min<int64_t>(a.ntile, ctx->num_sms);
  tc_forward_kernel<<<grid, kThreads, SMEM_BYTES, s>>>(a);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

void tc_free(tlp_ctx* ctx) {
  if (!ctx->tc) return;
  cudaFree(ctx->tc->wstream);
  cudaFree(ctx->tc->chunks);
  cudaFree(ctx->tc->pack);
  cudaFree(ctx->tc->vec);
  delete ctx->tc;
  ctx->tc = nullptr;
}

// ---------------------------------------------------------------- test hook
namespace {
// D[128 x N] = A[128 x K] * B[N x K]^T through one UMMA chain (descriptor test).
__global__ void umma_test_kernel(const float* A, const float* B, float* D, int N, int K) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t sb = tc::smem_u32(sm);
  const uint32_t offA = 0, offB = 128 * K * 2, offBar = offB + N * K * 2, offT = offBar + 8;
  for (int e = threadIdx.x; e < 128 * K; e += blockDim.x)
    *reinterpret_cast<__nv_bfloat16*>(sm + offA + tc::canon_off(e / K, e % K, K)) = __float2bfloat16_rn(A[e]);
  for (int e = threadIdx.x; e < N * K; e += blockDim.x)
    *reinterpret_cast<__nv_bfloat16*>(sm + offB + tc::canon_off(e / K, e % K, K)) = __float2bfloat16_rn(B[e]);
  uint32_t* tp = reinterpret_cast<uint32_t*>(sm + offT);
  if (threadIdx.x == 0) { tc::mbar_init(sb + offBar, 1); tc::fence_barrier_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(tc::smem_u32(tp), 256);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = *tp;
  if (threadIdx.x == 0) {
    const uint32_t id = tc::idesc_bf16(128, N);
    for (int ks = 0; ks < K; ks += 16)
      tc::mma_bf16(tm, tc::smem_desc(sb + offA + (ks >> 3) * 128, 128, K * 16),
                   tc::smem_desc(sb + offB + (ks >> 3) * 128, 128, K * 16), id, ks > 0);
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
}  // namespace

extern "C" tlp_status tlp_debug_umma(const float* A, const float* B, float* D, int32_t N,
                                     int32_t K, void* stream) {
  if (N < 16 || N > 256 || N % 16 || K < 16 || K % 16 || K > 256) return TLP_ERR_ARG;
  const size_t smem = (size_t)128 * K * 2 + (size_t)N * K * 2 + 64;
  cudaFuncSetAttribute(umma_test_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  umma_test_kernel<<<1, 128, smem, reinterpret_cast<cudaStream_t>(stream)>>>(A, B, D, N, K);
  return cudaGetLastError() == cudaSuccess ? TLP_OK : TLP_ERR_CUDA;
}
