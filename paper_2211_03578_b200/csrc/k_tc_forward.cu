// bf16 tensor-core fused forward of the TLP network (the scoring hot path).
//
// One persistent CTA per SM walks tiles of 5 candidates = 125 rows (+3 pad
// rows) = one M=128 UMMA tile, and runs the WHOLE network on chip for the tile
// (readings R8-R14, R28, R33, R34 in DESIGN.md):
//   X (fp32 [5,25,22] from HBM) -> bf16 smem
//   U1 = relu(X W1 + b1)             tcgen05, -> bf16 in TMEM (A operand of the next GEMM)
//   h  = relu(U1 W2 + b2)            tcgen05, -> bf16 smem (A operand + residual stream)
//   per attention layer, per head j (8 heads, d_h = 32):
//     [Q_j|K_j|V_j] = h W_qkv_j + b  tcgen05 N=96, issued two heads ahead (TMEM double buffer)
//     O_j = softmax(Q_j K_j^T / sqrt(32)) V_j   per candidate (25 x 25 in a padded
//           32 x 32 block), on 10 epilogue warps with warp-level mma.sync
//     acc += O_j Wo[32j:32j+32, :]   tcgen05, accumulated in TMEM
//   h = h + acc + bo
//   per residual block: r = relu(h Wa + a) in two N-halves (bf16 in TMEM as the
//     A operand), h = h + r Wb + b       tcgen05
//   per task t: s_t = sum_l relu(h_l W1_t + c1_t) . w2_t + 25 c2_t (fixed-order row sum)
// Only X (2,200 B/candidate) is read from HBM and n_tasks floats are written.
// Weights (bf16, UMMA canonical layout, consumption order) stream from L2
// through a 4-stage x 16 KB ring filled by 1-D bulk TMA (cp.async.bulk);
// biases / w2 / c2 are staged once per CTA in shared memory.
//
// Warp roles: warp 0 = TMA producer (one lane), warp 1 = tcgen05.mma issuer
// (one lane) and TMEM owner, warps 2..11 = epilogue.  Row-wise epilogues run on
// warps 2..9, two per TMEM lane quarter (thread = tile row = TMEM lane),
// splitting the columns.  The attention runs on all ten: QKV_j is converted by
// the warps of each lane quarter (2 or 3), and warp 2 + u computes the unit u =
// (candidate u/2, query half u%2).  MMA -> epilogue: tcgen05.commit on `acc`
// (generic) or `qkv[j%2]`; epilogue -> MMA: arrivals on `opnd` (256) or
// `attn[j%2]` (320) after fence.proxy.async / wait::st.
//
// The attention core is 1.5% of the FLOPs (0.64 of 44 MFLOP/candidate) and is
// block-diagonal 25x25 per candidate; doing it in registers removes two
// MMA<->epilogue round trips per head, which dominated v2 (ncu: TC 43% busy).
//
// Batch invariance (R34): Q, K, V of a candidate sit at padded positions
// 32*slot+kk (kk < 25, pad zero / masked); a unit only touches its candidate's
// block, at the same relative positions whatever the slot; everything else is
// row-local and the 25-row head sum runs in a fixed order.
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
constexpr int kStages = 4;
constexpr uint32_t kStageBytes = 16384;
constexpr int kThreads = 384;   // warp 0 TMA, warp 1 MMA, warps 2..11 epilogue
constexpr int kEpi = 256;       // row-wise epilogue threads: warps 2..9, 2 per TMEM lane quarter
constexpr int kAttn = 320;      // attention threads: warps 2..11, one (candidate, query half) each
constexpr uint32_t kRowB = 80;      // row stride (bytes) of the mma.sync Q/K/V tiles (64 + 16 pad)

// shared memory map (bytes)
constexpr uint32_t OFF_H = 0;                       // h      [128 x 256] bf16, canonical Kt=256
constexpr uint32_t OFF_X = OFF_H + 65536;           // X      [128 x 32]  canonical
constexpr uint32_t OFF_Q = OFF_X + 8192;            // Q_j    [160][32] row-major, 80 B rows (padded positions)
constexpr uint32_t OFF_K = OFF_Q + kKP * kRowB;     // K_j    [160][32] (padded key positions)
constexpr uint32_t OFF_V = OFF_K + kKP * kRowB;     // V_j    [160][32]
constexpr uint32_t OFF_O = OFF_V + kKP * kRowB;     // O_j    3 x [128 x 32] canonical (A of oproj), j % 3
constexpr uint32_t OFF_DOT = OFF_O + 3 * 8192;      // 2 x 128 fp32 row dots
constexpr uint32_t OFF_BAR = OFF_DOT + 1024;        // mbarriers (<= 64)
constexpr uint32_t OFF_TPTR = OFF_BAR + 512;
constexpr uint32_t OFF_KV = OFF_TPTR + 128;         // R42: key-valid byte per tile row (attn_mask)
constexpr uint32_t OFF_RING = OFF_KV + 128;         // kStages x 16 KB
constexpr uint32_t OFF_VEC = OFF_RING + kStages * kStageBytes;  // epilogue vectors (fp32)
constexpr uint32_t kMaxSmem = 232448;
static_assert(OFF_RING % 128 == 0, "ring alignment");

// TMEM column map (512 allocated)
constexpr uint32_t T_A = 0;      // 256: up1 / sum_j O_j Wo_j / residual-block output accumulator
constexpr uint32_t T_B = 256;    // 128: up0, residual-block first GEMM halves, head (scratch)
constexpr uint32_t T_QKV = 256;  // 2 x 96: QKV_j double buffer (attention phase only)
constexpr uint32_t T_AOP = 448;  // 64:  bf16 A operand (U1, residual-block second half)
constexpr uint32_t T_AOP0 = 384; // 64:  bf16 A operand (residual-block first half; res phase only)

// diagnostics (TLP_TC_TRACE=1): kTrEv epilogue timestamps per tile for 8 tiles
// of CTA 0, then 8 words of MMA-issuer wait totals per tile
// Compiled in only with -DTLP_TRACE (tools/abl_build.sh): even a never-taken
// timestamp branch per head cost ~13% of the kernel (clock reads pin the
// scheduling of the surrounding code).
constexpr int kTrEv = 160, kTrW = 8 * kTrEv, kTrM = 16;  // kTrM words per tile of MMA-issuer record
#ifdef TLP_TRACE
constexpr bool kTrace = true;
#else
constexpr bool kTrace = false;
#endif


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
  const float* vec;  // epilogue vectors (aligned slots), staged into smem
  int vec_floats;
  int64_t up_b0, up_b1;
  int64_t bq[TLP_MAX_ATTN], bk[TLP_MAX_ATTN], bv[TLP_MAX_ATTN], bo[TLP_MAX_ATTN];
  int64_t ra[TLP_MAX_RES], rb[TLP_MAX_RES];
  int64_t c1[TLP_MAX_TASKS], w2[TLP_MAX_TASKS], c2[TLP_MAX_TASKS];
  int n_attn, n_res, n_tasks;
  int attn_mask;     // R42: mask padding keys (all-zero X rows)
  const float* pos;  // R43: positional table [L, 256] (16-byte aligned copy) or null
  long long* trace;  // diagnostics (TLP_TC_TRACE=1): CTA 0 epilogue phase timestamps
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

// 32 bf16 (packed) -> plain row of the mma.sync tiles
__device__ __forceinline__ void store_plain32(uint8_t* smem, uint32_t off, const uint32_t (&pk)[16]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *reinterpret_cast<uint4*>(smem + off + 16 * i) =
        make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
}

// 32 consecutive fp32 from shared memory (same address across the warp: broadcast)
__device__ __forceinline__ void vec32(const float* v, float (&o)[32]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 x = reinterpret_cast<const float4*>(v)[i];
    o[4 * i] = x.x; o[4 * i + 1] = x.y; o[4 * i + 2] = x.z; o[4 * i + 3] = x.w;
  }
}

// relu(acc + bias) -> bf16 A operand in TMEM (two bf16 per column)
// The epilogue helpers below walk their column range 64 columns at a time:
// two tcgen05.ld in flight per tcgen05.wait::ld.
__device__ __forceinline__ void relu_pack32(const float (&v)[32], const float* bias,
                                            uint32_t (&pk)[16]) {
  float b[32];
  vec32(bias, b);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
#ifndef TLP_RELU_F32
    // round, then a bf16x2 max with 0: bitwise equal (RN is monotone, RN(0) = 0)
    // (acc + bias) as one FADD2 per pair
    const uint32_t a2 = tc::add_pack_bf16(v[2 * i], v[2 * i + 1], b[2 * i], b[2 * i + 1]);
    const __nv_bfloat162 r2 = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&a2), __float2bfloat162_rn(0.f));
    pk[i] = *reinterpret_cast<const uint32_t*>(&r2);
#else
    pk[i] = tc::pack_bf16(fmaxf(v[2 * i] + b[2 * i], 0.f), fmaxf(v[2 * i + 1] + b[2 * i + 1], 0.f));
#endif
  }
}

// relu(acc + bias) -> bf16 A operand in TMEM (two bf16 per column)
__device__ __forceinline__ void epi_relu_to_tmem(uint32_t tl, uint32_t src, int c0, int c1,
                                                 const float* bias, uint32_t dst) {
  for (int c = c0; c < c1; c += 64) {
    float v0[32], v1[32];
    uint32_t pk[16];
    tc::tmem_ld32(tl + src + c, v0);
    tc::tmem_ld32(tl + src + c + 32, v1);
    tc::tmem_wait_ld();
    relu_pack32(v0, bias + c, pk);
    tc::tmem_st16(tl + dst + c / 2, pk);
    relu_pack32(v1, bias + c + 32, pk);
    tc::tmem_st16(tl + dst + c / 2 + 16, pk);
  }
  tc::tmem_wait_st();
}

// same, 32 columns per tcgen05.ld (ranges that are multiples of 32)
__device__ __forceinline__ void epi_relu_to_tmem32(uint32_t tl, uint32_t src, int c0, int c1,
                                                   const float* bias, uint32_t dst) {
  for (int c = c0; c < c1; c += 32) {
    float v0[32];
    uint32_t pk[16];
    tc::tmem_ld32(tl + src + c, v0);
    tc::tmem_wait_ld();
    relu_pack32(v0, bias + c, pk);
    tc::tmem_st16(tl + dst + c / 2, pk);
  }
  tc::tmem_wait_st();
}

// relu(acc + bias) -> bf16 smem operand (row r)
// R43 (NEXT-3): + pos[row position][c] after the ReLU when `pos_row` is set
__device__ __forceinline__ void add_row32(float (&v)[32], const float* bias, const float* pos_row) {
  float b[32];
  vec32(bias, b);
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i] + b[i], 0.f);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 p = __ldg(reinterpret_cast<const float4*>(pos_row) + i);
    v[4 * i] += p.x; v[4 * i + 1] += p.y; v[4 * i + 2] += p.z; v[4 * i + 3] += p.w;
  }
}

__device__ __forceinline__ void epi_relu_to_smem(uint8_t* smem, uint32_t tl, uint32_t src,
                                                 int c0, int c1, const float* bias, uint32_t dst,
                                                 uint32_t Kt, uint32_t r, const float* pos_row) {
  for (int c = c0; c < c1; c += 64) {
    float v0[32], v1[32];
    uint32_t pk[16];
    tc::tmem_ld32(tl + src + c, v0);
    tc::tmem_ld32(tl + src + c + 32, v1);
    tc::tmem_wait_ld();
    if (pos_row) {
      add_row32(v0, bias + c, pos_row + c);
      add_row32(v1, bias + c + 32, pos_row + c + 32);
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = tc::pack_bf16(v0[2 * i], v0[2 * i + 1]);
      store_row32(smem, dst, r, c, Kt, pk);
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = tc::pack_bf16(v1[2 * i], v1[2 * i + 1]);
      store_row32(smem, dst, r, c + 32, Kt, pk);
      continue;
    }
    relu_pack32(v0, bias + c, pk);
    store_row32(smem, dst, r, c, Kt, pk);
    relu_pack32(v1, bias + c + 32, pk);
    store_row32(smem, dst, r, c + 32, Kt, pk);
  }
}

// h[r, c..c+32) = bf16(h + acc + bias)   (R10 / R12 residual, R33)
__device__ __forceinline__ void residual32(uint8_t* smem, const float (&v)[32], const float* bias,
                                           uint32_t r, int c) {
  float b[32];
  vec32(bias + c, b);
  uint4 old[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    old[i] = *reinterpret_cast<const uint4*>(smem + OFF_H + tc::canon_off(r, c + 8 * i, kH));
  uint32_t pk[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t w = (&old[i >> 2].x)[i & 3];
    __nv_bfloat162 hb = *reinterpret_cast<const __nv_bfloat162*>(&w);
#ifndef TLP_RESID_F32
    // (acc + bias) rounded to bf16, then one bf16x2 add (R33): 4 instructions per
    // pair instead of 7 -- the epilogues bound this kernel by issue slots (ncu:
    // 159K warp-instructions per 5-candidate tile); 23.6 -> 23.05 ms per round
    const uint32_t a2 = tc::add_pack_bf16(v[2 * i], v[2 * i + 1], b[2 * i], b[2 * i + 1]);  // FADD2
    const __nv_bfloat162 s2 = __hadd2(hb, *reinterpret_cast<const __nv_bfloat162*>(&a2));
    pk[i] = *reinterpret_cast<const uint32_t*>(&s2);
#else
    const float2 hf = __bfloat1622float2(hb);
    pk[i] = tc::pack_bf16(hf.x + (v[2 * i] + b[2 * i]), hf.y + (v[2 * i + 1] + b[2 * i + 1]));
#endif
  }
  store_row32(smem, OFF_H, r, c, kH, pk);
}

__device__ __forceinline__ void epi_residual(uint8_t* smem, uint32_t tl, const float* bias,
                                             uint32_t r, int c0, int c1) {
  for (int c = c0; c < c1; c += 64) {
    float v0[32], v1[32];
    tc::tmem_ld32(tl + T_A + c, v0);
    tc::tmem_ld32(tl + T_A + c + 32, v1);
    tc::tmem_wait_ld();
    residual32(smem, v0, bias, r, c);
    residual32(smem, v1, bias, r, c + 32);
  }
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));  // R29: bf16 path may use ex2.approx
  return y;
}

// Attention core of one head for one unit = (candidate c, query half mh): the
// 16 queries at padded positions 32c + 16mh .. +15 against the candidate's own
// 32 padded key positions (25 real), on one warp with mma.sync m16n8k16 bf16:
// S = Q K^T (4 n-tiles x 2 k-steps), masked softmax in registers (exp2 with the
// log2(e)/sqrt(d_h) scale folded in), P packed as A fragments (FA2-style register
// reuse), O = P V (4 d-tiles x 2 k-steps), O scaled by 1/rowsum and stored to
// the canonical bf16 [128 x 32] A operand of the output projection at tile rows
// 25c + kk.  Every candidate sees exactly its own block, at the same relative
// positions whatever its slot (batch invariance, R34).
template <bool MASK>
__device__ __forceinline__ void attn_unit_mma(uint8_t* smem, uint32_t sbase, uint32_t c,
                                              uint32_t mh, uint32_t lane, float sm_scale,
                                              uint32_t o_off, uint32_t kmask) {
  const uint32_t g = lane >> 2, tig = lane & 3;
  const uint32_t q0 = 32 * c + 16 * mh, k0 = 32 * c;
  uint32_t qa[2][4];  // Q A-fragments per k-step (d 0..15, 16..31)
#pragma unroll
  for (int ks = 0; ks < 2; ++ks)
    tc::ldsm_x4(sbase + OFF_Q + (q0 + (lane & 15)) * kRowB + (16 * ks + 8 * (lane >> 4)) * 2, qa[ks]);
  uint32_t vbe[2][2][4];  // V B-fragments, loaded before S so their latency hides under it
#pragma unroll
  for (int kbk = 0; kbk < 2; ++kbk)
#pragma unroll
    for (int dp = 0; dp < 2; ++dp) {
      const uint32_t krow = k0 + 16 * kbk + (lane & 7) + 8 * ((lane >> 3) & 1);
      const uint32_t dcol = 8 * (2 * dp + (lane >> 4));
      tc::ldsm_x4_t(sbase + OFF_V + krow * kRowB + dcol * 2, vbe[kbk][dp]);
    }
  float s[4][4];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
    for (int i = 0; i < 4; ++i) s[nt][i] = 0.f;
    uint32_t kb[4];  // (ks0: b0,b1) (ks1: b0,b1)
    tc::ldsm_x4(sbase + OFF_K + (k0 + 8 * nt + (lane & 7)) * kRowB + 16 * (lane >> 3), kb);
    tc::mma16816(s[nt], qa[0], kb[0], kb[1]);
    tc::mma16816(s[nt], qa[1], kb[2], kb[3]);
  }
  float inv[2];
#pragma unroll
  for (int half = 0; half < 2; ++half) {  // rows q0 + g (+8)
    float mx = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (MASK ? ((kmask >> (8 * nt + 2 * tig + e)) & 1u) : (8 * nt + 2 * (int)tig + e < kL))
          mx = fmaxf(mx, s[nt][2 * half + e]);
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float off = mx * sm_scale;  // kmask is never empty: mx finite
    float sum0 = 0.f, sum1 = 0.f;  // even / odd key columns, one FADD2 per pair
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      float x[2];  // s * scale - off for the pair, one FFMA2
      tc::fma2(x[0], x[1], s[nt][2 * half], s[nt][2 * half + 1], sm_scale, sm_scale, -off, -off);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool ok = MASK ? ((kmask >> (8 * nt + 2 * tig + e)) & 1u) : (8 * nt + 2 * (int)tig + e < kL);
        s[nt][2 * half + e] = ok ? ex2_approx(x[e]) : 0.f;
      }
      tc::add2(sum0, sum1, sum0, sum1, s[nt][2 * half], s[nt][2 * half + 1]);
    }
    float sum = sum0 + sum1;
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    // R29: approximate reciprocal on the bf16 path (sum >= 1: the row max term is
    // exp2(0)); the IEEE division's slow-path call cost 3.4% of the kernel
    inv[half] = __fdividef(1.0f, sum);
  }
  uint32_t pa[2][4];  // P as A fragments per 16-key block
#pragma unroll
  for (int kbk = 0; kbk < 2; ++kbk) {
    pa[kbk][0] = tc::pack_bf16(s[2 * kbk][0], s[2 * kbk][1]);
    pa[kbk][1] = tc::pack_bf16(s[2 * kbk][2], s[2 * kbk][3]);
    pa[kbk][2] = tc::pack_bf16(s[2 * kbk + 1][0], s[2 * kbk + 1][1]);
    pa[kbk][3] = tc::pack_bf16(s[2 * kbk + 1][2], s[2 * kbk + 1][3]);
  }
  float o[4][4];
#pragma unroll
  for (int dn = 0; dn < 4; ++dn)
#pragma unroll
    for (int i = 0; i < 4; ++i) o[dn][i] = 0.f;
#pragma unroll
  for (int kbk = 0; kbk < 2; ++kbk)
#pragma unroll
    for (int dp = 0; dp < 2; ++dp) {  // pairs of d n-tiles
      const uint32_t (&vb)[4] = vbe[kbk][dp];  // (dn=2dp: b0,b1) (dn=2dp+1: b0,b1)
      tc::mma16816(o[2 * dp], pa[kbk], vb[0], vb[1]);
      tc::mma16816(o[2 * dp + 1], pa[kbk], vb[2], vb[3]);
    }
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const uint32_t kk = 16 * mh + g + 8 * half;
    if (kk < (uint32_t)kL) {
      const uint32_t row = kL * c + kk;
#pragma unroll
      for (int dn = 0; dn < 4; ++dn) {
        float y0, y1;  // O / rowsum, one FMUL2
        tc::mul2(y0, y1, o[dn][2 * half], o[dn][2 * half + 1], inv[half], inv[half]);
        *reinterpret_cast<uint32_t*>(smem + o_off + tc::canon_off(row, 8 * dn + 2 * tig, kDH)) =
            tc::pack_bf16(y0, y1);
      }
    }
  }
}

// ---- cluster-pair (tcgen05 cta_group::2) helpers: two SMs run one M = 256 MMA
// per instruction, each holding its own 128-row tile (A) and half of every
// weight chunk (B split by N at the same SMEM offset); tools/umma2sm_probe.cu
// verified the operand split and measured the issue rate (M = 256 at the cost
// of M = 128).
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
// address of the same SMEM location in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
template <bool PAIR>
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t en) {
  if (PAIR)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(en) : "memory");
  else
    tc::mma_bf16(d, ad, bd, idesc, en);
}
template <bool PAIR>
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bd, uint32_t idesc, uint32_t en) {
  if (PAIR)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a_tmem), "l"(bd), "r"(idesc), "r"(en) : "memory");
  else
    tc::mma_bf16_ta(d, a_tmem, bd, idesc, en);
}
// commit: in pair mode the arrival is multicast to the same barrier in both CTAs
template <bool PAIR>
__device__ __forceinline__ void commit(uint32_t bar) {
  if (PAIR)
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(bar), "h"((uint16_t)3) : "memory");
  else
    tc::mma_commit(bar);
}

template <bool PAIR>
__global__ void __launch_bounds__(kThreads, 1) tc_forward_kernel(const TcArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sbase = tc::smem_u32(smem);
  // pair mode: every CTA holds half of each chunk, so the same 64 KB ring has
  // twice the stages (more weight bytes in flight per MMA-time)
  constexpr int NS = PAIR ? 2 * kStages : kStages;
  constexpr uint32_t SB = PAIR ? kStageBytes / 2 : kStageBytes;
  const uint32_t bar_full = sbase + OFF_BAR;             // [NS]
  const uint32_t bar_empty = bar_full + 8 * NS;          // [NS]
  const uint32_t bar_acc = bar_empty + 8 * NS;           // generic GEMM done
  // Attention-phase barriers, indexed so that phase n+1 of a barrier cannot
  // complete before every waiter has observed phase n (a parity wait can never
  // miss a phase): QKV_{j+2} is issued after conv_j is observed, O_{j+4} needs
  // QKV_{j+4}, issued after attn_j is observed.
  const uint32_t bar_qkv = bar_acc + 8;                  // [2] QKV_j done (j % 2)
  const uint32_t bar_opnd = bar_qkv + 16;                // epilogue -> MMA (kEpi arrivals)
  const uint32_t bar_conv = bar_opnd + 8;                // [2] QKV_j read, TMEM buffer free (j % 2)
  const uint32_t bar_attn = bar_conv + 16;               // [4] O_j ready (j % 4)
  const uint32_t bar_peer = bar_attn + 32;               // [NS] pair: the peer's half landed
  // second half of a K-split operand (h columns [128, 256), U1 columns [64, 128)):
  // the GEMM that follows starts on the first K half while the epilogue still
  // writes the second
  const uint32_t bar_opnd2 = bar_peer + 8 * NS;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;      // pair: 0 = leader (issues the MMAs)
  const uint32_t E = PAIR ? 2u : 1u;                     // epilogue arrivals scale (both CTAs)
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + OFF_TPTR);
  float* vs = reinterpret_cast<float*>(smem + OFF_VEC);

  // Q/K/V pad positions must stay exactly 0 (and O's pad rows finite): zero once.
  for (uint32_t o = OFF_Q + threadIdx.x * 16; o < OFF_O + 3 * 8192; o += kThreads * 16)
    *reinterpret_cast<uint4*>(smem + o) = make_uint4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < a.vec_floats / 4; i += kThreads)
    reinterpret_cast<float4*>(vs)[i] = __ldg(reinterpret_cast<const float4*>(a.vec) + i);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      tc::mbar_init(bar_full + 8 * s, 1);
      tc::mbar_init(bar_empty + 8 * s, 1);
    }
    tc::mbar_init(bar_acc, 1);
    tc::mbar_init(bar_qkv, 1);
    tc::mbar_init(bar_qkv + 8, 1);
    tc::mbar_init(bar_opnd, E * kEpi);
    tc::mbar_init(bar_opnd2, E * kEpi);
    for (int i = 0; i < 2; ++i) tc::mbar_init(bar_conv + 8 * i, E * kAttn);
    for (int i = 0; i < 4; ++i) tc::mbar_init(bar_attn + 8 * i, E * kAttn);
    for (int s = 0; s < NS; ++s) tc::mbar_init(bar_peer + 8 * s, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tptr)),
                   "r"(512) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tc::tmem_alloc(tc::smem_u32(tptr), 512);
    }
  }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tptr;
  const int NA = a.n_attn, NR = a.n_res, NT = a.n_tasks;
  // tile walk: single CTA -> tiles blockIdx.x + k gridDim.x; pair -> tile pairs
  // (2 it, 2 it + 1), the CTA of rank r taking 2 it + r (past ntile: an empty tile)
  const int64_t n_it = PAIR ? (a.ntile + 1) / 2 : a.ntile;
  const int64_t it0 = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int64_t it_step = PAIR ? gridDim.x / 2 : gridDim.x;
  auto tile_of = [&](int64_t it) -> int64_t { return PAIR ? 2 * it + rank : it; };
  // epilogue -> MMA arrivals go to the leader's barriers
  // (warp-uniform call sites: after each lane's fences the warp arrives once
  // with count 32 -- one remote operation per warp in pair mode)
  auto arrive_mma = [&](uint32_t bar) {
    __syncwarp();
    if (lane == 0) {
      if (PAIR && rank != 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0], 32;" ::"r"(map_to(bar, 0)) : "memory");
      else
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], 32;" ::"r"(bar) : "memory");
    }
  };

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uintptr_t xb = reinterpret_cast<uintptr_t>(a.X);
      const uintptr_t xe = (xb + (uintptr_t)a.N * kL * kE * sizeof(float)) & ~(uintptr_t)15;
      for (int64_t it = it0; it < n_it; it += it_step) {
        // this CTA's next tile of X into L2 a whole tile ahead: E0's row loads
        // then hit L2 instead of HBM (11,000 B per tile, 16-byte aligned cover)
        if (it + it_step < n_it) {
          const uintptr_t t0 = xb + (uintptr_t)tile_of(it + it_step) * kCand * kL * kE * sizeof(float);
          const uintptr_t p0 = t0 & ~(uintptr_t)15;
          const uintptr_t p1 = std::min<uintptr_t>((t0 + kCand * kL * kE * sizeof(float) + 15) & ~(uintptr_t)15, xe);
          if (p1 > p0) tc::bulk_prefetch_l2(reinterpret_cast<const void*>(p0), (uint32_t)(p1 - p0));
        }
        for (int c = 0; c < a.nchunks; ++c) {
          tc::mbar_wait(bar_empty + 8 * stage, phase ^ 1);
          const ChunkRef ch = a.chunks[c];
          // pair: this CTA's half of the chunk = rows [rank N/2, (rank+1) N/2) of the
          // canonical K-major B (8-row groups are contiguous: the first half of the bytes)
          const uint32_t bytes = PAIR ? ch.bytes / 2 : ch.bytes;
          tc::mbar_arrive_expect_tx(bar_full + 8 * stage, bytes);
          tc::bulk_g2s(sbase + OFF_RING + stage * SB,
                       a.wstream + (size_t)ch.off16 * 16 + (PAIR ? rank * bytes : 0u), bytes,
                       bar_full + 8 * stage);
          if (++stage == NS) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (the leader in pair mode)
    if (PAIR && rank != 0 && lane == 0) {
      // the peer's idle issuer warp relays: this CTA's half of a stage landed
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t peer_bar0 = map_to(bar_peer, 0);
      for (int64_t it = it0; it < n_it; it += it_step) {
        for (int c = 0; c < a.nchunks; ++c) {
          tc::mbar_wait(bar_full + 8 * stage, phase);
          mbar_arrive_remote(peer_bar0 + 8 * stage);
          if (++stage == NS) { stage = 0; phase ^= 1; }
        }
      }
    }
    if (lane == 0 && rank == 0) {
      int stage = 0;
      // per-buffer phases as bit masks (bit b = buffer b): a dynamically indexed
      // array lives in the stack frame (local loads on the issue path; 1.2%)
      uint32_t phase = 0, op_phase = 0, op2_phase = 0, cv_bits = 0, at_bits = 0;
      bool split = false;  // the next GEMM's second K half waits on bar_opnd2
      // diagnostics (a.trace, CTA 0): cycles the issuer spends waiting per tile on
      // weight chunks / QKV reads / O_j / other epilogue operands
      const bool trc = kTrace && a.trace != nullptr && blockIdx.x == 0;
      long long wt[4] = {0, 0, 0, 0}, wc[4] = {0, 0, 0, 0};  // wc: chunk waits per phase
      int cph = 0;  // phase: 0 upsample, 1 attention, 2 residual blocks, 3 heads
      auto timed_wait = [&](int k, uint32_t bar, uint32_t ph) {
        const long long t0 = trc ? clock64() : 0;
        if (PAIR) mbar_wait_cluster(bar, ph);  // arrivals include the peer CTA's
        else tc::mbar_wait(bar, ph);
        if (trc) {
          wt[k] += clock64() - t0;
          if (k == 0) wc[cph] += clock64() - t0;
        }
      };
      auto mark = [&](int ph, int mt) {  // phase start clock (diagnostics)
        cph = ph;
        if (trc && mt < 8) a.trace[kTrW + mt * kTrM + 4 + ph] = clock64();
      };
      auto wait_opnd = [&]() {
        timed_wait(3, bar_opnd, op_phase);
        op_phase ^= 1;
        tc::tc_fence_after();
      };
      // D (+)= A x (ring chunks of N x Kc)^T over K.  A in smem (canonical
      // layout with Kt = a_kt at byte offset a_off) or in TMEM (column a_off).
      auto gemm_w = [&](bool a_tmem, uint32_t a_off, uint32_t a_kt, uint32_t d_col, uint32_t N,
                        int K, int Kc, bool acc) {
        const uint32_t idesc = tc::idesc_bf16(PAIR ? 256 : 128, N);
        for (int kc = 0; kc < K; kc += Kc) {
          if (split && kc == K / 2) {  // K-split operand: second half written
            timed_wait(3, bar_opnd2, op2_phase);
            op2_phase ^= 1;
            tc::tc_fence_after();
            split = false;
          }
          timed_wait(0, bar_full + 8 * stage, phase);
          if (PAIR) timed_wait(0, bar_peer + 8 * stage, phase);  // the peer's half
          tc::tc_fence_after();
          const uint32_t b = sbase + OFF_RING + stage * SB;
#pragma unroll 4
          for (int ks = 0; ks < Kc; ks += 16) {
            const uint64_t bd = tc::smem_desc(b + (ks >> 3) * 128, 128, Kc * 16);
            const uint32_t en = (acc || kc + ks > 0) ? 1u : 0u;
            if (a_tmem)
              mma_ts<PAIR>(tmem + d_col, tmem + a_off + ((kc + ks) >> 1), bd, idesc, en);
            else
              mma_ss<PAIR>(tmem + d_col,
                           tc::smem_desc(sbase + a_off + ((kc + ks) >> 3) * 128, 128, a_kt * 16),
                           bd, idesc, en);
          }
          commit<PAIR>(bar_empty + 8 * stage);
          if (++stage == NS) { stage = 0; phase ^= 1; }
        }
      };
      int mt = 0;
      for (int64_t it = it0; it < n_it; it += it_step, ++mt) {
        if (trc && mt < 8)
          for (int k = 0; k < 4; ++k) wt[k] = wc[k] = 0;
        if (kTrace) mark(0, mt);
        wait_opnd();                                                      // E0: X
        gemm_w(false, OFF_X, kKX, T_B, 128, kKX, 32, false);              // up0 -> T_B
        commit<PAIR>(bar_acc);
        wait_opnd();                                                      // E1: U1[:, :64] -> T_AOP
        split = true;                                                     //     U1[:, 64:]
        gemm_w(true, T_AOP, 0, T_A, kH, 128, 32, false);                  // up1 -> T_A
        commit<PAIR>(bar_acc);
        wait_opnd();                                                      // E2: h[:, :128]
        split = true;                                                     //     h[:, 128:]
        if (kTrace) mark(1, mt);
        for (int l = 0; l < NA; ++l) {
          gemm_w(false, OFF_H, kH, T_QKV, 96, kH, 64, false);             // QKV_0 -> buf 0
          commit<PAIR>(bar_qkv);
          gemm_w(false, OFF_H, kH, T_QKV + 96, 96, kH, 64, false);        // QKV_1 -> buf 1
          commit<PAIR>(bar_qkv + 8);
          for (int j = 0; j < kHeads; ++j) {
            if (j + 2 < kHeads) {
              timed_wait(1, bar_conv + 8 * (j & 1), (cv_bits >> (j & 1)) & 1u);  // QKV_j read: buf j%2 free
              cv_bits ^= 1u << (j & 1);
              tc::tc_fence_after();
              gemm_w(false, OFF_H, kH, T_QKV + 96 * (j & 1), 96, kH, 64, false);  // QKV_{j+2}
              commit<PAIR>(bar_qkv + 8 * (j & 1));
            }
            timed_wait(2, bar_attn + 8 * (j & 3), (at_bits >> (j & 3)) & 1u);  // O_j ready
            at_bits ^= 1u << (j & 3);
            tc::tc_fence_after();
            gemm_w(false, OFF_O + 8192 * (j % 3), kDH, T_A, kH, kDH, 32, j > 0);  // acc += O_j Wo_j
          }
          commit<PAIR>(bar_acc);
          wait_opnd();                                                    // E_resid h[:, :128]
          split = true;                                                   //         h[:, 128:]
        }
        if (kTrace) mark(2, mt);
        for (int r = 0; r < NR; ++r) {
          // G1 half 1 goes ahead of G2 part 0 so that the epilogue of r_h1 overlaps
          // G2 part 0 (the two r halves live in separate TMEM operand slots)
          gemm_w(false, OFF_H, kH, T_B, 128, kH, 64, false);              // G1 half 0
          commit<PAIR>(bar_acc);
          wait_opnd();                                                    // r_h0 -> T_AOP0
          gemm_w(false, OFF_H, kH, T_B, 128, kH, 64, false);              // G1 half 1
          commit<PAIR>(bar_acc);
          gemm_w(true, T_AOP0, 0, T_A, kH, 128, 32, false);               // G2 part 0
          wait_opnd();                                                    // r_h1 -> T_AOP
          gemm_w(true, T_AOP, 0, T_A, kH, 128, 32, true);                 // G2 part 1
          commit<PAIR>(bar_acc);
          wait_opnd();                                                    // E_resid h[:, :128]
          split = true;                                                   //         h[:, 128:]
        }
        if (kTrace) mark(3, mt);
        for (int t = 0; t < NT; ++t) {
          gemm_w(false, OFF_H, kH, T_B, kHD, kH, 64, false);              // head t
          commit<PAIR>(bar_acc);
          if (t < NT - 1) wait_opnd();
        }
        if (trc && mt < 8)
          for (int k = 0; k < 4; ++k) {
            a.trace[kTrW + mt * kTrM + k] = wt[k];
            a.trace[kTrW + mt * kTrM + 8 + k] = wc[k];
          }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..11)
    const uint32_t q = warp & 3;                       // TMEM lane quarter
    const uint32_t hh = (warp - 2) >> 2;               // 0, 1 (row-wise phases) or 2 (quarters 2, 3)
    const bool rowwise = hh < 2;                       // warps 2..9 run the row-wise epilogues
    const uint32_t unit = warp - 2;                    // attention unit: candidate unit/2, query half unit%2
    const uint32_t r = 32 * q + lane;                  // tile row == TMEM lane
    const uint32_t tl = tmem + ((32 * q) << 16);       // this warp's lane quarter
    float* rowdot = reinterpret_cast<float*>(smem + OFF_DOT);   // [2][128]
    uint32_t ph_acc = 0, qkv_bits = 0;  // QKV buffer phases as bits (no stack array)
    int titer = 0, tev = 0;
    auto tr = [&]() {  // diagnostics only (a.trace == nullptr in production)
      if (kTrace && a.trace && blockIdx.x == 0 && threadIdx.x == 64 && titer < 8 && tev < kTrEv)
        a.trace[titer * kTrEv + tev] = clock64();
      ++tev;
    };
    auto wait_on = [&](uint32_t bar, uint32_t& ph) {
      tc::mbar_wait(bar, ph);
      ph ^= 1;
      tc::tc_fence_after();
      tr();
    };
    auto signal = [&]() {
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      arrive_mma(bar_opnd);
      tr();
    };
    auto signal2 = [&]() {  // second half of a K-split operand
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      arrive_mma(bar_opnd2);
    };
    // K-split operands: the quarter's two warps first write columns
    // [0, n/2) (n/4 each), signal, then [n/2, n)
    auto lo_of = [&](int n) { return (int)hh * (n / 2); };
    auto hi_of = [&](int n) { return ((int)hh + 1) * (n / 2); };
    auto kA = [&](int n) { return (int)hh * (n / 4); };
    auto kB = [&](int n) { return n / 2 + (int)hh * (n / 4); };
    auto signal_part = [&](int part) {
      if (part == 0) signal(); else signal2();
    };
    // h = h + acc + bias in two K halves (residual of an attention layer or a residual block)
    auto resid_split = [&](const float* bias) {
#pragma unroll 1
      for (int part = 0; part < 2; ++part) {
        const int c0 = part ? kB(kH) : kA(kH);
        epi_residual(smem, tl, bias, r, c0, c0 + 64);
        signal_part(part);
      }
    };
    // column split between the quarter's two warps
    const uint32_t slot = r / kL;                      // candidate slot (5 = pad rows)
    const uint32_t kk = r - slot * kL;
    const bool real = r < kCand * kL;
    const float sm_scale = 1.4426950408889634f / sqrtf((float)kDH);  // log2(e)/sqrt(d_h)

    for (int64_t it = it0; it < n_it; it += it_step, ++titer) {
      const int64_t tile = tile_of(it);
      tev = 0;
      tr();
      const int64_t n = tile * kCand + slot;
      if (rowwise) {
        if (hh == 0) {  // E0: X rows -> bf16 [128 x 32]
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = 0;
          bool nz = false;
          if (real && n < a.N) {
            const float2* src = reinterpret_cast<const float2*>(a.X + (tile * kCand * kL + r) * kE);
#pragma unroll
            for (int i = 0; i < kE / 2; ++i) {
              const float2 x = __ldg(src + i);
              pk[i] = tc::pack_bf16(x.x, x.y);
              nz |= (x.x != 0.f) | (x.y != 0.f);
            }
          }
          store_row32(smem, OFF_X, r, 0, kKX, pk);
          smem[OFF_KV + r] = nz ? 1 : 0;  // R42 key validity (read after barrier 2 of head 0)
        }
        signal();
        wait_on(bar_acc, ph_acc);
#pragma unroll 1
        for (int part = 0; part < 2; ++part) {  // U1 -> TMEM (K halves; one copy of the code)
          const int c0 = part ? kB(128) : kA(128);
          epi_relu_to_tmem32(tl, T_B, c0, c0 + 32, vs + a.up_b0, T_AOP);
          signal_part(part);
        }
        wait_on(bar_acc, ph_acc);
        const float* pos_row = a.pos ? a.pos + kk * kH : nullptr;  // h (+ pos, R43)
#pragma unroll 1
        for (int part = 0; part < 2; ++part) {
          const int c0 = part ? kB(kH) : kA(kH);
          epi_relu_to_smem(smem, tl, T_A, c0, c0 + 64, vs + a.up_b1, OFF_H, kH, r, pos_row);
          signal_part(part);
        }
      }
      for (int l = 0; l < NA; ++l) {
        for (int j = 0; j < kHeads; ++j) {
          {
            uint32_t ph = (qkv_bits >> (j & 1)) & 1u;
            wait_on(bar_qkv + 8 * (j & 1), ph);
            qkv_bits ^= 1u << (j & 1);
          }
          asm volatile("bar.sync 2, 320;" ::: "memory");  // all warps done reading head j-1
          tr();
          {  // QKV_j (TMEM) + bias -> Q, K, V tiles at padded positions 32 slot + kk
            const uint32_t tq = tl + T_QKV + 96 * (j & 1);
            const uint32_t pos = (32 * slot + kk) * kRowB;
            if (q >= 2) {  // three warps in this quarter: Q, K, V (32 columns each)
              float v[32], b[32];
              uint32_t pk[16];
              tc::tmem_ld32(tq + 32 * hh, v);
              vec32(vs + (hh == 0 ? a.bq[l] : hh == 1 ? a.bk[l] : a.bv[l]) + kDH * j, b);
              tc::tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) pk[i] = tc::add_pack_bf16(v[2 * i], v[2 * i + 1], b[2 * i], b[2 * i + 1]);
              if (real) store_plain32(smem, (hh == 0 ? OFF_Q : hh == 1 ? OFF_K : OFF_V) + pos, pk);
            } else {  // two warps: Q + K[0:16) / K[16:32) + V, both loads before one wait
              float v[32], v2[16], b[32], b2[16];
              uint32_t pk[16], pk2[8];
              const uint32_t c32 = hh == 0 ? 0u : 64u;       // Q or V (32 columns)
              const uint32_t c16 = hh == 0 ? 32u : 48u;      // K half (16 columns)
              tc::tmem_ld32(tq + c32, v);
              tc::tmem_ld16(tq + c16, v2);
              vec32(vs + (hh == 0 ? a.bq[l] : a.bv[l]) + kDH * j, b);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float4 x = reinterpret_cast<const float4*>(vs + a.bk[l] + kDH * j + 16 * hh)[i];
                b2[4 * i] = x.x; b2[4 * i + 1] = x.y; b2[4 * i + 2] = x.z; b2[4 * i + 3] = x.w;
              }
              tc::tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) pk[i] = tc::add_pack_bf16(v[2 * i], v[2 * i + 1], b[2 * i], b[2 * i + 1]);
#pragma unroll
              for (int i = 0; i < 8; ++i) pk2[i] = tc::add_pack_bf16(v2[2 * i], v2[2 * i + 1], b2[2 * i], b2[2 * i + 1]);
              if (real) {
                store_plain32(smem, (hh == 0 ? OFF_Q : OFF_V) + pos, pk);
                uint8_t* kd = smem + OFF_K + pos + 32 * hh;
                *reinterpret_cast<uint4*>(kd) = make_uint4(pk2[0], pk2[1], pk2[2], pk2[3]);
                *reinterpret_cast<uint4*>(kd + 16) = make_uint4(pk2[4], pk2[5], pk2[6], pk2[7]);
              }
            }
          }
          tc::tc_fence_before();                          // QKV_j read: TMEM buffer j%2 free
          if (j + 2 < kHeads) arrive_mma(bar_conv + 8 * (j & 1));
          tr();
          asm volatile("bar.sync 2, 320;" ::: "memory");  // Q/K/V of head j complete
          tr();
          {  // R42 key mask: drop padding keys (an all-padding slot keeps every key)
            const uint32_t cand = unit >> 1;
            uint32_t kmask = (1u << kL) - 1u;
            if (a.attn_mask) {
              kmask = __ballot_sync(0xffffffffu, lane < (uint32_t)kL && smem[OFF_KV + kL * cand + lane]);
              if (!kmask) kmask = (1u << kL) - 1u;
            }
            // two instantiations: the unmasked core tests key positions against
            // a constant (a runtime mask there measured 5% slower overall)
            if (a.attn_mask) attn_unit_mma<true>(smem, sbase, cand, unit & 1, lane, sm_scale, OFF_O + 8192 * (j % 3), kmask);
            else attn_unit_mma<false>(smem, sbase, cand, unit & 1, lane, sm_scale, OFF_O + 8192 * (j % 3), kmask);
          }
          tc::fence_proxy_async_smem();                   // O_j ready
          tc::tc_fence_before();
          arrive_mma(bar_attn + 8 * (j & 3));
          tr();
        }
        if (rowwise) {
          wait_on(bar_acc, ph_acc);
          resid_split(vs + a.bo[l]);
        }
      }
      if (!rowwise) continue;
      for (int rb = 0; rb < NR; ++rb) {
        wait_on(bar_acc, ph_acc);
        epi_relu_to_tmem(tl, T_B, lo_of(128), hi_of(128), vs + a.ra[rb], T_AOP0);
        signal();
        wait_on(bar_acc, ph_acc);
        epi_relu_to_tmem(tl, T_B, lo_of(128), hi_of(128), vs + a.ra[rb] + 128, T_AOP);
        signal();
        wait_on(bar_acc, ph_acc);
        resid_split(vs + a.rb[rb]);
      }
      for (int t = 0; t < NT; ++t) {
        wait_on(bar_acc, ph_acc);
        float dot = 0.f, dot1 = 0.f;
        for (int c = lo_of(kHD); c < hi_of(kHD); c += 32) {
          float v[32], b[32], w[32];
          tc::tmem_ld32(tl + T_B + c, v);
          vec32(vs + a.c1[t] + c, b);
          vec32(vs + a.w2[t] + c, w);
          tc::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {  // even / odd columns: FADD2, two max, FFMA2
            float x0, x1;
            tc::add2(x0, x1, v[2 * i], v[2 * i + 1], b[2 * i], b[2 * i + 1]);
            tc::fma2(dot, dot1, fmaxf(x0, 0.f), fmaxf(x1, 0.f), w[2 * i], w[2 * i + 1], dot, dot1);
          }
        }
        rowdot[hh * 128 + r] = dot + dot1;
        tc::tc_fence_before();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (hh == 0 && r < kCand) {
          const int64_t nn = tile * kCand + r;
          if (nn < a.N) {
            float s2 = 0.f;
            for (int l2 = 0; l2 < kL; ++l2)  // fixed order (R34)
              s2 += rowdot[r * kL + l2] + rowdot[128 + r * kL + l2];
            a.scores[nn * NT + t] = s2 + (float)kL * vs[a.c2[t]];
          }
        }
        // rowdot is rewritten by the next task / tile: order the fixed-order
        // sums above before any later write with a CTA barrier (the epilogue ->
        // MMA -> epilogue mbarrier chain already orders them, through the
        // warp-aggregated arrivals, but racecheck cannot follow that chain)
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (t < NT - 1) signal();
      }
    }
  }
  tc::tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    else tc::tmem_dealloc(tmem, 512);
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

// B operand chunk (N x Kc bf16, canonical K-major layout) from fp32 W [in, out]:
// B[n][k] = W[k0 + k][col(n)], zero beyond Kreal (the 22 -> 32 padding).
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
  // epilogue vectors (biases, w2, c2) copied to 16-byte aligned slots; staged
  // into shared memory by every CTA (flat R24 offsets are not all aligned)
  float* vec = nullptr;
  int vec_floats = 0;
  std::vector<std::array<int64_t, 3>> vec_copies;  // {src flat offset, dst offset, n}
  TcArgs slots{};                                  // offsets into `vec`
  uint32_t smem = 0;
  float* pos = nullptr;                            // R43: aligned copy of the positional table
};

bool tc_supported(const tlp_config& c) {
  return c.backbone == 0 && c.L == kL && c.E == kE && c.T == 11 && c.hidden == kH && c.n_up == 2 &&
         c.up_dims[0] == 128 && c.up_dims[1] == kH && c.attn_heads == kHeads &&
         c.head_dim == kHD && c.n_tasks <= TLP_MAX_TASKS;
}

// The weight chunks in the exact order tc_forward_kernel's MMA issuer consumes them.
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
  add(128, 32, 0, kE, {{0, o.up_W[0], 128, 0}});                                 // up0
  for (int k0 = 0; k0 < 128; k0 += 32) add(256, 32, k0, 128, {{0, o.up_W[1], 256, 0}});  // up1
  for (int l = 0; l < c.n_attn; ++l) {
    auto qkv = [&](int j) {
      for (int k0 = 0; k0 < kH; k0 += 64)
        add(96, 64, k0, kH, {{0, o.Wq[l], kH, kDH * j}, {32, o.Wk[l], kH, kDH * j}, {64, o.Wv[l], kH, kDH * j}});
    };
    qkv(0);
    qkv(1);
    for (int j = 0; j < kHeads; ++j) {
      if (j + 2 < kHeads) qkv(j + 2);                      // QKV two heads ahead once QKV_j is read
      add(256, 32, kDH * j, kH, {{0, o.Wo[l], kH, 0}});     // oproj_j once O_j is ready
    }
  }
  for (int r = 0; r < c.n_res; ++r) {
    for (int k0 = 0; k0 < kH; k0 += 64) add(128, 64, k0, kH, {{0, o.Wa[r], kH, 0}});    // G1 half 0
    for (int k0 = 0; k0 < kH; k0 += 64) add(128, 64, k0, kH, {{0, o.Wa[r], kH, 128}});  // G1 half 1
    for (int k0 = 0; k0 < 128; k0 += 32) add(256, 32, k0, kH, {{0, o.Wb[r], kH, 0}});   // G2 part 0
    for (int k0 = 128; k0 < kH; k0 += 32) add(256, 32, k0, kH, {{0, o.Wb[r], kH, 0}});  // G2 part 1
  }
  for (int t = 0; t < c.n_tasks; ++t)
    for (int k0 = 0; k0 < kH; k0 += 64) add(kHD, 64, k0, kH, {{0, o.W1[t], kHD, 0}});
  return v;
}

tlp_status tc_prepare(tlp_ctx* ctx, cudaStream_t s) {
  if (!ctx->tc) {
    ctx->tc = new TcWeights();
    TcWeights& w = *ctx->tc;
    w.host = build_schedule(ctx);
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
    // epilogue vector slots
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
    w.vec_floats = (int)dst;
    w.smem = OFF_VEC + (uint32_t)dst * 4u;
    if (w.smem > kMaxSmem) {
      ctx->last_error = "tc path: too many layers/tasks for the shared-memory budget";
      return TLP_ERR_UNSUPPORTED;
    }
    TLP_CUDA_TRY(cudaMalloc(&w.vec, dst * sizeof(float)));
    TLP_CUDA_TRY(cudaMemset(w.vec, 0, dst * sizeof(float)));
    TLP_CUDA_TRY(cudaMalloc(&w.wstream, w.bytes));
    TLP_CUDA_TRY(cudaMalloc(&w.chunks, w.nchunks * sizeof(ChunkRef)));
    TLP_CUDA_TRY(cudaMalloc(&w.pack, w.nchunks * sizeof(PackChunk)));
    TLP_CUDA_TRY(cudaMemcpy(w.chunks, refs.data(), w.nchunks * sizeof(ChunkRef), cudaMemcpyHostToDevice));
    TLP_CUDA_TRY(cudaMemcpy(w.pack, w.host.data(), w.nchunks * sizeof(PackChunk), cudaMemcpyHostToDevice));
    TLP_CUDA_TRY(cudaFuncSetAttribute(tc_forward_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kMaxSmem));
    TLP_CUDA_TRY(cudaFuncSetAttribute(tc_forward_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kMaxSmem));
  }
  TcWeights& w = *ctx->tc;
  if (ctx->cfg.pos_enc) {  // R43: the table, copied to an aligned buffer (read through L1 in E2)
    if (!w.pos) TLP_CUDA_TRY(cudaMalloc(&w.pos, (size_t)kL * kH * sizeof(float)));
    TLP_CUDA_TRY(cudaMemcpyAsync(w.pos, ctx->d_params + ctx->off.pos, (size_t)kL * kH * sizeof(float),
                                 cudaMemcpyDeviceToDevice, s));
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
  TcWeights& w = *ctx->tc;
  TcArgs a = w.slots;  // epilogue vector offsets into w.vec
  a.X = feats; a.scores = scores; a.N = N; a.ntile = cdiv(N, kCand);
  a.wstream = w.wstream; a.chunks = w.chunks; a.nchunks = w.nchunks;
  a.vec = w.vec; a.vec_floats = w.vec_floats;
  a.pos = ctx->cfg.pos_enc ? w.pos : nullptr;
  a.n_attn = c.n_attn; a.n_res = c.n_res; a.n_tasks = c.n_tasks;
  a.attn_mask = c.attn_mask;
  // Experimental (TLP_TC_PAIR=1): cluster pairs with tcgen05 cta_group::2 -- one
  // M = 256 MMA stream per pair of SMs, each SM on its own tile.  Correct (the
  // parity tests pass in this mode) but slower today: the two tiles advance in
  // lockstep and the cross-CTA handshakes (peer half of every weight chunk,
  // epilogue arrivals) leave the issuer waiting ~60% of the time.
  static const char* pe = getenv("TLP_TC_PAIR");
  const bool pair = pe && pe[0] == '1' && ctx->num_sms >= 2 && a.ntile >= 2;
  const int grid = pair ? (int)std::min<int64_t>((a.ntile + 1) / 2, ctx->num_sms / 2) * 2
                        : (int)std::min<int64_t>(a.ntile, ctx->num_sms);
  // Diagnostics: TLP_TC_TRACE=1 prints CTA 0's epilogue phase timeline (cycles
  // between successive waits/signals) for its first tiles to stderr.
  // (needs a -DTLP_TRACE build, tools/abl_build.sh NAME -DTLP_TRACE)
  static const bool trace = kTrace && getenv("TLP_TC_TRACE") != nullptr;
  long long* d_trace = nullptr;
  if (trace) {
    TLP_CUDA_TRY(cudaMalloc(&d_trace, (kTrW + 8 * kTrM) * sizeof(long long)));
    TLP_CUDA_TRY(cudaMemset(d_trace, 0, (kTrW + 8 * kTrM) * sizeof(long long)));
  }
  a.trace = d_trace;
  if (pair) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = w.smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    TLP_CUDA_TRY(cudaLaunchKernelEx(&cfg, tc_forward_kernel<true>, a));
  } else {
    tc_forward_kernel<false><<<grid, kThreads, w.smem, s>>>(a);
  }
  TLP_LAUNCH_CHECK();
  if (trace) {
    std::vector<long long> h(kTrW + 8 * kTrM);
    TLP_CUDA_TRY(cudaStreamSynchronize(s));
    TLP_CUDA_TRY(cudaMemcpy(h.data(), d_trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(d_trace);
    for (int t = 1; t < 4; ++t) {
      fprintf(stderr, "tile %d:", t);
      for (int e = 1; e < kTrEv && h[t * kTrEv + e]; ++e) fprintf(stderr, " %lld", h[t * kTrEv + e] - h[t * kTrEv + e - 1]);
      fprintf(stderr, " | total %lld\n", h[(t + 1) * kTrEv] ? h[(t + 1) * kTrEv] - h[t * kTrEv] : 0LL);
      const long long* m = &h[kTrW + t * kTrM];
      fprintf(stderr, "  mma issuer waits: chunks %lld, qkv-read %lld, O_j %lld, operands %lld (tile %lld)\n",
              m[0], m[1], m[2], m[3], m[kTrM + 4] ? m[kTrM + 4] - m[4] : 0LL);
      fprintf(stderr, "  mma phases (cycles / chunk waits): upsample %lld / %lld, attention %lld / %lld, "
              "residual %lld / %lld, heads %lld / %lld\n", m[5] - m[4], m[8], m[6] - m[5], m[9],
              m[7] - m[6], m[10], m[kTrM + 4] ? m[kTrM + 4] - m[7] : 0LL, m[11]);
    }
  }
  return TLP_OK;
}

void tc_free(tlp_ctx* ctx) {
  if (!ctx->tc) return;
  cudaFree(ctx->tc->wstream);
  cudaFree(ctx->tc->chunks);
  cudaFree(ctx->tc->pack);
  cudaFree(ctx->tc->vec);
  cudaFree(ctx->tc->pos);
  delete ctx->tc;
  ctx->tc = nullptr;
}

// ---------------------------------------------------------------- test hook
namespace {
// D[128 x N] = A[128 x K] * B[N x K]^T through one UMMA chain.  a_tmem != 0:
// the A operand is first written to TMEM (bf16 pairs) with tcgen05.st and the
// MMA reads it from there (the form used for U1, r-halves and P_j).
__global__ void umma_test_kernel(const float* A, const float* B, float* D, int N, int K,
                                 int a_tmem) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t sb = tc::smem_u32(sm);
  const uint32_t offA = 0, offB = 128 * K * 2, offBar = offB + N * K * 2, offT = offBar + 8;
  for (int e = threadIdx.x; e < 128 * K; e += blockDim.x)
    *reinterpret_cast<__nv_bfloat16*>(sm + offA + tc::canon_off(e / K, e % K, K)) = __float2bfloat16_rn(A[e]);
  for (int e = threadIdx.x; e < N * K; e += blockDim.x)
    *reinterpret_cast<__nv_bfloat16*>(sm + offB + tc::canon_off(e / K, e % K, K)) = __float2bfloat16_rn(B[e]);
  uint32_t* tp = reinterpret_cast<uint32_t*>(sm + offT);
  if (threadIdx.x == 0) { tc::mbar_init(sb + offBar, 1); tc::fence_barrier_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(tc::smem_u32(tp), 512);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = *tp;
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const uint32_t a_col = 256;  // A staged at TMEM columns [256, 256 + K/2)
  if (a_tmem) {
    const int r = 32 * w + ln;
    for (int c = 0; c < K; c += 32) {
      uint32_t pk[16];
      for (int i = 0; i < 16; ++i) pk[i] = tc::pack_bf16(A[r * K + c + 2 * i], A[r * K + c + 2 * i + 1]);
      tc::tmem_st16(tm + ((32 * w) << 16) + a_col + c / 2, pk);
    }
    tc::tmem_wait_st();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
  }
  if (threadIdx.x == 0) {
    const uint32_t id = tc::idesc_bf16(128, N);
    for (int ks = 0; ks < K; ks += 16) {
      const uint64_t bd = tc::smem_desc(sb + offB + (ks >> 3) * 128, 128, K * 16);
      if (a_tmem)
        tc::mma_bf16_ta(tm, tm + a_col + ks / 2, bd, id, ks > 0);
      else
        tc::mma_bf16(tm, tc::smem_desc(sb + offA + (ks >> 3) * 128, 128, K * 16), bd, id, ks > 0);
    }
    tc::mma_commit(sb + offBar);
  }
  tc::mbar_wait(sb + offBar, 0);
  tc::tc_fence_after();
  for (int c = 0; c < N; c += 32) {
    float v[32];
    tc::tmem_ld32(tm + ((32 * w) << 16) + c, v);
    tc::tmem_wait_ld();
    for (int i = 0; i < 32 && c + i < N; ++i) D[(32 * w + ln) * N + c + i] = v[i];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc::tc_fence_after(); tc::tmem_dealloc(tm, 512); }
}
}  // namespace

extern "C" tlp_status tlp_debug_umma(const float* A, const float* B, float* D, int32_t N,
                                     int32_t K, int32_t a_in_tmem, void* stream) {
  if (N < 16 || N > 256 || N % 16 || K < 32 || K % 32 || K > 256) return TLP_ERR_ARG;
  const size_t smem = (size_t)128 * K * 2 + (size_t)N * K * 2 + 64;
  cudaFuncSetAttribute(umma_test_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  umma_test_kernel<<<1, 128, smem, reinterpret_cast<cudaStream_t>(stream)>>>(A, B, D, N, K, a_in_tmem);
  return cudaGetLastError() == cudaSuccess ? TLP_OK : TLP_ERR_CUDA;
}
