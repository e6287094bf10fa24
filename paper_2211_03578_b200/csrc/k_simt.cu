// The layer-by-layer network: the fp32 SIMT kernels of the 1e-5-relative path
// (TLP_PREC_FP32), and the training forward/backward orchestration of both
// precisions -- a bf16 context routes every dense layer, dgrad and wgrad to the
// bf16x3 tcgen05 GEMMs of k_tc_gemm.cu and the attention core to k_attn_tc.cu.
//
// Forward (readings R8-R14 in DESIGN.md):
//   h = relu(relu(X W1 + b1) W2 + b2)                    upsample (R11)
//   h = h + softmax(Q K^T / sqrt(d_h)) V Wo + bo        per head, no mask (R8), no PE (R9), R10
//   h = h + relu(h Wa + a) Wb + b                        residual blocks (R12)
//   s_t = (sum_l relu(h_l W1_t + c1_t)) . w2_t + L c2_t  head + sum (R13)
// Backward: chain rule of the same (relu'(0) = 0), weight gradients reduced in
// a fixed order (split over rows + ordered partial sums) so training is
// deterministic.
//
// Kernels: a register-blocked 128x128x8 SGEMM with fused epilogues (bias,
// residual, ReLU, ReLU-mask, accumulate) used for every dense layer and every
// dgrad/wgrad, one-warp-per-(candidate, head) attention forward/backward, and
// the head pooling kernels.  No tensor cores here: TF32 could not meet 1e-5.
#include "tlp_internal.cuh"

#include <algorithm>
#include <cmath>

namespace {

constexpr int BM = 128, BN = 128, BK = 8, PADS = 4;

template <bool TA, bool TB>
__device__ __forceinline__ void load_tiles(const float* __restrict__ A, int64_t lda,
                                           const float* __restrict__ B, int64_t ldb, int64_t M,
                                           int64_t N, int64_t m0, int64_t n0, int64_t k0,
                                           int64_t kend, float ra[4], float rb[4]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int64_t i, k;
    if (TA) { k = t / 32; i = (t % 32) * 4 + q; }
    else { i = t / 2; k = (t % 2) * 4 + q; }
    const int64_t gi = m0 + i, gk = k0 + k;
    ra[q] = (gi < M && gk < kend) ? (TA ? A[gk * lda + gi] : A[gi * lda + gk]) : 0.f;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int64_t j, k;
    if (TB) { j = t / 2; k = (t % 2) * 4 + q; }
    else { k = t / 32; j = (t % 32) * 4 + q; }
    const int64_t gj = n0 + j, gk = k0 + k;
    rb[q] = (gj < N && gk < kend) ? (TB ? B[gj * ldb + gk] : B[gk * ldb + gj]) : 0.f;
  }
}

template <bool TA, bool TB>
__device__ __forceinline__ void store_tiles(float (*As)[BM + PADS], float (*Bs)[BN + PADS],
                                            const float ra[4], const float rb[4]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (TA) As[t / 32][(t % 32) * 4 + q] = ra[q];
    else As[(t % 2) * 4 + q][t / 2] = ra[q];
    if (TB) Bs[(t % 2) * 4 + q][t / 2] = rb[q];
    else Bs[t / 32][(t % 32) * 4 + q] = rb[q];
  }
}

struct EpiDev {
  const float* bias;
  const float* resid;
  int64_t ldr;
  const float* mask;
  int64_t ldm;
  int relu;
  int accumulate;
  int mask_after;
};

// C[M,N] = epi(op(A)[M,K] op(B)[K,N]).  blockIdx.z selects a K slice of
// length kslice; with gridDim.z > 1 the raw partial goes to C + z * M * ldc.
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) sgemm_kernel(int64_t M, int64_t N, int64_t K,
                                                    const float* __restrict__ A, int64_t lda,
                                                    const float* __restrict__ B, int64_t ldb,
                                                    float* __restrict__ C, int64_t ldc,
                                                    EpiDev ep, int64_t kslice) {
  __shared__ __align__(16) float As[2][BK][BM + PADS];
  __shared__ __align__(16) float Bs[2][BK][BN + PADS];
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t kb = (int64_t)blockIdx.z * kslice;
  const int64_t ke = std::min<int64_t>(K, kb + kslice);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  float ra[4], rb[4];
  load_tiles<TA, TB>(A, lda, B, ldb, M, N, m0, n0, kb, ke, ra, rb);
  store_tiles<TA, TB>(As[0], Bs[0], ra, rb);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    const bool more = k0 + BK < ke;
    if (more) load_tiles<TA, TB>(A, lda, B, ldb, M, N, m0, n0, k0 + BK, ke, ra, rb);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[8], b[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][k][64 + tx * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) {
      store_tiles<TA, TB>(As[buf ^ 1], Bs[buf ^ 1], ra, rb);
      __syncthreads();
      buf ^= 1;
    }
  }
  float* Cz = C + (int64_t)blockIdx.z * M * ldc;
  const bool partial = gridDim.z > 1;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t gi = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (gi >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t gj = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (gj >= N) continue;
      float v = acc[i][j];
      if (!partial) {
        if (ep.bias) v += ep.bias[gj];
        if (ep.resid) v += ep.resid[gi * ep.ldr + gj];
        if (ep.relu) v = fmaxf(v, 0.f);
        if (ep.mask && !ep.mask_after) v = ep.mask[gi * ep.ldm + gj] > 0.f ? v : 0.f;
        if (ep.accumulate) v += Cz[gi * ldc + gj];
        if (ep.mask && ep.mask_after) v = ep.mask[gi * ep.ldm + gj] > 0.f ? v : 0.f;
      }
      Cz[gi * ldc + gj] = v;
    }
  }
}

// out[j] = sum_z part[z][j], fixed order.  (A float4 variant with a quarter of
// the threads measured slower: 249 vs 142 us per step -- fewer loads in flight.)
__global__ void reduce_partials(const float* __restrict__ part, int64_t n, int Z,
                                float* __restrict__ out) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  // 16 loads in flight per thread (one partial row per load), then added in
  // z order: the same fixed-order sum, 16x the memory-level parallelism (a
  // (K+1) x N output is only ~65K threads -- 14 warps per SM)
  float s = 0.f;
  int z = 0;
  for (; z + 16 <= Z; z += 16) {
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __ldg(part + (int64_t)(z + i) * n + j);
#pragma unroll
    for (int i = 0; i < 16; ++i) s += v[i];
  }
  for (; z < Z; ++z) s += part[(int64_t)z * n + j];
  out[j] = s;
}

// X [M, E] -> [M, 32] with zero columns E..31 (16-byte rows for TMA)
__global__ void pad_cols_kernel(const float* __restrict__ X, int64_t M, int E, float* __restrict__ out) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  // one 16-byte output group (4 columns) per thread: 8 threads per row
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M * 8) return;
  const int64_t r = e >> 3;
  const int c = (int)(e & 7) * 4;
  const float* x = X + r * E;
  float4 v;
  v.x = c < E ? __ldg(x + c) : 0.f;
  v.y = c + 1 < E ? __ldg(x + c + 1) : 0.f;
  v.z = c + 2 < E ? __ldg(x + c + 2) : 0.f;
  v.w = c + 3 < E ? __ldg(x + c + 3) : 0.f;
  reinterpret_cast<float4*>(out)[e] = v;
}

// The padded first layer's weight + bias partials [Z][Kpad + 1][N] -> the R24
// (W [Kreal][N], b [N]) pair (contiguous at out): rows >= Kreal of W are the
// zero padding and are dropped; the bias is partial row Kpad.  Fixed order.
// One warp per output (few outputs, many partials): lane-strided partial sums
// combined by a fixed butterfly (deterministic).
__global__ void reduce_partials_pad(const float* __restrict__ part, int Kreal, int Kpad, int N, int Z,
                                    float* __restrict__ out) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= (int64_t)(Kreal + 1) * N) return;
  const int row = (int)(j / N), col = (int)(j % N);
  const int srow = row < Kreal ? row : Kpad;
  const int64_t stride = (int64_t)(Kpad + 1) * N;
  float s = 0.f;
  for (int z = lane; z < Z; z += 32) s += part[z * stride + (int64_t)srow * N + col];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[j] = s;
}

// Same sum for few outputs and many partials (column sums): one warp per
// output, lane-strided partial sums combined by a fixed butterfly
// (deterministic for given n, Z).
__global__ void reduce_partials_warp(const float* __restrict__ part, int64_t n, int Z,
                                     float* __restrict__ out) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  float s = 0.f;
  for (int z = lane; z < Z; z += 32) s += part[(int64_t)z * n + j];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[j] = s;
}

__global__ void colsum_partial(int64_t M, int64_t N, const float* __restrict__ X, int64_t ldx,
                               int64_t rows, float* __restrict__ part) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows, r1 = std::min<int64_t>(M, r0 + rows);
  // four interleaved partial sums (rows i, i+1, i+2, i+3 mod 4) for memory-level
  // parallelism, combined in a fixed order: deterministic for a given M
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  int64_t i = r0;
  for (; i + 3 < r1; i += 4) {
    a0 += X[i * ldx + j];
    a1 += X[(i + 1) * ldx + j];
    a2 += X[(i + 2) * ldx + j];
    a3 += X[(i + 3) * ldx + j];
  }
  for (; i < r1; ++i) a0 += X[i * ldx + j];
  part[(int64_t)blockIdx.y * N + j] = (a0 + a1) + (a2 + a3);
}

// ---------------------------------------------------------------------------
// attention, one warp per (candidate, head); lane = query row (L <= 32)
// R43 (NEXT-3): out[n*L + l, :] = h[n*L + l, :] + pos[l, :]
__global__ void add_pos_kernel(const float* __restrict__ h, const float* __restrict__ pos, int64_t M,
                               int L, int H, float* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M * H) return;
  const int64_t r = e / H;
  out[e] = h[e] + pos[(r % L) * H + (e % H)];
}

// R43: dpos[l, c] = sum_n dh[n*L + l, c], fixed order over n
__global__ void pos_grad_kernel(const float* __restrict__ dh, int64_t N, int L, int H,
                                float* __restrict__ dpos) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)L * H) return;
  float a0 = 0.f, a1 = 0.f;
  int64_t n = 0;
  for (; n + 1 < N; n += 2) {
    a0 += dh[(n * L) * H + e];
    a1 += dh[((n + 1) * L) * H + e];
  }
  if (n < N) a0 += dh[(n * L) * H + e];
  dpos[e] = a0 + a1;
}

// R42 (NEXT-3): kvalid[r] = 1 unless input row r is all zeros (a padding row)
__global__ void row_valid_kernel(const float* __restrict__ X, int64_t M, int E,
                                 float* __restrict__ kvalid) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  bool v = false;
  for (int c = 0; c < E; ++c) v |= X[r * E + c] != 0.f;
  kvalid[r] = v ? 1.f : 0.f;
}

template <int DH>
__global__ void __launch_bounds__(128) attn_fwd_kernel(const float* __restrict__ QKV, int L,
                                                       int H, int nh, int64_t pairs,
                                                       float* __restrict__ O,
                                                       float* __restrict__ Asave,
                                                       const float* __restrict__ kvalid) {
  extern __shared__ float sm[];
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t pair = (int64_t)blockIdx.x * (blockDim.x / 32) + w;
  if (pair >= pairs) return;
  float* Ks = sm + w * 2 * 32 * DH;
  float* Vs = Ks + 32 * DH;
  const int64_t n = pair / nh;
  const int hd = (int)(pair % nh);
  const int64_t row0 = n * L;
  const int64_t ld = 3 * (int64_t)H;
  for (int e = lane; e < L * DH; e += 32) {
    const int m = e / DH, d = e % DH;
    Ks[m * DH + d] = QKV[(row0 + m) * ld + H + hd * DH + d];
    Vs[m * DH + d] = QKV[(row0 + m) * ld + 2 * H + hd * DH + d];
  }
  __syncwarp();
  if (lane < L) {
    float q[DH];
#pragma unroll
    for (int d = 0; d < DH; ++d) q[d] = QKV[(row0 + lane) * ld + hd * DH + d];
    const float scale = 1.0f / sqrtf((float)DH);
    float s[32];
    float mx = -INFINITY;
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      if (m < L) {
        float a = 0.f;
#pragma unroll
        for (int d = 0; d < DH; ++d) a = fmaf(q[d], Ks[m * DH + d], a);
        s[m] = (kvalid && kvalid[row0 + m] == 0.f) ? -INFINITY : a * scale;  // R42 mask
        mx = fmaxf(mx, s[m]);
      }
    }
    if (mx == -INFINITY) {  // no valid key (cannot come from tlp_encode): attend uniformly
#pragma unroll
      for (int m = 0; m < 32; ++m)
        if (m < L) s[m] = 0.f;
      mx = 0.f;
    }
    float sum = 0.f;
#pragma unroll
    for (int m = 0; m < 32; ++m)
      if (m < L) { s[m] = expf(s[m] - mx); sum += s[m]; }
    const float inv = 1.0f / sum;
    float o[DH];
#pragma unroll
    for (int d = 0; d < DH; ++d) o[d] = 0.f;
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      if (m < L) {
        s[m] *= inv;
#pragma unroll
        for (int d = 0; d < DH; ++d) o[d] = fmaf(s[m], Vs[m * DH + d], o[d]);
      }
    }
#pragma unroll
    for (int d = 0; d < DH; ++d) O[(row0 + lane) * H + hd * DH + d] = o[d];
    if (Asave) {
      float* Ar = Asave + ((n * nh + hd) * L + lane) * (int64_t)L;
#pragma unroll
      for (int m = 0; m < 32; ++m)
        if (m < L) Ar[m] = s[m];
    }
  }
}

template <int DH>
__global__ void __launch_bounds__(64) attn_bwd_kernel(const float* __restrict__ QKV,
                                                      const float* __restrict__ Asave,
                                                      const float* __restrict__ dO, int L, int H,
                                                      int nh, int64_t pairs,
                                                      float* __restrict__ dQKV) {
  extern __shared__ float sm[];
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t pair = (int64_t)blockIdx.x * (blockDim.x / 32) + w;
  if (pair >= pairs) return;
  const int per = 4 * 32 * DH + 2 * 32 * 33;
  float* Qs = sm + w * per;
  float* Ks = Qs + 32 * DH;
  float* Vs = Ks + 32 * DH;
  float* dOs = Vs + 32 * DH;
  float* As = dOs + 32 * DH;   // [32][33]
  float* dSs = As + 32 * 33;   // [32][33]
  const int64_t n = pair / nh;
  const int hd = (int)(pair % nh);
  const int64_t row0 = n * L;
  const int64_t ld = 3 * (int64_t)H;
  for (int e = lane; e < L * DH; e += 32) {
    const int m = e / DH, d = e % DH;
    const int64_t r = (row0 + m) * ld + hd * DH + d;
    Qs[m * DH + d] = QKV[r];
    Ks[m * DH + d] = QKV[r + H];
    Vs[m * DH + d] = QKV[r + 2 * H];
    dOs[m * DH + d] = dO[(row0 + m) * H + hd * DH + d];
  }
  const float* Ab = Asave + (n * nh + hd) * (int64_t)L * L;
  for (int e = lane; e < L * L; e += 32) As[(e / L) * 33 + (e % L)] = Ab[e];
  __syncwarp();
  const float scale = 1.0f / sqrtf((float)DH);
  if (lane < L) {
    const int l = lane;
    float dA[32];
    float rowdot = 0.f;
    float dor[DH];  // this lane's dO row in registers (row reads of dOs would be 32-way bank conflicts)
#pragma unroll
    for (int d = 0; d < DH; ++d) dor[d] = dO[(row0 + l) * H + hd * DH + d];
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      if (m < L) {
        float a = 0.f;
#pragma unroll
        for (int d = 0; d < DH; ++d) a = fmaf(dor[d], Vs[m * DH + d], a);
        dA[m] = a;
        rowdot = fmaf(a, As[l * 33 + m], rowdot);
      }
    }
    float dq[DH];
#pragma unroll
    for (int d = 0; d < DH; ++d) dq[d] = 0.f;
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      if (m < L) {
        const float ds = As[l * 33 + m] * (dA[m] - rowdot);
        dSs[l * 33 + m] = ds;
#pragma unroll
        for (int d = 0; d < DH; ++d) dq[d] = fmaf(ds, Ks[m * DH + d], dq[d]);
      }
    }
#pragma unroll
    for (int d = 0; d < DH; ++d) dQKV[(row0 + l) * ld + hd * DH + d] = dq[d] * scale;
  }
  __syncwarp();
  if (lane < L) {
    const int m = lane;
    float dk[DH], dv[DH];
#pragma unroll
    for (int d = 0; d < DH; ++d) { dk[d] = 0.f; dv[d] = 0.f; }
    for (int l = 0; l < L; ++l) {
      const float ds = dSs[l * 33 + m], a = As[l * 33 + m];
#pragma unroll
      for (int d = 0; d < DH; ++d) {
        dk[d] = fmaf(ds, Qs[l * DH + d], dk[d]);
        dv[d] = fmaf(a, dOs[l * DH + d], dv[d]);
      }
    }
#pragma unroll
    for (int d = 0; d < DH; ++d) {
      dQKV[(row0 + m) * ld + H + hd * DH + d] = dk[d] * scale;
      dQKV[(row0 + m) * ld + 2 * H + hd * DH + d] = dv[d];
    }
  }
}

// ---------------------------------------------------------------------------
// head: pooled[n,k] = sum_l relu(U[n*L+l, k]); s[n,t] = pooled . w2 + L c2
__global__ void head_pool_kernel(const float* __restrict__ U, int64_t uld, int L, int hd, int64_t N,
                                 const float* __restrict__ w2, const float* __restrict__ c2,
                                 int t, int nt, float* __restrict__ pooled,
                                 float* __restrict__ scores) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t n = (int64_t)blockIdx.x * (blockDim.x / 32) + w;
  if (n >= N) return;
  float dot = 0.f;
  if (hd == 128 && uld % 4 == 0 && ((reinterpret_cast<uintptr_t>(U) | reinterpret_cast<uintptr_t>(w2) |
                                     reinterpret_cast<uintptr_t>(pooled)) & 15) == 0) {
    // hd = 128: lane owns columns 4 lane .. 4 lane + 3 (16-byte loads)
    const float4* U4 = reinterpret_cast<const float4*>(U);
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
    int l = 0;
    for (; l + 8 <= L; l += 8) {  // 8 row loads in flight, summed in row order
      float4 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __ldg(U4 + (n * L + l + i) * (uld >> 2) + lane);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        p.x += fmaxf(v[i].x, 0.f); p.y += fmaxf(v[i].y, 0.f);
        p.z += fmaxf(v[i].z, 0.f); p.w += fmaxf(v[i].w, 0.f);
      }
    }
    for (; l < L; ++l) {
      const float4 v = __ldg(U4 + (n * L + l) * (uld >> 2) + lane);
      p.x += fmaxf(v.x, 0.f); p.y += fmaxf(v.y, 0.f); p.z += fmaxf(v.z, 0.f); p.w += fmaxf(v.w, 0.f);
    }
    if (pooled) reinterpret_cast<float4*>(pooled + n * hd)[lane] = p;
    const float4 w = __ldg(reinterpret_cast<const float4*>(w2) + lane);
    dot = fmaf(p.w, w.w, fmaf(p.z, w.z, fmaf(p.y, w.y, p.x * w.x)));
  } else
  for (int k = lane; k < hd; k += 32) {
    float p = 0.f;
    int l = 0;
    for (; l + 8 <= L; l += 8) {  // 8 row loads in flight, summed in row order
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __ldg(U + (n * L + l + i) * uld + k);
#pragma unroll
      for (int i = 0; i < 8; ++i) p += fmaxf(v[i], 0.f);
    }
    for (; l < L; ++l) p += fmaxf(U[(n * L + l) * uld + k], 0.f);
    if (pooled) pooled[n * hd + k] = p;
    dot = fmaf(p, w2[k], dot);
  }
  for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  if (lane == 0) scores[n * nt + t] = dot + (float)L * c2[0];
}

// dU[n*L+l, k] = g[n,t] * w2[k] * (U > 0)
__global__ void head_bwd_kernel(const float* __restrict__ U, int64_t uld, int L, int hd, int64_t N,
                                const float* __restrict__ w2, const float* __restrict__ g, int t,
                                int nt, float* __restrict__ dU, int vec) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  if (vec) {  // float4 per thread, one row-segment: 32-bit row index, no 64-bit division
    const int q = hd >> 2;
    const int64_t e4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e4 >= N * L * q) return;
    const int64_t row = e4 / q;
    const int k = (int)(e4 - row * q) * 4;
    const float gn = __ldg(g + (row / L) * nt + t);
    const int64_t o4 = (row * uld + k) >> 2;  // U and dU share the row stride
    const float4 u = __ldg(reinterpret_cast<const float4*>(U) + o4);
    const float4 w = __ldg(reinterpret_cast<const float4*>(w2 + k));
    reinterpret_cast<float4*>(dU)[o4] = make_float4(u.x > 0.f ? gn * w.x : 0.f, u.y > 0.f ? gn * w.y : 0.f,
                                                    u.z > 0.f ? gn * w.z : 0.f, u.w > 0.f ? gn * w.w : 0.f);
    return;
  }
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * L * hd) return;
  const int k = (int)(e % hd);
  const int64_t row = e / hd, n = row / L, o = row * uld + k;
  dU[o] = U[o] > 0.f ? g[n * nt + t] * w2[k] : 0.f;
}

// Wcat = [Wq | Wk | Wv] rows side by side, then [bq | bk | bv] (the fused Q/K/V
// GEMM operands, k_simt.cu simt_forward / simt_backward): one launch instead of
// six device copies
__global__ void pack_wcat_kernel(const float* __restrict__ P, int64_t w0, int64_t w1, int64_t w2,
                                 int64_t b0, int64_t b1, int64_t b2, int H, float* __restrict__ wcat) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t H3 = 3 * (int64_t)H, nW = H3 * H;
  if (e < nW) {
    const int64_t i = e / H3;
    const int c = (int)(e - i * H3), j = c / H, k = c - j * H;
    wcat[e] = P[(j == 0 ? w0 : j == 1 ? w1 : w2) + i * H + k];
  } else if (e < nW + H3) {
    const int c = (int)(e - nW), j = c / H, k = c - j * H;
    wcat[e] = P[(j == 0 ? b0 : j == 1 ? b1 : b2) + k];
  }
}

// [W1_0 | W1_1 | ...] ([H, nt hd], row stride nt hd) then [c1_0 | c1_1 | ...]
struct HeadOffs { int64_t w[TLP_MAX_TASKS], c[TLP_MAX_TASKS]; };
__global__ void pack_heads_kernel(const float* __restrict__ P, HeadOffs o, int nt, int H, int hd,
                                  float* __restrict__ out) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t W = (int64_t)nt * hd, nW = (int64_t)H * W;
  if (e < nW) {
    const int64_t i = e / W;
    const int cc = (int)(e - i * W), t = cc / hd, k = cc - t * hd;
    out[e] = P[o.w[t] + i * hd + k];
  } else if (e < nW + W) {
    const int cc = (int)(e - nW), t = cc / hd, k = cc - t * hd;
    out[e] = P[o.c[t] + k];
  }
}

// out = L * sum_n g[n, t]   (single block, fixed order)
__global__ void dc2_kernel(const float* __restrict__ g, int64_t N, int t, int nt, int L,
                           float* __restrict__ out) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  __shared__ float red[256];
  float s = 0.f;
  for (int64_t n = threadIdx.x; n < N; n += blockDim.x) s += g[n * nt + t];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = (float)L * red[0];
}

// ---------------------------------------------------------------- R49 LSTM (NEXT-4)
// Step t of a layer, thread per (candidate, unit j).  gates row (n, t) holds
// the pre-activation z = h_t Wih + bih + h_{t-1} Whh + bhh (written by the step
// GEMM); it is overwritten by the activated [i, f, g, o] that backward needs.
// c_t -> C, h_t -> hprev row t+1 (the next step's GEMM operand and dWhh's
// A operand), layer output hin + h_t -> hout (identity residual, R49).
// Full-precision expf / tanhf (R29).
__device__ __forceinline__ float sigmoid_f(float x) { return 1.0f / (1.0f + expf(-x)); }

__global__ void lstm_cell_fwd(int64_t n, int L, int H, int t, float* __restrict__ gates,
                              float* __restrict__ C, float* __restrict__ hprev,
                              const float* __restrict__ hin, float* __restrict__ hout) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * H) return;
  const int64_t cand = idx / H;
  const int j = (int)(idx - cand * H);
  const int64_t row = cand * L + t;
  float* z = gates + row * 4 * H;
  const float i = sigmoid_f(z[j]), f = sigmoid_f(z[H + j]);
  const float g = tanhf(z[2 * H + j]), o = sigmoid_f(z[3 * H + j]);
  const float cp = t > 0 ? C[(row - 1) * H + j] : 0.f;
  const float c = f * cp + i * g;
  const float hl = o * tanhf(c);
  z[j] = i; z[H + j] = f; z[2 * H + j] = g; z[3 * H + j] = o;
  C[row * H + j] = c;
  if (t + 1 < L) hprev[(row + 1) * H + j] = hl;
  hout[row * H + j] = hin[row * H + j] + hl;
}

// Backward of step t: dh_t = dout_t + dhr (= dz_{t+1} Whh^T), carried dc;
// writes dz_t (pre-activation gradients) into dG.
__global__ void lstm_cell_bwd(int64_t n, int L, int H, int t, const float* __restrict__ gates,
                              const float* __restrict__ C, const float* __restrict__ dout,
                              const float* __restrict__ dhr, float* __restrict__ dcar,
                              float* __restrict__ dG) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * H) return;
  const int64_t cand = idx / H;
  const int j = (int)(idx - cand * H);
  const int64_t row = cand * L + t;
  const float* z = gates + row * 4 * H;
  const float i = z[j], f = z[H + j], g = z[2 * H + j], o = z[3 * H + j];
  const float c = C[row * H + j];
  const float cp = t > 0 ? C[(row - 1) * H + j] : 0.f;
  const float dht = dout[row * H + j] + (t + 1 < L ? dhr[cand * H + j] : 0.f);
  const float tc = tanhf(c);
  const float dc = (t + 1 < L ? dcar[cand * H + j] : 0.f) + dht * o * (1.f - tc * tc);
  dcar[cand * H + j] = dc * f;
  float* d = dG + row * 4 * H;
  d[j] = dc * g * i * (1.f - i);
  d[H + j] = dc * cp * f * (1.f - f);
  d[2 * H + j] = dc * i * (1.f - g * g);
  d[3 * H + j] = dht * tc * o * (1.f - o);
}

__global__ void relu_mask_inplace(float* __restrict__ d, const float* __restrict__ act,
                                  int64_t n) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n && !(act[e] > 0.f)) d[e] = 0.f;
}

// ---------------------------------------------------------------------------
// activation layout for a chunk of N candidates (fp32 elements)
struct ActLayout {
  int64_t up[TLP_MAX_UP];
  int64_t qkv[TLP_MAX_ATTN], A[TLP_MAX_ATTN], O[TLP_MAX_ATTN], hattn[TLP_MAX_ATTN];
  // R49 LSTM layers: input projection, gates (pre-activation -> activated),
  // cell states, shifted hidden states (row t holds h_{t-1}, row 0 zero)
  int64_t xg[TLP_MAX_ATTN], gates[TLP_MAX_ATTN], cst[TLP_MAX_ATTN], hprev[TLP_MAX_ATTN];
  int64_t dG, dcar, dhr;  // LSTM backward scratch
  int64_t r[TLP_MAX_RES], hres[TLP_MAX_RES];
  int64_t U[TLP_MAX_TASKS], pooled[TLP_MAX_TASKS];
  int64_t kvalid;  // R42 key-validity flags (attn_mask)
  int64_t hpos;    // R43 upsample output + positional table (pos_enc)
  int64_t xpad;    // X padded to 32 columns (bf16 training: 16-byte rows for TMA), or -1
  // backward scratch
  int64_t dh, dtmp, dqkv, dU;
  int64_t total_fwd, total;
};

ActLayout act_layout(const tlp_config& c, int64_t N) {
  ActLayout a{};
  const int64_t M = N * c.L, H = c.hidden;
  int64_t o = 0;
  auto take = [&](int64_t n) { int64_t r = o; o += (n + 63) / 64 * 64; return r; };
  for (int i = 0; i < c.n_up; ++i) a.up[i] = take(M * c.up_dims[i]);
  for (int l = 0; l < c.n_attn; ++l) {
    if (c.backbone == 1) {
      a.xg[l] = take(M * 4 * H);
      a.gates[l] = take(M * 4 * H);
      a.cst[l] = take(M * H);
      a.hprev[l] = take(M * H);
    } else {
      a.qkv[l] = take(M * 3 * H);
      a.A[l] = take(N * c.attn_heads * (int64_t)c.L * c.L);
      a.O[l] = take(M * H);
    }
    a.hattn[l] = take(M * H);
  }
  for (int r = 0; r < c.n_res; ++r) { a.r[r] = take(M * H); a.hres[r] = take(M * H); }
  // the heads' first-layer outputs side by side, [M, n_tasks hd] (row stride
  // uld): one GEMM for every task's first layer, one K = n_tasks hd dgrad
  const int64_t ucat = take(M * c.n_tasks * c.head_dim);
  for (int t = 0; t < c.n_tasks; ++t) { a.U[t] = ucat + t * c.head_dim; a.pooled[t] = take(N * c.head_dim); }
  a.kvalid = take(M);
  a.hpos = take(M * H);
  a.xpad = (c.precision == TLP_PREC_BF16 && c.E % 4 != 0 && c.E <= 32) ? take(M * 32) : -1;
  a.total_fwd = o;
  a.dh = take(M * H);
  a.dtmp = take(M * std::max<int64_t>(H, c.up_dims[0]));
  a.dqkv = take(M * 3 * H);
  a.dU = take(M * c.n_tasks * c.head_dim);  // [M, n_tasks hd] like U
  if (c.backbone == 1 && c.n_attn > 0) {
    a.dG = take(M * 4 * H);
    a.dcar = take(N * H);
    a.dhr = take(N * H);
  }
  a.total = o;
  return a;
}

template <int DH>
tlp_status launch_attn_fwd(tlp_ctx* ctx, const float* qkv, int64_t N, float* O, float* A,
                           const float* kvalid, cudaStream_t s) {
  const tlp_config& c = ctx->cfg;
  const int64_t pairs = N * c.attn_heads;
  const int warps = 4;
  const size_t smem = (size_t)warps * 2 * 32 * DH * sizeof(float);
  attn_fwd_kernel<DH><<<(unsigned)cdiv(pairs, warps), warps * 32, smem, s>>>(
      qkv, c.L, c.hidden, c.attn_heads, pairs, O, A, kvalid);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

template <int DH>
tlp_status launch_attn_bwd(tlp_ctx* ctx, const float* qkv, const float* A, const float* dO,
                           int64_t N, float* dqkv, cudaStream_t s) {
  const tlp_config& c = ctx->cfg;
  const int64_t pairs = N * c.attn_heads;
  const int warps = 2;
  const size_t smem = (size_t)warps * (4 * 32 * DH + 2 * 32 * 33) * sizeof(float);
  TLP_SMEM_ATTR(attn_bwd_kernel<DH>, smem);
  attn_bwd_kernel<DH><<<(unsigned)cdiv(pairs, warps), warps * 32, smem, s>>>(
      qkv, A, dO, c.L, c.hidden, c.attn_heads, pairs, dqkv);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

tlp_status attn_fwd(tlp_ctx* ctx, const float* qkv, int64_t N, float* O, float* A,
                    const float* kvalid, cudaStream_t s) {
  if (attn_tc_ok(ctx)) return attn_fwd_tc(ctx, qkv, N, O, A, kvalid, s);  // bf16 ctx: tensor cores
  switch (ctx->cfg.hidden / ctx->cfg.attn_heads) {
    case 8: return launch_attn_fwd<8>(ctx, qkv, N, O, A, kvalid, s);
    case 16: return launch_attn_fwd<16>(ctx, qkv, N, O, A, kvalid, s);
    case 32: return launch_attn_fwd<32>(ctx, qkv, N, O, A, kvalid, s);
    case 64: return launch_attn_fwd<64>(ctx, qkv, N, O, A, kvalid, s);
    default: ctx->last_error = "head dim must be 8/16/32/64"; return TLP_ERR_UNSUPPORTED;
  }
}

tlp_status attn_bwd(tlp_ctx* ctx, const float* qkv, const float* A, const float* dO, int64_t N,
                    float* dqkv, cudaStream_t s) {
  if (attn_tc_ok(ctx)) return attn_bwd_tc(ctx, qkv, A, dO, N, dqkv, s);  // bf16 ctx: tensor cores
  switch (ctx->cfg.hidden / ctx->cfg.attn_heads) {
    case 8: return launch_attn_bwd<8>(ctx, qkv, A, dO, N, dqkv, s);
    case 16: return launch_attn_bwd<16>(ctx, qkv, A, dO, N, dqkv, s);
    case 32: return launch_attn_bwd<32>(ctx, qkv, A, dO, N, dqkv, s);
    case 64: return launch_attn_bwd<64>(ctx, qkv, A, dO, N, dqkv, s);
    default: ctx->last_error = "head dim must be 8/16/32/64"; return TLP_ERR_UNSUPPORTED;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
tlp_status sgemm(tlp_ctx* ctx, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A,
                 int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                 const EpiParams& e, cudaStream_t s) {
  if (M == 0 || N == 0) return TLP_OK;
  // TLP_PREC_BF16 contexts train on the tensor cores (tf32 tcgen05) whenever the
  // operands allow 16-byte async copies; the fp32 context stays on FFMA (1e-5).
  if (ctx->cfg.precision == TLP_PREC_BF16)
    return tc_gemm(ctx, ta, tb, M, N, K, A, lda, B, ldb, C, ldc, e, 1, K, s);
  EpiDev ed{e.bias, e.resid, e.ldr, e.mask, e.ldm, e.relu ? 1 : 0, e.accumulate ? 1 : 0, e.mask_after ? 1 : 0};
  dim3 grid((unsigned)cdiv(N, BN), (unsigned)cdiv(M, BM), 1);
  const int64_t ks = K > 0 ? K : 1;
  if (!ta && !tb) sgemm_kernel<false, false><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, ed, ks);
  else if (!ta && tb) sgemm_kernel<false, true><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, ed, ks);
  else if (ta && !tb) sgemm_kernel<true, false><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, ed, ks);
  else sgemm_kernel<true, true><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, ed, ks);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

// dW[k] = sum_m A[m][k] dY[m] (a single output column: the head's w2
// gradient): row slices per block, thread per k (coalesced rows), fp32 FMA in
// row order; partials reduced in a fixed order.
__global__ void wgrad_n1_kernel(int64_t M, int K, const float* __restrict__ A, int64_t lda,
                                const float* __restrict__ dY, int64_t lddy, int64_t rows,
                                float* __restrict__ part) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  const int64_t m0 = (int64_t)blockIdx.x * rows;
  const int64_t m1 = M < m0 + rows ? M : m0 + rows;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    float acc = 0.f;
    int64_t m = m0;
    for (; m + 8 <= m1; m += 8) {  // 8 row loads in flight, then the same fixed-order chain
      float a[8], d[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        a[i] = __ldg(A + (m + i) * lda + k);
        d[i] = __ldg(dY + (m + i) * lddy);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) acc = fmaf(a[i], d[i], acc);
    }
    for (; m < m1; ++m) acc = fmaf(A[m * lda + k], dY[m * lddy], acc);
    part[(int64_t)blockIdx.x * K + k] = acc;
  }
}

tlp_status sgemm_wgrad(tlp_ctx* ctx, int64_t M, int64_t K, int64_t N, const float* A, int64_t lda,
                       const float* dY, int64_t lddy, float* dW, cudaStream_t s) {
  // dW[K,N] = A^T dY with A [M,K] (ld lda), dY [M,N] (ld lddy).  Split over the
  // M rows into Z fixed slices (a function of M only) -> ordered reduction.
  if (N == 1 && K <= 1024) {
    const int Zn = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(M, 32), 512));  // slices of 32 rows
    const int64_t rows = cdiv(M, Zn);
    TLP_CUDA_TRY(ctx->ws_partial.ensure((size_t)Zn * K * sizeof(float)));
    float* part = ctx->ws_partial.as<float>();
    TLP_LAUNCH_PDL(wgrad_n1_kernel, (unsigned)Zn, 128, 0, s, M, (int)K, A, lda, dY, lddy, rows, part);
    TLP_LAUNCH_CHECK();
    TLP_LAUNCH_PDL(reduce_partials, (unsigned)cdiv(K, 256), 256, 0, s, part, K, Zn, dW);
    TLP_LAUNCH_CHECK();
    return TLP_OK;
  }
  const int64_t slice = 2048;
  const int Z = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(M, slice), 256));
  const int64_t kslice = cdiv(cdiv(M, Z), BK) * BK;
  EpiDev ed{nullptr, nullptr, 0, nullptr, 0, 0, 0};
  dim3 grid((unsigned)cdiv(N, BN), (unsigned)cdiv(K, BM), (unsigned)Z);
  if (ctx->cfg.precision == TLP_PREC_BF16) {
    EpiParams none;
    if (Z == 1) return tc_gemm(ctx, true, false, K, N, M, A, lda, dY, lddy, dW, N, none, 1, M, s);
    TLP_CUDA_TRY(ctx->ws_partial.ensure((size_t)Z * K * N * sizeof(float)));
    float* part = ctx->ws_partial.as<float>();
    tlp_status st = tc_gemm(ctx, true, false, K, N, M, A, lda, dY, lddy, part, N, none, Z, kslice, s);
    if (st != TLP_OK) return st;
    TLP_LAUNCH_PDL(reduce_partials, (unsigned)cdiv(K * N, 256), 256, 0, s, part, K * N, Z, dW);
    TLP_LAUNCH_CHECK();
    return TLP_OK;
  }
  if (Z == 1) {
    sgemm_kernel<true, false><<<grid, 256, 0, s>>>(K, N, M, A, lda, dY, lddy, dW, N, ed, kslice);
    TLP_LAUNCH_CHECK();
    return TLP_OK;
  }
  TLP_CUDA_TRY(ctx->ws_partial.ensure((size_t)Z * K * N * sizeof(float)));
  float* part = ctx->ws_partial.as<float>();
  sgemm_kernel<true, false><<<grid, 256, 0, s>>>(K, N, M, A, lda, dY, lddy, part, N, ed, kslice);
  TLP_LAUNCH_CHECK();
  TLP_LAUNCH_PDL(reduce_partials, (unsigned)cdiv(K * N, 256), 256, 0, s, part, K * N, Z, dW);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

// R52: the TMA-fed kind::tf32 weight-gradient kernel (k_tc_tma.cu) on bf16
// contexts: one row slice per SM (J products share them), partials
// [J][Z][K + 1][N] reduced in a fixed order.  Returns TLP_ERR_UNSUPPORTED if the
// shapes do not fit it (nothing launched).
static tlp_status wgrad_bias_tma(tlp_ctx* ctx, int J, int64_t M, int64_t K, int64_t N, const float* A,
                                 int64_t lda, const float* dY, int64_t lddy, int64_t jcol,
                                 float* const* dW, cudaStream_t s) {
  if (ctx->cfg.precision != TLP_PREC_BF16) return TLP_ERR_UNSUPPORTED;
  for (int j = 0; j < J; ++j)
    if (dW[j] == nullptr) return TLP_ERR_UNSUPPORTED;
  int Z = std::max(1, ctx->num_sms / J);
  const int64_t kslice = cdiv(cdiv(M, Z), 32) * 32;
  Z = (int)cdiv(M, kslice);
  const int64_t pj = (int64_t)Z * (K + 1) * N;
  TLP_CUDA_TRY(ctx->ws_partial.ensure((size_t)J * pj * sizeof(float)));
  float* part = ctx->ws_partial.as<float>();
  tlp_status st = tc_wgrad_tma(ctx, M, K, N, A, lda, dY, lddy, part, Z, kslice, true, J, jcol, s);
  if (st != TLP_OK) return st;
  for (int j = 0; j < J; ++j) {
    TLP_LAUNCH_PDL(reduce_partials, (unsigned)cdiv((K + 1) * N, 256), 256, 0, s, part + j * pj, (K + 1) * N, Z, dW[j]);
    TLP_LAUNCH_CHECK();
  }
  return TLP_OK;
}

// The first layer's weight + bias gradient from the padded X [M, 32] (bf16
// contexts, E <= 32): the TMA tf32 wgrad kernel over Kpad = 32 columns, then
// reduce_partials_pad into W [Kreal][N] | b [N] (R52).  Falls back to the
// generic path on the original X if the kernel does not apply.
static tlp_status wgrad_bias_padded(tlp_ctx* ctx, int64_t M, int64_t Kreal, int64_t N, const float* X32,
                                    const float* dY, float* dWdb, cudaStream_t s) {
  int Z = std::max(1, ctx->num_sms);
  const int64_t kslice = cdiv(cdiv(M, Z), 32) * 32;
  Z = (int)cdiv(M, kslice);
  TLP_CUDA_TRY(ctx->ws_partial.ensure((size_t)Z * 33 * N * sizeof(float)));
  float* part = ctx->ws_partial.as<float>();
  tlp_status st = tc_wgrad_tma(ctx, M, 32, N, X32, 32, dY, N, part, Z, kslice, true, 1, 0, s);
  if (st == TLP_ERR_UNSUPPORTED)
    return sgemm_wgrad_bias(ctx, M, Kreal, N, ctx->train_X, Kreal, dY, N, dWdb, dWdb + Kreal * N, s);
  if (st != TLP_OK) return st;
  TLP_LAUNCH_PDL(reduce_partials_pad, (unsigned)cdiv((Kreal + 1) * N * 32, 256), 256, 0, s, part, (int)Kreal, 32, (int)N, Z, dWdb);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

tlp_status sgemm_wgrad_bias(tlp_ctx* ctx, int64_t M, int64_t K, int64_t N, const float* A, int64_t lda,
                            const float* dY, int64_t lddy, float* dW, float* db, cudaStream_t s) {
  if (db == dW + K * N) {
    float* const dws[1] = {dW};
    const tlp_status ts = wgrad_bias_tma(ctx, 1, M, K, N, A, lda, dY, lddy, 0, dws, s);
    if (ts != TLP_ERR_UNSUPPORTED) return ts;
  }
  const int64_t slice = 2048;
  const int Z = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(M, slice), 256));
  const int64_t kslice = cdiv(cdiv(M, Z), BK) * BK;
  if (ctx->cfg.precision == TLP_PREC_BF16 && db == dW + K * N && Z > 1) {
    TLP_CUDA_TRY(ctx->ws_partial.ensure((size_t)Z * (K + 1) * N * sizeof(float)));
    float* part = ctx->ws_partial.as<float>();
    tlp_status st = TLP_OK;
    if (tc_wgrad_bias(ctx, K, N, M, A, lda, dY, lddy, part, Z, kslice, s, &st)) {
      if (st != TLP_OK) return st;
      TLP_LAUNCH_PDL(reduce_partials, (unsigned)cdiv((K + 1) * N, 256), 256, 0, s, part, (K + 1) * N, Z, dW);
      TLP_LAUNCH_CHECK();
      return TLP_OK;
    }
  }
  tlp_status st = sgemm_wgrad(ctx, M, K, N, A, lda, dY, lddy, dW, s);
  if (st != TLP_OK) return st;
  return colsum(ctx, M, N, dY, lddy, db, s);
}

// J weight + bias gradients that share the activation A (the Q/K/V projections):
// dY_j = dY + j * jcol (columns of one [M, J*N] array), dW_j / db_j = dW[j] / dW[j] + K*N.
// bf16 contexts: one wgrad launch (A read from HBM once per slice); else J calls.
tlp_status sgemm_wgrad_bias_shared(tlp_ctx* ctx, int J, int64_t M, int64_t K, int64_t N, const float* A,
                                   int64_t lda, const float* dY, int64_t lddy, int64_t jcol,
                                   float* const* dW, cudaStream_t s) {
  {
    const tlp_status ts = wgrad_bias_tma(ctx, J, M, K, N, A, lda, dY, lddy, jcol, dW, s);
    if (ts != TLP_ERR_UNSUPPORTED) return ts;
  }
  const int64_t slice = 2048;
  const int Z = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(M, slice), 256));
  const int64_t kslice = cdiv(cdiv(M, Z), BK) * BK;
  if (ctx->cfg.precision == TLP_PREC_BF16 && Z > 1) {
    const int64_t pj = (int64_t)Z * (K + 1) * N;
    TLP_CUDA_TRY(ctx->ws_partial.ensure((size_t)J * pj * sizeof(float)));
    float* part = ctx->ws_partial.as<float>();
    tlp_status st = TLP_OK;
    if (tc_wgrad_bias(ctx, K, N, M, A, lda, dY, lddy, part, Z, kslice, s, &st, J, jcol, pj)) {
      if (st != TLP_OK) return st;
      for (int j = 0; j < J; ++j) {
        TLP_LAUNCH_PDL(reduce_partials, (unsigned)cdiv((K + 1) * N, 256), 256, 0, s, part + j * pj, (K + 1) * N, Z, dW[j]);
        TLP_LAUNCH_CHECK();
      }
      return TLP_OK;
    }
  }
  for (int j = 0; j < J; ++j) {
    tlp_status st = sgemm_wgrad_bias(ctx, M, K, N, A, lda, dY + j * jcol, lddy, dW[j], dW[j] + K * N, s);
    if (st != TLP_OK) return st;
  }
  return TLP_OK;
}

tlp_status colsum(tlp_ctx* ctx, int64_t M, int64_t N, const float* X, int64_t ldx, float* out,
                  cudaStream_t s) {
  const int64_t rows = 256;
  const int Z = (int)std::max<int64_t>(1, cdiv(M, rows));
  TLP_CUDA_TRY(ctx->ws_misc.ensure((size_t)Z * N * sizeof(float) + 4096));
  float* part = ctx->ws_misc.as<float>();
  colsum_partial<<<dim3((unsigned)cdiv(N, 128), (unsigned)Z), 128, 0, s>>>(M, N, X, ldx, rows, part);
  TLP_LAUNCH_CHECK();
  reduce_partials_warp<<<(unsigned)cdiv(N * 32, 256), 256, 0, s>>>(part, N, Z, out);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

#define TRY(x) do { tlp_status _s = (x); if (_s != TLP_OK) return _s; } while (0)

static bool heads_cat(const tlp_config& c) {
  const int64_t uld = (int64_t)c.n_tasks * c.head_dim;
  return c.n_tasks > 1 && (uld <= 256 || uld % 256 == 0);
}

tlp_status simt_forward(tlp_ctx* ctx, const float* X, int64_t N, float* scores, bool save,
                        cudaStream_t s) {
  const tlp_config& c = ctx->cfg;
  const ParamOffsets& o = ctx->off;
  const float* P = ctx->d_params;
  const int64_t H = c.hidden;
  // inference processes bounded chunks; training keeps the whole batch
  // (LSTM: larger chunks, so each of the L sequential step GEMMs has more rows)
  const int64_t chunk = save ? N : std::min<int64_t>(N, c.backbone == 1 ? 65536 : 8192);
  ActLayout lay = act_layout(c, chunk);
  TLP_CUDA_TRY(ctx->ws_act.ensure((size_t)(save ? lay.total : lay.total_fwd) * sizeof(float)));
  float* W = ctx->ws_act.as<float>();
  // Wcat[i][jH + k] = W_j[i][k] per attention layer, packed up front: the
  // weight images of the GEMMs are built ahead of their GEMMs (bimg_kernel)
  // and must only read operands final since the step began
  if (c.n_attn && c.backbone == 0) {
    const int64_t wcat_stride = ((3 * H * H + 3 * H) + 63) / 64 * 64;  // floats per layer
    TLP_CUDA_TRY(ctx->ws_wcat.ensure((size_t)c.n_attn * wcat_stride * sizeof(float)));
    for (int l = 0; l < c.n_attn; ++l) {
      TLP_LAUNCH_PDL(pack_wcat_kernel, (unsigned)cdiv(3 * H * H + 3 * H, 256), 256, 0, s, P, o.Wq[l], o.Wk[l],
                     o.Wv[l], o.bq[l], o.bk[l], o.bv[l], (int)H, ctx->ws_wcat.as<float>() + l * wcat_stride);
      TLP_LAUNCH_CHECK();
    }
  }
  // MTL: the heads' first layers side by side (one N = n_tasks hd GEMM) when
  // the TMA GEMM takes that width (<= 256 or a multiple of 256)
  const bool hcat = heads_cat(c);
  if (hcat) {
    const int64_t uld = (int64_t)c.n_tasks * c.head_dim;
    TLP_CUDA_TRY(ctx->ws_hcat.ensure((size_t)(H * uld + uld) * sizeof(float)));
    HeadOffs ho{};
    for (int t = 0; t < c.n_tasks; ++t) { ho.w[t] = o.W1[t]; ho.c[t] = o.c1[t]; }
    TLP_LAUNCH_PDL(pack_heads_kernel, (unsigned)cdiv(H * uld + uld, 256), 256, 0, s, P, ho, c.n_tasks, (int)H,
                   c.head_dim, ctx->ws_hcat.as<float>());
    TLP_LAUNCH_CHECK();
  }
  for (int64_t n0 = 0; n0 < N; n0 += chunk) {
    const int64_t n = std::min(chunk, N - n0);
    const int64_t M = n * c.L;
    const float* h = X + n0 * c.L * c.E;
    const float* kvalid = nullptr;
    if (c.attn_mask && c.n_attn > 0) {
      row_valid_kernel<<<(unsigned)cdiv(M, 256), 256, 0, s>>>(h, M, c.E, W + lay.kvalid);
      TLP_LAUNCH_CHECK();
      kvalid = W + lay.kvalid;
    }
    int64_t din = c.E, ldh = c.E;
    if (save && lay.xpad >= 0) {
      // E = 22 rows are 88 bytes, which TMA cannot address: one padded copy
      // [M, 32] (zero columns E..31) feeds the first layer's TMA GEMM here and
      // its weight gradient in the backward
      TLP_LAUNCH_PDL(pad_cols_kernel, (unsigned)cdiv(M * 8, 256), 256, 0, s, h, M, c.E, W + lay.xpad);
      TLP_LAUNCH_CHECK();
      h = W + lay.xpad;
      ldh = 32;
    }
    for (int i = 0; i < c.n_up; ++i) {
      EpiParams e; e.bias = P + o.up_b[i]; e.relu = true;
      TRY(sgemm(ctx, false, false, M, c.up_dims[i], din, h, ldh, P + o.up_W[i], c.up_dims[i],
                W + lay.up[i], c.up_dims[i], e, s));
      h = W + lay.up[i];
      din = c.up_dims[i];
      ldh = din;
    }
    if (c.pos_enc) {  // R43
      add_pos_kernel<<<(unsigned)cdiv(M * H, 256), 256, 0, s>>>(h, P + o.pos, M, c.L, (int)H, W + lay.hpos);
      TLP_LAUNCH_CHECK();
      h = W + lay.hpos;
    }
    for (int l = 0; l < c.n_attn && c.backbone == 1; ++l) {  // R49
      const int64_t H4 = 4 * H;
      float* xg = W + lay.xg[l];
      float* gt = W + lay.gates[l];
      float* hp = W + lay.hprev[l];
      EpiParams ex; ex.bias = P + o.bih[l];
      TRY(sgemm(ctx, false, false, M, H4, H, h, H, P + o.Wih[l], H4, xg, H4, ex, s));
      TLP_CUDA_TRY(cudaMemset2DAsync(hp, (size_t)c.L * H * sizeof(float), 0, (size_t)H * sizeof(float),
                                     (size_t)n, s));  // h_{-1} = 0
      for (int t = 0; t < c.L; ++t) {
        EpiParams eh; eh.bias = P + o.bhh[l]; eh.resid = xg + t * H4; eh.ldr = c.L * H4;
        TRY(sgemm(ctx, false, false, n, H4, H, hp + t * H, c.L * H, P + o.Whh[l], H4, gt + t * H4,
                  c.L * H4, eh, s));
        lstm_cell_fwd<<<(unsigned)cdiv(n * H, 256), 256, 0, s>>>(n, c.L, (int)H, t, gt, W + lay.cst[l], hp,
                                                                 h, W + lay.hattn[l]);
        TLP_LAUNCH_CHECK();
      }
      h = W + lay.hattn[l];
    }
    const int64_t wcat_stride = ((3 * H * H + 3 * H) + 63) / 64 * 64;  // floats per layer
    for (int l = 0; l < c.n_attn && c.backbone == 0; ++l) {
      float* qkv = W + lay.qkv[l];
      // [Q | K | V] = h [Wq | Wk | Wv] + [bq | bk | bv] as ONE N = 3H GEMM (h read
      // once); Wcat (packed before the chunk loop) kept for the backward's fused dgrad
      float* wcat = ctx->ws_wcat.as<float>() + l * wcat_stride;
      float* bcat = wcat + 3 * H * H;
      EpiParams eq; eq.bias = bcat;
      TRY(sgemm(ctx, false, false, M, 3 * H, H, h, H, wcat, 3 * H, qkv, 3 * H, eq, s));
      TRY(attn_fwd(ctx, qkv, n, W + lay.O[l], save ? W + lay.A[l] : nullptr, kvalid, s));
      EpiParams e; e.bias = P + o.bo[l]; e.resid = h; e.ldr = H;
      TRY(sgemm(ctx, false, false, M, H, H, W + lay.O[l], H, P + o.Wo[l], H, W + lay.hattn[l], H, e, s));
      h = W + lay.hattn[l];
    }
    for (int r = 0; r < c.n_res; ++r) {
      EpiParams e1; e1.bias = P + o.a[r]; e1.relu = true;
      TRY(sgemm(ctx, false, false, M, H, H, h, H, P + o.Wa[r], H, W + lay.r[r], H, e1, s));
      EpiParams e2; e2.bias = P + o.b[r]; e2.resid = h; e2.ldr = H;
      TRY(sgemm(ctx, false, false, M, H, H, W + lay.r[r], H, P + o.Wb[r], H, W + lay.hres[r], H, e2, s));
      h = W + lay.hres[r];
    }
    const int64_t uld = (int64_t)c.n_tasks * c.head_dim;
    if (hcat) {  // every task's first head layer as ONE GEMM (h read once)
      EpiParams e; e.bias = ctx->ws_hcat.as<float>() + H * uld;
      TRY(sgemm(ctx, false, false, M, uld, H, h, H, ctx->ws_hcat.as<float>(), uld, W + lay.U[0], uld, e, s));
    }
    for (int t = 0; t < c.n_tasks; ++t) {
      if (!hcat) {
        EpiParams e; e.bias = P + o.c1[t];
        TRY(sgemm(ctx, false, false, M, c.head_dim, H, h, H, P + o.W1[t], c.head_dim, W + lay.U[t],
                  uld, e, s));
      }
      TLP_LAUNCH_PDL(head_pool_kernel, (unsigned)cdiv(n, 8), 256, 0, s, 
          W + lay.U[t], uld, c.L, c.head_dim, n, P + o.w2[t], P + o.c2[t], t, c.n_tasks,
          save ? W + lay.pooled[t] : nullptr, scores + n0 * c.n_tasks);
      TLP_LAUNCH_CHECK();
    }
  }
  if (save) {
    ctx->train_N = N;
    ctx->train_X = X;
  }
  return TLP_OK;
}

tlp_status simt_backward(tlp_ctx* ctx, int64_t N, const float* g, cudaStream_t s) {
  const tlp_config& c = ctx->cfg;
  const ParamOffsets& o = ctx->off;
  const float* P = ctx->d_params;
  float* G = ctx->d_grads;
  if (ctx->train_N != N) { ctx->last_error = "backward without matching forward"; return TLP_ERR_STATE; }
  const ActLayout lay = act_layout(c, N);
  float* W = ctx->ws_act.as<float>();
  const int64_t H = c.hidden, M = N * c.L, hd = c.head_dim;
  float* dh = W + lay.dh;
  float* dtmp = W + lay.dtmp;
  float* dqkv = W + lay.dqkv;
  float* dU = W + lay.dU;
  const float* hfin = c.n_res ? W + lay.hres[c.n_res - 1]
                    : (c.n_attn ? W + lay.hattn[c.n_attn - 1] : (c.pos_enc ? W + lay.hpos : W + lay.up[c.n_up - 1]));
  // heads (dU of task t at columns [t hd, t hd + hd) of a [M, n_tasks hd] block)
  const int64_t uld = (int64_t)c.n_tasks * hd;
  const bool hcat = heads_cat(c);
  bool w1c1 = true;  // R24: c1_t right after W1_t (one shared-X weight-gradient launch)
  for (int t = 0; t < c.n_tasks; ++t) w1c1 &= o.c1[t] == o.W1[t] + H * hd;
  for (int t = 0; t < c.n_tasks; ++t) {
    // (the float4 path needs 16-byte aligned U / dU / w2: act_layout slots are
    // 64-float aligned; w2's flat offset may not be)
    const bool v4 = hd % 4 == 0 && (reinterpret_cast<uintptr_t>(P + o.w2[t]) & 15) == 0;
    TLP_LAUNCH_PDL(head_bwd_kernel, (unsigned)cdiv(v4 ? M * hd / 4 : M * hd, 256), 256, 0, s, 
        W + lay.U[t], uld, c.L, hd, N, P + o.w2[t], g, t, c.n_tasks, dU + t * hd, v4 ? 1 : 0);
    TLP_LAUNCH_CHECK();
    if (!(hcat && w1c1))
      TRY(sgemm_wgrad_bias(ctx, M, H, hd, hfin, H, dU + t * hd, uld, G + o.W1[t], G + o.c1[t], s));
    TRY(sgemm_wgrad(ctx, N, hd, 1, W + lay.pooled[t], hd, g + t, c.n_tasks, G + o.w2[t], s));
    TLP_LAUNCH_PDL(dc2_kernel, 1, 256, 0, s, g, N, t, c.n_tasks, c.L, G + o.c2[t]);
    TLP_LAUNCH_CHECK();
    if (!hcat) {
      EpiParams e; e.accumulate = t > 0;
      TRY(sgemm(ctx, false, true, M, H, hd, dU + t * hd, uld, P + o.W1[t], hd, dh, H, e, s));
    }
  }
  if (hcat && w1c1) {  // every task's W1 | c1 gradient from one pass over hfin
    float* dws[TLP_MAX_TASKS];
    for (int t = 0; t < c.n_tasks; ++t) dws[t] = G + o.W1[t];
    TRY(sgemm_wgrad_bias_shared(ctx, c.n_tasks, M, H, hd, hfin, H, dU, uld, hd, dws, s));
  }
  if (hcat) {  // dh = [dU_0 | dU_1 | ...] [W1_0 | W1_1 | ...]^T: one K = n_tasks hd GEMM
    EpiParams e;
    TRY(sgemm(ctx, false, true, M, H, uld, dU, uld, ctx->ws_hcat.as<float>(), uld, dh, H, e, s));
  }
  // C-1 buckets in reverse R24 order: heads | residual blocks | attention (or
  // LSTM) layers | upsample + positional table
  const int64_t b_heads = o.W1[0];
  const int64_t b_res = c.n_res ? o.Wa[0] : b_heads;
  const int64_t b_mid = c.n_attn ? (c.backbone == 1 ? o.Wih[0] : o.Wq[0]) : b_res;
  TRY(grad_bucket_ready(ctx, b_heads, o.total, s));
  // residual blocks
  for (int r = c.n_res - 1; r >= 0; --r) {
    const float* hin = r > 0 ? W + lay.hres[r - 1]
                     : (c.n_attn ? W + lay.hattn[c.n_attn - 1] : (c.pos_enc ? W + lay.hpos : W + lay.up[c.n_up - 1]));
    const float* rr = W + lay.r[r];
    TRY(sgemm_wgrad_bias(ctx, M, H, H, rr, H, dh, H, G + o.Wb[r], G + o.b[r], s));
    EpiParams em; em.mask = rr; em.ldm = H;
    TRY(sgemm(ctx, false, true, M, H, H, dh, H, P + o.Wb[r], H, dtmp, H, em, s));
    TRY(sgemm_wgrad_bias(ctx, M, H, H, hin, H, dtmp, H, G + o.Wa[r], G + o.a[r], s));
    EpiParams ea; ea.accumulate = true;
    TRY(sgemm(ctx, false, true, M, H, H, dtmp, H, P + o.Wa[r], H, dh, H, ea, s));
  }
  TRY(grad_bucket_ready(ctx, b_res, b_heads, s));
  // R49 LSTM layers: backpropagation through time, then the batched weight gradients
  for (int l = c.n_attn - 1; l >= 0 && c.backbone == 1; --l) {
    const float* hin = l > 0 ? W + lay.hattn[l - 1] : (c.pos_enc ? W + lay.hpos : W + lay.up[c.n_up - 1]);
    const int64_t H4 = 4 * H;
    float* dG = W + lay.dG;
    for (int t = c.L - 1; t >= 0; --t) {
      lstm_cell_bwd<<<(unsigned)cdiv(N * H, 256), 256, 0, s>>>(N, c.L, (int)H, t, W + lay.gates[l],
                                                               W + lay.cst[l], dh, W + lay.dhr,
                                                               W + lay.dcar, dG);
      TLP_LAUNCH_CHECK();
      if (t > 0) {
        EpiParams e0;
        TRY(sgemm(ctx, false, true, N, H, H4, dG + t * H4, c.L * H4, P + o.Whh[l], H4, W + lay.dhr, H, e0, s));
      }
    }
    TRY(sgemm_wgrad(ctx, M, H, H4, hin, H, dG, H4, G + o.Wih[l], s));
    TRY(sgemm_wgrad(ctx, M, H, H4, W + lay.hprev[l], H, dG, H4, G + o.Whh[l], s));
    TRY(colsum(ctx, M, H4, dG, H4, G + o.bih[l], s));
    TLP_CUDA_TRY(cudaMemcpyAsync(G + o.bhh[l], G + o.bih[l], H4 * sizeof(float), cudaMemcpyDeviceToDevice, s));
    EpiParams ea; ea.accumulate = true;
    TRY(sgemm(ctx, false, true, M, H, H4, dG, H4, P + o.Wih[l], H4, dh, H, ea, s));
  }
  // attention layers
  int up_masked = -1;  // upsample layer whose ReLU' a GEMM epilogue already applied to `cur`
  for (int l = c.n_attn - 1; l >= 0 && c.backbone == 0; --l) {
    const float* hin = l > 0 ? W + lay.hattn[l - 1] : (c.pos_enc ? W + lay.hpos : W + lay.up[c.n_up - 1]);
    TRY(sgemm_wgrad_bias(ctx, M, H, H, W + lay.O[l], H, dh, H, G + o.Wo[l], G + o.bo[l], s));
    EpiParams e0;
    TRY(sgemm(ctx, false, true, M, H, H, dh, H, P + o.Wo[l], H, dtmp, H, e0, s));  // dO
    TRY(attn_bwd(ctx, W + lay.qkv[l], W + lay.A[l], dtmp, N, dqkv, s));
    const int64_t wq[3] = {o.Wq[l], o.Wk[l], o.Wv[l]}, bq[3] = {o.bq[l], o.bk[l], o.bv[l]};
    bool contiguous = true;  // R24: each bias right after its weight
    for (int j = 0; j < 3; ++j) contiguous &= bq[j] == wq[j] + H * H;
    if (contiguous) {
      float* const dws[3] = {G + wq[0], G + wq[1], G + wq[2]};
      TRY(sgemm_wgrad_bias_shared(ctx, 3, M, H, H, hin, H, dqkv, 3 * H, H, dws, s));
    } else {
      for (int j = 0; j < 3; ++j)
        TRY(sgemm_wgrad_bias(ctx, M, H, H, hin, H, dqkv + j * H, 3 * H, G + wq[j], G + bq[j], s));
    }
    // dh += [dQ | dK | dV] [Wq | Wk | Wv]^T as ONE K = 3H GEMM (dqkv read once,
    // dh read and written once instead of three times), on the Wcat the
    // forward built (simt_backward always follows simt_forward(save))
    const float* wcat = ctx->ws_wcat.as<float>() + l * ((((3 * H * H + 3 * H) + 63) / 64) * 64);
    EpiParams ea; ea.accumulate = true;
    if (l == 0 && !c.pos_enc) {  // dh is final here: fold the upsample ReLU' (relu_mask) in
      ea.mask = W + lay.up[c.n_up - 1]; ea.ldm = H; ea.mask_after = true;
      up_masked = c.n_up - 1;
    }
    TRY(sgemm(ctx, false, true, M, H, 3 * H, dqkv, 3 * H, wcat, 3 * H, dh, H, ea, s));
  }
  TRY(grad_bucket_ready(ctx, b_mid, b_res, s));
  // R43: dpos = sum over candidates; d(up_out) = d(up_out + pos) unchanged
  if (c.pos_enc) {
    pos_grad_kernel<<<(unsigned)cdiv((int64_t)c.L * H, 256), 256, 0, s>>>(dh, N, c.L, (int)H, G + o.pos);
    TLP_LAUNCH_CHECK();
  }
  // upsample: dh is d(up_out[n_up-1])
  float* cur = dh;
  for (int i = c.n_up - 1; i >= 0; --i) {
    const int64_t w = c.up_dims[i];
    const int64_t din = i > 0 ? c.up_dims[i - 1] : c.E;
    if (up_masked != i) {
      relu_mask_inplace<<<(unsigned)cdiv(M * w, 256), 256, 0, s>>>(cur, W + lay.up[i], M * w);
      TLP_LAUNCH_CHECK();
    }
    const float* xin = i > 0 ? W + lay.up[i - 1] : ctx->train_X;
    if (i == 0 && lay.xpad >= 0) {
      TRY(wgrad_bias_padded(ctx, M, din, w, W + lay.xpad, cur, G + o.up_W[i], s));
    } else {
      TRY(sgemm_wgrad_bias(ctx, M, din, w, xin, din, cur, w, G + o.up_W[i], G + o.up_b[i], s));
    }
    if (i > 0) {
      float* nxt = (cur == dh) ? dtmp : dh;
      EpiParams e0;  // the next layer's ReLU' rides in this dgrad's epilogue
      e0.mask = W + lay.up[i - 1]; e0.ldm = din;
      up_masked = i - 1;
      TRY(sgemm(ctx, false, true, M, din, w, cur, w, P + o.up_W[i], w, nxt, din, e0, s));
      cur = nxt;
    }
  }
  TRY(grad_bucket_ready(ctx, 0, b_mid, s));
  return TLP_OK;
}

// ---------------------------------------------------------------- test hook
extern "C" tlp_status tlp_debug_wgrad(tlp_ctx* ctx, int64_t M, int64_t K, int64_t N, const float* X,
                                      int64_t ldx, const float* dY, int64_t ldy, float* dWdb,
                                      void* stream) {
  if (!ctx || !X || !dY || !dWdb || M < 1 || K < 1 || N < 1) return TLP_ERR_ARG;
  return sgemm_wgrad_bias(ctx, M, K, N, X, ldx, dY, ldy, dWdb, dWdb + K * N,
                          reinterpret_cast<cudaStream_t>(stream));
}
