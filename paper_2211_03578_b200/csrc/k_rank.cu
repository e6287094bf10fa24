// K9 LambdaRank loss + dL/ds per (group, task), and the strict-pair counts.
//
// Paper: "rank loss [cao2007learning, wang2018lambdaloss]"
// "lambda rank loss designed for ranking tasks", P:409 (chosen).  The formula
// is not printed; reading R16:
//   pi_i  = rank by (s desc, index asc)                       (R17)
//   G_i   = (2^{y_i} - 1) / maxDCG,  maxDCG = max(sum_r (2^{y_(r)}-1)/log2(1+r), 1e-10)
//   pair y_i > y_j:  w = |G_i - G_j| |1/log2(1+pi_i) - 1/log2(1+pi_j)|
//                    l = w log2(1 + exp(-(s_i - s_j)))
//                    dl/ds_i = -(1/ln2) w sigmoid(-(s_i - s_j)) = -dl/ds_j
//   L_t = sum l / P_t  (P_t = strict pairs of task t in the global batch)
// MTL (R19): per task, only items with a present (non-NaN) label.
//
// One CTA per (group, task).  Every item's gradient is the sum over all its
// partners computed by the thread that owns the item (no atomics), so the
// result is deterministic; the O(n^2) pair loop reads the group from shared
// memory (warp-broadcast of the partner j).  2^y - 1 is evaluated as
// expm1(y ln 2) to avoid cancellation for small labels.
#include "tlp_internal.cuh"

#include <algorithm>

namespace {

constexpr int kThreads = 512;
constexpr float kLn2 = 0.693147180559945309f;
constexpr float kInvLn2 = 1.44269504088896341f;  // 1 / ln 2

__device__ __forceinline__ float block_sum(float v, float* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = 0.f;
  if (threadIdx.x < 32) {
    r = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (threadIdx.x == 0) red[0] = r;
  }
  __syncthreads();
  r = red[0];
  __syncthreads();
  return r;
}

// Compact the present items of (group, task) into shared memory, in index order.
// Block-wide: one item per thread per pass, warp ballots + a prefix over the
// warps' counts (the single-warp version walked a 512-item group in 16
// dependent steps and dominated the rank kernels).  Call from every thread.
__device__ int gather_present(const float* __restrict__ scores, const float* __restrict__ labels,
                              int64_t lo, int64_t hi, int t, int nt, float* s, float* y,
                              int* idx) {
  __shared__ int wsum[32];  // inclusive prefix of the warps' present counts
  const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  int base = 0;
  for (int64_t c = lo; c < hi; c += blockDim.x) {
    const int64_t i = c + threadIdx.x;
    float yi = 0.f, si = 0.f;
    bool pres = false;
    if (i < hi) {
      yi = labels[i * nt + t];
      si = scores ? scores[i * nt + t] : 0.f;
      pres = !isnan(yi);
    }
    const unsigned m = __ballot_sync(0xffffffffu, pres);
    if (ln == 0) wsum[w] = __popc(m);
    __syncthreads();
    if (w == 0) {
      int v = ln < nw ? wsum[ln] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (ln >= o) v += u;
      }
      if (ln < nw) wsum[ln] = v;
    }
    __syncthreads();
    const int pos = base + (w ? wsum[w - 1] : 0) + __popc(m & ((1u << ln) - 1u));
    if (pres) { s[pos] = si; y[pos] = yi; idx[pos] = (int)(i - lo); }
    base += wsum[nw - 1];
    __syncthreads();
  }
  return base;
}

__global__ void __launch_bounds__(kThreads) pair_count_kernel(const float* __restrict__ labels,
                                                              const int64_t* __restrict__ goff,
                                                              int nt, double* __restrict__ part) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  extern __shared__ float sm[];
  const int g = blockIdx.x, t = blockIdx.y;
  const int64_t lo = goff[g], hi = goff[g + 1];
  const int cap = (int)(hi - lo);
  float* s = sm;
  float* y = s + cap;
  int* idx = reinterpret_cast<int*>(y + cap);
  const int n = gather_present(nullptr, labels, lo, hi, t, nt, s, y, idx);
  // slice blockIdx.z of the items i (gridDim.z slices: 16 groups alone left
  // 132 SMs idle), eight threads per i each scanning every eighth j
  const int S = gridDim.z, sl = blockIdx.z;
  const int chunk = (n + S - 1) / S, i0 = sl * chunk, i1 = min(n, i0 + chunk);
  unsigned long long cnt = 0;  // exact integers: any summation order
  for (int e = threadIdx.x; e < (i1 - i0) * 8; e += blockDim.x) {
    const float yi = y[i0 + (e >> 3)];
    int c = 0;
    for (int j = e & 7; j < n; j += 8) c += yi > y[j];
    cnt += (unsigned long long)c;
  }
  __shared__ unsigned long long tot;
  if (threadIdx.x == 0) tot = 0;
  __syncthreads();
  // warp sums first: one shared 64-bit atomic per warp (512 on one address
  // serialise) -- exact integers, any order
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&tot, cnt);
  __syncthreads();
  if (threadIdx.x == 0) part[((int64_t)t * gridDim.x + g) * S + sl] = (double)tot;
}

constexpr int kCountSplit = 8;  // pair_count_kernel slices per (group, task)

__global__ void sum_counts(const double* __restrict__ part, int G, int nt,
                           double* __restrict__ counts) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  double s = 0.0;  // integers < 2^53: exact
  for (int g = 0; g < G * kCountSplit; ++g) s += part[(int64_t)t * G * kCountSplit + g];
  counts[t] = s;
}

constexpr int kRankThreads = 1024;  // rank_kernel: two threads per item of a 512-item group; the split kernels size it to the slice

__global__ void __launch_bounds__(kRankThreads) rank_kernel(const float* __restrict__ scores,
                                                        const float* __restrict__ labels,
                                                        const int64_t* __restrict__ goff, int nt,
                                                        float* __restrict__ loss_part,
                                                        float* __restrict__ dscores) {
  extern __shared__ float sm[];
  __shared__ float red[32];
  const int g = blockIdx.x, t = blockIdx.y;
  const int64_t lo = goff[g], hi = goff[g + 1];
  const int cap = (int)(hi - lo);
  float* s = sm;
  float* y = s + cap;
  float* Gs = y + cap;
  float* iD = Gs + cap;
  int* idx = reinterpret_cast<int*>(iD + cap);
  const int n = gather_present(scores, labels, lo, hi, t, nt, s, y, idx);
  // Two threads per item (kRankThreads = 1024: item i = pair tid / 2, each half
  // of the pair scans half of the j range; the halves are combined with one
  // shuffle).  Every thread runs every round so the shuffles see full warps.
  const int half = threadIdx.x & 1, nth = blockDim.x >> 1;
  const int jm = n / 2, j0 = half ? jm : 0, j1 = half ? n : jm;
  // ranks (R17) and ideal ranks -> maxDCG
  float dcg = 0.f;
  for (int base = 0; base < n; base += nth) {
    const int i = base + (threadIdx.x >> 1);
    const bool act = i < n;
    const float si = act ? s[i] : 0.f, yi = act ? y[i] : 0.f;
    int rs = 0, ry = 0;
    if (act) {
      for (int j = j0; j < j1; ++j) {
        const float sj = s[j], yj = y[j];
        rs += (sj > si) || (sj == si && j < i);
        ry += (yj > yi) || (yj == yi && j < i);
      }
    }
    rs += __shfl_xor_sync(0xffffffffu, rs, 1);
    ry += __shfl_xor_sync(0xffffffffu, ry, 1);
    if (act && half == 0) {
      iD[i] = 1.0f / log2f(2.0f + (float)rs);               // rank = 1 + rs
      dcg += expm1f(yi * kLn2) / log2f(2.0f + (float)ry);
    }
  }
  const float maxdcg = fmaxf(block_sum(dcg, red), 1e-10f);
  for (int i = threadIdx.x; i < n; i += blockDim.x) Gs[i] = expm1f(y[i] * kLn2) / maxdcg;
  __syncthreads();
  float lsum = 0.f;
  for (int base = 0; base < n; base += nth) {
    const int i = base + (threadIdx.x >> 1);
    const bool act = i < n;
    float gi = 0.f, li = 0.f;
    if (act) {
      const float si = s[i], yi = y[i], Gi = Gs[i], iDi = iD[i];
      for (int j = j0; j < j1; ++j) {
        const float yj = y[j];
        if (yi == yj) continue;
        const float w = fabsf(Gi - Gs[j]) * fabsf(iDi - iD[j]);
        // z = s_hi - s_lo of the ordered pair
        const float z = (yi > yj) ? (si - s[j]) : (s[j] - si);
        const float e = expf(-fabsf(z));
        const float r = __frcp_rn(1.0f + e);                  // one correctly rounded reciprocal
        const float sig = (z >= 0.f) ? e * r : r;             // sigmoid(-z), sign-stable (R30)
        if (yi > yj) {
          li += w * (fmaxf(-z, 0.f) + log1pf(e));
          gi -= w * sig;
        } else {
          gi += w * sig;
        }
      }
    }
    gi += __shfl_xor_sync(0xffffffffu, gi, 1);
    li += __shfl_xor_sync(0xffffffffu, li, 1);
    if (act && half == 0) {
      // the 1/ln 2 of log2 and of d/ds log2(1 + e^{-z}) applied once per item
      dscores[(lo + idx[i]) * nt + t] = gi * kInvLn2;
      lsum += li * kInvLn2;
    }
  }
  const float L = block_sum(lsum, red);
  if (threadIdx.x == 0) loss_part[(int64_t)t * gridDim.x + g] = L;
}

// Split version (default): each (group, task) is spread over kRankSplit CTAs
// (one CTA per group left 132 of 148 SMs idle on the C3 step).  Pass 1: every
// CTA ranks its slice of the items against the whole group (R17) and writes
// 1/log2(1 + rank) plus its partial ideal DCG; pass 2: every CTA sums the
// partials in a fixed order (maxDCG), and runs the pair loop for its slice.
// Same per-item arithmetic and order as rank_kernel (deterministic).
constexpr int kRankSplit = 8;

__device__ __forceinline__ void slice_of(int n, int sub, int& i0, int& i1) {
  const int per = (n + kRankSplit - 1) / kRankSplit;
  i0 = min(n, sub * per);
  i1 = min(n, i0 + per);
}
// threads per item of a slice: the largest power of two <= 32 that still covers
// the slice's items with the block in one pass (a 512-item group split 8 ways
// leaves 64 items for 1024 threads: 16 per item, each scanning n / 16 of the
// j); the per-item partials combine by a fixed butterfly (deterministic)
__device__ __forceinline__ int threads_per_item(int items) {
  int tpi = 32;
  while (tpi > 2 && tpi * items > (int)blockDim.x) tpi >>= 1;
  return tpi;
}

__global__ void __launch_bounds__(kRankThreads) rank_prep_kernel(const float* __restrict__ scores,
                                                             const float* __restrict__ labels,
                                                             const int64_t* __restrict__ goff, int nt,
                                                             float* __restrict__ iD_out,
                                                             float* __restrict__ dcg_part) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  extern __shared__ float sm[];
  __shared__ float red[32];
  const int g = blockIdx.x / kRankSplit, sub = blockIdx.x % kRankSplit, t = blockIdx.y;
  const int64_t lo = goff[g], hi = goff[g + 1];
  const int cap = (int)(hi - lo);
  float* s = sm;
  float* y = s + cap;
  int* idx = reinterpret_cast<int*>(y + cap);
  const int n = gather_present(scores, labels, lo, hi, t, nt, s, y, idx);
  int i0, i1;
  slice_of(n, sub, i0, i1);
  const int tpi = threads_per_item(i1 - i0), lt = 31 - __clz(tpi);
  const int h = threadIdx.x & (tpi - 1), nth = blockDim.x >> lt;
  float dcg = 0.f;
  for (int base = i0; base < i1; base += nth) {
    const int i = base + (threadIdx.x >> lt);
    const bool act = i < i1;
    const float si = act ? s[i] : 0.f, yi = act ? y[i] : 0.f;
    int rs = 0, ry = 0;
    if (act) {
      for (int j = h; j < n; j += tpi) {  // interleaved j: conflict-free shared reads
        const float sj = s[j], yj = y[j];
        rs += (sj > si) || (sj == si && j < i);
        ry += (yj > yi) || (yj == yi && j < i);
      }
    }
    for (int o = 1; o < tpi; o <<= 1) {  // exact integer ranks
      rs += __shfl_xor_sync(0xffffffffu, rs, o);
      ry += __shfl_xor_sync(0xffffffffu, ry, o);
    }
    if (act && h == 0) {
      iD_out[(int64_t)t * goff[gridDim.x / kRankSplit] + lo + i] = 1.0f / log2f(2.0f + (float)rs);
      dcg += expm1f(yi * kLn2) / log2f(2.0f + (float)ry);
    }
  }
  const float d = block_sum(dcg, red);
  if (threadIdx.x == 0) dcg_part[((int64_t)t * (gridDim.x / kRankSplit) + g) * kRankSplit + sub] = d;
}

__global__ void __launch_bounds__(kRankThreads) rank_pair_kernel(const float* __restrict__ scores,
                                                             const float* __restrict__ labels,
                                                             const int64_t* __restrict__ goff, int nt,
                                                             const float* __restrict__ iD_in,
                                                             const float* __restrict__ dcg_part,
                                                             float* __restrict__ loss_part,
                                                             float* __restrict__ dscores) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  extern __shared__ float sm[];
  __shared__ float red[32];
  const int G = gridDim.x / kRankSplit;
  const int g = blockIdx.x / kRankSplit, sub = blockIdx.x % kRankSplit, t = blockIdx.y;
  const int64_t lo = goff[g], hi = goff[g + 1];
  const int cap = (int)(hi - lo);
  float* s = sm;
  float* y = s + cap;
  float* Gs = y + cap;
  float* iD = Gs + cap;
  int* idx = reinterpret_cast<int*>(iD + cap);
  const int n = gather_present(scores, labels, lo, hi, t, nt, s, y, idx);
  float dsum = 0.f;
  for (int k = 0; k < kRankSplit; ++k) dsum += dcg_part[((int64_t)t * G + g) * kRankSplit + k];  // fixed order
  const float maxdcg = fmaxf(dsum, 1e-10f);
  const float* iDg = iD_in + (int64_t)t * goff[G] + lo;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    Gs[i] = expm1f(y[i] * kLn2) / maxdcg;
    iD[i] = iDg[i];
  }
  __syncthreads();
  int i0, i1;
  slice_of(n, sub, i0, i1);
  const int tpi = threads_per_item(i1 - i0), lt = 31 - __clz(tpi);
  const int h = threadIdx.x & (tpi - 1), nth = blockDim.x >> lt;
  float lsum = 0.f;
  for (int base = i0; base < i1; base += nth) {
    const int i = base + (threadIdx.x >> lt);
    const bool act = i < i1;
    float gi = 0.f, li = 0.f;
    if (act) {
      const float si = s[i], yi = y[i], Gi = Gs[i], iDi = iD[i];
      for (int j = h; j < n; j += tpi) {  // interleaved j: conflict-free shared reads
        const float yj = y[j];
        if (yi == yj) continue;
        const float w = fabsf(Gi - Gs[j]) * fabsf(iDi - iD[j]);
        const float z = (yi > yj) ? (si - s[j]) : (s[j] - si);
        const float e = expf(-fabsf(z));
        const float r = __frcp_rn(1.0f + e);
        const float sig = (z >= 0.f) ? e * r : r;
        if (yi > yj) {
          li += w * (fmaxf(-z, 0.f) + log1pf(e));
          gi -= w * sig;
        } else {
          gi += w * sig;
        }
      }
    }
    for (int o = 1; o < tpi; o <<= 1) {  // fixed butterfly over the item's threads
      gi += __shfl_xor_sync(0xffffffffu, gi, o);
      li += __shfl_xor_sync(0xffffffffu, li, o);
    }
    if (act && h == 0) {
      dscores[(lo + idx[i]) * nt + t] = gi * kInvLn2;
      lsum += li * kInvLn2;
    }
  }
  const float L = block_sum(lsum, red);
  if (threadIdx.x == 0) loss_part[(int64_t)t * gridDim.x + blockIdx.x] = L;
}

__global__ void finalize_rank(const float* __restrict__ loss_part, int G, int nt,
                              const double* __restrict__ counts, float* __restrict__ dscores,
                              int64_t B, float* __restrict__ loss_out, uint32_t* err) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  // scale gradients by 1/P_t, sum the task losses in a fixed order
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < B * nt; e += stride) {
    const int t = (int)(e % nt);
    const double P = counts[t];
    dscores[e] = P > 0 ? (float)((double)dscores[e] / P) : 0.f;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double tot = 0.0;
    for (int t = 0; t < nt; ++t) {
      double lt = 0.0;
      for (int g = 0; g < G; ++g) lt += (double)loss_part[(int64_t)t * G + g];
      if (counts[t] > 0) tot += lt / counts[t];
    }
    const float lf = (float)tot;
    if (isnan(lf)) atomicOr(err, DERR_NAN_LOSS);
    *loss_out = lf;
  }
}

// ---- NEXT-3: MSE (MTL masking S:386-394; R41)
constexpr int kMseBlocks = 64;

// present labels per task (exact integer counts, summed into doubles)
__global__ void mse_count_kernel(const float* __restrict__ labels, int64_t B, int nt,
                                 unsigned long long* __restrict__ cnt) {
  const int t = blockIdx.y;
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x)
    c += !isnan(labels[i * nt + t]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt + t, c);
}

__global__ void mse_counts_to_double(const unsigned long long* __restrict__ cnt, int nt,
                                     double* __restrict__ counts) {
  if (threadIdx.x < nt) counts[threadIdx.x] = (double)cnt[threadIdx.x];
}

// gradient 2 r / n_t and per-(block, task) partial sums of r^2 in a fixed order
__global__ void mse_kernel(const float* __restrict__ scores, const float* __restrict__ labels,
                           int64_t B, int nt, const double* __restrict__ counts,
                           float* __restrict__ dscores, double* __restrict__ part) {
  const int t = blockIdx.y;
  const double n = counts[t];
  __shared__ double red[256];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * nt + t;
    const float y = labels[e];
    float g = 0.f;
    if (!isnan(y) && n > 0) {
      const double r = (double)scores[e] - (double)y;
      acc += r * r;
      g = (float)(2.0 * r / n);
    }
    dscores[e] = g;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(int64_t)t * gridDim.x + blockIdx.x] = red[0];
}

__global__ void mse_finalize(const double* __restrict__ part, int nblk, int nt,
                             const double* __restrict__ counts, float* __restrict__ loss_out,
                             uint32_t* err) {
  double tot = 0.0;
  for (int t = 0; t < nt; ++t) {
    if (!(counts[t] > 0)) continue;
    double lt = 0.0;
    for (int b = 0; b < nblk; ++b) lt += part[(int64_t)t * nblk + b];
    tot += lt / counts[t];
  }
  const float lf = (float)tot;
  if (isnan(lf)) atomicOr(err, DERR_NAN_LOSS);
  *loss_out = lf;
}

}  // namespace

tlp_status mse_counts(tlp_ctx* ctx, const float* labels, int64_t B, double* d_counts, cudaStream_t s) {
  const int nt = ctx->cfg.n_tasks;
  TLP_CUDA_TRY(ctx->ws_rank.ensure((size_t)nt * kMseBlocks * sizeof(double) + 64 * sizeof(unsigned long long)));
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(
      ctx->ws_rank.as<char>() + (size_t)nt * kMseBlocks * sizeof(double));
  TLP_CUDA_TRY(cudaMemsetAsync(cnt, 0, nt * sizeof(unsigned long long), s));
  mse_count_kernel<<<dim3(kMseBlocks, nt), 256, 0, s>>>(labels, B, nt, cnt);
  TLP_LAUNCH_CHECK();
  mse_counts_to_double<<<1, 32, 0, s>>>(cnt, nt, d_counts);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

tlp_status mse_loss_grad(tlp_ctx* ctx, const float* scores, const float* labels, int64_t B,
                         const double* d_counts, float* loss_out, float* dscores, cudaStream_t s) {
  const int nt = ctx->cfg.n_tasks;
  TLP_CUDA_TRY(ctx->ws_rank.ensure((size_t)nt * kMseBlocks * sizeof(double) + 64 * sizeof(unsigned long long)));
  double* part = ctx->ws_rank.as<double>();
  mse_kernel<<<dim3(kMseBlocks, nt), 256, 0, s>>>(scores, labels, B, nt, d_counts, dscores, part);
  TLP_LAUNCH_CHECK();
  mse_finalize<<<1, 1, 0, s>>>(part, kMseBlocks, nt, d_counts, loss_out, ctx->d_err);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

static size_t rank_ws_bytes(int G, int nt) {
  return (size_t)G * nt * (kCountSplit * sizeof(double) + (1 + 2 * kRankSplit) * sizeof(float)) + 64;
}

tlp_status rank_pair_counts(tlp_ctx* ctx, const float* labels, const int64_t* d_goff, int G,
                            int max_group, double* d_counts, cudaStream_t s) {
  const int nt = ctx->cfg.n_tasks;
  TLP_CUDA_TRY(ctx->ws_rank.ensure(rank_ws_bytes(G, nt)));
  double* part = ctx->ws_rank.as<double>();
  const size_t smem = (size_t)max_group * (2 * sizeof(float) + sizeof(int));
  cudaFuncSetAttribute(pair_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  TLP_LAUNCH_PDL(pair_count_kernel, dim3(G, nt, kCountSplit), kThreads, smem, s, labels, d_goff, nt, part);
  TLP_LAUNCH_CHECK();
  TLP_LAUNCH_PDL(sum_counts, 1, 32, 0, s, part, G, nt, d_counts);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

tlp_status rank_loss_grad(tlp_ctx* ctx, const float* scores, const float* labels,
                          const int64_t* d_goff, int G, int B, int max_group,
                          const double* d_counts, float* loss_out, float* dscores,
                          cudaStream_t s) {
  const int nt = ctx->cfg.n_tasks;
  TLP_CUDA_TRY(ctx->ws_rank.ensure(rank_ws_bytes(G, nt)));
  float* loss_part = reinterpret_cast<float*>(ctx->ws_rank.as<char>() + (size_t)G * nt * kCountSplit * sizeof(double));
  TLP_CUDA_TRY(cudaMemsetAsync(dscores, 0, (size_t)B * nt * sizeof(float), s));
  const size_t smem = (size_t)max_group * (4 * sizeof(float) + sizeof(int));
  static const char* env = getenv("TLP_RANK_SPLIT");
  if (env && env[0] == '0') {
    cudaFuncSetAttribute(rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rank_kernel<<<dim3(G, nt), kRankThreads, smem, s>>>(scores, labels, d_goff, nt, loss_part, dscores);
    TLP_LAUNCH_CHECK();
    TLP_LAUNCH_PDL(finalize_rank, (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv((int64_t)B * nt, 256), 1024)), 256, 0, s, 
        loss_part, G, nt, d_counts, dscores, B, loss_out, ctx->d_err);
    TLP_LAUNCH_CHECK();
    return TLP_OK;
  }
  // split: [nt][G][kRankSplit] loss and DCG partials, [nt][B] inverse discounts
  float* dcg_part = loss_part + (size_t)G * nt * kRankSplit;
  TLP_CUDA_TRY(ctx->ws_misc.ensure((size_t)nt * B * sizeof(float) + 256));
  float* iD = ctx->ws_misc.as<float>();
  const size_t smem1 = (size_t)max_group * (2 * sizeof(float) + sizeof(int));
  cudaFuncSetAttribute(rank_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
  TLP_LAUNCH_PDL(rank_prep_kernel, dim3(G * kRankSplit, nt), kRankThreads, smem1, s, scores, labels, d_goff, nt, iD, dcg_part);
  TLP_LAUNCH_CHECK();
  cudaFuncSetAttribute(rank_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  TLP_LAUNCH_PDL(rank_pair_kernel, dim3(G * kRankSplit, nt), kRankThreads, smem, s, scores, labels, d_goff, nt, iD, dcg_part,
                                                                       loss_part, dscores);
  TLP_LAUNCH_CHECK();
  TLP_LAUNCH_PDL(finalize_rank, (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv((int64_t)B * nt, 256), 1024)), 256, 0, s, 
      loss_part, G * kRankSplit, nt, d_counts, dscores, B, loss_out, ctx->d_err);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}
