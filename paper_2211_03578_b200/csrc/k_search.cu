// NEXT-1: the synthetic Ansor-style tuning round on the device.
//
// P:558 (§6.3): "Ansor will first generate some initial tensor programs for a
// subgraph according to predefined rules.  Then use the cost model to pick out
// potential tensor programs.  Use these potential tensor programs to generate
// more tensor programs through the genetic algorithm and use the cost model
// again to prune the poor performers.  This step will iterate multiple times."
// about 10,000 sequences per subgraph per round are featurised and
// scored.  The genetic operators, the random numbers and the pruning are the
// readings R44-R48 of DESIGN.md.
//
// Device layout: a candidate is a row of G uint8 domain indices ("genes");
// rows are grouped by subgraph.  Every random decision is a pure function of a
// Philox4x64-10 counter (candidate, subgraph, round/iter, stream/block), so the
// kernels need no state and any thread order gives the same result.  Integer
// decisions use only integer arithmetic on the 64-bit words (umulhi for a
// uniform index, a 53-bit threshold compare for a coin).
//
// Kernels:
//   ga_init_kernel        thread per candidate: uniform genes (R45)
//   ga_evolve_kernel      thread per child: rank-roulette parents, one-point
//                         crossover at a primitive boundary, +-1 mutation (R46/R47)
//   ga_materialize_kernel warp per candidate: skeleton copy + knob values ->
//                         the packed abstract-primitive batch tlp_encode reads
//   ga_dedup_kernel       CTA per subgraph: shared-memory open-addressing table
//                         of gene rows, lowest index of each class kept (R48)
//   ga_gather_kernel / ga_combine_kernel  survivors <- top-k order; pool =
//                         survivors ++ children
// The round (tlp_ga_round) chains them with encode_rows / score_launch /
// topk_launch on one stream; no host round trip inside a round.
#include "tlp_internal.cuh"

#include <algorithm>
#include <cmath>

namespace {

constexpr int kMaxGenes = 64;
constexpr uint64_t kKey1 = 0x544C50ull;
constexpr uint32_t kStreamInit = 1, kStreamSel = 2, kStreamMut = 3;
constexpr int kMaxPool = 16384;

struct Philox4 { uint64_t w[4]; };

// Philox4x64-10 (Salmon et al., SC'11); the same generator as numpy's Philox.
__device__ __forceinline__ Philox4 philox(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                          uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B97F4A7C15ull; k1 += 0xBB67AE8584CAA73Bull; }
    const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0), lo0 = 0xD2E7470EE14C6C93ull * c0;
    const uint64_t hi1 = __umul64hi(0xCA5A826395121157ull, c2), lo1 = 0xCA5A826395121157ull * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return Philox4{{c0, c1, c2, c3}};
}

// R44 counter layout: (c, s, round << 16 | iter, stream << 32 | block)
__device__ __forceinline__ Philox4 ga_block(uint64_t seed, int64_t c, int s, int rnd, int it,
                                            uint32_t stream, int block) {
  return philox((uint64_t)c, (uint64_t)s, ((uint64_t)(uint32_t)rnd << 16) | (uint32_t)it,
                ((uint64_t)stream << 32) | (uint32_t)block, seed, kKey1);
}

__device__ __forceinline__ uint64_t uniform_index(uint64_t w, uint64_t n) { return __umul64hi(w, n); }

__global__ void ga_init_kernel(const int64_t* __restrict__ knob_off, const int64_t* __restrict__ dom_off,
                               int S, int n, int G, int id_base, uint64_t seed, int rnd,
                               uint8_t* __restrict__ genes) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= (int64_t)S * n) return;
  const int s = (int)(row / n);
  const int64_t c = row - (int64_t)s * n;
  const int64_t k0 = knob_off[s];
  const int K = (int)(knob_off[s + 1] - k0);
  uint8_t* out = genes + row * G;
  for (int b = 0; b * 4 < G; ++b) {
    Philox4 r{};
    if (b * 4 < K) r = ga_block(seed, c, id_base + s, rnd, 0, kStreamInit, b);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = b * 4 + q;
      if (j >= G) break;
      uint8_t v = 0;
      if (j < K) v = (uint8_t)uniform_index(r.w[q], (uint64_t)(dom_off[k0 + j + 1] - dom_off[k0 + j]));
      out[j] = v;
    }
  }
}

// C(r) = sum_{q <= r} (n - q); smallest r with C(r) > u (binary search on a
// monotone integer sequence: the same r as the oracle's linear scan)
__device__ __forceinline__ int select_rank(uint64_t u, int64_t n) {
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const uint64_t C = (uint64_t)((mid + 1) * n - mid * (mid + 1) / 2);
    if (C > u) hi = mid; else lo = mid + 1;
  }
  return (int)lo;
}

__global__ void ga_evolve_kernel(const int64_t* __restrict__ knob_off, const int64_t* __restrict__ dom_off,
                                 const int32_t* __restrict__ knob_grp, int S, int G, int id_base,
                                 const uint8_t* __restrict__ pop, const float* __restrict__ pop_scores,
                                 int n_pop, int n_child, uint64_t th_cross, uint64_t th_mut,
                                 uint64_t seed, int rnd, int it, uint8_t* __restrict__ child) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= (int64_t)S * n_child) return;
  const int s = (int)(row / n_child);
  const int64_t c = row - (int64_t)s * n_child;
  const int64_t k0 = knob_off[s];
  const int K = (int)(knob_off[s + 1] - k0);
  // n_eff = finite-score prefix of the rank-ordered survivors (duplicates are -inf)
  const float* sc = pop_scores + (int64_t)s * n_pop;
  int lo = 0, hi = n_pop;  // first index with score == -inf
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sc[mid] == -INFINITY) hi = mid; else lo = mid + 1;
  }
  const int64_t n_eff = lo > 0 ? lo : 1;
  const uint64_t F = (uint64_t)(n_eff * (n_eff + 1) / 2);
  const Philox4 sel = ga_block(seed, c, id_base + s, rnd, it, kStreamSel, 0);
  const int ra = select_rank(uniform_index(sel.w[0], F), n_eff);
  const int rb = select_rank(uniform_index(sel.w[1], F), n_eff);
  const uint8_t* A = pop + ((int64_t)s * n_pop + ra) * G;
  const uint8_t* B = pop + ((int64_t)s * n_pop + rb) * G;
  uint8_t g[kMaxGenes];
#pragma unroll
  for (int j = 0; j < kMaxGenes; ++j) g[j] = j < G ? A[j] : 0;
  const int n_groups = K > 0 ? knob_grp[k0 + K - 1] + 1 : 0;
  if (n_groups >= 2 && (sel.w[2] >> 11) < th_cross) {
    const int cut = 1 + (int)uniform_index(sel.w[3], (uint64_t)(n_groups - 1));
    for (int j = 0; j < K; ++j)
      if (knob_grp[k0 + j] >= cut) g[j] = B[j];
  }
  if (th_mut > 0) {
    for (int b = 0; b * 4 < K; ++b) {
      const Philox4 m = ga_block(seed, c, id_base + s, rnd, it, kStreamMut, b);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = b * 4 + q;
        if (j >= K) break;
        const int D = (int)(dom_off[k0 + j + 1] - dom_off[k0 + j]);
        const uint64_t w = m.w[q];
        if (D >= 2 && (w >> 11) < th_mut) {
          int v = g[j];
          if (w & 1) v = v + 1 < D ? v + 1 : v - 1;
          else v = v > 0 ? v - 1 : v + 1;
          g[j] = (uint8_t)v;
        }
      }
    }
  }
  uint8_t* out = child + row * G;
  for (int j = 0; j < G; ++j) out[j] = g[j];
}

struct TmplView {
  const int64_t* seq_off;   // [S+1]
  const uint8_t* prim_type;
  const int64_t* arg_off;   // [P+1]
  const uint8_t* arg_kind;
  const double* arg_num;
  const int32_t* arg_name;
};

// warp per candidate row (s = row / n): candidate c of subgraph s occupies
// primitives [n * Ptmpl_before_s + c * P_s, +P_s) and the same for arguments
__global__ void ga_materialize_kernel(TmplView t, const int64_t* __restrict__ knob_off,
                                      const int64_t* __restrict__ knob_arg,
                                      const int64_t* __restrict__ dom_off,
                                      const double* __restrict__ dom_num,
                                      const int32_t* __restrict__ dom_name, int S, int64_t n, int G,
                                      const uint8_t* __restrict__ genes, int64_t* __restrict__ seq_off,
                                      uint8_t* __restrict__ prim_type, int64_t* __restrict__ arg_off,
                                      uint8_t* __restrict__ arg_kind, double* __restrict__ arg_num,
                                      int32_t* __restrict__ arg_name) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t N = (int64_t)S * n;
  if (row >= N) return;
  const int s = (int)(row / n);
  const int64_t c = row - (int64_t)s * n;
  const int64_t tp0 = t.seq_off[s], tp1 = t.seq_off[s + 1];
  const int64_t ta0 = t.arg_off[tp0], ta1 = t.arg_off[tp1];
  const int64_t Ps = tp1 - tp0, As = ta1 - ta0;
  const int64_t pb = n * tp0 + c * Ps;  // first primitive of this candidate
  const int64_t ab = n * ta0 + c * As;  // first argument
  if (lane == 0) {
    seq_off[row] = pb;
    if (row == N - 1) {
      seq_off[N] = n * t.seq_off[S];
      arg_off[n * t.seq_off[S]] = n * t.arg_off[t.seq_off[S]];
    }
  }
  for (int64_t p = lane; p < Ps; p += 32) {
    prim_type[pb + p] = t.prim_type[tp0 + p];
    arg_off[pb + p] = ab + (t.arg_off[tp0 + p] - ta0);
  }
  const int64_t k0 = knob_off[s];
  const int K = (int)(knob_off[s + 1] - k0);
  const uint8_t* g = genes + row * G;
  for (int64_t a = lane; a < As; a += 32) {
    arg_kind[ab + a] = t.arg_kind[ta0 + a];
    arg_num[ab + a] = t.arg_num[ta0 + a];
    arg_name[ab + a] = t.arg_name[ta0 + a];
  }
  __syncwarp();
  for (int j = lane; j < K; j += 32) {
    const int64_t d = dom_off[k0 + j] + g[j];
    const int64_t a = ab + (knob_arg[k0 + j] - ta0);
    arg_num[a] = dom_num[d];
    arg_name[a] = dom_name[d];
  }
}

__device__ __forceinline__ uint32_t row_hash(const uint8_t* r, int G) {
  uint32_t h = 2166136261u;  // FNV-1a, then a final avalanche
  for (int j = 0; j < G; ++j) h = (h ^ r[j]) * 16777619u;
  h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
  return h;
}

__device__ __forceinline__ bool rows_equal(const uint8_t* a, const uint8_t* b, int G) {
  for (int j = 0; j < G; ++j)
    if (a[j] != b[j]) return false;
  return true;
}

// CTA per subgraph: the n rows of subgraph blockIdx.x.  Shared table of cap
// int32 slots (power of two >= 2n).  Phase 1 inserts every row (CAS into an
// empty slot, or atomicMin into the slot of an equal row); phase 2 re-probes
// and marks a row a duplicate iff its class slot holds a lower index.
__global__ void ga_dedup_kernel(const uint8_t* __restrict__ genes, int n, int G, int cap,
                                float* __restrict__ scores) {
  extern __shared__ int32_t table[];
  const int s = blockIdx.x;
  const uint8_t* base = genes + (int64_t)s * n * G;
  for (int i = threadIdx.x; i < cap; i += blockDim.x) table[i] = -1;
  __syncthreads();
  const uint32_t mask = (uint32_t)cap - 1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint8_t* ri = base + (int64_t)i * G;
    uint32_t h = row_hash(ri, G) & mask;
    for (;;) {
      int cur = table[h];
      if (cur < 0) {
        cur = atomicCAS(&table[h], -1, i);
        if (cur < 0) break;  // inserted
      }
      if (rows_equal(base + (int64_t)cur * G, ri, G)) { atomicMin(&table[h], i); break; }
      h = (h + 1) & mask;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint8_t* ri = base + (int64_t)i * G;
    uint32_t h = row_hash(ri, G) & mask;
    for (;;) {
      const int cur = table[h];
      if (rows_equal(base + (int64_t)cur * G, ri, G)) {
        if (cur != i) scores[(int64_t)s * n + i] = -INFINITY;
        break;
      }
      h = (h + 1) & mask;
    }
  }
}

// survivors[s, r] <- pool row idx[s, r] (global pool row; -1 = pad)
__global__ void ga_gather_kernel(int S, int n_pop, int G, const int64_t* __restrict__ idx,
                                 const float* __restrict__ val, const uint8_t* __restrict__ pool,
                                 uint8_t* __restrict__ out, float* __restrict__ out_scores) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= (int64_t)S * n_pop) return;
  const int64_t src = idx[row];
  uint8_t* o = out + row * G;
  if (src < 0) {
    for (int j = 0; j < G; ++j) o[j] = 0;
    out_scores[row] = -INFINITY;
    return;
  }
  const uint8_t* in = pool + src * G;
  for (int j = 0; j < G; ++j) o[j] = in[j];
  out_scores[row] = val[row];
}

// pool[s] = survivors[s] (n_pop rows) ++ children[s] (n_child rows), with the
// children's scores taken from column `head` of the [*, stride] score array
__global__ void ga_combine_kernel(int S, int n_pop, int n_child, int G, const uint8_t* __restrict__ surv,
                                  const float* __restrict__ surv_scores, const uint8_t* __restrict__ ch,
                                  const float* __restrict__ ch_scores, int stride, int head,
                                  uint8_t* __restrict__ pool, float* __restrict__ pool_scores) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int n_pool = n_pop + n_child;
  if (row >= (int64_t)S * n_pool) return;
  const int s = (int)(row / n_pool);
  const int r = (int)(row - (int64_t)s * n_pool);
  const uint8_t* in;
  float sc;
  if (r < n_pop) {
    in = surv + ((int64_t)s * n_pop + r) * G;
    sc = surv_scores[(int64_t)s * n_pop + r];
  } else {
    const int64_t cr = (int64_t)s * n_child + (r - n_pop);
    in = ch + cr * G;
    sc = ch_scores[cr * stride + head];
  }
  uint8_t* o = pool + row * G;
  for (int j = 0; j < G; ++j) o[j] = in[j];
  pool_scores[row] = sc;
}

__global__ void ga_column_kernel(int64_t N, const float* __restrict__ in, int stride, int head,
                                 float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) out[i] = in[i * stride + head];
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

// ctx-owned device copy of the search space (tlp_ga_set_space)
struct GaSpace {
  int S = 0, G = 0, U = 0, id_base = 0;
  int64_t Ptot = 0, Atot = 0;  // skeleton primitives / arguments over all subgraphs
  DevBuf mem;
  TmplView t{};
  const int64_t *knob_off = nullptr, *knob_arg = nullptr, *dom_off = nullptr, *str_off = nullptr;
  const int32_t* knob_grp = nullptr;
  const double* dom_num = nullptr;
  const int32_t* dom_name = nullptr;
  const uint8_t* str_blob = nullptr;
  // round workspaces
  DevBuf ws_genes, ws_batch, ws_feats, ws_scores;
};

void ga_free(tlp_ctx* ctx) {
  if (!ctx->ga) return;
  ctx->ga->mem.release();
  ctx->ga->ws_genes.release(); ctx->ga->ws_batch.release();
  ctx->ga->ws_feats.release(); ctx->ga->ws_scores.release();
  delete ctx->ga;
  ctx->ga = nullptr;
}

namespace {

tlp_status ga_fail(tlp_ctx* ctx, tlp_status st, const char* msg) {
  ctx->last_error = msg;
  return st;
}

tlp_status need_space(tlp_ctx* ctx) {
  if (!ctx->ga) return ga_fail(ctx, TLP_ERR_STATE, "tlp_ga_set_space first");
  return TLP_OK;
}

struct BatchPtrs {
  int64_t* seq_off; uint8_t* prim_type; int64_t* arg_off; uint8_t* arg_kind; double* arg_num;
  int32_t* arg_name;
};

tlp_status materialize_launch(tlp_ctx* ctx, const uint8_t* genes, int64_t n, const BatchPtrs& b,
                              cudaStream_t s) {
  GaSpace& g = *ctx->ga;
  const int64_t N = (int64_t)g.S * n;
  if (N == 0) return TLP_OK;
  const int threads = 256;
  ga_materialize_kernel<<<(unsigned)cdiv(N * 32, threads), threads, 0, s>>>(
      g.t, g.knob_off, g.knob_arg, g.dom_off, g.dom_num, g.dom_name, g.S, n, g.G, genes, b.seq_off,
      b.prim_type, b.arg_off, b.arg_kind, b.arg_num, b.arg_name);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

tlp_status dedup_launch(tlp_ctx* ctx, const uint8_t* genes, int n, float* scores, cudaStream_t s) {
  GaSpace& g = *ctx->ga;
  if (n <= 0) return TLP_OK;
  int cap = 64;
  while (cap < 2 * n) cap <<= 1;
  const size_t smem = (size_t)cap * sizeof(int32_t);
  if (smem > 48 * 1024)
    TLP_CUDA_TRY(cudaFuncSetAttribute(ga_dedup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  ga_dedup_kernel<<<g.S, 512, smem, s>>>(genes, n, g.G, cap, scores);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

uint64_t threshold53(double p) { return (uint64_t)(p * 9007199254740992.0); }

tlp_status evolve_launch(tlp_ctx* ctx, const uint8_t* pop, const float* pop_scores, int n_pop,
                         int n_child, double p_cross, double p_mut, uint64_t seed, int rnd, int it,
                         uint8_t* child, cudaStream_t s) {
  GaSpace& g = *ctx->ga;
  const int64_t N = (int64_t)g.S * n_child;
  if (N == 0) return TLP_OK;
  ga_evolve_kernel<<<(unsigned)cdiv(N, 128), 128, 0, s>>>(
      g.knob_off, g.dom_off, g.knob_grp, g.S, g.G, g.id_base, pop, pop_scores, n_pop, n_child,
      threshold53(p_cross), threshold53(p_mut), seed, rnd, it, child);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

tlp_status init_launch(tlp_ctx* ctx, int n, uint64_t seed, int rnd, uint8_t* genes, cudaStream_t s) {
  GaSpace& g = *ctx->ga;
  const int64_t N = (int64_t)g.S * n;
  if (N == 0 || g.G == 0) return TLP_OK;
  ga_init_kernel<<<(unsigned)cdiv(N, 128), 128, 0, s>>>(g.knob_off, g.dom_off, g.S, n, g.G, g.id_base,
                                                         seed, rnd, genes);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

}  // namespace

extern "C" {

tlp_status tlp_ga_set_space(tlp_ctx* ctx, const tlp_ga_space* h) {
  if (!ctx) return TLP_ERR_ARG;
  if (!h || h->S < 1 || h->id_base < 0 || !h->knob_off || !h->tmpl.seq_off || !h->tmpl.arg_off)
    return ga_fail(ctx, TLP_ERR_ARG, "tlp_ga_set_space: null pointer or S < 1");
  const tlp_seq_batch& t = h->tmpl;
  const int S = h->S;
  if (t.P < 0 || t.A < 0 || t.U < 0) return ga_fail(ctx, TLP_ERR_ARG, "tlp_ga_set_space: negative sizes");
  if ((t.P > 0 && !t.prim_type) || (t.A > 0 && (!t.arg_kind || !t.arg_num || !t.arg_name)) ||
      (t.U > 0 && (!t.str_off || !t.str_blob)))
    return ga_fail(ctx, TLP_ERR_ARG, "tlp_ga_set_space: null skeleton arrays");
  if (t.seq_off[0] != 0 || t.seq_off[S] != t.P || t.arg_off[0] != 0 || t.arg_off[t.P] != t.A)
    return ga_fail(ctx, TLP_ERR_SHAPE, "tlp_ga_set_space: skeleton offsets must span [0, P] / [0, A]");
  for (int s = 0; s < S; ++s)
    if (t.seq_off[s + 1] < t.seq_off[s] + 1)
      return ga_fail(ctx, TLP_ERR_SHAPE, "tlp_ga_set_space: every skeleton needs >= 1 primitive");
  for (int64_t p = 0; p < t.P; ++p)
    if (t.arg_off[p + 1] < t.arg_off[p]) return ga_fail(ctx, TLP_ERR_SHAPE, "tlp_ga_set_space: arg_off");
  const int64_t blob = t.U > 0 ? t.str_off[t.U] : 0;
  if (h->knob_off[0] != 0) return ga_fail(ctx, TLP_ERR_SHAPE, "tlp_ga_set_space: knob_off[0] != 0");
  int G = 0;
  for (int s = 0; s < S; ++s) {
    const int64_t k0 = h->knob_off[s], k1 = h->knob_off[s + 1];
    if (k1 < k0 || k1 - k0 > kMaxGenes)
      return ga_fail(ctx, TLP_ERR_SHAPE, "tlp_ga_set_space: 0..64 knobs per subgraph");
    G = std::max<int>(G, (int)(k1 - k0));
    const int64_t a0 = t.arg_off[t.seq_off[s]], a1 = t.arg_off[t.seq_off[s + 1]];
    for (int64_t k = k0; k < k1; ++k) {
      if (k > k0 ? (h->knob_grp[k] < h->knob_grp[k - 1] || h->knob_grp[k] > h->knob_grp[k - 1] + 1)
                 : h->knob_grp[k] != 0)
        return ga_fail(ctx, TLP_ERR_SHAPE, "tlp_ga_set_space: knob_grp must start at 0, steps <= 1");
      const int64_t a = h->knob_arg[k];
      if (a < a0 || a >= a1) return ga_fail(ctx, TLP_ERR_SHAPE, "tlp_ga_set_space: knob_arg outside its skeleton");
      const int64_t d0 = h->dom_off[k], d1 = h->dom_off[k + 1];
      if (d1 - d0 < 1 || d1 - d0 > 255) return ga_fail(ctx, TLP_ERR_SHAPE, "tlp_ga_set_space: domain size 1..255");
      for (int64_t d = d0; d < d1; ++d) {
        const bool name = h->dom_name[d] >= 0;
        if (name != (t.arg_kind[a] == 1) || (name && h->dom_name[d] >= t.U) ||
            (!name && !std::isfinite(h->dom_num[d])))
          return ga_fail(ctx, TLP_ERR_SHAPE, "tlp_ga_set_space: domain value kind / index / finiteness");
      }
    }
  }
  const int64_t K = h->knob_off[S];
  if (K < 1) return ga_fail(ctx, TLP_ERR_SHAPE, "tlp_ga_set_space: the space needs >= 1 knob");
  if (h->dom_off[0] != 0) return ga_fail(ctx, TLP_ERR_SHAPE, "tlp_ga_set_space: dom_off[0] != 0");
  const int64_t D = h->dom_off[K];
  cudaSetDevice(ctx->device);
  if (!ctx->ga) ctx->ga = new GaSpace();
  GaSpace& g = *ctx->ga;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + std::max<size_t>(bytes, 1)); return r; };
  const size_t o_seq = take(8 * (S + 1)), o_pt = take(t.P), o_ao = take(8 * (t.P + 1)),
               o_ak = take(t.A), o_an = take(8 * t.A), o_am = take(4 * t.A), o_ko = take(8 * (S + 1)),
               o_ka = take(8 * K), o_kg = take(4 * K), o_do = take(8 * (K + 1)), o_dn = take(8 * D),
               o_dm = take(4 * D), o_so = take(8 * (t.U + 1)), o_sb = take(blob);
  TLP_CUDA_TRY(g.mem.ensure(o));
  uint8_t* b = g.mem.as<uint8_t>();
  auto put = [&](size_t off, const void* src, size_t bytes) -> cudaError_t {
    return bytes ? cudaMemcpy(b + off, src, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
  };
  TLP_CUDA_TRY(put(o_seq, t.seq_off, 8 * (S + 1)));
  TLP_CUDA_TRY(put(o_pt, t.prim_type, t.P));
  TLP_CUDA_TRY(put(o_ao, t.arg_off, 8 * (t.P + 1)));
  TLP_CUDA_TRY(put(o_ak, t.arg_kind, t.A));
  TLP_CUDA_TRY(put(o_an, t.arg_num, 8 * t.A));
  TLP_CUDA_TRY(put(o_am, t.arg_name, 4 * t.A));
  TLP_CUDA_TRY(put(o_ko, h->knob_off, 8 * (S + 1)));
  TLP_CUDA_TRY(put(o_ka, h->knob_arg, 8 * K));
  TLP_CUDA_TRY(put(o_kg, h->knob_grp, 4 * K));
  TLP_CUDA_TRY(put(o_do, h->dom_off, 8 * (K + 1)));
  TLP_CUDA_TRY(put(o_dn, h->dom_num, 8 * D));
  TLP_CUDA_TRY(put(o_dm, h->dom_name, 4 * D));
  if (t.U > 0) {
    TLP_CUDA_TRY(put(o_so, t.str_off, 8 * (t.U + 1)));
    TLP_CUDA_TRY(put(o_sb, t.str_blob, blob));
  }
  g.S = S; g.G = G; g.U = t.U; g.Ptot = t.P; g.Atot = t.A; g.id_base = h->id_base;
  g.t = TmplView{reinterpret_cast<const int64_t*>(b + o_seq), b + o_pt,
                 reinterpret_cast<const int64_t*>(b + o_ao), b + o_ak,
                 reinterpret_cast<const double*>(b + o_an), reinterpret_cast<const int32_t*>(b + o_am)};
  g.knob_off = reinterpret_cast<const int64_t*>(b + o_ko);
  g.knob_arg = reinterpret_cast<const int64_t*>(b + o_ka);
  g.knob_grp = reinterpret_cast<const int32_t*>(b + o_kg);
  g.dom_off = reinterpret_cast<const int64_t*>(b + o_do);
  g.dom_num = reinterpret_cast<const double*>(b + o_dn);
  g.dom_name = reinterpret_cast<const int32_t*>(b + o_dm);
  g.str_off = reinterpret_cast<const int64_t*>(b + o_so);
  g.str_blob = b + o_sb;
  return TLP_OK;
}

int32_t tlp_ga_num_genes(const tlp_ctx* ctx) { return ctx && ctx->ga ? ctx->ga->G : 0; }

tlp_status tlp_ga_batch_size(tlp_ctx* ctx, int64_t n, int64_t* P_out, int64_t* A_out) {
  if (!ctx) return TLP_ERR_ARG;
  if (tlp_status st = need_space(ctx)) return st;
  if (n < 0 || !P_out || !A_out) return ga_fail(ctx, TLP_ERR_ARG, "tlp_ga_batch_size: bad args");
  *P_out = n * ctx->ga->Ptot;
  *A_out = n * ctx->ga->Atot;
  return TLP_OK;
}

tlp_status tlp_ga_init(tlp_ctx* ctx, int32_t n, uint64_t seed, int32_t round, uint8_t* genes_out,
                       void* stream) {
  if (!ctx) return TLP_ERR_ARG;
  if (tlp_status st = need_space(ctx)) return st;
  if (n < 0 || round < 0 || (n > 0 && !genes_out)) return ga_fail(ctx, TLP_ERR_ARG, "tlp_ga_init: bad args");
  cudaSetDevice(ctx->device);
  return init_launch(ctx, n, seed, round, genes_out, reinterpret_cast<cudaStream_t>(stream));
}

tlp_status tlp_ga_evolve(tlp_ctx* ctx, const uint8_t* pop, const float* pop_scores, int32_t n_pop,
                         int32_t n_child, double p_cross, double p_mut, uint64_t seed, int32_t round,
                         int32_t iter, uint8_t* child_out, void* stream) {
  if (!ctx) return TLP_ERR_ARG;
  if (tlp_status st = need_space(ctx)) return st;
  if (n_pop < 1 || n_child < 0 || !pop || !pop_scores || (n_child > 0 && !child_out) || round < 0 ||
      iter < 1 || iter >= (1 << 16) || !(p_cross >= 0.0 && p_cross <= 1.0) ||
      !(p_mut >= 0.0 && p_mut <= 1.0))
    return ga_fail(ctx, TLP_ERR_ARG, "tlp_ga_evolve: bad args");
  cudaSetDevice(ctx->device);
  return evolve_launch(ctx, pop, pop_scores, n_pop, n_child, p_cross, p_mut, seed, round, iter,
                       child_out, reinterpret_cast<cudaStream_t>(stream));
}

tlp_status tlp_ga_materialize(tlp_ctx* ctx, const uint8_t* genes, int64_t n, int64_t* seq_off,
                              uint8_t* prim_type, int64_t* arg_off, uint8_t* arg_kind,
                              double* arg_num, int32_t* arg_name, void* stream) {
  if (!ctx) return TLP_ERR_ARG;
  if (tlp_status st = need_space(ctx)) return st;
  if (n < 0 || (n > 0 && (!genes || !seq_off || !prim_type || !arg_off || !arg_kind || !arg_num ||
                          !arg_name)))
    return ga_fail(ctx, TLP_ERR_ARG, "tlp_ga_materialize: bad args");
  cudaSetDevice(ctx->device);
  return materialize_launch(ctx, genes, n, BatchPtrs{seq_off, prim_type, arg_off, arg_kind, arg_num, arg_name},
                            reinterpret_cast<cudaStream_t>(stream));
}

tlp_status tlp_ga_drop_duplicates(tlp_ctx* ctx, const uint8_t* genes, int32_t n, float* scores,
                                  void* stream) {
  if (!ctx) return TLP_ERR_ARG;
  if (tlp_status st = need_space(ctx)) return st;
  if (n < 0 || n > kMaxPool || (n > 0 && (!genes || !scores)))
    return ga_fail(ctx, TLP_ERR_ARG, "tlp_ga_drop_duplicates: bad args (n <= 16384)");
  cudaSetDevice(ctx->device);
  return dedup_launch(ctx, genes, n, scores, reinterpret_cast<cudaStream_t>(stream));
}

tlp_status tlp_ga_round(tlp_ctx* ctx, int32_t n_pop, int32_t n_child, int32_t iters, double p_cross,
                        double p_mut, uint64_t seed, int32_t round, int32_t head, uint8_t* genes_out,
                        float* scores_out, void* stream) {
  if (!ctx) return TLP_ERR_ARG;
  if (tlp_status st = need_space(ctx)) return st;
  const tlp_config& c = ctx->cfg;
  if (n_pop < 1 || n_pop > 1024 || n_child < 1 || n_pop + n_child > kMaxPool || iters < 0 ||
      iters >= (1 << 16) || round < 0 || head < 0 || head >= c.n_tasks || !genes_out || !scores_out ||
      !(p_cross >= 0.0 && p_cross <= 1.0) || !(p_mut >= 0.0 && p_mut <= 1.0))
    return ga_fail(ctx, TLP_ERR_ARG, "tlp_ga_round: bad args");
  if (!ctx->have_scales) return ga_fail(ctx, TLP_ERR_STATE, "tlp_set_norm_scales first");
  if (!ctx->have_params) return ga_fail(ctx, TLP_ERR_STATE, "tlp_set_params first");
  if (!score_supported(c))
    return ga_fail(ctx, TLP_ERR_UNSUPPORTED, "bf16 scoring needs the paper shape");
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GaSpace& g = *ctx->ga;
  const int S = g.S, G = g.G;
  const int n_pool = n_pop + n_child;
  const int64_t Npool = (int64_t)S * n_pool;

  // workspaces: gene buffers (pool, survivors, children), the materialised
  // batch of up to Npool candidates, its features and scores
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + std::max<size_t>(bytes, 1)); return r; };
  const size_t o_pool = take((size_t)Npool * G), o_surv = take((size_t)S * n_pop * G),
               o_child = take((size_t)S * n_child * G);
  TLP_CUDA_TRY(g.ws_genes.ensure(o));
  uint8_t* pool = g.ws_genes.as<uint8_t>() + o_pool;
  uint8_t* surv = g.ws_genes.as<uint8_t>() + o_surv;
  uint8_t* child = g.ws_genes.as<uint8_t>() + o_child;
  o = 0;
  const size_t b_seq = take(8 * (Npool + 1)), b_pt = take(n_pool * g.Ptot), b_ao = take(8 * (n_pool * g.Ptot + 1)),
               b_ak = take(n_pool * g.Atot), b_an = take(8 * n_pool * g.Atot), b_am = take(4 * n_pool * g.Atot);
  TLP_CUDA_TRY(g.ws_batch.ensure(o));
  uint8_t* bb = g.ws_batch.as<uint8_t>();
  BatchPtrs bp{reinterpret_cast<int64_t*>(bb + b_seq), bb + b_pt, reinterpret_cast<int64_t*>(bb + b_ao),
               bb + b_ak, reinterpret_cast<double*>(bb + b_an), reinterpret_cast<int32_t*>(bb + b_am)};
  TLP_CUDA_TRY(g.ws_feats.ensure(sizeof(float) * (size_t)Npool * c.L * c.E));
  float* feats = g.ws_feats.as<float>();
  o = 0;
  const size_t s_all = take(sizeof(float) * (size_t)Npool * c.n_tasks), s_pool = take(sizeof(float) * Npool),
               s_surv = take(sizeof(float) * (size_t)S * n_pop),
               s_idx = take(sizeof(int64_t) * (size_t)S * n_pop), s_val = take(sizeof(float) * (size_t)S * n_pop);
  TLP_CUDA_TRY(g.ws_scores.ensure(o));
  uint8_t* sb = g.ws_scores.as<uint8_t>();
  float* sc_all = reinterpret_cast<float*>(sb + s_all);
  float* sc_pool = reinterpret_cast<float*>(sb + s_pool);
  float* sc_surv = reinterpret_cast<float*>(sb + s_surv);
  int64_t* tk_idx = reinterpret_cast<int64_t*>(sb + s_idx);
  float* tk_val = reinterpret_cast<float*>(sb + s_val);

  tlp_seq_batch batch{};
  batch.seq_off = bp.seq_off; batch.prim_type = bp.prim_type; batch.arg_off = bp.arg_off;
  batch.arg_kind = bp.arg_kind; batch.arg_num = bp.arg_num; batch.arg_name = bp.arg_name;
  batch.str_blob = g.str_blob; batch.str_off = g.str_off;
  batch.U = g.U;
  std::vector<int64_t> seg_off(S + 1);
  for (int i = 0; i <= S; ++i) seg_off[i] = (int64_t)i * n_pool;

  // score the S * n materialised candidates of `genes` into sc_all
  auto score_genes = [&](const uint8_t* genes, int64_t n) -> tlp_status {
    batch.P = n * g.Ptot;
    batch.A = n * g.Atot;
    tlp_status st = materialize_launch(ctx, genes, n, bp, s);
    if (st != TLP_OK) return st;
    st = encode_rows(ctx, &batch, (int64_t)S * n, feats, s);
    if (st != TLP_OK) return st;
    return score_launch(ctx, feats, (int64_t)S * n, sc_all, s);
  };
  auto prune = [&]() -> tlp_status {  // pool -> survivors (rank order)
    tlp_status st = dedup_launch(ctx, pool, n_pool, sc_pool, s);
    if (st != TLP_OK) return st;
    st = topk_launch(ctx, sc_pool, 1, 0, seg_off.data(), S, n_pop, 0, tk_idx, tk_val, s);
    if (st != TLP_OK) return st;
    ga_gather_kernel<<<(unsigned)cdiv((int64_t)S * n_pop, 128), 128, 0, s>>>(S, n_pop, G, tk_idx, tk_val,
                                                                             pool, surv, sc_surv);
    TLP_LAUNCH_CHECK();
    return TLP_OK;
  };

  // the batch string table is the space's: resolve its tokens once per round
  batch.P = 0; batch.A = 0;
  tlp_status st = encode_resolve(ctx, &batch, s);
  if (st != TLP_OK) return st;
  st = init_launch(ctx, n_pool, seed, round, pool, s);
  if (st != TLP_OK) return st;
  st = score_genes(pool, n_pool);
  if (st != TLP_OK) return st;
  ga_column_kernel<<<(unsigned)cdiv(Npool, 256), 256, 0, s>>>(Npool, sc_all, c.n_tasks, head, sc_pool);
  TLP_LAUNCH_CHECK();
  st = prune();
  if (st != TLP_OK) return st;
  for (int it = 1; it <= iters; ++it) {
    st = evolve_launch(ctx, surv, sc_surv, n_pop, n_child, p_cross, p_mut, seed, round, it, child, s);
    if (st != TLP_OK) return st;
    st = score_genes(child, n_child);
    if (st != TLP_OK) return st;
    ga_combine_kernel<<<(unsigned)cdiv(Npool, 128), 128, 0, s>>>(S, n_pop, n_child, G, surv, sc_surv, child,
                                                                 sc_all, c.n_tasks, head, pool, sc_pool);
    TLP_LAUNCH_CHECK();
    st = prune();
    if (st != TLP_OK) return st;
  }
  TLP_CUDA_TRY(cudaMemcpyAsync(genes_out, surv, (size_t)S * n_pop * G, cudaMemcpyDeviceToDevice, s));
  TLP_CUDA_TRY(cudaMemcpyAsync(scores_out, sc_surv, sizeof(float) * (size_t)S * n_pop,
                               cudaMemcpyDeviceToDevice, s));
  return TLP_OK;
}

}  // extern "C"
