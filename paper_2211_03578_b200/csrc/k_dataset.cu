// NEXT-2: dataset-side scans before training and the
// evaluation metric after it.
//
// tlp_dedup (§4.3; readings R39): duplicate classes of feature
// matrices within groups, their representative (lowest index), the class
// maximum label and the distinct count (duplicate rate = 1 - distinct / N).
//   1. hash_rows     one warp per sample: 64-bit hash of the row's bit pattern
//                    (coalesced 8-byte loads), mixed with the group id and a seed
//   2. table_insert  open addressing (linear probing, 2^p >= 2N slots): CAS the
//                    key, atomicMin the representative index
//   3. table_lookup  rep[i] = the slot's minimum index
//   4. verify_rows   one warp per non-representative: bitwise row compare with
//                    its representative; a mismatch is a hash collision and the
//                    host retries with a new seed (results never depend on it)
//   5. finish        keep / max label (int-ordered max of non-negative floats) /
//                    distinct count
// HBM-bound: each row is read twice (hash + verify of duplicates only).
//
// tlp_topk_score (§6.1; R40): per group the k best by (score desc,
// index asc) through the top-k kernels of k_select.cu, then one block per group
// for min latency overall / among the top k, and a single-block fp64 weighted
// sum in a fixed order.
#include "tlp_internal.cuh"

#include <algorithm>
#include <vector>

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

__global__ void hash_rows(const float* __restrict__ X, int64_t N, int row_len,
                          const int64_t* __restrict__ group_off, int G, uint64_t seed,
                          uint64_t* __restrict__ keys) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= N) return;
  uint64_t h = seed ^ (0x9e3779b97f4a7c15ull * (uint64_t)(lane + 1));
  if (((row_len & 1) == 0) && ((reinterpret_cast<uintptr_t>(X) & 7) == 0)) {
    // 8-byte loads (rows of an even number of floats are 8-byte aligned)
    const uint64_t* row = reinterpret_cast<const uint64_t*>(X + i * row_len);
    for (int w = lane; w < row_len / 2; w += 32) h = mix64(h ^ __ldg(row + w) ^ ((uint64_t)w * 0xd6e8feb86659fd93ull));
  } else {
    const uint32_t* row = reinterpret_cast<const uint32_t*>(X + i * row_len);
    for (int w = lane; w < row_len; w += 32)
      h = mix64(h ^ (((uint64_t)w << 32) | __ldg(row + w)));
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {  // fixed butterfly: every lane ends with the same value
    const uint64_t other = __shfl_xor_sync(0xffffffffu, h, o);
    h = (lane & o) ? mix64(other ^ (h * 0x2545f4914f6cdd1dull)) : mix64(h ^ (other * 0x2545f4914f6cdd1dull));
  }
  if (lane == 0) {
    int lo = 0, hi = G;  // group of i: group_off[g] <= i < group_off[g+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (group_off[mid] <= i) lo = mid; else hi = mid;
    }
    keys[i] = mix64(h ^ mix64((uint64_t)lo + seed)) | 1ull;  // 0 = empty slot
  }
}

__global__ void table_insert(const uint64_t* __restrict__ keys, int64_t N, uint64_t mask,
                             unsigned long long* __restrict__ tkey,
                             unsigned long long* __restrict__ trep) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const unsigned long long k = keys[i];
  uint64_t slot = k & mask;
  while (true) {
    const unsigned long long prev = atomicCAS(tkey + slot, 0ull, k);
    if (prev == 0ull || prev == k) {
      atomicMin(trep + slot, (unsigned long long)i);
      return;
    }
    slot = (slot + 1) & mask;
  }
}

__global__ void table_lookup(const uint64_t* __restrict__ keys, int64_t N, uint64_t mask,
                             const unsigned long long* __restrict__ tkey,
                             const unsigned long long* __restrict__ trep, int64_t* __restrict__ rep) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const unsigned long long k = keys[i];
  uint64_t slot = k & mask;
  while (tkey[slot] != k) slot = (slot + 1) & mask;
  rep[i] = (int64_t)trep[slot];
}

__global__ void verify_rows(const float* __restrict__ X, int64_t N, int row_len,
                            const int64_t* __restrict__ rep, unsigned int* __restrict__ collisions) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= N) return;
  const int64_t r = rep[i];
  if (r == i) return;
  const uint32_t* a = reinterpret_cast<const uint32_t*>(X + i * row_len);
  const uint32_t* b = reinterpret_cast<const uint32_t*>(X + r * row_len);
  bool diff = false;
  for (int w = lane; w < row_len; w += 32) diff |= __ldg(a + w) != __ldg(b + w);
  if (__any_sync(0xffffffffu, diff) && lane == 0) atomicAdd(collisions, 1u);
}

// labels >= 0 and finite: their int bit patterns order like the values
__global__ void label_max(const float* __restrict__ labels, const int64_t* __restrict__ rep,
                          int64_t N, int* __restrict__ acc, uint32_t* __restrict__ err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const float y = labels[i];
  if (!(y >= 0.f) || !isfinite(y)) {
    atomicOr(err, DERR_NONFINITE);
    return;
  }
  atomicMax(acc + rep[i], __float_as_int(y));
}

__global__ void finish(const int64_t* __restrict__ rep, int64_t N, const int* __restrict__ acc,
                       int32_t* __restrict__ keep, float* __restrict__ label_out,
                       unsigned long long* __restrict__ distinct) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool k = i < N && rep[i] == i;
  if (i < N) {
    keep[i] = k ? 1 : 0;
    if (label_out) label_out[i] = __int_as_float(acc[rep[i]]);
  }
  const unsigned int b = __ballot_sync(0xffffffffu, k);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(distinct, (unsigned long long)__popc(b));
}

// ---- top-k score: one block per group
__global__ void topk_score_groups(const float* __restrict__ latency, const int64_t* __restrict__ goff,
                                  const int64_t* __restrict__ idx, int k,
                                  double* __restrict__ best_true, double* __restrict__ best_pred) {
  const int g = blockIdx.x;
  const int64_t lo = goff[g], hi = goff[g + 1];
  __shared__ float red[256];
  float m = INFINITY;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) m = fminf(m, latency[i]);
  red[threadIdx.x] = m;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fminf(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    float p = INFINITY;
    for (int r = 0; r < k; ++r) {
      const int64_t j = idx[(int64_t)g * k + r];
      if (j >= 0) p = fminf(p, latency[j]);
    }
    best_true[g] = hi > lo ? (double)red[0] : 0.0;
    best_pred[g] = hi > lo ? (double)p : 0.0;
  }
}

__global__ void topk_score_sum(const double* __restrict__ best_true, const double* __restrict__ best_pred,
                               const double* __restrict__ w, int G, double* __restrict__ out) {
  __shared__ double rn[256], rd[256];
  double n = 0.0, d = 0.0;
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    n += best_true[g] * w[g];
    d += best_pred[g] * w[g];
  }
  rn[threadIdx.x] = n;
  rd[threadIdx.x] = d;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) {
      rn[threadIdx.x] += rn[threadIdx.x + o];
      rd[threadIdx.x] += rd[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = rd[0] > 0.0 ? rn[0] / rd[0] : 0.0;
}

tlp_status fail_msg(tlp_ctx* ctx, tlp_status st, const char* m) {
  ctx->last_error = m;
  return st;
}

size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

extern "C" tlp_status tlp_dedup(tlp_ctx* ctx, const float* feats, int64_t N, int32_t row_len,
                                const int64_t* group_off, int32_t G, const float* labels,
                                int32_t* keep_out, float* label_out, int64_t* n_distinct_out,
                                void* stream) {
  if (!ctx) return TLP_ERR_ARG;
  if (N < 0 || row_len < 1 || G < 1 || !group_off || !n_distinct_out || (N > 0 && (!feats || !keep_out)) ||
      (label_out && !labels))
    return fail_msg(ctx, TLP_ERR_ARG, "tlp_dedup: bad arguments");
  if (group_off[0] != 0 || group_off[G] != N)
    return fail_msg(ctx, TLP_ERR_SHAPE, "tlp_dedup: group_off must run from 0 to N");
  for (int g = 0; g < G; ++g)
    if (group_off[g + 1] < group_off[g]) return fail_msg(ctx, TLP_ERR_SHAPE, "tlp_dedup: group_off decreasing");
  *n_distinct_out = 0;
  if (N == 0) return TLP_OK;
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint64_t cap = 16;
  while (cap < 2 * (uint64_t)N) cap <<= 1;
  const size_t sz_goff = a256((G + 1) * sizeof(int64_t)), sz_keys = a256(N * sizeof(uint64_t));
  const size_t sz_tab = a256(cap * sizeof(unsigned long long)), sz_rep = a256(N * sizeof(int64_t));
  const size_t sz_acc = a256(N * sizeof(int)), sz_cnt = 256;
  TLP_CUDA_TRY(ctx->ws_misc.ensure(sz_goff + sz_keys + 2 * sz_tab + sz_rep + sz_acc + sz_cnt));
  char* p = ctx->ws_misc.as<char>();
  int64_t* d_goff = reinterpret_cast<int64_t*>(p); p += sz_goff;
  uint64_t* keys = reinterpret_cast<uint64_t*>(p); p += sz_keys;
  unsigned long long* tkey = reinterpret_cast<unsigned long long*>(p); p += sz_tab;
  unsigned long long* trep = reinterpret_cast<unsigned long long*>(p); p += sz_tab;
  int64_t* rep = reinterpret_cast<int64_t*>(p); p += sz_rep;
  int* acc = reinterpret_cast<int*>(p); p += sz_acc;
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(p);  // [0] collisions, [1] distinct
  TLP_CUDA_TRY(cudaMemcpyAsync(d_goff, group_off, (G + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  const unsigned wb = (unsigned)cdiv(N * 32, 256), tb = (unsigned)cdiv(N, 256);
  bool ok = false;
  for (int attempt = 0; attempt < 4 && !ok; ++attempt) {
    const uint64_t seed = 0x5851f42d4c957f2dull * (uint64_t)(attempt + 1);
    TLP_CUDA_TRY(cudaMemsetAsync(tkey, 0, cap * sizeof(unsigned long long), s));
    TLP_CUDA_TRY(cudaMemsetAsync(trep, 0xff, cap * sizeof(unsigned long long), s));
    TLP_CUDA_TRY(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), s));
    hash_rows<<<wb, 256, 0, s>>>(feats, N, row_len, d_goff, G, seed, keys);
    TLP_LAUNCH_CHECK();
    table_insert<<<tb, 256, 0, s>>>(keys, N, cap - 1, tkey, trep);
    TLP_LAUNCH_CHECK();
    table_lookup<<<tb, 256, 0, s>>>(keys, N, cap - 1, tkey, trep, rep);
    TLP_LAUNCH_CHECK();
    verify_rows<<<wb, 256, 0, s>>>(feats, N, row_len, rep, reinterpret_cast<unsigned int*>(cnt));
    TLP_LAUNCH_CHECK();
    if (labels) {
      TLP_CUDA_TRY(cudaMemsetAsync(acc, 0, N * sizeof(int), s));
      label_max<<<tb, 256, 0, s>>>(labels, rep, N, acc, ctx->d_err);
      TLP_LAUNCH_CHECK();
    }
    finish<<<tb, 256, 0, s>>>(rep, N, acc, keep_out, labels ? label_out : nullptr, cnt + 1);
    TLP_LAUNCH_CHECK();
    unsigned long long hc[2] = {0, 0};  // [0] collisions (low 32 bits), [1] distinct
    TLP_CUDA_TRY(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
    TLP_CUDA_TRY(cudaStreamSynchronize(s));
    ok = (hc[0] & 0xffffffffull) == 0;  // a collision invalidates the pass: re-hash
    *n_distinct_out = (int64_t)hc[1];
  }
  if (!ok) return fail_msg(ctx, TLP_ERR_STATE, "tlp_dedup: persistent 64-bit hash collisions");
  return TLP_OK;
}

extern "C" tlp_status tlp_topk_score(tlp_ctx* ctx, const float* scores, int32_t score_stride,
                                     int32_t head, const float* latency, const int64_t* group_off,
                                     const double* weight, int32_t G, int32_t k, double* out,
                                     void* stream) {
  if (!ctx) return TLP_ERR_ARG;
  if (!scores || !latency || !group_off || !weight || !out || G < 1 || k < 1 || k > 1024 ||
      score_stride < 1 || head < 0 || head >= score_stride)
    return fail_msg(ctx, TLP_ERR_ARG, "tlp_topk_score: bad arguments");
  for (int g = 0; g < G; ++g)
    if (group_off[g + 1] < group_off[g] || group_off[0] < 0)
      return fail_msg(ctx, TLP_ERR_SHAPE, "tlp_topk_score: group_off must be non-decreasing");
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t sz_idx = a256((size_t)G * k * sizeof(int64_t)), sz_val = a256((size_t)G * k * sizeof(float));
  const size_t sz_g = a256((G + 1) * sizeof(int64_t)), sz_d = a256(G * sizeof(double));
  TLP_CUDA_TRY(ctx->ws_merge.ensure(sz_idx + sz_val + sz_g + 3 * sz_d + 256));
  char* p = ctx->ws_merge.as<char>();
  int64_t* idx = reinterpret_cast<int64_t*>(p); p += sz_idx;
  float* val = reinterpret_cast<float*>(p); p += sz_val;
  int64_t* d_goff = reinterpret_cast<int64_t*>(p); p += sz_g;
  double* bt = reinterpret_cast<double*>(p); p += sz_d;
  double* bp = reinterpret_cast<double*>(p); p += sz_d;
  double* w = reinterpret_cast<double*>(p); p += sz_d;
  double* d_out = reinterpret_cast<double*>(p);
  tlp_status st = topk_launch(ctx, scores, score_stride, head, group_off, G, k, 0, idx, val, s);
  if (st != TLP_OK) return st;
  TLP_CUDA_TRY(cudaMemcpyAsync(d_goff, group_off, (G + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  TLP_CUDA_TRY(cudaMemcpyAsync(w, weight, G * sizeof(double), cudaMemcpyHostToDevice, s));
  topk_score_groups<<<G, 256, 0, s>>>(latency, d_goff, idx, k, bt, bp);
  TLP_LAUNCH_CHECK();
  topk_score_sum<<<1, 256, 0, s>>>(bt, bp, w, G, d_out);
  TLP_LAUNCH_CHECK();
  TLP_CUDA_TRY(cudaMemcpyAsync(out, d_out, sizeof(double), cudaMemcpyDeviceToHost, s));
  TLP_CUDA_TRY(cudaStreamSynchronize(s));
  return TLP_OK;
}
