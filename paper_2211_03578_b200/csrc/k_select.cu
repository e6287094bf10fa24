// K8 per-task top-k ("screens out the top-k potential candidates ...
// according to the prediction score"; "the i-th largest value of the
// output score" -> R15 higher is better; R21 total order (score desc, index
// asc), -0 == +0, NaN is an error, short segments padded with (-1, -inf)).
//
// K11 label normalisation ("label = min_latency / latency, where
// min_latency refers to the minimum value among all tensor programs of a
// subgraph"; R22 the min is over the whole group; fp64 quotient -> RN fp32).
//
// Top-k is a chunked tournament: every chunk of <= 2048 entries of a segment is
// bitonic-sorted in shared memory by one CTA under the total order and its
// best k survive; survivors of a segment are chunked and sorted again until
// one chunk per segment remains.  The order is total, so the result is the
// unique correct answer regardless of chunking (bit-exact vs a full sort).
#include "tlp_internal.cuh"

#include <algorithm>

namespace {

constexpr int kChunk = 2048;
constexpr int kThreads = 1024;

struct WorkItem {
  int64_t start;   // first entry (row for round 0, candidate slot otherwise)
  int32_t count;   // entries in this chunk (<= kChunk)
  int32_t out;     // output slot (candidate block index) -> out * k
};

// a strictly better than b under R21 (invalid entries: idx < 0, always last)
__device__ __forceinline__ bool better(float sa, int64_t ia, float sb, int64_t ib) {
  if (ia < 0) return false;
  if (ib < 0) return true;
  if (sa > sb) return true;
  if (sa < sb) return false;
  return ia < ib;
}

__global__ void __launch_bounds__(kThreads) topk_chunk_kernel(
    const WorkItem* __restrict__ items, int round0, const float* __restrict__ scores, int stride,
    int head, int64_t base, const float* __restrict__ in_s, const int64_t* __restrict__ in_i,
    float* __restrict__ out_s, int64_t* __restrict__ out_i, int k, uint32_t* __restrict__ err) {
  __shared__ float ss[kChunk];
  __shared__ int64_t si[kChunk];
  const WorkItem it = items[blockIdx.x];
  // Thread = warp w, lane l holds elements e = 64 w + 2 l + b (b = 0, 1) in
  // registers during the bitonic sort below; every stage with half <= 32 pairs
  // elements of one warp (half 1: inside the thread; 2..32: partner lane
  // l ^ half / 2, by shuffles).
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const int e0 = 64 * w + 2 * ln;
  float rs[2];
  int64_t ri[2];
  auto warp_stages = [&](int size, int top) {
    for (int half = top; half >= 2; half >>= 1) {
      const int lm = half >> 1;
      const bool lower = (ln & lm) == 0;
      const bool up = (e0 & size) == 0;
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const float ps = __shfl_xor_sync(0xffffffffu, rs[b], lm);
        const int64_t pi = __shfl_xor_sync(0xffffffffu, ri[b], lm);
        // the lower element keeps the better (up) / worse (down) of the pair
        const bool take = lower == up ? better(ps, pi, rs[b], ri[b]) : better(rs[b], ri[b], ps, pi);
        if (take) { rs[b] = ps; ri[b] = pi; }
      }
    }
    {  // half = 1: both elements in this thread
      const bool up = (e0 & size) == 0;
      const bool swap = up ? better(rs[1], ri[1], rs[0], ri[0]) : better(rs[0], ri[0], rs[1], ri[1]);
      if (swap) {
        const float ts = rs[0]; rs[0] = rs[1]; rs[1] = ts;
        const int64_t ti = ri[0]; ri[0] = ri[1]; ri[1] = ti;
      }
    }
  };
  if (it.count <= 64 && !round0) {
    // a merge chunk of <= 64 survivors (later rounds): one warp, registers only
    if (w != 0) return;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int j = 2 * ln + b;
      rs[b] = j < it.count ? in_s[it.start + j] : -INFINITY;
      ri[b] = j < it.count ? in_i[it.start + j] : -1;
    }
    for (int size = 2; size <= 64; size <<= 1) warp_stages(size, size >> 1);
    for (int jb = 0; jb < k; jb += 32) {  // (uniform trip count: every lane shuffles)
      const int j = jb + ln;              // element j sits in lane j / 2, slot j % 2
      const int src = (j < 64 ? j : 0) >> 1;
      const float s0 = __shfl_sync(0xffffffffu, rs[0], src), s1 = __shfl_sync(0xffffffffu, rs[1], src);
      const int64_t i0 = __shfl_sync(0xffffffffu, ri[0], src), i1 = __shfl_sync(0xffffffffu, ri[1], src);
      const float sv = (j & 1) ? s1 : s0;
      const int64_t iv = (j & 1) ? i1 : i0;
      if (j >= k) continue;
      const int64_t o = (int64_t)it.out * k + j;
      if (j < 64 && iv >= 0) { out_s[o] = sv; out_i[o] = iv; }
      else { out_s[o] = -INFINITY; out_i[o] = -1; }
    }
    return;
  }
  for (int j = threadIdx.x; j < kChunk; j += blockDim.x) {
    float s = -INFINITY;
    int64_t id = -1;
    if (j < it.count) {
      if (round0) {
        const int64_t row = it.start + j;
        s = scores[row * stride + head];
        id = base + row;
        if (isnan(s)) atomicOr(err, DERR_NONFINITE);
      } else {
        s = in_s[it.start + j];
        id = in_i[it.start + j];
      }
    }
    ss[j] = s;
    si[j] = id;
  }
  __syncthreads();
  // bitonic sort, "better" first: the warp stages above for half <= 32, only
  // half >= 64 goes through shared memory (15 block barriers instead of 66).
  // Same network, same result.
  rs[0] = ss[e0]; rs[1] = ss[e0 + 1];
  ri[0] = si[e0]; ri[1] = si[e0 + 1];
  for (int size = 2; size <= 64; size <<= 1) warp_stages(size, size >> 1);
  for (int size = 128; size <= kChunk; size <<= 1) {
    ss[e0] = rs[0]; ss[e0 + 1] = rs[1]; si[e0] = ri[0]; si[e0 + 1] = ri[1];
    __syncthreads();
    for (int half = size >> 1; half >= 64; half >>= 1) {
      const int t = threadIdx.x;  // kChunk / 2 compare-exchanges
      const int i = 2 * half * (t / half) + (t % half);
      const int j = i + half;
      const bool up = ((i & size) == 0);
      const float a = ss[i], b = ss[j];
      const int64_t ai = si[i], bi = si[j];
      const bool swap = up ? better(b, bi, a, ai) : better(a, ai, b, bi);
      if (swap) { ss[i] = b; ss[j] = a; si[i] = bi; si[j] = ai; }
      __syncthreads();
    }
    rs[0] = ss[e0]; rs[1] = ss[e0 + 1]; ri[0] = si[e0]; ri[1] = si[e0 + 1];
    __syncthreads();  // the next size's stores follow every thread's reads
    warp_stages(size, 32);
  }
  ss[e0] = rs[0]; ss[e0 + 1] = rs[1]; si[e0] = ri[0]; si[e0 + 1] = ri[1];
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const int64_t o = (int64_t)it.out * k + j;
    if (j < kChunk && si[j] >= 0) { out_s[o] = ss[j]; out_i[o] = si[j]; }
    else { out_s[o] = -INFINITY; out_i[o] = -1; }
  }
}

__global__ void finalize_topk(const float* __restrict__ s, const int64_t* __restrict__ i,
                              const int32_t* __restrict__ slot, int k, float* __restrict__ val,
                              int64_t* __restrict__ idx, int T) {
  const int t = blockIdx.x;
  if (t >= T) return;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const int32_t sl = slot[t];
    if (sl < 0) { val[(int64_t)t * k + j] = -INFINITY; idx[(int64_t)t * k + j] = -1; }
    else { val[(int64_t)t * k + j] = s[(int64_t)sl * k + j]; idx[(int64_t)t * k + j] = i[(int64_t)sl * k + j]; }
  }
}

__global__ void label_kernel(const float* __restrict__ lat, const int64_t* __restrict__ goff,
                             float* __restrict__ out, uint32_t* __restrict__ err) {
  const int64_t lo = goff[blockIdx.x], hi = goff[blockIdx.x + 1];
  __shared__ float red[32];
  float m = INFINITY;
  for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) {
    const float v = lat[j];
    if (!(v > 0.f) || isinf(v)) atomicOr(err, DERR_NONFINITE);
    m = fminf(m, v);
  }
  for (int o = 16; o; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : INFINITY;
    for (int o = 16; o; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  const double mn = (double)red[0];
  for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x)
    out[j] = __double2float_rn(mn / (double)lat[j]);
}

}  // namespace

// Shared tournament driver.  Round 0 reads either the strided score column
// (cand_s == nullptr) or (score, index) candidate pairs laid out contiguously
// per segment; every later round reads the survivors of the previous one.
static tlp_status topk_rounds(tlp_ctx* ctx, const float* scores, int stride, int head,
                              const float* cand_s, const int64_t* cand_i,
                              const std::vector<int64_t>& seg_lo, const std::vector<int64_t>& seg_hi,
                              int k, int64_t base, int64_t* idx_out, float* val_out,
                              cudaStream_t s) {
  const int T = (int)seg_lo.size();
  if (k <= 0 || k > kChunk / 2) {
    ctx->last_error = "tlp_topk: k must be in [1, 1024]";
    return TLP_ERR_ARG;
  }
  std::vector<WorkItem> items;
  std::vector<int32_t> seg_first(T), seg_n(T);
  for (int t = 0; t < T; ++t) {
    seg_first[t] = (int32_t)items.size();
    for (int64_t a = seg_lo[t]; a < seg_hi[t]; a += kChunk)
      items.push_back({a, (int32_t)std::min<int64_t>(kChunk, seg_hi[t] - a), (int32_t)items.size()});
    seg_n[t] = (int32_t)items.size() - seg_first[t];
  }
  const size_t max_blocks = items.size() + (size_t)T + 1;
  const size_t need = max_blocks * (size_t)k * 2 * (sizeof(float) + sizeof(int64_t)) +
                      (max_blocks + T) * sizeof(WorkItem) * 2 + T * sizeof(int32_t) + 256;
  TLP_CUDA_TRY(ctx->ws_topk.ensure(need));
  char* p = ctx->ws_topk.as<char>();
  float* bs[2];
  int64_t* bi[2];
  bi[0] = reinterpret_cast<int64_t*>(p); p += max_blocks * k * sizeof(int64_t);
  bi[1] = reinterpret_cast<int64_t*>(p); p += max_blocks * k * sizeof(int64_t);
  bs[0] = reinterpret_cast<float*>(p); p += max_blocks * k * sizeof(float);
  bs[1] = reinterpret_cast<float*>(p); p += max_blocks * k * sizeof(float);
  WorkItem* d_items = reinterpret_cast<WorkItem*>(p); p += (max_blocks + T) * sizeof(WorkItem) * 2;
  int32_t* d_slot = reinterpret_cast<int32_t*>(p);

  const float* src_s = cand_s;
  const int64_t* src_i = cand_i;
  bool first = true;
  int cur = 0;
  std::vector<int32_t> final_slot(T, -1);
  for (;;) {
    if (!items.empty()) {
      TLP_CUDA_TRY(cudaMemcpyAsync(d_items, items.data(), items.size() * sizeof(WorkItem),
                                   cudaMemcpyHostToDevice, s));
      const int r0 = (first && cand_s == nullptr) ? 1 : 0;
      topk_chunk_kernel<<<(unsigned)items.size(), kThreads, 0, s>>>(
          d_items, r0, scores, stride, head, base, src_s, src_i, bs[cur], bi[cur], k, ctx->d_err);
      TLP_LAUNCH_CHECK();
    }
    first = false;
    bool done = true;
    for (int t = 0; t < T; ++t) done = done && seg_n[t] <= 1;
    if (done) {
      for (int t = 0; t < T; ++t) final_slot[t] = seg_n[t] == 1 ? seg_first[t] : -1;
      break;
    }
    // next round: survivors of segment t are blocks [seg_first, +seg_n) of bs[cur]
    std::vector<WorkItem> next;
    std::vector<int32_t> nfirst(T), nn(T);
    for (int t = 0; t < T; ++t) {
      nfirst[t] = (int32_t)next.size();
      const int64_t f0 = (int64_t)seg_first[t] * k;
      const int64_t total = (int64_t)seg_n[t] * k;
      for (int64_t a = 0; a < total; a += kChunk)
        next.push_back({f0 + a, (int32_t)std::min<int64_t>(kChunk, total - a), (int32_t)next.size()});
      nn[t] = (int32_t)next.size() - nfirst[t];
    }
    items.swap(next);
    seg_first.swap(nfirst);
    seg_n.swap(nn);
    src_s = bs[cur];
    src_i = bi[cur];
    cur ^= 1;
  }
  TLP_CUDA_TRY(cudaMemcpyAsync(d_slot, final_slot.data(), T * sizeof(int32_t),
                               cudaMemcpyHostToDevice, s));
  finalize_topk<<<T, 128, 0, s>>>(bs[cur], bi[cur], d_slot, k, val_out, idx_out, T);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

tlp_status topk_launch(tlp_ctx* ctx, const float* scores, int stride, int head,
                       const int64_t* task_off, int T, int k, int64_t base, int64_t* idx_out,
                       float* val_out, cudaStream_t s) {
  std::vector<int64_t> lo(T), hi(T);
  for (int t = 0; t < T; ++t) { lo[t] = task_off[t]; hi[t] = task_off[t + 1]; }
  return topk_rounds(ctx, scores, stride, head, nullptr, nullptr, lo, hi, k, base, idx_out,
                     val_out, s);
}

tlp_status topk_merge_launch(tlp_ctx* ctx, const float* cand_s, const int64_t* cand_i, int T,
                             int64_t per_seg, int k, int64_t* idx_out, float* val_out,
                             cudaStream_t s) {
  std::vector<int64_t> lo(T), hi(T);
  for (int t = 0; t < T; ++t) { lo[t] = t * per_seg; hi[t] = (t + 1) * per_seg; }
  return topk_rounds(ctx, nullptr, 0, 0, cand_s, cand_i, lo, hi, k, 0, idx_out, val_out, s);
}

tlp_status normalize_labels_launch(tlp_ctx* ctx, const float* lat, const int64_t* group_off,
                                   int G, float* out, cudaStream_t s) {
  if (G <= 0) return TLP_OK;
  TLP_CUDA_TRY(ctx->ws_misc.ensure((G + 1) * sizeof(int64_t)));
  TLP_CUDA_TRY(cudaMemcpyAsync(ctx->ws_misc.p, group_off, (G + 1) * sizeof(int64_t),
                               cudaMemcpyHostToDevice, s));
  label_kernel<<<G, 256, 0, s>>>(lat, ctx->ws_misc.as<int64_t>(), out, ctx->d_err);
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}
