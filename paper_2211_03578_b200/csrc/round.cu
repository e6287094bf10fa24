// tlp_search_round: one search round of the auto-tuner from
// HOST memory -- encode -> score -> per-task top-k -- with the host->device
// copy of the packed batch pipelined against the kernels.
//
// The batch is copied into a device image with the SAME element offsets as the
// host arrays, so a chunk of candidates [c0, c1) is just a shifted view
// (seq_off + c0; every other offset is absolute) and the encode / score
// launchers run on it unchanged.  Chunk c+1 is copied on ctx->copy_stream while
// chunk c is encoded and scored on the caller's stream; events order the two.
// No arithmetic of the method happens here: orchestration only.
#include "tlp_internal.cuh"

#include <algorithm>
#include <vector>

namespace {

tlp_status round_fail(tlp_ctx* ctx, tlp_status st, const char* msg) {
  ctx->last_error = msg;
  return st;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t seq_off, prim_type, arg_off, arg_kind, arg_num, arg_name, str_off, str_blob, total;
};

Layout layout_of(int64_t N, int64_t P, int64_t A, int64_t U, int64_t blob) {
  Layout l{};
  size_t o = 0;
  l.seq_off = o;   o = align_up(o + sizeof(int64_t) * (size_t)(N + 1));
  l.prim_type = o; o = align_up(o + (size_t)P);
  l.arg_off = o;   o = align_up(o + sizeof(int64_t) * (size_t)(P + 1));
  l.arg_kind = o;  o = align_up(o + (size_t)A);
  l.arg_num = o;   o = align_up(o + sizeof(double) * (size_t)A);
  l.arg_name = o;  o = align_up(o + sizeof(int32_t) * (size_t)A);
  l.str_off = o;   o = align_up(o + sizeof(int64_t) * (size_t)(U + 1));
  l.str_blob = o;  o = align_up(o + (size_t)std::max<int64_t>(blob, 1));
  l.total = o;
  return l;
}

template <class T>
cudaError_t copy_range(uint8_t* dev_base, size_t off, const T* host, int64_t lo, int64_t hi,
                       cudaStream_t s) {
  if (hi <= lo) return cudaSuccess;
  return cudaMemcpyAsync(dev_base + off + sizeof(T) * (size_t)lo, host + lo,
                         sizeof(T) * (size_t)(hi - lo), cudaMemcpyHostToDevice, s);
}

}  // namespace

tlp_status tlp_search_round(tlp_ctx* ctx, const tlp_seq_batch* h, int64_t N,
                            const int64_t* task_off, int32_t T, int32_t k, int32_t head,
                            int64_t shard_base, int32_t chunks, int64_t* idx_out, float* val_out,
                            void* stream) {
  if (!ctx) return TLP_ERR_ARG;
  if (!h || !task_off || !idx_out || !val_out || N < 0 || T < 1 || k < 1)
    return round_fail(ctx, TLP_ERR_ARG, "tlp_search_round: null pointer or bad size");
  if (chunks < 1 || chunks > TLP_MAX_ROUND_CHUNKS)
    return round_fail(ctx, TLP_ERR_ARG, "tlp_search_round: chunks must be in [1, 64]");
  const tlp_config& c = ctx->cfg;
  if (head < 0 || head >= c.n_tasks) return round_fail(ctx, TLP_ERR_ARG, "tlp_search_round: bad head");
  if (!ctx->have_scales) return round_fail(ctx, TLP_ERR_STATE, "tlp_set_norm_scales first");
  if (!ctx->have_params) return round_fail(ctx, TLP_ERR_STATE, "tlp_set_params first");
  if (!score_supported(c))
    return round_fail(ctx, TLP_ERR_UNSUPPORTED, "bf16 scoring needs the paper shape");
  if (task_off[0] < 0 || task_off[T] > N)
    return round_fail(ctx, TLP_ERR_SHAPE, "tlp_search_round: task_off outside [0, N]");
  if (N > 0 && (!h->seq_off || !h->prim_type || !h->arg_off))
    return round_fail(ctx, TLP_ERR_ARG, "tlp_search_round: null batch arrays");
  if (h->A > 0 && (!h->arg_kind || !h->arg_num || !h->arg_name))
    return round_fail(ctx, TLP_ERR_ARG, "tlp_search_round: null argument arrays");
  if (h->U > 0 && (!h->str_blob || !h->str_off))
    return round_fail(ctx, TLP_ERR_ARG, "tlp_search_round: null string table");
  if (h->P < 0 || h->A < 0 || h->U < 0) return round_fail(ctx, TLP_ERR_ARG, "negative batch size");
  const int64_t blob = h->U > 0 ? h->str_off[h->U] : 0;
  if (blob < 0 || (h->U > 0 && h->str_off[0] != 0))
    return round_fail(ctx, TLP_ERR_SHAPE, "tlp_search_round: bad str_off");

  // chunk boundaries (multiples of 5 candidates = one tensor-core tile).  The
  // first two chunks are a quarter and a half of the others, so the kernels
  // start after a short copy (pipeline fill); only while the event array allows.
  const int64_t cs = std::max<int64_t>(5, cdiv(cdiv(std::max<int64_t>(N, 1), chunks), 5) * 5);
  std::vector<int64_t> bnd(1, 0);
  {
    const bool ramp = chunks + 2 <= TLP_MAX_ROUND_CHUNKS && cs >= 20;
    const int64_t first[2] = {ramp ? cdiv(cs / 4, 5) * 5 : cs, ramp ? cdiv(cs / 2, 5) * 5 : cs};
    for (int i = 0; bnd.back() < N; ++i) bnd.push_back(std::min<int64_t>(N, bnd.back() + (i < 2 ? first[i] : cs)));
  }
  const int nch = (int)bnd.size() - 1;
  // validate the host offsets the chunk copies rely on: seq_off in full
  // (non-decreasing within [0, P]), arg_off at the chunk boundaries
  if (N > 0) {
    if (h->seq_off[0] < 0 || h->seq_off[N] > h->P)
      return round_fail(ctx, TLP_ERR_SHAPE, "tlp_search_round: seq_off outside [0, P]");
    for (int64_t n = 0; n < N; ++n)
      if (h->seq_off[n + 1] < h->seq_off[n])
        return round_fail(ctx, TLP_ERR_SHAPE, "tlp_search_round: seq_off must be non-decreasing");
    int64_t prev = 0;
    for (int ci = 0; ci <= nch; ++ci) {
      const int64_t a = h->arg_off[h->seq_off[bnd[ci]]];
      if (a < prev || a > h->A)
        return round_fail(ctx, TLP_ERR_SHAPE, "tlp_search_round: arg_off outside [0, A]");
      prev = a;
    }
  }

  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!ctx->copy_stream)
    TLP_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  for (int i = 0; i <= nch; ++i)
    if (!ctx->round_ev[i]) TLP_CUDA_TRY(cudaEventCreateWithFlags(&ctx->round_ev[i], cudaEventDisableTiming));

  const Layout L = layout_of(N, h->P, h->A, h->U, blob);
  TLP_CUDA_TRY(ctx->ws_round_in.ensure(L.total));
  TLP_CUDA_TRY(ctx->ws_round_feats.ensure(sizeof(float) * (size_t)cs * c.L * c.E));
  const size_t nsc = (size_t)std::max<int64_t>(N, 1) * c.n_tasks;
  TLP_CUDA_TRY(ctx->ws_round_scores.ensure(sizeof(float) * nsc + 256 +
                                           (size_t)T * k * (sizeof(int64_t) + sizeof(float)) + 256));
  uint8_t* dev = ctx->ws_round_in.as<uint8_t>();
  float* scores = ctx->ws_round_scores.as<float>();
  int64_t* d_idx = reinterpret_cast<int64_t*>(ctx->ws_round_scores.as<uint8_t>() + align_up(sizeof(float) * nsc));
  float* d_val = reinterpret_cast<float*>(d_idx + (size_t)T * k);
  float* feats = ctx->ws_round_feats.as<float>();

  tlp_seq_batch d{};
  d.seq_off = reinterpret_cast<const int64_t*>(dev + L.seq_off);
  d.prim_type = dev + L.prim_type;
  d.arg_off = reinterpret_cast<const int64_t*>(dev + L.arg_off);
  d.arg_kind = dev + L.arg_kind;
  d.arg_num = reinterpret_cast<const double*>(dev + L.arg_num);
  d.arg_name = reinterpret_cast<const int32_t*>(dev + L.arg_name);
  d.str_off = reinterpret_cast<const int64_t*>(dev + L.str_off);
  d.str_blob = dev + L.str_blob;
  d.P = h->P; d.A = h->A; d.U = h->U;

  // the copy stream may only overwrite the device image once `stream` is done
  // with the previous round
  cudaEvent_t ev_start = ctx->round_ev[nch];
  TLP_CUDA_TRY(cudaEventRecord(ev_start, s));
  TLP_CUDA_TRY(cudaStreamWaitEvent(ctx->copy_stream, ev_start, 0));
  cudaStream_t cs_ = ctx->copy_stream;
  if (h->U > 0) {
    TLP_CUDA_TRY(copy_range(dev, L.str_off, h->str_off, 0, (int64_t)h->U + 1, cs_));
    TLP_CUDA_TRY(copy_range(dev, L.str_blob, h->str_blob, 0, blob, cs_));
  }
  for (int ci = 0; ci < nch; ++ci) {
    const int64_t c0 = bnd[ci], c1 = bnd[ci + 1];
    const int64_t p0 = h->seq_off[c0], p1 = h->seq_off[c1];
    const int64_t a0 = h->arg_off[p0], a1 = h->arg_off[p1];
    TLP_CUDA_TRY(copy_range(dev, L.seq_off, h->seq_off, c0, c1 + 1, cs_));
    TLP_CUDA_TRY(copy_range(dev, L.prim_type, h->prim_type, p0, p1, cs_));
    TLP_CUDA_TRY(copy_range(dev, L.arg_off, h->arg_off, p0, p1 + 1, cs_));
    TLP_CUDA_TRY(copy_range(dev, L.arg_kind, h->arg_kind, a0, a1, cs_));
    TLP_CUDA_TRY(copy_range(dev, L.arg_num, h->arg_num, a0, a1, cs_));
    TLP_CUDA_TRY(copy_range(dev, L.arg_name, h->arg_name, a0, a1, cs_));
    TLP_CUDA_TRY(cudaEventRecord(ctx->round_ev[ci], cs_));
  }
  if (nch == 0 && h->U > 0) {  // nothing to score; keep the stream order anyway
    TLP_CUDA_TRY(cudaEventRecord(ctx->round_ev[0], cs_));
    TLP_CUDA_TRY(cudaStreamWaitEvent(s, ctx->round_ev[0], 0));
  }

  tlp_status st = TLP_OK;
  for (int ci = 0; ci < nch && st == TLP_OK; ++ci) {
    const int64_t c0 = bnd[ci], c1 = bnd[ci + 1];
    TLP_CUDA_TRY(cudaStreamWaitEvent(s, ctx->round_ev[ci], 0));
    if (ci == 0) st = encode_resolve(ctx, &d, s);
    if (st != TLP_OK) break;
    tlp_seq_batch v = d;
    v.seq_off = d.seq_off + c0;
    st = encode_rows(ctx, &v, c1 - c0, feats, s);
    if (st == TLP_OK) st = score_launch(ctx, feats, c1 - c0, scores + (size_t)c0 * c.n_tasks, s);
  }
  if (st != TLP_OK) return st;
  st = tlp_topk(ctx, scores, c.n_tasks, head, task_off, T, k, shard_base, d_idx, d_val, stream);
  if (st != TLP_OK) return st;
  TLP_CUDA_TRY(cudaMemcpyAsync(idx_out, d_idx, sizeof(int64_t) * (size_t)T * k, cudaMemcpyDeviceToHost, s));
  TLP_CUDA_TRY(cudaMemcpyAsync(val_out, d_val, sizeof(float) * (size_t)T * k, cudaMemcpyDeviceToHost, s));
  return TLP_OK;
}
