// The C ABI of libtlp.so (include/tlp.h): ctx lifetime, state, and the four
// hot-path calls (tlp_encode, tlp_score, tlp_train_step, tlp_topk) plus label
// normalisation.  Host-side validation and orchestration only; every step of
// the path runs in the kernels of k_*.cu.  NCCL (torch's pip copy, 2.28) is
// used for the two data-parallel exchanges of SURVEY §8(e): the gradient /
// pair-count allreduce of training and the top-k allgather of sharded scoring.
#include "tlp_internal.cuh"

#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstring>
#include <vector>

tlp_status topk_merge_launch(tlp_ctx* ctx, const float* cand_s, const int64_t* cand_i, int T,
                             int64_t per_seg, int k, int64_t* idx_out, float* val_out,
                             cudaStream_t s);

namespace {

thread_local std::string g_tls_error;

tlp_status fail(tlp_ctx* ctx, tlp_status st, const std::string& msg) {
  if (ctx) ctx->last_error = msg;
  else g_tls_error = msg;
  return st;
}

// after a call enqueued collectives on stream s: tlp_sync's bounded wait
tlp_status note_collective(tlp_ctx* ctx, cudaStream_t s) {
  if (!ctx->coll_ev) TLP_CUDA_TRY(cudaEventCreateWithFlags(&ctx->coll_ev, cudaEventDisableTiming));
  TLP_CUDA_TRY(cudaEventRecord(ctx->coll_ev, s));
  return TLP_OK;
}

// tear the communicator down after a timeout or an asynchronous NCCL error
// (SURVEY §5 failure detection): ncclCommAbort unblocks any kernels still
// waiting on peers; the ctx then runs without collectives until tlp_set_comm
tlp_status abort_comm(tlp_ctx* ctx, const std::string& why) {
  ncclCommAbort(reinterpret_cast<ncclComm_t>(ctx->comm));
  ctx->comm = nullptr;
  ctx->world = 1;
  return fail(ctx, TLP_ERR_NCCL, why + " (communicator aborted)");
}

double nccl_timeout_s() {
  const char* e = getenv("TLP_NCCL_TIMEOUT_S");
  const double v = e ? atof(e) : 300.0;
  return v > 0 ? v : 300.0;
}

ParamOffsets compute_offsets(const tlp_config& c) {
  ParamOffsets o{};
  int64_t p = 0;
  int64_t din = c.E;
  for (int i = 0; i < c.n_up; ++i) {
    o.up_W[i] = p; p += din * c.up_dims[i];
    o.up_b[i] = p; p += c.up_dims[i];
    din = c.up_dims[i];
  }
  const int64_t H = c.hidden;
  o.pos = -1;
  if (c.pos_enc) { o.pos = p; p += (int64_t)c.L * H; }  // R43, right after the upsample (R24)
  for (int l = 0; l < c.n_attn; ++l) {
    if (c.backbone == 1) {  // R49: Wih [H, 4H], bih, Whh [H, 4H], bhh
      o.Wih[l] = p; p += 4 * H * H; o.bih[l] = p; p += 4 * H;
      o.Whh[l] = p; p += 4 * H * H; o.bhh[l] = p; p += 4 * H;
      continue;
    }
    o.Wq[l] = p; p += H * H; o.bq[l] = p; p += H;
    o.Wk[l] = p; p += H * H; o.bk[l] = p; p += H;
    o.Wv[l] = p; p += H * H; o.bv[l] = p; p += H;
    o.Wo[l] = p; p += H * H; o.bo[l] = p; p += H;
  }
  for (int r = 0; r < c.n_res; ++r) {
    o.Wa[r] = p; p += H * H; o.a[r] = p; p += H;
    o.Wb[r] = p; p += H * H; o.b[r] = p; p += H;
  }
  for (int t = 0; t < c.n_tasks; ++t) {
    o.W1[t] = p; p += H * c.head_dim; o.c1[t] = p; p += c.head_dim;
    o.w2[t] = p; p += c.head_dim; o.c2[t] = p; p += 1;
  }
  o.total = p;
  return o;
}

std::string check_config(const tlp_config& c) {
  if (c.L < 1 || c.L > 32) return "L must be in [1, 32]";
  if (c.E < 2 || c.E > 64) return "E must be in [2, 64]";
  if (c.T < 1 || c.T >= c.E) return "T must be in [1, E)";
  if (c.n_up < 1 || c.n_up > TLP_MAX_UP) return "n_up must be in [1, 4]";
  if (c.loss != TLP_LOSS_LAMBDARANK && c.loss != TLP_LOSS_MSE) return "loss must be 0 (LambdaRank) or 1 (MSE)";
  if (c.attn_mask != 0 && c.attn_mask != 1) return "attn_mask must be 0 or 1";
  if (c.pos_enc != 0 && c.pos_enc != 1) return "pos_enc must be 0 or 1";
  if (c.backbone != 0 && c.backbone != 1) return "backbone must be 0 (attention) or 1 (LSTM)";
  if (c.backbone == 1 && c.attn_mask) return "attn_mask applies to the attention backbone only";
  if (c.hidden < 8 || c.hidden > 512) return "hidden must be in [8, 512]";
  if (c.up_dims[c.n_up - 1] != c.hidden) return "up_dims[n_up-1] must equal hidden";
  for (int i = 0; i < c.n_up; ++i)
    if (c.up_dims[i] < 1 || c.up_dims[i] > c.hidden) return "up_dims must be in [1, hidden]";
  if (c.attn_heads < 1 || c.hidden % c.attn_heads) return "hidden % attn_heads must be 0";
  const int dh = c.hidden / c.attn_heads;
  if (c.backbone == 0 && c.n_attn > 0 && dh != 8 && dh != 16 && dh != 32 && dh != 64) return "hidden/attn_heads must be 8/16/32/64";
  if (c.n_attn < 0 || c.n_attn > TLP_MAX_ATTN) return "n_attn must be in [0, 4]";
  if (c.n_res < 0 || c.n_res > TLP_MAX_RES) return "n_res must be in [0, 4]";
  if (c.head_dim < 1 || c.head_dim > c.hidden) return "head_dim must be in [1, hidden]";
  if (c.n_tasks < 1 || c.n_tasks > TLP_MAX_TASKS) return "n_tasks must be in [1, 8]";
  if (c.precision != TLP_PREC_FP32 && c.precision != TLP_PREC_BF16) return "bad precision";
  return "";
}

#define CHECK_CTX() \
  if (!ctx) return fail(nullptr, TLP_ERR_ARG, "null ctx")

}  // namespace

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("TLP_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

tlp_status dev_error_status(tlp_ctx* ctx) {
  uint32_t e = 0;
  TLP_CUDA_TRY(cudaMemcpy(&e, ctx->d_err, sizeof(e), cudaMemcpyDeviceToHost));
  if (!e) return TLP_OK;
  TLP_CUDA_TRY(cudaMemset(ctx->d_err, 0, sizeof(uint32_t)));
  if (e & DERR_EMPTY_SEQ) return fail(ctx, TLP_ERR_EMPTY_SEQ, "empty primitive sequence");
  if (e & DERR_UNKNOWN_TYPE) return fail(ctx, TLP_ERR_UNKNOWN_TYPE, "primitive type id >= T");
  if (e & DERR_NONFINITE) return fail(ctx, TLP_ERR_NONFINITE, "non-finite number or score");
  if (e & DERR_NAN_LOSS) return fail(ctx, TLP_ERR_NAN_LOSS, "NaN loss");
  return fail(ctx, TLP_ERR_STATE, "unknown device error");
}

// C-1 gradient bucket (declared in tlp_internal.cuh; called from simt_backward)
tlp_status grad_bucket_ready(tlp_ctx* ctx, int64_t lo, int64_t hi, cudaStream_t s) {
  static const char* env = getenv("TLP_GRAD_BUCKETS");
  static const bool on = !(env && env[0] == '0');
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(ctx->comm);
  if (!comm || !on || hi <= lo) return TLP_OK;
  if (!ctx->comm_stream) {
    TLP_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    for (cudaEvent_t& e : ctx->bucket_ev) TLP_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaEvent_t ev = ctx->bucket_ev[ctx->buckets_issued % 4];
  TLP_CUDA_TRY(cudaEventRecord(ev, s));
  TLP_CUDA_TRY(cudaStreamWaitEvent(ctx->comm_stream, ev, 0));
  if (ncclAllReduce(ctx->d_grads + lo, ctx->d_grads + lo, (size_t)(hi - lo), ncclFloat32, ncclSum, comm,
                    ctx->comm_stream) != ncclSuccess)
    return fail(ctx, TLP_ERR_NCCL, "gradient bucket allreduce failed");
  ++ctx->buckets_issued;
  return TLP_OK;
}

extern "C" {

void tlp_default_config(tlp_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->L = 25; c->E = 22; c->T = 11;
  c->hidden = 256;
  c->up_dims[0] = 128; c->up_dims[1] = 256; c->n_up = 2;  // R11
  c->attn_heads = 8; c->n_attn = 1; c->n_res = 2;
  c->head_dim = 128; c->n_tasks = 1;        // R13
  c->precision = TLP_PREC_BF16;
  c->lr = 1e-3f; c->beta1 = 0.9f; c->beta2 = 0.999f; c->eps = 1e-8f;  // R23
}

tlp_status tlp_create(const tlp_config* cfg, int device, tlp_ctx** out) {
  if (!cfg || !out) return fail(nullptr, TLP_ERR_ARG, "null argument");
  const std::string why = check_config(*cfg);
  if (!why.empty()) return fail(nullptr, TLP_ERR_SHAPE, why);
  if (cudaSetDevice(device) != cudaSuccess) return fail(nullptr, TLP_ERR_CUDA, "cudaSetDevice failed");
  tlp_ctx* ctx = new tlp_ctx();
  ctx->cfg = *cfg;
  ctx->device = device;
  ctx->off = compute_offsets(*cfg);
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  const size_t pb = (size_t)ctx->off.total * sizeof(float);
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_params, pb);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_grads, pb);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_m, pb);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_v, pb);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_scale, cfg->E * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_err, sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(ctx->d_err, 0, sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(ctx->d_grads, 0, pb);
  if (e == cudaSuccess) e = cudaMemset(ctx->d_m, 0, pb);
  if (e == cudaSuccess) e = cudaMemset(ctx->d_v, 0, pb);
  if (e != cudaSuccess) {
    g_tls_error = std::string("CUDA: ") + cudaGetErrorString(e);
    tlp_destroy(ctx);
    return TLP_ERR_CUDA;
  }
  *out = ctx;
  return TLP_OK;
}

void tlp_destroy(tlp_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->comm) ncclCommDestroy(reinterpret_cast<ncclComm_t>(ctx->comm));
  tc_free(ctx);
  ga_free(ctx);
  cudaFree(ctx->d_params); cudaFree(ctx->d_grads); cudaFree(ctx->d_m); cudaFree(ctx->d_v);
  cudaFree(ctx->d_scale); cudaFree(ctx->d_err);
  cudaFree(ctx->d_hkeys); cudaFree(ctx->d_hval); cudaFree(ctx->d_hstr);
  cudaFree(ctx->d_tblob); cudaFree(ctx->d_toff);
  for (DevBuf* b : {&ctx->ws_tokens, &ctx->ws_act, &ctx->ws_train, &ctx->ws_rank, &ctx->ws_topk,
                    &ctx->ws_misc, &ctx->ws_partial, &ctx->ws_merge, &ctx->ws_round_in,
                    &ctx->ws_round_feats, &ctx->ws_round_scores, &ctx->ws_bimg, &ctx->ws_wcat, &ctx->ws_hcat})
    b->release();
  for (cudaEvent_t& e : ctx->round_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  for (cudaEvent_t e : ctx->bucket_ev)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < tlp_ctx::kGoffRing; ++i) {
    if (ctx->goff_ev[i]) cudaEventDestroy(ctx->goff_ev[i]);
    if (ctx->goff_pinned[i]) cudaFreeHost(ctx->goff_pinned[i]);
  }
  delete ctx;
}

const char* tlp_last_error(const tlp_ctx* ctx) {
  return ctx ? ctx->last_error.c_str() : g_tls_error.c_str();
}

tlp_status tlp_set_token_table(tlp_ctx* ctx, const uint8_t* blob, const int64_t* off, int32_t n) {
  CHECK_CTX();
  if (n < 0 || (n > 0 && (!off || (!blob && off[n] > 0))) || n >= (1 << 24) - 2)
    return fail(ctx, TLP_ERR_ARG, "bad token table");
  cudaSetDevice(ctx->device);
  return build_token_table(ctx, blob, off, n);
}

tlp_status tlp_set_norm_scales(tlp_ctx* ctx, const float* scale) {
  CHECK_CTX();
  if (!scale) return fail(ctx, TLP_ERR_ARG, "null scale");
  for (int c = 0; c < ctx->cfg.E; ++c)
    if (!(scale[c] > 0.f) || std::isinf(scale[c])) return fail(ctx, TLP_ERR_ARG, "scales must be finite and > 0");
  cudaSetDevice(ctx->device);
  TLP_CUDA_TRY(cudaMemcpy(ctx->d_scale, scale, ctx->cfg.E * sizeof(float), cudaMemcpyHostToDevice));
  ctx->have_scales = true;
  return TLP_OK;
}

tlp_status tlp_fit_token_table(tlp_ctx* ctx, const tlp_seq_batch* in, int64_t N) {
  CHECK_CTX();
  if (!in || N < 0 || (N > 0 && (!in->seq_off || !in->arg_off))) return fail(ctx, TLP_ERR_ARG, "null input");
  if (in->A > 0 && (!in->arg_kind || !in->arg_name)) return fail(ctx, TLP_ERR_ARG, "null argument arrays");
  if (in->U > 0 && (!in->str_blob || !in->str_off)) return fail(ctx, TLP_ERR_ARG, "null string table");
  // R1: tokens from 2 in first-occurrence order of the name arguments of the
  // training stream (candidates, primitives, arguments in order)
  const int64_t a_end = N > 0 ? in->arg_off[in->seq_off[N]] : 0;
  const int64_t a_beg = N > 0 ? in->arg_off[in->seq_off[0]] : 0;
  std::vector<uint8_t> seen(in->U > 0 ? in->U : 1, 0);
  std::vector<int64_t> off(1, 0);
  std::vector<uint8_t> blob;
  for (int64_t a = a_beg; a < a_end; ++a) {
    if (!in->arg_kind[a]) continue;
    const int32_t u = in->arg_name[a];
    if (u < 0 || u >= in->U) return fail(ctx, TLP_ERR_ARG, "name index outside the string table");
    if (seen[u]) continue;
    seen[u] = 1;
    const uint8_t* b = reinterpret_cast<const uint8_t*>(in->str_blob) + in->str_off[u];
    blob.insert(blob.end(), b, b + (in->str_off[u + 1] - in->str_off[u]));
    off.push_back((int64_t)blob.size());
  }
  // equal strings under different string-table indices keep the first token
  // (build_token_table skips later duplicates)
  const int32_t n = (int32_t)(off.size() - 1);
  if (n >= (1 << 24) - 2) return fail(ctx, TLP_ERR_ARG, "token table exceeds 2^24 entries");
  cudaSetDevice(ctx->device);
  return build_token_table(ctx, blob.data(), off.data(), n);
}

tlp_status tlp_fit_norm_scales(tlp_ctx* ctx, const tlp_seq_batch* in, int64_t N, float* scale_out,
                               void* stream) {
  CHECK_CTX();
  if (!in || N < 0 || (N > 0 && (!in->seq_off || !in->prim_type || !in->arg_off)))
    return fail(ctx, TLP_ERR_ARG, "null input");
  if (in->A > 0 && (!in->arg_kind || !in->arg_num || !in->arg_name))
    return fail(ctx, TLP_ERR_ARG, "null argument arrays");
  if (in->U > 0 && (!in->str_blob || !in->str_off)) return fail(ctx, TLP_ERR_ARG, "null string table");
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  tlp_status st = fit_scales_launch(ctx, in, N, s);
  if (st != TLP_OK) return st;
  if (scale_out)
    TLP_CUDA_TRY(cudaMemcpyAsync(scale_out, ctx->d_scale, ctx->cfg.E * sizeof(float), cudaMemcpyDefault, s));
  return TLP_OK;
}

int64_t tlp_num_params(const tlp_ctx* ctx) { return ctx ? ctx->off.total : -1; }

tlp_status tlp_set_params(tlp_ctx* ctx, const float* flat, int64_t n) {
  CHECK_CTX();
  if (!flat || n != ctx->off.total) return fail(ctx, TLP_ERR_SHAPE, "parameter count mismatch");
  cudaSetDevice(ctx->device);
  const size_t pb = (size_t)n * sizeof(float);
  TLP_CUDA_TRY(cudaMemcpy(ctx->d_params, flat, pb, cudaMemcpyDefault));
  TLP_CUDA_TRY(cudaMemset(ctx->d_m, 0, pb));
  TLP_CUDA_TRY(cudaMemset(ctx->d_v, 0, pb));
  ctx->adam_t = 0;
  ctx->have_params = true;
  ctx->tc_dirty = true;
  return TLP_OK;
}

tlp_status tlp_get_params(tlp_ctx* ctx, float* flat, int64_t n) {
  CHECK_CTX();
  if (!flat || n != ctx->off.total) return fail(ctx, TLP_ERR_SHAPE, "parameter count mismatch");
  cudaSetDevice(ctx->device);
  TLP_CUDA_TRY(cudaDeviceSynchronize());
  TLP_CUDA_TRY(cudaMemcpy(flat, ctx->d_params, (size_t)n * sizeof(float), cudaMemcpyDefault));
  return TLP_OK;
}

tlp_status tlp_get_grads(tlp_ctx* ctx, float* flat, int64_t n) {
  CHECK_CTX();
  if (!flat || n != ctx->off.total) return fail(ctx, TLP_ERR_SHAPE, "parameter count mismatch");
  cudaSetDevice(ctx->device);
  TLP_CUDA_TRY(cudaDeviceSynchronize());
  TLP_CUDA_TRY(cudaMemcpy(flat, ctx->d_grads, (size_t)n * sizeof(float), cudaMemcpyDefault));
  return TLP_OK;
}

tlp_status tlp_get_train_scores(tlp_ctx* ctx, float* out, int64_t n) {
  CHECK_CTX();
  if (!ctx->train_scores || ctx->train_N < 0) return fail(ctx, TLP_ERR_STATE, "no training step yet");
  if (!out || n != ctx->train_N * ctx->cfg.n_tasks) return fail(ctx, TLP_ERR_SHAPE, "score count mismatch");
  cudaSetDevice(ctx->device);
  TLP_CUDA_TRY(cudaDeviceSynchronize());
  TLP_CUDA_TRY(cudaMemcpy(out, ctx->train_scores, (size_t)n * sizeof(float), cudaMemcpyDefault));
  return TLP_OK;
}

tlp_status tlp_get_unique_id(void* out) {
  if (!out) return fail(nullptr, TLP_ERR_ARG, "null id buffer");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return fail(nullptr, TLP_ERR_NCCL, "ncclGetUniqueId failed");
  std::memcpy(out, &id, sizeof(id));
  return TLP_OK;
}

tlp_status tlp_set_comm(tlp_ctx* ctx, const void* nccl_id, int rank, int world) {
  CHECK_CTX();
  if (world < 1 || rank < 0 || rank >= world) return fail(ctx, TLP_ERR_ARG, "bad rank/world");
  cudaSetDevice(ctx->device);
  if (ctx->comm) {
    ncclCommDestroy(reinterpret_cast<ncclComm_t>(ctx->comm));
    ctx->comm = nullptr;
  }
  ctx->rank = rank;
  ctx->world = world;
  // world 1 without an id: no communicator (the single-GPU path).  World 1 WITH
  // an id builds a 1-rank communicator, so the collective code paths (count and
  // gradient allreduce, top-k allgather + merge) run on one GPU (tests).
  if (world == 1 && !nccl_id) return TLP_OK;
  if (!nccl_id) return fail(ctx, TLP_ERR_ARG, "null nccl id");
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof(id));
  ncclComm_t comm;
  ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
  if (r != ncclSuccess) return fail(ctx, TLP_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  ctx->comm = comm;
  return TLP_OK;
}

tlp_status tlp_broadcast_state(tlp_ctx* ctx, int root, void* stream) {
  CHECK_CTX();
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(ctx->comm);
  if (!comm) return fail(ctx, TLP_ERR_STATE, "tlp_set_comm first");
  if (root < 0 || root >= ctx->world) return fail(ctx, TLP_ERR_ARG, "bad root rank");
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // header: what the root holds (sizes the receivers must allocate)
  int64_t hdr[6] = {ctx->have_params ? 1 : 0, ctx->have_scales ? 1 : 0, (int64_t)ctx->hcap,
                    (int64_t)ctx->tok_n, ctx->tok_bytes, ctx->adam_t};
  TLP_CUDA_TRY(ctx->ws_misc.ensure(64));
  int64_t* d_hdr = ctx->ws_misc.as<int64_t>();
  TLP_CUDA_TRY(cudaMemcpyAsync(d_hdr, hdr, sizeof(hdr), cudaMemcpyHostToDevice, s));
  auto bc = [&](void* buf, size_t count, ncclDataType_t t) {
    return count == 0 || ncclBroadcast(buf, buf, count, t, root, comm, s) == ncclSuccess;
  };
  if (!bc(d_hdr, 6, ncclInt64)) return fail(ctx, TLP_ERR_NCCL, "state header broadcast failed");
  TLP_CUDA_TRY(cudaMemcpyAsync(hdr, d_hdr, sizeof(hdr), cudaMemcpyDeviceToHost, s));
  TLP_CUDA_TRY(cudaStreamSynchronize(s));
  const bool params = hdr[0] != 0, scales = hdr[1] != 0;
  const uint32_t cap = (uint32_t)hdr[2];
  const int32_t n = (int32_t)hdr[3];
  const int64_t nbytes = hdr[4];
  // receivers: token-table arrays of the root's size (contents arrive below)
  if (ctx->rank != root) {
    cudaFree(ctx->d_hkeys); cudaFree(ctx->d_hval); cudaFree(ctx->d_hstr);
    cudaFree(ctx->d_tblob); cudaFree(ctx->d_toff);
    ctx->d_hkeys = nullptr; ctx->d_hval = nullptr; ctx->d_hstr = nullptr;
    ctx->d_tblob = nullptr; ctx->d_toff = nullptr;
    if (cap) {
      TLP_CUDA_TRY(cudaMalloc(&ctx->d_hkeys, cap * sizeof(uint64_t)));
      TLP_CUDA_TRY(cudaMalloc(&ctx->d_hval, cap * sizeof(int32_t)));
      TLP_CUDA_TRY(cudaMalloc(&ctx->d_hstr, cap * sizeof(int32_t)));
      TLP_CUDA_TRY(cudaMalloc(&ctx->d_tblob, nbytes > 0 ? nbytes : 1));
      TLP_CUDA_TRY(cudaMalloc(&ctx->d_toff, ((size_t)n + 1) * sizeof(int64_t)));
    }
    ctx->hcap = cap;
    ctx->tok_n = n;
    ctx->tok_bytes = nbytes;
  }
  const size_t np = (size_t)ctx->off.total;
  bool ok = ncclGroupStart() == ncclSuccess;
  if (params) ok = ok && bc(ctx->d_params, np, ncclFloat32) && bc(ctx->d_m, np, ncclFloat32) &&
                   bc(ctx->d_v, np, ncclFloat32);
  if (scales) ok = ok && bc(ctx->d_scale, ctx->cfg.E, ncclFloat32);
  if (cap) ok = ok && bc(ctx->d_hkeys, cap, ncclUint64) && bc(ctx->d_hval, cap, ncclInt32) &&
                bc(ctx->d_hstr, cap, ncclInt32) && bc(ctx->d_tblob, (size_t)nbytes, ncclUint8) &&
                bc(ctx->d_toff, (size_t)n + 1, ncclInt64);
  ok = (ncclGroupEnd() == ncclSuccess) && ok;
  if (!ok) return fail(ctx, TLP_ERR_NCCL, "state broadcast failed");
  tlp_status st = note_collective(ctx, s);
  if (st != TLP_OK) return st;
  if (params) {
    ctx->have_params = true;
    ctx->adam_t = hdr[5];
    ctx->tc_dirty = true;  // the bf16 weight images are re-packed from the new parameters
  }
  if (scales) ctx->have_scales = true;
  return TLP_OK;
}

tlp_status tlp_encode(tlp_ctx* ctx, const tlp_seq_batch* in, int64_t N, float* feats, void* stream) {
  CHECK_CTX();
  if (!in || N < 0 || (N > 0 && (!feats || !in->seq_off || !in->prim_type || !in->arg_off)))
    return fail(ctx, TLP_ERR_ARG, "null input");
  if (in->A > 0 && (!in->arg_kind || !in->arg_num || !in->arg_name))
    return fail(ctx, TLP_ERR_ARG, "null argument arrays");
  if (in->U > 0 && (!in->str_blob || !in->str_off)) return fail(ctx, TLP_ERR_ARG, "null string table");
  if (!ctx->have_scales) return fail(ctx, TLP_ERR_STATE, "tlp_set_norm_scales first");
  cudaSetDevice(ctx->device);
  return encode_launch(ctx, in, N, feats, reinterpret_cast<cudaStream_t>(stream));
}

tlp_status tlp_score(tlp_ctx* ctx, const float* feats, int64_t N, float* scores, void* stream) {
  CHECK_CTX();
  if (N < 0 || (N > 0 && (!feats || !scores))) return fail(ctx, TLP_ERR_ARG, "null buffer");
  if (!ctx->have_params) return fail(ctx, TLP_ERR_STATE, "tlp_set_params first");
  if (!score_supported(ctx->cfg))
    return fail(ctx, TLP_ERR_UNSUPPORTED,
                "bf16 tensor-core scoring needs the paper shape (E=22, L=25, hidden=256, "
                "up_dims={128,256}, 8 heads, head_dim=128); use TLP_PREC_FP32");
  if (N == 0) return TLP_OK;
  cudaSetDevice(ctx->device);
  return score_launch(ctx, feats, N, scores, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"

tlp_status score_launch(tlp_ctx* ctx, const float* feats, int64_t N, float* scores, cudaStream_t s) {
  if (ctx->cfg.precision == TLP_PREC_BF16 && tc_supported(ctx->cfg)) {
    if (ctx->tc_dirty) {
      tlp_status st = tc_prepare(ctx, s);
      if (st != TLP_OK) return st;
      ctx->tc_dirty = false;
    }
    return tc_forward(ctx, feats, N, scores, s);
  }
  return simt_forward(ctx, feats, N, scores, false, s);
}

extern "C" {

namespace {

tlp_status check_groups(tlp_ctx* ctx, const int64_t* group_off, int32_t B, int32_t G, int* max_group) {
  if (!group_off || G < 1 || B < 1) return fail(ctx, TLP_ERR_ARG, "bad groups");
  if (group_off[0] != 0 || group_off[G] != B) return fail(ctx, TLP_ERR_SHAPE, "group_off must span [0, B]");
  int64_t mx = 0;
  for (int g = 0; g < G; ++g) {
    const int64_t n = group_off[g + 1] - group_off[g];
    if (n < 0) return fail(ctx, TLP_ERR_SHAPE, "group_off must be non-decreasing");
    mx = std::max(mx, n);
  }
  if (mx > 8192) return fail(ctx, TLP_ERR_UNSUPPORTED, "groups larger than 8192 items");
  *max_group = (int)std::max<int64_t>(mx, 1);
  return TLP_OK;
}

// Upload a step's group offsets to the device copy `dst`.  The same layout as
// the last upload to the same buffer on the same stream (a fixed training batch
// shape) needs no copy; otherwise the offsets go through one slot of a pinned
// staging ring (its previous copy is waited for first), never a pageable copy.
tlp_status upload_goff(tlp_ctx* ctx, int64_t* dst, const int64_t* group_off, int32_t G, cudaStream_t s) {
  const size_t n = (size_t)G + 1;
  if (ctx->goff_dev == dst && ctx->goff_stream == s && ctx->goff_last.size() == n &&
      std::memcmp(ctx->goff_last.data(), group_off, n * sizeof(int64_t)) == 0)
    return TLP_OK;
  if (n > ctx->goff_pinned_cap) {
    for (int i = 0; i < tlp_ctx::kGoffRing; ++i) {
      if (ctx->goff_ev[i]) TLP_CUDA_TRY(cudaEventSynchronize(ctx->goff_ev[i]));
      if (ctx->goff_pinned[i]) cudaFreeHost(ctx->goff_pinned[i]);
      ctx->goff_pinned[i] = nullptr;
    }
    ctx->goff_pinned_cap = 0;
    const size_t cap = std::max<size_t>(n, 1024);
    for (int i = 0; i < tlp_ctx::kGoffRing; ++i) {
      TLP_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&ctx->goff_pinned[i]), cap * sizeof(int64_t),
                                 cudaHostAllocDefault));
      if (!ctx->goff_ev[i]) TLP_CUDA_TRY(cudaEventCreateWithFlags(&ctx->goff_ev[i], cudaEventDisableTiming));
    }
    ctx->goff_pinned_cap = cap;
  }
  const int slot = ctx->goff_slot;
  ctx->goff_slot = (slot + 1) % tlp_ctx::kGoffRing;
  TLP_CUDA_TRY(cudaEventSynchronize(ctx->goff_ev[slot]));  // its last copy has read it
  std::memcpy(ctx->goff_pinned[slot], group_off, n * sizeof(int64_t));
  TLP_CUDA_TRY(cudaMemcpyAsync(dst, ctx->goff_pinned[slot], n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  TLP_CUDA_TRY(cudaEventRecord(ctx->goff_ev[slot], s));
  ctx->goff_last.assign(group_off, group_off + n);
  ctx->goff_dev = dst;
  ctx->goff_stream = s;
  return TLP_OK;
}

struct TrainWs {
  int64_t* goff;
  double* counts;
  float* scores;
  float* dscores;
  float* loss;
};

tlp_status train_ws(tlp_ctx* ctx, int B, int G, TrainWs* w) {
  const int nt = ctx->cfg.n_tasks;
  const size_t b_goff = ((size_t)(G + 1) * sizeof(int64_t) + 255) / 256 * 256;
  const size_t b_cnt = 256;
  const size_t b_sc = ((size_t)B * nt * sizeof(float) + 255) / 256 * 256;
  const size_t had = ctx->ws_train.bytes;
  TLP_CUDA_TRY(ctx->ws_train.ensure(b_goff + b_cnt + 2 * b_sc + 256));
  if (ctx->ws_train.bytes != had) ctx->goff_dev = nullptr;  // reallocated: the uploaded offsets are gone
  char* p = ctx->ws_train.as<char>();
  w->goff = reinterpret_cast<int64_t*>(p); p += b_goff;
  w->counts = reinterpret_cast<double*>(p); p += b_cnt;
  w->scores = reinterpret_cast<float*>(p); p += b_sc;
  w->dscores = reinterpret_cast<float*>(p); p += b_sc;
  w->loss = reinterpret_cast<float*>(p);
  return TLP_OK;
}

tlp_status grads_impl(tlp_ctx* ctx, const float* feats, const float* labels,
                      const int64_t* group_off, int32_t B, int32_t G, float* loss_out,
                      cudaStream_t s) {
  if (!feats || !labels || !loss_out) return fail(ctx, TLP_ERR_ARG, "null buffer");
  if (!ctx->have_params) return fail(ctx, TLP_ERR_STATE, "tlp_set_params first");
  int max_group = 0;
  tlp_status st = check_groups(ctx, group_off, B, G, &max_group);
  if (st != TLP_OK) return st;
  cudaSetDevice(ctx->device);
  TrainWs w;
  if ((st = train_ws(ctx, B, G, &w)) != TLP_OK) return st;
  if ((st = upload_goff(ctx, w.goff, group_off, G, s)) != TLP_OK) return st;
  const int nt = ctx->cfg.n_tasks;
  // C-0: per-task loss denominators (labels only), summed over ranks: strict
  // pairs for LambdaRank (R16), present labels for MSE (R41).
  const bool mse = ctx->cfg.loss == TLP_LOSS_MSE;
  st = mse ? mse_counts(ctx, labels, B, w.counts, s)
           : rank_pair_counts(ctx, labels, w.goff, G, max_group, w.counts, s);
  if (st != TLP_OK) return st;
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(ctx->comm);
  if (comm) {
    if (ncclAllReduce(w.counts, w.counts, nt, ncclFloat64, ncclSum, comm, s) != ncclSuccess)
      return fail(ctx, TLP_ERR_NCCL, "loss-count allreduce failed");
  }
  // From here on this rank has entered the step's collectives (C-0 above, the
  // gradient buckets during the backward): a failure must not leave its peers
  // waiting for collectives it will never issue.  Join any buckets in flight
  // (the next step's backward must not race their in-place allreduce) and
  // abort the communicator.
  auto bail = [&](tlp_status e) {
    if (comm) {
      if (ctx->buckets_issued && ctx->comm_stream) {
        cudaEventRecord(ctx->bucket_ev[4], ctx->comm_stream);
        cudaStreamWaitEvent(s, ctx->bucket_ev[4], 0);
      }
      const std::string why = ctx->last_error;
      abort_comm(ctx, why);
      ctx->last_error = why + " (communicator aborted: this rank left the step)";
    }
    return e;
  };
  ctx->buckets_issued = 0;
  if ((st = simt_forward(ctx, feats, B, w.scores, true, s)) != TLP_OK) return bail(st);
  ctx->train_scores = w.scores;
  st = mse ? mse_loss_grad(ctx, w.scores, labels, B, w.counts, loss_out, w.dscores, s)
           : rank_loss_grad(ctx, w.scores, labels, w.goff, G, B, max_group, w.counts, loss_out,
                            w.dscores, s);
  if (st != TLP_OK) return bail(st);
  if ((st = simt_backward(ctx, B, w.dscores, s)) != TLP_OK) return bail(st);
  if (comm) {
    // C-1: gradient allreduce (sum); every rank then applies the same Adam step.
    if (ctx->buckets_issued) {  // the buckets went out during the backward: join them
      TLP_CUDA_TRY(cudaEventRecord(ctx->bucket_ev[4], ctx->comm_stream));
      TLP_CUDA_TRY(cudaStreamWaitEvent(s, ctx->bucket_ev[4], 0));
    } else if (ncclAllReduce(ctx->d_grads, ctx->d_grads, ctx->off.total, ncclFloat32, ncclSum, comm, s) !=
               ncclSuccess) {
      return fail(ctx, TLP_ERR_NCCL, "gradient allreduce failed");
    }
    if (ncclAllReduce(loss_out, loss_out, 1, ncclFloat32, ncclSum, comm, s) != ncclSuccess)
      return fail(ctx, TLP_ERR_NCCL, "loss allreduce failed");
    if ((st = note_collective(ctx, s)) != TLP_OK) return st;
  }
  return TLP_OK;
}

// [W, T, k] per-shard top-k lists (scores + global indices) -> the global top-k
// per task, by the same deterministic tournament as tlp_topk (R21).
tlp_status merge_gathered(tlp_ctx* ctx, const float* gs, const int64_t* gi, float* ts, int64_t* ti,
                          int W, int T, int k, int64_t* idx_out, float* val_out, cudaStream_t s) {
  const size_t loc = (size_t)T * k;
  // [W, T, k] -> [T, W, k] so every segment's candidates are contiguous
  for (int r = 0; r < W; ++r) {
    TLP_CUDA_TRY(cudaMemcpy2DAsync(ts + (size_t)r * k, (size_t)W * k * sizeof(float),
                                   gs + (size_t)r * loc, (size_t)k * sizeof(float),
                                   (size_t)k * sizeof(float), T, cudaMemcpyDeviceToDevice, s));
    TLP_CUDA_TRY(cudaMemcpy2DAsync(ti + (size_t)r * k, (size_t)W * k * sizeof(int64_t),
                                   gi + (size_t)r * loc, (size_t)k * sizeof(int64_t),
                                   (size_t)k * sizeof(int64_t), T, cudaMemcpyDeviceToDevice, s));
  }
  return topk_merge_launch(ctx, ts, ti, T, (int64_t)W * k, k, idx_out, val_out, s);
}

}  // namespace

tlp_status tlp_compute_grads(tlp_ctx* ctx, const float* feats, const float* labels,
                             const int64_t* group_off, int32_t B, int32_t G, float* loss_out,
                             void* stream) {
  CHECK_CTX();
  return grads_impl(ctx, feats, labels, group_off, B, G, loss_out,
                    reinterpret_cast<cudaStream_t>(stream));
}

tlp_status tlp_train_step(tlp_ctx* ctx, const float* feats, const float* labels,
                          const int64_t* group_off, int32_t B, int32_t G, float* loss_out,
                          void* stream) {
  CHECK_CTX();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  tlp_status st = grads_impl(ctx, feats, labels, group_off, B, G, loss_out, s);
  if (st != TLP_OK) return st;
  return adam_launch(ctx, s);
}

tlp_status tlp_lambdarank(tlp_ctx* ctx, const float* scores, const float* labels,
                          const int64_t* group_off, int32_t B, int32_t G, float* loss_out,
                          float* dscores_out, void* stream) {
  CHECK_CTX();
  if (!scores || !labels || !loss_out || !dscores_out) return fail(ctx, TLP_ERR_ARG, "null buffer");
  int max_group = 0;
  tlp_status st = check_groups(ctx, group_off, B, G, &max_group);
  if (st != TLP_OK) return st;
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  TrainWs w;
  if ((st = train_ws(ctx, B, G, &w)) != TLP_OK) return st;
  if ((st = upload_goff(ctx, w.goff, group_off, G, s)) != TLP_OK) return st;
  if ((st = rank_pair_counts(ctx, labels, w.goff, G, max_group, w.counts, s)) != TLP_OK) return st;
  return rank_loss_grad(ctx, scores, labels, w.goff, G, B, max_group, w.counts, loss_out,
                        dscores_out, s);
}

tlp_status tlp_mse(tlp_ctx* ctx, const float* scores, const float* labels, int32_t B,
                   float* loss_out, float* dscores_out, void* stream) {
  CHECK_CTX();
  if (!scores || !labels || !loss_out || !dscores_out || B < 1) return fail(ctx, TLP_ERR_ARG, "bad MSE arguments");
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  TrainWs w;
  tlp_status st = train_ws(ctx, B, 1, &w);
  if (st != TLP_OK) return st;
  if ((st = mse_counts(ctx, labels, B, w.counts, s)) != TLP_OK) return st;
  return mse_loss_grad(ctx, scores, labels, B, w.counts, loss_out, dscores_out, s);
}

tlp_status tlp_topk(tlp_ctx* ctx, const float* scores, int32_t score_stride, int32_t head,
                    const int64_t* task_off, int32_t T, int32_t k, int64_t shard_base,
                    int64_t* idx_out, float* val_out, void* stream) {
  CHECK_CTX();
  if (!task_off || !idx_out || !val_out || T < 1 || k < 1 || score_stride < 1 || head < 0 ||
      head >= score_stride)
    return fail(ctx, TLP_ERR_ARG, "bad top-k arguments");
  for (int t = 0; t < T; ++t)
    if (task_off[t + 1] < task_off[t] || task_off[0] < 0)
      return fail(ctx, TLP_ERR_SHAPE, "task_off must be non-decreasing");
  if (task_off[T] > task_off[0] && !scores) return fail(ctx, TLP_ERR_ARG, "null scores");
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(ctx->comm);
  if (!comm) {
    return topk_launch(ctx, scores, score_stride, head, task_off, T, k, shard_base, idx_out,
                       val_out, s);
  }
  // C-2: local top-k -> allgather of T*k (score, index) -> the same merge everywhere.
  const int W = ctx->world;
  const size_t loc = (size_t)T * k;
  TLP_CUDA_TRY(ctx->ws_misc.ensure(loc * (sizeof(float) + sizeof(int64_t)) * (1 + 2 * (size_t)W) + 1024));
  char* p = ctx->ws_misc.as<char>();
  int64_t* li = reinterpret_cast<int64_t*>(p); p += loc * sizeof(int64_t);
  int64_t* gi = reinterpret_cast<int64_t*>(p); p += loc * W * sizeof(int64_t);
  int64_t* ti = reinterpret_cast<int64_t*>(p); p += loc * W * sizeof(int64_t);
  float* ls = reinterpret_cast<float*>(p); p += loc * sizeof(float);
  float* gs = reinterpret_cast<float*>(p); p += loc * W * sizeof(float);
  float* ts = reinterpret_cast<float*>(p);
  tlp_status st = topk_launch(ctx, scores, score_stride, head, task_off, T, k, shard_base, li, ls, s);
  if (st != TLP_OK) return st;
  if (ncclGroupStart() != ncclSuccess ||
      ncclAllGather(ls, gs, loc, ncclFloat32, comm, s) != ncclSuccess ||
      ncclAllGather(li, gi, loc, ncclInt64, comm, s) != ncclSuccess ||
      ncclGroupEnd() != ncclSuccess)
    return fail(ctx, TLP_ERR_NCCL, "top-k allgather failed");
  if ((st = note_collective(ctx, s)) != TLP_OK) return st;
  return merge_gathered(ctx, gs, gi, ts, ti, W, T, k, idx_out, val_out, s);
}

tlp_status tlp_topk_merge(tlp_ctx* ctx, const float* vals, const int64_t* idx, int32_t W, int32_t T,
                          int32_t k, int64_t* idx_out, float* val_out, void* stream) {
  CHECK_CTX();
  if (!vals || !idx || !idx_out || !val_out || W < 1 || T < 1 || k < 1)
    return fail(ctx, TLP_ERR_ARG, "bad top-k merge arguments");
  cudaSetDevice(ctx->device);
  const size_t n = (size_t)W * T * k;
  TLP_CUDA_TRY(ctx->ws_merge.ensure(n * (sizeof(float) + sizeof(int64_t)) + 256));
  int64_t* ti = ctx->ws_merge.as<int64_t>();
  float* ts = reinterpret_cast<float*>(ti + n);
  return merge_gathered(ctx, vals, idx, ts, ti, W, T, k, idx_out, val_out,
                        reinterpret_cast<cudaStream_t>(stream));
}

tlp_status tlp_normalize_labels(tlp_ctx* ctx, const float* latency, const int64_t* group_off,
                                int32_t G, float* label_out, void* stream) {
  CHECK_CTX();
  if (!latency || !group_off || !label_out || G < 0) return fail(ctx, TLP_ERR_ARG, "null buffer");
  for (int g = 0; g < G; ++g)
    if (group_off[g + 1] < group_off[g]) return fail(ctx, TLP_ERR_SHAPE, "group_off must be non-decreasing");
  cudaSetDevice(ctx->device);
  return normalize_labels_launch(ctx, latency, group_off, G, label_out,
                                 reinterpret_cast<cudaStream_t>(stream));
}

tlp_status tlp_sync(tlp_ctx* ctx) {
  CHECK_CTX();
  cudaSetDevice(ctx->device);
  if (ctx->comm && ctx->coll_ev) {
    // bounded wait on the last enqueued collective: a peer that never joins
    // would otherwise hang cudaDeviceSynchronize forever
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(ctx->comm);
    const auto t0 = std::chrono::steady_clock::now();
    const double limit = nccl_timeout_s();
    for (;;) {
      const cudaError_t q = cudaEventQuery(ctx->coll_ev);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) TLP_CUDA_TRY(q);
      ncclResult_t ar = ncclSuccess;
      ncclCommGetAsyncError(comm, &ar);
      if (ar != ncclSuccess && ar != ncclInProgress)
        return abort_comm(ctx, std::string("NCCL: ") + ncclGetErrorString(ar));
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > limit)
        return abort_comm(ctx, "NCCL collective not complete after " + std::to_string((int)limit) +
                                   " s (TLP_NCCL_TIMEOUT_S)");
      std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
  }
  TLP_CUDA_TRY(cudaDeviceSynchronize());
  if (ctx->comm) {
    ncclResult_t ar = ncclSuccess;
    ncclCommGetAsyncError(reinterpret_cast<ncclComm_t>(ctx->comm), &ar);
    if (ar != ncclSuccess) return fail(ctx, TLP_ERR_NCCL, ncclGetErrorString(ar));
  }
  return dev_error_status(ctx);
}

int64_t tlp_launch_count(const tlp_ctx* ctx) { return ctx ? ctx->launches : -1; }

}  // extern "C"
