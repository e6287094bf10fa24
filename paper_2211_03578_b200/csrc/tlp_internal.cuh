// Internal declarations shared by the libtlp.so translation units.
// Product code: nothing here is shared with oracle/ (the CPU checker).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>
#include <vector>
#include <mutex>
#include <atomic>

#include "../../include/tlp.h"

#define TLP_MAX_UP 4
#define TLP_MAX_ATTN 4
#define TLP_MAX_RES 4
#define TLP_MAX_TASKS 8
#define TLP_MAX_ROUND_CHUNKS 64

// Sticky device error bits (ctx->d_err), surfaced by tlp_sync.
enum : uint32_t {
  DERR_EMPTY_SEQ = 1u << 0,
  DERR_UNKNOWN_TYPE = 1u << 1,
  DERR_NONFINITE = 1u << 2,
  DERR_NAN_LOSS = 1u << 3,
};

// R24 flat-parameter offsets (fp32 elements).
struct ParamOffsets {
  int64_t up_W[TLP_MAX_UP], up_b[TLP_MAX_UP];
  int64_t pos;  // R43 positional table [L, hidden] (cfg.pos_enc), else -1
  int64_t Wq[TLP_MAX_ATTN], bq[TLP_MAX_ATTN], Wk[TLP_MAX_ATTN], bk[TLP_MAX_ATTN];
  int64_t Wv[TLP_MAX_ATTN], bv[TLP_MAX_ATTN], Wo[TLP_MAX_ATTN], bo[TLP_MAX_ATTN];
  int64_t Wa[TLP_MAX_RES], a[TLP_MAX_RES], Wb[TLP_MAX_RES], b[TLP_MAX_RES];
  int64_t W1[TLP_MAX_TASKS], c1[TLP_MAX_TASKS], w2[TLP_MAX_TASKS], c2[TLP_MAX_TASKS];
  // R49 LSTM layers (backbone == 1) in place of the attention layers
  int64_t Wih[TLP_MAX_ATTN], bih[TLP_MAX_ATTN], Whh[TLP_MAX_ATTN], bhh[TLP_MAX_ATTN];
  int64_t total;
};

// Grow-only device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t want = n + (n >> 3);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
  void release() { if (p) cudaFree(p); p = nullptr; bytes = 0; }
};

struct TcWeights;  // bf16 tcgen05 weight images (k_tc_forward.cu)
struct GaSpace;    // NEXT-1 search space + round workspaces (k_search.cu)

struct tlp_ctx {
  tlp_config cfg;
  int device = 0;
  int num_sms = 148;
  ParamOffsets off;
  std::string last_error;

  // parameters / optimizer (fp32, device)
  float* d_params = nullptr;
  float* d_grads = nullptr;
  float* d_m = nullptr;
  float* d_v = nullptr;
  int64_t adam_t = 0;
  bool have_params = false;

  // tokenizer state
  bool have_scales = false;
  float* d_scale = nullptr;          // [E]
  uint64_t* d_hkeys = nullptr;       // open-addressing hash: key (0 = empty)
  int32_t* d_hval = nullptr;         // token
  uint8_t* d_tblob = nullptr;        // table strings for verification
  int64_t* d_toff = nullptr;
  int32_t* d_hstr = nullptr;         // slot -> table string index
  uint32_t hcap = 0;                 // power of two (0 = no table)

  // sticky error word
  uint32_t* d_err = nullptr;

  // workspaces
  DevBuf ws_tokens, ws_act, ws_train, ws_rank, ws_topk, ws_misc, ws_partial, ws_merge;
  DevBuf ws_bimg;  // bf16 hi/lo images of the training GEMMs' weight operands, two halves
                   // used alternately (k_tc_gemm.cu: the next image is built while the
                   // previous GEMM still reads its own)
  size_t bimg_half = 0;
  int bimg_flip = 0;
  DevBuf ws_hcat;  // MTL heads side by side: [W1_0 | W1_1 | ...] [H, nt hd] then [c1_0 | c1_1 | ...]
  DevBuf ws_wcat;  // per attention layer [Wq | Wk | Wv] rows side by side, then [bq | bk | bv]:
                  // the fused Q/K/V forward GEMM and dgrad operands (k_simt.cu)

  // bf16 tensor-core path
  TcWeights* tc = nullptr;
  bool tc_dirty = true;

  // tlp_search_round (round.cu): device copy of the host batch (same offsets),
  // one chunk of features, all scores; copy stream + per-chunk events
  DevBuf ws_round_in, ws_round_feats, ws_round_scores;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t round_ev[TLP_MAX_ROUND_CHUNKS + 1] = {};

  // NCCL
  void* comm = nullptr;  // ncclComm_t
  // C-1 gradient buckets: each finished parameter range is
  // allreduced on comm_stream while the backward continues (TLP_GRAD_BUCKETS=0:
  // one allreduce after the backward, the no-overlap variant)
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t bucket_ev[5] = {};
  int buckets_issued = 0;
  int rank = 0, world = 1;
  // recorded after the last collective a call enqueued: tlp_sync waits on it
  // with a bound (TLP_NCCL_TIMEOUT_S) and aborts the communicator on timeout
  // or an asynchronous NCCL error
  cudaEvent_t coll_ev = nullptr;
  // training group offsets (api.cu upload_goff): the last offsets uploaded,
  // where and on which stream (an unchanged batch layout skips the copy), and a
  // pinned staging ring for changed ones (no pageable copy per step)
  std::vector<int64_t> goff_last;
  const void* goff_dev = nullptr;
  cudaStream_t goff_stream = nullptr;
  static constexpr int kGoffRing = 4;
  int64_t* goff_pinned[kGoffRing] = {};
  size_t goff_pinned_cap = 0;
  cudaEvent_t goff_ev[kGoffRing] = {};
  int goff_slot = 0;
  // size of the token table (tlp_broadcast_state)
  int32_t tok_n = 0;
  int64_t tok_bytes = 0;

  int64_t launches = 0;

  // NEXT-1 tuning-round search space (tlp_ga_set_space)
  GaSpace* ga = nullptr;

  // training forward state kept for backward (k_simt.cu)
  int64_t train_N = -1;
  const float* train_X = nullptr;
  // scores [train_N, n_tasks] of the last training forward (tlp_get_train_scores)
  const float* train_scores = nullptr;
};

// ---------------------------------------------------------------------------
// helpers
#define TLP_CUDA_TRY(expr)                                                    \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      ctx->last_error = std::string("CUDA: ") + cudaGetErrorString(_e) +      \
                        " at " __FILE__ ":" + std::to_string(__LINE__);       \
      return TLP_ERR_CUDA;                                                    \
    }                                                                         \
  } while (0)

#define TLP_LAUNCH_CHECK()                                                    \
  do {                                                                        \
    ctx->launches++;                                                          \
    cudaError_t _e = cudaGetLastError();                                      \
    if (_e != cudaSuccess) {                                                  \
      ctx->last_error = std::string("CUDA launch: ") +                        \
                        cudaGetErrorString(_e) + " at " __FILE__ ":" +        \
                        std::to_string(__LINE__);                             \
      return TLP_ERR_CUDA;                                                    \
    }                                                                         \
  } while (0)

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch (PDL) for the training step's chain of kernels
// (68 launches per C3 step, ~2 us of idle device time at each boundary): a
// kernel launched by TLP_LAUNCH_PDL may be scheduled while its predecessor in
// the stream drains, so it MUST call pdl_wait() before touching global memory
// (griddepcontrol.wait returns once every prerequisite grid has completed and
// its writes are visible; it is a no-op for a normal launch), and it calls
// pdl_trigger() once its own CTAs are resident so that the next kernel's
// launch overlaps its tail.  TLP_PDL=0 launches them normally (A/B).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
#define TLP_LAUNCH_PDL(kern, grid, block, smem, stream, ...)                  \
  do {                                                                        \
    cudaError_t _le = launch_pdl(kern, grid, block, smem, stream, __VA_ARGS__); \
    if (_le != cudaSuccess) {                                                 \
      ctx->last_error = std::string("CUDA launch: ") + cudaGetErrorString(_le) + \
                        " at " __FILE__ ":" + std::to_string(__LINE__);       \
      return TLP_ERR_CUDA;                                                    \
    }                                                                         \
  } while (0)  // follow with TLP_LAUNCH_CHECK() (launch count)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: remember per
// call site which devices already have it (bit = device ordinal), so a process
// with contexts on several GPUs sets it on each of them.
#define TLP_SMEM_ATTR(func, bytes)                                                       \
  do {                                                                                 \
    static std::atomic<uint64_t> _tlp_attr_mask{0};                                    \
    int _tlp_dev = 0;                                                                  \
    cudaGetDevice(&_tlp_dev);                                                          \
    const uint64_t _tlp_bit = 1ull << (_tlp_dev & 63);                                 \
    if (!(_tlp_attr_mask.load(std::memory_order_acquire) & _tlp_bit)) {                \
      cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes)); \
      _tlp_attr_mask.fetch_or(_tlp_bit, std::memory_order_acq_rel);                    \
    }                                                                                  \
  } while (0)

// ---------------------------------------------------------------------------
// kernels / launchers implemented in the .cu files

// k_encode.cu
tlp_status encode_launch(tlp_ctx* ctx, const tlp_seq_batch* in, int64_t N, float* feats,
                         cudaStream_t s);
// the two halves of encode_launch: batch strings -> tokens (ctx->ws_tokens), and
// rows of candidates [0, N) of `in` (seq_off may be a shifted view: offsets are absolute)
tlp_status encode_resolve(tlp_ctx* ctx, const tlp_seq_batch* in, cudaStream_t s);
tlp_status encode_rows(tlp_ctx* ctx, const tlp_seq_batch* in, int64_t N, float* feats,
                       cudaStream_t s);
// R3 scales fitted on the device from a packed training batch -> ctx->d_scale
tlp_status fit_scales_launch(tlp_ctx* ctx, const tlp_seq_batch* in, int64_t N, cudaStream_t s);
// api.cu: the bf16 / fp32 scoring dispatch behind tlp_score (no argument checks)
tlp_status score_launch(tlp_ctx* ctx, const float* feats, int64_t N, float* scores, cudaStream_t s);
tlp_status build_token_table(tlp_ctx* ctx, const uint8_t* blob, const int64_t* off, int32_t n);

// k_select.cu
tlp_status topk_launch(tlp_ctx* ctx, const float* scores, int stride, int head,
                       const int64_t* task_off, int T, int k, int64_t base, int64_t* idx_out,
                       float* val_out, cudaStream_t s);
tlp_status normalize_labels_launch(tlp_ctx* ctx, const float* lat, const int64_t* group_off,
                                   int G, float* out, cudaStream_t s);

// k_simt.cu : fp32 SIMT network (forward for scoring and training, backward)
struct EpiParams {
  const float* bias = nullptr;   // [N]
  const float* resid = nullptr;  // [M, ldr] added before activation
  int64_t ldr = 0;
  const float* mask = nullptr;   // [M, ldm] multiply by (mask > 0) (relu')
  int64_t ldm = 0;
  bool relu = false;
  bool accumulate = false;       // C += result (C read before write)
  bool mask_after = false;       // apply `mask` to the accumulated value (C + result)
};
tlp_status sgemm(tlp_ctx* ctx, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A,
                 int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                 const EpiParams& ep, cudaStream_t s);
// dW[K,N] (+)= A^T[K,M] * dY[M,N], deterministic split over M.
tlp_status sgemm_wgrad(tlp_ctx* ctx, int64_t M, int64_t K, int64_t N, const float* A, int64_t lda,
                       const float* dY, int64_t lddy, float* dW, cudaStream_t s);
tlp_status colsum(tlp_ctx* ctx, int64_t M, int64_t N, const float* X, int64_t ldx, float* out,
                  cudaStream_t s);
// dW = A^T dY and db = colsum(dY) (db must be dW + K*N, the R24 layout): one
// fused tcgen05 pass on bf16 contexts where the shape allows, else the two calls.
tlp_status sgemm_wgrad_bias(tlp_ctx* ctx, int64_t M, int64_t K, int64_t N, const float* A, int64_t lda,
                            const float* dY, int64_t lddy, float* dW, float* db, cudaStream_t s);
bool tc_wgrad_bias(tlp_ctx* ctx, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                   const float* B, int64_t ldb, float* part, int splits, int64_t kslice,
                   cudaStream_t s, tlp_status* st, int J = 1, int64_t bjs = 0, int64_t pjs = 0);
tlp_status simt_forward(tlp_ctx* ctx, const float* feats, int64_t N, float* scores, bool save,
                        cudaStream_t s);
// C-1 bucket: gradients [lo, hi) are final on stream s -> allreduce them on the
// comm stream (no-op without a communicator or with TLP_GRAD_BUCKETS=0)
tlp_status grad_bucket_ready(tlp_ctx* ctx, int64_t lo, int64_t hi, cudaStream_t s);
tlp_status simt_backward(tlp_ctx* ctx, int64_t N, const float* dscores, cudaStream_t s);

// k_tc_gemm.cu : bf16x3 tcgen05 GEMMs of the training path of bf16 contexts
// k_tc_tma.cu: the TMA-fed persistent variant for 128 < N <= 256, row-major A
// (img = bimg_kernel's weight image); TLP_ERR_UNSUPPORTED = not applicable
tlp_status tc_gemm_tma(tlp_ctx* ctx, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                       const uint8_t* img, float* C, int64_t ldc, const EpiParams& e, cudaStream_t s);
// k_tc_tma.cu: 2-D fp32 tensor map (row pitch ld floats, box box_rows x
// box_cols); swizzle = CUtensorMapSwizzle value; false if it cannot be encoded
bool make_tmap_f32_2d(CUtensorMap* m, const float* base, int64_t cols, int64_t rows, int64_t ld,
                      uint32_t box_cols, uint32_t box_rows, int swizzle);
// k_tc_tma.cu: TMA-fed kind::tf32 weight (+ bias) gradient partials, R52
tlp_status tc_wgrad_tma(tlp_ctx* ctx, int64_t R, int64_t Mf, int64_t Nf, const float* X, int64_t ldx,
                        const float* dY, int64_t ldy, float* part, int Z, int64_t kslice, bool colsum,
                        int J, int64_t cy0, cudaStream_t s);
tlp_status tc_gemm(tlp_ctx* ctx, bool ta, bool tb, int64_t M, int64_t N, int64_t K,
                   const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                   int64_t ldc, const EpiParams& e, int splits, int64_t kslice, cudaStream_t s);

// k_attn_tc.cu: tf32 mma.sync attention core of bf16-context training (d_h = 32)
bool attn_tc_ok(const tlp_ctx* ctx);
tlp_status attn_fwd_tc(tlp_ctx* ctx, const float* qkv, int64_t N, float* O, float* A,
                       const float* kvalid, cudaStream_t s);
tlp_status attn_bwd_tc(tlp_ctx* ctx, const float* qkv, const float* A, const float* dO, int64_t N,
                       float* dqkv, cudaStream_t s);
// k_rank.cu: MSE (NEXT-3): present-label counts per task, then loss + dscores
tlp_status mse_counts(tlp_ctx* ctx, const float* labels, int64_t B, double* d_counts, cudaStream_t s);
tlp_status mse_loss_grad(tlp_ctx* ctx, const float* scores, const float* labels, int64_t B,
                         const double* d_counts, float* loss_out, float* dscores, cudaStream_t s);
// k_rank.cu
tlp_status rank_pair_counts(tlp_ctx* ctx, const float* labels, const int64_t* d_goff, int G,
                            int max_group, double* d_counts, cudaStream_t s);
tlp_status rank_loss_grad(tlp_ctx* ctx, const float* scores, const float* labels,
                          const int64_t* d_goff, int G, int B, int max_group,
                          const double* d_counts, float* loss_out, float* dscores,
                          cudaStream_t s);

// k_adam.cu
tlp_status adam_launch(tlp_ctx* ctx, cudaStream_t s);

// k_tc_forward.cu : bf16 tcgen05 fused forward
bool tc_supported(const tlp_config& c);
// scoring is available: fp32, the fused bf16 kernel, or (LSTM, NEXT-4) the
// layer-by-layer bf16x3 GEMM path
inline bool score_supported(const tlp_config& c) {
  return c.precision != TLP_PREC_BF16 || c.backbone == 1 || tc_supported(c);
}
tlp_status tc_prepare(tlp_ctx* ctx, cudaStream_t s);
tlp_status tc_forward(tlp_ctx* ctx, const float* feats, int64_t N, float* scores, cudaStream_t s);
void tc_free(tlp_ctx* ctx);

// api.cu
tlp_status dev_error_status(tlp_ctx* ctx);

// k_search.cu
void ga_free(tlp_ctx* ctx);
