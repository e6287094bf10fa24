/*
 * tlp.h -- C ABI of libtlp.so, the B200 (sm_100a) hot path of TLP / MTL-TLP
 * (arXiv 2211.03578, "TLP: A Deep Learning-based Cost Model for Tensor Program
 * Tuning").  Citations: P:n = PAPER.md line n; R# = reading in DESIGN.md
 * "Readings" (= SURVEY.md §8(c)).
 *
 * The problem statement the calls follow (§3 "System Overview"):
 *   training:  "the TLP cost model forwardly propagates the finally extracted
 *               features and normalizes the latency of the corresponding tensor
 *               program as a label to calculate the loss.  Finally, the loss is
 *               back-propagated to update the weights"  -> tlp_normalize_labels,
 *               tlp_train_step
 *   inference: "the auto-tuner obtains the prediction score through the cost
 *               model and screens out the top-k potential candidates"
 *               -> tlp_encode, tlp_score, tlp_topk
 *
 * Conventions (all entry points):
 *   - Plain C types only.  "device" = CUDA global memory of the ctx's device;
 *     "host" = ordinary host memory.  The caller owns every buffer it passes;
 *     the ctx owns weights, optimizer state, the token table, scales,
 *     workspaces and the NCCL communicator.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Calls are stream-ordered; none synchronises the device except
 *     tlp_sync / tlp_get_params / tlp_get_grads / tlp_get_train_scores.
 *   - Host-detectable errors (NULL pointers, bad sizes, config mismatch) return
 *     immediately with a negative status and leave all outputs untouched.
 *     Device-detected data errors (empty sequence, type id >= T, non-finite
 *     number or score, NaN loss) set a sticky error word in the ctx that the
 *     next tlp_sync returns (and clears).  tlp_last_error() gives a message.
 *   - A ctx is single-threaded: calls on one ctx must not overlap in host
 *     time, and work queued on different streams of one ctx must not overlap
 *     on the device (ctx workspaces are shared).  Use one ctx per host thread.
 */
#ifndef TLP_H_
#define TLP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tlp_ctx tlp_ctx; /* opaque; created by tlp_create, owned by the library */

typedef enum {
  TLP_OK = 0,
  TLP_ERR_ARG = -1,           /* NULL pointer / negative size / bad enum */
  TLP_ERR_SHAPE = -2,         /* config or buffer shape mismatch */
  TLP_ERR_EMPTY_SEQ = -3,     /* a candidate has 0 primitives */
  TLP_ERR_UNKNOWN_TYPE = -4,  /* a kept primitive has type id >= T */
  TLP_ERR_NONFINITE = -5,     /* a kept numeric argument or a score is NaN/Inf */
  TLP_ERR_NAN_LOSS = -6,      /* training loss became NaN */
  TLP_ERR_NO_LABELS = -7,     /* reserved */
  TLP_ERR_CUDA = -8,          /* CUDA runtime error (message in tlp_last_error) */
  TLP_ERR_NCCL = -9,          /* NCCL error */
  TLP_ERR_STATE = -10,        /* call not valid in the ctx's state (e.g. no params) */
  TLP_ERR_UNSUPPORTED = -11   /* configuration outside what this build implements */
} tlp_status;

typedef enum {
  TLP_PREC_FP32 = 0,  /* fp32 SIMT everywhere: the 1e-5 relative path (no TF32) */
  TLP_PREC_BF16 = 1   /* bf16 tcgen05 tensor-core scoring, fp32 accumulation (1e-2 path) */
} tlp_precision;

/*
 * Model / feature configuration.  Defaults of the paper:
 * L=25, E=22, T=11, hidden=256, attn_heads=8, n_attn=1, n_res=2.  R11 upsample
 * widths up_dims[0..n_up) (ReLU after each, last == hidden); R13 head
 * hidden -> head_dim (ReLU) -> 1, summed over the L rows; n_tasks heads for
 * MTL-TLP.
 * Limits of this build: L <= 32, E <= 64, T < E, hidden % attn_heads == 0,
 * hidden <= 512, n_up <= 4, 1 <= n_tasks <= 8.  TLP_PREC_BF16 training runs
 * its dense layers on the tensor cores for any shape; TLP_PREC_BF16 scoring
 * (the fused kernel) requires the paper shape (E=22, hidden=256,
 * up_dims={128,256}, attn_heads=8, head_dim=128, L=25) and otherwise
 * tlp_score returns TLP_ERR_UNSUPPORTED (an LSTM backbone, NEXT-4, scores
 * through the layer-by-layer tensor-core GEMMs instead).
 */
typedef struct {
  int L, E, T;
  int hidden;
  int up_dims[4];
  int n_up;
  int attn_heads;
  int n_attn;
  int n_res;
  int head_dim;
  int n_tasks;
  int precision;              /* tlp_precision */
  float lr, beta1, beta2, eps; /* Adam (R23 / S:356: 1e-3, 0.9, 0.999, 1e-8) */
  unsigned long long seed;    /* reserved */
  int loss;                   /* tlp_loss: training loss ("MSE loss function or the rank loss") */
  int attn_mask;              /* NEXT-3 / R42: 1 = padding keys (all-zero input rows) are masked
                                 out of every attention softmax; 0 = no mask (the paper, R8) */
  int pos_enc;                /* NEXT-3 / R43: 1 = learned positional table pos [L, hidden] added
                                 after the upsample (R24: right after the upsample parameters);
                                 0 = none (the paper, R9) */
  int backbone;               /* NEXT-4 / R49: 0 = n_attn self-attention layers (the paper's
                                 choice); 1 = n_attn LSTM layers hidden -> hidden (gates
                                 i, f, g, o; h0 = c0 = 0; identity residual), "the
                                 self-attention or LSTM module".  LSTM contexts score through
                                 the layer-by-layer path (fp32 SIMT, or bf16x3 tcgen05 GEMMs for
                                 TLP_PREC_BF16) and require attn_mask = 0. */
} tlp_config;

typedef enum {
  TLP_LOSS_LAMBDARANK = 0,  /* R16 (the paper's choice) */
  TLP_LOSS_MSE = 1          /* NEXT-3: per-task mean squared residual over present labels (R41) */
} tlp_loss;

/* Packed abstract schedule primitives (S ::= p*, p ::= tau (id|num)*).
 * Structure of arrays; ALL pointers are device memory owned by the caller. */
typedef struct {
  const int64_t* seq_off;        /* [N+1] primitive offsets per candidate */
  const uint8_t* prim_type;      /* [P] type id tau in [0,T) (F1 -> one-hot) */
  const int64_t* arg_off;        /* [P+1] argument offsets per primitive */
  const uint8_t* arg_kind;       /* [A] 0 = Number (F3), 1 = NameParam (F2) */
  const double* arg_num;         /* [A] Number value (used when kind == 0) */
  const int32_t* arg_name;       /* [A] index into the batch string table (kind == 1) */
  const uint8_t* str_blob;       /* batch string table, UTF-8 bytes */
  const int64_t* str_off;        /* [U+1] byte offsets into str_blob */
  int64_t P, A;                  /* numbers of primitives / arguments */
  int32_t U;                     /* number of batch strings */
} tlp_seq_batch;

/* ---- lifetime ---------------------------------------------------------- */
tlp_status tlp_create(const tlp_config* cfg, int device, tlp_ctx** out);
void tlp_destroy(tlp_ctx* ctx);
/* Message of the last error on this ctx (valid until the next call on it). */
const char* tlp_last_error(const tlp_ctx* ctx);
/* Default configuration of the paper with Adam defaults (R23). */
void tlp_default_config(tlp_config* cfg);

/* ---- state -------------------------------------------------------------- */
/* F2's token table ("We map different character parameters to different
 * tokens"): string i (bytes blob[off[i]..off[i+1])) gets token i + 2; 0 = pad,
 * 1 = unknown (R1).  n < 2^24 - 2.  Host memory; copied. */
tlp_status tlp_set_token_table(tlp_ctx* ctx, const uint8_t* blob, const int64_t* off, int32_t n);
/* Post-processing normalisation scales ("normalization"; R3): [E] host
 * floats, all > 0.  Output column c is divided by scale[c] (IEEE fp32). */
tlp_status tlp_set_norm_scales(tlp_ctx* ctx, const float* scale);
/* R1 / R3 fitted by the library from a training split (the paper's
 * post-processing "normalization", fitted instead of supplied):
 * tlp_fit_token_table: token i + 2 for the i-th distinct name argument in
 *   first-occurrence order over the packed batch `in` (HOST memory; candidates,
 *   primitives, arguments in order; all arguments, cropped or not).  Replaces
 *   the ctx table.  TLP_ERR_ARG on a name index outside the string table.
 * tlp_fit_norm_scales: scale[c] = max over the kept data (crop R4) of |x[n,r,c]|
 *   of the un-normalised rows tlp_encode would build (one-hot 1, RN_f32 number,
 *   token of the ctx table), 1.0 for an all-zero column; `in` in DEVICE memory.
 *   Stream-ordered; sets the ctx scales and, if scale_out != NULL, copies the
 *   [E] floats there (host or device).  Device errors as tlp_encode. */
tlp_status tlp_fit_token_table(tlp_ctx* ctx, const tlp_seq_batch* in, int64_t N);
tlp_status tlp_fit_norm_scales(tlp_ctx* ctx, const tlp_seq_batch* in, int64_t N, float* scale_out,
                               void* stream);
/* Number of fp32 parameters in the R24 flat order. */
int64_t tlp_num_params(const tlp_ctx* ctx);
/* Flat fp32 parameters in R24 order (W stored [in,out] row-major).  `flat` may
 * be host or device memory.  Resets Adam state.  Synchronous. */
tlp_status tlp_set_params(tlp_ctx* ctx, const float* flat, int64_t n);
tlp_status tlp_get_params(tlp_ctx* ctx, float* flat, int64_t n);
/* Gradient of the last tlp_compute_grads / tlp_train_step (after allreduce). */
tlp_status tlp_get_grads(tlp_ctx* ctx, float* flat, int64_t n);
/* Test hook (R26): the scores [B, n_tasks] fp32 of the forward pass of the last
 * tlp_compute_grads / tlp_train_step -- the scores its LambdaRank ranked --
 * copied to `out` (host or device, n = B * n_tasks).  Synchronises the device.
 * TLP_ERR_STATE before the first training call, TLP_ERR_SHAPE on a count
 * mismatch. */
tlp_status tlp_get_train_scores(tlp_ctx* ctx, float* out, int64_t n);
/* Data-parallel communicator: `nccl_id` points to the 128-byte
 * ncclUniqueId created by rank 0 and broadcast by the caller; blocks until all
 * `world` ranks have joined.  world == 1 with nccl_id == NULL disables
 * collectives; world == 1 with an id builds a 1-rank communicator (the
 * collective code paths then run on one GPU, as the tests use it). */
tlp_status tlp_set_comm(tlp_ctx* ctx, const void* nccl_id, int rank, int world);
/* C-3: make every rank's model state rank `root`'s -- the
 * parameters and Adam moments / step count (if the root has parameters), the
 * normalisation scales (if set) and the token table -- by ncclBroadcast over
 * the ctx communicator.  Collective: every rank of the communicator calls it
 * with the same root.  Synchronises `stream` once (the sizes in a small header
 * decide the receivers' allocations).  TLP_ERR_STATE without a communicator. */
tlp_status tlp_broadcast_state(tlp_ctx* ctx, int root, void* stream);
/* Fill a 128-byte buffer with a fresh ncclUniqueId (rank 0 only). */
tlp_status tlp_get_unique_id(void* nccl_id_out);

/* ---- (1) tokenizer, P:215-225 + P:239 + P:273 ---------------------------
 * feats[n, r, c] (fp32 [N, L, E], device, row-major) =
 *   r < min(len_n, L):  c < T: (c == tau) ; T <= c < E: arg c-T (token or
 *   RN_f32(number)) or 0 past the last argument  -- then / scale[c]
 *   r >= len_n: 0.
 * Crops silently (R4).  Device errors: EMPTY_SEQ, UNKNOWN_TYPE, NONFINITE (kept
 * data only).  Requires tlp_set_norm_scales (token table optional: all names
 * -> 1 if unset). */
tlp_status tlp_encode(tlp_ctx* ctx, const tlp_seq_batch* in, int64_t N, float* feats, void* stream);

/* ---- (2) scoring, P:295 + P:355 ----------------------------------------
 * scores[n, t] (fp32 [N, n_tasks], device) = head_t(resblocks(attn(upsample(feats[n])))).
 * Per-candidate results do not depend on N or on the position of n (batch
 * invariance).  Requires tlp_set_params. */
tlp_status tlp_score(tlp_ctx* ctx, const float* feats, int64_t N, float* scores, void* stream);

/* ---- (3) training, P:182 + P:295-296 + P:355-362 ------------------------
 * One optimizer step on a batch of B candidates grouped into G contiguous
 * groups (subgraphs, R18): feats [B, L, E] device; labels [B, n_tasks] device
 * fp32 in (0,1], NaN = absent (MTL); group_off [G+1] HOST int64.
 * Forward, the configured loss (cfg.loss: LambdaRank R16, mean over the global
 * strict-pair count per task; or MSE, mean over the global present-label count
 * per task), backward, gradient allreduce when a communicator is set, Adam (R23).
 * loss_out: device fp32 scalar (sum over tasks of the per-task means; with a
 * communicator every rank receives the global loss). */
tlp_status tlp_train_step(tlp_ctx* ctx, const float* feats, const float* labels,
                          const int64_t* group_off, int32_t B, int32_t G,
                          float* loss_out, void* stream);
/* As tlp_train_step but without the Adam update (gradients via tlp_get_grads). */
tlp_status tlp_compute_grads(tlp_ctx* ctx, const float* feats, const float* labels,
                             const int64_t* group_off, int32_t B, int32_t G,
                             float* loss_out, void* stream);
/* The LambdaRank unit alone (R26): scores/labels [B, n_tasks] device; writes the
 * loss (device scalar) and dloss/dscores [B, n_tasks] (device).  Pair counts
 * are local (no communicator). */
tlp_status tlp_lambdarank(tlp_ctx* ctx, const float* scores, const float* labels,
                          const int64_t* group_off, int32_t B, int32_t G,
                          float* loss_out, float* dscores_out, void* stream);

/* The MSE unit alone (NEXT-3, MTL S:386-394, R41):
 * loss = sum_t (1/n_t) sum_{i: label present} (s_it - y_it)^2, n_t = present
 * labels of task t in the batch (a task with none contributes 0);
 * dscores = 2 (s - y) / n_t, 0 where the label is absent.  scores / labels /
 * dscores_out [B, n_tasks] device fp32, loss_out device fp32 scalar.  Counts
 * are local (no communicator). */
tlp_status tlp_mse(tlp_ctx* ctx, const float* scores, const float* labels, int32_t B,
                   float* loss_out, float* dscores_out, void* stream);

/* ---- (4) per-task top-k, P:182 + P:390 ----------------------------------
 * For task segment t = [task_off[t], task_off[t+1]) of `scores` (column `head`
 * of a row-major [*, score_stride] fp32 device array): the k best candidates by
 * (score desc, index asc), -0 == +0 (R15, R21).  idx_out [T, k] int64 device
 * (global index = shard_base + local row), val_out [T, k] fp32 device; a
 * segment shorter than k is padded with (-1, -inf).  task_off is HOST int64
 * [T+1].  NaN score -> NONFINITE device error.
 * With a communicator (world > 1) every rank passes its own shard (task_off
 * local, shard_base = global index of its row 0) and receives the merged global
 * top-k (one ncclAllGather of T*k (score, index) pairs, then the same
 * deterministic merge on every rank); T and k must agree across ranks. */
tlp_status tlp_topk(tlp_ctx* ctx, const float* scores, int32_t score_stride, int32_t head,
                    const int64_t* task_off, int32_t T, int32_t k, int64_t shard_base,
                    int64_t* idx_out, float* val_out, void* stream);

/* Merge of per-shard top-k lists (the second half of the sharded tlp_topk,
 * exposed for callers that gather the shards themselves): vals / idx are
 * [W, T, k] device arrays (shard r's tlp_topk output with its shard_base; pad
 * entries (-1, -inf) allowed); idx_out / val_out [T, k] device receive the
 * global top-k per task under the same total order (R21). */
tlp_status tlp_topk_merge(tlp_ctx* ctx, const float* vals, const int64_t* idx, int32_t W,
                          int32_t T, int32_t k, int64_t* idx_out, float* val_out, void* stream);

/* ---- one search round from host memory: (1) -> (2) -> (4) ---------------
 * The per-round call of the search loop ("the cost model ... predicts the
 * top-k candidates"): tlp_encode, tlp_score and tlp_topk over a batch of
 * N candidates held in HOST memory, with the top-k returned to HOST memory.
 *   host_in      tlp_seq_batch whose pointers are all HOST memory (page-locked
 *                for the copies to overlap the kernels; pageable is accepted
 *                and copied synchronously by the driver).  Not modified.
 *                Offsets as for tlp_encode; seq_off is checked in full
 *                (SHAPE), arg_off at the chunk boundaries.
 *   task_off     HOST int64 [T+1], candidate segments per task (as tlp_topk).
 *   head         score column ranked (0 <= head < n_tasks).
 *   shard_base   global index of candidate 0 (sharded rounds, as tlp_topk).
 *   chunks       1..64: the candidates are cut into about `chunks` ranges
 *                (multiples of 5 candidates; with chunks <= 62 the first two
 *                are a quarter and a half of the rest, a shorter pipeline
 *                fill); chunk c+1's host->device copy runs on an
 *                internal copy stream while chunk c is encoded and scored on
 *                `stream`.  The result does not depend on `chunks` (batch
 *                invariance, R34).
 *   idx_out / val_out  HOST [T, k] int64 / fp32 (page-locked for an
 *                asynchronous read-back), written by a copy ordered on `stream`.
 * Asynchronous on `stream`: outputs and the reuse of host_in are safe after
 * stream synchronisation or tlp_sync.  Device memory (a copy of the batch, one
 * chunk of features, N * n_tasks scores) is owned by the ctx and grows to the
 * largest round seen.  With a communicator the top-k is the merged global one
 * (as tlp_topk).  Errors: as tlp_encode / tlp_score / tlp_topk; ARG for chunks
 * outside [1, 64] or a null pointer. */
tlp_status tlp_search_round(tlp_ctx* ctx, const tlp_seq_batch* host_in, int64_t N,
                            const int64_t* task_off, int32_t T, int32_t k, int32_t head,
                            int64_t shard_base, int32_t chunks, int64_t* idx_out, float* val_out,
                            void* stream);

/* ---- NEXT-2 dataset scans: duplicates, P:276-278 ---------
 * Duplicate classes of feature matrices (§4.3 "8.56 million
 * different schedule primitive sequences in a total of 8.65 million tensor
 * programs"; R39): samples i, j are duplicates iff they lie in the same group
 * and their rows feats[i*row_len .. +row_len) are bitwise equal.
 *   feats      device fp32 [N, row_len] (row_len = L*E for tlp_encode output)
 *   group_off  HOST int64 [G+1], 0 = group_off[0] <= ... <= group_off[G] = N;
 *              pass G = 1, {0, N} for the global duplicate rate
 *   labels     device fp32 [N] finite and >= 0, or NULL (NONFINITE device error
 *              otherwise, returned by tlp_sync)
 *   keep_out   device int32 [N]: 1 iff i is the lowest index of its class
 *   label_out  device fp32 [N] or NULL (requires labels): the maximum label of
 *              i's class ("the optimal value of the labels ... can be used as
 *              the label") -- the kept sample carries it
 *   n_distinct_out  HOST: number of classes; duplicate rate = 1 - n/N.
 * Synchronous (returns after the count is on the host).  A 64-bit row hash
 * with full verification; collisions are detected and re-hashed, so the
 * result never depends on the hash. */
tlp_status tlp_dedup(tlp_ctx* ctx, const float* feats, int64_t N, int32_t row_len,
                     const int64_t* group_off, int32_t G, const float* labels, int32_t* keep_out,
                     float* label_out, int64_t* n_distinct_out, void* stream);

/* The top-k score metric (§6.1, R40):
 *   sum_g w_g min_{i in g} lat_i / sum_g w_g min_{i in topk_g} lat_i
 * with topk_g the min(k, |g|) best of group g by (score desc, index asc) as in
 * tlp_topk.  scores: column `head` of a row-major [N, score_stride] device
 * array; latency device fp32 [N] > 0; group_off HOST int64 [G+1]; weight HOST
 * fp64 [G]; 1 <= k <= 1024; empty groups contribute nothing.  *out (HOST) in
 * (0, 1].  Synchronous.  NaN score -> NONFINITE device error (as tlp_topk). */
tlp_status tlp_topk_score(tlp_ctx* ctx, const float* scores, int32_t score_stride, int32_t head,
                          const float* latency, const int64_t* group_off, const double* weight,
                          int32_t G, int32_t k, double* out, void* stream);

/* ---- NEXT-1: the synthetic Ansor-style tuning round --------
 * P:558 (§6.3): "Ansor will first generate some initial tensor programs for a
 * subgraph according to predefined rules.  Then use the cost model to pick out
 * potential tensor programs.  Use these potential tensor programs to generate
 * more tensor programs through the genetic algorithm and use the cost model
 * again to prune the poor performers.  This step will iterate multiple times."
 * "approximately 10,000 schedule primitive sequences ... for each
 * subgraph in one round".  The genetic operators, the counter-based random
 * numbers and the pruning follow DESIGN.md readings R44-R48.
 *
 * A search space holds S subgraphs.  Subgraph s is a skeleton sequence (one
 * candidate of `tmpl`) whose tunable arguments ("knobs") take a value from a
 * small domain; a candidate program is one domain index per knob (its "gene
 * vector", uint8).  Gene arrays are row-major [rows, G] uint8 with
 * G = tlp_ga_num_genes(ctx) (the largest knob count, <= 64; unused columns 0);
 * rows are grouped by subgraph: row s * n + c is candidate c of subgraph s. */
typedef struct {
  tlp_seq_batch tmpl;       /* HOST arrays: S skeletons, one candidate per subgraph */
  int32_t S;                /* subgraphs, >= 1 */
  const int64_t* knob_off;  /* HOST [S+1]: knobs of subgraph s = [knob_off[s], knob_off[s+1]), <= 64 */
  const int64_t* knob_arg;  /* HOST [K]: argument index (into tmpl's args) the knob sets, inside
                               its subgraph's skeleton */
  const int32_t* knob_grp;  /* HOST [K]: crossover group = ordinal of the knob's primitive among the
                               subgraph's knob-bearing primitives (0, non-decreasing, steps of <= 1) */
  const int64_t* dom_off;   /* HOST [K+1]: domain of knob k = entries [dom_off[k], dom_off[k+1]),
                               1..255 values */
  const double* dom_num;    /* HOST [D]: numeric value (knob on a Number argument) */
  const int32_t* dom_name;  /* HOST [D]: string index into tmpl's string table (knob on a NameParam
                               argument), -1 for numbers; must match the skeleton's arg_kind */
  int32_t id_base;          /* global id of subgraph 0: every random-number counter uses
                               id_base + s (R44), so a space sharded across ranks in contiguous
                               blocks draws exactly what the unsharded space draws */
} tlp_ga_space;

/* Copy a search space into ctx-owned device memory (replaces any previous one).
 * Validates every offset / index / kind (SHAPE or ARG on violation).  Sync. */
tlp_status tlp_ga_set_space(tlp_ctx* ctx, const tlp_ga_space* host_space);
/* Gene row width G of the ctx's space (0 if none set). */
int32_t tlp_ga_num_genes(const tlp_ctx* ctx);
/* Total primitives / arguments of n materialised candidates per subgraph
 * (sizes of tlp_ga_materialize's outputs). */
tlp_status tlp_ga_batch_size(tlp_ctx* ctx, int64_t n, int64_t* P_out, int64_t* A_out);

/* R45: genes_out [S*n, G] device <- n uniform candidates per subgraph drawn
 * with Philox4x64-10 (key (seed, 0x544C50), counter (c, s, round<<16, 1<<32|j/4)). */
tlp_status tlp_ga_init(tlp_ctx* ctx, int32_t n, uint64_t seed, int32_t round, uint8_t* genes_out,
                       void* stream);

/* R46/R47: child_out [S*n_child, G] device <- children of the survivors
 * pop [S*n_pop, G] (device, each subgraph's rows in rank order, best first);
 * pop_scores [S*n_pop] fp32 device: parents come from the finite-score prefix
 * of each subgraph's survivors.  0 <= p_cross, p_mut <= 1; iter >= 1. */
tlp_status tlp_ga_evolve(tlp_ctx* ctx, const uint8_t* pop, const float* pop_scores, int32_t n_pop,
                         int32_t n_child, double p_cross, double p_mut, uint64_t seed,
                         int32_t round, int32_t iter, uint8_t* child_out, void* stream);

/* The abstract primitive sequences of S*n gene rows (device, grouped by
 * subgraph, n per subgraph): skeleton s with knob k's argument set to its
 * domain value.  Outputs are caller-owned device arrays of the tlp_seq_batch
 * layout sized by tlp_ga_batch_size: seq_off [S*n+1], prim_type [P],
 * arg_off [P+1], arg_kind [A], arg_num [A], arg_name [A]; the string table is
 * the space's (str_blob / str_off as passed to tlp_ga_set_space). */
tlp_status tlp_ga_materialize(tlp_ctx* ctx, const uint8_t* genes, int64_t n, int64_t* seq_off,
                              uint8_t* prim_type, int64_t* arg_off, uint8_t* arg_kind,
                              double* arg_num, int32_t* arg_name, void* stream);

/* R48 duplicate dropping: within each subgraph's n rows of genes [S*n, G]
 * (device), every row equal to an earlier row of the same subgraph gets
 * scores[row] = -inf (scores [S*n] fp32 device, updated in place). */
tlp_status tlp_ga_drop_duplicates(tlp_ctx* ctx, const uint8_t* genes, int32_t n, float* scores,
                                  void* stream);

/* One tuning round of every subgraph entirely on the device (R48):
 * n_pop + n_child initial candidates -> materialise -> tlp_encode -> tlp_score
 * (column `head`) -> drop duplicates (-inf) -> keep the n_pop best (tlp_topk
 * order); then `iters` times: n_child children -> materialise -> encode ->
 * score -> pool = survivors + children -> drop duplicates -> keep n_pop best.
 * genes_out [S*n_pop, G] uint8 device and scores_out [S*n_pop] fp32 device
 * receive the final survivors in rank order (a -inf score marks a duplicate
 * survivor when a pool has fewer than n_pop distinct programs).  Requires
 * tlp_set_norm_scales and tlp_set_params; 1 <= n_pop <= 1024, n_child >= 1,
 * n_pop + n_child <= 16384, iters >= 0.  Device workspaces are ctx-owned and
 * grow to the largest round.  Asynchronous on `stream`. */
tlp_status tlp_ga_round(tlp_ctx* ctx, int32_t n_pop, int32_t n_child, int32_t iters,
                        double p_cross, double p_mut, uint64_t seed, int32_t round, int32_t head,
                        uint8_t* genes_out, float* scores_out, void* stream);

/* ---- training-data preparation, P:295-296 -------------------------------
 * label_i = min_{j in g} latency_j / latency_i per group g (fp64 quotient,
 * rounded to fp32).  latency [M] fp32 device > 0; group_off [G+1] HOST int64;
 * label_out [M] fp32 device. */
tlp_status tlp_normalize_labels(tlp_ctx* ctx, const float* latency, const int64_t* group_off,
                                int32_t G, float* label_out, void* stream);

/* Synchronise the device and return (then clear) the sticky device error.
 * With a communicator, first waits for the last collective the ctx enqueued,
 * at most TLP_NCCL_TIMEOUT_S seconds (default 300) while polling
 * ncclCommGetAsyncError; on a timeout or an asynchronous NCCL error the
 * communicator is aborted (ncclCommAbort, the ctx continues without one) and
 * TLP_ERR_NCCL is returned.  A training step that fails after entering its
 * collectives aborts the communicator the same way. */
tlp_status tlp_sync(tlp_ctx* ctx);
/* Number of kernels this ctx launched since creation (bench evidence). */
int64_t tlp_launch_count(const tlp_ctx* ctx);

/* Test hook for the tensor-core building block (not part of the hot path):
 * D[128, N] = bf16(A)[128, K] * bf16(B)[N, K]^T with fp32 accumulation through
 * one tcgen05.mma chain (UMMA descriptors, TMEM, tcgen05.ld).  A, B, D fp32
 * device row-major; 16 <= N <= 256, N % 16 == 0; 32 <= K <= 256, K % 32 == 0.
 * a_in_tmem != 0: A is staged in TMEM with tcgen05.st and read from there. */
tlp_status tlp_debug_umma(const float* A, const float* B, float* D, int32_t N, int32_t K,
                          int32_t a_in_tmem, void* stream);

/* Test hook for the bf16x3 tcgen05 GEMM of the bf16-context training path (R37:
 * fp32 operands split hi + lo, three bf16 MMAs per product, fp32 accumulation):
 * C = op(A) op(B) (op = transpose when ta / tb), fp32 device row-major with the
 * given leading dimensions (multiples of 4, 16-byte aligned pointers).  With
 * splits > 1, C receives `splits` partial products [splits, M, ldc] (fixed K
 * slices) instead of the sum. */
tlp_status tlp_debug_gemm(tlp_ctx* ctx, int32_t ta, int32_t tb, int64_t M, int64_t N, int64_t K,
                          const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                          int64_t ldc, int32_t splits, void* stream);

/* Test hook for the weight + bias gradient of one dense layer of the training
 * path: dWdb[0 : K*N] = X^T dY ([K, N] row-major, X [M][ldx] with K columns,
 * dY [M][ldy] with N columns, fp32 device) and dWdb[K*N : K*N + N] = the column
 * sums of dY -- the R24 (W, b) layout.  A bf16 ctx takes the kernels of its
 * training step (for 32 <= K, N <= 256 multiples of 32: TMA-fed kind::tf32
 * tiles per row slice + fixed-order slice reduction, R52). */
tlp_status tlp_debug_wgrad(tlp_ctx* ctx, int64_t M, int64_t K, int64_t N, const float* X, int64_t ldx,
                           const float* dY, int64_t ldy, float* dWdb, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TLP_H_ */
