// K1: the TLP tokenizer on the GPU.
//
//   f = F(p) ::= F1(tau) (F2(id) | F3(num))*       (fig 3_1_feature_extraction_abstract (b))
//   F1: type -> one-hot (T = 11 wide), F2: name -> token (R1/R2),
//   F3: number -> number (RN to fp32, R5); concatenated in original order;
//   post-processing: crop to L x E keeping the head (R4), zero padding (R7),
//   per-column division by the normalisation scale (R3, IEEE fp32 division --
//   this file must NOT be compiled with --use_fast_math / -prec-div=false).
//
// Two launches per batch:
//   resolve_tokens:     batch string table (U strings) -> token via the ctx hash
//                       table (FNV-1a 64, linear probing, byte-exact verification).
//   encode_warp_kernel: one warp per candidate; lane r builds row r in shared
//                       memory, then the warp streams the candidate's 2,200-byte
//                       fp32 block to HBM with coalesced 8-byte stores.
// tlp_fit_scales (R3's "normalization" fitted on the device): fit_scales_kernel
// computes the same un-normalised rows and reduces max |x| per column.
#include "tlp_internal.cuh"

#include <algorithm>
#include <cstring>

namespace {

__host__ __device__ inline uint64_t fnv1a(const uint8_t* p, int64_t n) {
  uint64_t h = 1469598103934665603ull;
  for (int64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h == 0 ? 1 : h;
}

__global__ void resolve_tokens(const uint8_t* __restrict__ blob, const int64_t* __restrict__ off,
                               int32_t U, const uint64_t* __restrict__ keys,
                               const int32_t* __restrict__ vals, const int32_t* __restrict__ sidx,
                               const uint8_t* __restrict__ tblob, const int64_t* __restrict__ toff,
                               uint32_t cap, int32_t* __restrict__ tokens) {
  int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= U) return;
  const uint8_t* s = blob + off[u];
  int64_t n = off[u + 1] - off[u];
  int32_t tok = 1;  // unknown (R1)
  if (cap) {
    uint64_t h = fnv1a(s, n);
    uint32_t slot = (uint32_t)h & (cap - 1);
    for (uint32_t probe = 0; probe < cap; ++probe) {
      uint64_t k = keys[slot];
      if (k == 0) break;
      if (k == h) {
        int32_t j = sidx[slot];
        const uint8_t* t = tblob + toff[j];
        int64_t tn = toff[j + 1] - toff[j];
        bool eq = tn == n;
        for (int64_t i = 0; eq && i < n; ++i) eq = t[i] == s[i];
        if (eq) { tok = vals[slot]; break; }
      }
      slot = (slot + 1) & (cap - 1);
    }
  }
  tokens[u] = tok;
}

// One warp per candidate: lane r < min(len, L) builds row r (one-hot, then its
// arguments in order, / scale) in shared memory; the warp then streams the
// candidate's L*E floats to HBM with coalesced 8-byte stores (a candidate
// block is 2,200 B, 8-byte aligned).
constexpr int kEncWarps = 8;

// R3's IEEE division x / s.  A zero numerator over a positive scale is
// answered directly (the quotient is x itself, sign included); otherwise the
// correctly rounded __fdiv_rn.  Most of a row's 22 entries are zeros (the
// one-hot's other columns, absent arguments), and a zero numerator sends
// __fdiv_rn down its slow path (FCHK), which dominated the kernel.
__device__ __forceinline__ float div_rn(float x, float s) {
  return (x == 0.f && s > 0.f) ? x : __fdiv_rn(x, s);
}
constexpr int kEncMaxElems = 32 * 64;  // L <= 32, E <= 64

template <int E_, int T_>
__global__ void __launch_bounds__(32 * kEncWarps) encode_warp_kernel(
    int64_t N, const int64_t* __restrict__ seq_off, const uint8_t* __restrict__ prim_type,
    const int64_t* __restrict__ arg_off, const uint8_t* __restrict__ arg_kind,
    const double* __restrict__ arg_num, const int32_t* __restrict__ arg_name,
    const int32_t* __restrict__ tokens, const float* __restrict__ scale, float* __restrict__ out,
    uint32_t* __restrict__ err, int L, int E, int T) {
  const int Er = E_ ? E_ : E, Tr = T_ ? T_ : T;
  extern __shared__ float enc_sm[];  // [kEncWarps][L*E] + scale[E]
  const int LE = L * Er;
  float* s_scale = enc_sm + kEncWarps * LE;
  if (threadIdx.x < Er) s_scale[threadIdx.x] = scale[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* buf = enc_sm + w * LE;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t n = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; n < N; n += nwarps) {
    const int64_t s0 = seq_off[n];
    const int64_t len = seq_off[n + 1] - s0;
    if (len <= 0 && lane == 0) atomicOr(err, DERR_EMPTY_SEQ);
    if (lane < L) {
      float* row = buf + lane * Er;
      int tau = -1, na = 0;
      int64_t a0 = 0;
      if (lane < len) {
        const int64_t p = s0 + lane;
        tau = prim_type[p];
        a0 = arg_off[p];
        na = (int)(arg_off[p + 1] - a0);
        if (tau >= Tr) {
          atomicOr(err, DERR_UNKNOWN_TYPE);
          tau = -1;  // row left zero
        }
      }
#pragma unroll
      for (int c = 0; c < Tr; ++c) row[c] = div_rn((tau >= 0 && c == tau) ? 1.f : 0.f, s_scale[c]);
      for (int a = 0; a < Er - Tr; ++a) {
        float v = 0.f;
        if (tau >= 0 && a < na) {
          const int64_t ai = a0 + a;
          if (arg_kind[ai]) {
            v = (float)tokens[arg_name[ai]];  // F2 (tokens < 2^24: exact)
          } else {
            const double d = arg_num[ai];
            v = __double2float_rn(d);  // F3, R5
            if (!isfinite(d) || !isfinite(v)) atomicOr(err, DERR_NONFINITE);
          }
        }
        row[Tr + a] = div_rn(v, s_scale[Tr + a]);  // R3: IEEE round-to-nearest division
      }
    }
    __syncwarp();
    float* o = out + n * (int64_t)LE;
    if ((LE & 1) == 0) {
      for (int j = lane; j < LE / 2; j += 32)
        reinterpret_cast<float2*>(o)[j] = reinterpret_cast<const float2*>(buf)[j];
    } else {
      for (int j = lane; j < LE; j += 32) o[j] = buf[j];
    }
    __syncwarp();
  }
}

// R3 on the device: max over the kept data of |x[n, r, c]| of the un-normalised
// rows (one-hot / RN_f32(number) / token), one thread per (candidate, row);
// per-block maxima in shared memory, then one atomicMax per column on the IEEE
// bits (non-negative floats order like their bit patterns, so the result does
// not depend on the reduction order).  Validation as in encode (kept data only).
__global__ void fit_scales_kernel(int64_t N, const int64_t* __restrict__ seq_off,
                                  const uint8_t* __restrict__ prim_type,
                                  const int64_t* __restrict__ arg_off,
                                  const uint8_t* __restrict__ arg_kind,
                                  const double* __restrict__ arg_num,
                                  const int32_t* __restrict__ arg_name,
                                  const int32_t* __restrict__ tokens, uint32_t* __restrict__ colmax,
                                  uint32_t* __restrict__ err, int L, int E, int T) {
  __shared__ uint32_t smax[64];
  if (threadIdx.x < 64) smax[threadIdx.x] = 0u;
  __syncthreads();
  const int64_t total = N * L;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i / L;
    const int r = (int)(i - n * L);
    const int64_t s0 = seq_off[n];
    const int64_t len = seq_off[n + 1] - s0;
    if (len <= 0) {
      if (r == 0) atomicOr(err, DERR_EMPTY_SEQ);
      continue;
    }
    if (r >= len) continue;  // padding row: zeros
    const int64_t p = s0 + r;
    const int tau = prim_type[p];
    if (tau >= T) {
      atomicOr(err, DERR_UNKNOWN_TYPE);
      continue;
    }
    atomicMax(&smax[tau], __float_as_uint(1.f));
    const int64_t a0 = arg_off[p];
    const int na = (int)(arg_off[p + 1] - a0);
    for (int a = 0; a < E - T && a < na; ++a) {
      const int64_t ai = a0 + a;
      float v;
      if (arg_kind[ai]) {
        v = (float)tokens[arg_name[ai]];
      } else {
        const double d = arg_num[ai];
        v = __double2float_rn(d);
        if (!isfinite(d) || !isfinite(v)) {
          atomicOr(err, DERR_NONFINITE);
          continue;
        }
      }
      atomicMax(&smax[T + a], __float_as_uint(fabsf(v)));
    }
  }
  __syncthreads();
  if (threadIdx.x < E && smax[threadIdx.x]) atomicMax(&colmax[threadIdx.x], smax[threadIdx.x]);
}

// scale[c] = max, or 1.0 where the column is all zero (R3)
__global__ void fit_scales_finish(const uint32_t* __restrict__ colmax, float* __restrict__ scale, int E) {
  const int c = threadIdx.x;
  if (c < E) scale[c] = colmax[c] ? __uint_as_float(colmax[c]) : 1.f;
}

}  // namespace

tlp_status build_token_table(tlp_ctx* ctx, const uint8_t* blob, const int64_t* off, int32_t n) {
  // Host-side construction (runtime plumbing), uploaded once.
  uint32_t cap = 0;
  if (n > 0) {
    cap = 16;
    while (cap < (uint32_t)n * 2u) cap <<= 1;
  }
  std::vector<uint64_t> keys(cap ? cap : 1, 0);
  std::vector<int32_t> vals(cap ? cap : 1, 0), sidx(cap ? cap : 1, -1);
  const int64_t nbytes = n > 0 ? off[n] : 0;
  for (int32_t i = 0; i < n; ++i) {
    const uint8_t* s = blob + off[i];
    int64_t len = off[i + 1] - off[i];
    uint64_t h = fnv1a(s, len);
    uint32_t slot = (uint32_t)h & (cap - 1);
    bool dup = false;
    while (keys[slot] != 0) {
      if (keys[slot] == h) {
        int32_t j = sidx[slot];
        if (off[j + 1] - off[j] == len && std::memcmp(blob + off[j], s, (size_t)len) == 0) {
          dup = true;  // first occurrence keeps its token (R1)
          break;
        }
      }
      slot = (slot + 1) & (cap - 1);
    }
    if (dup) continue;
    keys[slot] = h;
    vals[slot] = i + 2;
    sidx[slot] = i;
  }
  cudaFree(ctx->d_hkeys); cudaFree(ctx->d_hval); cudaFree(ctx->d_hstr);
  cudaFree(ctx->d_tblob); cudaFree(ctx->d_toff);
  ctx->d_hkeys = nullptr; ctx->d_hval = nullptr; ctx->d_hstr = nullptr;
  ctx->d_tblob = nullptr; ctx->d_toff = nullptr; ctx->hcap = 0;
  ctx->tok_n = 0; ctx->tok_bytes = 0;
  if (cap == 0) return TLP_OK;
  TLP_CUDA_TRY(cudaMalloc(&ctx->d_hkeys, cap * sizeof(uint64_t)));
  TLP_CUDA_TRY(cudaMalloc(&ctx->d_hval, cap * sizeof(int32_t)));
  TLP_CUDA_TRY(cudaMalloc(&ctx->d_hstr, cap * sizeof(int32_t)));
  TLP_CUDA_TRY(cudaMalloc(&ctx->d_tblob, nbytes > 0 ? nbytes : 1));
  TLP_CUDA_TRY(cudaMalloc(&ctx->d_toff, (n + 1) * sizeof(int64_t)));
  TLP_CUDA_TRY(cudaMemcpy(ctx->d_hkeys, keys.data(), cap * sizeof(uint64_t), cudaMemcpyHostToDevice));
  TLP_CUDA_TRY(cudaMemcpy(ctx->d_hval, vals.data(), cap * sizeof(int32_t), cudaMemcpyHostToDevice));
  TLP_CUDA_TRY(cudaMemcpy(ctx->d_hstr, sidx.data(), cap * sizeof(int32_t), cudaMemcpyHostToDevice));
  if (nbytes > 0) TLP_CUDA_TRY(cudaMemcpy(ctx->d_tblob, blob, nbytes, cudaMemcpyHostToDevice));
  TLP_CUDA_TRY(cudaMemcpy(ctx->d_toff, off, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
  ctx->hcap = cap;
  ctx->tok_n = n;
  ctx->tok_bytes = nbytes;
  return TLP_OK;
}

tlp_status encode_resolve(tlp_ctx* ctx, const tlp_seq_batch* in, cudaStream_t s) {
  if (in->U <= 0) return TLP_OK;
  TLP_CUDA_TRY(ctx->ws_tokens.ensure(sizeof(int32_t) * (size_t)in->U));
  resolve_tokens<<<(unsigned)cdiv(in->U, 128), 128, 0, s>>>(
      in->str_blob, in->str_off, in->U, ctx->d_hkeys, ctx->d_hval, ctx->d_hstr, ctx->d_tblob,
      ctx->d_toff, ctx->hcap, ctx->ws_tokens.as<int32_t>());
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

tlp_status encode_launch(tlp_ctx* ctx, const tlp_seq_batch* in, int64_t N, float* feats,
                         cudaStream_t s) {
  tlp_status st = encode_resolve(ctx, in, s);
  if (st != TLP_OK) return st;
  return encode_rows(ctx, in, N, feats, s);
}

tlp_status encode_rows(tlp_ctx* ctx, const tlp_seq_batch* in, int64_t N, float* feats,
                       cudaStream_t s) {
  const tlp_config& c = ctx->cfg;
  const int32_t* tokens = in->U > 0 ? ctx->ws_tokens.as<int32_t>() : nullptr;
  if (N == 0) return TLP_OK;
  const int64_t want = cdiv(N, kEncWarps);  // one warp per candidate
  const unsigned grid = (unsigned)(want < (int64_t)ctx->num_sms * 16 ? want : (int64_t)ctx->num_sms * 16);
  const size_t smem = ((size_t)kEncWarps * c.L * c.E + c.E) * sizeof(float);
  if (c.E == 22 && c.T == 11) {
    encode_warp_kernel<22, 11><<<grid, 32 * kEncWarps, smem, s>>>(
        N, in->seq_off, in->prim_type, in->arg_off, in->arg_kind, in->arg_num, in->arg_name,
        tokens, ctx->d_scale, feats, ctx->d_err, c.L, c.E, c.T);
  } else {
    encode_warp_kernel<0, 0><<<grid, 32 * kEncWarps, smem, s>>>(
        N, in->seq_off, in->prim_type, in->arg_off, in->arg_kind, in->arg_num, in->arg_name,
        tokens, ctx->d_scale, feats, ctx->d_err, c.L, c.E, c.T);
  }
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

tlp_status fit_scales_launch(tlp_ctx* ctx, const tlp_seq_batch* in, int64_t N, cudaStream_t s) {
  const tlp_config& c = ctx->cfg;
  tlp_status st = encode_resolve(ctx, in, s);
  if (st != TLP_OK) return st;
  const int32_t* tokens = in->U > 0 ? ctx->ws_tokens.as<int32_t>() : nullptr;
  TLP_CUDA_TRY(ctx->ws_misc.ensure(64 * sizeof(uint32_t)));
  uint32_t* colmax = ctx->ws_misc.as<uint32_t>();
  TLP_CUDA_TRY(cudaMemsetAsync(colmax, 0, 64 * sizeof(uint32_t), s));
  if (N > 0) {
    const int64_t want = cdiv(N * c.L, 256);
    const unsigned grid = (unsigned)std::min<int64_t>(want, (int64_t)ctx->num_sms * 8);
    fit_scales_kernel<<<grid, 256, 0, s>>>(N, in->seq_off, in->prim_type, in->arg_off, in->arg_kind,
                                           in->arg_num, in->arg_name, tokens, colmax, ctx->d_err,
                                           c.L, c.E, c.T);
    TLP_LAUNCH_CHECK();
  }
  fit_scales_finish<<<1, 64, 0, s>>>(colmax, ctx->d_scale, c.E);
  TLP_LAUNCH_CHECK();
  ctx->have_scales = true;
  return TLP_OK;
}
