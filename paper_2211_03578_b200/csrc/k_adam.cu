// K12 Adam (reading R23: the paper names no optimizer; torch.optim.Adam
// semantics with bias correction, lr 1e-3, betas (0.9, 0.999), eps 1e-8 as in
// S:356).  One elementwise pass over the flat fp32 parameters.
#include "tlp_internal.cuh"

#include <cmath>

namespace {

__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g,
                            float* __restrict__ m, float* __restrict__ v, int64_t n, float lr,
                            float b1, float b2, float eps, float bc1, float bc2) {
  pdl_wait();  // TLP_LAUNCH_PDL
  pdl_trigger();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
  }
}

}  // namespace

tlp_status adam_launch(tlp_ctx* ctx, cudaStream_t s) {
  const tlp_config& c = ctx->cfg;
  ctx->adam_t += 1;
  const double bc1 = 1.0 - std::pow((double)c.beta1, (double)ctx->adam_t);
  const double bc2 = 1.0 - std::pow((double)c.beta2, (double)ctx->adam_t);
  const int64_t n = ctx->off.total;
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(n, 256), (int64_t)ctx->num_sms * 8);
  TLP_LAUNCH_PDL(adam_kernel, grid, 256, 0, s, ctx->d_params, ctx->d_grads, ctx->d_m, ctx->d_v, n, c.lr,
                                   c.beta1, c.beta2, c.eps, (float)bc1, (float)bc2);
  TLP_LAUNCH_CHECK();
  ctx->tc_dirty = true;
  return TLP_OK;
}
