// bf16 tcgen05 fused forward (placeholder until the tensor-core kernel lands).
#include "tlp_internal.cuh"

bool tc_supported(const tlp_config& c) {
  return c.L == 25 && c.E == 22 && c.T == 11 && c.hidden == 256 && c.n_up == 2 &&
         c.up_dims[0] == 128 && c.up_dims[1] == 256 && c.attn_heads == 8 && c.head_dim == 128;
}
tlp_status tc_prepare(tlp_ctx* ctx, cudaStream_t) {
  ctx->last_error = "bf16 tensor-core path not built yet";
  return TLP_ERR_UNSUPPORTED;
}
tlp_status tc_forward(tlp_ctx* ctx, const float*, int64_t, float*, cudaStream_t) {
  ctx->last_error = "bf16 tensor-core path not built yet";
  return TLP_ERR_UNSUPPORTED;
}
void tc_free(tlp_ctx*) {}
