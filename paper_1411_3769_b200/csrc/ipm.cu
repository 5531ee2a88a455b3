// ipm.cu -- polya_ipm_step: one predictor-corrector iteration of Algorithm 2.
#include "polya_internal.h"

void polya_ipm_free(polya::Ctx& c) { (void)c; }

extern "C" polya_status polya_ipm_step(polya_ctx* ctx, polya_ipm_state* st, polya_ipm_stats* stats, void* stream) {
  (void)st; (void)stats; (void)stream;
  if (!ctx) return POLYA_EINVAL;
  ctx->c.last_error = "polya_ipm_step: not built yet";
  return POLYA_EINVAL;
}
