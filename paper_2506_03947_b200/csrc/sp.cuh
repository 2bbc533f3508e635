// sp.cuh -- saddle-point inner solver (placeholder until the SP kernels land).
#pragma once
#include "aac_internal.cuh"

static int sp_apply(aac_ctx* ctx, int k, const double* r, double* z) {
  (void)k; (void)r; (void)z;
  return aac_fail(ctx, AAC_EINVAL, "AAC_SP inner solver not built yet");
}
static int sp_prepare(aac_ctx* ctx, int k) {
  (void)k;
  return aac_fail(ctx, AAC_EINVAL, "AAC_SP inner solver not built yet");
}
static int sp_gmres_precond(aac_ctx* ctx, int k) { return sp_prepare(ctx, k); }
static int sp_gmres_finalize(aac_ctx* ctx) { return sp_prepare(ctx, 0); }
static long long sp_paper_matvecs(const aac_ctx* ctx, int k) { return 2LL * (ctx->ell - 1) * k; }
static void sp_destroy(aac_ctx* ctx) { (void)ctx; }
