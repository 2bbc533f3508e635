// exact_host.cuh -- host side of AAC_EXACT: the DST-I factorisation of the
// paper's operator and the exact P_alpha^{-1} apply (fp64 tensor-core GEMMs of exact.cuh). Textually
// included by aac.cu (one translation unit), after the NC helpers it uses.
#pragma once

// ------------------------------------------------------------------------------------------
// Exact P_alpha for the paper's operator (exact.cuh).
static int exact_prepare(aac_ctx* ctx) {
  if (ctx->exact_n > 0) return AAC_OK;
  const Geo& g = ctx->geo;
  if (ctx->dim != 2 || ctx->nranks != 1 || g.nx != g.ny || !g.dir)
    return aac_fail(ctx, AAC_EINVAL, "AAC_EXACT needs the paper's operator: 2D, square, one rank, Dirichlet faces");
  const int n = g.nx;
  const long long tot = ctx->wlen[0] + ctx->wlen[1];
  std::vector<double> hw(tot);
  CUDA_TRY(ctx, cudaMemcpy(hw.data(), ctx->d_w, tot * sizeof(double), cudaMemcpyDeviceToHost));
  const double w = hw[1];                       // wx of (x=1, y=0): an interior face
  auto same = [&](double v) { return fabs(v - w) <= 1e-12 * fabs(w); };
  bool ok = same(g.bdx) && same(g.bdy);
  for (int y = 0; y < n && ok; ++y)
    for (int x = 0; x < n && ok; ++x) {
      const long long p = (long long)y * n + x;
      if (x > 0) ok = ok && same(hw[p]);
      if (y > 0) ok = ok && same(hw[ctx->wlen[0] + p]);
    }
  if (!ok)
    return aac_fail(ctx, AAC_EINVAL,
                    "AAC_EXACT needs a constant face weight w on every interior and Dirichlet boundary face");
  std::vector<double> S((size_t)n * n), lam(n);
  const double sc = sqrt(2.0 / (n + 1));
  for (int i = 0; i < n; ++i) {
    const double si = sin(M_PI * (i + 1) / (2.0 * (n + 1)));
    lam[i] = w * 4.0 * si * si;
    for (int j = 0; j < n; ++j) S[(size_t)i * n + j] = sc * sin(M_PI * (double)(i + 1) * (j + 1) / (n + 1));
  }
  const long long L = (long long)ctx->ell * n * n;
  if (cudaMalloc((void**)&ctx->d_S, (size_t)n * n * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void**)&ctx->d_lam1, (size_t)n * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void**)&ctx->d_T, (size_t)L * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    return aac_fail(ctx, AAC_ENOMEM, "AAC_EXACT workspace allocation failed");
  }
  CUDA_TRY(ctx, cudaMemcpy(ctx->d_S, S.data(), S.size() * sizeof(double), cudaMemcpyHostToDevice));
  CUDA_TRY(ctx, cudaMemcpy(ctx->d_lam1, lam.data(), lam.size() * sizeof(double), cudaMemcpyHostToDevice));
  CUDA_TRY(ctx, cudaDeviceSynchronize());
  ctx->exact_n = n;
  return AAC_OK;
}

// C_q = A_q B_q for the ell planes (row-major n x n; S = S^T, stride 0 = the shared S)
static int gemm_planes(aac_ctx* ctx, const double* A, long long sa, const double* B, long long sb, double* C,
                       const IterState* st) {
  const int n = ctx->exact_n;
  const unsigned mt = (unsigned)((n + DG_T - 1) / DG_T);
  ctx->next_flops = 2.0 * ctx->ell * (double)n * n * n;
  // CTA tile 64 x 32 by default: more, smaller tiles fill the SMs more evenly than 64 x 64
  // (n = 500, ell = 10: 1280 CTAs over 3-4 resident per SM instead of 640)
  static const int tn = getenv("AAC_DST_TN") ? atoi(getenv("AAC_DST_TN")) : 32;
  if (tn == 64)
    LAUNCH(ctx, KID_SWEEP, 8.0 * ctx->ell * 3.0 * n * n,
           k_dst_gemm<64><<<dim3((n + 63) / 64, mt, ctx->ell), 128, 0, ctx->stream>>>(n, A, sa, B, sb, C,
                                                                                       (long long)n * n, st));
  else
    LAUNCH(ctx, KID_SWEEP, 8.0 * ctx->ell * 3.0 * n * n,
           k_dst_gemm<32><<<dim3((n + 31) / 32, mt, ctx->ell), 128, 0, ctx->stream>>>(n, A, sa, B, sb, C,
                                                                                       (long long)n * n, st));
  return AAC_OK;
}

static int exact_apply(aac_ctx* ctx, const double* r, double* zbase, bool gmres_mode, int host_j) {
  AAC_TRY(exact_prepare(ctx));
  const int n = ctx->exact_n, ell = ctx->ell, h = ell / 2;
  const long long N = ctx->geo.N, L = (long long)ell * N, NN = (long long)n * n;
  const double V = 8.0 * L;
  const Dft D = make_dft(ctx);
  const IterState* st = gmres_mode ? ctx->d_st : nullptr;
  if (gmres_mode) {
    const int rc = forward_step(ctx, (host_j == 0 ? 2 : host_j + 3) * V);
    if (rc != AAC_OK) return rc;
  } else if (ell <= 10) {
    LAUNCH(ctx, KID_FWD, 2 * V, (k_forward<10><<<grid1d(N, 256), 256, 0, ctx->stream>>>(N, D, r, ctx->d_what)));
  } else {
    LAUNCH(ctx, KID_FWD, 2 * V, (k_forward<16><<<grid1d(N, 256), 256, 0, ctx->stream>>>(N, D, r, ctx->d_what)));
  }
  double* X = ctx->d_X;
  // DST both sides: T = S W, X = T S; divide by mu - Lambda_k; back: T = S X, X = T S
  AAC_TRY(gemm_planes(ctx, ctx->d_S, 0, ctx->d_what, NN, ctx->d_T, st));
  AAC_TRY(gemm_planes(ctx, ctx->d_T, NN, ctx->d_S, 0, X, st));
  ExactShifts Sh{};
  for (int kb = 0; kb <= h; ++kb) shift_of_block(ctx, kb, &Sh.lr[kb], &Sh.li[kb]);
  LAUNCH(ctx, KID_SWEEP, 2 * V, k_exact_scale<<<grid1d(NN, 256), 256, 0, ctx->stream>>>(n, ell, ctx->d_lam1, X, Sh, st));
  AAC_TRY(gemm_planes(ctx, ctx->d_S, 0, X, NN, ctx->d_T, st));
  AAC_TRY(gemm_planes(ctx, ctx->d_T, NN, ctx->d_S, 0, X, st));
  NcFinal F{};
  for (int kb = 0; kb <= h; ++kb) {
    F.src[kb] = X + (long long)plane_of_block(ell, kb) * N;
    F.tr[kb] = 1.0;
    F.ti[kb] = 0.0;
  }
  return run_inverse(ctx, D, F, zbase, gmres_mode ? L : 0, st);
}

