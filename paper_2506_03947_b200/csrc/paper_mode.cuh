// paper_mode.cuh -- the paper-reproduction entry points: Dirichlet faces,
// explicit spectral bounds and the paper's outer CI. Textually included at the end of aac.cu.
#pragma once

// ------------------------------------------------------------------------------------------
// Paper-reproduction mode: Dirichlet boundary faces, explicit spectral
// bounds, the paper's outer CI.
static void invalidate_plans(aac_ctx* ctx) {
  for (auto& P : ctx->nc) P.method = 0;
  if (ctx->exact_n > 0) {                       // the DST factorisation belongs to the old operator
    cudaFree(ctx->d_S);
    cudaFree(ctx->d_lam1);
    cudaFree(ctx->d_T);
    ctx->d_S = ctx->d_lam1 = ctx->d_T = nullptr;
    ctx->exact_n = 0;
  }
  for (auto& ge : ctx->graphs) cudaGraphExecDestroy(ge.exec);
  ctx->graphs.clear();
  sp_destroy(ctx);
}

// ------------------------------------------------------------------------------------------
// Varying diagonal blocks (varying.cuh).
extern "C" int aac_set_blocks(aac_ctx* ctx, const double* kx, const double* ky, const double* kz) {
  if (!ctx) return aac_fail(nullptr, AAC_EINVAL, "aac_set_blocks: NULL ctx");
  if (ctx->nranks != 1 || ctx->host_tr || ctx->nccl_self)
    return aac_fail(ctx, AAC_EINVAL, "aac_set_blocks: one rank only");
  if (ctx->geo.dir) return aac_fail(ctx, AAC_EINVAL, "aac_set_blocks: the Neumann operator only");
  if (!kx || (ctx->dim >= 2 && !ky) || (ctx->dim >= 3 && !kz))
    return aac_fail(ctx, AAC_EINVAL, "aac_set_blocks: kappa arrays missing for a used axis");
  const long long nx = ctx->n[0], ny = ctx->n[1], nz = ctx->n[2];
  const long long sx = nz * ny * (nx - 1), sy = nz * (ny - 1) * nx, sz = (nz - 1) * ny * nx;
  aac_grid g{};
  g.dim = ctx->dim;
  g.n[0] = nx;
  g.n[1] = ny;
  g.n[2] = nz;
  g.rank = 0;
  g.nranks = 1;
  const long long wtot = ctx->wlen[0] + ctx->wlen[1] + ctx->wlen[2];
  std::vector<double> all((size_t)ctx->ell * wtot), mean((size_t)wtot, 0.0), hw;
  long long lens[3];
  for (int j = 0; j < ctx->ell; ++j) {
    double gm;
    if (!slab_weights(&g, kx + j * sx, ctx->dim >= 2 ? ky + j * sy : nullptr, ctx->dim >= 3 ? kz + j * sz : nullptr,
                      ctx->c, 0, ctx->dim == 1 ? 1 : ctx->n[ctx->dim - 1], hw, lens, &gm))
      return aac_fail(ctx, AAC_EINVAL, "aac_set_blocks: kappa of block %d must be finite and > 0", j);
    std::copy(hw.begin(), hw.end(), all.begin() + (size_t)j * wtot);
    for (long long i = 0; i < wtot; ++i) mean[i] += hw[i];
  }
  for (auto& v : mean) v /= ctx->ell;            // A_hat = mean_j A_j (affine in the weights)
  // Gershgorin bound of A_hat (reading R5); mu_min = 1 exactly (A_hat 1 = 1 under Neumann)
  const double* wx = mean.data();
  const double* wy = wx + ctx->wlen[0];
  const double* wz = wy + ctx->wlen[1];
  const Geo& G = ctx->geo;
  double gmax = 1.0;
  for (long long p = 0; p < G.N; ++p) {
    double sum = wx[p] + wx[p + 1];
    if (ctx->dim >= 2) sum += wy[p] + wy[p + G.nx];
    if (ctx->dim >= 3) sum += wz[p] + wz[p + G.S];
    gmax = fmax(gmax, 1.0 + 2.0 * sum);
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (!ctx->d_wblk && cudaMalloc((void**)&ctx->d_wblk, all.size() * sizeof(double)) != cudaSuccess) {
    ctx->d_wblk = nullptr;
    cudaGetLastError();
    return aac_fail(ctx, AAC_ENOMEM, "aac_set_blocks: allocation failed");
  }
  CUDA_TRY(ctx, cudaMemcpy(ctx->d_wblk, all.data(), all.size() * sizeof(double), cudaMemcpyHostToDevice));
  CUDA_TRY(ctx, cudaMemcpy(ctx->d_w, mean.data(), mean.size() * sizeof(double), cudaMemcpyHostToDevice));
  invalidate_plans(ctx);
  ctx->mu_min = 1.0;
  ctx->mu_max = gmax;
  ctx->varying = true;
  return AAC_OK;
}

extern "C" int aac_set_boundary(aac_ctx* ctx, double bx, double by, double bz) {
  if (!ctx) return aac_fail(nullptr, AAC_EINVAL, "aac_set_boundary: NULL ctx");
  if (ctx->varying) return aac_fail(ctx, AAC_EINVAL, "aac_set_boundary: not with varying blocks");
  if (!(bx >= 0.0 && by >= 0.0 && bz >= 0.0) || !std::isfinite(bx + by + bz))
    return aac_fail(ctx, AAC_EINVAL, "boundary face weights must be finite and >= 0");
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  Geo& g = ctx->geo;
  g.bdx = bx;
  g.bdy = ctx->dim >= 2 ? by : 0.0;
  g.bdz = ctx->dim >= 3 ? bz : 0.0;
  g.dir = (g.bdx != 0.0 || g.bdy != 0.0 || g.bdz != 0.0) ? 1 : 0;
  // Gershgorin bound with the boundary terms: max_P (1 + 2 sum_f w_f + sum_boundary bd)
  const long long tot = ctx->wlen[0] + ctx->wlen[1] + ctx->wlen[2];
  std::vector<double> hw(tot);
  CUDA_TRY(ctx, cudaMemcpy(hw.data(), ctx->d_w, tot * sizeof(double), cudaMemcpyDeviceToHost));
  const double* wx = hw.data();
  const double* wy = wx + ctx->wlen[0];
  const double* wz = wy + ctx->wlen[1];
  double gmax = 1.0;
  for (int z = 0; z < g.nz; ++z)
    for (int y = 0; y < g.ny; ++y)
      for (int x = 0; x < g.nx; ++x) {
        const long long p = ((long long)z * g.ny + y) * g.nx + x;
        double sum = wx[p] + wx[p + 1];
        if (ctx->dim >= 2) sum += wy[p] + wy[p + g.nx];
        if (ctx->dim >= 3) sum += wz[p] + wz[p + g.S];
        double d = g.bdx * ((x == 0) + (x == g.nx - 1));
        if (ctx->dim == 2) d += g.bdy * ((y == 0 && !g.has_lo) + (y == g.ny - 1 && !g.has_hi));
        if (ctx->dim == 3)
          d += g.bdy * ((y == 0) + (y == g.ny - 1)) + g.bdz * ((z == 0 && !g.has_lo) + (z == g.nz - 1 && !g.has_hi));
        gmax = fmax(gmax, 1.0 + 2.0 * sum + d);
      }
  if (ctx->nranks > 1) {
    ctx->h_stat[0] = gmax;
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_stat, ctx->h_stat, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    AAC_TRY(comm_allreduce(ctx, ctx->d_stat, 1, ncclMax));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_stat, ctx->d_stat, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    gmax = ctx->h_stat[0];
  }
  ctx->mu_min = 1.0;          // (a Dirichlet operator's mu_min is > 1: set it with aac_set_bounds)
  ctx->mu_max = gmax;
  invalidate_plans(ctx);
  return AAC_OK;
}

extern "C" int aac_set_bounds(aac_ctx* ctx, double mu_min, double mu_max) {
  if (!ctx) return aac_fail(nullptr, AAC_EINVAL, "aac_set_bounds: NULL ctx");
  if (!(mu_min > 0.0 && mu_max >= mu_min) || !std::isfinite(mu_max))
    return aac_fail(ctx, AAC_EINVAL, "need 0 < mu_min <= mu_max");
  if (!(pow(ctx->alpha, 1.0 / ctx->ell) < mu_min))
    return aac_fail(ctx, AAC_EINVAL, "alpha^{1/ell} must be below mu_min (Lemma lemma:Zalpha)");
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->mu_min = mu_min;
  ctx->mu_max = mu_max;
  invalidate_plans(ctx);
  return AAC_OK;
}

extern "C" int aac_ci(aac_ctx* ctx, int method, int k, const double* b, double* x, double lmin,
                      double lmax, double tol, int maxit, aac_gmres_info* info) {
  if (!ctx || !b || !x || b == x) return aac_fail(ctx, AAC_EINVAL, "aac_ci: bad pointers");
  NvtxRange nv("aac_ci");
  if (ctx->varying)   // the eigenvalue bounds behind the outer CI no longer hold
    return aac_fail(ctx, AAC_EINVAL, "aac_ci: varying blocks (aac_set_blocks) need GMRES, not CI (PAPER.md:991)");
  if (method != AAC_NONE && method != AAC_NC1 && method != AAC_NC2 && method != AAC_SP && method != AAC_EXACT)
    return aac_fail(ctx, AAC_EINVAL, "unknown method %d", method);
  if ((method == AAC_NC1 || method == AAC_NC2 || method == AAC_SP) && k < 1)
    return aac_fail(ctx, AAC_EINVAL, "k must be >= 1");
  if (!(lmin > 0.0 && lmax >= lmin) || !std::isfinite(lmax))
    return aac_fail(ctx, AAC_EINVAL, "need 0 < lmin <= lmax");
  if (!(tol >= 0.0) || maxit < 1) return aac_fail(ctx, AAC_EINVAL, "need tol >= 0, maxit >= 1");
  if (method == AAC_SP && ctx->geo.dir) return aac_fail(ctx, AAC_EINVAL, "AAC_SP needs the Neumann operator");
  if (method != AAC_NONE) AAC_TRY(check_alpha(ctx));
  StreamScope ss(ctx);
  const long long L = (long long)ctx->ell * ctx->geo.N;
  const long long sweeps0 = ctx->sweeps;
  double* xp = ctx->d_V;            // chi_{p-1}
  double* r = ctx->d_V + L;         // b - calA chi_p
  double* z = ctx->d_Z;             // P^{-1} r
  double* y = ctx->d_W;             // calA chi_p
  const unsigned nb = (unsigned)std::min<long long>(ctx->num_sms * 4, grid1d(L, 256));
  CUDA_TRY(ctx, cudaMemsetAsync(x, 0, L * sizeof(double), ctx->stream));
  CUDA_TRY(ctx, cudaMemsetAsync(xp, 0, L * sizeof(double), ctx->stream));
  CUDA_TRY(ctx, cudaMemsetAsync(y, 0, L * sizeof(double), ctx->stream));
  auto resid = [&](double* out) -> int {        // r = b - y, ||r||^2 -> host
    LAUNCH(ctx, KID_AXPY, 24.0 * L, k_ci_resid<<<nb, 256, 0, ctx->stream>>>(b, y, r, L, ctx->d_part));
    LAUNCH(ctx, KID_REDUCE, 0, k_sum<<<1, 256, 0, ctx->stream>>>(ctx->d_part, nb, ctx->d_stat));
    AAC_TRY(comm_allreduce(ctx, ctx->d_stat, 1, ncclSum));
    AAC_TRY(publish(ctx, ctx->d_stat, ctx->h_stat, sizeof(double)));   // (no copy engine, as aac_gmres)
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    *out = sqrt(ctx->h_stat[0]);
    return AAC_OK;
  };
  double bn = 0.0, rn = 0.0;
  AAC_TRY(resid(&bn));                           // r_0 = b
  if (method == AAC_SP) AAC_TRY(sp_prepare(ctx, k));
  if (method == AAC_EXACT) AAC_TRY(exact_prepare(ctx));
  int alloc_sum = 0;
  if (method == AAC_NC1 || method == AAC_NC2 || method == AAC_SP) {
    int al[AAC_MAX_ELL];
    allocation(ctx, method, k, al);
    for (int j = 0; j < ctx->ell; ++j) alloc_sum += al[j];
  }
  const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin);
  double rho = 0.0;
  int p = 0;
  rn = bn;
  bool conv = bn == 0.0;
  for (; p < maxit && !conv; ++p) {
    const double* zp = r;
    if (method == AAC_NC1 || method == AAC_NC2) {
      AAC_TRY(nc_apply(ctx, method, k, r, z, false));
      zp = z;
    } else if (method == AAC_EXACT) {
      AAC_TRY(exact_apply(ctx, r, z, false, 0));
      zp = z;
    } else if (method == AAC_SP) {
      const Dft D = make_dft(ctx);
      const long long N = ctx->geo.N;
      if (ctx->ell <= 10)
        LAUNCH(ctx, KID_FWD, 16.0 * L, (k_forward<10><<<grid1d(N, 256), 256, 0, ctx->stream>>>(N, D, r, ctx->d_what)));
      else
        LAUNCH(ctx, KID_FWD, 16.0 * L, (k_forward<16><<<grid1d(N, 256), 256, 0, ctx->stream>>>(N, D, r, ctx->d_what)));
      AAC_TRY(sp_solve(ctx, k, z, 0, nullptr));
      zp = z;
    }
    double a, c;
    if (p == 0 || delta == 0.0) {
      a = 0.0;
      c = 1.0 / theta;
      rho = delta / theta;
    } else {
      const double rho_new = 1.0 / (2.0 * theta / delta - rho);
      a = rho_new * rho;
      c = 2.0 * rho_new / delta;
      rho = rho_new;
    }
    LAUNCH(ctx, KID_AXPY, 32.0 * L, k_ci_update<<<nb, 256, 0, ctx->stream>>>(x, xp, zp, a, c, L));
    AAC_TRY(matvec_impl(ctx, x, y));
    AAC_TRY(resid(&rn));
    conv = rn < tol * bn;
  }
  if (info) {
    info->iters = p;
    info->converged = conv ? 1 : 0;
    info->relres_est = bn > 0.0 ? rn / bn : 0.0;
    info->relres_true = info->relres_est;
    info->matvecs_paper_units = (long long)p * (ctx->ell + (method == AAC_SP ? sp_paper_matvecs(ctx, k) : alloc_sum));
    info->stencil_sweeps = ctx->sweeps - sweeps0;
  }
  return conv ? AAC_OK : AAC_ENOCONV;
}
