// aac.cu -- libaac host side: the C ABI of include/aac.h (sm_100a, fp64).
//
// Call stacks:
//   aac_gmres  -> per Arnoldi step: aac_precond_apply -> aac_matvec -> CGS2 (3 passes)
//                 -> device Givens -> host poll of |g_{j+1}|/beta
//   aac_precond_apply (NC) -> k_forward -> (P_max - 1) x k_sweep -> k_inverse
#include <complex>
#include <cstdarg>
#include <mutex>

#include "aac_internal.cuh"
#include "comm.cuh"
#include "krylov.cuh"
#include "nc.cuh"
#include "sp.cuh"
#include "stencil.cuh"

static thread_local std::string g_last_err;

int aac_fail(aac_ctx* ctx, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  g_last_err = buf;
  return code;
}

static const char* kKernelNames[KID_COUNT] = {
    "matvec", "forward_dft", "cheb_sweep", "inverse_dft", "multidot", "cgs_update",
    "reduce", "scalar", "axpy", "sp_stencil", "sp_multigrid", "sp_vector", "halo"};

LaunchScope::LaunchScope(aac_ctx* c, int kid, double bytes) : ctx(c), id(kid) {
  ctx->launches++;
  ctx->prof_n[kid]++;
  ctx->prof_bytes[kid] += bytes;
  if (ctx->prof) {
    if (ctx->ev_pool.size() < 2) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->ev_pool.push_back(e);
      }
    }
    a = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    b = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    cudaEventRecord(a, ctx->stream);
  }
}

int LaunchScope::end() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return aac_fail(ctx, AAC_ECUDA, "launch of %s failed: %s", kKernelNames[id],
                    cudaGetErrorString(e));
  if (ctx->prof) {
    cudaEventRecord(b, ctx->stream);
    ctx->prof_recs.push_back({id, a, b});
  }
  return AAC_OK;
}

// Fold finished event pairs into the per-kernel totals and recycle the events.
static int prof_collect(aac_ctx* ctx) {
  if (ctx->prof_recs.empty()) return AAC_OK;
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  for (auto& r : ctx->prof_recs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    ctx->prof_ms[r.id] += ms;
    ctx->ev_pool.push_back(r.a);
    ctx->ev_pool.push_back(r.b);
  }
  ctx->prof_recs.clear();
  return AAC_OK;
}

// ------------------------------------------------------------------------------------------
extern "C" int aac_slab_range(int64_t n, int nranks, int rank, int64_t* lo, int64_t* hi) {
  if (nranks < 1 || rank < 0 || rank >= nranks || n < nranks || !lo || !hi)
    return aac_fail(nullptr, AAC_EINVAL, "aac_slab_range: bad arguments (n=%lld, nranks=%d, rank=%d)",
                    (long long)n, nranks, rank);
  const int64_t base = n / nranks, rem = n % nranks;
  *lo = rank * base + (rank < rem ? rank : rem);
  *hi = *lo + base + (rank < rem ? 1 : 0);
  return AAC_OK;
}

static bool finite_pos(double v) { return std::isfinite(v) && v > 0.0; }

extern "C" int aac_setup(const aac_grid* g, const double* kx, const double* ky, const double* kz,
                         double c, int ell, double alpha, int max_krylov, void* cuda_stream,
                         const void* nccl_id, aac_ctx** out) {
  if (!g || !out) return aac_fail(nullptr, AAC_EINVAL, "aac_setup: NULL grid or out");
  *out = nullptr;
  if (g->dim < 1 || g->dim > 3) return aac_fail(nullptr, AAC_EINVAL, "dim must be 1, 2 or 3");
  if (ell < 2 || ell > AAC_MAX_ELL || (ell & 1))
    return aac_fail(nullptr, AAC_EINVAL, "ell must be even, 2 <= ell <= %d (PAPER.md:47)", AAC_MAX_ELL);
  if (!(alpha > 0.0 && alpha < 1.0))
    return aac_fail(nullptr, AAC_EINVAL,
                    "alpha must lie in (0,1): mu_min(A) = 1 under Neumann BCs and P_alpha is "
                    "singular at alpha = mu^ell (Lemma lemma:Zalpha, PAPER.md:120)");
  if (!(c >= 0.0) || !std::isfinite(c)) return aac_fail(nullptr, AAC_EINVAL, "c must be finite and >= 0");
  if (max_krylov < 1) return aac_fail(nullptr, AAC_EINVAL, "max_krylov must be >= 1");
  const long long nx = g->n[0], ny = g->dim >= 2 ? g->n[1] : 1, nz = g->dim >= 3 ? g->n[2] : 1;
  if (nx < 2 || (g->dim >= 2 && ny < 2) || (g->dim >= 3 && nz < 2))
    return aac_fail(nullptr, AAC_EINVAL, "every used axis needs n >= 2");
  if (g->dim == 1 && g->nranks != 1) return aac_fail(nullptr, AAC_EINVAL, "1D problems run on one rank");
  const long long nslab = g->dim == 2 ? ny : (g->dim == 3 ? nz : 1);
  int64_t lo = 0, hi = nslab;
  if (g->dim > 1 && aac_slab_range(nslab, g->nranks, g->rank, &lo, &hi) != AAC_OK)
    return AAC_EINVAL;
  if (g->nranks > 1 && hi - lo < 1) return aac_fail(nullptr, AAC_EINVAL, "empty slab");
  if (!kx || (g->dim >= 2 && !ky) || (g->dim >= 3 && !kz))
    return aac_fail(nullptr, AAC_EINVAL, "kappa arrays missing for a used axis");

  aac_ctx* ctx = new aac_ctx();
  ctx->dim = g->dim;
  ctx->ell = ell;
  ctx->rank = g->rank;
  ctx->nranks = g->nranks;
  ctx->n[0] = nx;
  ctx->n[1] = ny;
  ctx->n[2] = nz;
  ctx->lo = lo;
  ctx->hi = hi;
  ctx->c = c;
  ctx->alpha = alpha;
  ctx->max_krylov = max_krylov;
  ctx->stream = (cudaStream_t)cuda_stream;
  cudaGetDevice(&ctx->device);

  Geo& G = ctx->geo;
  G.nx = (int)nx;
  G.ny = (int)(g->dim == 2 ? hi - lo : ny);
  G.nz = (int)(g->dim == 3 ? hi - lo : 1);
  G.N = (long long)G.nx * G.ny * G.nz;
  G.S = g->dim == 3 ? (long long)G.nx * G.ny : G.nx;
  G.has_lo = (g->nranks > 1 && g->rank > 0);
  G.has_hi = (g->nranks > 1 && g->rank < g->nranks - 1);
  const long long N = G.N;

  // Face weights w_f = c kappa_f n_a^2, lower-face layout with one padding layer (host build).
  const long long lenx = N + 1, leny = N + G.nx, lenz = N + G.S;
  std::vector<double> hw(lenx + leny + lenz, 0.0);
  double* wx = hw.data();
  double* wy = wx + lenx;
  double* wz = wy + leny;
  const double sx = c * (double)nx * (double)nx, sy = c * (double)ny * (double)ny,
               sz = c * (double)nz * (double)nz;
  bool bad = false;
  const long long z0 = g->dim == 3 ? lo : 0, y0 = g->dim == 2 ? lo : 0;
  for (long long zl = 0; zl < G.nz; ++zl)
    for (long long yl = 0; yl < G.ny; ++yl)
      for (long long x = 0; x < nx; ++x) {
        const long long p = (zl * G.ny + yl) * nx + x;
        const long long zg = z0 + zl, yg = y0 + yl;
        if (x > 0) {
          const double k = kx[(zg * ny + yg) * (nx - 1) + (x - 1)];
          bad |= !finite_pos(k);
          wx[p] = sx * k;
        }
        if (g->dim >= 2 && yg > 0) {
          const double k = ky[(zg * (ny - 1) + (yg - 1)) * nx + x];
          bad |= !finite_pos(k);
          wy[p] = sy * k;
        }
        if (g->dim == 3 && zg > 0) {
          const double k = kz[((zg - 1) * ny + yg) * nx + x];
          bad |= !finite_pos(k);
          wz[p] = sz * k;
        }
      }
  // the slab's top face (layer index = local extent) along the slab axis
  if (g->dim == 2 && hi < ny)
    for (long long x = 0; x < nx; ++x) {
      const double k = ky[(hi - 1) * nx + x];
      bad |= !finite_pos(k);
      wy[N + x] = sy * k;
    }
  if (g->dim == 3 && hi < nz)
    for (long long yx = 0; yx < G.S; ++yx) {
      const double k = kz[(hi - 1) * G.S + yx];
      bad |= !finite_pos(k);
      wz[N + yx] = sz * k;
    }
  if (bad) {
    delete ctx;
    return aac_fail(nullptr, AAC_EINVAL, "kappa must be finite and > 0 on every interior face");
  }
  // Gershgorin bound mu_max = max_P (1 + 2 sum_f w_f) (reading R5); mu_min = 1 exactly.
  double gmax = 1.0;
  for (long long p = 0; p < N; ++p) {
    double s = wx[p] + wx[p + 1];
    if (g->dim >= 2) s += wy[p] + wy[p + G.nx];
    if (g->dim >= 3) s += wz[p] + wz[p + G.S];
    gmax = fmax(gmax, 1.0 + 2.0 * s);
  }

  int rc = comm_init(ctx, nccl_id);
  if (rc != AAC_OK) {
    g_last_err = ctx->err;
    delete ctx;
    return rc;
  }

  // device allocations
  auto alloc = [&](double** p, long long n) -> bool {
    return cudaMalloc((void**)p, (size_t)(n > 0 ? n : 1) * sizeof(double)) == cudaSuccess;
  };
  const long long L = (long long)ell * N;
  const long long maxctas = (L + KRY_CHUNK - 1) / KRY_CHUNK;
  ctx->part_ctas = (int)maxctas;
  bool ok = alloc(&ctx->d_w, hw.size()) && alloc(&ctx->d_what, L) && alloc(&ctx->d_X, 3 * L) &&
            alloc(&ctx->d_tmp, L) && alloc(&ctx->d_V, (max_krylov + 1) * L) &&
            alloc(&ctx->d_Z, max_krylov * L) && alloc(&ctx->d_W, L) &&
            alloc(&ctx->d_halo, 2LL * ell * G.S) &&
            alloc(&ctx->d_part, maxctas * (max_krylov + 2)) &&
            alloc(&ctx->d_red, 4LL * (max_krylov + 2)) &&
            alloc(&ctx->d_H, (long long)(max_krylov + 1) * max_krylov) &&
            alloc(&ctx->d_giv, 4LL * (max_krylov + 2)) && alloc(&ctx->d_stat, 64);
  if (ok) ok = cudaMallocHost((void**)&ctx->h_stat, 64 * sizeof(double)) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    aac_destroy(ctx);
    return aac_fail(nullptr, AAC_ENOMEM, "device allocation failed (N=%lld, ell=%d, max_krylov=%d)", N,
                    ell, max_krylov);
  }
  G.wx = ctx->d_w;
  G.wy = ctx->d_w + lenx;
  G.wz = ctx->d_w + lenx + leny;
  if (cudaMemcpy(ctx->d_w, hw.data(), hw.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(ctx->d_halo, 0, 2LL * ell * G.S * sizeof(double)) != cudaSuccess) {
    aac_destroy(ctx);
    return aac_fail(nullptr, AAC_ECUDA, "setup copy failed");
  }
  // global Gershgorin max (all-reduce max over slabs)
  if (ctx->nranks > 1) {
    ctx->h_stat[0] = gmax;
    cudaMemcpy(ctx->d_stat, ctx->h_stat, sizeof(double), cudaMemcpyHostToDevice);
    rc = comm_allreduce(ctx, ctx->d_stat, 1, ncclMax);
    if (rc == AAC_OK && cudaStreamSynchronize(ctx->stream) == cudaSuccess)
      cudaMemcpy(&gmax, ctx->d_stat, sizeof(double), cudaMemcpyDeviceToHost);
    if (rc != AAC_OK) {
      g_last_err = ctx->err;
      aac_destroy(ctx);
      return rc;
    }
  }
  ctx->mu_min = 1.0;
  ctx->mu_max = gmax;
  *out = ctx;
  return AAC_OK;
}

extern "C" void aac_destroy(aac_ctx* ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->stream);
  sp_destroy(ctx);
  double* ptrs[] = {ctx->d_w, ctx->d_what, ctx->d_X, ctx->d_tmp, ctx->d_V, ctx->d_Z,
                    ctx->d_W, ctx->d_bx, ctx->d_halo, ctx->d_part, ctx->d_red, ctx->d_H,
                    ctx->d_giv, ctx->d_stat};
  for (double* p : ptrs)
    if (p) cudaFree(p);
  if (ctx->h_stat) cudaFreeHost(ctx->h_stat);
  for (auto& r : ctx->prof_recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  comm_destroy(ctx);
  delete ctx;
}

extern "C" const char* aac_last_error(const aac_ctx* ctx) {
  if (ctx && !ctx->err.empty()) return ctx->err.c_str();
  return g_last_err.c_str();
}

// ------------------------------------------------------------------------------------------
// calA apply
static int matvec_impl(aac_ctx* ctx, const double* x, double* y) {
  const Geo& g = ctx->geo;
  const int ell = ctx->ell;
  if (ctx->nranks > 1) {
    const double* planes[AAC_MAX_ELL];
    int qs[AAC_MAX_ELL];
    for (int j = 0; j < ell; ++j) {
      planes[j] = x + (long long)j * g.N;
      qs[j] = j;
    }
    AAC_TRY(comm_halo(ctx, planes, qs, ell));
  }
  const double* hlo = ctx->d_halo;
  const double* hhi = ctx->d_halo + (long long)ell * g.S;
  const double V = 8.0 * ell * g.N, C = 8.0 * ctx->dim * g.N;
  const unsigned grid = grid1d(g.N, 256);
  switch (ctx->dim) {
    case 1: LAUNCH(ctx, KID_MATVEC, 2 * V + C, k_matvec<1><<<grid, 256, 0, ctx->stream>>>(g, ell, x, y, hlo, hhi)); break;
    case 2: LAUNCH(ctx, KID_MATVEC, 2 * V + C, k_matvec<2><<<grid, 256, 0, ctx->stream>>>(g, ell, x, y, hlo, hhi)); break;
    default: LAUNCH(ctx, KID_MATVEC, 2 * V + C, k_matvec<3><<<grid, 256, 0, ctx->stream>>>(g, ell, x, y, hlo, hhi)); break;
  }
  ctx->sweeps += ell;
  return AAC_OK;
}

extern "C" int aac_matvec(aac_ctx* ctx, const double* x, double* y) {
  if (!ctx || !x || !y || x == y) return aac_fail(ctx, AAC_EINVAL, "aac_matvec: bad pointers");
  return matvec_impl(ctx, x, y);
}

// ------------------------------------------------------------------------------------------
// Inner Chebyshev plan: allocation (NC1 uniform / NC2 Algorithm 1) and coefficient tables.
static void allocation(const aac_ctx* ctx, int method, int k, int* out) {
  const int ell = ctx->ell;
  if (method == AAC_NC1 || method == AAC_SP) {
    for (int j = 0; j < ell; ++j) out[j] = k;
    return;
  }
  // Algorithm 1 with budget ell*k (reading R11)
  const double budget = (double)ell * (double)k;
  const double mu0 = ctx->mu_min, mu1 = ctx->mu_max;
  if (mu1 == mu0) {
    for (int j = 0; j < ell; ++j) out[j] = k > 1 ? k : 1;
    return;
  }
  double sig[AAC_MAX_ELL], r[AAC_MAX_ELL], tot = 0.0;
  const double root = pow(ctx->alpha, 1.0 / ell);
  for (int j = 0; j < ell; ++j) {
    const int jj = j < ell - j ? j : ell - j;          // reduced angle (conjugate pairs equal)
    const double re = root * cos(2.0 * M_PI * jj / ell);
    const double kap = (mu1 - re) / (mu0 - re);
    const double s = sqrt(kap);
    sig[j] = (s - 1.0) / (s + 1.0);
  }
  for (int j = 0; j < ell; ++j) {
    r[j] = log(sig[0]) / log(sig[j]);
    tot += r[j];
  }
  for (int j = 0; j < ell; ++j) {
    const int a = (int)floor(r[j] / tot * budget);
    out[j] = a < 1 ? 1 : a;
  }
}

static void shift_of_block(const aac_ctx* ctx, int kb, double* lr, double* li) {
  const int ell = ctx->ell, h = ell / 2;
  const double root = pow(ctx->alpha, 1.0 / ell);
  if (kb == 0) { *lr = root; *li = 0.0; return; }
  if (kb == h) { *lr = -root; *li = 0.0; return; }
  *lr = root * cos(2.0 * M_PI * kb / ell);          // Lambda_k = alpha^{1/ell} e^{-2 pi i k/ell}
  *li = -root * sin(2.0 * M_PI * kb / ell);
}

static const NcPlan& nc_plan(aac_ctx* ctx, int method, int k) {
  for (auto& P : ctx->nc)
    if (P.method == method && P.k == k) return P;
  NcPlan& P = ctx->nc[ctx->nc_next];
  ctx->nc_next ^= 1;
  const int ell = ctx->ell, h = ell / 2;
  int al[AAC_MAX_ELL];
  allocation(ctx, method, k, al);
  P.method = method;
  P.k = k;
  P.nblk = h + 1;
  const double delta = 0.5 * (ctx->mu_max - ctx->mu_min);
  P.pmax = 1;
  for (int kb = 0; kb <= h; ++kb) {
    P.p[kb] = delta == 0.0 ? 1 : al[kb];                 // delta = 0: x_1 is exact (R10)
    P.pmax = P.p[kb] > P.pmax ? P.p[kb] : P.pmax;
  }
  P.a_re.assign((size_t)P.nblk * P.pmax, 0.0);
  P.a_im = P.a_re; P.b_re = P.a_re; P.b_im = P.a_re;
  for (int kb = 0; kb <= h; ++kb) {
    double lr, li;
    shift_of_block(ctx, kb, &lr, &li);
    const std::complex<double> theta(0.5 * (ctx->mu_max + ctx->mu_min) - lr, -li);
    std::complex<double> rho_prev = delta / theta;
    for (int s = 1; s < P.p[kb]; ++s) {
      const std::complex<double> rho = 1.0 / (2.0 * theta / delta - rho_prev);
      const std::complex<double> a = rho * rho_prev, b = 2.0 * rho / delta;
      P.a_re[kb * P.pmax + s] = a.real();
      P.a_im[kb * P.pmax + s] = a.imag();
      P.b_re[kb * P.pmax + s] = b.real();
      P.b_im[kb * P.pmax + s] = b.imag();
      rho_prev = rho;
    }
  }
  return P;
}

static Dft make_dft(const aac_ctx* ctx) {
  Dft D{};
  const int ell = ctx->ell;
  D.ell = ell;
  for (int j = 0; j < ell; ++j) {
    D.g[j] = pow(ctx->alpha, (double)j / ell);
    D.gi[j] = 1.0 / D.g[j];
    D.c[j] = cos(2.0 * M_PI * j / ell);
    D.s[j] = sin(2.0 * M_PI * j / ell);
  }
  D.scale = 1.0 / sqrt((double)ell);
  return D;
}

static inline int plane_of_block(int ell, int kb) {
  const int h = ell / 2;
  return kb == 0 ? 0 : (kb == h ? ell - 1 : 2 * kb - 1);
}

static int nc_apply(aac_ctx* ctx, int method, int k, const double* r, double* z) {
  const NcPlan& P = nc_plan(ctx, method, k);
  const Geo& g = ctx->geo;
  const int ell = ctx->ell, h = ell / 2;
  const long long N = g.N, L = (long long)ell * N;
  const double V = 8.0 * L, C = 8.0 * ctx->dim * N;
  const Dft D = make_dft(ctx);
  const unsigned grid = grid1d(N, 256);
  LAUNCH(ctx, KID_FWD, 2 * V, k_forward<<<grid, 256, 0, ctx->stream>>>(N, D, r, ctx->d_what));
  double* X = ctx->d_X;
  auto slot = [&](int s, int q) { return X + (long long)(s % 3) * L + (long long)q * N; };
  const double* hlo = ctx->d_halo;
  const double* hhi = ctx->d_halo + (long long)ell * g.S;
  for (int t = 1; t < P.pmax; ++t) {
    NcSweep S{};
    S.nblk = h + 1;
    const double* planes[AAC_MAX_ELL];
    int qs[AAC_MAX_ELL], nh = 0, nplanes = 0;
    for (int kb = 0; kb <= h; ++kb) {
      NcBlk& B = S.b[kb];
      const int s = t - (P.pmax - P.p[kb]);          // aligned ends: block starts late
      if (s < 1) { B.kind = 0; continue; }
      const bool cplx = (kb != 0 && kb != h);
      const int q = plane_of_block(ell, kb);
      B.kind = cplx ? 2 : 1;
      B.q = q;
      B.first = (s == 1);
      B.xs = B.first ? nullptr : slot(s, q);
      B.xm = s <= 2 ? nullptr : slot(s - 1, q);
      B.xo = slot(s + 1, q);
      B.ar = P.a_re[kb * P.pmax + s]; B.ai = P.a_im[kb * P.pmax + s];
      B.br = P.b_re[kb * P.pmax + s]; B.bi = P.b_im[kb * P.pmax + s];
      shift_of_block(ctx, kb, &B.lr, &B.li);
      const std::complex<double> it = 1.0 / std::complex<double>(0.5 * (ctx->mu_max + ctx->mu_min) - B.lr, -B.li);
      B.tr = it.real();
      B.ti = cplx ? it.imag() : 0.0;
      const int np = cplx ? 2 : 1;
      for (int e = 0; e < np; ++e) {
        planes[nh] = (B.first ? ctx->d_what + (long long)q * N : slot(s, q)) + (long long)e * N;
        qs[nh++] = q + e;
      }
      nplanes += np;
    }
    AAC_TRY(comm_halo(ctx, planes, qs, nh));
    const double bytes = 8.0 * N * 4.0 * nplanes + C;
    switch (ctx->dim) {
      case 1: LAUNCH(ctx, KID_SWEEP, bytes, k_sweep<1><<<grid, 256, 0, ctx->stream>>>(g, S, ctx->d_what, hlo, hhi)); break;
      case 2: LAUNCH(ctx, KID_SWEEP, bytes, k_sweep<2><<<grid, 256, 0, ctx->stream>>>(g, S, ctx->d_what, hlo, hhi)); break;
      default: LAUNCH(ctx, KID_SWEEP, bytes, k_sweep<3><<<grid, 256, 0, ctx->stream>>>(g, S, ctx->d_what, hlo, hhi)); break;
    }
    ctx->sweeps += nplanes;
  }
  NcFinal F{};
  F.nblk = h + 1;
  for (int kb = 0; kb <= h; ++kb) {
    double lr, li;
    shift_of_block(ctx, kb, &lr, &li);
    const std::complex<double> it = 1.0 / std::complex<double>(0.5 * (ctx->mu_max + ctx->mu_min) - lr, -li);
    F.tr[kb] = it.real();
    F.ti[kb] = (kb != 0 && kb != h) ? it.imag() : 0.0;
    F.y[kb] = P.p[kb] == 1 ? nullptr : slot(P.p[kb], plane_of_block(ell, kb));
  }
  LAUNCH(ctx, KID_INV, 2 * V, k_inverse<<<grid, 256, 0, ctx->stream>>>(N, D, F, ctx->d_what, z));
  return AAC_OK;
}

extern "C" int aac_precond_apply(aac_ctx* ctx, int method, int k, const double* r, double* z) {
  if (!ctx || !r || !z || r == z) return aac_fail(ctx, AAC_EINVAL, "aac_precond_apply: bad pointers");
  if (k < 1) return aac_fail(ctx, AAC_EINVAL, "inner iteration count k must be >= 1");
  if (method == AAC_NC1 || method == AAC_NC2) return nc_apply(ctx, method, k, r, z);
  if (method == AAC_SP) return sp_apply(ctx, k, r, z);
  return aac_fail(ctx, AAC_EINVAL, "unknown method %d", method);
}

// ------------------------------------------------------------------------------------------
// Fixed-order reductions used by GMRES.
static int reduce_to(aac_ctx* ctx, int nctas, int nv, double* out) {
  LAUNCH(ctx, KID_REDUCE, 8.0 * nctas * nv,
         k_reduce<<<nv, 256, 0, ctx->stream>>>(ctx->d_part, nctas, nv, out));
  return comm_allreduce(ctx, out, nv, ncclSum);
}

static size_t red_smem(int nv) { return (size_t)(KRY_THREADS / 32) * (nv > 1 ? nv : 1) * sizeof(double); }

// out[0] = ||w - coef_sign*sum coef_i V_i||^2 ; optional store into w_out
static int norm2_update(aac_ctx* ctx, const double* V, int nv, const double* coef, double sign,
                        const double* w_in, double* w_out, double* out) {
  const long long L = (long long)ctx->ell * ctx->geo.N;
  const int nctas = (int)((L + KRY_CHUNK - 1) / KRY_CHUNK);
  const double bytes = 8.0 * L * (nv + 1 + (w_out ? 1 : 0));
  LAUNCH(ctx, KID_UPD, bytes,
         k_update<MODE_NORM><<<nctas, KRY_THREADS, red_smem(1), ctx->stream>>>(
             V, L, nv, coef, sign, w_in, w_out, L, ctx->d_part));
  return reduce_to(ctx, nctas, 1, out);
}

static int gmres_impl(aac_ctx* ctx, int method, int k, const double* b, double* x, double rtol,
                      int maxit, aac_gmres_info* info) {
  if (maxit < 1 || maxit > ctx->max_krylov)
    return aac_fail(ctx, AAC_EINVAL, "maxit must be in [1, max_krylov=%d]", ctx->max_krylov);
  if (!(rtol >= 0.0)) return aac_fail(ctx, AAC_EINVAL, "rtol must be >= 0");
  if (k < 1) return aac_fail(ctx, AAC_EINVAL, "k must be >= 1");
  if (method != AAC_NC1 && method != AAC_NC2 && method != AAC_SP)
    return aac_fail(ctx, AAC_EINVAL, "unknown method %d", method);
  const long long N = ctx->geo.N, L = (long long)ctx->ell * N;
  const int ldh = ctx->max_krylov + 1;
  const int nctas = (int)((L + KRY_CHUNK - 1) / KRY_CHUNK);
  double* h1 = ctx->d_red;
  double* h2 = ctx->d_red + (ctx->max_krylov + 2);
  double* nr = ctx->d_red + 2 * (ctx->max_krylov + 2);
  double* cs = ctx->d_giv;
  double* sn = cs + (ctx->max_krylov + 2);
  double* gg = sn + (ctx->max_krylov + 2);
  double* yy = gg + (ctx->max_krylov + 2);
  double* st = ctx->d_stat;
  const long long sweeps0 = ctx->sweeps;
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_giv, 0, 4LL * (ctx->max_krylov + 2) * sizeof(double), ctx->stream));
  // beta = ||b||, v_0 = b / beta
  AAC_TRY(norm2_update(ctx, nullptr, 0, nullptr, 1.0, b, nullptr, nr));
  LAUNCH(ctx, KID_SCALAR, 0, k_beta<<<1, 1, 0, ctx->stream>>>(nr, st, gg));
  LAUNCH(ctx, KID_AXPY, 16.0 * L, k_scale<<<grid1d(L, 256), 256, 0, ctx->stream>>>(b, st + ST_INV, ctx->d_V, L));
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_stat, st, ST_COUNT * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  const double beta = ctx->h_stat[ST_BETA];
  int m = 0, converged = 0;
  double relres = 1.0;
  if (beta == 0.0) {
    CUDA_TRY(ctx, cudaMemsetAsync(x, 0, L * sizeof(double), ctx->stream));
    converged = 1;
    relres = 0.0;
  }
  long long paper_mv = 0;
  int alloc_sum = 0;
  {
    int al[AAC_MAX_ELL];
    allocation(ctx, method, k, al);
    for (int j = 0; j < ctx->ell; ++j) alloc_sum += al[j];
  }
  for (int j = 0; j < maxit && !converged; ++j) {
    const double* vj = ctx->d_V + (long long)j * L;
    double* zj = ctx->d_Z + (long long)j * L;
    AAC_TRY(aac_precond_apply(ctx, method, k, vj, zj));
    AAC_TRY(matvec_impl(ctx, zj, ctx->d_W));
    paper_mv += ctx->ell + (method == AAC_SP ? sp_paper_matvecs(ctx, k) : alloc_sum);
    // CGS2 pass 1: h1 = V^T w
    LAUNCH(ctx, KID_DOT, 8.0 * L * (j + 2),
           k_mdot<<<nctas, KRY_THREADS, red_smem(j + 1), ctx->stream>>>(ctx->d_V, L, j + 1, ctx->d_W, L, ctx->d_part));
    AAC_TRY(reduce_to(ctx, nctas, j + 1, h1));
    // pass 2: w -= V h1 ; h2 = V^T w
    LAUNCH(ctx, KID_UPD, 8.0 * L * (j + 3),
           k_update<MODE_DOTS><<<nctas, KRY_THREADS, red_smem(j + 1), ctx->stream>>>(
               ctx->d_V, L, j + 1, h1, 1.0, ctx->d_W, ctx->d_W, L, ctx->d_part));
    AAC_TRY(reduce_to(ctx, nctas, j + 1, h2));
    // pass 3: w -= V h2 ; ||w||^2
    AAC_TRY(norm2_update(ctx, ctx->d_V, j + 1, h2, 1.0, ctx->d_W, ctx->d_W, nr));
    LAUNCH(ctx, KID_SCALAR, 0, k_arnoldi<<<1, 1, 0, ctx->stream>>>(j, ldh, h1, h2, nr, ctx->d_H, cs, sn, gg, st));
    LAUNCH(ctx, KID_AXPY, 16.0 * L,
           k_scale<<<grid1d(L, 256), 256, 0, ctx->stream>>>(ctx->d_W, st + ST_INV, ctx->d_V + (long long)(j + 1) * L, L));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_stat, st, ST_COUNT * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    m = j + 1;
    relres = ctx->h_stat[ST_RELRES];
    if (ctx->h_stat[ST_HNORM] == 0.0 || relres <= rtol) converged = 1;
  }
  if (m > 0) {
    LAUNCH(ctx, KID_SCALAR, 0, k_backsub<<<1, 1, 0, ctx->stream>>>(m, ldh, ctx->d_H, gg, yy));
    LAUNCH(ctx, KID_AXPY, 8.0 * L * (m + 1),
           k_lincomb<<<grid1d(L, 256), 256, 0, ctx->stream>>>(ctx->d_Z, L, m, yy, x, L));
  }
  double rtrue = 0.0;
  if (info && beta > 0.0) {
    // true residual ||b - calA x|| / ||b|| (one extra apply, not counted as an iteration)
    AAC_TRY(matvec_impl(ctx, x, ctx->d_tmp));
    AAC_TRY(norm2_update(ctx, ctx->d_tmp, 1, st + ST_ONE, 1.0, b, nullptr, nr));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_stat + ST_NRM2, nr, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    rtrue = sqrt(ctx->h_stat[ST_NRM2]) / beta;
  }
  if (info) {
    info->iters = m;
    info->converged = converged;
    info->relres_est = relres;
    info->relres_true = rtrue;
    info->matvecs_paper_units = paper_mv;
    info->stencil_sweeps = ctx->sweeps - sweeps0;
  }
  return converged ? AAC_OK : AAC_ENOCONV;
}

extern "C" int aac_gmres(aac_ctx* ctx, int method, int k, const double* b, double* x, double rtol,
                         int maxit, aac_gmres_info* info) {
  if (!ctx || !b || !x || b == x) return aac_fail(ctx, AAC_EINVAL, "aac_gmres: bad pointers");
  return gmres_impl(ctx, method, k, b, x, rtol, maxit, info);
}

extern "C" int aac_gmres_host(aac_ctx* ctx, int method, int k, const double* b_host, double* x_host,
                              double rtol, int maxit, aac_gmres_info* info) {
  if (!ctx || !b_host || !x_host) return aac_fail(ctx, AAC_EINVAL, "aac_gmres_host: bad pointers");
  const long long L = (long long)ctx->ell * ctx->geo.N;
  if (!ctx->d_bx && cudaMalloc((void**)&ctx->d_bx, 2 * L * sizeof(double)) != cudaSuccess) {
    ctx->d_bx = nullptr;
    return aac_fail(ctx, AAC_ENOMEM, "staging allocation failed");
  }
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_bx, b_host, L * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  const int rc = gmres_impl(ctx, method, k, ctx->d_bx, ctx->d_bx + L, rtol, maxit, info);
  if (rc < 0) return rc;
  CUDA_TRY(ctx, cudaMemcpyAsync(x_host, ctx->d_bx + L, L * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return rc;
}

extern "C" int aac_query(aac_ctx* ctx, int method, int k, double* mu_min, double* mu_max, int* alloc,
                         int64_t* n_local) {
  if (!ctx) return aac_fail(nullptr, AAC_EINVAL, "aac_query: NULL ctx");
  if (mu_min) *mu_min = ctx->mu_min;
  if (mu_max) *mu_max = ctx->mu_max;
  if (n_local) *n_local = ctx->geo.N;
  if (alloc) {
    if (method != AAC_NC1 && method != AAC_NC2 && method != AAC_SP)
      return aac_fail(ctx, AAC_EINVAL, "unknown method %d", method);
    if (k < 1) return aac_fail(ctx, AAC_EINVAL, "k must be >= 1");
    allocation(ctx, method, k, alloc);
  }
  return AAC_OK;
}

// ------------------------------------------------------------------------------------------
extern "C" int aac_profile_enable(aac_ctx* ctx, int enable) {
  if (!ctx) return aac_fail(nullptr, AAC_EINVAL, "NULL ctx");
  AAC_TRY(prof_collect(ctx));
  ctx->prof = enable != 0;
  return AAC_OK;
}
extern "C" int aac_profile_count(void) { return KID_COUNT; }
extern "C" int aac_profile_read(aac_ctx* ctx, int id, const char** name, double* ms, long long* launches,
                                double* model_bytes) {
  if (!ctx || id < 0 || id >= KID_COUNT) return aac_fail(ctx, AAC_EINVAL, "bad profile id");
  AAC_TRY(prof_collect(ctx));
  if (name) *name = kKernelNames[id];
  if (ms) *ms = ctx->prof_ms[id];
  if (launches) *launches = ctx->prof_n[id];
  if (model_bytes) *model_bytes = ctx->prof_bytes[id];
  return AAC_OK;
}
extern "C" int aac_profile_reset(aac_ctx* ctx) {
  if (!ctx) return aac_fail(nullptr, AAC_EINVAL, "NULL ctx");
  AAC_TRY(prof_collect(ctx));
  for (int i = 0; i < KID_COUNT; ++i) {
    ctx->prof_ms[i] = 0;
    ctx->prof_n[i] = 0;
    ctx->prof_bytes[i] = 0;
  }
  return AAC_OK;
}
extern "C" long long aac_launch_count(const aac_ctx* ctx) { return ctx ? ctx->launches : 0; }
