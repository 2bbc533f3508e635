// aac.cu -- libaac host side: the C ABI of include/aac.h (sm_100a, fp64).
//
// Call stacks:
//   aac_gmres  -> per Arnoldi step: aac_precond_apply -> aac_matvec -> CGS2 (3 passes)
//                 -> device Givens -> host poll of |g_{j+1}|/beta
//   aac_precond_apply (NC) -> k_forward -> (P_max - 1) x k_sweep -> k_inverse
#include <algorithm>
#include <complex>
#include <cstdarg>
#include <cstdlib>
#include <type_traits>

#include "aac_internal.cuh"
#include "arnoldi.cuh"
#include "ci.cuh"
#include "exact.cuh"
#include "comm.cuh"
#include "krylov.cuh"
#include "nc.cuh"
#include "wave.cuh"
#include "wave_r.cuh"
#include "stencil.cuh"
#include "stencil_tile.cuh"
#include "stencil_rows.cuh"

// saddle-point inner solver (sp.cuh, included below once make_dft / shift_of_block exist)
static int sp_prepare(aac_ctx* ctx, int k);
static int sp_solve(aac_ctx* ctx, int k, double* zbase, long long zjs, const IterState* st);
static void sp_destroy(aac_ctx* ctx);
static long long sp_paper_matvecs(const aac_ctx* ctx, int k);

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
    "reduce", "scalar", "axpy", "sp_stencil", "sp_multigrid", "sp_vector", "halo", "arnoldi"};

LaunchScope::LaunchScope(aac_ctx* c, int kid, double bytes) : ctx(c), id(kid) {
  ctx->launches++;
  ctx->prof_n[kid]++;
  ctx->prof_bytes[kid] += bytes;
  ctx->prof_flops[kid] += ctx->next_flops;
  ctx->next_flops = 0.0;
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

// Local face weights of slab [lo, hi) in the lower-face layout (see Geo), each sub-array
// padded to 4 doubles: wx | wy | wz. Returns false on a non-positive / non-finite kappa.
static bool slab_weights(const aac_grid* g, const double* kx, const double* ky, const double* kz,
                         double c, long long lo, long long hi, std::vector<double>& hw,
                         long long lens[3], double* gershgorin) {
  const long long nx = g->n[0], ny = g->dim >= 2 ? g->n[1] : 1, nz = g->dim >= 3 ? g->n[2] : 1;
  const long long lny = g->dim == 2 ? hi - lo : ny, lnz = g->dim == 3 ? hi - lo : 1;
  const long long N = nx * lny * lnz, S = g->dim == 3 ? nx * lny : nx;
  auto pad4 = [](long long v) { return (v + 3) / 4 * 4; };
  lens[0] = pad4(N + 1);
  lens[1] = pad4(N + nx);
  lens[2] = pad4(N + S);
  hw.assign(lens[0] + lens[1] + lens[2], 0.0);
  double* wx = hw.data();
  double* wy = wx + lens[0];
  double* wz = wy + lens[1];
  const double sx = c * (double)nx * (double)nx, sy = c * (double)ny * (double)ny,
               sz = c * (double)nz * (double)nz;
  bool bad = false;
  const long long z0 = g->dim == 3 ? lo : 0, y0 = g->dim == 2 ? lo : 0;
  for (long long zl = 0; zl < lnz; ++zl)
    for (long long yl = 0; yl < lny; ++yl)
      for (long long x = 0; x < nx; ++x) {
        const long long p = (zl * lny + yl) * nx + x;
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
    for (long long yx = 0; yx < S; ++yx) {
      const double k = kz[(hi - 1) * S + yx];
      bad |= !finite_pos(k);
      wz[N + yx] = sz * k;
    }
  // Gershgorin bound mu_max = max_P (1 + 2 sum_f w_f) (reading R5); mu_min = 1 exactly.
  double gmax = 1.0;
  for (long long p = 0; p < N; ++p) {
    double sum = wx[p] + wx[p + 1];
    if (g->dim >= 2) sum += wy[p] + wy[p + nx];
    if (g->dim >= 3) sum += wz[p] + wz[p + S];
    gmax = fmax(gmax, 1.0 + 2.0 * sum);
  }
  *gershgorin = gmax;
  return !bad;
}

extern "C" int aac_slab_weights(const aac_grid* g, const double* kx, const double* ky, const double* kz,
                                double c, double* w_out, int64_t* lens_out, double* gershgorin) {
  if (!g || !kx || !lens_out || g->dim < 1 || g->dim > 3 || g->nranks < 1)
    return aac_fail(nullptr, AAC_EINVAL, "aac_slab_weights: bad arguments");
  const long long nslab = g->dim == 2 ? g->n[1] : (g->dim == 3 ? g->n[2] : 1);
  int64_t lo = 0, hi = nslab;
  if (g->dim > 1 && aac_slab_range(nslab, g->nranks, g->rank, &lo, &hi) != AAC_OK) return AAC_EINVAL;
  if (g->dim == 1 && g->nranks != 1) return aac_fail(nullptr, AAC_EINVAL, "1D problems run on one rank");
  std::vector<double> hw;
  long long lens[3];
  double gm = 1.0;
  const bool ok = slab_weights(g, kx, ky, kz, c, lo, hi, hw, lens, &gm);
  for (int a = 0; a < 3; ++a) lens_out[a] = lens[a];
  if (gershgorin) *gershgorin = gm;
  if (w_out) std::copy(hw.begin(), hw.end(), w_out);
  return ok ? AAC_OK : aac_fail(nullptr, AAC_EINVAL, "kappa must be finite and > 0 on every interior face");
}

static int setup_impl(const aac_grid* g, const double* kx, const double* ky, const double* kz,
                      double c, int ell, double alpha, int max_krylov, void* cuda_stream,
                      const void* nccl_id, const aac_host_transport* tr, aac_ctx** out);

extern "C" int aac_setup(const aac_grid* g, const double* kx, const double* ky, const double* kz,
                         double c, int ell, double alpha, int max_krylov, void* cuda_stream,
                         const void* nccl_id, aac_ctx** out) {
  return setup_impl(g, kx, ky, kz, c, ell, alpha, max_krylov, cuda_stream, nccl_id, nullptr, out);
}

extern "C" int aac_setup_host_transport(const aac_grid* g, const double* kx, const double* ky,
                                        const double* kz, double c, int ell, double alpha,
                                        int max_krylov, void* cuda_stream,
                                        const aac_host_transport* tr, aac_ctx** out) {
  if (!tr || !tr->allreduce || !tr->sendrecv)
    return aac_fail(nullptr, AAC_EINVAL, "aac_setup_host_transport: incomplete transport");
  return setup_impl(g, kx, ky, kz, c, ell, alpha, max_krylov, cuda_stream, nullptr, tr, out);
}

static int setup_impl(const aac_grid* g, const double* kx, const double* ky, const double* kz,
                      double c, int ell, double alpha, int max_krylov, void* cuda_stream,
                      const void* nccl_id, const aac_host_transport* tr, aac_ctx** out) {
  NvtxRange nv("aac_setup");
  if (!g || !out) return aac_fail(nullptr, AAC_EINVAL, "aac_setup: NULL grid or out");
  *out = nullptr;
  if (g->dim < 1 || g->dim > 3) return aac_fail(nullptr, AAC_EINVAL, "dim must be 1, 2 or 3");
  if (ell < 2 || ell > AAC_MAX_ELL || (ell & 1))
    return aac_fail(nullptr, AAC_EINVAL, "ell must be even, 2 <= ell <= %d (PAPER.md:47)", AAC_MAX_ELL);
  if (!(alpha > 0.0) || !std::isfinite(alpha))
    return aac_fail(nullptr, AAC_EINVAL, "alpha must be finite and > 0");
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

  // Face weights w_f = c kappa_f n_a^2 of this slab (host build) + local Gershgorin max.
  std::vector<double> hw;
  long long lens[3];
  double gmax = 1.0;
  if (!slab_weights(g, kx, ky, kz, c, lo, hi, hw, lens, &gmax)) {
    delete ctx;
    return aac_fail(nullptr, AAC_EINVAL, "kappa must be finite and > 0 on every interior face");
  }
  const long long lenx = lens[0], leny = lens[1];
  ctx->wlen[0] = lens[0];
  ctx->wlen[1] = lens[1];
  ctx->wlen[2] = lens[2];

  if (tr) {
    ctx->host_tr = true;
    ctx->htr = *tr;
  }
  int rc = comm_init(ctx, nccl_id);
  if (rc != AAC_OK) {
    g_last_err = ctx->err;
    delete ctx;
    return rc;
  }

  // library-owned stream + events (graph capture cannot use the legacy default stream)
  ctx->user_stream = (cudaStream_t)cuda_stream;
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_it[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_it[1], cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    aac_destroy(ctx);
    return aac_fail(nullptr, AAC_ECUDA, "stream/event creation failed");
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device);
  if (getenv("AAC_NO_GRAPH")) ctx->use_graphs = false;
  {
    const int rev = getenv("AAC_REV") ? atoi(getenv("AAC_REV")) : AAC_REV_DEFAULT;
    cudaMemcpyToSymbol(c_rev, &rev, sizeof(int));
  }
  // wavefront temporal blocking (2D, one rank): depth 8 by default, AAC_WAVE_H=0 disables
  ctx->wave_h = getenv("AAC_WAVE_H") ? atoi(getenv("AAC_WAVE_H")) : 8;
  if (ctx->wave_h != 0 && ctx->wave_h != 4) ctx->wave_h = 8;
  ctx->wave_forced = getenv("AAC_WAVE_H") != nullptr;
  cudaDeviceGetAttribute(&ctx->l2_bytes, cudaDevAttrL2CacheSize, ctx->device);
  // host-staged transport: host syncs inside a step, eager launches; NCCL: captured in the graph
  if (ctx->host_tr) ctx->use_graphs = false;
  // one reduction per Arnoldi step on several ranks (it saves an all-reduce; on one GPU the
  // fused norm costs nothing and the lagged test would cost an extra apply); AAC_GMRES_1R=0/1
  ctx->one_reduce = getenv("AAC_GMRES_1R") ? atoi(getenv("AAC_GMRES_1R")) != 0 : ctx->multi();

  // device allocations
  auto alloc = [&](double** p, long long n) -> bool {
    return cudaMalloc((void**)p, (size_t)(n > 0 ? n : 1) * sizeof(double)) == cudaSuccess;
  };
  const long long L = (long long)ell * N;
  const int ldh = max_krylov + 1;
  ctx->ka_grid = 8 * ctx->num_sms;
  const long long fwd_ctas = (N + 255) / 256 + 1;
  ctx->part_len = std::max<long long>((long long)ctx->ka_grid * 2 * ldh, fwd_ctas);
  ctx->part_len = std::max<long long>(ctx->part_len, 4096);
  bool ok = alloc(&ctx->d_w, hw.size()) && alloc(&ctx->d_what, L) && alloc(&ctx->d_X, 4 * L) &&
            alloc(&ctx->d_tmp, L) && alloc(&ctx->d_V, (long long)(max_krylov + 1) * L) &&
            alloc(&ctx->d_Z, (long long)max_krylov * L) && alloc(&ctx->d_W, L) &&
            alloc(&ctx->d_halo, 2LL * ell * G.S) && alloc(&ctx->d_part, ctx->part_len) &&
            alloc(&ctx->d_red, 3LL * ldh + 8) && alloc(&ctx->d_H, (long long)ldh * max_krylov) &&
            alloc(&ctx->d_G, (long long)ldh * ldh) && alloc(&ctx->d_giv, 6LL * ldh) &&
            alloc(&ctx->d_stat, 64) &&
            cudaMalloc((void**)&ctx->d_grp, (size_t)(ctx->part_len / 32 + 2) * sizeof(unsigned)) == cudaSuccess &&
            cudaMalloc((void**)&ctx->d_st, sizeof(IterState)) == cudaSuccess;
  if (ok) ok = cudaMallocHost((void**)&ctx->h_stat, 64 * sizeof(double)) == cudaSuccess &&
               cudaMallocHost((void**)&ctx->h_st, sizeof(IterState)) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    aac_destroy(ctx);
    return aac_fail(nullptr, AAC_ENOMEM, "device allocation failed (N=%lld, ell=%d, max_krylov=%d)", N,
                    ell, max_krylov);
  }
  G.wx = ctx->d_w;
  G.wy = ctx->d_w + lenx;
  G.wz = ctx->d_w + lenx + leny;
  // (a pageable cudaMemcpy may return before its DMA completes; the library stream does not
  // order after the legacy stream: synchronise the device before any stream work)
  if (cudaMemcpy(ctx->d_w, hw.data(), hw.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(ctx->d_halo, 0, 2LL * ell * G.S * sizeof(double)) != cudaSuccess ||
      cudaMemset(ctx->d_st, 0, sizeof(IterState)) != cudaSuccess ||
      cudaMemset(ctx->d_grp, 0, (size_t)(ctx->part_len / 32 + 2) * sizeof(unsigned)) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    aac_destroy(ctx);
    return aac_fail(nullptr, AAC_ECUDA, "setup copy failed");
  }
  // slab-decomposed wavefront (2D): face weights of the slab +- WAVE_MAXH rows, halo buffers
  if (ctx->nranks > 1 && g->dim == 2) {
    // one row more than the deepest pass: the wavefront also produces the final iterates of the
    // ghost rows -1 and ny, from which the step forms Z_j's halo without an exchange
    const int hd = WAVE_MAXH + 1;
    bool thick = true;
    for (int r = 0; r < g->nranks; ++r) {
      int64_t rl, rh;
      aac_slab_range(ny, g->nranks, r, &rl, &rh);
      thick = thick && rh - rl >= hd;
    }
    if (thick) {
      const long long elo = std::max<long long>(0, lo - hd), ehi = std::min<long long>(ny, hi + hd);
      std::vector<double> he;
      long long le[3];
      double gdummy;
      slab_weights(g, kx, ky, kz, c, elo, ehi, he, le, &gdummy);
      if (cudaMalloc((void**)&ctx->d_wext, (size_t)(le[0] + le[1]) * sizeof(double)) != cudaSuccess ||
          cudaMalloc((void**)&ctx->d_whalo, (size_t)2 * ell * hd * nx * sizeof(double)) != cudaSuccess ||
          cudaMalloc((void**)&ctx->d_ghost, (size_t)2 * ell * nx * sizeof(double)) != cudaSuccess ||
          cudaMemcpy(ctx->d_wext, he.data(), (size_t)(le[0] + le[1]) * sizeof(double), cudaMemcpyHostToDevice) !=
              cudaSuccess ||
          cudaDeviceSynchronize() != cudaSuccess) {
        cudaGetLastError();
        aac_destroy(ctx);
        return aac_fail(nullptr, AAC_ENOMEM, "wavefront halo allocation failed");
      }
      ctx->wext_x = le[0];
      ctx->wext_off = (int)(lo - elo);
      ctx->wext_rows = (int)(ehi - elo);
      ctx->wave_hd = hd;
    }
  }
  // global Gershgorin max (all-reduce max over slabs)
  if (ctx->nranks > 1) {
    ctx->h_stat[0] = gmax;
    cudaMemcpyAsync(ctx->d_stat, ctx->h_stat, sizeof(double), cudaMemcpyHostToDevice, ctx->stream);
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
  // rank-ordered sums (comm.cuh): the gather buffer exists before any step graph is captured
  if (ctx->multi() &&
      cudaMalloc((void**)&ctx->d_gath, (size_t)ctx->nranks * AAC_GATHER_MAX * sizeof(double)) != cudaSuccess) {
    ctx->d_gath = nullptr;
    cudaGetLastError();
    aac_destroy(ctx);
    return aac_fail(nullptr, AAC_ENOMEM, "gather buffer allocation failed");
  }
  *out = ctx;
  return AAC_OK;
}

extern "C" void aac_destroy(aac_ctx* ctx) {
  if (!ctx) return;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  sp_destroy(ctx);
  for (auto& ge : ctx->graphs) cudaGraphExecDestroy(ge.exec);
  double* ptrs[] = {ctx->d_w, ctx->d_what, ctx->d_X, ctx->d_tmp, ctx->d_V, ctx->d_Z,
                    ctx->d_W, ctx->d_bx, ctx->d_bb, ctx->d_halo, ctx->d_part, ctx->d_red, ctx->d_H,
                    ctx->d_G, ctx->d_giv, ctx->d_stat};
  for (double* p : ptrs)
    if (p) cudaFree(p);
  if (ctx->d_st) cudaFree(ctx->d_st);
  if (ctx->d_grp) cudaFree(ctx->d_grp);
  if (ctx->d_wext) cudaFree(ctx->d_wext);
  if (ctx->d_wblk) cudaFree(ctx->d_wblk);
  if (ctx->d_S) cudaFree(ctx->d_S);
  if (ctx->d_lam1) cudaFree(ctx->d_lam1);
  if (ctx->d_T) cudaFree(ctx->d_T);
  if (ctx->d_whalo) cudaFree(ctx->d_whalo);
  if (ctx->d_ghost) cudaFree(ctx->d_ghost);
  if (ctx->d_gath) cudaFree(ctx->d_gath);
  if (ctx->h_stat) cudaFreeHost(ctx->h_stat);
  if (ctx->h_st) cudaFreeHost(ctx->h_st);
  cudaEvent_t evs[] = {ctx->ev_in, ctx->ev_out, ctx->ev_it[0], ctx->ev_it[1]};
  for (auto e : evs)
    if (e) cudaEventDestroy(e);
  for (auto e : ctx->ev_cp)
    if (e) cudaEventDestroy(e);
  if (ctx->cstream) cudaStreamDestroy(ctx->cstream);
  for (int a = 0; a < aac_ctx::NAUX; ++a) {
    if (ctx->aux[a]) cudaStreamDestroy(ctx->aux[a]);
    if (ctx->ev_join[a]) cudaEventDestroy(ctx->ev_join[a]);
  }
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  for (auto& r : ctx->prof_recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  comm_destroy(ctx);
  delete ctx;
}

// Lemma lemma:Zalpha: P_alpha is invertible for alpha != mu_j^ell; with the
// shifts |Lambda_k| = alpha^{1/ell} the block problems (A - Lambda_k) stay definite iff
// alpha^{1/ell} < mu_min -- for the Neumann operator (mu_min = 1) that is alpha < 1.
static int check_alpha(aac_ctx* ctx) {
  if (pow(ctx->alpha, 1.0 / ctx->ell) < ctx->mu_min) return AAC_OK;
  return aac_fail(ctx, AAC_EINVAL,
                  "alpha must lie in (0, mu_min^ell) = (0, %g): mu_min(A) = 1 under Neumann BCs and "
                  "P_alpha is singular at alpha = mu^ell (Lemma lemma:Zalpha, PAPER.md:120)",
                  pow(ctx->mu_min, (double)ctx->ell));
}

extern "C" const char* aac_last_error(const aac_ctx* ctx) {
  if (ctx && !ctx->err.empty()) return ctx->err.c_str();
  return g_last_err.c_str();
}

// ------------------------------------------------------------------------------------------
// Stream handoff: every entry point runs on the library stream, ordered after the caller's
// stream and before anything the caller enqueues afterwards.
struct StreamScope {
  aac_ctx* ctx;
  explicit StreamScope(aac_ctx* c) : ctx(c) {
    cudaEventRecord(ctx->ev_in, ctx->user_stream);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_in, 0);
  }
  ~StreamScope() {
    cudaEventRecord(ctx->ev_out, ctx->stream);
    cudaStreamWaitEvent(ctx->user_stream, ctx->ev_out, 0);
  }
};

// Two points per thread (16-byte loads) when nx is even (AAC_VEC3=1 forces one point per
// thread in 3D: measured 8% slower at 256^3 despite the higher occupancy).
static inline bool vec2(const aac_ctx* ctx) {
  static const bool v3_one = getenv("AAC_VEC3") && atoi(getenv("AAC_VEC3")) == 1;
  return (ctx->geo.nx % 2) == 0 && !(ctx->dim == 3 && v3_one);
}

#include "varying.cuh"      // varying diagonal blocks (N4)

// ------------------------------------------------------------------------------------------
// calA apply
// TMA-staged tile kernel (stencil_tile.cuh) on 2D one-rank Neumann grids with even nx, selected by
// AAC_MATVEC_TILE=1 (measured slower at the headline: 48.5 us against 33.5 us for k_matvec,
// ncu, cold L2 -- k_matvec's neighbour re-reads hit L1/L2, so staging saves no DRAM bytes, and
// the one-thread row-copy ring of 2 CTAs per SM keeps too few bytes in flight).
// x = xbase + j * xjs (j on the device if jdev).
static bool matvec_tile_on(const aac_ctx* ctx) {
  static const bool on = getenv("AAC_MATVEC_TILE") && atoi(getenv("AAC_MATVEC_TILE")) == 1;
  return on && !ctx->varying && mt_ok(ctx->geo, ctx->dim, ctx->nranks);
}

template <typename K>
static int smem_optin(aac_ctx* ctx, K kernel, size_t bytes);

static int launch_matvec_tile(aac_ctx* ctx, const double* xbase, long long xjs, const int* jdev, double* y,
                              double bytes) {
  const Geo& g = ctx->geo;
  MtGeo M;
  M.ntx = (g.nx + MT_TC - 1) / MT_TC;
  M.nty = (g.ny + MT_TR - 1) / MT_TR;
  M.nitems = (long long)M.ntx * M.nty * ctx->ell;
  const size_t smem = mt_smem();
  AAC_TRY(smem_optin(ctx, k_matvec_tile, smem));
  static thread_local int occ = 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_matvec_tile, MT_TC, smem);
    if (occ < 1) occ = 1;
  }
  const long long grid = std::min<long long>(M.nitems, (long long)occ * ctx->num_sms);
  LAUNCH(ctx, KID_MATVEC, bytes,
         k_matvec_tile<<<(unsigned)grid, MT_TC, smem, ctx->stream>>>(g, M, ctx->ell, xbase, xjs, jdev, y));
  return AAC_OK;
}

// Row-marching kernel (stencil_rows.cuh) on 2D grids with even nx (one rank or slabs), opt-in:
// AAC_MATVEC_ROWS=1 (AAC_MATVEC_RY sets the rows per thread). Measured slower at the headline
// (profiles/r02/ab_matvec_rows: 62-89 us per apply at 2-16 rows per thread against 37.9 us for
// k_matvec, graph replay): each row step waits one DRAM latency for its south rows with only
// 12 warps per SM (168 registers), where k_matvec's short-lived CTAs keep more bytes in flight.
// Returns 0 when not selected or not applicable (the caller launches k_matvec).
static int matvec_rows_ry(const aac_ctx* ctx) {
  static const int off = !(getenv("AAC_MATVEC_ROWS") && atoi(getenv("AAC_MATVEC_ROWS")) == 1);
  static const int ry_env = getenv("AAC_MATVEC_RY") ? atoi(getenv("AAC_MATVEC_RY")) : 0;
  if (off || ctx->dim != 2 || ctx->varying || (ctx->geo.nx % 2) != 0) return 0;
  const int ell = ctx->ell;
  if (!(ell == 2 || ell == 4 || ell == 6 || ell == 8 || ell == 10 || ell == 12)) return 0;
  if (ry_env > 0) return ry_env;
  // rows per thread: the most that still gives two waves of resident CTAs (MR_MINB per SM)
  const long long strips = (ctx->geo.nx / 2 + MR_NT - 1) / MR_NT;
  int ry = 16;
  while (ry > 1 && strips * ((ctx->geo.ny + ry - 1) / ry) < 2LL * MR_MINB * ctx->num_sms) ry /= 2;
  return ry;
}

static int launch_matvec_rows(aac_ctx* ctx, int ry, const double* xbase, long long xjs, const int* jdev,
                              double* y, const double* hlo, const double* hhi, double bytes) {
  const Geo& g = ctx->geo;
  const dim3 grid((unsigned)((g.nx / 2 + MR_NT - 1) / MR_NT), (unsigned)((g.ny + ry - 1) / ry));
#define MR_CASE(E)                                                                                  \
  case E:                                                                                           \
    LAUNCH(ctx, KID_MATVEC, bytes,                                                                  \
           k_matvec_rows<E><<<grid, MR_NT, 0, ctx->stream>>>(g, xbase, xjs, jdev, y, hlo, hhi, ry)); \
    return AAC_OK;
  switch (ctx->ell) {
    MR_CASE(2) MR_CASE(4) MR_CASE(6) MR_CASE(8) MR_CASE(10) MR_CASE(12)
    default: break;
  }
#undef MR_CASE
  return aac_fail(ctx, AAC_EINVAL, "k_matvec_rows: unsupported ell %d", ctx->ell);
}

template <int DIM, int VEC>
static int launch_matvec(aac_ctx* ctx, const double* x, double* y, double bytes) {
  const Geo& g = ctx->geo;
  if (DIM == 2 && matvec_tile_on(ctx)) return launch_matvec_tile(ctx, x, 0, nullptr, y, bytes);
  if (DIM == 2) {
    if (const int ry = matvec_rows_ry(ctx))
      return launch_matvec_rows(ctx, ry, x, 0, nullptr, y, ctx->d_halo, ctx->d_halo + (long long)ctx->ell * g.S,
                                bytes);
  }
  const double* hlo = ctx->d_halo;
  const double* hhi = ctx->d_halo + (long long)ctx->ell * g.S;
  const dim3 grid(grid1d(g.nx / VEC, 256), g.ny, g.nz);
  LAUNCH(ctx, KID_MATVEC, bytes,
         k_matvec<DIM, VEC><<<grid, 256, 0, ctx->stream>>>(g, ctx->ell, x, 0, nullptr, y, hlo, hhi));
  return AAC_OK;
}

static int halo_planes(aac_ctx* ctx, const double* x) {
  if (ctx->nranks == 1) return AAC_OK;
  const double* planes[AAC_MAX_ELL];
  int qs[AAC_MAX_ELL];
  for (int j = 0; j < ctx->ell; ++j) {
    planes[j] = x + (long long)j * ctx->geo.N;
    qs[j] = j;
  }
  return comm_halo(ctx, planes, qs, ctx->ell);
}

static int matvec_impl(aac_ctx* ctx, const double* x, double* y) {
  if (ctx->varying) {
    AAC_TRY(matvec_var(ctx, x, 0, nullptr, y));
    ctx->sweeps += ctx->ell;
    return AAC_OK;
  }
  AAC_TRY(halo_planes(ctx, x));
  const double V = 8.0 * ctx->ell * ctx->geo.N, C = 8.0 * ctx->dim * ctx->geo.N;
  const double bytes = 2 * V + C;
  const bool v2 = vec2(ctx);
  switch (ctx->dim) {
    case 1: AAC_TRY(v2 ? launch_matvec<1, 2>(ctx, x, y, bytes) : launch_matvec<1, 1>(ctx, x, y, bytes)); break;
    case 2: AAC_TRY(v2 ? launch_matvec<2, 2>(ctx, x, y, bytes) : launch_matvec<2, 1>(ctx, x, y, bytes)); break;
    default: AAC_TRY(v2 ? launch_matvec<3, 2>(ctx, x, y, bytes) : launch_matvec<3, 1>(ctx, x, y, bytes)); break;
  }
  ctx->sweeps += ctx->ell;
  return AAC_OK;
}

extern "C" int aac_matvec(aac_ctx* ctx, const double* x, double* y) {
  if (!ctx || !x || !y || x == y) return aac_fail(ctx, AAC_EINVAL, "aac_matvec: bad pointers");
  NvtxRange nv("aac_matvec");
  StreamScope ss(ctx);
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

static void inv_theta(const aac_ctx* ctx, int kb, double* tr, double* ti) {
  double lr, li;
  shift_of_block(ctx, kb, &lr, &li);
  const std::complex<double> it =
      1.0 / std::complex<double>(0.5 * (ctx->mu_max + ctx->mu_min) - lr, -li);
  const int h = ctx->ell / 2;
  *tr = it.real();
  *ti = (kb != 0 && kb != h) ? it.imag() : 0.0;
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

// z = Gamma^{-1} U y from per-block sources (streaming; one point per thread measured faster
// than two: the per-block register arrays stay small)
// The inverse transform over N points (planes N apart in source and destination).
static int run_inverse_n(aac_ctx* ctx, const Dft& D, const NcFinal& F, double* zbase, long long zjs,
                         const IterState* st, long long N) {
  const double V = 8.0 * ctx->ell * N;
  if (ctx->ell == 10)
    LAUNCH(ctx, KID_INV, 2 * V, k_inverse_exact<10><<<grid1d(N, 256), 256, 0, ctx->stream>>>(N, D, F, zbase, zjs, st));
  else if (ctx->ell == 12)
    LAUNCH(ctx, KID_INV, 2 * V, k_inverse_exact<12><<<grid1d(N, 256), 256, 0, ctx->stream>>>(N, D, F, zbase, zjs, st));
  else
    LAUNCH(ctx, KID_INV, 2 * V, k_inverse<1><<<grid1d(N, 256), 256, 0, ctx->stream>>>(N, D, F, zbase, zjs, st));
  return AAC_OK;
}

static int run_inverse(aac_ctx* ctx, const Dft& D, const NcFinal& F, double* zbase, long long zjs,
                       const IterState* st) {
  return run_inverse_n(ctx, D, F, zbase, zjs, st, ctx->geo.N);
}

#include "sp.cuh"

static inline int plane_of_block(int ell, int kb) {
  const int h = ell / 2;
  return kb == 0 ? 0 : (kb == h ? ell - 1 : 2 * kb - 1);
}

static ArnoldiCtx arnoldi_ctx(aac_ctx* ctx) {
  ArnoldiCtx ac{};
  const int ldh = ctx->max_krylov + 1;
  ac.st = ctx->d_st;
  ac.H = ctx->d_H;
  ac.ldh = ldh;
  ac.cs = ctx->d_giv;
  ac.sn = ctx->d_giv + ldh;
  ac.g = ctx->d_giv + 2 * ldh;
  ac.sigma = ctx->d_giv + 4 * ldh;
  ac.c = ctx->d_giv + 5 * ldh;
  ac.G = ctx->d_G;
  ac.red = ctx->d_red;
  ac.local_only = ctx->multi();
  ac.one_reduce = ctx->one_reduce ? 1 : 0;
  ac.pub = ctx->pub_fold;
  return ac;
}

// Eager GMRES (profiling, AAC_NO_GRAPH, host transport): after the forward step of an Arnoldi
// step -- the kernel that forms V_j, its norm and the Givens update, so the step where the
// solve converges -- read the state back; a converged solve then launches nothing more for
// that step. (Graph replay instead runs the whole speculative step, whose kernels return at
// once; profile counters are only collected in eager mode, so they count work that ran.)
static constexpr int AAC_STEP_DONE = 100;              // internal: the solve finished
static int publish(aac_ctx* ctx, const void* dsrc, void* hdst, size_t bytes);
static int poll_after_forward(aac_ctx* ctx) {
  if (!ctx->eager_poll) return AAC_OK;
  AAC_TRY(publish(ctx, ctx->d_st, ctx->h_st, sizeof(IterState)));
  AAC_TRY(comm_sync(ctx));
  return ctx->h_st->done ? AAC_STEP_DONE : AAC_OK;
}

// ------------------------------------------------------------------------------------------
// Dynamic shared memory beyond 48 KB needs an explicit opt-in per kernel.
// The opt-in is per kernel and process-wide: raise it whenever a launch needs more than any
// earlier one (contexts with a larger max_krylov need more shared memory in k_arnoldi).
template <typename K>
static int smem_optin(aac_ctx* ctx, K kernel, size_t bytes) {
  static thread_local std::vector<std::pair<const void*, size_t>> done;
  if (bytes <= 48 * 1024) return AAC_OK;
  const void* key = reinterpret_cast<const void*>(kernel);
  for (auto& d : done)
    if (d.first == key && d.second >= bytes) return AAC_OK;
  CUDA_TRY(ctx, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  for (auto& d : done)
    if (d.first == key) { d.second = bytes; return AAC_OK; }
  done.emplace_back(key, bytes);
  return AAC_OK;
}

template <int ELLC, bool TMA>
static int launch_fwd_upd_t(aac_ctx* ctx, double bytes, bool norm) {
  const long long N = ctx->geo.N, L = (long long)ctx->ell * N;
  FwdUpd U{ctx->d_W, ctx->d_V, L, ctx->d_part, arnoldi_ctx(ctx), ctx->d_grp, norm ? 1 : 0};
  const Dft D = make_dft(ctx);
  const size_t smem = TMA ? (size_t)FS * ELLC * FT * sizeof(double) : 0;
  AAC_TRY(smem_optin(ctx, k_fwd_upd<ELLC, TMA>, smem));
  LAUNCH(ctx, KID_FWD, bytes,
         (k_fwd_upd<ELLC, TMA><<<grid1d(N, FT), FT + 32, smem, ctx->stream>>>(N, D, ctx->d_what, U)));
  return AAC_OK;
}

// Forward step of an Arnoldi step: the update forming V_j + its transform; `norm`: also reduce
// ||V_j||^2 and run the norm step (always, except in one-reduce mode inside the loop).
static int launch_fwd_upd(aac_ctx* ctx, double bytes, bool norm) {
  const bool tma = (ctx->geo.N % 2) == 0;         // 16-byte aligned plane tiles
  // plane capacity = ell rounded up to 10 / 12 / 16: the shared-memory ring scales with it
  if (ctx->ell <= 10) return tma ? launch_fwd_upd_t<10, true>(ctx, bytes, norm) : launch_fwd_upd_t<10, false>(ctx, bytes, norm);
  if (ctx->ell <= 12) return tma ? launch_fwd_upd_t<12, true>(ctx, bytes, norm) : launch_fwd_upd_t<12, false>(ctx, bytes, norm);
  return tma ? launch_fwd_upd_t<16, true>(ctx, bytes, norm) : launch_fwd_upd_t<16, false>(ctx, bytes, norm);
}

// The forward step inside the Arnoldi loop: with the norm step (+ its all-reduce on several
// ranks and the eager poll), or without it in one-reduce mode.
static int forward_step(aac_ctx* ctx, double bytes) {
  AAC_TRY(launch_fwd_upd(ctx, bytes, !ctx->one_reduce));
  if (ctx->one_reduce) return AAC_OK;
  if (ctx->multi()) {
    AAC_TRY(comm_allreduce(ctx, ctx->d_red, 1, ncclSum));
    LAUNCH(ctx, KID_SCALAR, 0, k_scalar_norm<<<1, 1, 0, ctx->stream>>>(arnoldi_ctx(ctx)));
  }
  return poll_after_forward(ctx);
}

// ------------------------------------------------------------------------------------------
// Per-block wavefront launches (wave_r.cuh): one kernel instantiation per (steps, real/complex,
// general, first pass), the active blocks of a pass forked over the auxiliary streams and joined
// back into the library stream (a fork/join subgraph under graph capture).
template <int H, int NT, int NS, bool CPLX, bool GEN, bool VIRT, typename T>
static int waver_launch_t(aac_ctx* ctx, const WROne& P, int ncta, const WSlab& sl, const IterState* st,
                          cudaStream_t s, bool clu) {
  if constexpr (!GEN && std::is_same<T, double>::value) {
    if (clu) {                          // the strips of a row chunk as one cluster (no x-halo)
      auto kern = k_waver<H, NT, NS, CPLX, GEN, VIRT, true, T>;
      const size_t smem = waver_smem_clu<NT, T>(NS, CPLX ? 2 : 1);
      AAC_TRY(smem_optin(ctx, kern, smem));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)ncta);
      cfg.blockDim = dim3(NT);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)P.nstrip;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, kern, ctx->geo, P, (const double*)ctx->d_what, st, sl));
      return AAC_OK;
    }
  }
  auto kern = k_waver<H, NT, NS, CPLX, GEN, VIRT, false, T>;
  const size_t smem = waver_smem<NT, T>(NS, CPLX ? 2 : 1);
  AAC_TRY(smem_optin(ctx, kern, smem));
  kern<<<ncta, NT, smem, s>>>(ctx->geo, P, ctx->d_what, st, sl);
  return AAC_OK;
}

template <int H, int NT, int NS, typename T>
static int waver_launch_ns(aac_ctx* ctx, const WROne& P, int ncta, const WSlab& sl, const IterState* st,
                           cudaStream_t s, bool gen, bool clu) {
  if constexpr (NS >= 1) {
    if (P.b.ns != NS) return waver_launch_ns<H, NT, NS - 1, T>(ctx, P, ncta, sl, st, s, gen, clu);
    const bool c = P.b.np == 2, v = P.b.virt != 0;
    if (gen) {
      if (c) return v ? waver_launch_t<H, NT, NS, true, true, true, T>(ctx, P, ncta, sl, st, s, clu)
                      : waver_launch_t<H, NT, NS, true, true, false, T>(ctx, P, ncta, sl, st, s, clu);
      return v ? waver_launch_t<H, NT, NS, false, true, true, T>(ctx, P, ncta, sl, st, s, clu)
               : waver_launch_t<H, NT, NS, false, true, false, T>(ctx, P, ncta, sl, st, s, clu);
    }
    if (c) return v ? waver_launch_t<H, NT, NS, true, false, true, T>(ctx, P, ncta, sl, st, s, clu)
                    : waver_launch_t<H, NT, NS, true, false, false, T>(ctx, P, ncta, sl, st, s, clu);
    return v ? waver_launch_t<H, NT, NS, false, false, true, T>(ctx, P, ncta, sl, st, s, clu)
             : waver_launch_t<H, NT, NS, false, false, false, T>(ctx, P, ncta, sl, st, s, clu);
  }
  return aac_fail(ctx, AAC_EINVAL, "wavefront: bad step count %d", P.b.ns);
}

static int aux_streams(aac_ctx* ctx) {
  if (ctx->ev_fork) return AAC_OK;
  for (int a = 0; a < aac_ctx::NAUX; ++a) {
    CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->aux[a], cudaStreamNonBlocking));
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_join[a], cudaEventDisableTiming));
  }
  CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
  return AAC_OK;
}

// Cluster wavefront (k_waver CLU, opt-in: AAC_WAVE_CLUSTER=1): the strips of a row chunk
// exchange edge columns through distributed shared memory, so no strip recomputes an x-halo.
// Needs all strips of a row in one cluster (ceil(nx / NT) <= 8, the portable cluster size).
// Bit-identical to the halo kernel but measured slower at the headline (9.10-9.49 vs 8.31 ms per
// solve): the per-step neighbour coupling costs more than the halo columns.
static bool wave_cluster(const aac_ctx* ctx, int nt) {
  const char* e = getenv("AAC_WAVE_CLUSTER");        // (read per pass: tests switch it)
  const int env = e ? atoi(e) : 0;
  const int nstrip = (ctx->geo.nx + nt - 1) / nt;
  return env != 0 && ctx->dim == 2 && nstrip >= 2 && nstrip <= 8;
}

// All blocks of one wavefront pass: block 0 (the heaviest) on the library stream, the others
// round-robin over the auxiliary streams. Profiled as ONE launch group (its events bracket the
// fork and the join); every kernel counts in aac_launch_count.
template <int H, int NT>
static int waver_group(aac_ctx* ctx, const WSweep& S, int nchunk, const WSlab& sl, const IterState* st,
                       double bytes, int ybeg, int yend) {
  AAC_TRY(aux_streams(ctx));
  const bool gen = ctx->geo.dir || ctx->nranks > 1;
  const int naux = std::min(aac_ctx::NAUX, S.nb - 1);
  LaunchScope ls_(ctx, KID_SWEEP, bytes);
  if (naux > 0) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fork, ctx->stream));
    for (int a = 0; a < naux; ++a) CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->aux[a], ctx->ev_fork, 0));
  }
  const bool clu = wave_cluster(ctx, NT) && !gen && !ctx->inner_f32;
  for (int i = 0; i < S.nb; ++i) {
    // strips of NT - 2 ns columns: the x-halo of a block is its step count; with a cluster
    // (wave_cluster) strips of NT columns without a halo
    const int halo = clu ? 0 : S.b[i].ns;
    const int nstrip = (ctx->geo.nx + (NT - 2 * halo) - 1) / (NT - 2 * halo);
    const cudaStream_t s = i == 0 ? ctx->stream : ctx->aux[(i - 1) % naux];
    const WROne P{S.b[i], nstrip, S.ly[i], ybeg, yend};
    if (ctx->inner_f32)                 // mixed precision (AAC_F32): fp32 recurrence, fp64 storage
      AAC_TRY((waver_launch_ns<H, NT, H, float>(ctx, P, P.nstrip * nchunk, sl, st, s, gen, false)));
    else
      AAC_TRY((waver_launch_ns<H, NT, H, double>(ctx, P, P.nstrip * nchunk, sl, st, s, gen, clu)));
  }
  for (int a = 0; a < naux; ++a) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_join[a], ctx->aux[a]));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_join[a], 0));
  }
  ctx->launches += S.nb - 1;
  return ls_.end();
}

// ------------------------------------------------------------------------------------------
// Preconditioner: forward DFT (optionally fused with the Arnoldi update), Chebyshev sweeps,
// last sweep fused with the inverse DFT. gmres_mode: input is the Arnoldi update (W, V, c),
// output Z_j with j read on the device; otherwise r -> z.
// Wavefront passes (wave.cuh, 2D, one rank): each pass advances every block still running
// by up to H steps in one read of its inputs; passes ping-pong between the iterate slot sets
// d_X + (2k, 2k+1) * L; the final iterates feed the streaming inverse transform.
template <int H, int NT>
static int wave_passes_t(aac_ctx* ctx, const NcPlan& P, double* zbase, long long zjs, const IterState* st) {
  using WG = WGeom<H, NT>;
  const Geo& g = ctx->geo;
  const int ell = ctx->ell, h = ell / 2;
  const long long N = g.N, L = (long long)ell * N;
  const double C = 8.0 * ctx->dim * N;
  const Dft D = make_dft(ctx);
  // register-resident wavefront (wave_r.cuh) by default; AAC_WAVE_OLD=1: the shared-memory
  // history kernel of wave.cuh
  static const bool old = getenv("AAC_WAVE_OLD") != nullptr;
  const size_t smem = WG::SMEM;
  AAC_TRY(smem_optin(ctx, k_wave<H, NT, false>, WG::SMEM));
  AAC_TRY(smem_optin(ctx, k_wave<H, NT, true>, WG::SMEM));
  const int nstrip = (g.nx + WG::TX - 1) / WG::TX;
  // rows per chunk: AAC_WAVE_LY overrides the default below
  const int ly_env = getenv("AAC_WAVE_LY") ? atoi(getenv("AAC_WAVE_LY")) : 0;
  const double* fin[AAC_MAX_BLK] = {};
  const int steps_max = P.pmax - 1;
  // Ghost mode (several ranks, one pass, no passive block): the wavefront also computes x_{p_k}
  // on the slab's ghost rows (-1, ny; the hat-w halo is one row deeper than the deepest pass),
  // and their inverse transform below is Z_j's halo -- the step needs no exchange of Z_j.
  static const bool ghost_off = getenv("AAC_WAVE_GHOST") && atoi(getenv("AAC_WAVE_GHOST")) == 0;
  bool ghost = !old && !ghost_off && ctx->nranks > 1 && ctx->d_ghost && steps_max <= H &&
               ctx->wave_hd >= steps_max + 1;
  for (int kb = 0; kb <= h; ++kb) ghost = ghost && P.p[kb] >= 2;
  const int ybeg = (ghost && g.has_lo) ? -1 : 0, yend = (ghost && g.has_hi) ? g.ny + 1 : g.ny;
  for (int pass = 0; pass * H < steps_max; ++pass) {
    const int s0 = 1 + pass * H;
    const int set = pass & 1, prev_set = set ^ 1;
    WSweep S{};
    S.nstrip = nstrip;
    int nb = 0;
    double passes = 0.0, flops = 0.0;
    for (int kb = 0; kb <= h; ++kb) {
      const int steps = P.p[kb] - 1;
      if (steps < s0) continue;                       // finished (or passive)
      const int ns = std::min(H, steps - s0 + 1);
      const bool cplx = (kb != 0 && kb != h);
      const int q = plane_of_block(ell, kb);
      WBlk& B = S.b[nb++];
      B.q = q;
      B.np = cplx ? 2 : 1;
      B.ns = ns;
      B.virt = pass == 0;
      if (pass == 0) {
        inv_theta(ctx, kb, &B.sr, &B.si);
        B.ps = B.pm = ctx->d_what + (long long)q * N;
        B.mr = B.mi = 0.0;
      } else {
        B.ps = ctx->d_X + (long long)(2 * prev_set) * L + (long long)q * N;
        B.pm = ctx->d_X + (long long)(2 * prev_set + 1) * L + (long long)q * N;
        B.sr = 1.0; B.si = 0.0; B.mr = 1.0; B.mi = 0.0;
      }
      const bool final_pass = s0 + ns - 1 == steps;
      B.out_last = ctx->d_X + (long long)(2 * set) * L + (long long)q * N;
      B.out_prev = final_pass ? nullptr : ctx->d_X + (long long)(2 * set + 1) * L + (long long)q * N;
      B.glo = ghost ? ctx->d_ghost + (long long)q * g.nx : nullptr;
      B.ghi = ghost ? ctx->d_ghost + (long long)(ell + q) * g.nx : nullptr;
      if (final_pass) fin[kb] = B.out_last;
      for (int l = 0; l < ns; ++l) {
        const int s = s0 + l;
        B.ar[l] = P.a_re[kb * P.pmax + s]; B.ai[l] = P.a_im[kb * P.pmax + s];
        B.br[l] = P.b_re[kb * P.pmax + s]; B.bi[l] = P.b_im[kb * P.pmax + s];
      }
      shift_of_block(ctx, kb, &B.lr, &B.li);
      passes += B.np * ((pass == 0 ? 1.0 : 3.0) + (final_pass ? 1.0 : 2.0));
      // algorithmic fp64 flops of the recurrence per point and step:
      // complex 58 (2 x 5-point stencils in difference form + complex three-term update), real 21
      flops += (double)N * ns * (cplx ? 58.0 : 21.0);
      ctx->sweeps += (long long)ns * B.np;
    }
    if (nb == 0) break;
    // heaviest blocks first (lowest CTA indices are dispatched first)
    auto cost = [](const WBlk& b) { return (double)b.ns * (b.np == 2 ? 58.0 : 21.0); };
    std::stable_sort(S.b, S.b + nb, [&](const WBlk& a, const WBlk& b) { return cost(a) > cost(b); });
    S.nb = nb;
    // rows per chunk (all blocks alike): ~2 CTAs per resident slot over the active blocks,
    // at least 8 steps' worth of rows (measured at the headline: 9.29 ms at 80 rows, within 3%
    // from 48 to 140; an equal-work split with taller chunks for cheaper blocks was 20% slower)
    auto layout = [&](int ly0) {                      // fills S.ly / S.cta0, returns #CTAs
      int ncta = 0;
      for (int i = 0; i < nb; ++i) {
        S.ly[i] = std::max(1, std::min(ly0, g.ny));
        S.cta0[i] = ncta;
        ncta += nstrip * ((g.ny + S.ly[i] - 1) / S.ly[i]);
      }
      S.cta0[nb] = ncta;
      return ncta;
    };
    int ly0 = ly_env;
    if (ly0 <= 0 && !old) {
      // per-block register wavefront: latency-bound at 2-3 CTAs per SM, so more, shorter chunks
      // pay for their warm-up rows -- about 64 rows, ny split evenly (measured at the headline:
      // 8.41 ms per solve at 64 rows, 8.46-8.57 at 40-72, 8.63 at 80, 9.21 at 160)
      const int rows = yend - ybeg;                    // (ghost mode: the slab + its ghost rows)
      const int nch = std::max(1, (rows + 63) / 64);
      ly0 = (rows + nch - 1) / nch;
      const long long slots = 2LL * ctx->num_sms;
      const long long cols = (long long)g.ny * nstrip * nb;
      if (cols / ly0 < slots) {                        // small grids: fill the resident slots
        int ns_max = 1;
        for (int i = 0; i < nb; ++i) ns_max = std::max(ns_max, S.b[i].ns);
        ly0 = (int)std::max<long long>(2LL * ns_max, (cols + slots - 1) / slots);
      }
    }
    if (ly0 <= 0) {
      const long long slots = (long long)(NT > 128 ? 2 : 3) * ctx->num_sms;
      const long long want = std::max<long long>(1, 2 * slots / std::max(1, nstrip * nb));
      ly0 = (int)std::max<long long>(10LL * H, (g.ny + want - 1) / want);
      // small grids: 10 H rows per chunk would leave most SMs idle -- fill the resident slots
      // instead (at least 2 ns rows, the warm-up, per chunk)
      const long long cols = (long long)g.ny * nstrip * nb;
      if (cols / ly0 < slots) {
        int ns_max = 1;
        for (int i = 0; i < nb; ++i) ns_max = std::max(ns_max, S.b[i].ns);
        ly0 = (int)std::max<long long>(2LL * ns_max, (cols + slots - 1) / slots);
      }
    }
    const int ncta = layout(ly0);
    WSlab sl{g.wx, g.wy, 0, g.ny, nullptr, nullptr, 0, (int)ctx->lo, (int)ctx->n[1]};
    if (ctx->nranks > 1) {                             // hd rows of hat w from each neighbour
      const int hd = ctx->wave_hd;
      Geo gh = g;
      gh.S = (long long)hd * g.nx;
      const double* planes[AAC_MAX_ELL];
      int qs[AAC_MAX_ELL];
      for (int q = 0; q < ell; ++q) {
        planes[q] = ctx->d_what + (long long)q * N;
        qs[q] = q;
      }
      double* hl = ctx->d_whalo;
      double* hh = ctx->d_whalo + (long long)ell * hd * g.nx;
      AAC_TRY(comm_halo_ex(ctx, gh, planes, qs, ell, hl, hh));
      sl = WSlab{ctx->d_wext, ctx->d_wext + ctx->wext_x, ctx->wext_off, ctx->wext_rows, hl, hh, hd,
                 (int)ctx->lo, (int)ctx->n[1]};
    }
    ctx->next_flops = flops;
    if (old) {
      LAUNCH(ctx, KID_SWEEP, 8.0 * N * passes + C,
             ((g.dir || ctx->nranks > 1)
                  ? k_wave<H, NT, true><<<ncta, NT, smem, ctx->stream>>>(g, S, ctx->d_what, st, sl)
                  : k_wave<H, NT, false><<<ncta, NT, smem, ctx->stream>>>(g, S, ctx->d_what, st, sl)));
    } else {
      AAC_TRY(waver_group<H, NT>(ctx, S, (yend - ybeg + S.ly[0] - 1) / S.ly[0], sl, st, 8.0 * N * passes + C,
                                 ybeg, yend));
    }
  }
  if (ghost) {                                         // Z_j on the ghost rows -> d_halo
    NcFinal G{};
    for (int side = 0; side < 2; ++side) {
      if (side == 0 ? !g.has_lo : !g.has_hi) continue;
      for (int kb = 0; kb <= h; ++kb) {
        G.tr[kb] = 1.0;
        G.ti[kb] = 0.0;
        G.src[kb] = ctx->d_ghost + (long long)(side * ell + plane_of_block(ell, kb)) * g.nx;
      }
      AAC_TRY(run_inverse_n(ctx, D, G, ctx->d_halo + (long long)side * ell * g.S, 0, st, g.nx));
    }
    ctx->z_ghost = true;
  }
  NcFinal F{};
  for (int kb = 0; kb <= h; ++kb) {
    if (P.p[kb] == 1) {                                // passive: y = w / theta
      inv_theta(ctx, kb, &F.tr[kb], &F.ti[kb]);
      F.src[kb] = ctx->d_what + (long long)plane_of_block(ell, kb) * N;
    } else {
      F.tr[kb] = 1.0;
      F.ti[kb] = 0.0;
      F.src[kb] = fin[kb];
    }
  }
  return run_inverse(ctx, D, F, zbase, zjs, st);
}

// The wavefront pays when every step of a block fits in ONE pass (no iterate ever goes to memory),
// or when the iterates do not fit in L2 (then a multi-pass wave still moves fewer HBM bytes than
// per-step sweeps). With many steps on an L2-resident problem (the paper's n_x = 500 runs: 144
// steps, 5V = 100 MB) the per-step sweeps win: no halo / warm-up recomputation, L2 bandwidth
// (measured 563 vs 348 outer its/s). AAC_WAVE_H forces the setting.
static bool wave_pays(const aac_ctx* ctx, const NcPlan& P) {
  if (ctx->wave_forced || P.pmax - 1 <= ctx->wave_h) return true;
  const double V = 8.0 * ctx->ell * ctx->geo.N;      // one block-vector; the sweeps keep 3 iterate
  return 5.0 * V > (double)ctx->l2_bytes;            // slots + hat w + z in flight
}

static int wave_passes(aac_ctx* ctx, const NcPlan& P, double* zbase, long long zjs, const IterState* st) {
  if (ctx->wave_h == 4) return wave_passes_t<4, 128>(ctx, P, zbase, zjs, st);
  // strip width 128 threads (112 columns + 2 x 8 halo); AAC_WAVE_NT=192 selects 176-column
  // strips (fewer halo columns at nx = 1024, 1152 vs 1280 thread-columns, but 2 instead of 3
  // CTAs per SM: measured no faster)
  static const int nt_env = getenv("AAC_WAVE_NT") ? atoi(getenv("AAC_WAVE_NT")) : 0;
  if (nt_env == 192) return wave_passes_t<8, 192>(ctx, P, zbase, zjs, st);
  return wave_passes_t<8, 128>(ctx, P, zbase, zjs, st);
}

template <int DIM, int VEC>
static int nc_apply_t(aac_ctx* ctx, const NcPlan& P, const double* r, double* zbase, bool gmres_mode, int host_j) {
  const Geo& g = ctx->geo;
  const int ell = ctx->ell, h = ell / 2;
  const long long N = g.N, L = (long long)ell * N;
  const double V = 8.0 * L, C = 8.0 * ctx->dim * N;
  const Dft D = make_dft(ctx);
  const IterState* st = gmres_mode ? ctx->d_st : nullptr;
  if (gmres_mode) {
    // algorithmic bytes: W + V_0..V_{j-1} in, V_j and hat w out (j = 0: V_0 in, hat w out)
    const int rc = forward_step(ctx, (host_j == 0 ? 2 : host_j + 3) * V);
    if (rc != AAC_OK) return rc;
  } else {
    if (ell <= 10)
      LAUNCH(ctx, KID_FWD, 2 * V, (k_forward<10><<<grid1d(N, 256), 256, 0, ctx->stream>>>(N, D, r, ctx->d_what)));
    else
      LAUNCH(ctx, KID_FWD, 2 * V, (k_forward<16><<<grid1d(N, 256), 256, 0, ctx->stream>>>(N, D, r, ctx->d_what)));
  }
  const long long zjs = gmres_mode ? L : 0;
  if (P.pmax == 1) {
    NcFinal F{};
    for (int kb = 0; kb <= h; ++kb) {
      inv_theta(ctx, kb, &F.tr[kb], &F.ti[kb]);
      F.src[kb] = ctx->d_what + (long long)plane_of_block(ell, kb) * N;
    }
    AAC_TRY(run_inverse(ctx, D, F, zbase, zjs, st));
    return AAC_OK;
  }
  // wavefront: one rank, or slabs of >= WAVE_MAXH rows with every block done in one pass (the
  // halo exchange covers hat w only)
  if (DIM == 2 && ctx->wave_h > 0 && (wave_pays(ctx, P) || ctx->inner_f32) &&
      (ctx->nranks == 1 || (ctx->wave_hd > 0 && P.pmax - 1 <= WAVE_MAXH && ctx->wave_h == WAVE_MAXH)))
    return wave_passes(ctx, P, zbase, zjs, st);
  if (ctx->inner_f32)
    return aac_fail(ctx, AAC_EINVAL, "AAC_F32 (mixed precision) needs the 2D wavefront path (dim 2)");
  double* X = ctx->d_X;
  auto slot = [&](int s, int q) { return X + (long long)(s % 3) * L + (long long)q * N; };
  const double* hlo = ctx->d_halo;
  const double* hhi = ctx->d_halo + (long long)ell * g.S;
  const unsigned ncx_last = grid1d(g.nx / VEC, SW_TX), ncx = grid1d(g.nx / VEC, SW_FX);
  // the last step as a regular sweep writing x_{p_k}, then the streaming inverse transform
  // (measured faster than the fused k_sweep<LAST>, which stays available: AAC_FUSED_LAST=1)
  static const bool split_last = getenv("AAC_FUSED_LAST") == nullptr;
  const double* fin[AAC_MAX_BLK] = {};
  for (int t = 1; t < P.pmax; ++t) {
    const bool last = (t == P.pmax - 1) && !split_last;
    NcSweep S{};
    S.nblk = h + 1;
    const double* planes[AAC_MAX_ELL];
    int qs[AAC_MAX_ELL], nh = 0, nplanes = 0;
    double passes = 0.0;             // compulsory plane passes (virtual x_1 = w/theta, x_0 = 0 read nothing)
    for (int kb = 0; kb <= h; ++kb) {
      const int s = t - (P.pmax - P.p[kb]);          // aligned ends: block starts late
      const bool cplx = (kb != 0 && kb != h);
      const int q = plane_of_block(ell, kb);
      if (s < 1) {                                     // inactive now; passive at the end
        S.passive[kb] = 1;
        inv_theta(ctx, kb, &S.ptr[kb], &S.pti[kb]);
        continue;
      }
      NcBlk& B = S.b[S.nact++];
      B.kb = kb;
      B.cplx = cplx ? 1 : 0;
      B.q = q;
      double tr, ti;
      inv_theta(ctx, kb, &tr, &ti);
      const double* wq = ctx->d_what + (long long)q * N;
      if (s == 1) {                    // x_1 = w/theta, x_0 = 0
        B.ps = wq; B.sr = tr; B.si = ti;
        B.pm = wq; B.mr = 0.0; B.mi = 0.0;
      } else {
        B.ps = slot(s, q); B.sr = 1.0; B.si = 0.0;
        if (s == 2) { B.pm = wq; B.mr = tr; B.mi = ti; }
        else { B.pm = slot(s - 1, q); B.mr = 1.0; B.mi = 0.0; }
      }
      B.xo = last ? nullptr : slot(s + 1, q);
      fin[kb] = slot(s + 1, q);
      B.ar = P.a_re[kb * P.pmax + s]; B.ai = P.a_im[kb * P.pmax + s];
      B.br = P.b_re[kb * P.pmax + s]; B.bi = P.b_im[kb * P.pmax + s];
      shift_of_block(ctx, kb, &B.lr, &B.li);
      const int np = cplx ? 2 : 1;
      for (int e = 0; e < np; ++e) {
        planes[nh] = B.ps + (long long)e * N;
        qs[nh++] = q + e;
      }
      nplanes += np;
      passes += np * ((s == 1 ? 1.0 : s == 2 ? 2.0 : 3.0) + (last ? 0.0 : 1.0));
    }
    AAC_TRY(comm_halo(ctx, planes, qs, nh));
    const dim3 blk = last ? dim3(SW_TX, S.nact) : dim3(SW_FX, 1);
    const dim3 gsw(last ? ncx_last : ncx * S.nact, g.ny, g.nz);
    if (last) {
      const size_t smem = (size_t)ell * SW_TX * VEC * sizeof(double);
      const double bytes = 8.0 * N * passes + C + V;           // x_s, x_{s-1}, w in; z out
      LAUNCH(ctx, KID_INV, bytes,
             (k_sweep<DIM, VEC, true><<<gsw, blk, smem, ctx->stream>>>(g, S, D, ctx->d_what, hlo, hhi, zbase, zjs, st)));
    } else {
      const double bytes = 8.0 * N * passes + C;
      LAUNCH(ctx, KID_SWEEP, bytes,
             (k_sweep<DIM, VEC, false><<<gsw, blk, 0, ctx->stream>>>(g, S, D, ctx->d_what, hlo, hhi, nullptr, 0, st)));
    }
    ctx->sweeps += nplanes;
  }
  if (split_last) {
    NcFinal F{};
    for (int kb = 0; kb <= h; ++kb) {
      if (P.p[kb] == 1) {                              // passive: y = w / theta
        inv_theta(ctx, kb, &F.tr[kb], &F.ti[kb]);
        F.src[kb] = ctx->d_what + (long long)plane_of_block(ell, kb) * N;
      } else {
        F.tr[kb] = 1.0;
        F.ti[kb] = 0.0;
        F.src[kb] = fin[kb];
      }
    }
    AAC_TRY(run_inverse(ctx, D, F, zbase, zjs, st));
  }
  return AAC_OK;
}

static int nc_apply(aac_ctx* ctx, int method, int k, const double* r, double* z, bool gmres_mode, int host_j = 0) {
  const NcPlan& P = nc_plan(ctx, method, k);
  // two points per thread (16-byte loads) when nx is even; AAC_SWEEP_VEC=1 forces one
  static const bool sweep_v1 = getenv("AAC_SWEEP_VEC") && atoi(getenv("AAC_SWEEP_VEC")) == 1;
  const bool v2 = vec2(ctx) && !sweep_v1;
  switch (ctx->dim) {
    case 1: return v2 ? nc_apply_t<1, 2>(ctx, P, r, z, gmres_mode, host_j) : nc_apply_t<1, 1>(ctx, P, r, z, gmres_mode, host_j);
    case 2: return v2 ? nc_apply_t<2, 2>(ctx, P, r, z, gmres_mode, host_j) : nc_apply_t<2, 1>(ctx, P, r, z, gmres_mode, host_j);
    default: return v2 ? nc_apply_t<3, 2>(ctx, P, r, z, gmres_mode, host_j) : nc_apply_t<3, 1>(ctx, P, r, z, gmres_mode, host_j);
  }
}

#include "exact_host.cuh"   // exact P_alpha for the paper operator (N3): host side

// method | AAC_F32: this call's NC inner solves in fp32 (reset on return)
struct F32Scope {
  aac_ctx* c;
  F32Scope(aac_ctx* c_, bool on) : c(c_) { c->inner_f32 = on; }
  ~F32Scope() { c->inner_f32 = false; }
};

static int split_f32(aac_ctx* ctx, int* method, bool* f32) {
  *f32 = (*method & AAC_F32) != 0;
  *method &= ~AAC_F32;
  if (*f32 && *method != AAC_NC1 && *method != AAC_NC2)
    return aac_fail(ctx, AAC_EINVAL, "AAC_F32 applies to the nested Chebyshev methods (AAC_NC1 / AAC_NC2)");
  return AAC_OK;
}

extern "C" int aac_precond_apply(aac_ctx* ctx, int method, int k, const double* r, double* z) {
  if (!ctx || !r || !z || r == z) return aac_fail(ctx, AAC_EINVAL, "aac_precond_apply: bad pointers");
  bool f32 = false;
  AAC_TRY(split_f32(ctx, &method, &f32));
  F32Scope fs(ctx, f32);
  if (k < 1 && method != AAC_EXACT) return aac_fail(ctx, AAC_EINVAL, "inner iteration count k must be >= 1");
  AAC_TRY(check_alpha(ctx));
  NvtxRange nv("aac_precond_apply");
  StreamScope ss(ctx);
  if (method == AAC_NC1 || method == AAC_NC2) return nc_apply(ctx, method, k, r, z, false);
  if (method == AAC_EXACT) return exact_apply(ctx, r, z, false, 0);
  if (method == AAC_SP) {
    AAC_TRY(sp_prepare(ctx, k));
    const long long N = ctx->geo.N;
    const Dft D = make_dft(ctx);
    const double V = 8.0 * ctx->ell * N;
    if (ctx->ell <= 10)
      LAUNCH(ctx, KID_FWD, 2 * V, (k_forward<10><<<grid1d(N, 256), 256, 0, ctx->stream>>>(N, D, r, ctx->d_what)));
    else
      LAUNCH(ctx, KID_FWD, 2 * V, (k_forward<16><<<grid1d(N, 256), 256, 0, ctx->stream>>>(N, D, r, ctx->d_what)));
    return sp_solve(ctx, k, z, 0, nullptr);
  }
  return aac_fail(ctx, AAC_EINVAL, "unknown method %d", method);
}

// ------------------------------------------------------------------------------------------
// GMRES
template <int DIM, int ELLC, bool TMA, bool FUSED>
static int launch_arnoldi(aac_ctx* ctx, int host_j) {
  const Geo& g = ctx->geo;
  const int ldh = ctx->max_krylov + 1;
  const long long L = (long long)ctx->ell * g.N;
  const double V = 8.0 * ctx->ell * g.N, C = 8.0 * ctx->dim * g.N;
  KAParams P{ctx->d_Z, ctx->d_V, ctx->d_W, L, ctx->d_part,
             ctx->d_halo, ctx->d_halo + (long long)ctx->ell * g.S, arnoldi_ctx(ctx)};
  if (!FUSED && ctx->varying) {      // varying blocks: each plane its own operator
    AAC_TRY(matvec_var(ctx, ctx->d_Z, L, reinterpret_cast<const int*>(ctx->d_st), ctx->d_W));
    ctx->sweeps += ctx->ell;
  } else if (!FUSED && DIM == 2 && matvec_tile_on(ctx)) {
    AAC_TRY(launch_matvec_tile(ctx, ctx->d_Z, L, reinterpret_cast<const int*>(ctx->d_st), ctx->d_W, 2 * V + C));
    ctx->sweeps += ctx->ell;
  } else if (!FUSED && DIM == 2 && matvec_rows_ry(ctx)) {
    AAC_TRY(launch_matvec_rows(ctx, matvec_rows_ry(ctx), ctx->d_Z, L, reinterpret_cast<const int*>(ctx->d_st),
                               ctx->d_W, ctx->d_halo, ctx->d_halo + (long long)ctx->ell * g.S, 2 * V + C));
    ctx->sweeps += ctx->ell;
  } else if (!FUSED) {               // w = calA Z_j by the stencil kernel (j read on the device)
    const bool v2 = vec2(ctx);
    const dim3 gm(grid1d(g.nx / (v2 ? 2 : 1), 256), g.ny, g.nz);
    const int* jd = reinterpret_cast<const int*>(ctx->d_st);
    const double* hlo = ctx->d_halo;
    const double* hhi = ctx->d_halo + (long long)ctx->ell * g.S;
    if (v2)
      LAUNCH(ctx, KID_MATVEC, 2 * V + C, (k_matvec<DIM, 2><<<gm, 256, 0, ctx->stream>>>(g, ctx->ell, ctx->d_Z, L, jd, ctx->d_W, hlo, hhi)));
    else
      LAUNCH(ctx, KID_MATVEC, 2 * V + C, (k_matvec<DIM, 1><<<gm, 256, 0, ctx->stream>>>(g, ctx->ell, ctx->d_Z, L, jd, ctx->d_W, hlo, hhi)));
    ctx->sweeps += ctx->ell;
  }
  const size_t smem = (arnoldi_ring_doubles<ELLC>() + (size_t)(AW + 1) * 2 * ldh) * sizeof(double);
  // persistent grid: exactly the resident capacity (no partial second wave)
  static thread_local int occ_cache[3][4][2][2] = {};
  int& occ = occ_cache[ELLC == 10 ? 0 : (ELLC == 12 ? 1 : 2)][DIM][TMA ? 1 : 0][FUSED ? 1 : 0];
  AAC_TRY(smem_optin(ctx, k_arnoldi<DIM, ELLC, TMA, FUSED>, smem));
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_arnoldi<DIM, ELLC, TMA, FUSED>, AT + 32, smem);
    if (occ < 1) occ = 1;
  }
  const long long ntile = (long long)((g.nx + AT - 1) / AT) * g.ny * g.nz;
  const int grid = (int)std::min<long long>((long long)occ * ctx->num_sms, ARN_NGF > 2 ? ntile * ARN_NGF / 2 : ntile);
  // algorithmic bytes: Z_j + C in (fused) or W in (split), W out (fused), basis V_0..V_j in
  const double bytes = FUSED ? (host_j + 3) * V + C : (host_j + 2) * V;
  LAUNCH(ctx, KID_ARNOLDI, bytes, (k_arnoldi<DIM, ELLC, TMA, FUSED><<<grid, AT + 32, smem, ctx->stream>>>(g, ctx->ell, P)));
  return AAC_OK;
}

template <int DIM>
static int arnoldi_dim(aac_ctx* ctx, int host_j) {
  const bool tma = (ctx->geo.nx % 2) == 0;          // row-aligned tiles start at row * nx
  // split (k_matvec + dot kernel) by default; AAC_FUSED_ARNOLDI=1 keeps the stencil in-kernel
  static const bool fused_env = getenv("AAC_FUSED_ARNOLDI") != nullptr;
  const bool fused = fused_env && !ctx->varying;   // (the fused stencil knows one operator)
  if (ctx->ell <= 10) {
    if (fused) return tma ? launch_arnoldi<DIM, 10, true, true>(ctx, host_j) : launch_arnoldi<DIM, 10, false, true>(ctx, host_j);
    return tma ? launch_arnoldi<DIM, 10, true, false>(ctx, host_j) : launch_arnoldi<DIM, 10, false, false>(ctx, host_j);
  }
  if (ctx->ell <= 12) {
    if (fused) return tma ? launch_arnoldi<DIM, 12, true, true>(ctx, host_j) : launch_arnoldi<DIM, 12, false, true>(ctx, host_j);
    return tma ? launch_arnoldi<DIM, 12, true, false>(ctx, host_j) : launch_arnoldi<DIM, 12, false, false>(ctx, host_j);
  }
  if (fused) return tma ? launch_arnoldi<DIM, 16, true, true>(ctx, host_j) : launch_arnoldi<DIM, 16, false, true>(ctx, host_j);
  return tma ? launch_arnoldi<DIM, 16, true, false>(ctx, host_j) : launch_arnoldi<DIM, 16, false, false>(ctx, host_j);
}

static int arnoldi_impl(aac_ctx* ctx, int host_j) {
  switch (ctx->dim) {
    case 1: return arnoldi_dim<1>(ctx, host_j);
    case 2: return arnoldi_dim<2>(ctx, host_j);
    default: return arnoldi_dim<3>(ctx, host_j);
  }
}

// One Arnoldi step (device j): precondition V_j -> Z_j (forward fused with the update that
// forms V_j), then w = calA Z_j with the CGS2 projections and Gram column.
static int arnoldi_step(aac_ctx* ctx, int method, int k, int host_j) {
  int rc = AAC_OK;
  ctx->z_ghost = false;
  if (method == AAC_SP) {
    const double V = 8.0 * ctx->ell * ctx->geo.N;
    rc = forward_step(ctx, (host_j + 3) * V);
    if (rc != AAC_OK) return rc;
    AAC_TRY(sp_solve(ctx, k, ctx->d_Z, (long long)ctx->ell * ctx->geo.N, ctx->d_st));
  } else if (method == AAC_EXACT) {
    rc = exact_apply(ctx, nullptr, ctx->d_Z, true, host_j);
  } else {
    rc = nc_apply(ctx, method, k, nullptr, ctx->d_Z, true, host_j);
  }
  if (rc != AAC_OK) return rc;                         // error, or the solve finished
  // Z_j's halo: exchanged, unless the wavefront formed it from its ghost rows (ghost mode)
  if (ctx->nranks > 1 && !ctx->z_ghost) AAC_TRY(halo_planes(ctx, ctx->d_Z + (long long)host_j * ctx->ell * ctx->geo.N));
  ctx->z_ghost = false;
  AAC_TRY(arnoldi_impl(ctx, host_j));
  if (ctx->multi()) {
    AAC_TRY(comm_allreduce(ctx, ctx->d_red, 2 * (host_j + 1), ncclSum));
    LAUNCH(ctx, KID_SCALAR, 0, k_scalar_cgs2<<<1, 128, 0, ctx->stream>>>(arnoldi_ctx(ctx)));
  }
  return AAC_OK;
}

// IterState (or n doubles) device -> pinned host without a copy engine (k_publish)
static int publish(aac_ctx* ctx, const void* dsrc, void* hdst, size_t bytes) {
  void* hd = nullptr;
  CUDA_TRY(ctx, cudaHostGetDevicePointer(&hd, hdst, 0));
  const int n = (int)(bytes / sizeof(unsigned));
  LAUNCH(ctx, KID_SCALAR, 0, k_publish<<<1, 32, 0, ctx->stream>>>(static_cast<const unsigned*>(dsrc),
                                                                  static_cast<unsigned*>(hd), n));
  return AAC_OK;
}

static int get_graph(aac_ctx* ctx, int method, int k, GraphEntry** out) {
  for (auto& ge : ctx->graphs)
    if (ge.method == method && ge.k == k) { *out = &ge; return AAC_OK; }
  const long long l0 = ctx->launches;
  CUDA_TRY(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  // one rank: k_arnoldi's last CTA publishes the state itself (AAC_PUB_KERNEL=1: a k_publish node)
  static const bool pub_kernel = getenv("AAC_PUB_KERNEL") && atoi(getenv("AAC_PUB_KERNEL")) == 1;
  if (!ctx->multi() && !pub_kernel) {
    void* hd = nullptr;
    if (cudaHostGetDevicePointer(&hd, ctx->h_st, 0) == cudaSuccess) ctx->pub_fold = static_cast<unsigned*>(hd);
  }
  int rc = arnoldi_step(ctx, method & ~AAC_F32, k, 0);       // (the key keeps the AAC_F32 flag)
  const bool folded = ctx->pub_fold != nullptr;
  ctx->pub_fold = nullptr;
  if (rc == AAC_OK && !folded) rc = publish(ctx, ctx->d_st, ctx->h_st, sizeof(IterState));
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
  if (rc != AAC_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (e != cudaSuccess) return aac_fail(ctx, AAC_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
  GraphEntry ge{method, k, nullptr, (int)(ctx->launches - l0)};
  ctx->launches = l0;                      // capture launched nothing
  e = cudaGraphInstantiate(&ge.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return aac_fail(ctx, AAC_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
  ctx->graphs.push_back(ge);
  *out = &ctx->graphs.back();
  return AAC_OK;
}

static int gmres_impl(aac_ctx* ctx, int method, int k, const double* b, double* x, double rtol,
                      int maxit, aac_gmres_info* info) {
  NvtxRange nv("aac_gmres");
  bool f32 = false;
  AAC_TRY(split_f32(ctx, &method, &f32));
  F32Scope fs(ctx, f32);
  if (maxit < 1 || maxit > ctx->max_krylov)
    return aac_fail(ctx, AAC_EINVAL, "maxit must be in [1, max_krylov=%d]", ctx->max_krylov);
  if (!(rtol >= 0.0)) return aac_fail(ctx, AAC_EINVAL, "rtol must be >= 0");
  if (method != AAC_NC1 && method != AAC_NC2 && method != AAC_SP && method != AAC_EXACT)
    return aac_fail(ctx, AAC_EINVAL, "unknown method %d", method);
  if (k < 1 && method != AAC_EXACT) return aac_fail(ctx, AAC_EINVAL, "k must be >= 1");
  AAC_TRY(check_alpha(ctx));
  if (method == AAC_EXACT) AAC_TRY(exact_prepare(ctx));
  const long long N = ctx->geo.N, L = (long long)ctx->ell * N;
  const int ldh = ctx->max_krylov + 1;
  const long long sweeps0 = ctx->sweeps;
  if (method == AAC_SP) AAC_TRY(sp_prepare(ctx, k));
  // init: V_0 = b (raw), state, Givens/Gram workspaces
  IterState init{};
  init.maxit = maxit;
  init.rtol = rtol;
  *ctx->h_st = init;
  // (kernels, not copy engines: a concurrent host transfer of aac_gmres_host_batch must not
  // delay the solve)
  LAUNCH(ctx, KID_SCALAR, 0, k_set_state<<<1, 1, 0, ctx->stream>>>(ctx->d_st, init));
  LAUNCH(ctx, KID_AXPY, 16.0 * L,
         k_copy<<<std::min<long long>(4LL * ctx->num_sms, grid1d(L, 256)), 256, 0, ctx->stream>>>(b, ctx->d_V, L));
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_giv, 0, 6LL * ldh * sizeof(double), ctx->stream));
  int alloc_sum = 0;
  if (method != AAC_EXACT) {
    int al[AAC_MAX_ELL];
    allocation(ctx, method, k, al);
    for (int j = 0; j < ctx->ell; ++j) alloc_sum += al[j];
  }
  GraphEntry* ge = nullptr;
  const bool graphs = ctx->use_graphs && !ctx->prof;
  if (graphs) AAC_TRY(get_graph(ctx, method | (f32 ? AAC_F32 : 0), k, &ge));
  // Arnoldi steps. Graph path: replay one captured step per iteration and poll the state of
  // the PREVIOUS step (speculative: a step launched after convergence returns at once).
  int it = 0;
  for (; it < maxit; ++it) {
    if (graphs) {
      CUDA_TRY(ctx, cudaGraphLaunch(ge->exec, ctx->stream));
      ctx->launches += ge->nodes;
      CUDA_TRY(ctx, cudaEventRecord(ctx->ev_it[it & 1], ctx->stream));
      if (it >= 1) {
        AAC_TRY(comm_wait_event(ctx, ctx->ev_it[(it - 1) & 1]));
        if (ctx->h_st->done) break;
      }
    } else {
      ctx->eager_poll = true;
      const int rc = arnoldi_step(ctx, method, k, it);
      ctx->eager_poll = false;
      if (rc == AAC_STEP_DONE) break;
      AAC_TRY(rc);
      AAC_TRY(publish(ctx, ctx->d_st, ctx->h_st, sizeof(IterState)));
      AAC_TRY(comm_sync(ctx));
      if (ctx->h_st->done) break;
    }
  }
  // finalise the last column and form x = sum y_i Z_i. The finalising forward step does work
  // only when the loop stopped at maxit; after convergence (h_st->done, final) it is skipped.
  if (!ctx->h_st->done) {
    // finalise the last Arnoldi column (same kernel; its transform output is unused)
    AAC_TRY(launch_fwd_upd(ctx, 0, true));
    if (ctx->multi()) {
      AAC_TRY(comm_allreduce(ctx, ctx->d_red, 1, ncclSum));
      LAUNCH(ctx, KID_SCALAR, 0, k_scalar_norm<<<1, 1, 0, ctx->stream>>>(arnoldi_ctx(ctx)));
    }
  }
  double* yy = ctx->d_giv + 3 * ldh;
  LAUNCH(ctx, KID_SCALAR, 0,
         k_backsub<<<1, 32, 0, ctx->stream>>>(ctx->d_st, ldh, ctx->d_H, ctx->d_giv + 2 * ldh, ctx->d_giv + 4 * ldh, yy));
  AAC_TRY(publish(ctx, ctx->d_st, ctx->h_st, sizeof(IterState)));
  AAC_TRY(comm_sync(ctx));
  const IterState fin = *ctx->h_st;
  const int m = fin.m;
  if (m > 0)
    LAUNCH(ctx, KID_AXPY, 8.0 * L * (m + 1),
           k_lincomb<<<grid1d((L + 1) / 2, 256), 256, 0, ctx->stream>>>(ctx->d_Z, L, ctx->d_st, yy, x, L));
  else
    CUDA_TRY(ctx, cudaMemsetAsync(x, 0, L * sizeof(double), ctx->stream));
  const bool converged = fin.relres <= rtol || fin.hn == 0.0 || fin.beta == 0.0;
  double rtrue = 0.0;
  if (info && fin.beta > 0.0) {
    // true residual ||b - calA x|| / ||b|| (one extra apply, not an Arnoldi step)
    AAC_TRY(matvec_impl(ctx, x, ctx->d_tmp));
    const int nb = std::min<int>(ctx->num_sms * 4, (int)grid1d(L, 256));
    LAUNCH(ctx, KID_AXPY, 16.0 * L, k_diffnorm<<<nb, 256, 0, ctx->stream>>>(b, ctx->d_tmp, L, ctx->d_part));
    LAUNCH(ctx, KID_REDUCE, 0, k_sum<<<1, 256, 0, ctx->stream>>>(ctx->d_part, nb, ctx->d_stat));
    AAC_TRY(comm_allreduce(ctx, ctx->d_stat, 1, ncclSum));
    AAC_TRY(publish(ctx, ctx->d_stat, ctx->h_stat, sizeof(double)));
    AAC_TRY(comm_sync(ctx));
    rtrue = sqrt(ctx->h_stat[0]) / fin.beta;
  }
  if (info) {
    info->iters = m;
    info->converged = converged ? 1 : 0;
    info->relres_est = fin.relres;
    info->relres_true = rtrue;
    info->matvecs_paper_units = (long long)m * (ctx->ell + (method == AAC_SP ? sp_paper_matvecs(ctx, k) : alloc_sum));
    info->stencil_sweeps = ctx->sweeps - sweeps0;
  }
  return converged ? AAC_OK : AAC_ENOCONV;
}

extern "C" int aac_gmres(aac_ctx* ctx, int method, int k, const double* b, double* x, double rtol,
                         int maxit, aac_gmres_info* info) {
  if (!ctx || !b || !x || b == x) return aac_fail(ctx, AAC_EINVAL, "aac_gmres: bad pointers");
  StreamScope ss(ctx);
  return gmres_impl(ctx, method, k, b, x, rtol, maxit, info);
}

extern "C" int aac_gmres_host(aac_ctx* ctx, int method, int k, const double* b_host, double* x_host,
                              double rtol, int maxit, aac_gmres_info* info) {
  if (!ctx || !b_host || !x_host) return aac_fail(ctx, AAC_EINVAL, "aac_gmres_host: bad pointers");
  const long long L = (long long)ctx->ell * ctx->geo.N;
  if (!ctx->d_bx && cudaMalloc((void**)&ctx->d_bx, 2 * L * sizeof(double)) != cudaSuccess) {
    ctx->d_bx = nullptr;
    cudaGetLastError();
    return aac_fail(ctx, AAC_ENOMEM, "staging allocation failed");
  }
  StreamScope ss(ctx);
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_bx, b_host, L * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  const int rc = gmres_impl(ctx, method, k, ctx->d_bx, ctx->d_bx + L, rtol, maxit, info);
  if (rc < 0) return rc;
  CUDA_TRY(ctx, cudaMemcpyAsync(x_host, ctx->d_bx + L, L * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return rc;
}

// Several right-hand sides from the host, copies overlapped with the solves: the H2D copy of
// b_{i+1} and the D2H copy of x_{i-1} run on a copy stream while system i is solved (two device
// slots each for b and x; events order every reuse of a slot).
extern "C" int aac_gmres_host_batch(aac_ctx* ctx, int method, int k, int nrhs, const double* const* b_host,
                                    double* const* x_host, double rtol, int maxit, aac_gmres_info* info) {
  if (!ctx || nrhs < 0 || (nrhs > 0 && (!b_host || !x_host)))
    return aac_fail(ctx, AAC_EINVAL, "aac_gmres_host_batch: bad arguments");
  for (int i = 0; i < nrhs; ++i)
    if (!b_host[i] || !x_host[i]) return aac_fail(ctx, AAC_EINVAL, "aac_gmres_host_batch: NULL vector %d", i);
  if (nrhs == 0) return AAC_OK;
  const long long L = (long long)ctx->ell * ctx->geo.N;
  const size_t bytes = L * sizeof(double);
  if (!ctx->d_bb && cudaMalloc((void**)&ctx->d_bb, 4 * bytes) != cudaSuccess) {
    ctx->d_bb = nullptr;
    cudaGetLastError();
    return aac_fail(ctx, AAC_ENOMEM, "batch staging allocation failed");
  }
  if (!ctx->cstream) {
    CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
    for (auto& e : ctx->ev_cp) CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaEvent_t* ev_in = ctx->ev_cp;
  cudaEvent_t* ev_done = ctx->ev_cp + 2;
  cudaEvent_t* ev_out = ctx->ev_cp + 4;
  auto B = [&](int s) { return ctx->d_bb + (long long)s * L; };
  auto X = [&](int s) { return ctx->d_bb + (long long)(2 + s) * L; };
  StreamScope ss(ctx);
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->cstream, ctx->ev_in, 0));   // after the caller's work
  CUDA_TRY(ctx, cudaMemcpyAsync(B(0), b_host[0], bytes, cudaMemcpyHostToDevice, ctx->cstream));
  CUDA_TRY(ctx, cudaEventRecord(ev_in[0], ctx->cstream));
  int worst = AAC_OK;
  for (int i = 0; i < nrhs; ++i) {
    const int s = i & 1;
    if (i + 1 < nrhs) {                          // prefetch b_{i+1} into the other slot
      const int s1 = (i + 1) & 1;
      if (i >= 1) CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->cstream, ev_done[s1], 0));   // solve i-1 done with it
      CUDA_TRY(ctx, cudaMemcpyAsync(B(s1), b_host[i + 1], bytes, cudaMemcpyHostToDevice, ctx->cstream));
      CUDA_TRY(ctx, cudaEventRecord(ev_in[s1], ctx->cstream));
    }
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ev_in[s], 0));
    if (i >= 2) CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ev_out[s], 0));       // x_{i-2} copied out
    const int rc = gmres_impl(ctx, method, k, B(s), X(s), rtol, maxit, info ? info + i : nullptr);
    if (rc < 0) {
      cudaStreamSynchronize(ctx->cstream);
      return rc;
    }
    worst = std::max(worst, rc);
    CUDA_TRY(ctx, cudaEventRecord(ev_done[s], ctx->stream));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->cstream, ev_done[s], 0));
    CUDA_TRY(ctx, cudaMemcpyAsync(x_host[i], X(s), bytes, cudaMemcpyDeviceToHost, ctx->cstream));
    CUDA_TRY(ctx, cudaEventRecord(ev_out[s], ctx->cstream));
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->cstream));
  return worst;
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
extern "C" int aac_profile_flops(aac_ctx* ctx, int id, double* model_flops) {
  if (!ctx || id < 0 || id >= KID_COUNT || !model_flops) return aac_fail(ctx, AAC_EINVAL, "bad profile id");
  *model_flops = ctx->prof_flops[id];
  return AAC_OK;
}
extern "C" int aac_profile_reset(aac_ctx* ctx) {
  if (!ctx) return aac_fail(nullptr, AAC_EINVAL, "NULL ctx");
  AAC_TRY(prof_collect(ctx));
  for (int i = 0; i < KID_COUNT; ++i) {
    ctx->prof_ms[i] = 0;
    ctx->prof_n[i] = 0;
    ctx->prof_bytes[i] = 0;
    ctx->prof_flops[i] = 0;
  }
  return AAC_OK;
}
extern "C" long long aac_launch_count(const aac_ctx* ctx) { return ctx ? ctx->launches : 0; }
extern "C" int aac_comm_kind(const aac_ctx* ctx) {
  if (!ctx) return 0;
  if (ctx->host_tr) return 2;
  return ctx->nccl_comm ? 1 : 0;
}

#include "paper_mode.cuh"   // aac_set_boundary / aac_set_bounds / aac_ci (N1)
