// sp.cuh -- saddle-point inner solver P_SP (§4; §5.1, 694-697).
//
// Per packed Fourier block (after the same gamma-scale + DFT as NC):
//   complex block k (1 <= k < ell/2): lambda = conj(Lambda_k) (Im lambda > 0), b = conj(w_k);
//     MINRES (k_in iterations from 0) on the real saddle system Eq. (eq:saddlesystem)
//       S [u; v] = [Im lam u + Psi v; Psi u - Im lam v] = [-Im b; Re b] = [Im w_k; Re w_k],
//       Psi = A - Re lam, preconditioned by P_D = diag(M, M) (Eq. eq:minresprecond),
//       M ~ (A + (Im lam - Re lam) I)^{-1} = one V-cycle;  y_k = conj(u - i v) = u + i v.
//   real blocks k = 0, ell/2: PCG (k_in iterations) on (A - Lambda_k) y = w_k, M = one V-cycle
//     of A - Lambda_k.
// then the inverse DFT + gamma^{-1}. Reading R16: V(1,1) cycle, damped Jacobi
// omega = 0.8, aggregation by 2 per axis with Galerkin coarse operators (a coarse face weight is
// the sum of the fine faces between the two aggregates; the identity becomes the child count),
// dense solve once every axis <= 8. The oracle (oracle/saddle.py) follows the same algorithm
// with scipy sparse products; it shares no code with this file.
//
// All blocks advance in lock step; every kernel is batched over the ell packed planes
// (blockIdx.y = plane or block); the Krylov scalars live on the device and are updated by the
// last CTA of the kernel that produces the dot products (fixed-order sums).
#pragma once

#include <algorithm>
#include <vector>

#include "krylov.cuh"
#include "nc.cuh"
#include "stencil.cuh"

constexpr double SP_OMEGA = 0.8;
constexpr int SP_COARSE_MAX_AXIS = 8;
constexpr int SP_T = 256;

struct SpBlk {                 // device scalars of one packed block
  // MINRES (Elman-Silvester-Wathen form, as oracle/saddle.py::minres)
  double gamma, gamma_prev, eta, s_prev, s_cur, c_prev, c_cur, delta;
  double a1, a2, a3, xcoef, dcoef, vcoef;
  // PCG (as oracle/saddle.py::pcg)
  double rho, alpha, beta;
  int stop;                    // 1: the oracle's loop has broken out; 2: break after this update
  int pad;
};

struct SpConst {               // per-block constants, passed by value
  double lre[AAC_MAX_BLK], lim[AAC_MAX_BLK];   // lambda (complex blocks: conj Lambda_k)
  double s[AAC_MAX_ELL];                        // MG shift per plane: A + s I
  int ell;
};

struct SpLevel {               // one multigrid level (device arrays)
  Geo g;                       // extents + face weights (lower-face convention); has_lo / has_hi
                               // on the slab-decomposed levels of a multi-rank run
  double* cnt;                 // Galerkin image of I: fine cells per aggregate
  double* b;                   // [ell][N] right-hand sides (levels >= 1)
  double* x;                   // [ell][N] pre-smoothed iterate
  double* x2;                  // [ell][N] post-smoothed iterate (the level's result, levels >= 1)
  double* dinv = nullptr;      // [h+1][N] 1 / diag(A_l + s_k I) per block shift (setup; the
                               // smoother multiplies instead of dividing -- fp64 division is
                               // ~10x the cost of the rest of the point update)
  int local = 1;               // 1: this rank's slab (halo exchanges); 0: the global level
  Geo gl{};                    // gathered level: this rank's slab of it (extents only) ...
  long long goff = 0;          // ... and its offset in the global arrays (points)
};

struct SpfRed {               // two-level reduction of the fused kernels (sp_fused.cuh):
  double* gpart;               // group partials [nq][ngroups]
  unsigned* gtick;             // group tickets (SPF_TICK_STRIDE apart), then the global one
};

struct SpPlan {
  int ell = 0, h = 0;
  std::vector<SpLevel> lev;
  std::vector<void*> owned;    // device allocations
  double* minv = nullptr;      // [h+1][nc][nc] dense inverses of the coarsest operator
  int nc = 0;
  SpConst K;
  double* X = nullptr;
  double* Vb[3] = {nullptr, nullptr, nullptr};
  double* Zb[2] = {nullptr, nullptr};
  double* Wb[3] = {nullptr, nullptr, nullptr};
  double *SZ = nullptr, *R = nullptr, *P = nullptr, *Zr = nullptr;
  SpBlk* blk = nullptr;        // [h+1]
  double* part = nullptr;      // partials [planes or blocks][tiles]
  unsigned* tick = nullptr;
  double* red = nullptr;       // multi-rank: local sums for the all-reduce (AAC_MAX_ELL)
  SpfRed red2{};               // two-level reduction workspace of the fused kernels (sp_fused.cuh)
  int gather = -1;             // multi-rank: index of the gathered (first global) level
};

// ------------------------------------------------------------------------------------------
__device__ __forceinline__ int sp_block_of(int ell, int pl) {
  const int h = ell / 2;
  return pl == 0 ? 0 : (pl == ell - 1 ? h : (pl + 1) / 2);
}

// A_l(s) u at the point: m u_p + sum_f w_f (u_p - u_nb), m = (1 + s) cnt_p
// hlo / hhi: the plane's halo layers (slab-decomposed levels; unused when g has no neighbours)
template <int DIM>
__device__ __forceinline__ double mg_apply(const Geo& g, const PtV<DIM, 1>& q, const double* u, double m,
                                           const double* hlo = nullptr, const double* hhi = nullptr) {
  double a[1], c[1];
  apply_Av<DIM, 1>(g, q, u, hlo, hhi, a, c);
  return a[0] + (m - 1.0) * c[0];
}

template <int DIM>
__device__ __forceinline__ double diag_of(const PtV<DIM, 1>& q, double m) {
  double d = m + q.wx[0] + q.wx[1];
  if constexpr (DIM >= 2) d += q.wym[0] + q.wyp[0];
  if constexpr (DIM >= 3) d += q.wzm[0] + q.wzp[0];
  return d;
}

struct MgIo {                  // per-plane fine-level pointers
  const double* in[AAC_MAX_ELL];
  double* out[AAC_MAX_ELL];
};

struct SpStepCtx {
  SpBlk* blk;
  double* part;
  unsigned* tick;
  SpConst K;
  int phase;                   // step B: 0 = initial (gamma / rho), 1 = iteration
  const IterState* st;
  double* red;                 // multi-rank: the last CTA stores the local sums here (an
                               // all-reduce and k_sp_scalar follow); NULL: it runs the step
  const double* hlo;           // level-0 halo layers (slab decomposition), plane stride g.S
  const double* hhi;
};

// ---- scalar steps (thread 0 of the last CTA) ---------------------------------------------
// A: after K1. tot[kb] = <S z, z> (complex) or <p, A' p> (real).
__device__ void sp_scalar_A(const SpStepCtx& S, const double* tot) {
  const int h = S.K.ell / 2;
  for (int kb = 0; kb <= h; ++kb) {
    SpBlk& b = S.blk[kb];
    if (b.stop == 2) b.stop = 1;
    if (kb == 0 || kb == h) {
      if (!b.stop) b.alpha = b.rho / tot[kb];
    } else {
      b.delta = tot[kb];
      b.dcoef = b.delta / b.gamma;
      b.vcoef = b.gamma / b.gamma_prev;
    }
  }
}

// B: after the V-cycle. tot[plane] = <M v, v> per plane (complex blocks: two planes).
__device__ void sp_scalar_B(const SpStepCtx& S, const double* tot) {
  const int ell = S.K.ell, h = ell / 2;
  for (int kb = 0; kb <= h; ++kb) {
    SpBlk& b = S.blk[kb];
    if (kb == 0 || kb == h) {
      const double rho_new = tot[kb == 0 ? 0 : ell - 1];
      if (S.phase == 0) {
        b.rho = rho_new;
        b.stop = (rho_new == 0.0) ? 1 : 0;
      } else if (!b.stop) {
        b.beta = rho_new / b.rho;
        b.rho = rho_new;
        if (rho_new == 0.0) b.stop = 1;
      }
      continue;
    }
    const double d = tot[2 * kb - 1] + tot[2 * kb];
    const double gn = sqrt(d > 0.0 ? d : 0.0);
    if (S.phase == 0) {
      b.gamma = gn;
      b.gamma_prev = 1.0;
      b.eta = gn;
      b.s_prev = b.s_cur = 0.0;
      b.c_prev = b.c_cur = 1.0;
      b.stop = (gn == 0.0) ? 1 : 0;
      continue;
    }
    if (b.stop) continue;
    const double a0 = b.c_cur * b.delta - b.c_prev * b.s_cur * b.gamma;
    const double a1 = sqrt(a0 * a0 + gn * gn);
    const double a2 = b.s_cur * b.delta + b.c_prev * b.c_cur * b.gamma;
    const double a3 = b.s_prev * b.gamma;
    const double c_next = a0 / a1, s_next = gn / a1;
    b.a1 = a1;
    b.a2 = a2;
    b.a3 = a3;
    b.xcoef = c_next * b.eta;
    b.eta = -s_next * b.eta;
    b.gamma_prev = b.gamma;            // K6 scales z by 1/gamma_prev (= the old gamma)
    b.gamma = gn;
    b.s_prev = b.s_cur;
    b.s_cur = s_next;
    b.c_prev = b.c_cur;
    b.c_cur = c_next;
    if (gn == 0.0) b.stop = 2;
  }
}

// Per-(plane or block, CTA) partials; the last CTA sums in a fixed order and runs a step.
__device__ __forceinline__ void sp_reduce(const SpStepCtx& S, double v, bool stepB) {
  __shared__ double red[SP_T / 32];
  __shared__ bool last;
  __shared__ double tot[AAC_MAX_ELL];
  v = warp_sum(v);
  const int t = threadIdx.x;
  if ((t & 31) == 0) red[t >> 5] = v;
  __syncthreads();
  const int ntile = gridDim.x;
  if (t == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    S.part[(long long)blockIdx.y * ntile + blockIdx.x] = s;
    __threadfence();
    const unsigned tk = atomicAdd(S.tick, 1u);
    last = (tk == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int q = 0; q < (int)gridDim.y; ++q) {
    const double s = block_sum_fixed(S.part + (long long)q * ntile, ntile);
    if (t == 0) tot[q] = s;
  }
  if (t == 0) {
    *S.tick = 0;
    if (S.red) {
      for (int q = 0; q < (int)gridDim.y; ++q) S.red[q] = tot[q];
    } else if (stepB) {
      sp_scalar_B(S, tot);
    } else {
      sp_scalar_A(S, tot);
    }
  }
}

// Multi-rank: the scalar step on the all-reduced sums.
__global__ void k_sp_scalar(SpStepCtx S, int stepB) {
  if (S.st && S.st->done) return;
  double tot[AAC_MAX_ELL];
  for (int q = 0; q < AAC_MAX_ELL; ++q) tot[q] = S.red[q];
  if (stepB) sp_scalar_B(S, tot);
  else sp_scalar_A(S, tot);
}

// ---- multigrid kernels (grid: tiles x planes) ----------------------------------------------
// Slab-decomposed levels carry has_lo / has_hi in their Geo and read the neighbours' boundary
// layers from hlo / hhi (plane stride g.S).
// x = omega b / D (pre-smoothing from zero)
template <int DIM>
__global__ void __launch_bounds__(SP_T) k_mg_smooth0(Geo g, const double* __restrict__ dinv, SpConst K,
                                                     MgIo io, const double* bl, double* xl,
                                                     const IterState* st) {
  if (st && st->done) return;
  const int pl = blockIdx.y;
  const long long p = (long long)blockIdx.x * SP_T + threadIdx.x;
  if (p >= g.N) return;
  const double* b = bl ? bl + (long long)pl * g.N : io.in[pl];
  xl[(long long)pl * g.N + p] = SP_OMEGA * b[p] * dinv[(long long)sp_block_of(K.ell, pl) * g.N + p];
}

// b_{l+1} = P^T (b - A_l x): one thread per COARSE point sums its children
// gc: this rank's part of the coarse level; the result goes to bc[pl * cstride + coff + pc]
// (cstride / coff: the plane stride and slab offset of the coarse array -- the global array of
// a gathered level, or the local one).
template <int DIM>
__global__ void __launch_bounds__(SP_T) k_mg_restrict(Geo g, const double* __restrict__ cnt, Geo gc,
                                                      SpConst K, MgIo io, const double* bl,
                                                      const double* xl, double* bc,
                                                      const IterState* st, const double* hlo,
                                                      const double* hhi, long long cstride, long long coff) {
  if (st && st->done) return;
  const int pl = blockIdx.y;
  const long long pc = (long long)blockIdx.x * SP_T + threadIdx.x;
  if (pc >= gc.N) return;
  const int X = (int)(pc % gc.nx);
  const long long rr = pc / gc.nx;
  const int Y = (int)(rr % gc.ny), Z = (int)(rr / gc.ny);
  const double s = K.s[pl];
  const double* b = bl ? bl + (long long)pl * g.N : io.in[pl];
  const double* x = xl + (long long)pl * g.N;
  double acc = 0.0;
  for (int dz = 0; dz < (DIM >= 3 ? 2 : 1); ++dz)
    for (int dy = 0; dy < (DIM >= 2 ? 2 : 1); ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const int fx = 2 * X + dx, fy = DIM >= 2 ? 2 * Y + dy : 0, fz = DIM >= 3 ? 2 * Z + dz : 0;
        if (fx >= g.nx || fy >= g.ny || fz >= g.nz) continue;
        const long long p = ((long long)fz * g.ny + fy) * g.nx + fx;
        PtV<DIM, 1> q;
        load_ptv<DIM, 1>(g, p, q);
        acc += b[p] - mg_apply<DIM>(g, q, x, (1.0 + s) * cnt[p], hlo + (long long)pl * g.S,
                                    hhi + (long long)pl * g.S);
      }
  bc[(long long)pl * cstride + coff + pc] = acc;
}

// ---- plane-pair variants: one CTA per (tile, plane pair) -- the pair shares the point's face
// weights, aggregate count and index arithmetic (loaded once for both planes) and gives each
// thread two independent chains. Pair 0 = planes (0, ell-1) (the real blocks), pair k = the
// (Re, Im) planes of complex block k.
__device__ __forceinline__ void sp_pair(int ell, int pi, int& p0, int& p1) {
  p0 = pi == 0 ? 0 : 2 * pi - 1;
  p1 = pi == 0 ? ell - 1 : 2 * pi;
}

template <int DIM>
__global__ void __launch_bounds__(SP_T) k_mg_restrict_pair(Geo g, const double* __restrict__ cnt, Geo gc,
                                                           SpConst K, MgIo io, const double* bl,
                                                           const double* xl, double* bc,
                                                           const IterState* st, const double* hlo,
                                                           const double* hhi, long long cstride,
                                                           long long coff) {
  if (st && st->done) return;
  int pa, pb;
  sp_pair(K.ell, blockIdx.y, pa, pb);
  const long long pc = (long long)blockIdx.x * SP_T + threadIdx.x;
  if (pc >= gc.N) return;
  const int X = (int)(pc % gc.nx);
  const long long rr = pc / gc.nx;
  const int Y = (int)(rr % gc.ny), Z = (int)(rr / gc.ny);
  const double sa = K.s[pa], sb = K.s[pb];
  const double* ba = bl ? bl + (long long)pa * g.N : io.in[pa];
  const double* bb = bl ? bl + (long long)pb * g.N : io.in[pb];
  const double* xa = xl + (long long)pa * g.N;
  const double* xb = xl + (long long)pb * g.N;
  double acca = 0.0, accb = 0.0;
  for (int dz = 0; dz < (DIM >= 3 ? 2 : 1); ++dz)
    for (int dy = 0; dy < (DIM >= 2 ? 2 : 1); ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const int fx = 2 * X + dx, fy = DIM >= 2 ? 2 * Y + dy : 0, fz = DIM >= 3 ? 2 * Z + dz : 0;
        if (fx >= g.nx || fy >= g.ny || fz >= g.nz) continue;
        PtV<DIM, 1> q;
        load_ptv_xyz<DIM, 1>(g, fx, fy, fz, q);
        const long long p = q.p;
        const double c = cnt[p];
        acca += ba[p] - mg_apply<DIM>(g, q, xa, (1.0 + sa) * c, hlo + (long long)pa * g.S, hhi + (long long)pa * g.S);
        accb += bb[p] - mg_apply<DIM>(g, q, xb, (1.0 + sb) * c, hlo + (long long)pb * g.S, hhi + (long long)pb * g.S);
      }
  bc[(long long)pa * cstride + coff + pc] = acca;
  bc[(long long)pb * cstride + coff + pc] = accb;
}

// per-(plane, CTA) partials of a pair kernel; the last CTA sums every plane in a fixed order
__device__ __forceinline__ void sp_reduce_pair(const SpStepCtx& S, double va, double vb, int pa, int pb) {
  __shared__ double red[2][SP_T / 32];
  __shared__ bool last;
  __shared__ double tot[AAC_MAX_ELL];
  va = warp_sum(va);
  vb = warp_sum(vb);
  const int t = threadIdx.x;
  if ((t & 31) == 0) {
    red[0][t >> 5] = va;
    red[1][t >> 5] = vb;
  }
  __syncthreads();
  const int ntile = gridDim.x;
  if (t == 0) {
    double sa = 0.0, sb = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {     // (<= SP_T threads)
      sa += red[0][w];
      sb += red[1][w];
    }
    S.part[(long long)pa * ntile + blockIdx.x] = sa;
    S.part[(long long)pb * ntile + blockIdx.x] = sb;
    __threadfence();
    const unsigned tk = atomicAdd(S.tick, 1u);
    last = (tk == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int ell = S.K.ell;
  for (int q = 0; q < ell; ++q) {
    const double sum = block_sum_fixed(S.part + (long long)q * ntile, ntile);
    if (t == 0) tot[q] = sum;
  }
  if (t == 0) {
    *S.tick = 0;
    if (S.red) {
      for (int q = 0; q < ell; ++q) S.red[q] = tot[q];
    } else {
      sp_scalar_B(S, tot);
    }
  }
}

template <int DIM>
__global__ void __launch_bounds__(SP_T) k_mg_prolong_post_pair(Geo g, const double* __restrict__ cnt,
                                                               const double* __restrict__ dinv, Geo gc,
                                                               MgIo io, const double* bl, const double* xl,
                                                               const double* __restrict__ xc, double* x2l,
                                                               SpStepCtx S, int level0) {
  if (S.st && S.st->done) return;
  int pa, pb;
  sp_pair(S.K.ell, blockIdx.y, pa, pb);
  double dota = 0.0, dotb = 0.0;
  const double* xa = xl + (long long)pa * g.N;
  const double* xb = xl + (long long)pb * g.N;
  const double* ca = xc + (long long)pa * gc.N;
  const double* cb = xc + (long long)pb * gc.N;
  const double* ba = bl ? bl + (long long)pa * g.N : io.in[pa];
  const double* bb = bl ? bl + (long long)pb * g.N : io.in[pb];
  const double* da = dinv + (long long)sp_block_of(S.K.ell, pa) * g.N;
  const double* db = dinv + (long long)sp_block_of(S.K.ell, pb) * g.N;
  const double sa = S.K.s[pa], sb = S.K.s[pb];
  for (long long p = (long long)blockIdx.x * SP_T + threadIdx.x; p < g.N; p += (long long)gridDim.x * SP_T) {
    PtV<DIM, 1> q;
    load_ptv<DIM, 1>(g, p, q);
    // neighbour offsets and aggregates (a boundary neighbour aliases the point); a neighbour's
    // aggregate differs from the point's only across an aggregate edge (coordinate parity)
    const long long ac = ((long long)(q.z / 2) * gc.ny + q.y / 2) * gc.nx + q.x / 2;
    const long long ow = q.x > 0 ? -1 : 0, oe = q.x < g.nx - 1 ? 1 : 0;
    const long long aw = ac - (ow != 0 && !(q.x & 1)), ae = ac + (oe != 0 && (q.x & 1));
    long long on = 0, os = 0, od = 0, ou = 0, an = ac, as = ac, ad = ac, au = ac;
    if constexpr (DIM >= 2) {
      on = q.y > 0 ? -(long long)g.nx : 0;
      os = q.y < g.ny - 1 ? (long long)g.nx : 0;
      an = ac - (on != 0 && !(q.y & 1)) * (long long)gc.nx;
      as = ac + (os != 0 && (q.y & 1)) * (long long)gc.nx;
    }
    if constexpr (DIM >= 3) {
      const long long cS = (long long)gc.nx * gc.ny;
      od = q.z > 0 ? -g.S : 0;
      ou = q.z < g.nz - 1 ? g.S : 0;
      ad = ac - (od != 0 && !(q.z & 1)) * cS;
      au = ac + (ou != 0 && (q.z & 1)) * cS;
    }
    const double c = cnt ? cnt[p] : 1.0;
    // both planes computed before either is stored (the stores may alias the inputs as far as
    // the compiler knows: storing between them would serialise the two planes' loads)
    auto one = [&](const double* x, const double* xcp, const double* b, const double* di, double s,
                   double& bp) -> double {
      const double u0 = x[p] + xcp[ac];
      const double m = (1.0 + s) * c;
      double a = m * u0;
      a = fma(q.wx[0], u0 - (x[p + ow] + xcp[aw]), a);
      a = fma(q.wx[1], u0 - (x[p + oe] + xcp[ae]), a);
      if constexpr (DIM >= 2) {
        a = fma(q.wym[0], u0 - (x[p + on] + xcp[an]), a);
        a = fma(q.wyp[0], u0 - (x[p + os] + xcp[as]), a);
      }
      if constexpr (DIM >= 3) {
        a = fma(q.wzm[0], u0 - (x[p + od] + xcp[ad]), a);
        a = fma(q.wzp[0], u0 - (x[p + ou] + xcp[au]), a);
      }
      bp = b[p];
      return u0 + SP_OMEGA * (bp - a) * di[p];
    };
    double bpa, bpb;
    const double xna = one(xa, ca, ba, da, sa, bpa);
    const double xnb = one(xb, cb, bb, db, sb, bpb);
    if (level0) {
      io.out[pa][p] = xna;
      io.out[pb][p] = xnb;
      dota = fma(xna, bpa, dota);
      dotb = fma(xnb, bpb, dotb);
    } else {
      x2l[(long long)pa * g.N + p] = xna;
      x2l[(long long)pb * g.N + p] = xnb;
    }
  }
  if (level0) sp_reduce_pair(S, dota, dotb, pa, pb);
}

// 2D variant of k_mg_prolong_post_pair on a row grid (grid-stride over rows, threads over x):
// the generic kernel spends ~70% of its ~310 instructions per point pair on flat-index and
// aggregate arithmetic; here every neighbour is a row pointer fixed once per row plus the column,
// and the aggregate of a neighbour follows from the coordinate parity. Same operations in the
// same order: bit-identical results.
__global__ void __launch_bounds__(SP_T) k_mg_prolong_post_pair2(Geo g, const double* __restrict__ cnt,
                                                                const double* __restrict__ dinv, Geo gc,
                                                                MgIo io, const double* bl, const double* xl,
                                                                const double* __restrict__ xc, double* x2l,
                                                                SpStepCtx S, int level0) {
  if (S.st && S.st->done) return;
  int pa, pb;
  sp_pair(S.K.ell, blockIdx.y, pa, pb);
  double dota = 0.0, dotb = 0.0;
  const int nx = g.nx, ny = g.ny, cnx = gc.nx;
  const double sa = S.K.s[pa], sb = S.K.s[pb];
  const double* xa = xl + (long long)pa * g.N;
  const double* xb = xl + (long long)pb * g.N;
  const double* ca = xc + (long long)pa * gc.N;
  const double* cb = xc + (long long)pb * gc.N;
  const double* ba = bl ? bl + (long long)pa * g.N : io.in[pa];
  const double* bb = bl ? bl + (long long)pb * g.N : io.in[pb];
  const double* da = dinv + (long long)sp_block_of(S.K.ell, pa) * g.N;
  const double* db = dinv + (long long)sp_block_of(S.K.ell, pb) * g.N;
  double* oa = level0 ? io.out[pa] : x2l + (long long)pa * g.N;
  double* ob = level0 ? io.out[pb] : x2l + (long long)pb * g.N;
  for (int y = blockIdx.x; y < ny; y += gridDim.x) {
    const long long r0 = (long long)y * nx;
    const int on = y > 0 ? -nx : 0, os = y < ny - 1 ? nx : 0;   // boundary neighbour = the point
    const long long cr = (long long)(y / 2) * cnx;
    const int can = (on != 0 && !(y & 1)) ? -cnx : 0, cas = (os != 0 && (y & 1)) ? cnx : 0;
    const double* wxr = g.wx + r0;
    const double* wyr = g.wy + r0;
    const double* cntr = cnt ? cnt + r0 : nullptr;
    for (int x = threadIdx.x; x < nx; x += SP_T) {
      const int ow = x > 0 ? -1 : 0, oe = x < nx - 1 ? 1 : 0;
      const int cx = x >> 1;
      const int caw = (ow != 0 && !(x & 1)) ? -1 : 0, cae = (oe != 0 && (x & 1)) ? 1 : 0;
      const double wx0 = __ldg(wxr + x), wx1 = __ldg(wxr + x + 1);
      const double wym = __ldg(wyr + x), wyp = __ldg(wyr + nx + x);
      const double c = cntr ? cntr[x] : 1.0;
      auto one = [&](const double* xp_, const double* cp_, const double* b_, const double* d_, double s,
                     double& bp) -> double {
        const double* xr = xp_ + r0 + x;
        const double* cc = cp_ + cr + cx;
        const double u0 = xr[0] + cc[0];
        const double m = (1.0 + s) * c;
        double a = m * u0;
        a = fma(wx0, u0 - (xr[ow] + cc[caw]), a);
        a = fma(wx1, u0 - (xr[oe] + cc[cae]), a);
        a = fma(wym, u0 - (xr[on] + cc[can]), a);
        a = fma(wyp, u0 - (xr[os] + cc[cas]), a);
        bp = b_[r0 + x];
        return u0 + SP_OMEGA * (bp - a) * d_[r0 + x];
      };
      double bpa, bpb;
      const double xna = one(xa, ca, ba, da, sa, bpa);
      const double xnb = one(xb, cb, bb, db, sb, bpb);
      oa[r0 + x] = xna;
      ob[r0 + x] = xnb;
      if (level0) {
        dota = fma(xna, bpa, dota);
        dotb = fma(xnb, bpb, dotb);
      }
    }
  }
  if (level0) sp_reduce_pair(S, dota, dotb, pa, pb);
}

// x_c = A_c(s)^{-1} b_c with the precomputed dense inverse of the plane's block (CTA per plane)
__global__ void __launch_bounds__(SP_T) k_mg_coarse(int nc, const double* __restrict__ minv, int ell,
                                                    const double* bc, double* xc, const IterState* st) {
  griddep();
  if (st && st->done) return;
  const int pl = blockIdx.x;
  const double* M = minv + (long long)sp_block_of(ell, pl) * nc * nc;
  const double* b = bc + (long long)pl * nc;
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nc; ++k) s = fma(M[(long long)i * nc + k], b[k], s);
    xc[(long long)pl * nc + i] = s;
  }
}

// x_l += P x_c (injection from the aggregate)
template <int DIM>
__global__ void __launch_bounds__(SP_T) k_mg_prolong(Geo g, Geo gc, double* xl, const double* xc,
                                                     const IterState* st, long long cstride, long long coff) {
  if (st && st->done) return;
  const int pl = blockIdx.y;
  const long long p = (long long)blockIdx.x * SP_T + threadIdx.x;
  if (p >= g.N) return;
  const int x = (int)(p % g.nx);
  const long long r = p / g.nx;
  const int y = (int)(r % g.ny), z = (int)(r / g.ny);
  const long long pc = ((long long)(z / 2) * gc.ny + y / 2) * gc.nx + x / 2;
  xl[(long long)pl * g.N + p] += xc[(long long)pl * cstride + coff + pc];
}

// x2 = x + omega (b - A x)/D. Level 0: written to io.out[pl], dot partial <x2, b> per plane,
// last CTA: scalar step B.
template <int DIM>
__global__ void __launch_bounds__(SP_T) k_mg_post(Geo g, const double* __restrict__ cnt,
                                                  const double* __restrict__ dinv, MgIo io,
                                                  const double* bl, const double* xl, double* x2l,
                                                  SpStepCtx S, int level0, const double* hlo,
                                                  const double* hhi) {
  if (S.st && S.st->done) return;
  const int pl = blockIdx.y;
  double dotp = 0.0;
  // grid-stride over tiles: on level 0 the grid is kept small, because every CTA of a
  // reducing kernel takes a ticket on ONE counter (tens of thousands of same-address atomics
  // serialised in L2 cost more than the kernel's memory traffic)
  for (long long p = (long long)blockIdx.x * SP_T + threadIdx.x; p < g.N; p += (long long)gridDim.x * SP_T) {
    PtV<DIM, 1> q;
    load_ptv<DIM, 1>(g, p, q);
    const double m = (1.0 + S.K.s[pl]) * cnt[p];
    const double* b = bl ? bl + (long long)pl * g.N : io.in[pl];
    const double* x = xl + (long long)pl * g.N;
    const double xn = x[p] + SP_OMEGA * (b[p] - mg_apply<DIM>(g, q, x, m, hlo + (long long)pl * g.S,
                                                              hhi + (long long)pl * g.S)) *
                                 dinv[(long long)sp_block_of(S.K.ell, pl) * g.N + p];
    if (level0) {
      io.out[pl][p] = xn;
      dotp = fma(xn, b[p], dotp);
    } else {
      x2l[(long long)pl * g.N + p] = xn;
    }
  }
  if (level0) sp_reduce(S, dotp, true);
}

// Prolongation fused into the post-smoothing (saves the prolonged iterate's write and re-read):
// xt = x + P x_c evaluated at the point and its stencil neighbours (halo layers: the neighbour
// rank's x AFTER its own prolongation, i.e. exchanged by the caller -- so on slab-decomposed
// levels the unfused pair k_mg_prolong + halo + k_mg_post is used instead).
template <int DIM>
__global__ void __launch_bounds__(SP_T) k_mg_prolong_post(Geo g, const double* __restrict__ cnt,
                                                          const double* __restrict__ dinv, Geo gc,
                                                          MgIo io, const double* bl, const double* xl,
                                                          const double* __restrict__ xc, double* x2l,
                                                          SpStepCtx S, int level0) {
  if (S.st && S.st->done) return;
  const int pl = blockIdx.y;
  double dotp = 0.0;
  const double* x = xl + (long long)pl * g.N;
  const double* xcp = xc + (long long)pl * gc.N;
  for (long long p = (long long)blockIdx.x * SP_T + threadIdx.x; p < g.N; p += (long long)gridDim.x * SP_T) {
    PtV<DIM, 1> q;
    load_ptv<DIM, 1>(g, p, q);
    const Nbr nb = nbr<DIM, 1>(g, q, x, nullptr, nullptr);
    // aggregates of the point and its neighbours from the coordinates (a boundary neighbour
    // aliases the point and so its aggregate)
    auto agg = [&](int xx, int yy, int zz) { return ((long long)(zz / 2) * gc.ny + yy / 2) * gc.nx + xx / 2; };
    const long long ac = agg(q.x, q.y, q.z);
    const double u0 = *nb.c + xcp[ac];
    const double m = (1.0 + S.K.s[pl]) * (cnt ? cnt[p] : 1.0);
    double a = m * u0;
    a = fma(q.wx[0], u0 - (*nb.w + xcp[q.x > 0 ? agg(q.x - 1, q.y, q.z) : ac]), a);
    a = fma(q.wx[1], u0 - (*nb.e + xcp[q.x < g.nx - 1 ? agg(q.x + 1, q.y, q.z) : ac]), a);
    if constexpr (DIM >= 2) {
      a = fma(q.wym[0], u0 - (*nb.n + xcp[q.y > 0 ? agg(q.x, q.y - 1, q.z) : ac]), a);
      a = fma(q.wyp[0], u0 - (*nb.s + xcp[q.y < g.ny - 1 ? agg(q.x, q.y + 1, q.z) : ac]), a);
    }
    if constexpr (DIM >= 3) {
      a = fma(q.wzm[0], u0 - (*nb.d + xcp[q.z > 0 ? agg(q.x, q.y, q.z - 1) : ac]), a);
      a = fma(q.wzp[0], u0 - (*nb.u + xcp[q.z < g.nz - 1 ? agg(q.x, q.y, q.z + 1) : ac]), a);
    }
    const double* b = bl ? bl + (long long)pl * g.N : io.in[pl];
    const double bp = b[p];
    const double xn = u0 + SP_OMEGA * (bp - a) * dinv[(long long)sp_block_of(S.K.ell, pl) * g.N + p];
    if (level0) {
      io.out[pl][p] = xn;
      dotp = fma(xn, bp, dotp);
    } else {
      x2l[(long long)pl * g.N + p] = xn;
    }
  }
  if (level0) sp_reduce(S, dotp, true);
}

// ---- coarse tail of the V-cycle in ONE launch ----------------------------------------------
// Levels T..L (all global, each <= SP_TAIL_MAX points) for one plane per CTA: the same
// smoothing / restriction / dense solve / prolongation / post-smoothing steps as the per-level
// kernels, separated by __syncthreads instead of kernel boundaries (the small levels are
// launch- and latency-bound: ~16 launches of a few hundred points each per cycle).
constexpr int SP_TAIL_MAX = 4096;
constexpr int SP_TAIL_T = 1024;
constexpr int SP_TAIL_LEV = 8;
struct MgTail {
  int nlev;                      // levels T .. T + nlev - 1 (the last one is the coarsest)
  Geo g[SP_TAIL_LEV];
  const double* cnt[SP_TAIL_LEV];
  const double* dinv[SP_TAIL_LEV];
  double* b[SP_TAIL_LEV];        // b[0] = the tail's input (written by the level above)
  double* x[SP_TAIL_LEV];
  double* x2[SP_TAIL_LEV];       // x2[0] = the tail's output
  const double* minv;
  int nc;
};

template <int DIM>
__device__ __forceinline__ void tail_xyz(const Geo& g, long long p, int& x, int& y, int& z) {
  x = (int)(p % g.nx);
  const long long r = p / g.nx;
  y = (int)(r % g.ny);
  z = (int)(r / g.ny);
}

template <int DIM>
__global__ void __launch_bounds__(SP_TAIL_T) k_mg_tail(MgTail T, SpConst K, const IterState* st) {
  griddep();
  if (st && st->done) return;
  const int pl = blockIdx.x;
  const double s = K.s[pl];
  const int t = threadIdx.x;
  for (int l = 0; l + 1 < T.nlev; ++l) {                   // down
    const Geo& g = T.g[l];
    const Geo& gc = T.g[l + 1];
    const double* b = T.b[l] + (long long)pl * g.N;
    double* x = T.x[l] + (long long)pl * g.N;
    const double* di = T.dinv[l] + (long long)sp_block_of(K.ell, pl) * g.N;
    for (long long p = t; p < g.N; p += blockDim.x) x[p] = SP_OMEGA * b[p] * di[p];
    __syncthreads();
    double* bc = T.b[l + 1] + (long long)pl * gc.N;
    for (long long pc = t; pc < gc.N; pc += blockDim.x) {
      int X, Y, Z;
      tail_xyz<DIM>(gc, pc, X, Y, Z);
      double acc = 0.0;
      for (int dz = 0; dz < (DIM >= 3 ? 2 : 1); ++dz)
        for (int dy = 0; dy < (DIM >= 2 ? 2 : 1); ++dy)
          for (int dx = 0; dx < 2; ++dx) {
            const int fx = 2 * X + dx, fy = DIM >= 2 ? 2 * Y + dy : 0, fz = DIM >= 3 ? 2 * Z + dz : 0;
            if (fx >= g.nx || fy >= g.ny || fz >= g.nz) continue;
            PtV<DIM, 1> q;
            load_ptv_xyz<DIM, 1>(g, fx, fy, fz, q);
            acc += b[q.p] - mg_apply<DIM>(g, q, x, (1.0 + s) * T.cnt[l][q.p]);
          }
      bc[pc] = acc;
    }
    __syncthreads();
  }
  {                                                        // coarsest: dense solve
    const int nc = T.nc, L = T.nlev - 1;
    const double* M = T.minv + (long long)sp_block_of(K.ell, pl) * nc * nc;
    const double* b = T.b[L] + (long long)pl * nc;
    double* xc = T.x2[L] + (long long)pl * nc;
    for (int i = t; i < nc; i += blockDim.x) {
      double acc = 0.0;
      for (int k = 0; k < nc; ++k) acc = fma(M[(long long)i * nc + k], b[k], acc);
      xc[i] = acc;
    }
    __syncthreads();
  }
  for (int l = T.nlev - 2; l >= 0; --l) {                  // up
    const Geo& g = T.g[l];
    const Geo& gc = T.g[l + 1];
    double* x = T.x[l] + (long long)pl * g.N;
    const double* xc = T.x2[l + 1] + (long long)pl * gc.N;
    for (long long p = t; p < g.N; p += blockDim.x) {
      int xx, yy, zz;
      tail_xyz<DIM>(g, p, xx, yy, zz);
      x[p] += xc[((long long)(zz / 2) * gc.ny + yy / 2) * gc.nx + xx / 2];
    }
    __syncthreads();
    const double* b = T.b[l] + (long long)pl * g.N;
    double* x2 = T.x2[l] + (long long)pl * g.N;
    for (long long p = t; p < g.N; p += blockDim.x) {
      PtV<DIM, 1> q;
      load_ptv<DIM, 1>(g, p, q);
      const double m = (1.0 + s) * T.cnt[l][p];
      x2[p] = x[p] + SP_OMEGA * (b[p] - mg_apply<DIM>(g, q, x, m)) *
                     T.dinv[l][(long long)sp_block_of(K.ell, pl) * g.N + p];
    }
    __syncthreads();
  }
}

// ---- Krylov kernels -------------------------------------------------------------------------
struct SpVec {
  double* X;
  double *Vp, *Vc, *Vn, *Zc, *Wp, *Wc, *Wn, *SZ;
  double *R, *P, *Zr;
  const double* what;
};

// complex planes: Vc = [Im w; Re w] (u-plane <- Im w, v-plane <- Re w), Vp = Wp = Wc = X = 0;
// real planes: R = w, X = 0.
__global__ void __launch_bounds__(SP_T) k_sp_init(long long N, int ell, SpVec v, const IterState* st) {
  griddep();
  if (st && st->done) return;
  const long long p = (long long)blockIdx.x * SP_T + threadIdx.x;
  if (p >= N) return;
  const int h = ell / 2;
  for (int pl = 0; pl < ell; ++pl) {
    const long long o = (long long)pl * N + p;
    v.X[o] = 0.0;
    const int kb = sp_block_of(ell, pl);
    if (kb == 0 || kb == h) {
      v.R[o] = v.what[o];
    } else {
      v.Vc[o] = (pl & 1) ? v.what[o + N] : v.what[o - N];   // 2k-1 is the u (Re) plane
      v.Vp[o] = 0.0;
      v.Wp[o] = 0.0;
      v.Wc[o] = 0.0;
    }
  }
}

// K1 (grid: tiles x blocks): complex: SZ = S (z / gamma), partial <S z, z> / gamma^2-scaled;
// real: Q = SZ = (A - Lambda) P, partial <P, Q>. Last CTA: scalar step A.
template <int DIM>
__global__ void __launch_bounds__(SP_T) k_sp_apply(Geo g, SpVec v, SpStepCtx S) {
  if (S.st && S.st->done) return;
  const int kb = blockIdx.y, ell = S.K.ell, h = ell / 2;
  const long long N = g.N;
  // block scalars read once (SZ stores may alias S.blk as far as the compiler knows, which
  // would re-load them after every store and serialise the loop)
  const bool stopped = S.blk[kb].stop != 0;
  const double invg = stopped ? 0.0 : 1.0 / S.blk[kb].gamma;
  double dotp = 0.0;
  for (long long p = (long long)blockIdx.x * SP_T + threadIdx.x; p < N && !stopped;
       p += (long long)gridDim.x * SP_T) {     // grid-stride: few reducing CTAs (see k_mg_post)
    PtV<DIM, 1> q;
    load_ptv<DIM, 1>(g, p, q);
    if (kb == 0 || kb == h) {
      const int pl = kb == 0 ? 0 : ell - 1;
      const double* pp = v.P + (long long)pl * N;
      const double a = mg_apply<DIM>(g, q, pp, 1.0 + S.K.s[pl], S.hlo + (long long)pl * g.S,
                                     S.hhi + (long long)pl * g.S);   // (A - Lambda) p
      v.SZ[(long long)pl * N + p] = a;
      dotp = fma(pp[p], a, dotp);
    } else {
      const int qu = 2 * kb - 1, qv = qu + 1;
      double azu[1], azv[1], zu[1], zv[1];
      apply_Av<DIM, 1>(g, q, v.Zc + (long long)qu * N, S.hlo + (long long)qu * g.S, S.hhi + (long long)qu * g.S,
                       azu, zu);
      apply_Av<DIM, 1>(g, q, v.Zc + (long long)qv * N, S.hlo + (long long)qv * g.S, S.hhi + (long long)qv * g.S,
                       azv, zv);
      const double us = zu[0] * invg, vs = zv[0] * invg;
      const double Au = azu[0] * invg, Av = azv[0] * invg;
      const double lr = S.K.lre[kb], li = S.K.lim[kb];
      const double Su = li * us + (Av - lr * vs);
      const double Sv = (Au - lr * us) - li * vs;
      v.SZ[(long long)qu * N + p] = Su;
      v.SZ[(long long)qv * N + p] = Sv;
      dotp = fma(Sv, vs, fma(Su, us, dotp));
    }
  }
  sp_reduce(S, dotp, false);
}

// 2D row-grid variant of k_sp_apply (grid-stride over rows, threads over x): row pointers for the
// y-neighbours (slab halo rows at the ends), no flat-index arithmetic. Same operations in the same
// order as apply_Av / mg_apply: bit-identical.
__global__ void __launch_bounds__(SP_T) k_sp_apply2(Geo g, SpVec v, SpStepCtx S) {
  if (S.st && S.st->done) return;
  const int kb = blockIdx.y, ell = S.K.ell, h = ell / 2;
  const long long N = g.N;
  const int nx = g.nx, ny = g.ny;
  const bool stopped = S.blk[kb].stop != 0;
  const double invg = stopped ? 0.0 : 1.0 / S.blk[kb].gamma;
  const bool real = kb == 0 || kb == h;
  const int q0 = real ? (kb == 0 ? 0 : ell - 1) : 2 * kb - 1;
  const double* u0p = real ? v.P + (long long)q0 * N : v.Zc + (long long)q0 * N;
  const double* u1p = real ? u0p : v.Zc + (long long)(q0 + 1) * N;
  const double* hl0 = S.hlo + (long long)q0 * g.S;
  const double* hh0 = S.hhi + (long long)q0 * g.S;
  const double* hl1 = S.hlo + (long long)(q0 + 1) * g.S;
  const double* hh1 = S.hhi + (long long)(q0 + 1) * g.S;
  const double m = 1.0 + S.K.s[q0];
  const double lr = S.K.lre[kb], li = S.K.lim[kb];
  double* sz0 = v.SZ + (long long)q0 * N;
  double* sz1 = v.SZ + (long long)(q0 + 1) * N;
  double dotp = 0.0;
  for (int y = blockIdx.x; y < ny && !stopped; y += gridDim.x) {
    const long long r0 = (long long)y * nx;
    // y-neighbour rows: in the slab, a halo row (slab boundary), or the row itself (boundary)
    const double* n0 = y > 0 ? u0p + r0 - nx : (g.has_lo ? hl0 : u0p + r0);
    const double* s0 = y < ny - 1 ? u0p + r0 + nx : (g.has_hi ? hh0 : u0p + r0);
    const double* n1 = y > 0 ? u1p + r0 - nx : (g.has_lo ? hl1 : u1p + r0);
    const double* s1 = y < ny - 1 ? u1p + r0 + nx : (g.has_hi ? hh1 : u1p + r0);
    const double* wxr = g.wx + r0;
    const double* wyr = g.wy + r0;
    for (int x = threadIdx.x; x < nx; x += SP_T) {
      const int ow = x > 0 ? -1 : 0, oe = x < nx - 1 ? 1 : 0;
      const double wx0 = __ldg(wxr + x), wx1 = __ldg(wxr + x + 1);
      const double wym = __ldg(wyr + x), wyp = __ldg(wyr + nx + x);
      const double dbd = g.dir ? dirichlet_diag<2>(g, x, y, 0) : 0.0;
      auto av = [&](const double* u, const double* nr, const double* sr, double& c) {
        const double* ur = u + r0 + x;
        c = ur[0];
        double acc = c;
        acc = fma(wx0, c - ur[ow], acc);
        acc = fma(wx1, c - ur[oe], acc);
        acc = fma(wym, c - nr[x], acc);
        acc = fma(wyp, c - sr[x], acc);
        acc = fma(dbd, c, acc);
        return acc;
      };
      if (real) {
        double c;
        const double a0 = av(u0p, n0, s0, c);
        const double a = a0 + (m - 1.0) * c;                 // (A - Lambda) p
        sz0[r0 + x] = a;
        dotp = fma(c, a, dotp);
      } else {
        double zu, zv;
        const double azu = av(u0p, n0, s0, zu);
        const double azv = av(u1p, n1, s1, zv);
        const double us = zu * invg, vs = zv * invg;
        const double Au = azu * invg, Av = azv * invg;
        const double Su = li * us + (Av - lr * vs);
        const double Sv = (Au - lr * us) - li * vs;
        sz0[r0 + x] = Su;
        sz1[r0 + x] = Sv;
        dotp = fma(Sv, vs, fma(Su, us, dotp));
      }
    }
  }
  sp_reduce(S, dotp, false);
}

// K3 (grid: tiles x planes): complex: Vn = SZ - (delta/gamma) Vc - (gamma/gamma_prev) Vp;
// real: X += alpha P, R -= alpha Q.
__global__ void __launch_bounds__(SP_T) k_sp_upd1(long long N, int ell, SpVec v, const SpBlk* blk,
                                                  const IterState* st) {
  if (st && st->done) return;
  const int pl = blockIdx.y, h = ell / 2, kb = sp_block_of(ell, pl);
  const SpBlk& b = blk[kb];
  if (b.stop == 1) return;
  // block scalars once per thread; grid-stride over the plane (the vectors are not aliased with
  // blk, but the compiler cannot know: loading the scalars inside the loop would re-load them)
  const double alpha = b.alpha, dcoef = b.dcoef, vcoef = b.vcoef;
  const bool real = kb == 0 || kb == h;
  const long long o0 = (long long)pl * N;
  for (long long p = (long long)blockIdx.x * SP_T + threadIdx.x; p < N; p += (long long)gridDim.x * SP_T) {
    const long long o = o0 + p;
    if (real) {
      v.X[o] = fma(alpha, v.P[o], v.X[o]);
      v.R[o] = fma(-alpha, v.SZ[o], v.R[o]);
    } else {
      v.Vn[o] = v.SZ[o] - dcoef * v.Vc[o] - vcoef * v.Vp[o];
    }
  }
}

// K6 (grid: tiles x planes): complex: Wn = (z/gamma_old - a3 Wp - a2 Wc) / a1, X += xcoef Wn;
// real: P = Zr + beta P.
__global__ void __launch_bounds__(SP_T) k_sp_upd2(long long N, int ell, SpVec v, const SpBlk* blk,
                                                  const IterState* st) {
  griddep();
  if (st && st->done) return;
  const int pl = blockIdx.y, h = ell / 2, kb = sp_block_of(ell, pl);
  const SpBlk& b = blk[kb];
  if (b.stop == 1) return;
  const double beta = b.beta, gp = b.gamma_prev, a1 = b.a1, a2 = b.a2, a3 = b.a3, xcoef = b.xcoef;
  const bool real = kb == 0 || kb == h;
  const long long o0 = (long long)pl * N;
  for (long long p = (long long)blockIdx.x * SP_T + threadIdx.x; p < N; p += (long long)gridDim.x * SP_T) {
    const long long o = o0 + p;
    if (real) {
      v.P[o] = fma(beta, v.P[o], v.Zr[o]);
    } else {
      const double zs = v.Zc[o] / gp;
      const double wn = (zs - a3 * v.Wp[o] - a2 * v.Wc[o]) / a1;
      v.Wn[o] = wn;
      v.X[o] = fma(xcoef, wn, v.X[o]);
    }
  }
}

// Real planes of K3 alone (the complex planes' update is formed inside the fused level-0
// restriction, sp_fused.cuh): X += alpha P, R -= alpha Q for planes 0 and ell - 1.
__global__ void __launch_bounds__(SP_T) k_sp_upd1_real(long long N, int ell, SpVec v, const SpBlk* blk,
                                                       const IterState* st) {
  griddep();
  if (st && st->done) return;
  const int pl = blockIdx.y == 0 ? 0 : ell - 1, kb = sp_block_of(ell, pl);
  const SpBlk& b = blk[kb];
  if (b.stop == 1) return;
  const double alpha = b.alpha;
  const long long o0 = (long long)pl * N;
  for (long long p = (long long)blockIdx.x * SP_T + threadIdx.x; p < N; p += (long long)gridDim.x * SP_T) {
    const long long o = o0 + p;
    v.X[o] = fma(alpha, v.P[o], v.X[o]);
    v.R[o] = fma(-alpha, v.SZ[o], v.R[o]);
  }
}

#include "sp_fused.cuh"

// ------------------------------------------------------------------------------------------
// host side
static int sp_alloc(aac_ctx* ctx, SpPlan* P, double** p, long long n) {
  if (cudaMalloc((void**)p, (size_t)std::max<long long>(n, 1) * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    return aac_fail(ctx, AAC_ENOMEM, "SP workspace allocation failed");
  }
  P->owned.push_back(*p);
  return AAC_OK;
}

static void sp_destroy(aac_ctx* ctx) {
  if (!ctx->sp) return;
  for (void* p : ctx->sp->owned) cudaFree(p);
  delete ctx->sp;
  ctx->sp = nullptr;
}

struct HostLevel {
  int nx, ny, nz;
  std::vector<double> wx, wy, wz, cnt;      // lower-face layout, padded like aac_setup
};

static inline long long pad4l(long long v) { return (v + 3) / 4 * 4; }

static HostLevel coarsen(const HostLevel& f, int dim) {
  HostLevel c;
  c.nx = f.nx > 1 ? (f.nx + 1) / 2 : 1;
  c.ny = f.ny > 1 ? (f.ny + 1) / 2 : 1;
  c.nz = f.nz > 1 ? (f.nz + 1) / 2 : 1;
  const long long Nc = (long long)c.nx * c.ny * c.nz, Nf = (long long)f.nx * f.ny * f.nz;
  const long long Sc = dim == 3 ? (long long)c.nx * c.ny : c.nx;
  c.wx.assign(pad4l(Nc + 1), 0.0);
  c.wy.assign(pad4l(Nc + c.nx), 0.0);
  c.wz.assign(pad4l(Nc + Sc), 0.0);
  c.cnt.assign(Nc, 0.0);
  auto fi = [&](long long x, long long y, long long z) { return (z * f.ny + y) * f.nx + x; };
  auto ci = [&](long long x, long long y, long long z) { return (z * c.ny + y) * c.nx + x; };
  (void)Nf;
  for (long long z = 0; z < f.nz; ++z)
    for (long long y = 0; y < f.ny; ++y)
      for (long long x = 0; x < f.nx; ++x) {
        const long long pf = fi(x, y, z);
        const long long X = x / 2, Y = f.ny > 1 ? y / 2 : 0, Z = f.nz > 1 ? z / 2 : 0;
        const long long pc = ci(X, Y, Z);
        c.cnt[pc] += f.cnt[pf];
        // a fine lower face between two different aggregates adds to the coarse lower face
        // (index 0 included: zero on a physical boundary, the face to the neighbour rank's
        // slab on a slab boundary -- slab boundaries are aggregate boundaries)
        if ((x & 1) == 0) c.wx[pc] += f.wx[pf];
        if (dim >= 2 && (y & 1) == 0) c.wy[pc] += f.wy[pf];
        if (dim >= 3 && (z & 1) == 0) c.wz[pc] += f.wz[pf];
      }
  // the upper face of the slab (extra layer of the slab axis) when it bounds an aggregate
  if (dim == 2 && (f.ny & 1) == 0)
    for (long long x = 0; x < f.nx; ++x) c.wy[(long long)c.ny * c.nx + x / 2] += f.wy[(long long)f.ny * f.nx + x];
  if (dim == 3 && (f.nz & 1) == 0)
    for (long long y = 0; y < f.ny; ++y)
      for (long long x = 0; x < f.nx; ++x)
        c.wz[(long long)c.nz * c.nx * c.ny + (y / 2) * c.nx + x / 2] += f.wz[(long long)f.nz * f.nx * f.ny + y * f.nx + x];
  return c;
}

// dense A_c(s) = diag((1+s) cnt + sum w) - W, inverted by Cholesky (SPD)
static bool dense_inverse(const HostLevel& c, int dim, double s, std::vector<double>& inv) {
  const int n = c.nx * c.ny * c.nz;
  std::vector<double> A((size_t)n * n, 0.0);
  const long long S = dim == 3 ? (long long)c.nx * c.ny : c.nx;
  for (int z = 0; z < c.nz; ++z)
    for (int y = 0; y < c.ny; ++y)
      for (int x = 0; x < c.nx; ++x) {
        const int p = (z * c.ny + y) * c.nx + x;
        A[(size_t)p * n + p] += (1.0 + s) * c.cnt[p];
        auto edge = [&](int q, double w) {
          A[(size_t)p * n + p] += w;
          A[(size_t)q * n + q] += w;
          A[(size_t)p * n + q] -= w;
          A[(size_t)q * n + p] -= w;
        };
        if (x > 0) edge(p - 1, c.wx[p]);
        if (dim >= 2 && y > 0) edge(p - c.nx, c.wy[p]);
        if (dim >= 3 && z > 0) edge((int)(p - S), c.wz[p]);
      }
  // Cholesky A = L L^T (lower, in place)
  for (int j = 0; j < n; ++j) {
    double d = A[(size_t)j * n + j];
    for (int k = 0; k < j; ++k) d -= A[(size_t)j * n + k] * A[(size_t)j * n + k];
    if (!(d > 0.0)) {
      if (getenv("AAC_SP_DEBUG"))
        fprintf(stderr, "[sp] dense Cholesky failed at %d of %d (%dx%dx%d), d=%g s=%g\n", j, n, c.nx, c.ny, c.nz, d, s);
      return false;
    }
    d = sqrt(d);
    A[(size_t)j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double v = A[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) v -= A[(size_t)i * n + k] * A[(size_t)j * n + k];
      A[(size_t)i * n + j] = v / d;
    }
  }
  inv.assign((size_t)n * n, 0.0);
  std::vector<double> col(n);
  for (int e = 0; e < n; ++e) {          // solve L L^T x = e_e
    for (int i = 0; i < n; ++i) {
      double v = (i == e) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) v -= A[(size_t)i * n + k] * col[k];
      col[i] = v / A[(size_t)i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double v = col[i];
      for (int k = i + 1; k < n; ++k) v -= A[(size_t)k * n + i] * col[k];
      col[i] = v / A[(size_t)i * n + i];
    }
    for (int i = 0; i < n; ++i) inv[(size_t)i * n + e] = col[i];
  }
  return true;
}

static void shift_of_block(const aac_ctx* ctx, int kb, double* lr, double* li);

static int sp_prepare_impl(aac_ctx* ctx, int k);

// Build the SP plan once per context. The plan is attached to ctx->sp while it is built (the
// helpers read it from there); any failure frees the partial plan and leaves ctx->sp NULL, so a
// later call retries from scratch instead of running on a half-built hierarchy.
static int sp_prepare(aac_ctx* ctx, int k) {
  if (ctx->sp) return AAC_OK;
  const int rc = sp_prepare_impl(ctx, k);
  if (rc != AAC_OK) {
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    cudaGetLastError();
    sp_destroy(ctx);
  }
  return rc;
}

static int sp_prepare_impl(aac_ctx* ctx, int k) {
  (void)k;
  if (ctx->geo.dir)   // the aggregation hierarchy carries no Dirichlet boundary terms
    return aac_fail(ctx, AAC_EINVAL, "AAC_SP needs the Neumann operator (no aac_set_boundary)");
  SpPlan* P = new SpPlan();
  ctx->sp = P;
  const int ell = ctx->ell, h = ell / 2, dim = ctx->dim;
  P->ell = ell;
  P->h = h;
  const Geo& g0 = ctx->geo;
  const long long N = g0.N, L = (long long)ell * N;
  // block shifts
  P->K.ell = ell;
  for (int kb = 0; kb <= h; ++kb) {
    double lr, li;
    shift_of_block(ctx, kb, &lr, &li);
    if (kb == 0 || kb == h) {
      P->K.lre[kb] = lr;
      P->K.lim[kb] = 0.0;
    } else {                                    // lambda = conj(Lambda_k): Im lambda > 0
      P->K.lre[kb] = lr;
      P->K.lim[kb] = -li;
    }
  }
  for (int pl = 0; pl < ell; ++pl) {
    const int kb = pl == 0 ? 0 : (pl == ell - 1 ? h : (pl + 1) / 2);
    P->K.s[pl] = (kb == 0 || kb == h) ? -P->K.lre[kb] : P->K.lim[kb] - P->K.lre[kb];
  }
  // level 0 from the device face weights
  HostLevel f;
  f.nx = g0.nx;
  f.ny = g0.ny;
  f.nz = g0.nz;
  const long long lenx = pad4l(N + 1), leny = pad4l(N + g0.nx), lenz = pad4l(N + g0.S);
  f.wx.resize(lenx);
  f.wy.resize(leny);
  f.wz.resize(lenz);
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  CUDA_TRY(ctx, cudaMemcpy(f.wx.data(), g0.wx, lenx * sizeof(double), cudaMemcpyDeviceToHost));
  CUDA_TRY(ctx, cudaMemcpy(f.wy.data(), g0.wy, leny * sizeof(double), cudaMemcpyDeviceToHost));
  CUDA_TRY(ctx, cudaMemcpy(f.wz.data(), g0.wz, lenz * sizeof(double), cudaMemcpyDeviceToHost));
  f.cnt.assign(N, 1.0);
  std::vector<HostLevel> hl{f};
  int G = -1;                                   // multi-rank: first global (gathered) level
  long long gLo = 0;                            // this rank's slab start on the gathered level
  if (ctx->nranks == 1) {
    while (std::max(hl.back().nx, std::max(hl.back().ny, hl.back().nz)) > SP_COARSE_MAX_AXIS)
      hl.push_back(coarsen(hl.back(), dim));
  } else {
    // Coarsen inside the slabs while every slab boundary is an aggregate boundary of the
    // GLOBAL hierarchy (even offsets; an odd count only at the top of the domain), so the
    // levels are exactly those of the one-rank hierarchy; then gather the last local level
    // on every rank and continue (and solve) redundantly.
    const int P_ = ctx->nranks;
    const long long n0 = dim == 2 ? ctx->n[1] : ctx->n[2];
    std::vector<int64_t> lo(P_), hi(P_);
    for (int r = 0; r < P_; ++r) aac_slab_range(n0, P_, r, &lo[r], &hi[r]);
    long long nslab = n0;
    auto gmax = [&](const HostLevel& H) {
      return std::max<long long>(H.nx, dim == 2 ? nslab : std::max<long long>(H.ny, nslab));
    };
    while (gmax(hl.back()) > SP_COARSE_MAX_AXIS) {
      bool ok = true;
      for (int r = 0; r < P_; ++r)
        ok = ok && lo[r] % 2 == 0 && (hi[r] % 2 == 0 || hi[r] == nslab) && hi[r] - lo[r] >= 2;
      if (!ok) break;
      hl.push_back(coarsen(hl.back(), dim));
      for (int r = 0; r < P_; ++r) {
        lo[r] /= 2;
        hi[r] = (hi[r] + 1) / 2;
      }
      nslab = (nslab + 1) / 2;
    }
    if (hl.size() < 2)
      return aac_fail(ctx, AAC_EINVAL,
                      "AAC_SP on %d ranks needs even slab boundaries (slab rows per rank even)", P_);
    G = (int)hl.size() - 1;
    gLo = lo[ctx->rank];
    // global level G: every rank contributes the lower faces / counts of its own layers
    const HostLevel& Lg = hl.back();
    HostLevel Gg;
    Gg.nx = Lg.nx;
    Gg.ny = dim == 2 ? (int)nslab : Lg.ny;
    Gg.nz = dim == 3 ? (int)nslab : 1;
    const long long Ng = (long long)Gg.nx * Gg.ny * Gg.nz, Sg = dim == 3 ? (long long)Gg.nx * Gg.ny : Gg.nx;
    const long long Nl = (long long)Lg.nx * Lg.ny * Lg.nz, off = gLo * Sg;
    Gg.wx.assign(pad4l(Ng + 1), 0.0);
    Gg.wy.assign(pad4l(Ng + Gg.nx), 0.0);
    Gg.wz.assign(pad4l(Ng + Sg), 0.0);
    Gg.cnt.assign(Ng, 0.0);
    const long long tot = (long long)Gg.wx.size() + Gg.wy.size() + Gg.wz.size() + Ng;
    std::vector<double> buf(tot, 0.0);
    double* bx = buf.data();
    double* by = bx + Gg.wx.size();
    double* bz = by + Gg.wy.size();
    double* bc = bz + Gg.wz.size();
    for (long long i = 0; i < Nl; ++i) {
      bx[off + i] = Lg.wx[i];
      if (dim >= 2) by[off + i] = Lg.wy[i];
      if (dim >= 3) bz[off + i] = Lg.wz[i];
      bc[off + i] = Lg.cnt[i];
    }
    double* dbuf = nullptr;
    AAC_TRY(sp_alloc(ctx, P, &dbuf, tot));
    // (stream-ordered copies: a pageable cudaMemcpy may return before its DMA completes, and
    // the library stream does not synchronise with the legacy stream)
    CUDA_TRY(ctx, cudaMemcpyAsync(dbuf, buf.data(), tot * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    AAC_TRY(comm_allreduce(ctx, dbuf, (int)tot, ncclSum));
    CUDA_TRY(ctx, cudaMemcpyAsync(buf.data(), dbuf, tot * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::copy(bx, bx + Gg.wx.size(), Gg.wx.begin());
    std::copy(by, by + Gg.wy.size(), Gg.wy.begin());
    std::copy(bz, bz + Gg.wz.size(), Gg.wz.begin());
    std::copy(bc, bc + Ng, Gg.cnt.begin());
    hl.push_back(Gg);                            // hl[G] = local slab, hl[G + 1] = global level G
    while (std::max(hl.back().nx, std::max(hl.back().ny, hl.back().nz)) > SP_COARSE_MAX_AXIS)
      hl.push_back(coarsen(hl.back(), dim));
  }
  P->gather = G;
  // device levels (multi-rank: hl[G] is only the slab geometry of the gathered level hl[G+1])
  Geo gslab{};
  for (size_t l = 0; l < hl.size(); ++l) {
    const HostLevel& H = hl[l];
    if (G >= 0 && (int)l == G) {
      gslab.nx = H.nx;
      gslab.ny = H.ny;
      gslab.nz = H.nz;
      gslab.N = (long long)H.nx * H.ny * H.nz;
      gslab.S = dim == 3 ? (long long)H.nx * H.ny : H.nx;
      continue;
    }
    SpLevel lv{};
    Geo& g = lv.g;
    g.nx = H.nx;
    g.ny = H.ny;
    g.nz = H.nz;
    g.N = (long long)H.nx * H.ny * H.nz;
    g.S = dim == 3 ? (long long)H.nx * H.ny : H.nx;
    lv.local = (G < 0 || (int)l < G) ? 1 : 0;
    g.has_lo = (G >= 0 && lv.local) ? ctx->geo.has_lo : 0;
    g.has_hi = (G >= 0 && lv.local) ? ctx->geo.has_hi : 0;
    if (G >= 0 && (int)l == G + 1) {
      lv.gl = gslab;
      lv.goff = gLo * g.S;
    }
    double* w = nullptr;
    const size_t nw = H.wx.size() + H.wy.size() + H.wz.size();
    AAC_TRY(sp_alloc(ctx, P, &w, nw));
    CUDA_TRY(ctx, cudaMemcpy(w, H.wx.data(), H.wx.size() * sizeof(double), cudaMemcpyHostToDevice));
    CUDA_TRY(ctx, cudaMemcpy(w + H.wx.size(), H.wy.data(), H.wy.size() * sizeof(double), cudaMemcpyHostToDevice));
    CUDA_TRY(ctx, cudaMemcpy(w + H.wx.size() + H.wy.size(), H.wz.data(), H.wz.size() * sizeof(double),
                             cudaMemcpyHostToDevice));
    g.wx = w;
    g.wy = w + H.wx.size();
    g.wz = w + H.wx.size() + H.wy.size();
    AAC_TRY(sp_alloc(ctx, P, &lv.cnt, g.N));
    {                                            // 1 / diag, in diag_of's summation order
      std::vector<double> di((size_t)(h + 1) * g.N);
      for (int kb = 0; kb <= h; ++kb) {
        const double sk = P->K.s[kb == 0 ? 0 : (kb == h ? ell - 1 : 2 * kb - 1)];
        for (long long pt = 0; pt < g.N; ++pt) {
          double d = (1.0 + sk) * H.cnt[pt] + H.wx[pt] + H.wx[pt + 1];
          if (dim >= 2) d += H.wy[pt] + H.wy[pt + g.nx];
          if (dim >= 3) d += H.wz[pt] + H.wz[pt + g.S];
          di[(size_t)kb * g.N + pt] = 1.0 / d;
        }
      }
      AAC_TRY(sp_alloc(ctx, P, &lv.dinv, (long long)di.size()));
      CUDA_TRY(ctx, cudaMemcpy(lv.dinv, di.data(), di.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    CUDA_TRY(ctx, cudaMemcpy(lv.cnt, H.cnt.data(), g.N * sizeof(double), cudaMemcpyHostToDevice));
    if (l > 0) AAC_TRY(sp_alloc(ctx, P, &lv.b, (long long)ell * g.N));
    AAC_TRY(sp_alloc(ctx, P, &lv.x, (long long)ell * g.N));
    if (l > 0) AAC_TRY(sp_alloc(ctx, P, &lv.x2, (long long)ell * g.N));
    P->lev.push_back(lv);
  }
  if (G >= 0) P->gather = G;                    // index into P->lev of the global level
  AAC_TRY(sp_alloc(ctx, P, &P->red, AAC_MAX_ELL));
  // coarsest dense inverses, one per block shift
  const HostLevel& Hc = hl.back();
  P->nc = Hc.nx * Hc.ny * Hc.nz;
  std::vector<double> allinv((size_t)(h + 1) * P->nc * P->nc);
  for (int kb = 0; kb <= h; ++kb) {
    const int pl = kb == 0 ? 0 : (kb == h ? ell - 1 : 2 * kb - 1);
    std::vector<double> inv;
    if (!dense_inverse(Hc, dim, P->K.s[pl], inv))
      return aac_fail(ctx, AAC_EINVAL, "coarsest multigrid operator not SPD");
    std::copy(inv.begin(), inv.end(), allinv.begin() + (size_t)kb * P->nc * P->nc);
  }
  AAC_TRY(sp_alloc(ctx, P, &P->minv, (long long)allinv.size()));
  CUDA_TRY(ctx, cudaMemcpy(P->minv, allinv.data(), allinv.size() * sizeof(double), cudaMemcpyHostToDevice));
  // Krylov workspaces
  double** bufs[] = {&P->X, &P->Vb[0], &P->Vb[1], &P->Vb[2], &P->Zb[0], &P->Zb[1], &P->Wb[0],
                     &P->Wb[1], &P->Wb[2], &P->SZ, &P->R, &P->P, &P->Zr};
  for (double** b : bufs) AAC_TRY(sp_alloc(ctx, P, b, L));
  double* blk = nullptr;
  AAC_TRY(sp_alloc(ctx, P, &blk, (long long)(h + 1) * (sizeof(SpBlk) / sizeof(double) + 1)));
  P->blk = reinterpret_cast<SpBlk*>(blk);
  CUDA_TRY(ctx, cudaMemset(P->blk, 0, (h + 1) * sizeof(SpBlk)));
  long long ntile = (N + SP_T - 1) / SP_T;
  if (P->lev.size() > 1) {                      // the fused level-0 kernels' tiles (sp_fused.cuh)
    int nsx, nt;
    spf_tiles(P->lev[1].g.nx, P->lev[1].g.ny, nsx, nt);
    ntile = std::max<long long>(ntile, nt);
  }
  AAC_TRY(sp_alloc(ctx, P, &P->part, ntile * ell + 8));
  {                                             // fused kernels: group partials and tickets
    const long long ng = (ntile + SPF_GROUP - 1) / SPF_GROUP;
    AAC_TRY(sp_alloc(ctx, P, &P->red2.gpart, ng * ell + 8));
    double* gt = nullptr;
    const long long nticks = (ng + 1) * SPF_TICK_STRIDE;
    AAC_TRY(sp_alloc(ctx, P, &gt, (nticks + 1) / 2));
    CUDA_TRY(ctx, cudaMemset(gt, 0, (size_t)nticks * sizeof(unsigned)));
    P->red2.gtick = reinterpret_cast<unsigned*>(gt);
  }
  double* tk = nullptr;
  AAC_TRY(sp_alloc(ctx, P, &tk, 1));
  P->tick = reinterpret_cast<unsigned*>(tk);
  CUDA_TRY(ctx, cudaMemset(P->tick, 0, sizeof(double)));
  CUDA_TRY(ctx, cudaDeviceSynchronize());     // legacy-stream uploads complete before stream work
  return AAC_OK;
}

// Halo exchange of the ell planes of a slab-decomposed level (no-op on one rank).
static int sp_halo(aac_ctx* ctx, const Geo& g, const double* x) {
  if (ctx->nranks == 1) return AAC_OK;
  const double* planes[AAC_MAX_ELL];
  int qs[AAC_MAX_ELL];
  for (int pl = 0; pl < ctx->ell; ++pl) {
    planes[pl] = x + (long long)pl * g.N;
    qs[pl] = pl;
  }
  return comm_halo_ex(ctx, g, planes, qs, ctx->ell, ctx->d_halo, ctx->d_halo + (long long)ctx->ell * ctx->geo.S);
}

// One V(1,1) cycle on all ell planes. Multi-rank: the slab-decomposed levels exchange halos
// after the pre-smoothing (restriction stencil) and after the prolongation (post-smoothing
// stencil); the restriction into the gathered level writes this rank's rows of the zeroed
// global right-hand side, which an all-reduce completes on every rank; the global levels run
// redundantly and the prolongation back reads this rank's rows of their result.
// CTAs per SM of the fused kernels that reduce (AAC_SPF_CPS overrides; measured: 4).
static int spf_cps() {
  static const int v = getenv("AAC_SPF_CPS") ? atoi(getenv("AAC_SPF_CPS")) : 4;
  return std::max(1, v);
}

// The fused 2D level kernels (sp_fused.cuh) run on one rank; AAC_SP_FUSED=0 selects the
// per-step kernels (smoothing, restriction, prolongation + post-smoothing).
static bool sp_fused_on(const aac_ctx* ctx, int dim) {
  static const bool off = getenv("AAC_SP_FUSED") && atoi(getenv("AAC_SP_FUSED")) == 0;
  return dim == 2 && ctx->nranks == 1 && !off;
}

template <int DIM>
static int sp_vcycle(aac_ctx* ctx, const MgIo& io, SpStepCtx S, const SpfUpd& U = SpfUpd{}) {
  SpPlan* P = ctx->sp;
  const int ell = P->ell;
  const int nl = (int)P->lev.size();
  const bool fused = sp_fused_on(ctx, DIM);
  const IterState* st = S.st;
  const double* hlo = ctx->d_halo;
  const double* hhi = ctx->d_halo + (long long)ell * ctx->geo.S;
  // first level of the fused coarse tail: global, <= SP_TAIL_MAX points, and not level 0
  // (level 0 takes the V-cycle's input and output pointers); AAC_SP_TAIL=0 disables it
  static const bool tail_on = !(getenv("AAC_SP_TAIL") && atoi(getenv("AAC_SP_TAIL")) == 0);
  int tl = nl;                                             // nl: no tail
  if (tail_on)
    for (int l = 1; l < nl; ++l)
      if (!(P->lev[l].local && ctx->nranks > 1) && P->lev[l].g.N <= SP_TAIL_MAX && nl - l <= SP_TAIL_LEV &&
          nl - l >= 2) {
        tl = l;
        break;
      }
  const int ldown = tl < nl ? tl : nl - 1;                 // per-level kernels above the tail
  for (int l = 0; l < ldown; ++l) {                        // down
    SpLevel& a = P->lev[l];
    SpLevel& c = P->lev[l + 1];
    const double* bl = l == 0 ? nullptr : a.b;
    const bool gat = a.local && !c.local;                  // restriction into the gathered level
    const Geo& gcl = gat ? c.gl : c.g;                     // this rank's part of the coarse level
    const dim3 gf(grid1d(a.g.N, SP_T), ell), gc(grid1d(gcl.N, SP_T), ell);
    if (fused) {                                           // smoothing + restriction in one pass
      int nsx, nt;
      spf_tiles(c.g.nx, c.g.ny, nsx, nt);
      const SpfUpd u = l == 0 ? U : SpfUpd{};
      // compulsory bytes: b (or the update operands + v_{j+1}), 1/D per block, wx, wy, cnt, b_c
      const double nb = u.on ? (4.0 * (ell - 2) + 2.0) : (double)ell;
      const double bytes = 8.0 * a.g.N * (nb + (ell / 2 + 1) + 3.0) + 8.0 * ell * c.g.N;
      // (AAC_SPF_TMA=2: also the staged-row level-0 restriction -- measured slower: 133 vs 95 us)
      static const bool rtma_on = getenv("AAC_SPF_TMA") && atoi(getenv("AAC_SPF_TMA")) == 2;
      if (l == 0 && a.g.nx % 2 == 0 && rtma_on) {
        // level 0: rows staged by the bulk-copy engine (k_spf_restrict_tma), ~2 CTAs per SM
        static thread_local bool attr = false;
        if (!attr) {
          CUDA_TRY(ctx, cudaFuncSetAttribute(k_spf_restrict_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)spr_smem()));
          attr = true;
        }
        const int nyp = (a.g.ny + 1) / 2;
        const int nch = std::min(nyp, std::max(1, 2 * ctx->num_sms / (nsx * (ell / 2))));
        const int nyc = (nyp + nch - 1) / nch, nchr = (nyp + nyc - 1) / nyc;
        LAUNCH(ctx, KID_SP_MG, bytes,
               launch_pdl(k_spf_restrict_tma, dim3(nsx * nchr, ell / 2), dim3(SPF_T), spr_smem(), ctx->stream, a.g,
                          c.g, (const double*)a.cnt, (const double*)a.dinv, P->K, io, c.b, u, nsx, nyc, st));
      } else if (a.g.nx % 2 == 0)
        LAUNCH(ctx, KID_SP_MG, bytes, launch_pdl(k_spf_restrict<true>, dim3(nt, ell / 2), dim3(SPF_T), 0, ctx->stream,
                                          a.g, c.g, a.cnt, a.dinv, P->K, io, bl, c.b, u, nsx, st));
      else
        LAUNCH(ctx, KID_SP_MG, bytes, launch_pdl(k_spf_restrict<false>, dim3(nt, ell / 2), dim3(SPF_T), 0, ctx->stream,
                                          a.g, c.g, a.cnt, a.dinv, P->K, io, bl, c.b, u, nsx, st));
      continue;
    }
    LAUNCH(ctx, KID_SP_MG, 16.0 * ell * a.g.N,
           k_mg_smooth0<DIM><<<gf, SP_T, 0, ctx->stream>>>(a.g, a.dinv, P->K, io, bl, a.x, st));
    if (a.local) AAC_TRY(sp_halo(ctx, a.g, a.x));
    if (gat) CUDA_TRY(ctx, cudaMemsetAsync(c.b, 0, (size_t)ell * c.g.N * sizeof(double), ctx->stream));
    static const bool no_pair = getenv("AAC_SP_PAIR") && atoi(getenv("AAC_SP_PAIR")) == 0;
    if (no_pair)
      LAUNCH(ctx, KID_SP_MG, 24.0 * ell * a.g.N,
             k_mg_restrict<DIM><<<gc, SP_T, 0, ctx->stream>>>(a.g, a.cnt, gcl, P->K, io, bl, a.x, c.b, st, hlo,
                                                              hhi, c.g.N, gat ? c.goff : 0));
    else
      LAUNCH(ctx, KID_SP_MG, 24.0 * ell * a.g.N,
             k_mg_restrict_pair<DIM><<<dim3(gc.x, ell / 2), SP_T, 0, ctx->stream>>>(
                 a.g, a.cnt, gcl, P->K, io, bl, a.x, c.b, st, hlo, hhi, c.g.N, gat ? c.goff : 0));
    if (gat) AAC_TRY(comm_allreduce(ctx, c.b, (int)(ell * c.g.N), ncclSum));
  }
  SpLevel& cl = P->lev[nl - 1];
  if (nl == 1) return aac_fail(ctx, AAC_EINVAL, "SP needs at least one coarsening (grid too small)");
  if (tl < nl) {
    MgTail T{};
    T.nlev = nl - tl;
    double bytes = 8.0 * ell * P->nc * P->nc;
    for (int i = 0; i < T.nlev; ++i) {
      const SpLevel& L = P->lev[tl + i];
      T.g[i] = L.g;
      T.cnt[i] = L.cnt;
      T.dinv[i] = L.dinv;
      T.b[i] = L.b;
      T.x[i] = L.x;
      T.x2[i] = L.x2;
      bytes += 8.0 * ell * L.g.N * 6;
    }
    T.minv = P->minv;
    T.nc = P->nc;
    LAUNCH(ctx, KID_SP_MG, bytes, launch_pdl(k_mg_tail<DIM>, dim3(ell), dim3(SP_TAIL_T), 0, ctx->stream, T, P->K, st));
  } else {
    LAUNCH(ctx, KID_SP_MG, 8.0 * ell * P->nc * P->nc,
           k_mg_coarse<<<ell, SP_T, 0, ctx->stream>>>(P->nc, P->minv, ell, cl.b, cl.x2, st));
  }
  for (int l = (tl < nl ? tl : nl - 1) - 1; l >= 0; --l) { // up
    SpLevel& a = P->lev[l];
    SpLevel& c = P->lev[l + 1];
    const double* bl = l == 0 ? nullptr : a.b;
    const bool gat = a.local && !c.local;
    const dim3 gf(grid1d(a.g.N, SP_T), ell);
    const dim3 gp(l == 0 ? std::min<unsigned>(gf.x, std::max(1, 8 * ctx->num_sms / ell)) : gf.x, ell);
    if (fused) {
      int nsx, nt;
      spf_tiles(c.g.nx, c.g.ny, nsx, nt);
      // level 0 (dot partials): grid-stride, ~SPF_CPS CTAs per SM -- the per-CTA fence and ticket
      // of the reduction made one row pair per CTA (10 240 CTAs) 1.4x slower
      if (l == 0) nt = nsx * std::min(c.g.ny, std::max(1, spf_cps() * ctx->num_sms / (nsx * (ell / 2))));
      const double bytes = 8.0 * a.g.N * (2.0 * ell + (ell / 2 + 1) + 3.0) + 8.0 * ell * c.g.N;
      // (AAC_SPF_TMA=2: also the staged-row level-0 prolongation -- measured slower: 83 vs 65 us)
      static const bool ptma_on = getenv("AAC_SPF_TMA") && atoi(getenv("AAC_SPF_TMA")) == 2;
      if (l == 0 && a.g.nx % 4 == 0 && ptma_on) {
        // level 0: rows staged by the bulk-copy engine (k_spf_prolong_tma), ~2 CTAs per SM
        static thread_local bool attr = false;
        if (!attr) {
          CUDA_TRY(ctx, cudaFuncSetAttribute(k_spf_prolong_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)spp_smem()));
          attr = true;
        }
        const int nyp = (a.g.ny + 1) / 2;
        const int nch = std::min(nyp, std::max(1, 2 * ctx->num_sms / (nsx * (ell / 2))));
        const int nyc = (nyp + nch - 1) / nch, nchr = (nyp + nyc - 1) / nyc;
        LAUNCH(ctx, KID_SP_MG, bytes,
               launch_pdl(k_spf_prolong_tma, dim3(nsx * nchr, ell / 2), dim3(SPF_T), spp_smem(), ctx->stream, a.g, c.g,
                          (const double*)a.cnt, (const double*)a.dinv, io, (const double*)c.x2, S, P->red2, nsx, nyc));
      } else if (a.g.nx % 2 == 0)
        LAUNCH(ctx, KID_SP_MG, bytes, launch_pdl(k_spf_prolong_post<true>, dim3(nt, ell / 2), dim3(SPF_T), 0, ctx->stream,
                                          a.g, c.g, a.cnt, a.dinv, io, bl, c.x2, a.x2, S, P->red2, l == 0 ? 1 : 0, nsx));
      else
        LAUNCH(ctx, KID_SP_MG, bytes, launch_pdl(k_spf_prolong_post<false>, dim3(nt, ell / 2), dim3(SPF_T), 0, ctx->stream,
                                          a.g, c.g, a.cnt, a.dinv, io, bl, c.x2, a.x2, S, P->red2, l == 0 ? 1 : 0, nsx));
      continue;
    }
    if (ctx->nranks > 1 && a.local) {                      // slab level: prolong, halo, post
      LAUNCH(ctx, KID_SP_MG, 24.0 * ell * a.g.N,
             k_mg_prolong<DIM><<<gf, SP_T, 0, ctx->stream>>>(a.g, gat ? c.gl : c.g, a.x, c.x2, st, c.g.N,
                                                             gat ? c.goff : 0));
      AAC_TRY(sp_halo(ctx, a.g, a.x));
      LAUNCH(ctx, KID_SP_MG, 24.0 * ell * a.g.N,
             k_mg_post<DIM><<<gp, SP_T, 0, ctx->stream>>>(a.g, a.cnt, a.dinv, io, bl, a.x, a.x2, S, l == 0 ? 1 : 0,
                                                          hlo, hhi));
    } else {                                               // x, x_c, b in; x2 out (+ C)
      static const bool no_pair = getenv("AAC_SP_PAIR") && atoi(getenv("AAC_SP_PAIR")) == 0;
      static const bool no_row2d = getenv("AAC_SP_ROW2D") && atoi(getenv("AAC_SP_ROW2D")) == 0;
      if (no_pair)
        LAUNCH(ctx, KID_SP_MG, 8.0 * ell * (3.0 * a.g.N + c.g.N) + 8.0 * DIM * a.g.N,
               k_mg_prolong_post<DIM><<<gp, SP_T, 0, ctx->stream>>>(a.g, a.cnt, a.dinv, c.g, io, bl, a.x, c.x2,
                                                                    a.x2, S, l == 0 ? 1 : 0));
      else if (DIM == 2 && !no_row2d)                      // row grid: grid-stride over rows
        LAUNCH(ctx, KID_SP_MG, 8.0 * ell * (3.0 * a.g.N + c.g.N) + 8.0 * DIM * a.g.N,
               k_mg_prolong_post_pair2<<<dim3(std::min<unsigned>(gp.x, (unsigned)a.g.ny), ell / 2), SP_T, 0,
                                         ctx->stream>>>(a.g, a.cnt, a.dinv, c.g, io, bl, a.x, c.x2, a.x2, S,
                                                        l == 0 ? 1 : 0));
      else
        LAUNCH(ctx, KID_SP_MG, 8.0 * ell * (3.0 * a.g.N + c.g.N) + 8.0 * DIM * a.g.N,
               k_mg_prolong_post_pair<DIM><<<dim3(gp.x, ell / 2), SP_T, 0, ctx->stream>>>(
                   a.g, a.cnt, a.dinv, c.g, io, bl, a.x, c.x2, a.x2, S, l == 0 ? 1 : 0));
    }
  }
  return AAC_OK;
}

// Inner solve on hat w (ctx->d_what) -> packed y in P->X -> inverse DFT -> z (zbase + j*zjs).
template <int DIM>
static int sp_solve_t(aac_ctx* ctx, int k, double* zbase, long long zjs, const IterState* st) {
  SpPlan* P = ctx->sp;
  const int ell = P->ell, h = P->h;
  const long long N = ctx->geo.N;
  const double V = 8.0 * ell * N;
  double *Vp = P->Vb[0], *Vc = P->Vb[1], *Vn = P->Vb[2];
  double *Zc = P->Zb[0], *Zn = P->Zb[1];
  double *Wp = P->Wb[0], *Wc = P->Wb[1], *Wn = P->Wb[2];
  auto vecs = [&]() {
    SpVec v{P->X, Vp, Vc, Vn, Zc, Wp, Wc, Wn, P->SZ, P->R, P->P, P->Zr, ctx->d_what};
    return v;
  };
  auto io_for = [&](bool init) {
    MgIo io{};
    for (int pl = 0; pl < ell; ++pl) {
      const int kb = pl == 0 ? 0 : (pl == ell - 1 ? h : (pl + 1) / 2);
      const long long o = (long long)pl * N;
      if (kb == 0 || kb == h) {
        io.in[pl] = P->R + o;
        io.out[pl] = (init ? P->P : P->Zr) + o;
      } else {
        io.in[pl] = (init ? Vc : Vn) + o;
        io.out[pl] = (init ? Zc : Zn) + o;
      }
    }
    return io;
  };
  const bool multi = ctx->multi();
  SpStepCtx S{P->blk, P->part, P->tick, P->K, 0, st, multi ? P->red : nullptr, ctx->d_halo,
              ctx->d_halo + (long long)ell * ctx->geo.S};
  // multi-rank: all-reduce the local sums of the last kernel, then the scalar step
  auto finish = [&](int nq, int stepB) -> int {
    if (!multi) return AAC_OK;
    AAC_TRY(comm_allreduce(ctx, P->red, nq, ncclSum));
    LAUNCH(ctx, KID_SCALAR, 0, k_sp_scalar<<<1, 1, 0, ctx->stream>>>(S, stepB));
    return AAC_OK;
  };
  const unsigned gt = grid1d(N, SP_T);
  LAUNCH(ctx, KID_SP_VEC, 2.0 * V, launch_pdl(k_sp_init, dim3(gt), dim3(SP_T), 0, ctx->stream, N, ell, vecs(), st));
  S.phase = 0;
  AAC_TRY(sp_vcycle<DIM>(ctx, io_for(true), S));          // z_1 = M v_1 ; p_0 = M r_0
  AAC_TRY(finish(ell, 1));
  S.phase = 1;
  for (int it = 0; it < k; ++it) {
    if (multi) {                                           // halos of P (real) and Z (complex)
      const double* planes[AAC_MAX_ELL];
      int qs[AAC_MAX_ELL];
      for (int pl = 0; pl < ell; ++pl) {
        const int kb = pl == 0 ? 0 : (pl == ell - 1 ? h : (pl + 1) / 2);
        planes[pl] = ((kb == 0 || kb == h) ? P->P : Zc) + (long long)pl * N;
        qs[pl] = pl;
      }
      AAC_TRY(comm_halo(ctx, planes, qs, ell));
    }
    static const bool no_row2d = getenv("AAC_SP_ROW2D") && atoi(getenv("AAC_SP_ROW2D")) == 0;
    const unsigned gsa = std::min<unsigned>(gt, std::max(1, 8 * ctx->num_sms / (h + 1)));
    if (sp_fused_on(ctx, DIM)) {
      const int nsx = ((ctx->geo.nx + 1) / 2 + SPF_T - 1) / SPF_T, nyp = (ctx->geo.ny + 1) / 2;
      const int nry = std::min(nyp, std::max(1, spf_cps() * ctx->num_sms / (nsx * h)));
      static const bool tma_off = getenv("AAC_SPF_TMA") && atoi(getenv("AAC_SPF_TMA")) == 0;
      if (ctx->geo.nx % 2 == 0 && !tma_off) {
        // rows staged by the bulk-copy engine; ~SPT_MINB CTAs per SM, chunks of nyc aggregate rows
        static thread_local bool attr = false;
        if (!attr) {
          CUDA_TRY(ctx, cudaFuncSetAttribute(k_spf_apply_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)spt_smem()));
          attr = true;
        }
        const int nch = std::min(nyp, std::max(1, SPT_MINB * ctx->num_sms / (nsx * h)));
        const int nyc = (nyp + nch - 1) / nch;
        const int nchr = (nyp + nyc - 1) / nyc;
        LAUNCH(ctx, KID_SP_STENCIL, 2.0 * V,
               launch_pdl(k_spf_apply_tma, dim3(nsx * nchr, h), dim3(SPF_T), spt_smem(), ctx->stream, ctx->geo, vecs(),
                          S, P->red2, nsx, nyc));
      } else if (ctx->geo.nx % 2 == 0)
        LAUNCH(ctx, KID_SP_STENCIL, 2.0 * V,
               launch_pdl(k_spf_apply<true>, dim3(nsx * nry, h), dim3(SPF_T), 0, ctx->stream, ctx->geo, vecs(), S, P->red2, nsx));
      else
        LAUNCH(ctx, KID_SP_STENCIL, 2.0 * V,
               launch_pdl(k_spf_apply<false>, dim3(nsx * nry, h), dim3(SPF_T), 0, ctx->stream, ctx->geo, vecs(), S, P->red2, nsx));
    } else if (DIM == 2 && !no_row2d)
      LAUNCH(ctx, KID_SP_STENCIL, 2.0 * V,
             k_sp_apply2<<<dim3(std::min<unsigned>(gsa, (unsigned)ctx->geo.ny), h + 1), SP_T, 0, ctx->stream>>>(
                 ctx->geo, vecs(), S));
    else
      LAUNCH(ctx, KID_SP_STENCIL, 2.0 * V,
             k_sp_apply<DIM><<<dim3(gsa, h + 1), SP_T, 0, ctx->stream>>>(ctx->geo, vecs(), S));
    AAC_TRY(finish(h + 1, 0));
    // CTAs per plane of the vector updates (grid-stride): 4 x SMs per plane (measured: 237 -> 592
    // took the saddle solve from 64.8 to 63.3 ms; a full one-element-per-thread grid was slower)
    static const int upd_env = getenv("AAC_SP_UPD_CAP") ? atoi(getenv("AAC_SP_UPD_CAP")) : 0;
    const unsigned upd_cap = upd_env > 0 ? (unsigned)upd_env : (unsigned)(4 * ctx->num_sms);
    if (sp_fused_on(ctx, DIM)) {
      // complex planes: v_{j+1} formed inside the level-0 restriction; real planes here
      LAUNCH(ctx, KID_SP_VEC, 3.0 * V * 2 / ell,
             launch_pdl(k_sp_upd1_real, dim3(std::min<unsigned>(gt, upd_cap), 2), dim3(SP_T), 0, ctx->stream,
                        N, ell, vecs(), P->blk, st));
      AAC_TRY(sp_vcycle<DIM>(ctx, io_for(false), S, SpfUpd{P->SZ, Vc, Vp, P->blk, 1}));
    } else {
      LAUNCH(ctx, KID_SP_VEC, 3.0 * V,
             k_sp_upd1<<<dim3(std::min<unsigned>(gt, upd_cap), ell), SP_T, 0, ctx->stream>>>(
                 N, ell, vecs(), P->blk, st));
      AAC_TRY(sp_vcycle<DIM>(ctx, io_for(false), S));
    }
    AAC_TRY(finish(ell, 1));
    LAUNCH(ctx, KID_SP_VEC, 4.0 * V,
           launch_pdl(k_sp_upd2, dim3(std::min<unsigned>(gt, upd_cap), ell), dim3(SP_T), 0, ctx->stream,
                      N, ell, vecs(), P->blk, st));
    // rotate: v_prev <- v <- v_next, z <- z_next, w_prev <- w <- w_next
    double* t = Vp; Vp = Vc; Vc = Vn; Vn = t;
    t = Zc; Zc = Zn; Zn = t;
    t = Wp; Wp = Wc; Wc = Wn; Wn = t;
  }
  // z = Gamma^{-1} U y (y packed in X): the same inverse transform with unit block scales
  NcFinal F{};
  for (int kb = 0; kb <= h; ++kb) {
    F.tr[kb] = 1.0;
    F.ti[kb] = 0.0;
    F.src[kb] = P->X + (long long)(kb == 0 ? 0 : (kb == h ? ell - 1 : 2 * kb - 1)) * N;
  }
  const Dft D = make_dft(ctx);
  AAC_TRY(run_inverse(ctx, D, F, zbase, zjs, st));
  return AAC_OK;
}

static int sp_solve(aac_ctx* ctx, int k, double* zbase, long long zjs, const IterState* st) {
  switch (ctx->dim) {
    case 1: return sp_solve_t<1>(ctx, k, zbase, zjs, st);
    case 2: return sp_solve_t<2>(ctx, k, zbase, zjs, st);
    default: return sp_solve_t<3>(ctx, k, zbase, zjs, st);
  }
}

static long long sp_paper_matvecs(const aac_ctx* ctx, int k) { return 2LL * (ctx->ell - 1) * k; }
