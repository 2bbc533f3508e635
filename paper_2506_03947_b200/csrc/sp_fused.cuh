// sp_fused.cuh -- 2D one-rank V-cycle level kernels of P_SP (§5.1, 694-697; reading R16):
// the same pre-smoothing / restriction / prolongation / post-smoothing as k_mg_smooth0,
// k_mg_restrict_pair and k_mg_prolong_post_pair2 (sp.cuh), organised for HBM instead of for
// simplicity:
//  * the pre-smoothed iterate x = omega b / D (smoothing from zero) is never stored: the
//    restriction and the post-smoothing form it from b and 1/D where they need it (the
//    separate smoothing pass and the iterate's write and two re-reads go away);
//  * one thread owns one aggregate (fine columns 2X, 2X+1: one 16-byte load per array and row;
//    fine rows 2Y, 2Y+1 plus the neighbour rows above and below) of a plane pair; the
//    x-neighbours come from the adjacent lanes (warp shuffles; the two warp-edge lanes form
//    their outside column themselves). A row-marching variant (each thread walking 16 rows with
//    the y-neighbours in registers) was slower: 3 CTAs per SM by registers and one dependent
//    load round trip per row (saddle solve 86 ms against 63.6 ms for the per-step kernels);
//  * level 0 of an inner MINRES iteration also forms its right-hand side v_{j+1} = S z -
//    (delta/gamma) v_j - (gamma/gamma_prev) v_{j-1} (k_sp_upd1 of the complex blocks) on the fly
//    and stores it: the update pass disappears into the restriction.
// Per point and plane pair the arithmetic is the generic kernels', in the same order (up to the
// association of the fixed-order dot reduction).
#pragma once

#include "tma.cuh"

constexpr int SPF_T = 128;                     // threads = aggregate columns per CTA
#ifndef SPF_MINB
#define SPF_MINB 4                             // __launch_bounds__ min CTAs per SM (register cap)
#endif

struct SpfUpd {                                // level 0, inner iteration: v_{j+1} on the fly
  const double* SZ;
  const double* Vc;
  const double* Vp;
  const SpBlk* blk;
  int on;
};

// Row y of a plane pair at fine columns c0 = 2X, c0 + 1 (value 0 outside the domain).
template <bool EVEN>
__device__ __forceinline__ void spf_ld2(const double* p, int c0, bool v0, bool v1, double& a, double& b) {
  if (EVEN) {
    if (v0) {
      const double2 t = __ldg(reinterpret_cast<const double2*>(p + c0));
      a = t.x;
      b = t.y;
    } else {
      a = b = 0.0;
    }
  } else {
    a = v0 ? __ldg(p + c0) : 0.0;
    b = v1 ? __ldg(p + c0 + 1) : 0.0;
  }
}

template <bool EVEN>
__device__ __forceinline__ void spf_st2(double* p, int c0, bool v0, bool v1, double a, double b) {
  if (EVEN) {
    if (v0) *reinterpret_cast<double2*>(p + c0) = make_double2(a, b);
  } else {
    if (v0) p[c0] = a;
    if (v1) p[c0 + 1] = b;
  }
}

// One thread per aggregate (X, Y): fine columns c0 = 2X, c0 + 1 and rows y0 = 2Y, y0 + 1, with
// the rows y0 - 1 and y0 + 2 of their y-neighbours. Every load of a thread is issued before any
// arithmetic (rows and columns outside the level are clamped to valid addresses and their values
// discarded): one memory round trip per thread. (Loads behind row-validity branches cost one
// round trip per branch: 2-3x slower.)
struct SpfGeom {
  int X, Y, c0, lane;
  int cl;                      // load column: c0, clamped into the level
  int ce;                      // this lane's warp-edge column (lanes < 16: west of the warp,
                               // >= 16: east of it), clamped
  bool v0, v1;                 // columns inside the level
  bool r1;                     // row y0 + 1 inside the level
  bool rm, rp;                 // rows y0 - 1 / y0 + 2 inside the level
  bool ew, ee;                 // lane 0: west column inside; lane 31: east column inside
  long long rA, rB, rM, rP;    // row offsets (clamped: rB = rA, rM = rA, rP = rB outside)
};

__device__ __forceinline__ SpfGeom spf_geom(const Geo& g, int nsx, int Y) {
  SpfGeom G;
  G.X = (blockIdx.x % nsx) * SPF_T + threadIdx.x;
  G.Y = Y;
  G.c0 = 2 * G.X;
  G.lane = threadIdx.x & 31;
  G.v0 = G.c0 < g.nx;
  G.v1 = G.c0 + 1 < g.nx;
  G.cl = G.v0 ? G.c0 : (g.nx - 1) & ~1;
  const int ce = G.lane < 16 ? G.c0 - 2 * G.lane - 1 : G.c0 + 2 * (31 - G.lane) + 2;
  G.ce = min(max(ce, 0), g.nx - 1);
  G.ew = G.c0 - 1 >= 0;
  G.ee = G.c0 + 2 < g.nx;
  const int y0 = 2 * G.Y;
  G.r1 = y0 + 1 < g.ny;
  G.rm = G.Y > 0;
  G.rp = y0 + 2 < g.ny;
  G.rA = (long long)y0 * g.nx;
  G.rB = G.r1 ? G.rA + g.nx : G.rA;
  G.rM = G.rm ? G.rA - g.nx : G.rA;
  G.rP = G.rp ? G.rB + g.nx : G.rB;
  return G;
}

// Unconditional pair load at the clamped column (EVEN: one 16-byte load).
template <bool EVEN>
__device__ __forceinline__ double2 spf_l2(const double* p, const SpfGeom& G, int nx) {
  if (EVEN) return __ldg(reinterpret_cast<const double2*>(p + G.cl));
  return make_double2(__ldg(p + G.cl), __ldg(p + min(G.cl + 1, nx - 1)));
}

// Lane-to-lane x-neighbours: west of c0 (lane - 1's right column or, at lane 0, the warp-edge
// value `ed` of lane 0) and east of c0 + 1 (lane + 1's left column or, at lane 31, lane 31's `ed`).
__device__ __forceinline__ void spf_xnb(double x0, double x1, double ed, int lane, double& w, double& ea) {
  const double up = __shfl_up_sync(0xffffffffu, x1, 1);
  const double dn = __shfl_down_sync(0xffffffffu, x0, 1);
  w = lane == 0 ? ed : up;
  ea = lane == 31 ? ed : dn;
}

// Face weights and counts of the rows y0 (A) and y0 + 1 (B), lower wy of y0 + 2 (P).
struct SpfW {
  double wxA0, wxA1, wxA2, wyA0, wyA1, kA0, kA1;
  double wxB0, wxB1, wxB2, wyB0, wyB1, kB0, kB1;
  double wyP0, wyP1;
};

// Raw loads of the face weights and counts (issued first; spf_wfin forms SpfW from them -- its
// shuffles wait for the loads, so a kernel issues its other loads in between).
struct SpfWRaw {
  double2 xa, xb, ya, yb, ka, kb, yp;
  double xa2, xb2;
};

template <bool EVEN, bool CNT = true>
__device__ __forceinline__ void spf_wload(const Geo& g, const double* cnt, const SpfGeom& G, SpfWRaw& R) {
  const int nx = g.nx;
  R.xa = spf_l2<EVEN>(g.wx + G.rA, G, nx);
  R.xb = spf_l2<EVEN>(g.wx + G.rB, G, nx);
  R.ya = spf_l2<EVEN>(g.wy + G.rA, G, nx);
  R.yb = spf_l2<EVEN>(g.wy + G.rB, G, nx);
  R.ka = CNT ? spf_l2<EVEN>(cnt + G.rA, G, nx) : make_double2(1.0, 1.0);
  R.kb = CNT ? spf_l2<EVEN>(cnt + G.rB, G, nx) : make_double2(1.0, 1.0);
  R.yp = spf_l2<EVEN>(g.wy + G.rB + nx, G, nx);   // row y0 + 2 or the zero padding row
  // face (c0+1 | c0+2): lane + 1's wx[c0'], lane 31 loads it (c0 + 2 <= nx: wx has nx + 1 entries
  // per row position in the padded layout)
  const int c2 = min(G.c0 + 2, nx);
  R.xa2 = __ldg(g.wx + G.rA + c2);
  R.xb2 = __ldg(g.wx + G.rB + c2);
}

__device__ __forceinline__ void spf_wfin(const Geo& g, const SpfGeom& G, const SpfWRaw& R, SpfW& W) {
  const int nx = g.nx;
  const bool in = G.v0;
  // (lane + 1 outside the level: its clamped load is not a face of this row -- shuffle zero)
  const double na = __shfl_down_sync(0xffffffffu, in ? R.xa.x : 0.0, 1);
  const double nb = __shfl_down_sync(0xffffffffu, in ? R.xb.x : 0.0, 1);
  W.wxA0 = in ? R.xa.x : 0.0;
  W.wxA1 = in ? R.xa.y : 0.0;
  W.wxA2 = G.lane == 31 ? (G.c0 + 2 <= nx ? R.xa2 : 0.0) : na;
  W.wyA0 = in ? R.ya.x : 0.0;
  W.wyA1 = in ? R.ya.y : 0.0;
  W.kA0 = R.ka.x;
  W.kA1 = R.ka.y;
  const bool inB = in && G.r1;
  W.wxB0 = inB ? R.xb.x : 0.0;
  W.wxB1 = inB ? R.xb.y : 0.0;
  W.wxB2 = G.lane == 31 ? (G.c0 + 2 <= nx && G.r1 ? R.xb2 : 0.0) : (G.r1 ? nb : 0.0);
  W.wyB0 = inB ? R.yb.x : 0.0;
  W.wyB1 = inB ? R.yb.y : 0.0;
  W.kB0 = R.kb.x;
  W.kB1 = R.kb.y;
  W.wyP0 = inB ? R.yp.x : 0.0;
  W.wyP1 = inB ? R.yp.y : 0.0;
}

template <bool EVEN, bool CNT = true>
__device__ __forceinline__ void spf_weights(const Geo& g, const double* cnt, const SpfGeom& G, SpfW& W) {
  SpfWRaw R;
  spf_wload<EVEN, CNT>(g, cnt, G, R);
  spf_wfin(g, G, R, W);
}

// ---- reductions of the fused kernels ----------------------------------------------------------
// Two levels, fixed order (bitwise reproducible): the CTAs of tile group g (SPF_GROUP consecutive
// tiles of every pair) count on their own ticket; the group's last CTA sums the group's partials
// into gpart[q][g]; the last group sums those (one group: the group sum is the total). The
// kernels launch ~4 CTAs per SM (one group): with one row pair per CTA (10 240 CTAs, 40 groups)
// the per-CTA fence and ticket made them 1.4x slower.
constexpr int SPF_GROUP = 256;
constexpr int SPF_TICK_STRIDE = 8;             // 32 bytes between group tickets

// tot[q] = sum_{i < n} base[q * stride + i], q < nq; thread t sums i = t, t + T, ... ascending, then
// the warps' sums in warp order.
__device__ void spf_sum_multi(const double* base, int nq, int n, long long stride, double* tot) {
  __shared__ double ws[AAC_MAX_ELL][SPF_T / 32];
  double acc[AAC_MAX_ELL];
#pragma unroll
  for (int q = 0; q < AAC_MAX_ELL; ++q) acc[q] = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
#pragma unroll
    for (int q = 0; q < AAC_MAX_ELL; ++q)
      if (q < nq) acc[q] += __ldcg(base + (long long)q * stride + i);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < AAC_MAX_ELL; ++q) {
    if (q < nq) {
      const double v = warp_sum(acc[q]);
      if (lane == 0) ws[q][w] = v;
    }
  }
  __syncthreads();
  if ((int)threadIdx.x < nq) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += ws[threadIdx.x][k];
    tot[threadIdx.x] = t;
  }
  __syncthreads();
}

// After this CTA stored its partials part[q * gridDim.x + blockIdx.x] (thread 0, fenced): true in
// the one CTA that ends with tot[q] = the total of plane q, q < nq.
__device__ bool spf_reduce2(const double* part, const SpfRed& R, int nq, double* tot) {
  __shared__ bool lastg, lasta;
  const int ntile = gridDim.x, ng = (ntile + SPF_GROUP - 1) / SPF_GROUP, g = blockIdx.x / SPF_GROUP;
  const int t0 = g * SPF_GROUP, nt = min(SPF_GROUP, ntile - t0);
  if (threadIdx.x == 0) {
    const unsigned tk = atomicAdd(R.gtick + (long long)g * SPF_TICK_STRIDE, 1u);
    lastg = (tk == (unsigned)(nt * gridDim.y) - 1);
  }
  __syncthreads();
  if (!lastg) return false;
  __threadfence();
  spf_sum_multi(part + t0, nq, nt, ntile, tot);
  if (ng == 1) {                                           // one group: that was the total
    if (threadIdx.x == 0) R.gtick[0] = 0;
    return true;
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < nq; ++q) R.gpart[(long long)q * ng + g] = tot[q];
    R.gtick[(long long)g * SPF_TICK_STRIDE] = 0;
    __threadfence();
    const unsigned tk = atomicAdd(R.gtick + (long long)ng * SPF_TICK_STRIDE, 1u);
    lasta = (tk == (unsigned)ng - 1);
  }
  __syncthreads();
  if (!lasta) return false;
  __threadfence();
  spf_sum_multi(R.gpart, nq, ng, ng, tot);
  if (threadIdx.x == 0) R.gtick[(long long)ng * SPF_TICK_STRIDE] = 0;
  return true;
}

// Per-(pair, CTA) partials (va -> plane pa, vb -> plane pb); the CTA that completes the sum of
// every plane runs scalar step B (k_mg_prolong_post_pair's sp_reduce_pair).
__device__ __forceinline__ void spf_reduce_pair(const SpStepCtx& S, const SpfRed& R, double va, double vb, int pa,
                                                int pb) {
  __shared__ double red[2][SPF_T / 32];
  __shared__ double tot[AAC_MAX_ELL];
  va = warp_sum(va);
  vb = warp_sum(vb);
  const int t = threadIdx.x, ntile = gridDim.x;
  if ((t & 31) == 0) {
    red[0][t >> 5] = va;
    red[1][t >> 5] = vb;
  }
  __syncthreads();
  if (t == 0) {
    double sa = 0.0, sb = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      sa += red[0][w];
      sb += red[1][w];
    }
    S.part[(long long)pa * ntile + blockIdx.x] = sa;
    S.part[(long long)pb * ntile + blockIdx.x] = sb;
    __threadfence();
  }
  const int ell = S.K.ell;
  if (!spf_reduce2(S.part, R, ell, tot)) return;
  if (t == 0) {
    if (S.red) {
      for (int q = 0; q < ell; ++q) S.red[q] = tot[q];
    } else {
      sp_scalar_B(S, tot);
    }
  }
}

// ---- restriction with the pre-smoothing on the fly ------------------------------------------
// bc(X, Y) = sum over the (<= 4) children, row-major, of (b - A_l(s) x)_child, x = omega b / D,
// A_l(s) u = m u + sum_f w_f (u - u_nb), m = (1 + s) cnt -- k_mg_smooth0 + k_mg_restrict_pair.
// A neighbour outside the level is the point itself (its face weight is zero).
template <bool EVEN>
__global__ void __launch_bounds__(SPF_T, SPF_MINB) k_spf_restrict(Geo g, Geo gc, const double* __restrict__ cnt,
                                                           const double* __restrict__ dinv, SpConst K, MgIo io,
                                                           const double* bl, double* bc, SpfUpd U, int nsx,
                                                           const IterState* st) {
  griddep();
  if (st && st->done) return;
  int pa, pb;
  sp_pair(K.ell, blockIdx.y, pa, pb);
  const SpfGeom G = spf_geom(g, nsx, blockIdx.x / nsx);
  const int nx = g.nx;
  SpfW W;
  spf_weights<EVEN>(g, cnt, G, W);
  const int pls[2] = {pa, pb};
  double acc[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int pl = pls[e];
    const int kb = sp_block_of(K.ell, pl);
    const double* dq = dinv + (long long)kb * g.N;
    const double m = 1.0 + K.s[pl];
    const bool upd = U.on && kb != 0 && kb != K.ell / 2 && U.blk[kb].stop != 1;
    // b of rows A, B, M, P and of the warp-edge column of rows A, B: stored, or v_{j+1} formed
    // from the update operands exactly as k_sp_upd1 does
    double2 bA, bB, bM, bP;
    double beA, beB;
    if (upd) {
      const long long o = (long long)pl * g.N;
      const double *sz = U.SZ + o, *vc = U.Vc + o, *vp = U.Vp + o;
      const double dc = U.blk[kb].dcoef, vcf = U.blk[kb].vcoef;
      auto v2 = [&](long long r) {
        const double2 a = spf_l2<EVEN>(sz + r, G, nx), b = spf_l2<EVEN>(vc + r, G, nx), c = spf_l2<EVEN>(vp + r, G, nx);
        return make_double2(a.x - dc * b.x - vcf * c.x, a.y - dc * b.y - vcf * c.y);
      };
      auto v1 = [&](long long r) {
        const long long q = r + G.ce;
        return __ldg(sz + q) - dc * __ldg(vc + q) - vcf * __ldg(vp + q);
      };
      bA = v2(G.rA);
      bB = v2(G.rB);
      bM = v2(G.rM);
      bP = v2(G.rP);
      beA = v1(G.rA);
      beB = v1(G.rB);
      double* vn = const_cast<double*>(io.in[pl]);         // v_{j+1} of the own points
      spf_st2<EVEN>(vn + G.rA, G.c0, G.v0, G.v1, bA.x, bA.y);
      if (G.r1) spf_st2<EVEN>(vn + G.rB, G.c0, G.v0, G.v1, bB.x, bB.y);
    } else {
      const double* bq = bl ? bl + (long long)pl * g.N : io.in[pl];
      bA = spf_l2<EVEN>(bq + G.rA, G, nx);
      bB = spf_l2<EVEN>(bq + G.rB, G, nx);
      bM = spf_l2<EVEN>(bq + G.rM, G, nx);
      bP = spf_l2<EVEN>(bq + G.rP, G, nx);
      beA = __ldg(bq + G.rA + G.ce);
      beB = __ldg(bq + G.rB + G.ce);
    }
    const double2 dA = spf_l2<EVEN>(dq + G.rA, G, nx), dB = spf_l2<EVEN>(dq + G.rB, G, nx);
    const double2 dM = spf_l2<EVEN>(dq + G.rM, G, nx), dP = spf_l2<EVEN>(dq + G.rP, G, nx);
    const double deA = __ldg(dq + G.rA + G.ce), deB = __ldg(dq + G.rB + G.ce);
    // pre-smoothed iterate x = omega b / D (outside rows: the row itself)
    const double xA0 = SP_OMEGA * bA.x * dA.x, xA1 = SP_OMEGA * bA.y * dA.y;
    const double xB0 = SP_OMEGA * bB.x * dB.x, xB1 = SP_OMEGA * bB.y * dB.y;
    const double xM0 = SP_OMEGA * bM.x * dM.x, xM1 = SP_OMEGA * bM.y * dM.y;
    const double xP0 = SP_OMEGA * bP.x * dP.x, xP1 = SP_OMEGA * bP.y * dP.y;
    double wA, eA, wB, eB;
    spf_xnb(xA0, xA1, SP_OMEGA * beA * deA, G.lane, wA, eA);
    spf_xnb(xB0, xB1, SP_OMEGA * beB * deB, G.lane, wB, eB);
    auto res = [&](double c, double b, double xw, double xe, double xn, double xs, double fw, double fe, double fn,
                   double fs, double k) {
      double a = c;
      a = fma(fw, c - xw, a);
      a = fma(fe, c - xe, a);
      a = fma(fn, c - xn, a);
      a = fma(fs, c - xs, a);
      a = a + (m * k - 1.0) * c;
      return b - a;
    };
    double s = 0.0;
    if (G.v0) s += res(xA0, bA.x, wA, xA1, xM0, xB0, W.wxA0, W.wxA1, W.wyA0, W.wyB0, W.kA0);
    if (G.v1) s += res(xA1, bA.y, xA0, eA, xM1, xB1, W.wxA1, W.wxA2, W.wyA1, W.wyB1, W.kA1);
    if (G.r1) {
      if (G.v0) s += res(xB0, bB.x, wB, xB1, xA0, xP0, W.wxB0, W.wxB1, W.wyB0, W.wyP0, W.kB0);
      if (G.v1) s += res(xB1, bB.y, xB0, eB, xA1, xP1, W.wxB1, W.wxB2, W.wyB1, W.wyP1, W.kB1);
    }
    acc[e] = s;
  }
  if (G.X < gc.nx) {
    const long long oc = (long long)G.Y * gc.nx + G.X;
    bc[(long long)pa * gc.N + oc] = acc[0];
    bc[(long long)pb * gc.N + oc] = acc[1];
  }
}

// ---- prolongation + post-smoothing with the pre-smoothed iterate on the fly ---------------
// u = x + P x_c (x = omega b / D), x2 = u + omega (b - A_l(s) u) / D; level 0: x2 -> io.out
// and the per-plane dot <x2, b> (scalar step B by the last CTA) -- k_mg_prolong_post_pair2.
template <bool EVEN>
__global__ void __launch_bounds__(SPF_T, SPF_MINB) k_spf_prolong_post(Geo g, Geo gc, const double* __restrict__ cnt,
                                                               const double* __restrict__ dinv, MgIo io,
                                                               const double* bl, const double* __restrict__ xc,
                                                               double* x2l, SpStepCtx S, SpfRed R, int level0,
                                                               int nsx) {
  griddep();
  if (S.st && S.st->done) return;
  int pa, pb;
  sp_pair(S.K.ell, blockIdx.y, pa, pb);
  double dot[2] = {0.0, 0.0};
  const int nry = gridDim.x / nsx;
  for (int Y = blockIdx.x / nsx; Y < gc.ny; Y += nry) {     // (one row pair per CTA by default)
  const SpfGeom G = spf_geom(g, nsx, Y);
  const int nx = g.nx;
  SpfW W;
  spf_weights<EVEN>(g, cnt, G, W);
  // aggregates: (X, Y) of rows A, B; (X, Y -+ 1) of rows M, P (clamped); the warp-edge column's
  const int Xc = min(G.X, gc.nx - 1);
  const long long cA = (long long)G.Y * gc.nx, cM = G.rm ? cA - gc.nx : cA, cP = G.rp ? cA + gc.nx : cA;
  const int pls[2] = {pa, pb};
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int pl = pls[e];
    const double* bq = bl ? bl + (long long)pl * g.N : io.in[pl];
    const double* dq = dinv + (long long)sp_block_of(S.K.ell, pl) * g.N;
    const double* cq = xc + (long long)pl * gc.N;
    double* oq = level0 ? io.out[pl] : x2l + (long long)pl * g.N;
    const double m1 = 1.0 + S.K.s[pl];
    const double2 bA = spf_l2<EVEN>(bq + G.rA, G, nx), bB = spf_l2<EVEN>(bq + G.rB, G, nx);
    const double2 bM = spf_l2<EVEN>(bq + G.rM, G, nx), bP = spf_l2<EVEN>(bq + G.rP, G, nx);
    const double2 dA = spf_l2<EVEN>(dq + G.rA, G, nx), dB = spf_l2<EVEN>(dq + G.rB, G, nx);
    const double2 dM = spf_l2<EVEN>(dq + G.rM, G, nx), dP = spf_l2<EVEN>(dq + G.rP, G, nx);
    const double xcA = __ldg(cq + cA + Xc), xcM = __ldg(cq + cM + Xc), xcP = __ldg(cq + cP + Xc);
    const double beA = __ldg(bq + G.rA + G.ce), beB = __ldg(bq + G.rB + G.ce);
    const double deA = __ldg(dq + G.rA + G.ce), deB = __ldg(dq + G.rB + G.ce);
    const double xce = __ldg(cq + cA + (G.ce >> 1));
    const double uA0 = SP_OMEGA * bA.x * dA.x + xcA, uA1 = SP_OMEGA * bA.y * dA.y + xcA;
    const double uB0 = SP_OMEGA * bB.x * dB.x + xcA, uB1 = SP_OMEGA * bB.y * dB.y + xcA;
    const double uM0 = G.rm ? SP_OMEGA * bM.x * dM.x + xcM : uA0, uM1 = G.rm ? SP_OMEGA * bM.y * dM.y + xcM : uA1;
    const double uP0 = G.rp ? SP_OMEGA * bP.x * dP.x + xcP : uB0, uP1 = G.rp ? SP_OMEGA * bP.y * dP.y + xcP : uB1;
    double wA, eA, wB, eB;
    spf_xnb(uA0, uA1, SP_OMEGA * beA * deA + xce, G.lane, wA, eA);
    spf_xnb(uB0, uB1, SP_OMEGA * beB * deB + xce, G.lane, wB, eB);
    auto post = [&](double u0, double b, double d, double uw, double ue, double un, double us, double fw, double fe,
                    double fn, double fs, double k) {
      double a = (m1 * k) * u0;
      a = fma(fw, u0 - uw, a);
      a = fma(fe, u0 - ue, a);
      a = fma(fn, u0 - un, a);
      a = fma(fs, u0 - us, a);
      return u0 + SP_OMEGA * (b - a) * d;
    };
    const double oA0 = post(uA0, bA.x, dA.x, wA, uA1, uM0, uB0, W.wxA0, W.wxA1, W.wyA0, W.wyB0, W.kA0);
    const double oA1 = post(uA1, bA.y, dA.y, uA0, eA, uM1, uB1, W.wxA1, W.wxA2, W.wyA1, W.wyB1, W.kA1);
    spf_st2<EVEN>(oq + G.rA, G.c0, G.v0, G.v1, oA0, oA1);
    double s = dot[e];
    if (level0) {
      if (G.v0) s = fma(oA0, bA.x, s);
      if (G.v1) s = fma(oA1, bA.y, s);
    }
    if (G.r1) {
      const double oB0 = post(uB0, bB.x, dB.x, wB, uB1, uA0, uP0, W.wxB0, W.wxB1, W.wyB0, W.wyP0, W.kB0);
      const double oB1 = post(uB1, bB.y, dB.y, uB0, eB, uA1, uP1, W.wxB1, W.wxB2, W.wyB1, W.wyP1, W.kB1);
      spf_st2<EVEN>(oq + G.rB, G.c0, G.v0, G.v1, oB0, oB1);
      if (level0) {
        if (G.v0) s = fma(oB0, bB.x, s);
        if (G.v1) s = fma(oB1, bB.y, s);
      }
    }
    dot[e] = s;
  }
  }
  if (level0) spf_reduce_pair(S, R, dot[0], dot[1], pa, pb);
}

// ---- K1 of the inner solvers (k_sp_apply2) in the same organisation ------------------------
// CTA = (row-pair tile, plane pair): pair 0 = the two real blocks (planes 0 and ell - 1: Q = (A -
// Lambda) P and <P, Q> each), pair k = complex block k (S z / gamma of Eq. (eq:saddlesystem) and
// <S z, z> / gamma^2) -- equal work per CTA. Thread = fine columns (c0, c0 + 1) x rows (2Y, 2Y + 1),
// every load issued first; grid-stride over row pairs (one dot partial per CTA and block).
__device__ __forceinline__ void spf_reduce_apply(const SpStepCtx& S, const SpfRed& R, double va, double vb,
                                                 int pair) {
  __shared__ double red[2][SPF_T / 32];
  __shared__ double tot[AAC_MAX_ELL];
  va = warp_sum(va);
  vb = warp_sum(vb);
  const int t = threadIdx.x, ntile = gridDim.x, np = gridDim.y;
  if ((t & 31) == 0) {
    red[0][t >> 5] = va;
    red[1][t >> 5] = vb;
  }
  __syncthreads();
  if (t == 0) {
    double sa = 0.0, sb = 0.0;
    for (int w = 0; w < SPF_T / 32; ++w) {
      sa += red[0][w];
      sb += red[1][w];
    }
    S.part[(long long)pair * ntile + blockIdx.x] = sa;
    S.part[(long long)(np + pair) * ntile + blockIdx.x] = sb;
    __threadfence();
  }
  // tot[q] = pair q's first sums (block q), tot[np] = pair 0's second (block h = np)
  if (!spf_reduce2(S.part, R, np + 1, tot)) return;
  if (t == 0) {
    const int h = S.K.ell / 2;
    if (S.red) {
      for (int q = 0; q <= h; ++q) S.red[q] = tot[q];
    } else {
      sp_scalar_A(S, tot);
    }
  }
}

template <bool EVEN>
__global__ void __launch_bounds__(SPF_T, SPF_MINB) k_spf_apply(Geo g, SpVec v, SpStepCtx S, SpfRed R, int nsx) {
  griddep();
  if (S.st && S.st->done) return;
  const int pair = blockIdx.y, ell = S.K.ell, h = ell / 2;
  const long long N = g.N;
  const int nx = g.nx;
  const bool real = pair == 0;
  // plane e of the pair and its block
  const int q[2] = {real ? 0 : 2 * pair - 1, real ? ell - 1 : 2 * pair};
  const int kbs[2] = {real ? 0 : pair, real ? h : pair};
  const bool stop0 = S.blk[kbs[0]].stop != 0, stop1 = S.blk[kbs[1]].stop != 0;
  const double invg = real || stop0 ? 0.0 : 1.0 / S.blk[pair].gamma;
  const double* u0p = (real ? v.P : v.Zc) + (long long)q[0] * N;
  const double* u1p = (real ? v.P : v.Zc) + (long long)q[1] * N;
  const double ms[2] = {1.0 + S.K.s[q[0]], 1.0 + S.K.s[q[1]]};
  const double lr = S.K.lre[pair], li = S.K.lim[pair];
  double* sz0 = v.SZ + (long long)q[0] * N;
  double* sz1 = v.SZ + (long long)q[1] * N;
  double dot0 = 0.0, dot1 = 0.0;
  const int nry = gridDim.x / nsx, nyp = (g.ny + 1) / 2;
  const bool idle = real ? (stop0 && stop1) : stop0;
  for (int Y = blockIdx.x / nsx; Y < nyp && !idle; Y += nry) {
    const SpfGeom G = spf_geom(g, nsx, Y);
    // u of rows M, A, B, P and of the warp-edge column of rows A, B, for one plane
    auto rows = [&](const double* u, double2& a, double2& b, double2& mm, double2& pp, double& ea, double& eb) {
      a = spf_l2<EVEN>(u + G.rA, G, nx);
      b = spf_l2<EVEN>(u + G.rB, G, nx);
      mm = spf_l2<EVEN>(u + G.rM, G, nx);
      pp = spf_l2<EVEN>(u + G.rP, G, nx);
      ea = __ldg(u + G.rA + G.ce);
      eb = __ldg(u + G.rB + G.ce);
    };
    double2 a0, b0, m0, p0, a1, b1, m1, p1;
    double ea0, eb0, ea1, eb1;
    rows(u0p, a0, b0, m0, p0, ea0, eb0);
    rows(u1p, a1, b1, m1, p1, ea1, eb1);
    // the weights after the planes' loads: their shuffles wait for the weight loads only
    SpfWRaw WR;
    spf_wload<EVEN, false>(g, nullptr, G, WR);
    SpfW W;
    spf_wfin(g, G, WR, W);
    // (A u) at the four points of one plane in apply_Av's order: c + sum_f w_f (c - nb_f)
    auto av4 = [&](const double2& A, const double2& B, const double2& M, const double2& P, double ea, double eb,
                   double out[4]) {
      double wA, eA, wB, eB;
      spf_xnb(A.x, A.y, ea, G.lane, wA, eA);
      spf_xnb(B.x, B.y, eb, G.lane, wB, eB);
      auto one = [&](double c, double xw, double xe, double xn, double xs, double fw, double fe, double fn, double fs) {
        double acc = c;
        acc = fma(fw, c - xw, acc);
        acc = fma(fe, c - xe, acc);
        acc = fma(fn, c - xn, acc);
        acc = fma(fs, c - xs, acc);
        return acc;
      };
      const double mA0 = G.rm ? M.x : A.x, mA1 = G.rm ? M.y : A.y;
      const double pB0 = G.rp ? P.x : B.x, pB1 = G.rp ? P.y : B.y;
      out[0] = one(A.x, wA, A.y, mA0, B.x, W.wxA0, W.wxA1, W.wyA0, W.wyB0);
      out[1] = one(A.y, A.x, eA, mA1, B.y, W.wxA1, W.wxA2, W.wyA1, W.wyB1);
      out[2] = one(B.x, wB, B.y, A.x, pB0, W.wxB0, W.wxB1, W.wyB0, W.wyP0);
      out[3] = one(B.y, B.x, eB, A.y, pB1, W.wxB1, W.wxB2, W.wyB1, W.wyP1);
    };
    const double c0v[4] = {a0.x, a0.y, b0.x, b0.y};
    const double c1v[4] = {a1.x, a1.y, b1.x, b1.y};
    const bool ok[4] = {G.v0, G.v1, G.v0 && G.r1, G.v1 && G.r1};
    double A0[4], A1[4], o0[4], o1[4];
    av4(a0, b0, m0, p0, ea0, eb0, A0);
    av4(a1, b1, m1, p1, ea1, eb1, A1);
    if (real) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        o0[i] = A0[i] + (ms[0] - 1.0) * c0v[i];             // (A - Lambda) p, both real blocks
        o1[i] = A1[i] + (ms[1] - 1.0) * c1v[i];
        if (ok[i]) {
          dot0 = fma(c0v[i], o0[i], dot0);
          dot1 = fma(c1v[i], o1[i], dot1);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double us = c0v[i] * invg, vs = c1v[i] * invg;
        const double Au = A0[i] * invg, Av = A1[i] * invg;
        const double Su = li * us + (Av - lr * vs);
        const double Sv = (Au - lr * us) - li * vs;
        o0[i] = Su;
        o1[i] = Sv;
        if (ok[i]) dot0 = fma(Sv, vs, fma(Su, us, dot0));
      }
    }
    if (!stop0) {
      spf_st2<EVEN>(sz0 + G.rA, G.c0, G.v0, G.v1, o0[0], o0[1]);
      if (G.r1) spf_st2<EVEN>(sz0 + G.rB, G.c0, G.v0, G.v1, o0[2], o0[3]);
    }
    if (real ? !stop1 : !stop0) {
      spf_st2<EVEN>(sz1 + G.rA, G.c0, G.v0, G.v1, o1[0], o1[1]);
      if (G.r1) spf_st2<EVEN>(sz1 + G.rB, G.c0, G.v0, G.v1, o1[2], o1[3]);
    }
  }
  if (real) {
    if (stop0) dot0 = 0.0;
    if (stop1) dot1 = 0.0;
  }
  spf_reduce_apply(S, R, dot0, dot1, pair);
}

// ---- K1 with the rows staged by the bulk-copy engine (even nx) --------------------------------
// k_spf_apply keeps ~16 warps per SM (128 registers) and every operand of an aggregate row in
// registers: ncu shows it latency-bound (long-scoreboard stalls, 2.1 TB/s). Here a CTA owns a
// strip of 2 SPF_T fine columns (+2 halo columns each side) and a chunk of aggregate rows of one
// plane pair, and marches down the chunk: thread 0 streams each fine row (u of both planes, the
// x- and y-face weights) through a ring of SPT_D row slots with cp.async.bulk + one mbarrier per
// slot, so the bytes in flight are bounded by shared memory, not registers; the x-neighbours
// come from the staged row (no shuffles, no warp-edge loads) and every row is loaded once per
// chunk instead of twice. The arithmetic per point is k_spf_apply's, in its order (columns
// outside the level hold zero and carry zero face weights, rows outside it are selected away).
#ifndef SPT_MINB
#define SPT_MINB 3
#endif
#ifndef SPT_DSLOT
#define SPT_DSLOT 8
#endif
constexpr int SPT_D = SPT_DSLOT;               // row slots
constexpr int SPT_W = 2 * SPF_T + 4;           // staged columns: cb - 2 .. cb + 2 SPF_T + 1
constexpr int SPT_NA = 4;                      // arrays per row: u (plane a), u (plane b), wx, wy

__host__ __device__ constexpr size_t spt_smem() {
  return (size_t)SPT_D * SPT_NA * SPT_W * sizeof(double) + SPT_D * sizeof(uint64_t);
}

__global__ void __launch_bounds__(SPF_T, SPT_MINB) k_spf_apply_tma(Geo g, SpVec v, SpStepCtx S, SpfRed R, int nsx,
                                                                   int nyc) {
  // (programmatic dependent launch: wait for the predecessor here, but let the successor launch
  //  only at the end -- its early CTAs would otherwise compete with this smem-heavy grid: measured
  //  53.7 vs 48.8 ms per saddle solve)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (S.st && S.st->done) return;
  extern __shared__ __align__(16) double sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + SPT_D * SPT_NA * SPT_W);
  const int pair = blockIdx.y, ell = S.K.ell, h = ell / 2;
  const int nx = g.nx, ny = g.ny, t = threadIdx.x;
  const bool real = pair == 0;
  const int q[2] = {real ? 0 : 2 * pair - 1, real ? ell - 1 : 2 * pair};
  const int kbs[2] = {real ? 0 : pair, real ? h : pair};
  const bool stop0 = S.blk[kbs[0]].stop != 0, stop1 = S.blk[kbs[1]].stop != 0;
  const double invg = real || stop0 ? 0.0 : 1.0 / S.blk[pair].gamma;
  const double* u0p = (real ? v.P : v.Zc) + (long long)q[0] * g.N;
  const double* u1p = (real ? v.P : v.Zc) + (long long)q[1] * g.N;
  const double ms[2] = {1.0 + S.K.s[q[0]], 1.0 + S.K.s[q[1]]};
  const double lr = S.K.lre[pair], li = S.K.lim[pair];
  double* sz0 = v.SZ + (long long)q[0] * g.N;
  double* sz1 = v.SZ + (long long)q[1] * g.N;
  double dot0 = 0.0, dot1 = 0.0;
  const int strip = blockIdx.x % nsx, chunk = blockIdx.x / nsx;
  const int nyp = (ny + 1) / 2;
  const int Y0 = chunk * nyc, Y1 = min(Y0 + nyc, nyp);
  const bool idle = (real ? (stop0 && stop1) : stop0) || Y0 >= Y1;
  const int cs = strip * 2 * SPF_T - 2;          // fine column of staged column 0
  const int clo = max(cs, 0), chi = min(cs + SPT_W, nx);
  const uint32_t bytes = (uint32_t)(chi - clo) * 8u;
  const int off = clo - cs;
  // columns outside the level: zero in every slot (the bulk copies never write them)
  for (int k = t; k < SPT_D * SPT_NA * SPT_W; k += SPF_T) {
    const int c = cs + k % SPT_W;
    if (c < 0 || c >= nx) sm[k] = 0.0;
  }
  if (t == 0) {
    for (int s = 0; s < SPT_D; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int r0 = 2 * Y0 - 1, nrow = 2 * (Y1 - Y0) + 2;   // fine rows r0 .. r0 + nrow - 1
  auto issue = [&](int i) {                      // relative row i into slot i % SPT_D
    const int r = r0 + i, s = i % SPT_D;
    double* d = sm + (size_t)s * SPT_NA * SPT_W + off;
    if (r >= 0 && r < ny) {
      mbar_arrive_expect_tx(&bar[s], 4u * bytes);
      const long long ro = (long long)r * nx + clo;
      bulk_g2s(d, u0p + ro, bytes, &bar[s]);
      bulk_g2s(d + SPT_W, u1p + ro, bytes, &bar[s]);
      bulk_g2s(d + 2 * SPT_W, g.wx + ro, bytes, &bar[s]);
      bulk_g2s(d + 3 * SPT_W, g.wy + ro, bytes, &bar[s]);
    } else {
      mbar_arrive(&bar[s]);                      // (row outside the level: never read)
    }
  };
  if (!idle) {
    if (t == 0)
      for (int i = 0; i < min(SPT_D, nrow); ++i) issue(i);
    const int c0 = 2 * (strip * SPF_T + t);
    const bool v0 = c0 < nx, v1 = c0 + 1 < nx;
    const int j0 = c0 - cs;                      // staged column of c0
    for (int Y = Y0; Y < Y1; ++Y) {
      const int k = Y - Y0;
      for (int i = (k == 0 ? 0 : 2 * k + 2); i <= 2 * k + 3; ++i)
        mbar_wait(&bar[i % SPT_D], (uint32_t)((i / SPT_D) & 1));
      const int y0 = 2 * Y;
      const bool r1 = y0 + 1 < ny, rm = Y > 0, rp = y0 + 2 < ny;
      const double* sM = sm + (size_t)((2 * k) % SPT_D) * SPT_NA * SPT_W;
      const double* sA = sm + (size_t)((2 * k + 1) % SPT_D) * SPT_NA * SPT_W;
      const double* sB = r1 ? sm + (size_t)((2 * k + 2) % SPT_D) * SPT_NA * SPT_W : sA;
      const double* sP = sm + (size_t)((2 * k + 3) % SPT_D) * SPT_NA * SPT_W;
      // face weights (k_spf_apply's SpfW without the counts)
      const bool inB = v0 && r1;
      const double* wxA = sA + 2 * SPT_W + j0;
      const double* wyA = sA + 3 * SPT_W + j0;
      const double* wxB = sB + 2 * SPT_W + j0;
      const double* wyB = sB + 3 * SPT_W + j0;
      const double wxA0 = v0 ? wxA[0] : 0.0, wxA1 = v0 ? wxA[1] : 0.0;
      const double wxA2 = c0 + 2 < nx ? wxA[2] : 0.0;
      const double wyA0 = v0 ? wyA[0] : 0.0, wyA1 = v0 ? wyA[1] : 0.0;
      const double wxB0 = inB ? wxB[0] : 0.0, wxB1 = inB ? wxB[1] : 0.0;
      const double wxB2 = (c0 + 2 < nx && r1) ? wxB[2] : 0.0;
      const double wyB0 = inB ? wyB[0] : 0.0, wyB1 = inB ? wyB[1] : 0.0;
      const double wyP0 = (inB && rp) ? sP[3 * SPT_W + j0] : 0.0;
      const double wyP1 = (inB && rp) ? sP[3 * SPT_W + j0 + 1] : 0.0;
      auto one = [&](double c, double xw, double xe, double xn, double xs, double fw, double fe, double fn, double fs) {
        double acc = c;
        acc = fma(fw, c - xw, acc);
        acc = fma(fe, c - xe, acc);
        acc = fma(fn, c - xn, acc);
        acc = fma(fs, c - xs, acc);
        return acc;
      };
      double cv[2][4], Av[2][4];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double* a = sA + e * SPT_W + j0;
        const double* b = sB + e * SPT_W + j0;
        const double* m = (rm ? sM : sA) + e * SPT_W + j0;
        const double* pp = (rp ? sP : sB) + e * SPT_W + j0;
        const double a0 = a[0], a1 = a[1], b0 = b[0], b1 = b[1];
        cv[e][0] = a0; cv[e][1] = a1; cv[e][2] = b0; cv[e][3] = b1;
        Av[e][0] = one(a0, a[-1], a1, m[0], b0, wxA0, wxA1, wyA0, wyB0);
        Av[e][1] = one(a1, a0, a[2], m[1], b1, wxA1, wxA2, wyA1, wyB1);
        Av[e][2] = one(b0, b[-1], b1, a0, pp[0], wxB0, wxB1, wyB0, wyP0);
        Av[e][3] = one(b1, b0, b[2], a1, pp[1], wxB1, wxB2, wyB1, wyP1);
      }
      const bool ok[4] = {v0, v1, v0 && r1, v1 && r1};
      double o0[4], o1[4];
      if (real) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          o0[i] = Av[0][i] + (ms[0] - 1.0) * cv[0][i];
          o1[i] = Av[1][i] + (ms[1] - 1.0) * cv[1][i];
          if (ok[i]) {
            dot0 = fma(cv[0][i], o0[i], dot0);
            dot1 = fma(cv[1][i], o1[i], dot1);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double us = cv[0][i] * invg, vs = cv[1][i] * invg;
          const double Au = Av[0][i] * invg, Avv = Av[1][i] * invg;
          const double Su = li * us + (Avv - lr * vs);
          const double Sv = (Au - lr * us) - li * vs;
          o0[i] = Su;
          o1[i] = Sv;
          if (ok[i]) dot0 = fma(Sv, vs, fma(Su, us, dot0));
        }
      }
      const long long rA = (long long)y0 * nx, rB = rA + nx;
      if (!stop0) {
        spf_st2<true>(sz0 + rA, c0, v0, v1, o0[0], o0[1]);
        if (r1) spf_st2<true>(sz0 + rB, c0, v0, v1, o0[2], o0[3]);
      }
      if (real ? !stop1 : !stop0) {
        spf_st2<true>(sz1 + rA, c0, v0, v1, o1[0], o1[1]);
        if (r1) spf_st2<true>(sz1 + rB, c0, v0, v1, o1[2], o1[3]);
      }
      __syncthreads();                           // rows 2k, 2k + 1 are free
      if (t == 0) {
        if (2 * k + SPT_D < nrow) issue(2 * k + SPT_D);
        if (2 * k + 1 + SPT_D < nrow) issue(2 * k + 1 + SPT_D);
      }
    }
  }
  if (real) {
    if (stop0) dot0 = 0.0;
    if (stop1) dot1 = 0.0;
  }
  spf_reduce_apply(S, R, dot0, dot1, pair);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- level-0 restriction with the rows staged by the bulk-copy engine (even nx) ---------------
// k_spf_restrict at level 0 (one aggregate row per CTA, every operand in registers) as a
// row-marching kernel in the organisation of k_spf_apply_tma: per fine row the b operands of
// both planes (or the update operands SZ, V_j, V_{j-1} of v_{j+1}), 1/D of their blocks and the
// weights wx, wy, cnt stream through an SPR_D-slot ring; the arithmetic per point is
// k_spf_restrict's, in its order.
constexpr int SPR_D = 4;                       // row slots
constexpr int SPR_NA = 11;                     // [plane 0: a0 a1 a2 d][plane 1: a0 a1 a2 d][wx wy cnt]

__host__ __device__ constexpr size_t spr_smem() {
  return (size_t)SPR_D * SPR_NA * SPT_W * sizeof(double) + SPR_D * sizeof(uint64_t);
}

__global__ void __launch_bounds__(SPF_T, 2) k_spf_restrict_tma(Geo g, Geo gc, const double* __restrict__ cnt,
                                                               const double* __restrict__ dinv, SpConst K, MgIo io,
                                                               double* bc, SpfUpd U, int nsx, int nyc,
                                                               const IterState* st) {
  asm volatile("griddepcontrol.wait;" ::: "memory");   // (dependents triggered at the end)
  if (st && st->done) return;
  extern __shared__ __align__(16) double sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + SPR_D * SPR_NA * SPT_W);
  int pa, pb;
  sp_pair(K.ell, blockIdx.y, pa, pb);
  const int pls[2] = {pa, pb};
  const int nx = g.nx, ny = g.ny, t = threadIdx.x;
  const long long N = g.N;
  bool upd[2];
  int kbs[2];
  const double* src[2][4];
  double dc[2], vcf[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int pl = pls[e];
    kbs[e] = sp_block_of(K.ell, pl);
    upd[e] = U.on && kbs[e] != 0 && kbs[e] != K.ell / 2 && U.blk[kbs[e]].stop != 1;
    const long long o = (long long)pl * N;
    src[e][0] = upd[e] ? U.SZ + o : io.in[pl];
    src[e][1] = upd[e] ? U.Vc + o : nullptr;
    src[e][2] = upd[e] ? U.Vp + o : nullptr;
    src[e][3] = dinv + (long long)kbs[e] * N;
    dc[e] = upd[e] ? U.blk[kbs[e]].dcoef : 0.0;
    vcf[e] = upd[e] ? U.blk[kbs[e]].vcoef : 0.0;
  }
  const bool dsame = kbs[0] == kbs[1];           // one 1/D row for both planes
  const int strip = blockIdx.x % nsx, chunk = blockIdx.x / nsx;
  const int nyp = (ny + 1) / 2;
  const int Y0 = chunk * nyc, Y1 = min(Y0 + nyc, nyp);
  const bool idle = Y0 >= Y1;
  const int cs = strip * 2 * SPF_T - 2;
  const int clo = max(cs, 0), chi = min(cs + SPT_W, nx);
  const uint32_t bytes = (uint32_t)(chi - clo) * 8u;
  const int off = clo - cs;
  for (int k = t; k < SPR_D * SPR_NA * SPT_W; k += SPF_T) {
    const int c = cs + k % SPT_W;
    if (c < 0 || c >= nx) sm[k] = 0.0;
  }
  if (t == 0) {
    for (int s = 0; s < SPR_D; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int r0 = 2 * Y0 - 1, nrow = 2 * (Y1 - Y0) + 2;
  int ncopy = 3;                                 // arrays per row: wx, wy, cnt + the planes'
#pragma unroll
  for (int e = 0; e < 2; ++e) ncopy += (upd[e] ? 3 : 1) + ((e == 1 && dsame) ? 0 : 1);
  auto issue = [&](int i) {
    const int r = r0 + i, s = i % SPR_D;
    double* d = sm + (size_t)s * SPR_NA * SPT_W + off;
    if (r >= 0 && r < ny) {
      mbar_arrive_expect_tx(&bar[s], (uint32_t)ncopy * bytes);
      const long long ro = (long long)r * nx + clo;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int na = upd[e] ? 3 : 1;
        for (int a = 0; a < na; ++a) bulk_g2s(d + (e * 4 + a) * SPT_W, src[e][a] + ro, bytes, &bar[s]);
        if (!(e == 1 && dsame)) bulk_g2s(d + (e * 4 + 3) * SPT_W, src[e][3] + ro, bytes, &bar[s]);
      }
      bulk_g2s(d + 8 * SPT_W, g.wx + ro, bytes, &bar[s]);
      bulk_g2s(d + 9 * SPT_W, g.wy + ro, bytes, &bar[s]);
      bulk_g2s(d + 10 * SPT_W, cnt + ro, bytes, &bar[s]);
    } else {
      mbar_arrive(&bar[s]);
    }
  };
  if (!idle) {
    if (t == 0)
      for (int i = 0; i < min(SPR_D, nrow); ++i) issue(i);
    const int X = strip * SPF_T + t, c0 = 2 * X;
    const bool v0 = c0 < nx, v1 = c0 + 1 < nx;
    const int j0 = c0 - cs;
    for (int Y = Y0; Y < Y1; ++Y) {
      const int k = Y - Y0;
      for (int i = (k == 0 ? 0 : 2 * k + 2); i <= 2 * k + 3; ++i)
        mbar_wait(&bar[i % SPR_D], (uint32_t)((i / SPR_D) & 1));
      const int y0 = 2 * Y;
      const bool r1 = y0 + 1 < ny, rm = Y > 0, rp = y0 + 2 < ny;
      const double* sA = sm + (size_t)((2 * k + 1) % SPR_D) * SPR_NA * SPT_W;
      const double* sB = r1 ? sm + (size_t)((2 * k + 2) % SPR_D) * SPR_NA * SPT_W : sA;
      const double* sM = rm ? sm + (size_t)((2 * k) % SPR_D) * SPR_NA * SPT_W : sA;
      const double* sP = rp ? sm + (size_t)((2 * k + 3) % SPR_D) * SPR_NA * SPT_W : sB;
      const double* sPw = sm + (size_t)((2 * k + 3) % SPR_D) * SPR_NA * SPT_W;
      const bool inB = v0 && r1;
      const double* wxA = sA + 8 * SPT_W + j0;
      const double* wyA = sA + 9 * SPT_W + j0;
      const double* wxB = sB + 8 * SPT_W + j0;
      const double* wyB = sB + 9 * SPT_W + j0;
      const double wxA0 = v0 ? wxA[0] : 0.0, wxA1 = v0 ? wxA[1] : 0.0;
      const double wxA2 = c0 + 2 < nx ? wxA[2] : 0.0;
      const double wyA0 = v0 ? wyA[0] : 0.0, wyA1 = v0 ? wyA[1] : 0.0;
      const double wxB0 = inB ? wxB[0] : 0.0, wxB1 = inB ? wxB[1] : 0.0;
      const double wxB2 = (c0 + 2 < nx && r1) ? wxB[2] : 0.0;
      const double wyB0 = inB ? wyB[0] : 0.0, wyB1 = inB ? wyB[1] : 0.0;
      const double wyP0 = (inB && rp) ? sPw[9 * SPT_W + j0] : 0.0;
      const double wyP1 = (inB && rp) ? sPw[9 * SPT_W + j0 + 1] : 0.0;
      const double kA0 = sA[10 * SPT_W + j0], kA1 = sA[10 * SPT_W + j0 + 1];
      const double kB0 = sB[10 * SPT_W + j0], kB1 = sB[10 * SPT_W + j0 + 1];
      double acc[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double m = 1.0 + K.s[pls[e]];
        const int dd = (e == 1 && dsame) ? 3 : e * 4 + 3;
        // b at staged column jj of a row (the update formed exactly as k_sp_upd1 does)
        auto bval = [&](const double* row, int jj) {
          const double a0 = row[(e * 4) * SPT_W + jj];
          if (!upd[e]) return a0;
          return a0 - dc[e] * row[(e * 4 + 1) * SPT_W + jj] - vcf[e] * row[(e * 4 + 2) * SPT_W + jj];
        };
        auto xval = [&](const double* row, int jj, double b) { return SP_OMEGA * b * row[dd * SPT_W + jj]; };
        const double bA0 = bval(sA, j0), bA1 = bval(sA, j0 + 1), bB0 = bval(sB, j0), bB1 = bval(sB, j0 + 1);
        const double bM0 = bval(sM, j0), bM1 = bval(sM, j0 + 1), bP0 = bval(sP, j0), bP1 = bval(sP, j0 + 1);
        if (upd[e]) {                            // v_{j+1} of the own points
          double* vn = const_cast<double*>(io.in[pls[e]]);
          spf_st2<true>(vn + (long long)y0 * nx, c0, v0, v1, bA0, bA1);
          if (r1) spf_st2<true>(vn + (long long)(y0 + 1) * nx, c0, v0, v1, bB0, bB1);
        }
        const double xA0 = xval(sA, j0, bA0), xA1 = xval(sA, j0 + 1, bA1);
        const double xB0 = xval(sB, j0, bB0), xB1 = xval(sB, j0 + 1, bB1);
        const double xM0 = xval(sM, j0, bM0), xM1 = xval(sM, j0 + 1, bM1);
        const double xP0 = xval(sP, j0, bP0), xP1 = xval(sP, j0 + 1, bP1);
        const double wA = xval(sA, j0 - 1, bval(sA, j0 - 1)), eA = xval(sA, j0 + 2, bval(sA, j0 + 2));
        const double wB = xval(sB, j0 - 1, bval(sB, j0 - 1)), eB = xval(sB, j0 + 2, bval(sB, j0 + 2));
        auto res = [&](double c, double b, double xw, double xe, double xn, double xs, double fw, double fe, double fn,
                       double fs, double kk) {
          double a = c;
          a = fma(fw, c - xw, a);
          a = fma(fe, c - xe, a);
          a = fma(fn, c - xn, a);
          a = fma(fs, c - xs, a);
          a = a + (m * kk - 1.0) * c;
          return b - a;
        };
        double s = 0.0;
        if (v0) s += res(xA0, bA0, wA, xA1, xM0, xB0, wxA0, wxA1, wyA0, wyB0, kA0);
        if (v1) s += res(xA1, bA1, xA0, eA, xM1, xB1, wxA1, wxA2, wyA1, wyB1, kA1);
        if (r1) {
          if (v0) s += res(xB0, bB0, wB, xB1, xA0, xP0, wxB0, wxB1, wyB0, wyP0, kB0);
          if (v1) s += res(xB1, bB1, xB0, eB, xA1, xP1, wxB1, wxB2, wyB1, wyP1, kB1);
        }
        acc[e] = s;
      }
      if (X < gc.nx) {
        const long long oc = (long long)Y * gc.nx + X;
        bc[(long long)pa * gc.N + oc] = acc[0];
        bc[(long long)pb * gc.N + oc] = acc[1];
      }
      __syncthreads();
      if (t == 0) {
        if (2 * k + SPR_D < nrow) issue(2 * k + SPR_D);
        if (2 * k + 1 + SPR_D < nrow) issue(2 * k + 1 + SPR_D);
      }
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- level-0 prolongation + post-smoothing with the rows staged by the bulk-copy engine -------
// k_spf_prolong_post at level 0 (nx % 4 == 0: the coarse rows are 16-byte aligned too) as a
// row-marching kernel: per fine row b and 1/D of both planes, wx, wy, cnt, and the coarse row
// (r / 2) of x_c of both planes stream through an SPP_D-slot ring. Arithmetic per point as
// k_spf_prolong_post.
constexpr int SPP_D = 6;
constexpr int SPC_W = SPF_T + 4;               // staged coarse columns: X0 - 2 .. X0 + SPF_T + 1
constexpr int SPP_SLOT = 7 * SPT_W + 2 * SPC_W; // [b0 d0 b1 d1 wx wy cnt][xc0 xc1]

__host__ __device__ constexpr size_t spp_smem() {
  return (size_t)SPP_D * SPP_SLOT * sizeof(double) + SPP_D * sizeof(uint64_t);
}

__global__ void __launch_bounds__(SPF_T, 2) k_spf_prolong_tma(Geo g, Geo gc, const double* __restrict__ cnt,
                                                              const double* __restrict__ dinv, MgIo io,
                                                              const double* __restrict__ xc, SpStepCtx S, SpfRed R,
                                                              int nsx, int nyc) {
  asm volatile("griddepcontrol.wait;" ::: "memory");   // (dependents triggered at the end)
  if (S.st && S.st->done) return;
  extern __shared__ __align__(16) double sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + SPP_D * SPP_SLOT);
  int pa, pb;
  sp_pair(S.K.ell, blockIdx.y, pa, pb);
  const int pls[2] = {pa, pb};
  const int nx = g.nx, ny = g.ny, t = threadIdx.x;
  const long long N = g.N;
  const double* bsrc[2] = {io.in[pa], io.in[pb]};
  const double* dsrc[2] = {dinv + (long long)sp_block_of(S.K.ell, pa) * N, dinv + (long long)sp_block_of(S.K.ell, pb) * N};
  const double* csrc[2] = {xc + (long long)pa * gc.N, xc + (long long)pb * gc.N};
  const bool dsame = dsrc[0] == dsrc[1];
  const int strip = blockIdx.x % nsx, chunk = blockIdx.x / nsx;
  const int nyp = (ny + 1) / 2;
  const int Y0 = chunk * nyc, Y1 = min(Y0 + nyc, nyp);
  const bool idle = Y0 >= Y1;
  const int cs = strip * 2 * SPF_T - 2;
  const int clo = max(cs, 0), chi = min(cs + SPT_W, nx);
  const uint32_t bytes = (uint32_t)(chi - clo) * 8u;
  const int off = clo - cs;
  const int xs = strip * SPF_T - 2;              // coarse column of staged coarse column 0
  const int xlo = max(xs, 0), xhi = min(xs + SPC_W, gc.nx);
  const uint32_t cbytes = (uint32_t)(xhi - xlo) * 8u;
  const int coff = xlo - xs;
  for (int k = t; k < SPP_D * SPP_SLOT; k += SPF_T) {
    const int q = k % SPP_SLOT;
    bool out;
    if (q < 7 * SPT_W) {
      const int c = cs + q % SPT_W;
      out = c < 0 || c >= nx;
    } else {
      const int c = xs + (q - 7 * SPT_W) % SPC_W;
      out = c < 0 || c >= gc.nx;
    }
    if (out) sm[k] = 0.0;
  }
  if (t == 0) {
    for (int s = 0; s < SPP_D; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int r0 = 2 * Y0 - 1, nrow = 2 * (Y1 - Y0) + 2;
  const uint32_t tx = (uint32_t)(dsame ? 6 : 7) * bytes + 2u * cbytes;
  auto issue = [&](int i) {
    const int r = r0 + i, s = i % SPP_D;
    double* d = sm + (size_t)s * SPP_SLOT;
    if (r >= 0 && r < ny) {
      mbar_arrive_expect_tx(&bar[s], tx);
      const long long ro = (long long)r * nx + clo;
      bulk_g2s(d + off, bsrc[0] + ro, bytes, &bar[s]);
      bulk_g2s(d + SPT_W + off, dsrc[0] + ro, bytes, &bar[s]);
      bulk_g2s(d + 2 * SPT_W + off, bsrc[1] + ro, bytes, &bar[s]);
      if (!dsame) bulk_g2s(d + 3 * SPT_W + off, dsrc[1] + ro, bytes, &bar[s]);
      bulk_g2s(d + 4 * SPT_W + off, g.wx + ro, bytes, &bar[s]);
      bulk_g2s(d + 5 * SPT_W + off, g.wy + ro, bytes, &bar[s]);
      bulk_g2s(d + 6 * SPT_W + off, cnt + ro, bytes, &bar[s]);
      const long long co = (long long)(r >> 1) * gc.nx + xlo;
      bulk_g2s(d + 7 * SPT_W + coff, csrc[0] + co, cbytes, &bar[s]);
      bulk_g2s(d + 7 * SPT_W + SPC_W + coff, csrc[1] + co, cbytes, &bar[s]);
    } else {
      mbar_arrive(&bar[s]);
    }
  };
  double dot[2] = {0.0, 0.0};
  if (!idle) {
    if (t == 0)
      for (int i = 0; i < min(SPP_D, nrow); ++i) issue(i);
    const int X = strip * SPF_T + t, c0 = 2 * X;
    const bool v0 = c0 < nx, v1 = c0 + 1 < nx;
    const int j0 = c0 - cs, jc = X - xs;         // staged fine / coarse column of this thread
    for (int Y = Y0; Y < Y1; ++Y) {
      const int k = Y - Y0;
      for (int i = (k == 0 ? 0 : 2 * k + 2); i <= 2 * k + 3; ++i)
        mbar_wait(&bar[i % SPP_D], (uint32_t)((i / SPP_D) & 1));
      const int y0 = 2 * Y;
      const bool r1 = y0 + 1 < ny, rm = Y > 0, rp = y0 + 2 < ny;
      const double* sA = sm + (size_t)((2 * k + 1) % SPP_D) * SPP_SLOT;
      const double* sB = r1 ? sm + (size_t)((2 * k + 2) % SPP_D) * SPP_SLOT : sA;
      const double* sM = sm + (size_t)((2 * k) % SPP_D) * SPP_SLOT;
      const double* sP = sm + (size_t)((2 * k + 3) % SPP_D) * SPP_SLOT;
      const bool inB = v0 && r1;
      const double* wxA = sA + 4 * SPT_W + j0;
      const double* wyA = sA + 5 * SPT_W + j0;
      const double* wxB = sB + 4 * SPT_W + j0;
      const double* wyB = sB + 5 * SPT_W + j0;
      const double wxA0 = v0 ? wxA[0] : 0.0, wxA1 = v0 ? wxA[1] : 0.0;
      const double wxA2 = c0 + 2 < nx ? wxA[2] : 0.0;
      const double wyA0 = v0 ? wyA[0] : 0.0, wyA1 = v0 ? wyA[1] : 0.0;
      const double wxB0 = inB ? wxB[0] : 0.0, wxB1 = inB ? wxB[1] : 0.0;
      const double wxB2 = (c0 + 2 < nx && r1) ? wxB[2] : 0.0;
      const double wyB0 = inB ? wyB[0] : 0.0, wyB1 = inB ? wyB[1] : 0.0;
      const double wyP0 = (inB && rp) ? sP[5 * SPT_W + j0] : 0.0;
      const double wyP1 = (inB && rp) ? sP[5 * SPT_W + j0 + 1] : 0.0;
      const double kA0 = sA[6 * SPT_W + j0], kA1 = sA[6 * SPT_W + j0 + 1];
      const double kB0 = sB[6 * SPT_W + j0], kB1 = sB[6 * SPT_W + j0 + 1];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double m1 = 1.0 + S.K.s[pls[e]];
        const int ob = 2 * e * SPT_W, od = (e == 1 && dsame) ? SPT_W : (2 * e + 1) * SPT_W;
        const int oc = 7 * SPT_W + e * SPC_W;
        // u = omega b / D + P x_c at staged fine column jj of a row (coarse column jj_c)
        auto uval = [&](const double* row, int jj, int jjc) {
          return SP_OMEGA * row[ob + jj] * row[od + jj] + row[oc + jjc];
        };
        const double uA0 = uval(sA, j0, jc), uA1 = uval(sA, j0 + 1, jc);
        const double uB0 = uval(sB, j0, jc), uB1 = uval(sB, j0 + 1, jc);
        const double uM0 = rm ? uval(sM, j0, jc) : uA0, uM1 = rm ? uval(sM, j0 + 1, jc) : uA1;
        const double uP0 = rp ? uval(sP, j0, jc) : uB0, uP1 = rp ? uval(sP, j0 + 1, jc) : uB1;
        const double wA = uval(sA, j0 - 1, jc - 1), eA = uval(sA, j0 + 2, jc + 1);
        const double wB = uval(sB, j0 - 1, jc - 1), eB = uval(sB, j0 + 2, jc + 1);
        auto post = [&](double u0, double b, double d, double uw, double ue, double un, double us, double fw, double fe,
                        double fn, double fs, double kk) {
          double a = (m1 * kk) * u0;
          a = fma(fw, u0 - uw, a);
          a = fma(fe, u0 - ue, a);
          a = fma(fn, u0 - un, a);
          a = fma(fs, u0 - us, a);
          return u0 + SP_OMEGA * (b - a) * d;
        };
        const double bA0 = sA[ob + j0], bA1 = sA[ob + j0 + 1], bB0 = sB[ob + j0], bB1 = sB[ob + j0 + 1];
        const double oA0 = post(uA0, bA0, sA[od + j0], wA, uA1, uM0, uB0, wxA0, wxA1, wyA0, wyB0, kA0);
        const double oA1 = post(uA1, bA1, sA[od + j0 + 1], uA0, eA, uM1, uB1, wxA1, wxA2, wyA1, wyB1, kA1);
        double* oq = io.out[pls[e]];
        spf_st2<true>(oq + (long long)y0 * nx, c0, v0, v1, oA0, oA1);
        double s = dot[e];
        if (v0) s = fma(oA0, bA0, s);
        if (v1) s = fma(oA1, bA1, s);
        if (r1) {
          const double oB0 = post(uB0, bB0, sB[od + j0], wB, uB1, uA0, uP0, wxB0, wxB1, wyB0, wyP0, kB0);
          const double oB1 = post(uB1, bB1, sB[od + j0 + 1], uB0, eB, uA1, uP1, wxB1, wxB2, wyB1, wyP1, kB1);
          spf_st2<true>(oq + (long long)(y0 + 1) * nx, c0, v0, v1, oB0, oB1);
          if (v0) s = fma(oB0, bB0, s);
          if (v1) s = fma(oB1, bB1, s);
        }
        dot[e] = s;
      }
      __syncthreads();
      if (t == 0) {
        if (2 * k + SPP_D < nrow) issue(2 * k + SPP_D);
        if (2 * k + 1 + SPP_D < nrow) issue(2 * k + 1 + SPP_D);
      }
    }
  }
  spf_reduce_pair(S, R, dot[0], dot[1], pa, pb);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Tiles of the fused kernels on a level of `ncx` x `ncy` aggregates: strips of SPF_T aggregate
// columns x one aggregate row.
static inline void spf_tiles(int ncx, int ncy, int& nsx, int& ntile) {
  nsx = (ncx + SPF_T - 1) / SPF_T;
  ntile = nsx * ncy;
}
