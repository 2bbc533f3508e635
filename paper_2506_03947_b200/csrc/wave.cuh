// wave.cuh -- temporally blocked Chebyshev solves for 2D grids: a y-wavefront over all steps.
//
// The block problems (A - Lambda_k) y_k = w_k (PAPER.md:266-275 Eq. eq:blockproblem) are
// independent after the forward transform, and the Chebyshev recurrence of reading R8
//   x_0 = 0, x_1 = w/theta, x_{s+1} = x_s + a_s (x_s - x_{s-1}) + b_s (w - (A - Lambda) x_s)
// only couples a point to its 5-point neighbourhood from one step to the next. So the whole
// solve of one block (p_k - 1 stencil steps) can run in ONE pass over HBM: read w, write
// x_{p_k}, instead of 4 plane-passes per step (k_sweep).
//
// Organisation (one CTA = one packed block x one strip of columns x one chunk of rows):
//  * thread t owns column x = x0 - H + t of the strip (NT columns = TX interior + 2H halo);
//  * the CTA marches down the rows: at step tau it loads row tau of w (level L_1 = x_{s0}
//    enters at row tau) and computes level L_{i+1} at row tau - i for i = 1..ns (a skewed
//    wavefront: L_{i+1}(r) needs L_i at rows r-1, r, r+1 and L_{i-1}(r), all computed by the
//    same thread in this or an earlier step);
//  * the y-neighbours live in per-thread register rings (3 rows per level), the x-neighbours
//    come from the two adjacent threads through a double-buffered shared-memory exchange of
//    the previous step's rows (one __syncthreads per row);
//  * w rows are kept in a per-thread shared-memory history (H+1 rows), face weights are
//    read from L1/L2.
// Halo columns (H per side) and the warm-up rows of a chunk are computed redundantly and
// discarded; values outside the domain are zero and carry zero face weights (Neumann), so
// they never reach an in-domain point. Passes of up to H steps chain through ping-pong
// iterate buffers when p_k - 1 > H.
#pragma once

#include "nc.cuh"

constexpr int WAVE_MAXH = 8;

struct WBlk {
  int q, np, ns;             // first plane, planes (1 real | 2 complex), steps this pass (1..H)
  int virt;                  // 1: first pass, x_0 = 0 and x_1 = w/theta (sr, si) from w itself
  const double* ps;          // x_{s0}   plane q (virt == 0), scaled by (sr, si)
  const double* pm;          // x_{s0-1} plane q (virt == 0), scaled by (mr, mi)
  double sr, si, mr, mi;
  double* out_last;          // x_{s0+ns}   plane q
  double* out_prev;          // x_{s0+ns-1} plane q, or NULL (final pass)
  double* glo;               // slab ghost rows (k_waver, single pass): x_{p_k} of local row -1 / ny,
  double* ghi;               // plane q of [ell][nx] buffers (plane stride nx); NULL: none
  double lr, li;             // Lambda_k
  double ar[WAVE_MAXH], ai[WAVE_MAXH], br[WAVE_MAXH], bi[WAVE_MAXH];   // steps s0 .. s0+ns-1
};
// Slab decomposition (several ranks): rows outside this rank's slab come from halo buffers
// (the neighbours' last / first hd rows of hat w, exchanged once per preconditioner apply) and
// the face weights from arrays extended by hd rows on each side (built at setup from the global
// kappa). One rank: no halo rows, the extended arrays are the slab's own.
struct WSlab {
  const double* wxe;         // extended lower x-faces, row e = local row + eoff
  const double* wye;         // extended lower y-faces (row ne = the top face of the range)
  int eoff, ne;              // local row r lies in the global domain iff 0 <= r + eoff < ne
  const double* whlo;        // [ell][hd][nx] rows -hd .. -1 of hat w (NULL: none)
  const double* whhi;        // [ell][hd][nx] rows ny .. ny+hd-1
  int hd;
  int lo, nyg;               // global row of local row 0, global rows (Dirichlet faces)
};

struct WSweep {
  WBlk b[AAC_MAX_BLK];
  int nb;                    // blocks in this launch
  int nstrip;                // strips of TX columns
  int ly[AAC_MAX_BLK];       // rows per chunk of each block (equal work per CTA: a block with
                             // fewer steps or a real plane gets taller chunks)
  int cta0[AAC_MAX_BLK + 1]; // first CTA of each block (prefix sums of nstrip x chunks)
};

template <int H, int NT>
struct WGeom {
  static constexpr int TX = NT - 2 * H;                 // interior columns per strip
  static constexpr int NSLOT = H + 2;                   // ages 0 .. H, +1: thread t+1 may run a step ahead
  static constexpr int HW = NT + 1;                     // history row: one pad column
  static constexpr int XW = NT + 2;                     // exchange row: zero pad at both ends
  static constexpr int XCH = 2 * H * 2 * XW;            // [2 buffers][H levels][2 planes][XW]
  static constexpr int HIST = NSLOT * 4 * HW;           // [slot][w_re, w_im, wxl, wyl][HW]
  static constexpr size_t SMEM = (size_t)(XCH + HIST) * sizeof(double);
};

// Per-thread register rings: 3 rows per level (age 0 = newest), shifted by moves. (Renaming
// the slots by unrolling the row loop 3 times saves the moves but triples the loop body, and
// the instruction cache (L1.5 ~32 KB) then misses when CTAs of different blocks share an SM.)
template <int H>
struct WState {
  double L[H + 1][3][2];           // L[0] = x_{s0-1}, L[i] = L_i (i = 1..ns): [age][plane]
  double co[H][4];                 // step coefficients a_r, b_r, a_i, b_i held in registers
};

template <int H, int NT>
struct WCtx {                      // per-CTA constants
  const WBlk* B;
  const double* what;
  Geo g;
  WSlab sl;
  double* xch;
  double* hist;                    // this thread's column of the history (x+1: next thread)
  int t, x, y0, y1;
  bool colin, colout;
};

struct WRow { double w0, w1, s0, s1, m0, m1, fxl, fyl; };

template <int H, int NT, bool CPLX, bool GEN>
__device__ __forceinline__ void wave_load_row(const WCtx<H, NT>& C, int r, WRow& R) {
  R.w0 = R.w1 = R.s0 = R.s1 = R.m0 = R.m1 = R.fxl = R.fyl = 0.0;
  const Geo& g = C.g;
  if constexpr (!GEN) {                                  // one rank, Neumann: the slab itself
    if (C.colin && r >= 0 && r < g.ny) {
      const long long p = (long long)r * g.nx + C.x;
      const double* wq = C.what + (long long)C.B->q * g.N + p;
      R.w0 = __ldg(wq);
      if (CPLX) R.w1 = __ldg(wq + g.N);
      R.fxl = __ldg(g.wx + p);
      R.fyl = __ldg(g.wy + p);
      if (!C.B->virt) {
        R.s0 = C.B->ps[p];
        R.m0 = C.B->pm[p];
        if (CPLX) {
          R.s1 = C.B->ps[g.N + p];
          R.m1 = C.B->pm[g.N + p];
        }
      }
    } else if (C.colin && r == g.ny) {
      R.fyl = __ldg(g.wy + (long long)r * g.nx + C.x);
    }
    return;
  }
  const int er = r + C.sl.eoff;                          // row of the extended weight arrays
  if (C.colin && er >= 0 && er < C.sl.ne) {
    const long long p = (long long)r * g.nx + C.x;
    const long long pe = (long long)er * g.nx + C.x;
    const double* wq;                                    // hat w: own slab or a halo row
    long long ws;
    if (r < 0) {
      ws = (long long)C.sl.hd * g.nx;
      wq = C.sl.whlo + (long long)C.B->q * ws + (long long)(r + C.sl.hd) * g.nx + C.x;
    } else if (r >= g.ny) {
      ws = (long long)C.sl.hd * g.nx;
      wq = C.sl.whhi + (long long)C.B->q * ws + (long long)(r - g.ny) * g.nx + C.x;
    } else {
      ws = g.N;
      wq = C.what + (long long)C.B->q * g.N + p;
    }
    R.w0 = __ldg(wq);
    if (CPLX) R.w1 = __ldg(wq + ws);
    R.fxl = __ldg(C.sl.wxe + pe);
    R.fyl = __ldg(C.sl.wye + pe);
    if (!C.B->virt) {                                    // (later passes: one rank only)
      R.s0 = C.B->ps[p];
      R.m0 = C.B->pm[p];
      if (CPLX) {
        R.s1 = C.B->ps[g.N + p];
        R.m1 = C.B->pm[g.N + p];
      }
    }
  } else if (C.colin && er == C.sl.ne) {
    R.fyl = __ldg(C.sl.wye + (long long)er * g.nx + C.x);   // upper face of the last row
  }
}

template <int H, int NT, int ns, bool CPLX, bool GEN>
__device__ __forceinline__ void wave_step(const WCtx<H, NT>& C, WState<H>& S, int tau, int slot,
                                          WRow& nxt, int tau1) {
  using G = WGeom<H, NT>;
  const WBlk& B = *C.B;
  const int t = C.t;
  double* xb = C.xch + (tau & 1) * (H * 2 * G::XW) + 1 + t;
  // (1) publish the newest row of every level (L_i at row tau - i) for the x-neighbours
#pragma unroll
  for (int i = 1; i <= H; ++i) {
    if (i > ns) break;
    xb[((i - 1) * 2 + 0) * G::XW] = S.L[i][0][0];
    if (CPLX) xb[((i - 1) * 2 + 1) * G::XW] = S.L[i][0][1];
  }
  // (2) row tau enters: history, L_0, L_1; prefetch row tau + 1
  const WRow cur = nxt;
  if (tau + 1 < tau1) wave_load_row<H, NT, CPLX, GEN>(C, tau + 1, nxt);
  {
    double* hs = C.hist + slot * (4 * G::HW);
    hs[0] = cur.w0;
    if (CPLX) hs[G::HW] = cur.w1;
    hs[2 * G::HW] = cur.fxl;
    hs[3 * G::HW] = cur.fyl;
  }
#pragma unroll
  for (int e = 0; e < (CPLX ? 2 : 1); ++e) {
    S.L[0][1][e] = S.L[0][0][e];
    S.L[1][2][e] = S.L[1][1][e];
    S.L[1][1][e] = S.L[1][0][e];
  }
  if (B.virt) {
    S.L[0][0][0] = 0.0;
    S.L[1][0][0] = B.sr * cur.w0 - B.si * cur.w1;
    if (CPLX) {
      S.L[0][0][1] = 0.0;
      S.L[1][0][1] = B.sr * cur.w1 + B.si * cur.w0;
    }
  } else {
    S.L[1][0][0] = B.sr * cur.s0 - B.si * cur.s1;
    S.L[0][0][0] = B.mr * cur.m0 - B.mi * cur.m1;
    if (CPLX) {
      S.L[1][0][1] = B.sr * cur.s1 + B.si * cur.s0;
      S.L[0][0][1] = B.mr * cur.m1 + B.mi * cur.m0;
    }
  }
  __syncthreads();
  // (3) levels: L_{i+1} at row r = tau - i
  const double lr = B.lr, li = B.li;
  int su = slot;                                        // history slot of row r + 1
#pragma unroll
  for (int i = 1; i <= H; ++i) {
    if (i > ns) break;
    const int sl = su == 0 ? G::NSLOT - 1 : su - 1;     // history slot of row r
    const double* hr = C.hist + sl * (4 * G::HW);
    // upper x-face = lower x-face of the next column (stored by thread t+1 in an earlier step)
    const double fxl = hr[2 * G::HW], fxh = hr[2 * G::HW + 1], fyl = hr[3 * G::HW];
    const double fyh = C.hist[su * (4 * G::HW) + 3 * G::HW];
    const double w0 = hr[0];
    const double* xl = xb + ((i - 1) * 2) * G::XW;
    // everything except the y+1 neighbour (L_i at row r + 1, computed just before in this
    // step) is folded first; the serial chain through the levels is 4 operations deep:
    //   x_new = c + a (c - m) + b (w - (A - Lambda) c) = Q - b Ap,  Ap = fyh (c - dn) + Bp.
    const double c0 = S.L[i][1][0];
    double B0 = fma(fyl, c0 - S.L[i][2][0], fma(fxh, c0 - xl[1], fma(fxl, c0 - xl[-1], c0)));
    double dB = 0.0;                                    // Dirichlet boundary faces (paper mode)
    if (GEN && C.g.dir) {
      const int rg = tau - i + C.sl.lo;
      dB = C.g.bdx * ((C.x == 0) + (C.x == C.g.nx - 1)) + C.g.bdy * ((rg == 0) + (rg == C.sl.nyg - 1));
      B0 = fma(dB, c0, B0);
    }
    const double m0 = i == 1 ? S.L[0][1][0] : S.L[i - 1][2][0];
    const double ar = S.co[i - 1][0], br = S.co[i - 1][1];
    double o0, o1 = 0.0;
    if (CPLX) {
      const double w1 = hr[G::HW];
      const double c1 = S.L[i][1][1];
      const double B1 = fma(dB, c1, fma(fyl, c1 - S.L[i][2][1],
                                        fma(fxh, c1 - xl[G::XW + 1], fma(fxl, c1 - xl[G::XW - 1], c1))));
      const double m1 = i == 1 ? S.L[0][1][1] : S.L[i - 1][2][1];
      const double ai = S.co[i - 1][2], bi = S.co[i - 1][3];
      const double P0 = fma(-li, c1, fma(lr, c0, w0));      // w + Lambda c (r = P - Ap)
      const double P1 = fma(li, c0, fma(lr, c1, w1));
      const double dr = c0 - m0, di = c1 - m1;
      const double X0 = fma(-ai, di, fma(ar, dr, c0));
      const double X1 = fma(ai, dr, fma(ar, di, c1));
      const double Q0 = fma(-bi, P1, fma(br, P0, X0));
      const double Q1 = fma(bi, P0, fma(br, P1, X1));
      const double Ap0 = fma(fyh, c0 - S.L[i][0][0], B0);
      const double Ap1 = fma(fyh, c1 - S.L[i][0][1], B1);
      o0 = fma(bi, Ap1, fma(-br, Ap0, Q0));
      o1 = fma(-bi, Ap0, fma(-br, Ap1, Q1));
    } else {
      const double P0 = fma(lr, c0, w0);
      const double Q0 = fma(br, P0, fma(ar, c0 - m0, c0));
      const double Ap0 = fma(fyh, c0 - S.L[i][0][0], B0);
      o0 = fma(-br, Ap0, Q0);
    }
    if (i == ns) {
      const int r = tau - i;
      if (C.colout && r >= C.y0 && r < C.y1) {
        const long long p = (long long)r * C.g.nx + C.x;
        B.out_last[p] = o0;
        if (CPLX) B.out_last[C.g.N + p] = o1;
        if (B.out_prev) {                                // L_ns at row r (age 1)
          B.out_prev[p] = S.L[i][1][0];
          if (CPLX) B.out_prev[C.g.N + p] = S.L[i][1][1];
        }
      }
    } else if (i < H) {
      S.L[i + 1][2][0] = S.L[i + 1][1][0];
      S.L[i + 1][1][0] = S.L[i + 1][0][0];
      S.L[i + 1][0][0] = o0;
      if (CPLX) {
        S.L[i + 1][2][1] = S.L[i + 1][1][1];
        S.L[i + 1][1][1] = S.L[i + 1][0][1];
        S.L[i + 1][0][1] = o1;
      }
    }
    su = sl;
  }
}

template <int H, int NT, int ns, bool CPLX, bool GEN>
__device__ __forceinline__ void wave_block(const WCtx<H, NT>& C) {
  using G = WGeom<H, NT>;
  WState<H> S;
#pragma unroll
  for (int i = 0; i <= H; ++i)
#pragma unroll
    for (int a = 0; a < 3; ++a) S.L[i][a][0] = S.L[i][a][1] = 0.0;
#pragma unroll
  for (int i = 0; i < ns; ++i) {
    S.co[i][0] = C.B->ar[i];
    S.co[i][1] = C.B->br[i];
    S.co[i][2] = CPLX ? C.B->ai[i] : 0.0;
    S.co[i][3] = CPLX ? C.B->bi[i] : 0.0;
  }
  const int tau0 = C.y0 - ns, tau1 = C.y1 + ns;         // L_1 rows tau0 .. tau1-1
  WRow nxt;
  wave_load_row<H, NT, CPLX, GEN>(C, tau0, nxt);
  int slot = (tau0 % G::NSLOT + G::NSLOT) % G::NSLOT;   // history slot of row tau
  for (int tau = tau0; tau < tau1; ++tau) {
    wave_step<H, NT, ns, CPLX, GEN>(C, S, tau, slot, nxt, tau1);
    slot = slot + 1 == G::NSLOT ? 0 : slot + 1;
  }
}

// one compact specialised loop per (steps, real/complex): no level guards in the loop
template <int H, int NT, int NS, bool GEN>
__device__ __forceinline__ void wave_dispatch_ns(const WCtx<H, NT>& C, int ns, bool cplx) {
  if constexpr (NS >= 1) {
    if (ns == NS) {
      if (cplx) wave_block<H, NT, NS, true, GEN>(C);
      else wave_block<H, NT, NS, false, GEN>(C);
      return;
    }
    wave_dispatch_ns<H, NT, NS - 1, GEN>(C, ns, cplx);
  }
}

// GEN: the general variant (Dirichlet boundary faces of paper mode, halo rows of a slab);
// GEN = false is the one-rank Neumann path with neither compiled in
template <int H, int NT, bool GEN>
__global__ void __launch_bounds__(NT, NT > 128 ? 2 : 3) k_wave(Geo g, WSweep W, const double* __restrict__ what,
                                                            const IterState* st, WSlab sl) {
  using G = WGeom<H, NT>;
  if (st && st->done) return;
  extern __shared__ __align__(16) double wsm[];
  WCtx<H, NT> C;
  int bi = 0;                                           // this CTA's block (flat 1-D grid)
  while (bi + 1 < W.nb && (int)blockIdx.x >= W.cta0[bi + 1]) ++bi;
  const int cta = (int)blockIdx.x - W.cta0[bi];
  C.B = &W.b[bi];
  C.what = what;
  C.g = g;
  C.sl = sl;
  C.xch = wsm;
  C.hist = wsm + G::XCH + threadIdx.x;
  C.t = threadIdx.x;
  const int strip = cta % W.nstrip, chunk = cta / W.nstrip;
  C.x = strip * G::TX - H + C.t;
  C.colin = C.x >= 0 && C.x < g.nx;
  C.colout = C.t >= H && C.t < NT - H && C.x < g.nx;
  C.y0 = chunk * W.ly[bi];
  C.y1 = min(C.y0 + W.ly[bi], g.ny);
  // zero pads of the exchange rows and of the history rows (never written)
  for (int k = threadIdx.x; k < 2 * H * 2; k += NT) {
    wsm[k * G::XW] = 0.0;
    wsm[k * G::XW + G::XW - 1] = 0.0;
  }
  for (int k = threadIdx.x; k < G::NSLOT * 4; k += NT) wsm[G::XCH + k * G::HW + NT] = 0.0;
  wave_dispatch_ns<H, NT, H, GEN>(C, C.B->ns, C.B->np == 2);
}
