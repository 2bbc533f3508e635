// wave_r.cuh -- temporally blocked Chebyshev solves (2D): the y-wavefront with every per-row
// operand in registers.
//
// Same method and wavefront as wave.cuh (PAPER.md:266-275 Eq. eq:blockproblem; recurrence of
// reading R8), organised for the B200 SM's measured limits (scripts/ubench_smem.cu on the pool's
// B200: LDS.64 / STS.64 cost 2 SM-cycles per warp on the 128 B/clk shared-memory crossbar, a
// 32-bit SHFL 1 cycle on the SAME crossbar, a DFMA 0.5 cycle):
//  * wave.cuh kept the ŵ rows and face weights of the last H+2 rows in a shared-memory history
//    and read six of them per level: with the x-neighbour exchange, 12 crossbar operations
//    (24 cycles) against 34 DFMA/DADD (17 cycles) per complex point-step -- crossbar-bound;
//  * here each level i keeps the row it works on (row tau - i) in registers -- ŵ, the face
//    weights and e = 1 + sum of the four face weights - Re Lambda -- and the rows move one
//    level down per step (register moves, 0.25 cycle each); only the x-neighbour exchange
//    goes through shared memory (1 STS + 2 LDS per plane);
//  * the residual in diagonal form, r = w - e c - i Im(Lambda) c + sum_f w_f c_nb(f):
//    22 fp64 instructions per complex point-step (12 for r, 10 for the three-term update)
//    instead of 34, 8 per real one instead of 13.
// Halo columns (H per side) and the 2 ns warm-up rows of a chunk are computed redundantly and
// discarded; out-of-domain points hold zero and carry zero face weights, so they stay zero.
#pragma once

#include "tma.cuh"
#include "wave.cuh"

#ifndef WR_PAIRX
#define WR_PAIRX 1                                      // -DWR_PAIRX=0: one exchange row per plane
#endif

template <typename T> struct WRVec;
template <> struct WRVec<double> {
  using T2 = double2;
  static __device__ __forceinline__ double2 make(double a, double b) { return make_double2(a, b); }
};
template <> struct WRVec<float> {
  using T2 = float2;
  static __device__ __forceinline__ float2 make(float a, float b) { return make_float2(a, b); }
};

template <int NT>
struct WRGeom {
  static constexpr int XW = NT + 2;                     // exchange row: zero pad at both ends
};

// Thread-block cluster helpers (k_waver with CLU: the strips of one row chunk form a cluster and
// exchange their edge columns through distributed shared memory instead of recomputing an x-halo).
__device__ __forceinline__ uint32_t wr_mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// st.async: store into a neighbour CTA's shared memory and complete `bytes` of the transaction
// count of its mbarrier (the consumer waits on its own barrier at CTA scope -- no cluster-scope
// acquire, which would invalidate L1 on every step). Predicated inside the asm (no branch: a
// divergent branch per level made ptxas fence every level into its own reconvergence region),
// and no "memory" clobber: the stores only touch the neighbour's pad slots, which this thread
// never reads.
#define WR_STA(TY, REGS, ...)                                                                         \
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %0, 0;\n@q st.async.shared::cluster.mbarrier::complete_tx::bytes" \
               TY " [%1], " REGS ", [%2];\n}" ::"r"((int)p), "r"(a), "r"(bar), __VA_ARGS__)
__device__ __forceinline__ void wr_st_async(bool p, uint32_t a, double v, uint32_t bar) {
  WR_STA(".f64", "%3", "d"(v));
}
__device__ __forceinline__ void wr_st_async(bool p, uint32_t a, double2 v, uint32_t bar) {
  WR_STA(".v2.f64", "{%3, %4}", "d"(v.x), "d"(v.y));
}
__device__ __forceinline__ void wr_st_async(bool p, uint32_t a, float v, uint32_t bar) {
  WR_STA(".f32", "%3", "f"(v));
}
__device__ __forceinline__ void wr_st_async(bool p, uint32_t a, float2 v, uint32_t bar) {
  WR_STA(".v2.f32", "{%3, %4}", "f"(v.x), "f"(v.y));
}
#undef WR_STA
// Cluster-side state of a thread (k_waver CLU). Exchange rows and step barriers are indexed by
// the step's phase mod 3 (three buffers): a strip sends the values of step tau + 1 during step
// tau, as soon as each level produces them, so they have most of a step to cross the cluster.
struct WRClu {
  uint32_t rem;      // edge threads: the neighbour strip's exchange rows (shared::cluster), else 0
  uint32_t rbar;     // the neighbour's step barriers (shared::cluster)
  int roff;          // the neighbour's pad slot this thread fills (0 or XW - 1)
  uint64_t* bar;     // this CTA's step barriers [3][WRC_G]
  uint32_t tx0, tx1; // bytes the neighbours deliver per step to barrier group 0 / 1
  int tau0, nend;    // first step; one past the last step the loop runs
};
// Barrier groups per step: levels 1..NS/2 and NS/2+1..NS complete separate barriers, so the
// edge threads wait for the second half only before level NS/2 + 1 (followed by a CTA barrier:
// the wait stays outside the branch-free level code).
#ifndef WRC_SPLIT
#define WRC_SPLIT 1                                      // 0: one barrier group per step
#endif
template <int NS> struct WRCG {
  static constexpr int G = (WRC_SPLIT && NS >= 4) ? 2 : 1;
  static constexpr int H0 = G == 2 ? NS / 2 : NS;
};

__device__ __forceinline__ void wr_cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void wr_cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

struct WRRow { double w0, w1, xl, xh, yl, yh, s0, s1, m0, m1; };

// Row r of the block's inputs (zero outside the domain / the strip).
template <bool CPLX, bool GEN, bool VIRT>
__device__ __forceinline__ void waver_load(const WBlk& B, const double* __restrict__ what, const Geo& g,
                                           const WSlab& sl, int x, bool colin, int r, WRRow& R) {
  R.w0 = R.w1 = R.xl = R.xh = R.yl = R.yh = R.s0 = R.s1 = R.m0 = R.m1 = 0.0;
  if constexpr (!GEN) {
    if (colin && r >= 0 && r < g.ny) {
      const long long p = (long long)r * g.nx + x;
      const double* wq = what + (long long)B.q * g.N + p;
      R.w0 = __ldg(wq);
      if (CPLX) R.w1 = __ldg(wq + g.N);
      R.xl = __ldg(g.wx + p);
      R.xh = __ldg(g.wx + p + 1);
      R.yl = __ldg(g.wy + p);
      R.yh = __ldg(g.wy + p + g.nx);
      if constexpr (!VIRT) {
        R.s0 = B.ps[p];
        R.m0 = B.pm[p];
        if (CPLX) {
          R.s1 = B.ps[g.N + p];
          R.m1 = B.pm[g.N + p];
        }
      }
    }
    return;
  }
  const int er = r + sl.eoff;                            // row of the extended weight arrays
  if (colin && er >= 0 && er < sl.ne) {
    const long long p = (long long)r * g.nx + x;
    const long long pe = (long long)er * g.nx + x;
    const double* wq;
    long long ws;
    if (r < 0) {
      ws = (long long)sl.hd * g.nx;
      wq = sl.whlo + (long long)B.q * ws + (long long)(r + sl.hd) * g.nx + x;
    } else if (r >= g.ny) {
      ws = (long long)sl.hd * g.nx;
      wq = sl.whhi + (long long)B.q * ws + (long long)(r - g.ny) * g.nx + x;
    } else {
      ws = g.N;
      wq = what + (long long)B.q * g.N + p;
    }
    R.w0 = __ldg(wq);
    if (CPLX) R.w1 = __ldg(wq + ws);
    R.xl = __ldg(sl.wxe + pe);
    R.xh = __ldg(sl.wxe + pe + 1);
    R.yl = __ldg(sl.wye + pe);
    R.yh = __ldg(sl.wye + pe + g.nx);
    if constexpr (!VIRT) {                               // (later passes: one rank only)
      R.s0 = B.ps[p];
      R.m0 = B.pm[p];
      if (CPLX) {
        R.s1 = B.ps[g.N + p];
        R.m1 = B.pm[g.N + p];
      }
    }
  }
}

// One point-step of the recurrence of reading R8 in diagonal form (L_{i+1} at row r from L_i at
// rows r-1 (dn), r (c), r+1 (up), its x-neighbours (xl_nb, xr_nb) and L_{i-1} at row r (m)):
//   res = w - e c - i Im(Lambda) c + sum_f w_f c_nb(f),  x_new = c + a (c - m) + b res,
// e = 1 + sum_f w_f - Re Lambda; the y+1 neighbour enters last (it is the newest value).
template <bool CPLX, typename T>
__device__ __forceinline__ void wr_level(T c0, T c1, T up0, T up1, T dn0, T dn1, T m0, T m1, T l0, T l1, T rr0,
                                         T rr1, T w0, T w1, T e, T fxl, T fxh, T fyl, T fyh, T li, T ar, T ai,
                                         T br, T bi, T& o0, T& o1) {
  T q0 = fma(-e, c0, w0);
  if constexpr (CPLX) {
    T q1 = fma(-e, c1, w1);
    q0 = fma(-li, c1, q0);
    q1 = fma(li, c0, q1);
    q0 = fma(fxl, l0, q0);
    q1 = fma(fxl, l1, q1);
    q0 = fma(fxh, rr0, q0);
    q1 = fma(fxh, rr1, q1);
    q0 = fma(fyl, dn0, q0);
    q1 = fma(fyl, dn1, q1);
    const T dr = c0 - m0, di = c1 - m1;
    const T X0 = fma(-ai, di, fma(ar, dr, c0));
    const T X1 = fma(ai, dr, fma(ar, di, c1));
    const T r0 = fma(fyh, up0, q0);
    const T r1 = fma(fyh, up1, q1);
    o0 = fma(-bi, r1, fma(br, r0, X0));
    o1 = fma(bi, r0, fma(br, r1, X1));
  } else {
    q0 = fma(fxl, l0, q0);
    q0 = fma(fxh, rr0, q0);
    q0 = fma(fyl, dn0, q0);
    const T X0 = fma(ar, c0 - m0, c0);
    o0 = fma(br, fma(fyh, up0, q0), X0);
    o1 = T(0);
  }
}

// Register state of one thread for one block.
//   L[i][slot][e]: level i (L_0 = x_{s0-1}, L_i = x_{s0+i-1}), plane e, as a 3-slot ring: at step
//                  tau the row of age a (0 = newest, row tau - i + 1 after this step's push)
//                  sits in slot (a - tau) mod 3, so pushing a row overwrites the oldest and the
//                  ring never moves (the step loop is unrolled by 3: slot indices are static)
//   R*[i]:         operands of the row level i works on (row tau - i); index 0 = the row that
//                  entered at this step. These rows move one level down per step (register
//                  moves). A 9-slot row ring with the step loop unrolled by 9 needs no moves but
//                  measured slower (8.58 vs 8.36 ms per headline solve: a 58 KB loop body and
//                  uniform-register spills).
template <int NS, int NP, typename T>
struct WRState {
  T L[NS + 1][3][NP];
  T Rw[NS + 1][NP], Re[NS + 1], Rxl[NS + 1], Rxh[NS + 1], Ryl[NS + 1];
};

template <int PH, int A>
struct WSlot { static constexpr int v = ((A - PH) % 3 + 3) % 3; };

// One step tau (tau mod 3 == PH) of the wavefront.
template <int NT, int NS, bool CPLX, bool GEN, bool VIRT, bool CLU, int PH, typename T>
__device__ __forceinline__ void waver_step(WRState<NS, CPLX ? 2 : 1, T>& S, const WBlk& B,
                                           const double* __restrict__ what, const Geo& g, const WSlab& sl,
                                           T* xch, int t, int x, bool colin, bool colout, int y0,
                                           int y1, int tau, int tau1, double e0, double dB, WRRow& nxt,
                                           const WRClu& C) {
  constexpr int XW = WRGeom<NT>::XW;
  constexpr int NP = CPLX ? 2 : 1;
  constexpr int S0 = WSlot<PH, 0>::v, S1 = WSlot<PH, 1>::v, S2 = WSlot<PH, 2>::v;
  constexpr int NB = CLU ? 3 : 2;                       // exchange buffers
  const int buf = CLU ? PH : (tau & 1);
  T* xb = xch + buf * (NS * NP * XW) + 1 + t;
  // complex blocks: the (Re, Im) pair of a column is one 2-vector in the exchange rows (one
  // STS.128 + two LDS.128 per level instead of two STS.64 + four LDS.64)
  using T2 = typename WRVec<T>::T2;
  T2* xb2 = reinterpret_cast<T2*>(xch) + buf * (NS * XW) + 1 + t;
  (void)NB;
  // cluster: values of step tau + 1 go to the neighbour's buffer (PH + 1) % 3, completing bytes
  // on its barrier PH (group of the level); sent only if step tau + 1 runs
  constexpr int G = WRCG<NS>::G, H0 = WRCG<NS>::H0;
  const bool snd = CLU && C.rem && tau + 1 < C.nend;
  auto send = [&](int k, T v0, T v1) {                  // index k (1-based) of step tau + 1
    if constexpr (CLU) {
      constexpr int bn = (PH + 1) % 3;
      const uint32_t rb = C.rbar + 8u * (uint32_t)(PH * G + (k > H0 ? 1 : 0));
      if constexpr (CPLX && WR_PAIRX) {
        wr_st_async(snd, C.rem + (uint32_t)(((bn * NS + (k - 1)) * XW + C.roff) * sizeof(T2)), WRVec<T>::make(v0, v1),
                    rb);
      } else {
        wr_st_async(snd, C.rem + (uint32_t)(((bn * NS * NP + (k - 1) * NP) * XW + C.roff) * sizeof(T)), v0, rb);
        if (CPLX)
          wr_st_async(snd, C.rem + (uint32_t)(((bn * NS * NP + (k - 1) * NP + 1) * XW + C.roff) * sizeof(T)), v1, rb);
      }
    }
  };
  // (1) publish the newest row of every level (L_i at row tau - i; age 1 after this step's
  //     push) for the x-neighbours
#pragma unroll
  for (int i = 1; i <= NS; ++i) {
    if constexpr (CPLX && WR_PAIRX) {
      xb2[(i - 1) * XW] = WRVec<T>::make(S.L[i][S1][0], S.L[i][S1][1]);
    } else {
#pragma unroll
      for (int e = 0; e < NP; ++e) xb[((i - 1) * NP + e) * XW] = S.L[i][S1][e];
    }
  }
  // cluster: the phases of step tau + 1 complete when the neighbours' bytes have landed
  if (CLU && t == NT / 2 && tau + 1 < C.nend) {
    mbar_arrive_expect_tx(C.bar + PH * G, C.tx0);
    if (G == 2) mbar_arrive_expect_tx(C.bar + PH * G + 1, C.tx1);
  }
  // (2) rows move one level down; row tau enters (L_0, L_1 and its operands)
#pragma unroll
  for (int i = NS; i >= 1; --i) {
#pragma unroll
    for (int e = 0; e < NP; ++e) S.Rw[i][e] = S.Rw[i - 1][e];
    S.Re[i] = S.Re[i - 1];
    S.Rxl[i] = S.Rxl[i - 1];
    S.Rxh[i] = S.Rxh[i - 1];
    S.Ryl[i] = S.Ryl[i - 1];
  }
  const WRRow cur = nxt;
  if (tau + 1 < tau1) waver_load<CPLX, GEN, VIRT>(B, what, g, sl, x, colin, tau + 1, nxt);
  // (the operands are stored in fp64; T = float computes the recurrence in fp32: the
  //  mixed-precision inner solve of AAC_F32, fp64 GMRES outside)
  S.Rw[0][0] = T(cur.w0);
  if (CPLX) S.Rw[0][1] = T(cur.w1);
  S.Rxl[0] = T(cur.xl);
  S.Rxh[0] = T(cur.xh);
  S.Ryl[0] = T(cur.yl);
  {
    double dd = dB;
    if (GEN && g.dir) {
      const int rg = tau + sl.lo;
      dd += g.bdy * ((rg == 0) + (rg == sl.nyg - 1));
    }
    // (out of the domain: e = 1 - Re Lambda on zero iterates and zero weights -- harmless)
    S.Re[0] = T(((e0 + dd) + (cur.xl + cur.xh)) + (cur.yl + cur.yh));
  }
  if constexpr (VIRT) {                                  // x_0 = 0, x_1 = w / theta
    S.L[1][S0][0] = T(B.sr * cur.w0 - B.si * cur.w1);
    if (CPLX) S.L[1][S0][1] = T(B.sr * cur.w1 + B.si * cur.w0);
  } else {
    S.L[1][S0][0] = T(cur.s0);
    S.L[0][S0][0] = T(cur.m0);
    if (CPLX) {
      S.L[1][S0][1] = T(cur.s1);
      S.L[0][S0][1] = T(cur.m1);
    }
  }
  send(1, S.L[1][S0][0], CPLX ? S.L[1][S0][1] : T(0));
  // cluster: step tau's values from the neighbours (barrier (PH + 2) % 3; none at the first step)
  constexpr int BW = (PH + 2) % 3;
  const bool rcv = CLU && C.rem && tau > C.tau0;
  const uint32_t par = (uint32_t)(((tau - C.tau0 - 1) / 3) & 1);
  if (rcv) mbar_wait(C.bar + BW * G, par);
  __syncthreads();
  // (3) levels: L_{i+1} at row r = tau - i
  const T li = T(B.li);
#pragma unroll
  for (int i = 1; i <= NS; ++i) {
    if (G == 2 && i == H0 + 1) {
      if (rcv) mbar_wait(C.bar + BW * G + 1, par);
      __syncthreads();
    }
    const T* xr = xb + ((i - 1) * NP) * XW;
    const int e1 = CPLX ? 1 : 0;
    T nl0, nl1, nr0, nr1;                                // x-neighbours (left, right)
    if constexpr (CPLX && WR_PAIRX) {
      const T2 a = xb2[(i - 1) * XW - 1], b = xb2[(i - 1) * XW + 1];
      nl0 = a.x; nl1 = a.y; nr0 = b.x; nr1 = b.y;
    } else {
      nl0 = xr[-1]; nl1 = CPLX ? xr[XW - 1] : T(0); nr0 = xr[1]; nr1 = CPLX ? xr[XW + 1] : T(0);
    }
    T o0, o1;
    wr_level<CPLX, T>(S.L[i][S1][0], S.L[i][S1][e1], S.L[i][S0][0], S.L[i][S0][e1], S.L[i][S2][0], S.L[i][S2][e1],
                      i == 1 ? (VIRT ? T(0) : S.L[0][S1][0]) : S.L[i - 1][S2][0],
                      i == 1 ? (VIRT ? T(0) : S.L[0][S1][e1]) : S.L[i - 1][S2][e1],
                      nl0, nl1, nr0, nr1,
                      S.Rw[i][0], S.Rw[i][e1], S.Re[i], S.Rxl[i], S.Rxh[i], S.Ryl[i], S.Ryl[i - 1], li,
                      T(B.ar[i - 1]), CPLX ? T(B.ai[i - 1]) : T(0), T(B.br[i - 1]), CPLX ? T(B.bi[i - 1]) : T(0),
                      o0, o1);
    if (i == NS) {
      const int r = tau - i;
      if (colout && r >= y0 && r < y1) {
        if (GEN && (r < 0 || r >= g.ny)) {               // slab ghost row (-1 or ny): the
          double* gq = (r < 0 ? B.glo : B.ghi) + x;      // neighbour's boundary row of x_{p_k}
          gq[0] = o0;
          if (CPLX) gq[g.nx] = o1;
          continue;
        }
        const long long p = (long long)r * g.nx + x;
        B.out_last[p] = o0;
        if (CPLX) B.out_last[g.N + p] = o1;
        if (B.out_prev) {                                // L_ns at row r (age 1)
          B.out_prev[p] = S.L[i][S1][0];
          if (CPLX) B.out_prev[g.N + p] = S.L[i][S1][1];
        }
      }
    } else {                                             // push: overwrites the oldest row
      S.L[i + 1][S0][0] = o0;
      if (CPLX) S.L[i + 1][S0][1] = o1;
      send(i + 1, o0, o1);
    }
  }
}

// All ns steps of one block over this CTA's strip x row chunk.
template <int NT, int NS, bool CPLX, bool GEN, bool VIRT, bool CLU, typename T>
__device__ __forceinline__ void waver_block(const WBlk& B, const double* __restrict__ what, const Geo& g,
                                            const WSlab& sl, T* xch, int t, int x, bool colin,
                                            bool colout, int y0, int y1, WRClu& C) {
  constexpr int NP = CPLX ? 2 : 1;
  WRState<NS, NP, T> S;
#pragma unroll
  for (int i = 0; i <= NS; ++i) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int e = 0; e < NP; ++e) S.L[i][a][e] = T(0);
#pragma unroll
    for (int e = 0; e < NP; ++e) S.Rw[i][e] = T(0);
    S.Re[i] = S.Rxl[i] = S.Rxh[i] = S.Ryl[i] = T(0);
  }
  const double e0 = 1.0 - B.lr;                          // diagonal shift: 1 - Re Lambda
  double dB = 0.0;                                       // Dirichlet boundary faces (paper mode)
  if (GEN && g.dir) dB = g.bdx * ((x == 0) + (x == g.nx - 1));
  // L_1 rows tau0 .. tau1-1; the loop runs whole triples of steps (a step past tau1 computes
  // rows past the chunk, which are never stored). Phase 0 at tau0 (shifted into [0, 3) so the
  // slot of a row never depends on the sign of tau).
  const int tau0 = y0 - NS, tau1 = y1 + NS;
  C.tau0 = tau0;
  C.nend = tau0 + 3 * ((tau1 - tau0 + 2) / 3);
  WRRow nxt;
  waver_load<CPLX, GEN, VIRT>(B, what, g, sl, x, colin, tau0, nxt);
  for (int tau = tau0; tau < tau1; tau += 3) {
    waver_step<NT, NS, CPLX, GEN, VIRT, CLU, 0, T>(S, B, what, g, sl, xch, t, x, colin, colout, y0, y1, tau, tau1, e0, dB, nxt, C);
    waver_step<NT, NS, CPLX, GEN, VIRT, CLU, 1, T>(S, B, what, g, sl, xch, t, x, colin, colout, y0, y1, tau + 1, tau1, e0, dB, nxt, C);
    waver_step<NT, NS, CPLX, GEN, VIRT, CLU, 2, T>(S, B, what, g, sl, xch, t, x, colin, colout, y0, y1, tau + 2, tau1, e0, dB, nxt, C);
  }
}

// One launch per packed block (the host launches the active blocks concurrently on several
// streams): with the block's step count, planes and pass kind compile-time, ptxas keeps the
// block's scalars (a_s, b_s, Lambda, 1/theta) in uniform registers and the DFMAs take them as
// uniform operands -- a DFMA with three 64-bit register operands costs 3 register-file cycles per
// warp on the B200 SMSP (scripts/ubench_dp.cu: 3.2 vs 2.3 cycles with a uniform operand), and an
// in-kernel dispatch over the variants made ptxas fall back to per-thread LDC loads.
struct WROne {
  WBlk b;
  int nstrip;                // strips of NT - 2H columns
  int ly;                    // rows per chunk
  int ybeg, yend;            // output rows [ybeg, yend): [0, ny), or one slab ghost row more per
                             // side with a neighbour (ghost mode)
};

// Shared memory: the x-exchange rows [2 buffers][NS levels][planes][NT + 2].
template <int NT, typename T>
__host__ __device__ constexpr size_t waver_smem(int ns, int np) { return (size_t)2 * ns * np * (NT + 2) * sizeof(T); }
// + the two step barriers of the cluster kernel
template <int NT, typename T>
__host__ __device__ constexpr size_t waver_smem_clu(int ns, int np) {
  return (size_t)3 * ns * np * (NT + 2) * sizeof(T) + 8 * 3 * ((WRC_SPLIT && ns >= 4) ? 2 : 1);
}

// CLU (one rank, nx <= 8 NT): the nstrip strips of a row chunk are one thread-block cluster and
// the strips carry NO x-halo -- every step each strip's edge threads also store their columns
// into the neighbouring strips' pad slots (st.async, completing bytes on the neighbour's step
// barrier), and the edge threads wait on their own CTA's barrier (CTA scope) before the levels
// read the pads. Only neighbours couple (no cluster-wide barrier per step: barrier.cluster with
// its cluster-scope acquire measured 10.1 vs 8.3 ms per headline solve -- it also invalidates L1).
// The points computed and their operands are those of the halo kernel: bit-identical results.
template <int H, int NT, int NS, bool CPLX, bool GEN, bool VIRT, bool CLU, typename T>
__global__ void __launch_bounds__(NT, CPLX ? 2 : 3) k_waver(Geo g, const __grid_constant__ WROne P,
                                                            const double* __restrict__ what,
                                                            const IterState* st, WSlab sl) {
  if (st && st->done) return;
  extern __shared__ __align__(16) unsigned char wsm_raw[];
  T* wsm = reinterpret_cast<T*>(wsm_raw);
  const WBlk& B = P.b;
  const int t = threadIdx.x;
  // x-halo of NS columns per side: a wrong edge value reaches one column further per level
  constexpr int HX = CLU ? 0 : NS;
  constexpr int TX = NT - 2 * HX;
  const int cta = (!CLU && (c_rev & AAC_REV_WAVE)) ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x;
  const int strip = cta % P.nstrip, chunk = cta / P.nstrip;
  const int x = strip * TX - HX + t;
  const bool colin = x >= 0 && x < g.nx;
  const bool colout = t >= HX && t < NT - HX && x < g.nx;
  const int y0 = P.ybeg + chunk * P.ly;
  const int y1 = min(y0 + P.ly, P.yend);
  // zero pads of the exchange rows (never written without a cluster; with one, written by the
  // neighbouring strips only -- the strips at the domain edges keep zero there)
  constexpr int XW = NT + 2;
  if constexpr (CPLX && WR_PAIRX) {                     // rows of XW (Re, Im) pairs
    using T2 = typename WRVec<T>::T2;
    T2* w2 = reinterpret_cast<T2*>(wsm);
    for (int k = t; k < (CLU ? 3 : 2) * NS; k += NT) {
      w2[k * XW] = WRVec<T>::make(T(0), T(0));
      w2[k * XW + XW - 1] = WRVec<T>::make(T(0), T(0));
    }
  } else {
    constexpr int NROW = (CLU ? 3 : 2) * NS * (CPLX ? 2 : 1);
    for (int k = t; k < NROW; k += NT) {
      wsm[k * XW] = T(0);
      wsm[k * XW + XW - 1] = T(0);
    }
  }
  WRClu C{0u, 0u, 0, nullptr, 0u, 0u, 0, 0};
  if constexpr (CLU) {
    constexpr int G = WRCG<NS>::G, H0 = WRCG<NS>::H0;
    C.bar = reinterpret_cast<uint64_t*>(wsm_raw + waver_smem_clu<NT, T>(NS, CPLX ? 2 : 1) - 8 * 3 * G);
    const uint32_t lb = (uint32_t)__cvta_generic_to_shared(wsm);
    const uint32_t bb = (uint32_t)__cvta_generic_to_shared(C.bar);
    if (t == 0 && strip > 0) {
      C.rem = wr_mapa(lb, (uint32_t)(strip - 1));
      C.rbar = wr_mapa(bb, (uint32_t)(strip - 1));
      C.roff = XW - 1;
    } else if (t == NT - 1 && strip < P.nstrip - 1) {
      C.rem = wr_mapa(lb, (uint32_t)(strip + 1));
      C.rbar = wr_mapa(bb, (uint32_t)(strip + 1));
      C.roff = 0;
    }
    const int nnb = (strip > 0) + (strip < P.nstrip - 1);
    C.tx0 = (uint32_t)(nnb * H0 * (CPLX ? 2 : 1) * (int)sizeof(T));
    C.tx1 = (uint32_t)(nnb * (NS - H0) * (CPLX ? 2 : 1) * (int)sizeof(T));
    if (t == 0) {
      for (int k = 0; k < 3 * G; ++k) mbar_init(C.bar + k, 1);
      fence_mbar_init();
    }
    wr_cluster_arrive();                                 // barriers initialised and pads zeroed
    wr_cluster_wait();                                   // everywhere before any neighbour writes
  }
  waver_block<NT, NS, CPLX, GEN, VIRT, CLU, T>(B, what, g, sl, wsm, t, x, colin, colout, y0, y1, C);
  if constexpr (CLU) {                                   // (every store into this CTA was waited
    wr_cluster_arrive();                                 //  for; keep the cluster alive anyway until
    wr_cluster_wait();                                   //  all strips are done)
  }
}
