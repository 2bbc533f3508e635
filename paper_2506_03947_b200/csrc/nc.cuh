// nc.cuh -- nested Chebyshev application of the block alpha-circulant preconditioner.
//
// P_alpha^{-1} r = (Gamma^{-1} U (x) I)(I (x) A - Lambda (x) I)^{-1}(U^* Gamma (x) I) r
// (PAPER.md:252-254 Eq. eq:Paform, pairing of reading R6), block problems
// (A - Lambda_k) y_k = w_k (Eq. eq:blockproblem) solved by p_k Chebyshev iterations
// (recurrence of reading R8):
//   x_0 = 0, x_1 = w/theta, x_{s+1} = x_s + a_s (x_s - x_{s-1}) + b_s (w - (A - Lambda) x_s).
//
// Packed half-complex layout: for real input the ell Fourier blocks satisfy
// w_{ell-k} = conj(w_k), so only k = 0..ell/2 are solved:
//   plane 0            = block 0 (real, Lambda_0 = alpha^{1/ell})
//   planes 2k-1, 2k    = Re, Im of block k, k = 1..ell/2-1
//   plane ell-1        = block ell/2 (real, Lambda = -alpha^{1/ell})
// i.e. ell real planes, the same bytes as the real block vector.
//
// Kernels (one GMRES iteration = k_forward, P_max-2 x k_sweep, k_sweep<LAST>):
//   k_forward   (optional fused Arnoldi update u = s_w W - sum_i c_i s_i V_i, its squared
//                norm and the new basis vector) + gamma-scale + real->half-complex DFT
//   k_sweep     one Chebyshev step for every block active at this sweep (aligned ends:
//                block k starts at sweep P_max - p_k), threadIdx.y = block
//   k_sweep<LAST> the final step of every block fused with the inverse DFT and
//                gamma^{-1} scaling: x_{p_k} never goes to HBM
#pragma once

#include "krylov.cuh"
#include "stencil.cuh"
#include "tma.cuh"

struct Dft {
  int ell;
  double g[AAC_MAX_ELL];     // gamma_j = alpha^{j/ell}
  double gi[AAC_MAX_ELL];    // 1/gamma_j
  double c[AAC_MAX_ELL];     // cos(2 pi m/ell)
  double s[AAC_MAX_ELL];     // sin(2 pi m/ell)
  double scale;              // ell^{-1/2}
};

__device__ __forceinline__ int plane_of(int ell, int kb) {
  const int h = ell / 2;
  return kb == 0 ? 0 : (kb == h ? ell - 1 : 2 * kb - 1);
}

// Arnoldi update fused into the forward transform (GMRES mode, see krylov.cuh):
//   u = sigma_{j-1} W - sum_{i<j} c_i sigma_i V_i   written to V_j (unnormalised), ||u||^2 reduced.
struct FwdUpd {
  const double* W;           // calA Z_{j-1} (raw)
  double* V;                 // raw basis base pointer, stride L (V_0 = b on entry)
  long long L;
  double* part;              // per-CTA partials of ||u||^2
  ArnoldiCtx ac;             // st, sigma, c (CGS2 coefficients of column j-1), Givens state
  unsigned* grp;             // per-32-CTA ticket counters (zero between launches)
  int norm;                  // 1: reduce ||u||^2 and run the norm step here; 0: one-reduce mode
                             // (the projection pass measures it, krylov.cuh arnoldi_lagged_step)
};

// gamma-scale + real -> packed half-complex DFT of the ell values w[] of one point.
template <int ELLC>
__device__ __forceinline__ void dft_store(const Dft& D, long long N, long long p, double* w,
                                          double* __restrict__ what) {
  const int ell = D.ell, h = ell / 2;
  FOR_PL(pl) w[pl] *= D.g[pl];
  double s0 = 0.0, sh = 0.0;
  FOR_PL(pl) {
    s0 += w[pl];
    sh += (pl & 1) ? -w[pl] : w[pl];
  }
  what[p] = D.scale * s0;
  what[(long long)(ell - 1) * N + p] = D.scale * sh;
  for (int k = 1; k < h; ++k) {
    double re = 0.0, im = 0.0;
    int m = 0;
    FOR_PL(pl) {
      re = fma(w[pl], D.c[m], re);
      im = fma(-w[pl], D.s[m], im);
      m += k;
      if (m >= ell) m -= ell;
    }
    what[(long long)(2 * k - 1) * N + p] = D.scale * re;
    what[(long long)(2 * k) * N + p] = D.scale * im;
  }
}

// Same with ell == ELLC known at compile time: every twiddle index (k*pl mod ell) is static,
// so the transform is straight-line FMAs on registers with constant-bank twiddles.
template <int ELLC>
__device__ __forceinline__ void dft_store_exact(const Dft& D, long long N, long long p, double* w,
                                                double* __restrict__ what) {
  constexpr int h = ELLC / 2;
#pragma unroll
  for (int pl = 0; pl < ELLC; ++pl) w[pl] *= D.g[pl];
  double s0 = 0.0, sh = 0.0;
#pragma unroll
  for (int pl = 0; pl < ELLC; ++pl) {
    s0 += w[pl];
    sh += (pl & 1) ? -w[pl] : w[pl];
  }
  what[p] = D.scale * s0;
  what[(long long)(ELLC - 1) * N + p] = D.scale * sh;
#pragma unroll
  for (int k = 1; k < h; ++k) {
    double re = 0.0, im = 0.0;
#pragma unroll
    for (int pl = 0; pl < ELLC; ++pl) {
      re = fma(w[pl], D.c[(k * pl) % ELLC], re);
      im = fma(-w[pl], D.s[(k * pl) % ELLC], im);
    }
    what[(long long)(2 * k - 1) * N + p] = D.scale * re;
    what[(long long)(2 * k) * N + p] = D.scale * im;
  }
}

// Standalone forward transform: hat w = U^* Gamma r.
template <int ELLC>
__global__ void __launch_bounds__(256) k_forward(long long N, Dft D, const double* __restrict__ r,
                                                 double* __restrict__ what) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int ell = D.ell;
  double w[ELLC];
  FOR_PL(pl) w[pl] = __ldg(r + (long long)pl * N + p);
  dft_store<ELLC>(D, N, p, w, what);
}

constexpr int FT = 256;        // tile points per CTA (one per consumer thread)
#define AAC_FWD_MAXC 128       // update coefficients staged in shared memory (more: global loads)
constexpr int FS = 3;          // bulk-copy pipeline stages
constexpr int FW = FT / 32;    // consumer warps; warp FW is the TMA producer

// GMRES mode: form u from W and V_0..V_{j-1} (streamed through a TMA bulk-copy ring fed by
// a producer warp), store V_j, reduce ||u||^2 (last CTA: Arnoldi norm step), transform u.
template <int ELLC, bool TMA>
__global__ void __launch_bounds__(FT + 32) k_fwd_upd(long long N, Dft D, double* __restrict__ what,
                                                     FwdUpd U) {
  extern __shared__ __align__(16) double sm[];      // [FS][ELLC][FT]
  __shared__ __align__(8) uint64_t full[FS], empty[FS];
  __shared__ double red[FW];
  __shared__ double coefs[AAC_FWD_MAXC];       // update coefficients, loaded once per CTA
  __shared__ bool last;
  IterState* st = U.ac.st;
  if (st->done) return;
  const int j = st->j;
  const int ell = D.ell;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const unsigned bid = (c_rev & AAC_REV_FWD) ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
  const long long base = (long long)bid * FT;
  const int len = (int)((N - base) < FT ? (N - base) : FT);
  const int lb = len & ~1;
  const long long L = U.L;
  const int nitems = j == 0 ? 1 : j + 1;   // item 0: W (or V_0 when j == 0); item k: V_{k-1}
  auto src_of = [&](int k) -> const double* {
    return k == 0 ? (j == 0 ? U.V : U.W) : U.V + (long long)(k - 1) * L;
  };
  if (TMA && t == 0) {
    for (int s = 0; s < FS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], FW);
    }
    fence_mbar_init();
  }
  // the item coefficients are read by every consumer thread for every item: one parallel load
  // into shared memory instead of a dependent global load per item
  for (int k = t; k < nitems && k < AAC_FWD_MAXC; k += blockDim.x)
    coefs[k] = k == 0 ? (j == 0 ? 1.0 : U.ac.sigma[j - 1]) : -U.ac.c[k - 1] * U.ac.sigma[k - 1];
  __syncthreads();
  double nrm = 0.0;
  if (warp == FW) {                                 // ---- producer warp
    if (TMA && lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      for (int k = 0; k < nitems; ++k) {
        const int s = k % FS;
        if (k >= FS) mbar_wait(&empty[s], (uint32_t)(((k / FS) - 1) & 1));
        const bool hint = k == 0 ? (c_rev & AAC_L2_FWD_W) : (c_rev & AAC_L2_FWD);
        bulk_planes(sm + (long long)s * ELLC * FT, FT, src_of(k) + base, N, ell, len, &full[s], hint, pol);
      }
    }
  } else {                                          // ---- consumer warps
    const bool valid = t < len;
    double w[ELLC];
    FOR_PL(pl) w[pl] = 0.0;
    for (int k = 0; k < nitems; ++k) {
      const int s = k % FS;
      const double coef = k < AAC_FWD_MAXC ? coefs[k]
                          : (k == 0 ? (j == 0 ? 1.0 : U.ac.sigma[j - 1]) : -U.ac.c[k - 1] * U.ac.sigma[k - 1]);
      const double* src = src_of(k) + base;
      if constexpr (TMA) mbar_wait(&full[s], (uint32_t)((k / FS) & 1));
      if (valid) {
        FOR_PL(pl) {
          const double v = (TMA && t < lb) ? sm[((long long)s * ELLC + pl) * FT + t] : src[(long long)pl * N + t];
          w[pl] = fma(coef, v, w[pl]);
        }
      }
      if constexpr (TMA) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
    if (valid) {
      const long long p = base + t;
      if (j > 0) {
        double* vj = U.V + (long long)j * L;
        if (c_rev & AAC_L2_FWD_VJ) {                 // (streaming store: next read four kernels later)
          FOR_PL(pl) __stcs(vj + (long long)pl * N + p, w[pl]);
        } else {
          FOR_PL(pl) vj[(long long)pl * N + p] = w[pl];
        }
      }
      FOR_PL(pl) nrm = fma(w[pl], w[pl], nrm);
      if (ell == ELLC) dft_store_exact<ELLC>(D, N, p, w, what);
      else dft_store<ELLC>(D, N, p, w, what);
    }
    nrm = warp_sum(nrm);
    if (lane == 0) red[warp] = nrm;
  }
  // ||u||^2: CTA partial, then the last CTA reduces in a fixed order and finalises Arnoldi
  // column j-1 (or beta when j == 0).
  if (!U.norm) return;
  __syncthreads();
  if (t == 0) {
    double tot = 0.0;
    for (int w2 = 0; w2 < FW; ++w2) tot += red[w2];
    U.part[bid] = tot;
    __threadfence();
    // two-level ticket: thousands of CTAs taking a ticket on ONE counter serialise in L2;
    // the last CTA of each group of 32 takes the global ticket (and resets its group counter)
    const unsigned gid = bid >> 5;
    const unsigned gsz = min(32u, gridDim.x - (gid << 5));
    bool lst = false;
    if (atomicAdd(&U.grp[gid], 1u) == gsz - 1) {
      U.grp[gid] = 0;
      __threadfence();
      lst = atomicAdd(&st->tick, 1u) == ((gridDim.x + 31) >> 5) - 1;
    }
    last = lst;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    const double tot = block_sum_fixed(U.part, gridDim.x);
    if (t == 0) st->tick = 0;
    if (U.ac.local_only) {
      if (t == 0) U.ac.red[0] = tot;
    } else {
      arnoldi_norm_step_cta(U.ac, j, tot);
    }
  }
}

// ------------------------------------------------------------------------------------------
struct NcBlk {
  int kb;                    // packed block index (0..ell/2)
  int cplx;                  // 1: Re/Im plane pair
  int q;                     // first plane of the block
  // x_s = scs * (*ps), x_{s-1} = scm * (*pm): the virtual iterates x_1 = w/theta and x_0 = 0
  // become a pointer to hat w with a complex scale (theta^{-1}, or 0), so every block runs
  // the same branch-free code path.
  const double* ps;
  const double* pm;
  double* xo;                // x_{s+1}, plane q (unused in the LAST sweep)
  double sr, si;             // scs
  double mr, mi;             // scm
  double ar, ai, br, bi;     // a_s = rho_s rho_{s-1}, b_s = 2 rho_s / delta (complex)
  double lr, li;             // Lambda_k
};
struct NcSweep {
  NcBlk b[AAC_MAX_BLK];      // the active blocks of this sweep, compacted (threadIdx.y)
  int nact;
  // LAST sweep: every packed block, active or passive (p_k == 1: y_k = w_k / theta_k)
  int passive[AAC_MAX_BLK];
  double ptr[AAC_MAX_BLK], pti[AAC_MAX_BLK];
  int nblk;
};

constexpr int SW_TX = 64;                 // LAST: point groups per CTA along x (threadIdx.y = block)
constexpr int SW_FX = 128;                // otherwise: one block per CTA, flat grid (chunk, block)

template <int DIM, int VEC, bool LAST>
__global__ void __launch_bounds__(LAST ? SW_TX * AAC_MAX_BLK : SW_FX, LAST ? 2 : 4) k_sweep(Geo g, NcSweep P, Dft D,
                                                                 const double* __restrict__ what,
                                                                 const double* __restrict__ hlo,
                                                                 const double* __restrict__ hhi,
                                                                 double* __restrict__ zbase,
                                                                 long long zjs,
                                                                 const IterState* st) {
  if (st && st->done) return;
  // output: z (standalone) or Z_j = zbase + j * zjs (GMRES mode, j on the device)
  double* zout = zbase + (st ? (long long)st->j * zjs : 0LL);
  // LAST: final iterates of all blocks at this CTA's points, then the inverse DFT
  extern __shared__ double ysh[];         // [ell planes][SW_TX*VEC]
  const long long N = g.N;
  // grid (x-chunks of SW_TX*VEC points, ny, nz): coordinates without index division
  // (not LAST: blocks are independent, so each CTA runs one block and the grid is flat over
  // (x-chunk, block): full occupancy whatever the number of active blocks)
  constexpr int TXB = LAST ? SW_TX : SW_FX;
  const int cx = LAST ? (int)blockIdx.x : (int)blockIdx.x / P.nact;
  const int xx = (cx * TXB + threadIdx.x) * VEC;
  const long long row0 = ((long long)blockIdx.z * g.ny + blockIdx.y) * g.nx;
  const long long p = row0 + xx;
  const NcBlk& B = P.b[LAST ? (int)threadIdx.y : (int)blockIdx.x % P.nact];
  double out_r[VEC], out_i[VEC];
  if (xx < g.nx) {
    PtV<DIM, VEC> q;
    load_ptv_xyz<DIM, VEC>(g, xx, blockIdx.y, blockIdx.z, q);
    const double* wr = what + (long long)B.q * N;
    const double* hl = hlo + B.q * g.S;
    const double* hh = hhi + B.q * g.S;
    // all loads of the block first (stencil operands of both planes, x_{s-1}, hat w), then
    // the arithmetic: the loads are independent and stay in flight together
    SV<VEC> v0, v1;
    double m0[VEC], m1[VEC], w0[VEC], w1[VEC];
    load_sv<DIM, VEC>(g, q, B.ps, hl, hh, v0);
    ldc<VEC>(B.pm, p, m0);
    ldv<VEC>(wr, p, w0);
    if (B.cplx) {
      load_sv<DIM, VEC>(g, q, B.ps + N, hl + g.S, hh + g.S, v1);
      ldc<VEC>(B.pm + N, p, m1);
      ldv<VEC>(wr + N, p, w1);
    }
    double a0[VEC], a1[VEC];
    stencil_sv<DIM, VEC>(g, q, v0, a0);
    if (!B.cplx) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const double xs = B.sr * v0.c[e], Axs = B.sr * a0[e], xm = B.mr * m0[e];
        const double res = w0[e] - (Axs - B.lr * xs);
        out_r[e] = xs + B.ar * (xs - xm) + B.br * res;
      }
      if (!LAST) stv<VEC>(B.xo, p, out_r);
    } else {
      stencil_sv<DIM, VEC>(g, q, v1, a1);
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const double c0 = v0.c[e], c1 = v1.c[e];
        const double ur = B.sr * c0 - B.si * c1, ui = B.sr * c1 + B.si * c0;
        const double Aur = B.sr * a0[e] - B.si * a1[e], Aui = B.sr * a1[e] + B.si * a0[e];
        const double mr = B.mr * m0[e] - B.mi * m1[e], mi = B.mr * m1[e] + B.mi * m0[e];
        // residual w - (A - Lambda) x
        const double rr = w0[e] - (Aur - (B.lr * ur - B.li * ui));
        const double ri = w1[e] - (Aui - (B.lr * ui + B.li * ur));
        const double dr = ur - mr, di = ui - mi;
        out_r[e] = ur + (B.ar * dr - B.ai * di) + (B.br * rr - B.bi * ri);
        out_i[e] = ui + (B.ar * di + B.ai * dr) + (B.br * ri + B.bi * rr);
      }
      if (!LAST) {
        stv<VEC>(B.xo, p, out_r);
        stv<VEC>(B.xo + N, p, out_i);
      }
    }
    if (LAST) {
      const int tp = threadIdx.x * VEC;
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        ysh[B.q * (SW_TX * VEC) + tp + e] = out_r[e];
        if (B.cplx) ysh[(B.q + 1) * (SW_TX * VEC) + tp + e] = out_i[e];
      }
    }
  }
  if constexpr (LAST) {
    __syncthreads();
    // passive blocks (p_k == 1): y = w / theta straight from hat w
    const int ell = D.ell, h = ell / 2;
    const int npts = SW_TX * VEC;
    const long long p0 = row0 + (long long)blockIdx.x * npts;
    const int xlim = g.nx - blockIdx.x * npts;       // valid points of this CTA's row chunk
    const int nthr = blockDim.x * blockDim.y;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    for (int kb = 0; kb <= h; ++kb) {
      if (!P.passive[kb]) continue;
      const int qq = plane_of(ell, kb);
      const bool cp = (kb != 0 && kb != h);
      for (int t = tid; t < npts; t += nthr) {
        if (t >= xlim) continue;
        const double a = what[(long long)qq * N + p0 + t];
        const double b = cp ? what[(long long)(qq + 1) * N + p0 + t] : 0.0;
        ysh[qq * npts + t] = a * P.ptr[kb] - b * P.pti[kb];
        if (cp) ysh[(qq + 1) * npts + t] = a * P.pti[kb] + b * P.ptr[kb];
      }
    }
    __syncthreads();
    // z_j = ell^{-1/2} gamma_j^{-1} (y_0 + (-1)^j y_{ell/2} + 2 sum_{k=1}^{ell/2-1} Re(y_k e^{2 pi i jk/ell}))
    // thread (x, y) -> its VEC points, output planes j = y, y + nact, ...
    const int tp = threadIdx.x * VEC;
    if (tp < xlim) {
      for (int jj = threadIdx.y; jj < ell; jj += blockDim.y) {
        double acc[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] = 0.0;
        int m = jj;
        for (int kb = 1; kb < h; ++kb) {
          double yr[VEC], yi[VEC];
          ldc<VEC>(ysh, (2 * kb - 1) * npts + tp, yr);
          ldc<VEC>(ysh, (2 * kb) * npts + tp, yi);
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            acc[e] = fma(yr[e], D.c[m], acc[e]);
            acc[e] = fma(-yi[e], D.s[m], acc[e]);
          }
          m += jj;
          if (m >= ell) m -= ell;
        }
        double y0[VEC], yh[VEC], o[VEC];
        ldc<VEC>(ysh, tp, y0);
        ldc<VEC>(ysh, (ell - 1) * npts + tp, yh);
        const double f = D.scale * D.gi[jj];
#pragma unroll
        for (int e = 0; e < VEC; ++e) o[e] = f * (y0[e] + ((jj & 1) ? -yh[e] : yh[e]) + 2.0 * acc[e]);
        stv<VEC>(zout, (long long)jj * N + p0 + tp, o);
      }
    }
  }
}

// Inverse transform from per-block sources: y_k = (tr_k + i ti_k) * src_k (planes of block k),
// z = Gamma^{-1} U y (real by construction). Used when P_max == 1 (y = w / theta), after the
// temporally blocked sweeps (y = x_{p_k}, passive blocks w / theta) and by the SP solver.
struct NcFinal {
  const double* src[AAC_MAX_BLK];   // first plane of block k in its source array
  double tr[AAC_MAX_BLK], ti[AAC_MAX_BLK];
};

template <int VEC>
__global__ void __launch_bounds__(256) k_inverse(long long N, Dft D, NcFinal F,
                                                 double* __restrict__ zbase, long long zjs,
                                                 const IterState* st) {
  if (st && st->done) return;
  double* z = zbase + (st ? (long long)st->j * zjs : 0LL);
  const unsigned bid = (c_rev & AAC_REV_INV) ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
  const long long p = ((long long)bid * blockDim.x + threadIdx.x) * VEC;
  if (p >= N) return;
  const int ell = D.ell, h = ell / 2;
  double yr[AAC_MAX_BLK][VEC], yi[AAC_MAX_BLK][VEC];
#pragma unroll
  for (int kb = 0; kb < AAC_MAX_BLK; ++kb) {       // all loads first
    if (kb > h) break;
    const bool cplx = (kb != 0 && kb != h);
    ldc<VEC>(F.src[kb], p, yr[kb]);
    if (cplx) ldc<VEC>(F.src[kb] + N, p, yi[kb]);
  }
#pragma unroll
  for (int kb = 0; kb < AAC_MAX_BLK; ++kb) {
    if (kb > h) break;
    const bool cplx = (kb != 0 && kb != h);
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const double w0 = yr[kb][e], w1 = cplx ? yi[kb][e] : 0.0;
      yr[kb][e] = w0 * F.tr[kb] - w1 * F.ti[kb];
      yi[kb][e] = cplx ? (w0 * F.ti[kb] + w1 * F.tr[kb]) : 0.0;
    }
  }
  for (int j = 0; j < ell; ++j) {
    double acc[VEC], o[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] = 0.0;
    int m = j;
#pragma unroll
    for (int kb = 1; kb < AAC_MAX_BLK; ++kb) {
      if (kb >= h) break;
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        acc[e] = fma(yr[kb][e], D.c[m], acc[e]);
        acc[e] = fma(-yi[kb][e], D.s[m], acc[e]);
      }
      m += j;
      if (m >= ell) m -= ell;
    }
    const double f = D.scale * D.gi[j];
#pragma unroll
    for (int e = 0; e < VEC; ++e) o[e] = f * (yr[0][e] + ((j & 1) ? -yr[h][e] : yr[h][e]) + 2.0 * acc[e]);
    stv<VEC>(z + (long long)j * N, p, o);
  }
}

// k_inverse with ell == ELL at compile time (static twiddle indices, all planes in registers).
template <int ELL>
__global__ void __launch_bounds__(256) k_inverse_exact(long long N, Dft D, NcFinal F,
                                                       double* __restrict__ zbase, long long zjs,
                                                       const IterState* st) {
  if (st && st->done) return;
  double* z = zbase + (st ? (long long)st->j * zjs : 0LL);
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  constexpr int h = ELL / 2;
  double yr[h + 1], yi[h + 1];
#pragma unroll
  for (int kb = 0; kb <= h; ++kb) {                // all loads first
    yr[kb] = F.src[kb][p];
    yi[kb] = (kb != 0 && kb != h) ? F.src[kb][N + p] : 0.0;
  }
#pragma unroll
  for (int kb = 0; kb <= h; ++kb) {
    const double a = yr[kb], b = yi[kb];
    yr[kb] = a * F.tr[kb] - b * F.ti[kb];
    yi[kb] = (kb != 0 && kb != h) ? (a * F.ti[kb] + b * F.tr[kb]) : 0.0;
  }
#pragma unroll
  for (int j = 0; j < ELL; ++j) {
    double acc = 0.0;
#pragma unroll
    for (int kb = 1; kb < h; ++kb) {
      acc = fma(yr[kb], D.c[(j * kb) % ELL], acc);
      acc = fma(-yi[kb], D.s[(j * kb) % ELL], acc);
    }
    z[(long long)j * N + p] = D.scale * D.gi[j] * (yr[0] + ((j & 1) ? -yr[h] : yr[h]) + 2.0 * acc);
  }
}
