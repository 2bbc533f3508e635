// nc.cuh -- nested Chebyshev application of the block alpha-circulant preconditioner.
//
// P_alpha^{-1} r = (Gamma^{-1} U (x) I)(I (x) A - Lambda (x) I)^{-1}(U^* Gamma (x) I) r
// (PAPER.md:252-254 Eq. eq:Paform, pairing of reading R6), block problems
// (A - Lambda_k) y_k = w_k (Eq. eq:blockproblem) solved by p_k Chebyshev iterations
// (recurrence of reading R8).
//
// Packed half-complex layout: for real input the ell Fourier
// blocks satisfy w_{ell-k} = conj(w_k), so only k = 0..ell/2 are solved:
//   plane 0            = block 0 (real, Lambda_0 = alpha^{1/ell})
//   planes 2k-1, 2k    = Re, Im of block k, k = 1..ell/2-1
//   plane ell-1        = block ell/2 (real, Lambda = -alpha^{1/ell})
// i.e. ell real planes, the same bytes as the real block vector.
#pragma once

#include "stencil.cuh"

struct Dft {
  int ell;
  double g[AAC_MAX_ELL];     // gamma_j = alpha^{j/ell}
  double gi[AAC_MAX_ELL];    // 1/gamma_j
  double c[AAC_MAX_ELL];     // cos(2 pi m/ell)
  double s[AAC_MAX_ELL];     // sin(2 pi m/ell)
  double scale;              // ell^{-1/2}
};

// hat w = U^* Gamma r, packed. One thread per point, ell loads / ell stores.
__global__ void __launch_bounds__(256) k_forward(long long N, Dft D, const double* __restrict__ r,
                                                 double* __restrict__ what) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int ell = D.ell, h = ell / 2;
  double w[AAC_MAX_ELL];
#pragma unroll
  for (int j = 0; j < AAC_MAX_ELL; ++j)
    if (j < ell) w[j] = D.g[j] * r[(long long)j * N + p];
  // k = 0 and k = ell/2 (real)
  double s0 = 0.0, sh = 0.0;
#pragma unroll
  for (int j = 0; j < AAC_MAX_ELL; ++j)
    if (j < ell) {
      s0 += w[j];
      sh += (j & 1) ? -w[j] : w[j];
    }
  what[p] = D.scale * s0;
  what[(long long)(ell - 1) * N + p] = D.scale * sh;
  for (int k = 1; k < h; ++k) {
    double re = 0.0, im = 0.0;
    int m = 0;
#pragma unroll
    for (int j = 0; j < AAC_MAX_ELL; ++j)
      if (j < ell) {
        re = fma(w[j], D.c[m], re);
        im = fma(-w[j], D.s[m], im);
        m += k;
        if (m >= ell) m -= ell;
      }
    what[(long long)(2 * k - 1) * N + p] = D.scale * re;
    what[(long long)(2 * k) * N + p] = D.scale * im;
  }
}

// One Chebyshev step for every ACTIVE packed block at this global sweep.
struct NcBlk {
  int kind;                  // 0 inactive, 1 real (1 plane), 2 complex (2 planes)
  int q;                     // first plane of the block
  int first;                 // local step s == 1: x_1 = w/theta (virtual), x_0 = 0
  const double* xs;          // x_s, plane q (ignored when first)
  const double* xm;          // x_{s-1}, plane q (NULL when s <= 2: x_1 = w/theta is virtual)
  double* xo;                // x_{s+1}, plane q
  double ar, ai, br, bi;     // a_s = rho_s rho_{s-1}, b_s = 2 rho_s / delta (complex)
  double lr, li;             // Lambda_k
  double tr, ti;             // 1/theta_k
};
struct NcSweep {
  NcBlk b[AAC_MAX_BLK];
  int nblk;
};

template <int DIM>
__global__ void __launch_bounds__(256) k_sweep(Geo g, NcSweep P, const double* __restrict__ what,
                                               const double* __restrict__ hlo,
                                               const double* __restrict__ hhi) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.N) return;
  Pt<DIM> q;
  load_pt<DIM>(g, p, q);
  const long long N = g.N;
  for (int kb = 0; kb < P.nblk; ++kb) {
    const NcBlk& B = P.b[kb];
    if (B.kind == 0) continue;
    const double* wr = what + (long long)B.q * N;
    const double* hl = hlo + B.q * g.S;
    const double* hh = hhi + B.q * g.S;
    if (B.kind == 1) {
      double xs, Axs, xm;
      if (B.first) {
        xs = wr[p] * B.tr;
        Axs = apply_A<DIM>(g, q, wr, hl, hh) * B.tr;
        xm = 0.0;
      } else {
        xs = B.xs[p];
        Axs = apply_A<DIM>(g, q, B.xs, hl, hh);
        xm = B.xm ? B.xm[p] : wr[p] * B.tr;
      }
      const double res = wr[p] - (Axs - B.lr * xs);
      B.xo[p] = xs + B.ar * (xs - xm) + B.br * res;
    } else {
      const double* wi = wr + N;
      double ur, ui, Aur, Aui, mr, mi;
      if (B.first) {
        const double w0 = wr[p], w1 = wi[p];
        const double Aw0 = apply_A<DIM>(g, q, wr, hl, hh);
        const double Aw1 = apply_A<DIM>(g, q, wi, hl + g.S, hh + g.S);
        ur = w0 * B.tr - w1 * B.ti;
        ui = w0 * B.ti + w1 * B.tr;
        Aur = Aw0 * B.tr - Aw1 * B.ti;
        Aui = Aw0 * B.ti + Aw1 * B.tr;
        mr = mi = 0.0;
      } else {
        ur = B.xs[p];
        ui = B.xs[N + p];
        Aur = apply_A<DIM>(g, q, B.xs, hl, hh);
        Aui = apply_A<DIM>(g, q, B.xs + N, hl + g.S, hh + g.S);
        if (B.xm) {
          mr = B.xm[p];
          mi = B.xm[N + p];
        } else {                               // x_1 = w / theta
          const double w0 = wr[p], w1 = wi[p];
          mr = w0 * B.tr - w1 * B.ti;
          mi = w0 * B.ti + w1 * B.tr;
        }
      }
      // residual w - (A - Lambda) x
      const double rr = wr[p] - (Aur - (B.lr * ur - B.li * ui));
      const double ri = wi[p] - (Aui - (B.lr * ui + B.li * ur));
      const double dr = ur - mr, di = ui - mi;
      B.xo[p] = ur + (B.ar * dr - B.ai * di) + (B.br * rr - B.bi * ri);
      B.xo[N + p] = ui + (B.ar * di + B.ai * dr) + (B.br * ri + B.bi * rr);
    }
  }
}

// Final iterates y_k -> z = Gamma^{-1} U y (real by construction of the packing).
struct NcFinal {
  const double* y[AAC_MAX_BLK];   // x_{p_k} (plane q of the block) or NULL when p_k == 1
  double tr[AAC_MAX_BLK], ti[AAC_MAX_BLK];
  int nblk;
};

__global__ void __launch_bounds__(256) k_inverse(long long N, Dft D, NcFinal F,
                                                 const double* __restrict__ what,
                                                 double* __restrict__ z) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int ell = D.ell, h = ell / 2;
  double yr[AAC_MAX_BLK], yi[AAC_MAX_BLK];
  for (int kb = 0; kb <= h; ++kb) {
    const int q = (kb == 0) ? 0 : (kb == h ? ell - 1 : 2 * kb - 1);
    const bool cplx = (kb != 0 && kb != h);
    if (F.y[kb]) {
      yr[kb] = F.y[kb][p];
      yi[kb] = cplx ? F.y[kb][N + p] : 0.0;
    } else {
      const double w0 = what[(long long)q * N + p];
      const double w1 = cplx ? what[(long long)(q + 1) * N + p] : 0.0;
      yr[kb] = w0 * F.tr[kb] - w1 * F.ti[kb];
      yi[kb] = cplx ? (w0 * F.ti[kb] + w1 * F.tr[kb]) : 0.0;
    }
  }
  for (int j = 0; j < ell; ++j) {
    double acc = 0.0;
    int m = j;                                    // m = j*k mod ell
    for (int kb = 1; kb < h; ++kb) {
      acc = fma(yr[kb], D.c[m], acc);
      acc = fma(-yi[kb], D.s[m], acc);
      m += j;
      if (m >= ell) m -= ell;
    }
    const double u = yr[0] + ((j & 1) ? -yr[h] : yr[h]) + 2.0 * acc;
    z[(long long)j * N + p] = D.scale * u * D.gi[j];
  }
}
