// exact.cuh -- the exact block alpha-circulant preconditioner P_alpha^{-1} at scale for the
// paper's operator. A = I - (nu/h^2) L with Dirichlet faces on a square
// n x n grid is diagonalised by the orthonormal DST-I S (Appendix A):
//   A = S diag(mu) S,  mu_ij = 1 + w (l_i + l_j),  l_i = 4 sin^2(pi (i+1) / (2 (n+1))),
// so each block problem (A - Lambda_k) y_k = w_k (Eq. eq:blockproblem) is solved exactly:
//   y_k = S ((S W_k S) ./ (mu - Lambda_k)) S      (W_k = block k as an n x n matrix).
// The two-sided transforms are dense n x n x n products per plane: batched fp64 GEMMs through
// cuBLAS (a plain library GEMM, loaded at run time); the spectral division is a kernel.
#pragma once

#include <dlfcn.h>

#include "aac_internal.cuh"

struct CublasApi {
  void* h = nullptr;
  void* handle = nullptr;
  int (*Create)(void**) = nullptr;
  int (*Destroy)(void*) = nullptr;
  int (*SetStream)(void*, cudaStream_t) = nullptr;
  int (*DgemmStridedBatched)(void*, int, int, int, int, int, const double*, const double*, int, long long,
                             const double*, int, long long, const double*, double*, int, long long, int) = nullptr;
};

struct ExactShifts {
  double lr[AAC_MAX_BLK], li[AAC_MAX_BLK];
};

// Spectral division of the packed Fourier planes (DST domain): real blocks divide by
// mu_xy - Lambda_k, complex blocks by the complex mu_xy - Lambda_k (plane pair Re, Im).
__global__ void __launch_bounds__(256) k_exact_scale(int n, int ell, const double* __restrict__ lam1d,
                                                     double* __restrict__ X, ExactShifts Sh) {
  const long long N = (long long)n * n;
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int x = (int)(p % n), y = (int)(p / n);
  const double mu = 1.0 + lam1d[x] + lam1d[y];
  const int h = ell / 2;
  for (int kb = 0; kb <= h; ++kb) {
    const int q = kb == 0 ? 0 : (kb == h ? ell - 1 : 2 * kb - 1);
    const double dr = mu - Sh.lr[kb], di = -Sh.li[kb];
    if (kb == 0 || kb == h) {
      X[(long long)q * N + p] /= dr;
    } else {                                    // (a + i b) / (dr + i di)
      const double a = X[(long long)q * N + p], b = X[(long long)(q + 1) * N + p];
      const double den = dr * dr + di * di;
      X[(long long)q * N + p] = (a * dr + b * di) / den;
      X[(long long)(q + 1) * N + p] = (b * dr - a * di) / den;
    }
  }
}
