// ci.cuh -- the paper's outer solver: Chebyshev semi-iteration on the left-preconditioned
// all-at-once system (PAPER.md:102-107 Eq. eq:precondsystem; foci Cor. cor:extremeevals,
// PAPER.md:204-210; stopping rule PAPER.md:647). SURVEY.md §8(f) N1 (paper-reproduction mode).
//   chi_{p+1} = chi_p + a_p (chi_p - chi_{p-1}) + c_p z_p,  z_p = P^{-1}(b - calA chi_p)
// with the three-term Chebyshev-acceleration coefficients of reading R8 (real theta, delta).
#pragma once

#include "krylov.cuh"

// In place: t = x; x = t + a (t - xp) + c z; xp = t.
__global__ void __launch_bounds__(256) k_ci_update(double* __restrict__ x, double* __restrict__ xp,
                                                   const double* __restrict__ z, double a, double c,
                                                   long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double t = x[i];
    x[i] = fma(c, z[i], fma(a, t - xp[i], t));
    xp[i] = t;
  }
}

// r = b - y and per-CTA partials of ||r||^2 (summed by k_sum in a fixed order).
__global__ void __launch_bounds__(256) k_ci_resid(const double* __restrict__ b, const double* __restrict__ y,
                                                  double* __restrict__ r, long long n,
                                                  double* __restrict__ part) {
  __shared__ double red[8];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double d = b[i] - y[i];
    r[i] = d;
    s = fma(d, d, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}
