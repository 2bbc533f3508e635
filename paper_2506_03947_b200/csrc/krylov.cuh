// krylov.cuh -- flexible GMRES building blocks (BASELINE.json north_star; not in the paper).
//
// CGS2 (reading R14) as three streaming passes over the Krylov basis:
//   pass 1  h  = V^T w                         (k_mdot)
//   pass 2  w -= V h ;  h' = V^T w             (k_update<MODE_DOTS>, one read of V)
//   pass 3  w -= V h';  ||w||^2                (k_update<MODE_NORM>)
// Every pass writes per-CTA partial sums; k_reduce sums them in a FIXED order (the result
// is bitwise reproducible run to run). Scalars (Givens rotations, residual estimate, the
// triangular solve) stay on the device (single-thread kernels).
#pragma once

#include "aac_internal.cuh"

constexpr int KRY_THREADS = 256;
constexpr int KRY_E = 8;                        // elements per thread per CTA chunk
constexpr long long KRY_CHUNK = (long long)KRY_THREADS * KRY_E;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-reduce one value per thread into red[warp][i]; caller syncs and combines.
__device__ __forceinline__ void stash(double* red, int nv, int i, double v) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[(threadIdx.x >> 5) * nv + i] = v;
}

__device__ __forceinline__ void flush_partials(const double* red, int nv, double* part) {
  __syncthreads();
  const int nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w * nv + i];
    part[(long long)blockIdx.x * nv + i] = s;
  }
}

// part[cta][i] = sum over the CTA's chunk of V_i . w, i < nv
__global__ void __launch_bounds__(KRY_THREADS) k_mdot(const double* __restrict__ V, long long ldv,
                                                      int nv, const double* __restrict__ w,
                                                      long long n, double* __restrict__ part) {
  extern __shared__ double red[];
  const long long base = (long long)blockIdx.x * KRY_CHUNK + threadIdx.x;
  double wr[KRY_E];
#pragma unroll
  for (int e = 0; e < KRY_E; ++e) {
    const long long idx = base + (long long)e * KRY_THREADS;
    wr[e] = idx < n ? w[idx] : 0.0;
  }
  for (int i = 0; i < nv; ++i) {
    const double* v = V + (long long)i * ldv;
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < KRY_E; ++e) {
      const long long idx = base + (long long)e * KRY_THREADS;
      if (idx < n) acc = fma(v[idx], wr[e], acc);
    }
    stash(red, nv, i, acc);
  }
  flush_partials(red, nv, part);
}

enum { MODE_DOTS = 0, MODE_NORM = 1 };

// w_out = w_in - sum_i coef[i] V_i, then per-CTA partials of V^T w_out (MODE_DOTS) or of
// ||w_out||^2 (MODE_NORM, partial slot 0). w_out may be NULL (no store), nv may be 0.
template <int MODE>
__global__ void __launch_bounds__(KRY_THREADS) k_update(const double* __restrict__ V, long long ldv,
                                                        int nv, const double* __restrict__ coef,
                                                        double coef_sign,
                                                        const double* __restrict__ w_in,
                                                        double* __restrict__ w_out, long long n,
                                                        double* __restrict__ part) {
  extern __shared__ double red[];
  const long long base = (long long)blockIdx.x * KRY_CHUNK + threadIdx.x;
  double wr[KRY_E];
#pragma unroll
  for (int e = 0; e < KRY_E; ++e) {
    const long long idx = base + (long long)e * KRY_THREADS;
    wr[e] = idx < n ? w_in[idx] : 0.0;
  }
  for (int i = 0; i < nv; ++i) {
    const double* v = V + (long long)i * ldv;
    const double c = coef_sign * coef[i];
#pragma unroll
    for (int e = 0; e < KRY_E; ++e) {
      const long long idx = base + (long long)e * KRY_THREADS;
      if (idx < n) wr[e] = fma(-c, v[idx], wr[e]);
    }
  }
  if (w_out) {
#pragma unroll
    for (int e = 0; e < KRY_E; ++e) {
      const long long idx = base + (long long)e * KRY_THREADS;
      if (idx < n) w_out[idx] = wr[e];
    }
  }
  if (MODE == MODE_DOTS) {
    for (int i = 0; i < nv; ++i) {
      const double* v = V + (long long)i * ldv;
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < KRY_E; ++e) {
        const long long idx = base + (long long)e * KRY_THREADS;
        if (idx < n) acc = fma(v[idx], wr[e], acc);
      }
      stash(red, nv, i, acc);
    }
    flush_partials(red, nv, part);
  } else {
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < KRY_E; ++e) acc = fma(wr[e], wr[e], acc);
    stash(red, 1, 0, acc);
    flush_partials(red, 1, part);
  }
}

// out[i] = sum_c part[c][i] in a fixed order (one CTA per i).
__global__ void __launch_bounds__(256) k_reduce(const double* __restrict__ part, int nctas, int nv,
                                                double* __restrict__ out) {
  __shared__ double red[8];
  const int i = blockIdx.x;
  double s = 0.0;
  for (int c = threadIdx.x; c < nctas; c += blockDim.x) s += part[(long long)c * nv + i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    out[i] = t;
  }
}

// Status block layout (device d_stat, mirrored to pinned host):
enum {
  ST_RELRES = 0,   // |g_{j+1}| / beta
  ST_HNORM,        // H[j+1, j]
  ST_INV,          // 1 / H[j+1, j] (scale for v_{j+1}); 1/beta for v_0
  ST_BETA,         // ||b||
  ST_ONE,          // constant 1.0
  ST_NRM2,         // scratch: reduced squared norm
  ST_COUNT
};

// beta = sqrt(nrm2); g = (beta, 0, ...); inv = 1/beta.
__global__ void k_beta(const double* __restrict__ nrm2, double* __restrict__ stat,
                       double* __restrict__ g) {
  const double beta = sqrt(nrm2[0]);
  stat[ST_BETA] = beta;
  stat[ST_INV] = beta > 0.0 ? 1.0 / beta : 0.0;
  stat[ST_RELRES] = 1.0;
  stat[ST_ONE] = 1.0;
  g[0] = beta;
}

// Arnoldi column j: H[0..j, j] = h1 + h2, H[j+1, j] = ||w||; apply old rotations, form the
// new one (r = hypot, c = h_jj/r, s = h_{j+1,j}/r; reading R14) and update g.
__global__ void k_arnoldi(int j, int ldh, const double* __restrict__ h1,
                          const double* __restrict__ h2, const double* __restrict__ nrm2,
                          double* __restrict__ H, double* __restrict__ cs, double* __restrict__ sn,
                          double* __restrict__ g, double* __restrict__ stat) {
  double* col = H + (long long)j * ldh;
  for (int i = 0; i <= j; ++i) col[i] = h1[i] + h2[i];
  const double hn = sqrt(nrm2[0]);
  col[j + 1] = hn;
  for (int i = 0; i < j; ++i) {
    const double t = cs[i] * col[i] + sn[i] * col[i + 1];
    col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
    col[i] = t;
  }
  const double r = hypot(col[j], col[j + 1]);
  cs[j] = col[j] / r;
  sn[j] = col[j + 1] / r;
  col[j] = r;
  col[j + 1] = 0.0;
  g[j + 1] = -sn[j] * g[j];
  g[j] = cs[j] * g[j];
  stat[ST_HNORM] = hn;
  stat[ST_INV] = hn > 0.0 ? 1.0 / hn : 0.0;
  stat[ST_RELRES] = fabs(g[j + 1]) / stat[ST_BETA];
}

// y = R^{-1} g for the m x m upper-triangular rotated Hessenberg.
__global__ void k_backsub(int m, int ldh, const double* __restrict__ H, const double* __restrict__ g,
                          double* __restrict__ y) {
  for (int i = m - 1; i >= 0; --i) {
    double s = g[i];
    for (int k = i + 1; k < m; ++k) s -= H[(long long)k * ldh + i] * y[k];
    y[i] = s / H[(long long)i * ldh + i];
  }
}

// out = scale[0] * w
__global__ void __launch_bounds__(256) k_scale(const double* __restrict__ w,
                                               const double* __restrict__ scale,
                                               double* __restrict__ out, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = scale[0] * w[i];
}

// x = sum_i y[i] Z_i
__global__ void __launch_bounds__(256) k_lincomb(const double* __restrict__ Z, long long ldz, int m,
                                                 const double* __restrict__ y,
                                                 double* __restrict__ x, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int k = 0; k < m; ++k) s = fma(y[k], Z[(long long)k * ldz + i], s);
  x[i] = s;
}
