// exact.cuh -- the exact block alpha-circulant preconditioner P_alpha^{-1} at scale for the
// paper's operator. A = I - (nu/h^2) L with Dirichlet faces on a square
// n x n grid is diagonalised by the orthonormal DST-I S (Appendix A):
//   A = S diag(mu) S,  mu_ij = 1 + w (l_i + l_j),  l_i = 4 sin^2(pi (i+1) / (2 (n+1))),
// so each block problem (A - Lambda_k) y_k = w_k (Eq. eq:blockproblem) is solved exactly:
//   y_k = S ((S W_k S) ./ (mu - Lambda_k)) S      (W_k = block k as an n x n matrix).
// The two-sided transforms are dense n x n x n products per plane -- the one dense contraction
// on any path of this library -- so they run on the fp64 tensor cores: k_dst_gemm, a batched
// DMMA (mma.sync m8n8k4 f64) GEMM written here (scripts/ubench_dmma.cu: DMMA sustains 36.6
// TFLOP/s on the B200, the full fp64 rate, where a DFMA with three register operands is capped
// near 62% of it by register-file bank reads). The spectral division is k_exact_scale.
#pragma once

#include "krylov.cuh"

struct ExactShifts {
  double lr[AAC_MAX_BLK], li[AAC_MAX_BLK];
};

// Spectral division of the packed Fourier planes (DST domain): real blocks divide by
// mu_xy - Lambda_k, complex blocks by the complex mu_xy - Lambda_k (plane pair Re, Im).
__global__ void __launch_bounds__(256) k_exact_scale(int n, int ell, const double* __restrict__ lam1d,
                                                     double* __restrict__ X, ExactShifts Sh,
                                                     const IterState* st) {
  if (st && st->done) return;
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

// ------------------------------------------------------------------------------------------
// C_b = A_b B_b for b = blockIdx.z (row-major n x n; sa / sb = 0: one matrix shared by the
// batch). CTA tile 64 x TN (4 warps in 2 x 2, each 32 x TN/2 = 4 x TN/16 DMMA tiles of 8 x 8), k
// in chunks of 16 through double-buffered shared memory (the next chunk is loaded into registers
// while the current one is multiplied). Fragments of m8n8k4 (PTX ISA): thread t holds A[t/4][t%4],
// B[t%4][t/4] and C[t/4][2(t%4) + {0,1}]. Shared-memory row strides 20 / TN + 8 doubles make
// every 64-bit fragment load two conflict-free wavefronts (the minimum for 256 bytes).
constexpr int DG_T = 64, DG_K = 16, DG_AS = DG_K + 4;

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int TN>
__global__ void __launch_bounds__(128) k_dst_gemm(int n, const double* __restrict__ A, long long sa,
                                                  const double* __restrict__ B, long long sb,
                                                  double* __restrict__ C, long long sc, const IterState* st) {
  constexpr int BS = TN + 8, NJ = TN / 16, NB = DG_K * TN / 128;   // B values per thread and chunk
  if (st && st->done) return;
  __shared__ __align__(16) double As[2][DG_T][DG_AS];
  __shared__ __align__(16) double Bs[2][DG_K][BS];
  const int b = blockIdx.z;
  A += (long long)b * sa;
  B += (long long)b * sb;
  C += (long long)b * sc;
  const int m0 = blockIdx.y * DG_T, n0 = blockIdx.x * TN;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * (TN / 2);
  const int gr = lane >> 2, gc = lane & 3;
  double acc[4][NJ][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // global -> registers: A chunk 64 x 16 (8 per thread), B chunk 16 x TN (NB per thread)
  double ra[8], rb[NB];
  auto gload = [&](int k0) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int ia = t + u * 128;                       // A: row ia / 16, col ia % 16
      const int ar = m0 + (ia >> 4), ac = k0 + (ia & 15);
      ra[u] = (ar < n && ac < n) ? __ldg(A + (long long)ar * n + ac) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int ib = t + u * 128;                       // B: row ib / TN, col ib % TN
      const int br = k0 + ib / TN, bc = n0 + ib % TN;
      rb[u] = (br < n && bc < n) ? __ldg(B + (long long)br * n + bc) : 0.0;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int ia = t + u * 128;
      As[buf][ia >> 4][ia & 15] = ra[u];
    }
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int ib = t + u * 128;
      Bs[buf][ib / TN][ib % TN] = rb[u];
    }
  };
  const int nk = (n + DG_K - 1) / DG_K;
  gload(0);
  sstore(0);
  __syncthreads();
  for (int kc = 0; kc < nk; ++kc) {
    const int cur = kc & 1;
    if (kc + 1 < nk) gload((kc + 1) * DG_K);
#pragma unroll
    for (int kk = 0; kk < DG_K; kk += 4) {
      double fa[4], fb[NJ];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = As[cur][wm + i * 8 + gr][kk + gc];
#pragma unroll
      for (int j = 0; j < NJ; ++j) fb[j] = Bs[cur][kk + gc][wn + j * 8 + gr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma884(acc[i][j], fa[i], fb[j]);
    }
    if (kc + 1 < nk) {
      sstore(cur ^ 1);
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm + i * 8 + gr;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = n0 + wn + j * 8 + 2 * gc;
      if (c < n) C[(long long)r * n + c] = acc[i][j][0];
      if (c + 1 < n) C[(long long)r * n + c + 1] = acc[i][j][1];
    }
  }
}
