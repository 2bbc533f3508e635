// krylov.cuh -- flexible GMRES building blocks (BASELINE.json north_star; not in the paper).
//
// Arnoldi with CGS2 (reading R14) organised for HBM traffic:
//   * the basis is stored UNNORMALISED (V_i raw, sigma_i = 1/||V_i||), so the update that
//     forms the next vector u = w - V c can be fused into the next preconditioner's forward
//     transform (k_forward<UPD>) without waiting for ||u||;
//   * pass 1 (k_arnoldi, fused with the calA apply): s = V^T w and the new Gram column
//     V^T v_j in ONE read of the basis; the second CGS pass is formed algebraically,
//     h2 = V^T (w - V h1) = h1 - G h1 with G = V^T V the (normalised) Gram matrix, which is
//     identical to classical CGS2 in exact arithmetic; c = h1 + h2 is column j of H;
//   * every reduction is per-CTA partials + a fixed-order sum in the LAST CTA (bitwise
//     reproducible), followed by the scalar algebra (Givens, residual estimate, flags) on
//     the device: no host round trip inside an Arnoldi step.
// Multi-rank: the last CTA only reduces locally; an NCCL all-reduce and k_scalar_* follow.
#pragma once

#include "aac_internal.cuh"

struct IterState {
  int j;            // column under construction
  int done;         // 1: converged / breakdown / maxit -> every iteration kernel returns
  int m;            // completed Arnoldi columns
  int maxit;
  unsigned tick;    // last-CTA ticket (reset by the last CTA)
  unsigned pad;
  double beta;      // ||b||
  double relres;    // |g_m| / beta
  double rtol;
  double hn;        // last H[j+1, j]
};

// Publish n 32-bit words of device state into pinned (mapped) host memory from a kernel: the
// host reads it after an event / stream sync. Unlike a D2H memcpy this needs no copy engine, so
// the per-step poll never queues behind a large host transfer on another stream
// (aac_gmres_host_batch moves whole vectors in and out while the solves run).
// Programmatic dependent launch (PDL): a kernel launched with the programmatic-serialisation
// attribute may start while its predecessor drains; it waits here for the predecessor's completion
// (and memory flush) before touching anything, then lets its own successor launch. A no-op for
// kernels launched normally.
#ifndef GRIDDEP_EARLY
#define GRIDDEP_EARLY 1
#endif
__device__ __forceinline__ void griddep() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (GRIDDEP_EARLY) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void k_publish(const unsigned* __restrict__ src, unsigned* dst, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// Solve start without copy engines (see k_publish): the state from a kernel argument, V_0 = b.
__global__ void k_set_state(IterState* st, IterState v) { *st = v; }
__global__ void __launch_bounds__(256) k_copy(const double* __restrict__ src, double* __restrict__ dst,
                                              long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

struct ArnoldiCtx {
  IterState* st;
  double* H;        // (ldh x max_krylov) column-major, ldh = max_krylov + 1
  int ldh;
  double* cs;       // Givens cosines
  double* sn;       // Givens sines
  double* g;        // rotated rhs
  double* sigma;    // 1/||V_i raw||
  double* c;        // CGS2 coefficients of the pending column (normalised basis)
  double* G;        // Gram matrix (ldh x ldh)
  double* red;      // multi-rank: locally reduced raw sums before the all-reduce
  int local_only;   // 1 when nranks > 1
  unsigned* pub;    // graph replay on one rank: the last CTA of k_arnoldi copies the IterState here
                    // (host-mapped pinned memory) itself -- no k_publish node at the end of the step
  int one_reduce;   // 1: lagged normalisation -- ||V_j||^2 is taken from the Gram column of the
                    // projection pass (one reduction / all-reduce per Arnoldi step), see below
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// s = sum over c = start, start + step, ... < n of base[c * stride], in ascending c (the order of the
// plain loop), with the loads issued KU at a time: the values were written by other CTAs and sit
// in L2, and a loop that adds each value before loading the next pays one L2 round trip per value.
template <int KU = 8>
__device__ __forceinline__ double strided_sum_ordered(const double* base, long long stride, int start, int step,
                                                      int n) {
  double s = 0.0;
  int c = start;
  for (; c + (KU - 1) * step < n; c += KU * step) {
    double v[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) v[u] = __ldcg(base + (long long)(c + u * step) * stride);
#pragma unroll
    for (int u = 0; u < KU; ++u) s += v[u];
  }
  for (; c < n; c += step) s += __ldcg(base + (long long)c * stride);
  return s;
}

// Fixed-order sum of n values by one CTA (lane-strided, warp tree, warps in order).
__device__ double block_sum_fixed(const double* v, int n) {
  __shared__ double wsum[32];
  // written by other CTAs: bypass L1 (loads batched, same order as a plain strided loop)
  double s = strided_sum_ordered(v, 1, threadIdx.x + threadIdx.y * blockDim.x, blockDim.x * blockDim.y, n);
  s = warp_sum(s);
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int nw = (blockDim.x * blockDim.y + 31) >> 5;
  if ((tid & 31) == 0) wsum[tid >> 5] = s;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += wsum[w];
  __syncthreads();
  return t;
}

// ||u||^2 of the vector just formed: j == 0 -> beta; else H[j, j-1] and Givens of column j-1.
__device__ void arnoldi_norm_step(const ArnoldiCtx& ac, int j, double nrm2) {
  IterState* st = ac.st;
  const double nu = sqrt(nrm2);
  ac.sigma[j] = nu > 0.0 ? 1.0 / nu : 0.0;
  if (j == 0) {
    st->beta = nu;
    ac.g[0] = nu;
    st->relres = 1.0;
    st->m = 0;
    if (nu == 0.0) {
      st->relres = 0.0;
      st->done = 1;
    }
    return;
  }
  const int col = j - 1;
  double* h = ac.H + (long long)col * ac.ldh;
  for (int i = 0; i < j; ++i) h[i] = ac.c[i];
  h[j] = nu;
  for (int i = 0; i < col; ++i) {
    const double t = ac.cs[i] * h[i] + ac.sn[i] * h[i + 1];
    h[i + 1] = -ac.sn[i] * h[i] + ac.cs[i] * h[i + 1];
    h[i] = t;
  }
  const double r = hypot(h[col], h[col + 1]);
  ac.cs[col] = h[col] / r;
  ac.sn[col] = h[col + 1] / r;
  h[col] = r;
  h[col + 1] = 0.0;
  ac.g[col + 1] = -ac.sn[col] * ac.g[col];
  ac.g[col] = ac.cs[col] * ac.g[col];
  st->hn = nu;
  st->m = j;
  st->relres = fabs(ac.g[col + 1]) / st->beta;
  if (st->relres <= st->rtol || nu == 0.0 || j >= st->maxit) st->done = 1;
}

// arnoldi_norm_step by a whole CTA: the column's entries, cos and sin of the previous rotations
// are staged in shared memory by all threads, thread 0 runs the (inherently serial) rotation chain
// on them, and the column goes back to H in parallel. The serial version reloads h from global
// memory at every rotation (one L2 round trip per rotation in the last CTA's tail).
__device__ void arnoldi_norm_step_cta(const ArnoldiCtx& ac, int j, double nrm2) {
  constexpr int CAP = 256;
  __shared__ double sh_h[CAP + 2], sh_cs[CAP], sh_sn[CAP];
  if (j == 0 || j > CAP) {
    if (threadIdx.x == 0) arnoldi_norm_step(ac, j, nrm2);
    __syncthreads();
    return;
  }
  const int col = j - 1;
  for (int i = threadIdx.x; i < j; i += blockDim.x) sh_h[i] = ac.c[i];
  for (int i = threadIdx.x; i < col; i += blockDim.x) {
    sh_cs[i] = ac.cs[i];
    sh_sn[i] = ac.sn[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    IterState* st = ac.st;
    const double nu = sqrt(nrm2);
    ac.sigma[j] = nu > 0.0 ? 1.0 / nu : 0.0;
    double* h = sh_h;
    h[j] = nu;
    for (int i = 0; i < col; ++i) {
      const double t = sh_cs[i] * h[i] + sh_sn[i] * h[i + 1];
      h[i + 1] = -sh_sn[i] * h[i] + sh_cs[i] * h[i + 1];
      h[i] = t;
    }
    const double r = hypot(h[col], h[col + 1]);
    ac.cs[col] = h[col] / r;
    ac.sn[col] = h[col + 1] / r;
    h[col] = r;
    h[col + 1] = 0.0;
    ac.g[col + 1] = -ac.sn[col] * ac.g[col];
    ac.g[col] = ac.cs[col] * ac.g[col];
    st->hn = nu;
    st->m = j;
    st->relres = fabs(ac.g[col + 1]) / st->beta;
    if (st->relres <= st->rtol || nu == 0.0 || j >= st->maxit) st->done = 1;
  }
  __syncthreads();
  double* hc = ac.H + (long long)col * ac.ldh;
  for (int i = threadIdx.x; i <= j; i += blockDim.x) hc[i] = sh_h[i];
  __syncthreads();
}

// CGS2 coefficients of column j from the raw sums s_i = <V_i, W>, gg_i = <V_i, V_j>.
__device__ void arnoldi_cgs2_step(const ArnoldiCtx& ac, int j, const double* s, const double* gg) {
  const int ld = ac.ldh;
  const double sj = ac.sigma[j];
  double* h1 = ac.red + 2 * ld;              // scratch
  for (int i = 0; i <= j; ++i) {
    h1[i] = ac.sigma[i] * sj * s[i];
    const double gij = ac.sigma[i] * sj * gg[i];
    ac.G[(long long)j * ld + i] = gij;
    ac.G[(long long)i * ld + j] = gij;
  }
  for (int i = 0; i <= j; ++i) {             // h2 = h1 - G h1 ;  c = h1 + h2
    double t = 0.0;
    for (int k = 0; k <= j; ++k) t = fma(ac.G[(long long)k * ld + i], h1[k], t);
    ac.c[i] = h1[i] + (h1[i] - t);
  }
  ac.st->j = j + 1;
}

// The same CGS2 coefficients computed by all threads of the calling CTA (thread i: h1_i, the Gram
// entries (i, j), then c_i = h1_i + (h1_i - (G h1)_i) with the sum over k in ascending order, as the
// one-thread version): O(j) per thread instead of O(j^2) on one thread -- the serial form was
// the last CTA's tail of every Arnoldi launch (at the 2d256 config, 39 steps: ~9% of a solve).
__device__ void arnoldi_cgs2_step_cta(const ArnoldiCtx& ac, int j, const double* s, const double* gg) {
  const int ld = ac.ldh;
  const double sj = ac.sigma[j];
  double* h1 = ac.red + 2 * ld;              // scratch
  for (int i = threadIdx.x; i <= j; i += blockDim.x) {
    h1[i] = ac.sigma[i] * sj * s[i];
    const double gij = ac.sigma[i] * sj * gg[i];
    ac.G[(long long)j * ld + i] = gij;
    ac.G[(long long)i * ld + j] = gij;
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= j; i += blockDim.x) {
    double t = 0.0;
    for (int k = 0; k <= j; ++k) t = fma(ac.G[(long long)k * ld + i], h1[k], t);
    ac.c[i] = h1[i] + (h1[i] - t);
  }
  __syncthreads();
  if (threadIdx.x == 0) ac.st->j = j + 1;
}

// One-reduce Arnoldi step (not in the paper, GMRES is the north star's). The
// projection pass already measures the Gram column <V_i, V_j>, i <= j, whose last entry is
// ||V_j||^2 -- so the norm of the vector formed by the previous update need not be reduced on
// its own: its normalisation (beta or H[j, j-1], the Givens rotation of column j-1 and the
// convergence test) is lagged into the same reduction as column j's CGS2 coefficients. One
// all-reduce per step instead of two on several ranks; the price is that convergence of column
// j-1 is seen one preconditioner apply and calA apply later. In exact arithmetic identical to
// the two-reduction form (and to the oracle's literal CGS2).
__device__ void arnoldi_lagged_step(const ArnoldiCtx& ac, int j, const double* s, const double* gg) {
  arnoldi_norm_step(ac, j, gg[j]);
  arnoldi_cgs2_step(ac, j, s, gg);
}

// Multi-rank scalar kernels (after the NCCL all-reduce of the local sums).
__global__ void k_scalar_norm(ArnoldiCtx ac) {
  if (ac.st->done) return;
  arnoldi_norm_step(ac, ac.st->j, ac.red[0]);
}
__global__ void k_scalar_cgs2(ArnoldiCtx ac) {       // one CTA
  const bool done = ac.st->done;                     // (read by every thread before thread 0's
  const int j = ac.st->j;                            //  norm step may set it)
  __syncthreads();
  if (done) return;
  if (ac.one_reduce) arnoldi_norm_step_cta(ac, j, ac.red[(j + 1) + j]);
  arnoldi_cgs2_step_cta(ac, j, ac.red, ac.red + (j + 1));
}

// y = R^{-1} g for the m x m upper-triangular rotated Hessenberg; y_i *= sigma_i so that
// x = sum_i y_i Z_i with the RAW preconditioned vectors Z_i = P^{-1} V_i(raw).
// One warp: row i's sum over k > i split over the lanes (lane-strided, then the warp tree), y_i by
// lane 0 -- m steps of a warp reduction instead of m^2 / 2 dependent global loads on one thread.
__global__ void k_backsub(const IterState* st, int ldh, const double* __restrict__ H,
                          const double* __restrict__ g, const double* __restrict__ sigma,
                          double* y) {
  const int m = st->m;
  const int lane = threadIdx.x & 31;
  for (int i = m - 1; i >= 0; --i) {
    double s = 0.0;
    for (int k = i + 1 + lane; k < m; k += 32) s = fma(H[(long long)k * ldh + i], y[k], s);
    s = warp_sum(s);
    if (lane == 0) y[i] = (g[i] - s) / H[(long long)i * ldh + i];
    __syncwarp();
  }
  for (int i = lane; i < m; i += 32) y[i] *= sigma[i];
}

// x = sum_{i<m} y[i] Z_i
__global__ void __launch_bounds__(256) k_lincomb(const double* __restrict__ Z, long long ldz,
                                                 const IterState* st, const double* __restrict__ y,
                                                 double* __restrict__ x, long long n) {
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (i >= n) return;
  const int m = st->m;
  double s0 = 0.0, s1 = 0.0;
  const bool two = i + 1 < n;
  for (int k = 0; k < m; ++k) {
    const double yk = y[k];
    const double* z = Z + (long long)k * ldz + i;
    s0 = fma(yk, z[0], s0);
    if (two) s1 = fma(yk, z[1], s1);
  }
  x[i] = s0;
  if (two) x[i + 1] = s1;
}

// part[cta] = sum over the CTA's elements of (a - b)^2   (b may be NULL)
__global__ void __launch_bounds__(256) k_diffnorm(const double* __restrict__ a,
                                                  const double* __restrict__ b, long long n,
                                                  double* __restrict__ part) {
  __shared__ double red[8];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double d = a[i] - (b ? b[i] : 0.0);
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

// out[0] = sum_c part[c] (fixed order, one CTA)
__global__ void __launch_bounds__(256) k_sum(const double* __restrict__ part, int n,
                                             double* __restrict__ out) {
  const double t = block_sum_fixed(part, n);
  if (threadIdx.x == 0) out[0] = t;
}
