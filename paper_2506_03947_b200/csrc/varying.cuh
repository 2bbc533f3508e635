// varying.cuh -- varying diagonal blocks A_1..A_ell (PAPER.md:991 Conclusions:
// "the block alpha-circulant preconditioner can be extended to a problem ... with varying
// diagonal blocks A_1, ..., A_ell using some 'representative' or average choice A_hat").
//   calA_var x:  y_0 = A_0 x_0, y_j = A_j x_j - x_{j-1}   (each block its own face weights),
//   P_alpha(A_hat), A_hat = (1/ell) sum_j A_j: A is affine in the face weights, so A_hat is the
//   operator of the averaged weights and every preconditioner kernel runs unchanged on it.
// GMRES only: the paper notes the eigenvalue bounds behind the outer CI no longer hold.
// Textually included by aac.cu.
#pragma once

// y = calA_var x over all ell planes; block j's face weights at wblk + j * wstride (the same
// padded wx | wy | wz layout as Geo). x = xbase + j_dev * xjs in GMRES mode (as k_matvec).
template <int DIM, int VEC>
__global__ void __launch_bounds__(256) k_matvec_var(Geo g, int ell, const double* __restrict__ xbase,
                                                    long long xjs, const int* jdev, double* __restrict__ y,
                                                    const double* __restrict__ wblk, long long wstride,
                                                    long long leny_off, long long lenz_off) {
  if (jdev && jdev[1]) return;                    // IterState {j, done, ...}: done
  const double* x = xbase + (jdev ? (long long)jdev[0] * xjs : 0LL);
  const int xx = (blockIdx.x * blockDim.x + threadIdx.x) * VEC;
  if (xx >= g.nx) return;
  double prev[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) prev[e] = 0.0;
  for (int j = 0; j < ell; ++j) {
    Geo gj = g;                                   // block j's operator
    gj.wx = wblk + (long long)j * wstride;
    gj.wy = gj.wx + leny_off;
    gj.wz = gj.wx + lenz_off;
    PtV<DIM, VEC> q;
    load_ptv_xyz<DIM, VEC>(gj, xx, blockIdx.y, blockIdx.z, q);
    SV<VEC> v;
    load_sv<DIM, VEC>(gj, q, x + (long long)j * g.N, nullptr, nullptr, v);
    double a[VEC];
    stencil_sv<DIM, VEC>(gj, q, v, a);
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      a[e] -= prev[e];
      prev[e] = v.c[e];
    }
    stv<VEC>(y + (long long)j * g.N, q.p, a);
  }
}

template <int DIM, int VEC>
static int launch_matvec_var(aac_ctx* ctx, const double* xbase, long long xjs, const int* jdev, double* y) {
  const Geo& g = ctx->geo;
  const long long wtot = ctx->wlen[0] + ctx->wlen[1] + ctx->wlen[2];
  const double V = 8.0 * ctx->ell * g.N, C = 8.0 * ctx->dim * g.N;
  const dim3 grid(grid1d(g.nx / VEC, 256), g.ny, g.nz);
  LAUNCH(ctx, KID_MATVEC, 2 * V + ctx->ell * C,
         (k_matvec_var<DIM, VEC><<<grid, 256, 0, ctx->stream>>>(g, ctx->ell, xbase, xjs, jdev, y, ctx->d_wblk, wtot,
                                                                ctx->wlen[0], ctx->wlen[0] + ctx->wlen[1])));
  return AAC_OK;
}

static int matvec_var(aac_ctx* ctx, const double* xbase, long long xjs, const int* jdev, double* y) {
  const bool v2 = (ctx->geo.nx % 2) == 0;
  switch (ctx->dim) {
    case 1: return v2 ? launch_matvec_var<1, 2>(ctx, xbase, xjs, jdev, y) : launch_matvec_var<1, 1>(ctx, xbase, xjs, jdev, y);
    case 2: return v2 ? launch_matvec_var<2, 2>(ctx, xbase, xjs, jdev, y) : launch_matvec_var<2, 1>(ctx, xbase, xjs, jdev, y);
    default: return v2 ? launch_matvec_var<3, 2>(ctx, xbase, xjs, jdev, y) : launch_matvec_var<3, 1>(ctx, xbase, xjs, jdev, y);
  }
}
