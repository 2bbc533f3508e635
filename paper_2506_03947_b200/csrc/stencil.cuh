// stencil.cuh -- the variable-coefficient 3/5/7-point operator A (device side).
//
// (A u)_P = u_P + sum_{interior faces f of P} w_f (u_P - u_nb(f)),  w_f = c kappa_f n_a^2
// (BASELINE.json operator; readings R2/R3). Zero-flux Neumann boundaries carry
// w_f = 0, so a boundary neighbour is replaced by u_P itself (contribution exactly 0, no
// out-of-range load). Across the slab axis the neighbour comes from the halo layer of the
// adjacent rank.
#pragma once

#include "aac_internal.cuh"

template <int DIM>
struct Pt {
  long long p;
  int x, y, z;
  long long li;                      // index inside the slab layer (for halo reads)
  double wxm, wxp, wym, wyp, wzm, wzp;
};

template <int DIM>
__device__ __forceinline__ void load_pt(const Geo& g, long long p, Pt<DIM>& q) {
  q.p = p;
  q.x = (int)(p % g.nx);
  long long r = p / g.nx;
  q.y = (int)(r % g.ny);
  q.z = (int)(r / g.ny);
  q.li = p % g.S;
  q.wxm = __ldg(g.wx + p);
  q.wxp = __ldg(g.wx + p + 1);
  if (DIM >= 2) {
    q.wym = __ldg(g.wy + p);
    q.wyp = __ldg(g.wy + p + g.nx);
  } else {
    q.wym = q.wyp = 0.0;
  }
  if (DIM >= 3) {
    q.wzm = __ldg(g.wz + p);
    q.wzp = __ldg(g.wz + p + g.S);
  } else {
    q.wzm = q.wzp = 0.0;
  }
}

// (A u)_p for one plane u (base pointer of the plane); hlo / hhi = this plane's halo layers.
template <int DIM>
__device__ __forceinline__ double apply_A(const Geo& g, const Pt<DIM>& q,
                                          const double* __restrict__ u,
                                          const double* __restrict__ hlo,
                                          const double* __restrict__ hhi) {
  const double u0 = u[q.p];
  const double xm = (q.x > 0) ? u[q.p - 1] : u0;
  const double xp = (q.x < g.nx - 1) ? u[q.p + 1] : u0;
  double acc = u0;
  acc = fma(q.wxm, u0 - xm, acc);
  acc = fma(q.wxp, u0 - xp, acc);
  if (DIM == 2) {                    // y is the slab axis
    const double ym = (q.y > 0) ? u[q.p - g.nx] : (g.has_lo ? hlo[q.li] : u0);
    const double yp = (q.y < g.ny - 1) ? u[q.p + g.nx] : (g.has_hi ? hhi[q.li] : u0);
    acc = fma(q.wym, u0 - ym, acc);
    acc = fma(q.wyp, u0 - yp, acc);
  }
  if (DIM == 3) {                    // z is the slab axis
    const double ym = (q.y > 0) ? u[q.p - g.nx] : u0;
    const double yp = (q.y < g.ny - 1) ? u[q.p + g.nx] : u0;
    const double zm = (q.z > 0) ? u[q.p - g.S] : (g.has_lo ? hlo[q.li] : u0);
    const double zp = (q.z < g.nz - 1) ? u[q.p + g.S] : (g.has_hi ? hhi[q.li] : u0);
    acc = fma(q.wym, u0 - ym, acc);
    acc = fma(q.wyp, u0 - yp, acc);
    acc = fma(q.wzm, u0 - zm, acc);
    acc = fma(q.wzp, u0 - zp, acc);
  }
  return acc;
}

// ------------------------------------------------------------------------------------------
// y = calA x over all ell planes: y_0 = A x_0, y_j = A x_j - x_{j-1}.
// One thread per spatial point; the face weights are loaded once and reused for all planes.
template <int DIM>
__global__ void __launch_bounds__(256) k_matvec(Geo g, int ell, const double* __restrict__ x,
                                                double* __restrict__ y,
                                                const double* __restrict__ hlo,
                                                const double* __restrict__ hhi) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.N) return;
  Pt<DIM> q;
  load_pt<DIM>(g, p, q);
  double prev = 0.0;
  for (int j = 0; j < ell; ++j) {
    const double* u = x + (long long)j * g.N;
    const double ax = apply_A<DIM>(g, q, u, hlo + j * g.S, hhi + j * g.S);
    y[(long long)j * g.N + p] = ax - prev;
    prev = u[p];
  }
}
