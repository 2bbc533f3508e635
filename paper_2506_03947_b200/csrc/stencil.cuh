// stencil.cuh -- the variable-coefficient 3/5/7-point operator A (device side).
//
// (A u)_P = u_P + sum_{interior faces f of P} w_f (u_P - u_nb(f)),  w_f = c kappa_f n_a^2
// (BASELINE.json operator; readings R2/R3). Zero-flux Neumann boundaries carry
// w_f = 0, so a boundary neighbour is replaced by u_P itself (contribution exactly 0, no
// out-of-range load). Across the slab axis the neighbour comes from the halo layer of the
// adjacent rank.
//
// Every thread owns VEC consecutive points along x (VEC = 2 when nx is even: 16-byte
// loads of the centre / north / south values and of the face weights).
#pragma once

#include "aac_internal.cuh"

template <int VEC>
__device__ __forceinline__ void ldv(const double* __restrict__ u, long long p, double* out) {
  if constexpr (VEC == 2) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(u + p));
    out[0] = t.x;
    out[1] = t.y;
  } else {
    out[0] = __ldg(u + p);
  }
}

// Plain (coherent) load: for buffers written earlier in the same kernel sequence.
template <int VEC>
__device__ __forceinline__ void ldc(const double* u, long long p, double* out) {
  if constexpr (VEC == 2) {
    const double2 t = *reinterpret_cast<const double2*>(u + p);
    out[0] = t.x;
    out[1] = t.y;
  } else {
    out[0] = u[p];
  }
}

template <int VEC>
__device__ __forceinline__ void stv(double* u, long long p, const double* v) {
  if constexpr (VEC == 2) {
    *reinterpret_cast<double2*>(u + p) = make_double2(v[0], v[1]);
  } else {
    u[p] = v[0];
  }
}

// Store with an L2 cache-hint policy (createpolicy): w = calA Z_j kept in L2 (evict_last) for the
// two kernels that read it next.
template <int VEC>
__device__ __forceinline__ void stv_hint(double* u, long long p, const double* v, uint64_t pol) {
  if constexpr (VEC == 2) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(u + p), "d"(v[0]), "d"(v[1]), "l"(pol)
                 : "memory");
  } else {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(u + p), "d"(v[0]), "l"(pol) : "memory");
  }
}

// Geometry + face weights of the VEC points p .. p+VEC-1 (same row).
template <int DIM, int VEC>
struct PtV {
  long long p, li;
  int x, y, z;
  double wx[VEC + 1];             // lower x-faces of the VEC points, then the last upper face
  double wym[VEC], wyp[VEC], wzm[VEC], wzp[VEC];
  double dbd[VEC];                // Dirichlet boundary-face diagonal (0 for Neumann)
};

// Dirichlet boundary faces of the point (x, y, z) on the physical boundary (paper operator,
// PAPER.md:630-637 Eq. IminusLap): sum of bd_a over its faces to a zero ghost value.
template <int DIM>
__device__ __forceinline__ double dirichlet_diag(const Geo& g, int x, int y, int z) {
  double d = g.bdx * ((x == 0) + (x == g.nx - 1));
  if constexpr (DIM == 2) d += g.bdy * ((y == 0 && !g.has_lo) + (y == g.ny - 1 && !g.has_hi));
  if constexpr (DIM == 3) {
    d += g.bdy * ((y == 0) + (y == g.ny - 1));
    d += g.bdz * ((z == 0 && !g.has_lo) + (z == g.nz - 1 && !g.has_hi));
  }
  return d;
}

// Face weights of the VEC-point group at (x, y, z) (local slab coordinates).
template <int DIM, int VEC>
__device__ __forceinline__ void load_ptv_xyz(const Geo& g, int x, int y, int z, PtV<DIM, VEC>& q) {
  q.x = x;
  q.y = y;
  q.z = z;
  q.li = (long long)y * g.nx + x;                 // index inside the slab layer (3D); 2D: S = nx
  if (DIM == 2) q.li = x;
  q.p = ((long long)z * g.ny + y) * g.nx + x;
  const long long p = q.p;
  ldv<VEC>(g.wx, p, q.wx);
  q.wx[VEC] = __ldg(g.wx + p + VEC);
  if constexpr (DIM >= 2) {
    ldv<VEC>(g.wy, p, q.wym);
    ldv<VEC>(g.wy, p + g.nx, q.wyp);
  }
  if constexpr (DIM >= 3) {
    ldv<VEC>(g.wz, p, q.wzm);
    ldv<VEC>(g.wz, p + g.S, q.wzp);
  }
#pragma unroll
  for (int e = 0; e < VEC; ++e) q.dbd[e] = 0.0;
  if (g.dir) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) q.dbd[e] = dirichlet_diag<DIM>(g, x + e, y, z);
  }
}

// Same from a flat index (32-bit index arithmetic: slabs hold < 2^32 points).
template <int DIM, int VEC>
__device__ __forceinline__ void load_ptv(const Geo& g, long long p, PtV<DIM, VEC>& q) {
  const unsigned pp = (unsigned)p, nx = (unsigned)g.nx, ny = (unsigned)g.ny;
  const unsigned r = pp / nx;
  load_ptv_xyz<DIM, VEC>(g, (int)(pp - r * nx), (int)(r % ny), (int)(r / ny), q);
}

// Neighbour pointers of the VEC-point group for one plane (branch-free: boundary neighbours
// alias the centre, slab neighbours point into the halo layer). All loads of a stencil are
// then independent and issue back to back.
struct Nbr {
  const double* c;   // centre (VEC values)
  const double* w;   // west of the first point
  const double* e;   // east of the last point
  const double* n;   // y - 1   (VEC values)
  const double* s;   // y + 1
  const double* d;   // z - 1
  const double* u;   // z + 1
};

template <int DIM, int VEC>
__device__ __forceinline__ Nbr nbr(const Geo& g, const PtV<DIM, VEC>& q, const double* u,
                                   const double* hlo, const double* hhi) {
  Nbr b;
  b.c = u + q.p;
  b.w = (q.x > 0) ? b.c - 1 : b.c;
  b.e = (q.x + VEC < g.nx) ? b.c + VEC : b.c + (VEC - 1);
  b.n = b.s = b.d = b.u = b.c;
  if constexpr (DIM == 2) {
    b.n = (q.y > 0) ? b.c - g.nx : (g.has_lo ? hlo + q.li : b.c);
    b.s = (q.y < g.ny - 1) ? b.c + g.nx : (g.has_hi ? hhi + q.li : b.c);
  }
  if constexpr (DIM == 3) {
    b.n = (q.y > 0) ? b.c - g.nx : b.c;
    b.s = (q.y < g.ny - 1) ? b.c + g.nx : b.c;
    b.d = (q.z > 0) ? b.c - g.S : (g.has_lo ? hlo + q.li : b.c);
    b.u = (q.z < g.nz - 1) ? b.c + g.S : (g.has_hi ? hhi + q.li : b.c);
  }
  return b;
}

// Stencil operands of one plane at the VEC-point group (loads only: lets a kernel issue the
// loads of several planes before any arithmetic or store).
template <int VEC>
struct SV {
  double c[VEC], n[VEC], s[VEC], d[VEC], u[VEC];
  double w, e;
};

template <int DIM, int VEC>
__device__ __forceinline__ void load_sv(const Geo& g, const PtV<DIM, VEC>& q, const double* u,
                                        const double* hlo, const double* hhi, SV<VEC>& v) {
  const Nbr b = nbr<DIM, VEC>(g, q, u, hlo, hhi);
  ldc<VEC>(b.c, 0, v.c);
  v.w = *b.w;
  v.e = *b.e;
  if constexpr (DIM >= 2) {
    ldc<VEC>(b.n, 0, v.n);
    ldc<VEC>(b.s, 0, v.s);
  }
  if constexpr (DIM >= 3) {
    ldc<VEC>(b.d, 0, v.d);
    ldc<VEC>(b.u, 0, v.u);
  }
}

// out[e] = (A u)_{p+e} from loaded operands
template <int DIM, int VEC>
__device__ __forceinline__ void stencil_sv(const Geo& g, const PtV<DIM, VEC>& q, const SV<VEC>& v, double* out) {
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    const double l = e == 0 ? v.w : v.c[e - 1];
    const double r = e == VEC - 1 ? v.e : v.c[e + 1];
    const double c = v.c[e];
    double acc = c;
    acc = fma(q.wx[e], c - l, acc);
    acc = fma(q.wx[e + 1], c - r, acc);
    if constexpr (DIM >= 2) {
      acc = fma(q.wym[e], c - v.n[e], acc);
      acc = fma(q.wyp[e], c - v.s[e], acc);
    }
    if constexpr (DIM >= 3) {
      acc = fma(q.wzm[e], c - v.d[e], acc);
      acc = fma(q.wzp[e], c - v.u[e], acc);
    }
    acc = fma(q.dbd[e], c, acc);                   // Dirichlet boundary faces (0: Neumann)
    out[e] = acc;
  }
}

// out[e] = (A u)_{p+e}, centre[e] = u_{p+e}, e < VEC.
template <int DIM, int VEC>
__device__ __forceinline__ void apply_Av(const Geo& g, const PtV<DIM, VEC>& q, const double* u,
                                         const double* hlo, const double* hhi, double* out,
                                         double* centre) {
  SV<VEC> v;
  load_sv<DIM, VEC>(g, q, u, hlo, hhi, v);
  stencil_sv<DIM, VEC>(g, q, v, out);
#pragma unroll
  for (int e = 0; e < VEC; ++e) centre[e] = v.c[e];
}

// ------------------------------------------------------------------------------------------
// y = calA x over all ell planes: y_0 = A x_0, y_j = A x_j - x_{j-1}.
// x = xbase + j * xjs with j read on the device when st != NULL (GMRES mode: x = Z_j).
template <int DIM, int VEC>
__global__ void __launch_bounds__(256) k_matvec(Geo g, int ell, const double* __restrict__ xbase,
                                                long long xjs, const int* jdev,
                                                double* __restrict__ y,
                                                const double* __restrict__ hlo,
                                                const double* __restrict__ hhi) {
  if (jdev && jdev[1]) return;                    // IterState {j, done, ...}: done
  const double* x = xbase + (jdev ? (long long)jdev[0] * xjs : 0LL);
  // grid (x-chunks, ny, nz): no index division
  const int xx = (blockIdx.x * blockDim.x + threadIdx.x) * VEC;
  if (xx >= g.nx) return;
  // (GMRES step only: a stand-alone aac_matvec has no producer to walk against, and the descending
  //  row order alone measured 3% slower back to back -- 70.7 against 73.1% of the copy rate)
  const bool rev = jdev && (c_rev & AAC_REV_MATVEC);
  const bool keep = c_rev & AAC_L2_MATVEC_W;
  uint64_t pol = 0;
  if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  PtV<DIM, VEC> q;
  load_ptv_xyz<DIM, VEC>(g, xx, rev ? gridDim.y - 1 - blockIdx.y : blockIdx.y,
                         rev ? gridDim.z - 1 - blockIdx.z : blockIdx.z, q);
  const long long p = q.p;
  double prev[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) prev[e] = 0.0;
  // planes in pairs: the loads of both planes are in flight together
  for (int j = 0; j < ell; j += 2) {
    const bool two = j + 1 < ell;
    SV<VEC> v0, v1;
    load_sv<DIM, VEC>(g, q, x + (long long)j * g.N, hlo + j * g.S, hhi + j * g.S, v0);
    if (two) load_sv<DIM, VEC>(g, q, x + (long long)(j + 1) * g.N, hlo + (j + 1) * g.S, hhi + (j + 1) * g.S, v1);
    double a0[VEC], a1[VEC];
    stencil_sv<DIM, VEC>(g, q, v0, a0);
#pragma unroll
    for (int e = 0; e < VEC; ++e) a0[e] -= prev[e];
    if (keep) stv_hint<VEC>(y + (long long)j * g.N, p, a0, pol);
    else stv<VEC>(y + (long long)j * g.N, p, a0);
    if (two) {
      stencil_sv<DIM, VEC>(g, q, v1, a1);
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        a1[e] -= v0.c[e];
        prev[e] = v1.c[e];
      }
      if (keep) stv_hint<VEC>(y + (long long)(j + 1) * g.N, p, a1, pol);
      else stv<VEC>(y + (long long)(j + 1) * g.N, p, a1);
    }
  }
}
