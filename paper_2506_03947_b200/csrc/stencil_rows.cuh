// stencil_rows.cuh -- the calA apply (operator A of stencil.cuh) as a row-marching
// kernel for 2D grids with even nx.
//
// k_matvec (stencil.cuh) gives every thread one 2-point group of one row and loads the north and
// south rows again for every row: 3 row requests per row and plane from L1/L2, each issued after
// the previous plane pair's arithmetic. Here a thread owns a 2-column group over RY consecutive rows
// and keeps, per plane, the rows y - 1 and y in registers; each row step first issues the loads of
// row y + 1 of all ell planes (ell 16-byte loads in flight per thread), so every plane row is
// requested once per chunk (+ the two boundary rows of the chunk). x-neighbours come from the
// adjacent lanes by warp shuffles (a load only at the warp edges). The arithmetic is stencil_sv's, operation for operation (same fma order): results are
// bit-identical to k_matvec. Opt-in (AAC_MATVEC_ROWS=1): measured slower than k_matvec (aac.cu,
// matvec_rows_ry).
#pragma once

#include "stencil.cuh"

#ifndef MR_NT
#define MR_NT 128                                       // threads per CTA (2 columns each)
#endif
#ifndef MR_MINB
#define MR_MINB 3                                       // resident CTAs per SM (register cap 168:
#endif                                                  // ell = 10 without spills)

__device__ __forceinline__ double2 mr_ld2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

// Rows -1 and ny are the halo layers of the neighbouring slabs (several ranks), else absent: the
// neighbour then aliases the centre (zero-flux face, w = 0, contribution exactly 0 as in nbr()).
template <int ELL>
__global__ void __launch_bounds__(MR_NT, ELL >= 12 ? 2 : MR_MINB) k_matvec_rows(Geo g, const double* __restrict__ xbase, long long xjs,
                                                       const int* jdev, double* __restrict__ y,
                                                       const double* __restrict__ hlo,
                                                       const double* __restrict__ hhi, int ry) {
  if (jdev && jdev[1]) return;                    // IterState {j, done, ...}: done
  const double* x = xbase + (jdev ? (long long)jdev[0] * xjs : 0LL);
  const int nx = g.nx, ny = g.ny;
  const long long N = g.N, S = g.S;
  const int lane = threadIdx.x & 31;
  const int x0 = (blockIdx.x * MR_NT + threadIdx.x) * 2;
  const bool act = x0 < nx;                       // inactive lanes still take part in the shuffles
  const int xc = act ? x0 : nx - 2;               // (and load a valid address)
  const int ya = blockIdx.y * ry, yb = min(ya + ry, ny);
  const bool has_lo = g.has_lo, has_hi = g.has_hi;
  auto valid = [&](int r) { return (r >= 0 && r < ny) || (r == -1 && has_lo) || (r == ny && has_hi); };
  auto src = [&](int j, int r) -> const double* {
    if (r < 0) return hlo + (long long)j * S + xc;
    if (r >= ny) return hhi + (long long)j * S + xc;
    return x + (long long)j * N + (long long)r * nx + xc;
  };
  double2 rm[ELL], rc[ELL];
  const bool vm = valid(ya - 1);
#pragma unroll
  for (int j = 0; j < ELL; ++j) {
    rc[j] = mr_ld2(src(j, ya));
    if (vm) rm[j] = mr_ld2(src(j, ya - 1));
  }
#pragma unroll
  for (int j = 0; j < ELL; ++j)
    if (!vm) rm[j] = rc[j];
  long long pw = (long long)ya * nx + xc;
  double2 wym = mr_ld2(g.wy + pw);                 // lower y faces of row ya (wy padded: row ny = 0)
  for (int r = ya; r < yb; ++r) {
    // the south row r + 1 of every plane (or the centre: zero-flux face) and row r's weights
    const bool vs = valid(r + 1);
    double2 rp[ELL];
#pragma unroll
    for (int j = 0; j < ELL; ++j) rp[j] = vs ? mr_ld2(src(j, r + 1)) : rc[j];
    const double2 wxa = mr_ld2(g.wx + pw);          // lower x faces of the two points
    const double wxe = __ldg(g.wx + pw + 2);        // upper x face of the second
    const double2 wyp = mr_ld2(g.wy + pw + nx);     // upper y faces
    double dbd0 = 0.0, dbd1 = 0.0;                 // Dirichlet boundary faces (0: Neumann)
    if (g.dir) {
      dbd0 = dirichlet_diag<2>(g, xc, r, 0);
      dbd1 = dirichlet_diag<2>(g, xc + 1, r, 0);
    }
    const long long pr = (long long)r * nx + xc;
    double prev0 = 0.0, prev1 = 0.0;
#pragma unroll
    for (int j = 0; j < ELL; ++j) {
      const double2 c = rc[j];
      double l = __shfl_up_sync(0xffffffffu, c.y, 1);
      double e = __shfl_down_sync(0xffffffffu, c.x, 1);
      if (lane == 0) l = (xc > 0) ? __ldg(x + (long long)j * N + pr - 1) : c.x;
      if (lane == 31 || xc + 2 >= nx) e = (xc + 2 < nx) ? __ldg(x + (long long)j * N + pr + 2) : c.y;
      // stencil_sv, e = 0 then e = 1
      double a0 = c.x;
      a0 = fma(wxa.x, c.x - l, a0);
      a0 = fma(wxa.y, c.x - c.y, a0);
      a0 = fma(wym.x, c.x - rm[j].x, a0);
      a0 = fma(wyp.x, c.x - rp[j].x, a0);
      a0 = fma(dbd0, c.x, a0);
      double a1 = c.y;
      a1 = fma(wxa.y, c.y - c.x, a1);
      a1 = fma(wxe, c.y - e, a1);
      a1 = fma(wym.y, c.y - rm[j].y, a1);
      a1 = fma(wyp.y, c.y - rp[j].y, a1);
      a1 = fma(dbd1, c.y, a1);
      a0 -= prev0;
      a1 -= prev1;
      prev0 = c.x;
      prev1 = c.y;
      if (act) *reinterpret_cast<double2*>(y + (long long)j * N + pr) = make_double2(a0, a1);
    }
#pragma unroll
    for (int j = 0; j < ELL; ++j) {
      rm[j] = rc[j];
      rc[j] = rp[j];
    }
    wym = wyp;                                     // upper face of row r = lower face of r + 1
    pw += nx;
  }
}
