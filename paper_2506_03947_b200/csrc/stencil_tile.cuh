// stencil_tile.cuh -- the calA apply (PAPER.md:35-46 Eq. eq:A: y_0 = A x_0, y_j = A x_j - x_{j-1})
// for 2D one-rank Neumann grids with TMA-staged tiles.
//
// k_matvec (stencil.cuh) loads every operand of a point through registers: the y-neighbours are
// separate 16-byte loads of the rows above and below (three L1/L2 requests per x value), and the
// bytes a thread can keep in flight are bounded by its registers. Here a tile of TR rows x TC
// columns of one plane, with its one-row / two-column halo, is copied row by row into shared
// memory by the bulk-copy engine (cp.async.bulk + mbarrier transaction counts, one issuing
// thread), through an NBUF-deep ring that runs across planes and tiles; the threads (one column
// each) read the five stencil operands from shared memory. The work is the flat sequence of
// (tile, plane) items split evenly over a persistent grid, so every CTA does the same number of
// plane tiles (+-1) whatever the tile count; a CTA starting mid-tile reloads x_{j-1} at its
// column. The face weights of a tile are loaded once per tile into registers (all planes share
// them). Operations per point in stencil_sv's order: results are bit-identical to k_matvec.
#pragma once

#include "tma.cuh"

constexpr int MT_TC = 256;                     // columns per tile = threads per CTA
constexpr int MT_TR = 8;                       // rows per tile
constexpr int MT_NBUF = 3;                     // ring depth (plane tiles)
constexpr int MT_SW = MT_TC + 4;               // smem row: columns c0 - 2 .. c0 + TC + 1

constexpr size_t mt_smem() {
  return (size_t)MT_NBUF * (MT_TR + 2) * MT_SW * sizeof(double) + MT_NBUF * sizeof(uint64_t) + 16;
}

struct MtGeo {
  int ntx, nty;                // tiles along x / y
  long long nitems;            // tiles x ell
};

// Issue the bulk copies of item `it` (tile-major, plane-minor) into ring slot `slot`.
__device__ __forceinline__ void mt_issue(const Geo& g, const MtGeo& M, int ell, const double* x, long long it,
                                         double* buf, uint64_t* bar) {
  const long long tile = it / ell;
  const int j = (int)(it % ell);
  const int ty = (int)(tile / M.ntx), tx = (int)(tile % M.ntx);
  const int r0 = ty * MT_TR, c0 = tx * MT_TC;
  const int cs = max(c0 - 2, 0), ce = min(c0 + MT_TC + 2, g.nx);
  const int ra = max(r0 - 1, 0), rb = min(r0 + MT_TR + 1, g.ny);
  const uint32_t rowb = (uint32_t)(ce - cs) * 8u;
  mbar_arrive_expect_tx(bar, rowb * (uint32_t)(rb - ra));
  const double* xp = x + (long long)j * g.N;
  for (int r = ra; r < rb; ++r)
    bulk_g2s(buf + (r - (r0 - 1)) * MT_SW + (cs - (c0 - 2)), xp + (long long)r * g.nx + cs, rowb, bar);
}

__global__ void __launch_bounds__(MT_TC, 2) k_matvec_tile(Geo g, MtGeo M, int ell, const double* __restrict__ xbase,
                                                          long long xjs, const int* jdev, double* __restrict__ y) {
  if (jdev && jdev[1]) return;                    // IterState {j, done, ...}: done
  const double* x = xbase + (jdev ? (long long)jdev[0] * xjs : 0LL);
  extern __shared__ __align__(16) unsigned char mt_raw[];
  double* ring = reinterpret_cast<double*>(mt_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + MT_NBUF * (MT_TR + 2) * MT_SW);
  const int t = threadIdx.x;
  // this CTA's items [i0, i1): the flat (tile, plane) sequence split evenly
  const long long per = M.nitems / gridDim.x, rem = M.nitems % gridDim.x;
  const long long bx = blockIdx.x;
  const long long i0 = bx * per + (bx < rem ? bx : rem);
  const long long i1 = i0 + per + (blockIdx.x < rem ? 1 : 0);
  if (t == 0) {
    for (int b = 0; b < MT_NBUF; ++b) mbar_init(&bars[b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (t == 0)
    for (int b = 0; b < MT_NBUF && i0 + b < i1; ++b)
      mt_issue(g, M, ell, x, i0 + b, ring + b * (MT_TR + 2) * MT_SW, &bars[b]);
  double wxl[MT_TR], wxr[MT_TR], wy[MT_TR + 1], prev[MT_TR];
  long long cur_tile = -1;
  for (long long it = i0; it < i1; ++it) {
    const long long k = it - i0;
    const int slot = (int)(k % MT_NBUF);
    const long long tile = it / ell;
    const int j = (int)(it % ell);
    const int ty = (int)(tile / M.ntx), tx = (int)(tile % M.ntx);
    const int r0 = ty * MT_TR, c0 = tx * MT_TC;
    const int xc = c0 + t;
    const bool colin = xc < g.nx;
    if (tile != cur_tile) {                       // face weights of the tile; x_{j-1} if mid-tile
      cur_tile = tile;
#pragma unroll
      for (int r = 0; r < MT_TR; ++r) {
        const int yr = r0 + r;
        const bool in = colin && yr < g.ny;
        const long long p = (long long)yr * g.nx + xc;
        wxl[r] = in ? __ldg(g.wx + p) : 0.0;
        wxr[r] = in ? __ldg(g.wx + p + 1) : 0.0;
        wy[r] = in ? __ldg(g.wy + p) : 0.0;
        prev[r] = (in && j > 0) ? __ldg(x + (long long)(j - 1) * g.N + p) : 0.0;
      }
      const int yr = r0 + MT_TR;
      wy[MT_TR] = (colin && yr - 1 < g.ny) ? __ldg(g.wy + (long long)yr * g.nx + xc) : 0.0;
    }
    mbar_wait(&bars[slot], (uint32_t)((k / MT_NBUF) & 1));
    const double* S = ring + slot * (MT_TR + 2) * MT_SW + 2 + t;   // column xc, smem row 0 = r0 - 1
    double* yp = y + (long long)j * g.N;
#pragma unroll
    for (int r = 0; r < MT_TR; ++r) {
      const int yr = r0 + r;
      const double* s = S + (r + 1) * MT_SW;
      const double c = s[0];
      // neighbours outside the domain: the point itself (their face weight is zero anyway; the
      // unloaded shared memory there may hold anything)
      const double l = xc > 0 ? s[-1] : c;
      const double rr = xc + 1 < g.nx ? s[1] : c;
      const double n = yr > 0 ? s[-MT_SW] : c;
      const double so = yr + 1 < g.ny ? s[MT_SW] : c;
      double acc = c;
      acc = fma(wxl[r], c - l, acc);
      acc = fma(wxr[r], c - rr, acc);
      acc = fma(wy[r], c - n, acc);
      acc = fma(wy[r + 1], c - so, acc);
      if (colin && yr < g.ny) yp[(long long)yr * g.nx + xc] = acc - prev[r];
      prev[r] = c;
    }
    __syncthreads();                              // every thread is done with this slot
    if (t == 0 && it + MT_NBUF < i1) mt_issue(g, M, ell, x, it + MT_NBUF, ring + slot * (MT_TR + 2) * MT_SW, &bars[slot]);
  }
}

// Usable for this context: 2D, one rank, Neumann faces, nx even (16-byte row segments).
static inline bool mt_ok(const Geo& g, int dim, int nranks) {
  return dim == 2 && nranks == 1 && !g.dir && g.nx % 2 == 0 && g.nx >= 2 && g.ny >= 1;
}
