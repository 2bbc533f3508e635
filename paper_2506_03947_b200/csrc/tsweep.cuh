// tsweep.cuh -- temporally blocked Chebyshev sweeps for 2D grids (one rank).
//
// The three-term recurrence (reading R8) reads x_s, x_{s-1} and hat w and writes x_{s+1} for
// every step: 4 plane-passes of HBM per step. Here a CTA owns one TX x TY output tile of ONE
// packed Fourier block, loads x_{s0}, x_{s0-1}, hat w and the face weights on the tile plus
// an S-point halo into shared memory once, and advances ns <= S Chebyshev steps in shared
// memory (level l is computed on the tile + (S - l) halo, so every level only needs values
// of the previous level that the CTA itself computed). Only the last two iterates of the
// interior go back to HBM (the next pass needs x_s and x_{s-1}); the final pass writes x_{p_k}
// only. Per plane and pass: 3 reads + 2 writes instead of 4 per step.
//
// Out-of-domain halo positions are zero-filled; their face weights are zero, so they never
// contribute to an in-domain point (Neumann: zero flux), and they stay exactly zero.
// Inputs and outputs use disjoint slot sets (ping-pong), so no CTA overwrites what another
// CTA still reads as halo.
#pragma once

#include "nc.cuh"

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct TBlk {
  int cplx, q, ns, s0;       // complex?, first plane, steps this pass, local step of x_{s0}
  const double* ps;          // x_{s0} source (plane q), scaled by (sr, si)
  const double* pm;          // x_{s0-1} source, scaled by (mr, mi)
  double sr, si, mr, mi;
  double* out_last;          // x_{s0+ns}   (plane q) or NULL
  double* out_prev;          // x_{s0+ns-1} (plane q) or NULL
  double lr, li;             // Lambda_k
  double ar[8], ai[8], br[8], bi[8];   // step coefficients for local steps s0 .. s0+ns-1
};
struct TSweep {
  TBlk b[AAC_MAX_BLK];
};

template <int S, int TX, int TY>
struct TGeom {
  static constexpr int RX = TX + 2 * S, RY = TY + 2 * S, R = RX * RY;
  static constexpr int WXN = RY * (RX + 1);      // x-faces incl. the upper face of the last column
  static constexpr int WYN = (RY + 1) * RX;      // y-faces incl. the upper face of the last row
  static constexpr int NDBL = 8 * R + WXN + WYN; // 3 levels x 2 planes, hat w x 2 planes
};

template <int S, int TX, int TY>
__global__ void __launch_bounds__(256) k_tsweep(Geo g, TSweep T, const double* __restrict__ what,
                                                const IterState* st) {
  using G = TGeom<S, TX, TY>;
  if (st && st->done) return;
  extern __shared__ __align__(16) double sh[];
  double* buf = sh;                       // [3 levels][2 planes][R]
  double* wsh = sh + 6 * G::R;            // [2 planes][R]
  double* wx = sh + 8 * G::R;             // [RY][RX+1]
  double* wy = wx + G::WXN;               // [RY+1][RX]
  const TBlk& B = T.b[blockIdx.y];
  const int ntx = (g.nx + TX - 1) / TX;
  const int tx0 = (blockIdx.x % ntx) * TX - S, ty0 = (blockIdx.x / ntx) * TY - S;
  const long long N = g.N;
  const int np = B.cplx ? 2 : 1;
  const int tid = threadIdx.x;
  // ---- load phase: asynchronous copies (cp.async, zero-fill outside the domain) so every
  // thread has all of its loads in flight at once, then an in-place complex scaling when the
  // source is a virtual iterate (x_1 = w/theta, x_0 = 0).
  const bool scale_s = !(B.sr == 1.0 && B.si == 0.0), scale_m = !(B.mr == 1.0 && B.mi == 0.0);
  const bool load_m = !(B.mr == 0.0 && B.mi == 0.0);
  for (int c2 = tid; c2 < G::R / 2; c2 += blockDim.x) {       // pairs along x (16 bytes)
    const int c = 2 * c2;
    const int cx = c % G::RX, cy = c / G::RX;
    const int gx = tx0 + cx, gy = ty0 + cy;
    const bool in = gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny;
    const long long p = in ? (long long)gy * g.nx + gx : 0;
    const int sz = in ? 16 : 0;
    for (int e = 0; e < np; ++e) {
      cp_async16(buf + e * G::R + c, B.ps + (long long)e * N + p, sz);
      if (load_m) cp_async16(buf + 4 * G::R + e * G::R + c, B.pm + (long long)e * N + p, sz);
      cp_async16(wsh + e * G::R + c, what + (long long)(B.q + e) * N + p, sz);
    }
  }
  for (int c = tid; c < G::WXN; c += blockDim.x) {
    const int cx = c % (G::RX + 1), cy = c / (G::RX + 1);
    const int gx = tx0 + cx, gy = ty0 + cy;
    const bool in = gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny;
    cp_async8(wx + c, g.wx + (in ? (long long)gy * g.nx + gx : 0), in ? 8 : 0);
  }
  for (int c = tid; c < G::WYN; c += blockDim.x) {
    const int cx = c % G::RX, cy = c / G::RX;
    const int gx = tx0 + cx, gy = ty0 + cy;
    const bool in = gx >= 0 && gx < g.nx && gy >= 0 && gy <= g.ny;
    cp_async8(wy + c, g.wy + (in ? (long long)gy * g.nx + gx : 0), in ? 8 : 0);
  }
  cp_async_wait_all();
  __syncthreads();
  if (scale_s || scale_m) {
    for (int c = tid; c < G::R; c += blockDim.x) {
      if (scale_s) {
        const double a = buf[c], b = np == 2 ? buf[G::R + c] : 0.0;
        buf[c] = B.sr * a - B.si * b;
        if (np == 2) buf[G::R + c] = B.sr * b + B.si * a;
      }
      if (scale_m) {
        const double a = load_m ? buf[4 * G::R + c] : 0.0;
        const double b = (load_m && np == 2) ? buf[5 * G::R + c] : 0.0;
        buf[4 * G::R + c] = B.mr * a - B.mi * b;
        if (np == 2) buf[5 * G::R + c] = B.mr * b + B.mi * a;
      }
    }
    __syncthreads();
  }
  // ---- ns Chebyshev steps in shared memory
  for (int l = 1; l <= B.ns; ++l) {
    const double* cur = buf + ((l - 1) % 3) * 2 * G::R;
    const double* prv = buf + ((l + 1) % 3) * 2 * G::R;      // (l - 2) mod 3
    double* out = buf + (l % 3) * 2 * G::R;
    const double ar = B.ar[l - 1], ai = B.ai[l - 1], br = B.br[l - 1], bi = B.bi[l - 1];
    const int lo = l, hx = G::RX - l, hy = G::RY - l;
    const int wdt = hx - lo, cnt = wdt * (hy - lo);
    for (int i = tid; i < cnt; i += blockDim.x) {
      const int cx = lo + i % wdt, cy = lo + i / wdt;
      const int c = cy * G::RX + cx;
      const double fxl = wx[cy * (G::RX + 1) + cx], fxr = wx[cy * (G::RX + 1) + cx + 1];
      const double fyl = wy[c], fyr = wy[c + G::RX];
      double ax[2], xc[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (e < np) {
          const double* u = cur + e * G::R;
          const double u0 = u[c];
          double a = u0;
          a = fma(fxl, u0 - u[c - 1], a);
          a = fma(fxr, u0 - u[c + 1], a);
          a = fma(fyl, u0 - u[c - G::RX], a);
          a = fma(fyr, u0 - u[c + G::RX], a);
          ax[e] = a;
          xc[e] = u0;
        } else {
          ax[e] = xc[e] = 0.0;
        }
      }
      const double mr = prv[c], mi = np == 2 ? prv[G::R + c] : 0.0;
      const double w0 = wsh[c], w1 = np == 2 ? wsh[G::R + c] : 0.0;
      const double rr = w0 - (ax[0] - (B.lr * xc[0] - B.li * xc[1]));
      const double ri = w1 - (ax[1] - (B.lr * xc[1] + B.li * xc[0]));
      const double dr = xc[0] - mr, di = xc[1] - mi;
      out[c] = xc[0] + (ar * dr - ai * di) + (br * rr - bi * ri);
      if (np == 2) out[G::R + c] = xc[1] + (ar * di + ai * dr) + (br * ri + bi * rr);
    }
    __syncthreads();
  }
  // ---- write the tile interior of the last two levels
  const double* last = buf + (B.ns % 3) * 2 * G::R;
  const double* prev = buf + ((B.ns + 2) % 3) * 2 * G::R;
  for (int i = tid; i < TX * TY; i += blockDim.x) {
    const int ix = i % TX, iy = i / TX;
    const int gx = tx0 + S + ix, gy = ty0 + S + iy;
    if (gx >= g.nx || gy >= g.ny) continue;
    const long long p = (long long)gy * g.nx + gx;
    const int c = (iy + S) * G::RX + ix + S;
    if (B.out_last) {
      B.out_last[p] = last[c];
      if (np == 2) B.out_last[N + p] = last[G::R + c];
    }
    if (B.out_prev) {
      B.out_prev[p] = prev[c];
      if (np == 2) B.out_prev[N + p] = prev[G::R + c];
    }
  }
}
