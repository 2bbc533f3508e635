// aac_internal.cuh -- context, geometry and launch plumbing of libaac (sm_100a, fp64).
// Not part of the C ABI (include/aac.h is). See DESIGN.md §5 for the data layout.
#pragma once
#include <cstdlib>

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/aac.h"
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: no-ops unless a profiler is attached

#define AAC_MAX_ELL 16
#define AAC_MAX_BLK (AAC_MAX_ELL / 2 + 1)
#define AAC_GATHER_MAX 1024    // longest sum reduced by all-gather + rank-order sum

// Traversal direction of the streaming kernels of a GMRES step (AAC_REV bit mask, set once at
// aac_setup): a kernel that walks the grid in the direction OPPOSITE to its producer starts on
// the producer's most recent output, which is still in the 126 MB L2 (the vectors are 84 MB at
// the headline, so a same-direction consumer starts on lines already evicted). The logical
// CTA index is flipped, so every CTA computes the same points in the same order and the
// cross-CTA partial sums keep their slots: bit-identical to the forward order (k_arnoldi's
// persistent CTAs walk their own tiles backwards too, which reorders their private sums).
// bit 0 k_matvec, 1 k_arnoldi, 2 k_fwd_upd, 3 k_waver, 4 k_inverse.
__constant__ int c_rev;
#define AAC_REV_MATVEC 1
#define AAC_REV_ARNOLDI 2
#define AAC_REV_FWD 4
#define AAC_REV_WAVE 8
#define AAC_REV_INV 16
#define AAC_L2_ARNOLDI 32   // basis stream of k_arnoldi with an L2 evict_first policy
#define AAC_L2_FWD 64       // ... of k_fwd_upd (bit 7: W too)
#define AAC_L2_FWD_W 128
#define AAC_L2_FWD_VJ 256    // k_fwd_upd stores V_j with a streaming (evict-first) store
#define AAC_L2_MATVEC_W 512  // k_matvec stores w with an L2 evict_last policy
#ifndef AAC_REV_DEFAULT
// measured best at the headline: k_matvec and k_fwd_upd reversed (8.34 -> 8.18 ms per solve, all
// 32 direction masks tried), k_fwd_upd's input streams evict_first and its V_j store streaming so
// that hat w stays in L2 for the wavefront (8.15; 2d256 3.98 -> 3.92 ms)
#define AAC_REV_DEFAULT (AAC_REV_MATVEC | AAC_REV_FWD | AAC_L2_FWD | AAC_L2_FWD_W | AAC_L2_FWD_VJ)
#endif

// ------------------------------------------------------------------------------------------
// Geometry of this rank's slab, passed BY VALUE to every stencil kernel.
// Points p = (z*ny + y)*nx + x of the local slab (x fastest). The slab axis is y for dim 2
// and z for dim 3; `S` is the size of one layer across the slab axis (nx in 2D, nx*ny in 3D).
// Face weights use the "lower face" convention: wx[p] = weight of the face between (x-1) and
// x (0 at x = 0), and likewise wy, wz; each array carries one extra layer so that the upper
// face of p is always w?[p + stride] (zero on physical boundaries; the slab's top face on
// the last local layer of the slab axis). Halo layers (ell planes of S values) hold the
// neighbour ranks' boundary layers of the stencil input.
struct Geo {
  int nx, ny, nz;        // LOCAL extents (slab axis already cut)
  long long N;           // nx*ny*nz
  long long S;           // layer size across the slab axis
  int has_lo, has_hi;    // neighbour ranks below / above along the slab axis
  int dir;               // 1: Dirichlet boundary faces (paper operator, aac_set_boundary)
  double bdx, bdy, bdz;  // Dirichlet boundary-face weights per axis: (A u)_P += bd u_P per face
  const double* wx;
  const double* wy;
  const double* wz;
};

// ------------------------------------------------------------------------------------------
// Kernel classes for per-kernel CUDA-event profiling (aac_profile_*).
enum KernelId {
  KID_MATVEC = 0,      // calA apply (stencil over all ell planes)
  KID_FWD,             // gamma-scale + block DFT (+ first Chebyshev step when fused)
  KID_SWEEP,           // Chebyshev three-term sweep (stencil + axpby) on active planes
  KID_INV,             // last Chebyshev step + inverse DFT + gamma^{-1}
  KID_DOT,             // multi-dot partials
  KID_UPD,             // CGS update (+ fused dots / norm)
  KID_REDUCE,          // fixed-order reduction of partials
  KID_SCALAR,          // single-thread Arnoldi / Givens / back substitution
  KID_AXPY,            // vector scale / lincomb
  KID_SP_STENCIL,      // SP: shifted / saddle stencil applies
  KID_SP_MG,           // SP: multigrid smoother / transfer / coarse solve
  KID_SP_VEC,          // SP: Krylov vector updates and dots
  KID_HALO,            // halo pack/copy
  KID_ARNOLDI,         // calA apply fused with the CGS2 projections + Gram column
  KID_COUNT
};

struct ProfRec { int id; cudaEvent_t a, b; };

struct NcPlan {            // inner Chebyshev plan for (method, k)
  int method = 0, k = 0;
  int nblk = 0;            // ell/2 + 1 packed blocks
  int p[AAC_MAX_BLK];      // iterations per packed block
  int pmax = 0;
  std::vector<double> a_re, a_im, b_re, b_im;   // [blk][s] s = 1..p-1, row stride pmax
};

struct SpPlan;             // saddle-point plan (sp.cuh)
struct IterState;          // GMRES device state (krylov.cuh)

struct GraphEntry {        // one captured Arnoldi step per (method, k)
  int method, k;
  cudaGraphExec_t exec;
  int nodes;
};

struct aac_ctx {
  // problem
  int dim = 0, ell = 0, rank = 0, nranks = 1;
  long long n[3] = {1, 1, 1};          // global extents
  long long lo = 0, hi = 0;            // slab range along the slab axis
  double c = 0.0, alpha = 0.0;
  double mu_min = 1.0, mu_max = 1.0;
  Geo geo{};
  int max_krylov = 0;
  cudaStream_t user_stream = nullptr;  // caller's stream (entry / exit ordering)
  cudaStream_t stream = nullptr;       // library-owned non-blocking stream (graph capture)
  cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_it[2] = {nullptr, nullptr};
  int device = 0;
  int num_sms = 148;
  int ka_grid = 0;                     // persistent grid of k_arnoldi
  // device memory (library-owned)
  double* d_w = nullptr;               // wx | wy | wz
  long long wlen[3] = {0, 0, 0};       // their padded lengths
  double* d_what = nullptr;            // [ell][N] packed half-complex DFT of the input
  double* d_X = nullptr;               // [3][ell][N] Chebyshev iterate slots
  double* d_tmp = nullptr;             // [ell][N] scratch (true residual, SP)
  double* d_V = nullptr;               // [(max_krylov+1)][ell][N]
  double* d_Z = nullptr;               // [max_krylov][ell][N]
  double* d_W = nullptr;               // [ell][N] Arnoldi work vector
  double* d_bx = nullptr;              // [2][ell][N] staging for aac_gmres_host
  double* d_bb = nullptr;              // [4][ell][N] b | b | x | x for aac_gmres_host_batch
  cudaStream_t cstream = nullptr;      // copy stream of aac_gmres_host_batch
  cudaEvent_t ev_cp[6] = {};           // in[2] | done[2] | out[2]
  // fork/join streams of the per-block wavefront launches (wave_r.cuh)
  static constexpr int NAUX = 4;
  cudaStream_t aux[NAUX] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[NAUX] = {};
  double* d_halo = nullptr;            // [2][ell][S]  lo | hi
  double* d_part = nullptr;            // per-CTA partial sums
  unsigned* d_grp = nullptr;           // two-level ticket counters (zeroed)
  long long part_len = 0;
  double* d_red = nullptr;             // reduced sums / scratch (3 * ldh)
  double* d_H = nullptr;               // Hessenberg ldh x max_krylov, col-major
  double* d_G = nullptr;               // Gram matrix ldh x ldh
  double* d_giv = nullptr;             // cs | sn | g | y | sigma | c   (ldh each)
  double* d_stat = nullptr;            // small scalars (device)
  double* h_stat = nullptr;            // pinned mirror
  IterState* d_st = nullptr;
  IterState* h_st = nullptr;           // pinned mirror (graph memcpy node target)
  std::vector<GraphEntry> graphs;
  bool use_graphs = true;
  int wave_h = 8;                      // wavefront depth (wave.cuh; 0 = per-step sweeps)
  bool wave_forced = false;            // AAC_WAVE_H given: no automatic choice (wave_pays)
  int l2_bytes = 0;                    // L2 size (the wave / per-step choice)
  // slab-decomposed wavefront (2D, several ranks): face weights of rows [elo, ehi) of the
  // global grid (this slab +- WAVE halo rows) and halo rows of hat w
  double* d_wext = nullptr;            // wx | wy of the extended row range
  long long wext_x = 0;                // offset of wy in d_wext
  int wext_off = 0, wext_rows = 0;     // lo - elo, ehi - elo
  double* d_whalo = nullptr;           // [2][ell][hd][nx]
  double* d_gath = nullptr;            // [nranks][AAC_GATHER_MAX]: rank-ordered sums (comm.cuh)
  double* d_ghost = nullptr;           // [2][ell][nx]: final Chebyshev iterates of the slab ghost rows
  bool z_ghost = false;                // this step's preconditioner wrote Z_j's halo rows (d_halo)
  unsigned* pub_fold = nullptr;        // set while the step graph is captured: k_arnoldi publishes the IterState
  int wave_hd = 0;                     // halo depth (0: slabs too thin, per-step sweeps)
  // plans
  NcPlan nc[2];                        // cached NC plans
  int nc_next = 0;
  SpPlan* sp = nullptr;
  // exact P_alpha (N3, exact.cuh): DST-I matrix, 1D eigenvalues, GEMM workspace
  double* d_S = nullptr;               // [n][n] orthonormal DST-I
  double* d_lam1 = nullptr;            // [n] w * 4 sin^2(pi (i+1) / (2 (n+1)))
  double* d_T = nullptr;               // [ell][n][n] GEMM intermediate
  int exact_n = 0;                     // > 0 once prepared
  // varying diagonal blocks (aac_set_blocks): per-block face weights; d_w then holds
  // the mean-block A_hat the preconditioner uses
  double* d_wblk = nullptr;            // [ell][wlen[0] + wlen[1] + wlen[2]]
  bool varying = false;
  // NCCL (dlopen'ed), or the host-staged transport
  void* nccl_comm = nullptr;
  bool nccl_self = false;              // AAC_NCCL_SELF=1: a one-rank NCCL communicator (test switch)
  cudaEvent_t ev_sync = nullptr;       // NCCL waits: polled with the async-error check + timeout
  bool host_tr = false;
  aac_host_transport htr{};
  double* h_stage = nullptr;           // pinned staging for host-transport exchanges
  long long stage_len = 0;
  // bookkeeping
  long long launches = 0;
  long long sweeps = 0;
  bool prof = false;
  bool eager_poll = false;             // eager GMRES: read the state back after each forward step
  bool one_reduce = false;             // lagged normalisation: one reduction per Arnoldi step
  bool inner_f32 = false;              // this call's NC inner solves in fp32 (method | AAC_F32)
  std::vector<ProfRec> prof_recs;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[KID_COUNT] = {0};
  long long prof_n[KID_COUNT] = {0};
  double prof_bytes[KID_COUNT] = {0};
  double prof_flops[KID_COUNT] = {0};  // model fp64 flops (set for ALU-bound kernels)
  double next_flops = 0.0;             // attached to the next launch
  std::string err;
  // the multi-rank code path runs (local partial sums + all-reduce + scalar kernels)
  bool multi() const { return nranks > 1 || nccl_self; }
};

// ------------------------------------------------------------------------------------------
int aac_fail(aac_ctx* ctx, int code, const char* fmt, ...);

#define CUDA_TRY(ctx, call)                                                                 \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return aac_fail((ctx), AAC_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,         \
                      cudaGetErrorString(e_));                                              \
  } while (0)

#define AAC_TRY(...)         \
  do {                       \
    int r_ = (__VA_ARGS__);  \
    if (r_ < 0) return r_;   \
  } while (0)

// NVTX range over a C-ABI call (setup, matvec, precond_apply, gmres, ci): the phases show up
// in nsys / ncu --nvtx timelines.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Bracket one launch with profiling events when enabled; count it; check launch errors.
struct LaunchScope {
  aac_ctx* ctx;
  int id;
  cudaEvent_t a = nullptr, b = nullptr;
  LaunchScope(aac_ctx* c, int kid, double bytes);
  int end();
};

// Launch with programmatic stream serialisation (PDL): the kernel may be scheduled while its
// predecessor drains and waits in griddep() (krylov.cuh); AAC_PDL=0 launches normally.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  static const bool off = getenv("AAC_PDL") && atoi(getenv("AAC_PDL")) == 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = off ? 0 : 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

#define LAUNCH(ctx, kid, bytes, ...)                                                         \
  do {                                                                                      \
    LaunchScope ls_((ctx), (kid), (bytes));                                                 \
    __VA_ARGS__;                                                                            \
    AAC_TRY(ls_.end());                                                                     \
  } while (0)

// Loop over the ell planes of a point with compile-time indices (register-resident arrays).
// ELLC is the compile-time plane capacity of the kernel (10 or 16; ell <= ELLC).
#define FOR_PL(pl) _Pragma("unroll") for (int pl = 0; pl < ELLC; ++pl) if (pl < ell)

inline unsigned grid1d(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  return (unsigned)(g < 1 ? 1 : g);
}
