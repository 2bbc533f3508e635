/*
 * aac.h -- C ABI of the B200-native all-at-once diffusion-covariance solver
 * (arXiv 2506.03947, "Block alpha-circulant preconditioners for all-at-once
 * diffusion-based covariance operators").
 *
 * The library solves calA x = b (Eq. eq:A), where
 *     calA = I_ell (x) A - Sigma (x) I_N,   Sigma = lower block shift,
 *     A    = I + c (-div kappa grad)_h      (cell-centred, zero-flux Neumann),
 * by flexible GMRES right-preconditioned with the block alpha-circulant
 * preconditioner P_alpha (Eq. eq:exactPBE) applied approximately
 * through its DFT form (Eqs. eq:Paform, eq:blockproblem):
 *     Gamma_alpha scaling -> length-ell DFT across blocks -> ell shifted solves
 *     (A - Lambda_k I) y_k = w_k -> inverse DFT -> Gamma_alpha^{-1} unscaling,
 * the shifted solves by nested Chebyshev semi-iteration (NC1 / NC2 = Algorithm 1,
 * PAPER.md:286-446, 652-690) or by the real saddle-point reformulation with
 * MINRES / PCG (SP).
 *
 * Conventions (all calls):
 *  - fp64 everywhere. Block vectors are DEVICE pointers to ell contiguous planes
 *    of this rank's slab: x[j * n_local + p], p = (z*ny + y)*nx + x (x fastest),
 *    j = 0..ell-1 the time block. Slabs split the slowest non-trivial axis
 *    (y in 2D, z in 3D) into contiguous ranges, rank order = slab order
 *    (aac_slab_range). The caller owns every vector; the library never retains
 *    a caller pointer after a call returns.
 *  - All work is enqueued on the cudaStream_t given to aac_setup, in stream
 *    order. aac_gmres / aac_gmres_host synchronise that stream (they poll the
 *    Arnoldi residual); aac_matvec / aac_precond_apply do not.
 *  - Multi-rank (nranks > 1): every rank calls every function collectively
 *    (SPMD) with the same scalar arguments; NCCL (loaded at run time) carries
 *    the halo exchange and the reductions over NVLink.
 *  - A context is not thread-safe.
 *  - Return codes: AAC_OK, AAC_ENOCONV (> 0: completed with a condition) or a
 *    negative error; aac_last_error() then holds a message.
 */
#ifndef AAC_H
#define AAC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct aac_ctx aac_ctx;

enum {
  AAC_OK = 0,
  AAC_ENOCONV = 1,   /* GMRES reached maxit; x holds the last iterate, info filled */
  AAC_EINVAL = -1,   /* bad argument (message in aac_last_error)                   */
  AAC_ECUDA = -2,    /* a CUDA runtime call or kernel launch failed                */
  AAC_ENCCL = -3,    /* NCCL unavailable or failed                                 */
  AAC_ENOMEM = -4    /* device or host allocation failed                           */
};

enum { AAC_NONE = 0, AAC_NC1 = 1, AAC_NC2 = 2, AAC_SP = 3, AAC_EXACT = 4 };
/* Flag OR'ed into AAC_NC1 / AAC_NC2 (aac_precond_apply, aac_gmres*): mixed precision
 * -- the Chebyshev recurrence of the shifted solves runs in fp32 (operands
 * and iterates stay fp64 in memory), the transforms, calA and GMRES in fp64. The
 * preconditioner is then no longer the fp64 one (FGMRES absorbs the difference). 2D only
 * (the wavefront path); other geometries return AAC_EINVAL.                              */
enum { AAC_F32 = 16 };

typedef struct {
  int dim;          /* 1, 2 or 3                                                     */
  int64_t n[3];     /* global cells per axis (x, y, z); unused axes = 1               */
  int rank;         /* this rank, 0 <= rank < nranks                                  */
  int nranks;       /* number of slabs (1 for a single GPU; must be 1 when dim == 1)  */
} aac_grid;

/* Half-open slab [lo, hi) of the slab axis owned by `rank` (balanced contiguous
 * split, the first n % nranks ranks get one extra layer). Host-only, needs no GPU.
 * Returns AAC_EINVAL on nranks < 1, rank out of range or n < nranks.             */
int aac_slab_range(int64_t n, int nranks, int rank, int64_t* lo, int64_t* hi);

/* Host-only (no GPU needed): this rank's face weights w_f = c kappa_f n_a^2 in the device
 * layout used by the kernels -- three "lower face" arrays wx | wy | wz, concatenated, lengths
 * lens[0..2] (each padded to a multiple of 4 doubles): w?[p] is the face between point p and
 * its lower neighbour along the axis (0 on physical boundaries), and w?[p + stride] is p's
 * upper face, so the slab's top face sits in the extra layer at the end of the slab axis.
 * Call with w_out == NULL to get the lengths; gershgorin (may be NULL) receives the local
 * max_P (1 + 2 sum_f w_f). Same inputs and errors as aac_setup.                             */
int aac_slab_weights(const aac_grid* g, const double* kx, const double* ky, const double* kz,
                     double c, double* w_out, int64_t* lens, double* gershgorin);

/* Create a solver context on the current CUDA device.
 *  kx, ky, kz : HOST pointers to the GLOBAL interior-face diffusivities kappa_f
 *               (anisotropy already applied), natural layouts
 *                 kx[nz][ny][nx-1], ky[nz][ny-1][nx], kz[nz-1][ny][nx]
 *               (NULL allowed for an axis with n = 1). Copied; not retained.
 *  c          : diffusion coefficient; face weight w_f = c * kappa_f * n_a^2
 *               (h_a = 1/n_a), so A = I + c(-div kappa grad)_h (BASELINE.json).
 *  ell        : number of time blocks, even, 2 <= ell <= 16.
 *  alpha      : > 0. Every call that applies P_alpha then needs alpha^{1/ell} < mu_min
 *               (Lemma lemma:Zalpha; AAC_EINVAL otherwise): alpha < 1 for
 *               the Neumann operator (mu_min = 1 exactly), alpha <= 1 allowed for the
 *               paper's Dirichlet operator once aac_set_bounds gives its mu_min > 1.
 *  max_krylov : Krylov storage for aac_gmres (maxit <= max_krylov).
 *  cuda_stream: cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 *               NULL = legacy default stream.
 *  nccl_id    : HOST pointer to a 128-byte ncclUniqueId shared by all ranks;
 *               ignored (may be NULL) when nranks == 1.
 * Errors: AAC_EINVAL (odd/small ell, alpha <= 0, c < 0, kappa <= 0 or
 * non-finite, n < 2 on a used axis, bad slab), AAC_ENOMEM, AAC_ECUDA, AAC_ENCCL. */
int aac_setup(const aac_grid* g, const double* kx, const double* ky, const double* kz,
              double c, int ell, double alpha, int max_krylov, void* cuda_stream,
              const void* nccl_id, aac_ctx** out);

/* Host-staged transport for the slab exchanges (alternative to NCCL). The library copies
 * the data of every exchange step to pinned host memory, synchronises its stream, calls the
 * callback and copies the result back: slow, but it lets any host process group (e.g.
 * torch.distributed "gloo") carry the slab decomposition -- used to verify the multi-rank
 * path with several processes sharing fewer GPUs than ranks, where NCCL cannot run.
 *  allreduce(user, buf, n, op): in-place all-reduce of n HOST doubles over all ranks,
 *                               op 0 = sum, 1 = max; op 2 = all-gather: buf holds nranks * n
 *                               doubles, this rank's n at offset rank * n on entry, every
 *                               rank's at its offset on return (the library then sums them in
 *                               rank order). Return 0 on success.
 *  sendrecv(user, n, send_lo, recv_lo, send_hi, recv_hi): exchange n HOST doubles with
 *      the rank below (send_lo -> its recv_hi, its send_hi -> recv_lo) and the rank above;
 *      the pointers of a missing neighbour are NULL. Return 0 on success.
 * A non-zero return makes the calling entry point fail with AAC_ENCCL.                 */
typedef struct {
  void* user;
  int (*allreduce)(void* user, double* buf, int n, int op);
  int (*sendrecv)(void* user, int64_t n, const double* send_lo, double* recv_lo,
                  const double* send_hi, double* recv_hi);
} aac_host_transport;

/* aac_setup with the host-staged transport instead of NCCL (same arguments otherwise;
 * `tr` is copied; its callbacks must stay valid until aac_destroy).                    */
int aac_setup_host_transport(const aac_grid* g, const double* kx, const double* ky,
                             const double* kz, double c, int ell, double alpha, int max_krylov,
                             void* cuda_stream, const aac_host_transport* tr, aac_ctx** out);

/* y = calA x: y_0 = A x_0, y_j = A x_j - x_{j-1}.
 * x, y: device, [ell][n_local]; x != y. One halo exchange when nranks > 1.       */
int aac_matvec(aac_ctx* ctx, const double* x, double* y);

/* z ~= P_alpha^{-1} r (Eq. eq:Paform) with inner method AAC_NC1 / AAC_NC2
 * (k Chebyshev iterations per shifted system, NC2 redistributes a budget of
 * ell*k by Algorithm 1) or AAC_SP (k MINRES / PCG iterations).
 * r, z: device, [ell][n_local]; r != z. Errors: AAC_EINVAL on k < 1 or an
 * unknown method.                                                                */
int aac_precond_apply(aac_ctx* ctx, int method, int k, const double* r, double* z);

typedef struct {
  int iters;                    /* Arnoldi steps = preconditioner applications     */
  int converged;                /* 1 if |g_{j+1}| <= rtol ||b|| (or breakdown)     */
  double relres_est;            /* |g_{j+1}| / ||b|| at exit                       */
  double relres_true;           /* ||b - calA x|| / ||b|| (one extra apply)        */
  long long matvecs_paper_units;/* products with A in the paper's Table 1 units    */
  long long stencil_sweeps;     /* stencil passes actually executed (per plane)    */
} aac_gmres_info;

/* Flexible GMRES (x_0 = 0, unrestarted, CGS2, Givens) for calA x = b, right-
 * preconditioned by aac_precond_apply(method, k) (BASELINE.json north_star).
 * b, x: device [ell][n_local]; b != x. info may be NULL.
 * Returns AAC_OK on convergence, AAC_ENOCONV after maxit steps.                   */
int aac_gmres(aac_ctx* ctx, int method, int k, const double* b, double* x,
              double rtol, int maxit, aac_gmres_info* info);

/* As aac_gmres with HOST b and x (pinned or pageable); the host<->device copies
 * are enqueued inside the call (the end-to-end path).                            */
int aac_gmres_host(aac_ctx* ctx, int method, int k, const double* b_host, double* x_host,
                   double rtol, int maxit, aac_gmres_info* info);

/* aac_gmres_host for nrhs independent systems (BASELINE.json north_star: one
 * solve per right-hand side), pipelined: while system i is solved on the
 * context stream, b_{i+1} is copied in and x_{i-1} copied out on a second
 * stream (two device slots each; pinned host memory makes the copies
 * asynchronous, pageable memory still works but stages through the driver).
 * b_host[i], x_host[i]: host [ell][n_local] each (x_host[i] may repeat a
 * buffer: the copies out are ordered). info: NULL or nrhs entries. Returns
 * the worst code over the systems (AAC_ENOCONV if any reached maxit); on an
 * error (< 0) the systems after the failing one are not solved.               */
int aac_gmres_host_batch(aac_ctx* ctx, int method, int k, int nrhs, const double* const* b_host,
                         double* const* x_host, double rtol, int maxit, aac_gmres_info* info);

/* Spectral bounds used by the inner solvers (mu_min = 1 exactly, mu_max =
 * global Gershgorin max) and the per-block inner iteration counts for
 * (method, k), block k = 0..ell-1 (alloc may be NULL). n_local may be NULL.      */
int aac_query(aac_ctx* ctx, int method, int k, double* mu_min, double* mu_max, int* alloc,
              int64_t* n_local);

/* Per-kernel CUDA-event timing (off by default). When enabled, every launch of
 * the library is bracketed by events on the context stream; aac_profile_read
 * returns the accumulated device milliseconds, launch count and the model
 * (algorithmic) DRAM bytes of kernel class `id` (0 <= id < aac_profile_count()),
 * and its name. aac_launch_count counts every kernel launch since setup.         */
int aac_profile_enable(aac_ctx* ctx, int enable);
int aac_profile_count(void);
int aac_profile_read(aac_ctx* ctx, int id, const char** name, double* ms, long long* launches,
                     double* model_bytes);
/* ---- paper-reproduction mode ------------------------------------- */

/* Dirichlet boundary faces: (A u)_P += b_a u_P for every face of P on the physical boundary
 * along axis a (a zero ghost value), the paper's operator A = I - (nu/h^2) L (PAPER.md:630-637,
 * Eq. IminusLap: interior AND boundary faces carry nu/h^2). b = 0 restores the BASELINE
 * zero-flux operator. Recomputes the Gershgorin mu_max (mu_min resets to 1: set the true bound
 * with aac_set_bounds), drops cached plans and graphs. Collective. AAC_SP then returns
 * AAC_EINVAL (its multigrid hierarchy has no boundary terms).                            */
int aac_set_boundary(aac_ctx* ctx, double bx, double by, double bz);

/* Spectral bounds of A used by the inner Chebyshev solves and Algorithm 1 (default: 1 and the
 * Gershgorin max, reading R5), e.g. the exact Appendix A bounds of the paper's operator
 * (PAPER.md:998-1020). Needs 0 < mu_min <= mu_max and alpha^{1/ell} < mu_min.           */
int aac_set_bounds(aac_ctx* ctx, double mu_min, double mu_max);

/* method AAC_EXACT, for aac_precond_apply / aac_gmres / aac_ci: the exact
 * P_alpha^{-1} (PAPER.md:229-275 with exact block solves) for the paper's operator only -- 2D,
 * square n x n, one rank, every interior face and the Dirichlet boundary faces of both axes
 * carrying the same weight w (aac_set_boundary(w, w, 0)): A is then diagonalised by the
 * orthonormal DST-I (Appendix A) and every block solve is two-sided DST
 * products (batched fp64 GEMMs through cuBLAS, loaded at run time) and a spectral division.
 * AAC_EINVAL for any other operator; k is ignored.                                       */

/* The paper's outer solver: Chebyshev semi-iteration on P^{-1} calA x = P^{-1} b (PAPER.md:
 * 102-107 Eq. eq:precondsystem) with foci [lmin, lmax] -- Cor. cor:extremeevals gives
 * [1, mu_min^ell/(mu_min^ell - alpha)] -- from x_0 = 0, stopping when ||b - calA x_p|| <
 * tol ||b|| (the paper uses tol = 1e-6). method AAC_NONE: unpreconditioned, foci
 * = the extreme eigenvalues of A. info->iters = p (preconditioner applications); info->
 * matvecs_paper_units = p (ell + inner budget) (Table 1). b, x: device [ell][n_local], b != x.
 * Uses the Krylov workspace (max_krylov >= 1). Returns AAC_OK or AAC_ENOCONV.             */
int aac_ci(aac_ctx* ctx, int method, int k, const double* b, double* x, double lmin, double lmax,
           double tol, int maxit, aac_gmres_info* info);

/* Model (algorithmic) fp64 flops accumulated by kernel class `id` -- non-zero only for the
 * classes whose roofline is arithmetic (the wavefront Chebyshev kernel).                 */
int aac_profile_flops(aac_ctx* ctx, int id, double* model_flops);
int aac_profile_reset(aac_ctx* ctx);
long long aac_launch_count(const aac_ctx* ctx);

/* Varying diagonal blocks: from now on calA has block j's own
 * operator A_j = I + c(-div kappa_j grad)_h (y_0 = A_0 x_0, y_j = A_j x_j - x_{j-1}), and every
 * preconditioner is built on the average A_hat = (1/ell) sum_j A_j (= the operator of the mean
 * face weights; mu_max its Gershgorin bound, mu_min = 1). kx, ky, kz: HOST, the ell blocks'
 * GLOBAL face diffusivities stacked block after block, each in aac_setup's layout; copied.
 * One rank, Neumann only; aac_ci is refused afterwards (the eigenvalue bounds behind the
 * outer CI no longer hold) -- use aac_gmres. Drops cached plans and graphs.
 * Errors: AAC_EINVAL (several ranks, Dirichlet faces, missing or non-positive kappa),
 * AAC_ENOMEM, AAC_ECUDA.                                                                  */
int aac_set_blocks(aac_ctx* ctx, const double* kx, const double* ky, const double* kz);

/* Transport of the slab exchanges: 0 = none (one rank), 1 = NCCL (nranks > 1,
 * or the one-rank communicator AAC_NCCL_SELF=1 creates so that a single GPU runs the whole
 * multi-rank code path), 2 = the host-staged transport of aac_setup_host_transport.
 * NCCL waits watch ncclCommGetAsyncError and give up after AAC_NCCL_TIMEOUT_S seconds
 * (default 300): the communicator is then aborted and calls return AAC_ENCCL.           */
int aac_comm_kind(const aac_ctx* ctx);

const char* aac_last_error(const aac_ctx* ctx);   /* also valid for ctx == NULL */
void aac_destroy(aac_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* AAC_H */
