// comm.cuh -- NCCL over NVLink/NVSwitch for the slab decomposition.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy torch already mapped into the
// process), only when nranks > 1, so single-GPU use and CPU-only imports never touch it.
// Exchange steps of the path: one halo exchange of the stencil input before every stencil
// sweep (neighbour boundary layers along the slab axis, contiguous per plane) and sum
// all-reduces of the GMRES inner products / max all-reduce of the Gershgorin bound.
#pragma once

#include <dlfcn.h>
#include <nccl.h>
#include <time.h>
#include <unistd.h>

#include "aac_internal.cuh"

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};

static NcclApi g_nccl;

static int nccl_load(aac_ctx* ctx) {
  if (g_nccl.h) return AAC_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return aac_fail(ctx, AAC_ENCCL, "dlopen libnccl.so.2 failed: %s", dlerror());
#define SYM(name, field)                                                               \
  *(void**)(&g_nccl.field) = dlsym(h, name);                                           \
  if (!g_nccl.field) return aac_fail(ctx, AAC_ENCCL, "NCCL symbol %s missing", name);
  SYM("ncclCommInitRank", CommInitRank)
  SYM("ncclCommDestroy", CommDestroy)
  SYM("ncclAllReduce", AllReduce)
  SYM("ncclAllGather", AllGather)
  SYM("ncclSend", Send)
  SYM("ncclRecv", Recv)
  SYM("ncclGroupStart", GroupStart)
  SYM("ncclGroupEnd", GroupEnd)
  SYM("ncclGetErrorString", GetErrorString)
  SYM("ncclGetUniqueId", GetUniqueId)
  SYM("ncclCommGetAsyncError", CommGetAsyncError)
  SYM("ncclCommAbort", CommAbort)
#undef SYM
  g_nccl.h = h;
  return AAC_OK;
}

#define NCCL_TRY(ctx, call)                                                                 \
  do {                                                                                      \
    ncclResult_t r_ = (call);                                                               \
    if (r_ != ncclSuccess)                                                                  \
      return aac_fail((ctx), AAC_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call,         \
                      g_nccl.GetErrorString(r_));                                           \
  } while (0)

// nranks > 1: the caller's unique id (rank 0 created it). nranks == 1 with AAC_NCCL_SELF=1: a
// one-rank communicator of this process, so a single GPU runs the whole multi-rank code path --
// local partial sums, NCCL all-reduces captured in the step graph, the scalar kernels -- which
// is how that path is exercised where only one GPU exists (tests/test_gpu_nccl.py).
static int comm_init(aac_ctx* ctx, const void* nccl_id) {
  if (ctx->host_tr) return AAC_OK;
  ncclUniqueId id;
  if (ctx->nranks == 1) {
    const char* e = getenv("AAC_NCCL_SELF");
    if (!e || atoi(e) != 1) return AAC_OK;
    AAC_TRY(nccl_load(ctx));
    NCCL_TRY(ctx, g_nccl.GetUniqueId(&id));
    ctx->nccl_self = true;
  } else {
    if (!nccl_id) return aac_fail(ctx, AAC_EINVAL, "nccl_id required when nranks > 1");
    AAC_TRY(nccl_load(ctx));
    memcpy(&id, nccl_id, sizeof(id));
  }
  ncclComm_t comm;
  NCCL_TRY(ctx, g_nccl.CommInitRank(&comm, ctx->nranks, id, ctx->rank));
  ctx->nccl_comm = (void*)comm;
  return AAC_OK;
}

static void comm_destroy(aac_ctx* ctx) {
  if (ctx->nccl_comm && g_nccl.CommDestroy) g_nccl.CommDestroy((ncclComm_t)ctx->nccl_comm);
  ctx->nccl_comm = nullptr;
  if (ctx->ev_sync) cudaEventDestroy(ctx->ev_sync);
  ctx->ev_sync = nullptr;
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  ctx->h_stage = nullptr;
}

// Pinned staging for the host transport: [send_lo | recv_lo | send_hi | recv_hi] halo layers of
// up to ell planes, or the all-reduce payload.
static int host_stage(aac_ctx* ctx, long long need) {
  if (ctx->stage_len >= need) return AAC_OK;
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  ctx->h_stage = nullptr;
  ctx->stage_len = 0;
  CUDA_TRY(ctx, cudaMallocHost((void**)&ctx->h_stage, (size_t)need * sizeof(double)));
  ctx->stage_len = need;
  return AAC_OK;
}

static int host_allreduce(aac_ctx* ctx, double* d, int n, int op) {
  AAC_TRY(host_stage(ctx, n));
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_stage, d, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (ctx->htr.allreduce(ctx->htr.user, ctx->h_stage, n, op) != 0)
    return aac_fail(ctx, AAC_ENCCL, "host transport all-reduce failed");
  CUDA_TRY(ctx, cudaMemcpyAsync(d, ctx->h_stage, (size_t)n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));   // the staging buffer is reused next call
  return AAC_OK;
}

// Wait for `ev` while watching the communicator: a peer that died or an NCCL failure
// (ncclCommGetAsyncError) or no progress within AAC_NCCL_TIMEOUT_S seconds (default 300)
// aborts the communicator and returns AAC_ENCCL instead of hanging the solve.
static double comm_now() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

static int comm_wait_event(aac_ctx* ctx, cudaEvent_t ev) {
  if (!ctx->nccl_comm) {
    CUDA_TRY(ctx, cudaEventSynchronize(ev));
    return AAC_OK;
  }
  static const double limit = getenv("AAC_NCCL_TIMEOUT_S") ? atof(getenv("AAC_NCCL_TIMEOUT_S")) : 300.0;
  const double t0 = comm_now();
  for (int spin = 0;; ++spin) {
    const cudaError_t e = cudaEventQuery(ev);
    if (e == cudaSuccess) return AAC_OK;
    if (e != cudaErrorNotReady) return aac_fail(ctx, AAC_ECUDA, "wait: %s", cudaGetErrorString(e));
    ncclResult_t ar = ncclSuccess;
    g_nccl.CommGetAsyncError((ncclComm_t)ctx->nccl_comm, &ar);
    const bool late = comm_now() - t0 > limit;
    if ((ar != ncclSuccess && ar != ncclInProgress) || late) {
      g_nccl.CommAbort((ncclComm_t)ctx->nccl_comm);
      ctx->nccl_comm = nullptr;
      return aac_fail(ctx, AAC_ENCCL, late ? "NCCL: no progress within %.0f s (communicator aborted)"
                                           : "NCCL asynchronous error: %s (communicator aborted)",
                      late ? limit : 0.0, late ? "" : g_nccl.GetErrorString(ar));
    }
    if (spin > 64) usleep(20);
  }
}

// Profiling only: keep the library stream busy for `ns` nanoseconds (globaltimer) so that the
// host enqueues the next launches, with their timing events, before the GPU reaches them --
// otherwise the first event pair after a host sync measures the host's enqueue latency too.
__global__ void k_prof_hold(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

// cudaStreamSynchronize of the library stream with the same watch (NCCL contexts). In profile
// mode the stream is then held for 400 us (k_prof_hold; not counted as a launch).
static int comm_sync_impl(aac_ctx* ctx) {
  if (!ctx->nccl_comm) {
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return AAC_OK;
  }
  if (!ctx->ev_sync) CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_sync, cudaEventDisableTiming));
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_sync, ctx->stream));
  return comm_wait_event(ctx, ctx->ev_sync);
}
static int comm_sync(aac_ctx* ctx) {
  AAC_TRY(comm_sync_impl(ctx));
  if (ctx->prof) k_prof_hold<<<1, 1, 0, ctx->stream>>>(400000ULL);
  return AAC_OK;
}

// In-place all-reduce of n doubles on the context stream (no-op on one rank).
// d[i] = sum_{r < P} g[r * n + i], ranks in order (a fixed association on every rank and run).
__global__ void k_rank_sum(const double* __restrict__ g, int P, int n, double* d) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < P; ++r) s += g[(long long)r * n + i];
    d[i] = s;
  }
}

// Sums of at most AAC_GATHER_MAX doubles (the GMRES / CI / SP inner products) are all-gathered
// and added in rank order (the reductions across ranks do not depend on NCCL's
// algorithm or on the host group's order); longer sums (the zero-padded gathered multigrid
// level, where every entry has one non-zero contribution, so any order is exact) and maxima use
// the transport's all-reduce.
static int comm_gather_sum(aac_ctx* ctx, double* d, int n) {
  const int P = ctx->nranks;
  if (!ctx->d_gath) {
    if (cudaMalloc((void**)&ctx->d_gath, (size_t)P * AAC_GATHER_MAX * sizeof(double)) != cudaSuccess) {
      ctx->d_gath = nullptr;
      cudaGetLastError();
      return aac_fail(ctx, AAC_ENOMEM, "gather buffer allocation failed");
    }
  }
  double* mine = ctx->d_gath + (long long)ctx->rank * n;
  CUDA_TRY(ctx, cudaMemcpyAsync(mine, d, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  if (ctx->host_tr) {
    AAC_TRY(host_stage(ctx, (long long)P * n));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_stage + (long long)ctx->rank * n, d, (size_t)n * sizeof(double),
                                  cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->htr.allreduce(ctx->htr.user, ctx->h_stage, n, 2) != 0)
      return aac_fail(ctx, AAC_ENCCL, "host transport all-gather failed");
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_gath, ctx->h_stage, (size_t)P * n * sizeof(double),
                                  cudaMemcpyHostToDevice, ctx->stream));
  } else {
    NCCL_TRY(ctx, g_nccl.AllGather(mine, ctx->d_gath, (size_t)n, ncclFloat64, (ncclComm_t)ctx->nccl_comm,
                                   ctx->stream));
  }
  k_rank_sum<<<1, 256, 0, ctx->stream>>>(ctx->d_gath, P, n, d);
  CUDA_TRY(ctx, cudaGetLastError());
  if (ctx->host_tr) CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));   // h_stage reused next call
  return AAC_OK;
}

static int comm_allreduce(aac_ctx* ctx, double* d, int n, ncclRedOp_t op) {
  if (!ctx->multi() || n <= 0) return AAC_OK;
  if (!ctx->host_tr && !ctx->nccl_comm) return aac_fail(ctx, AAC_ENCCL, "NCCL communicator aborted");
  if (op == ncclSum && n <= AAC_GATHER_MAX) return comm_gather_sum(ctx, d, n);
  if (ctx->host_tr) return host_allreduce(ctx, d, n, op == ncclMax ? 1 : 0);
  NCCL_TRY(ctx, g_nccl.AllReduce(d, d, (size_t)n, ncclFloat64, op, (ncclComm_t)ctx->nccl_comm,
                                 ctx->stream));
  return AAC_OK;
}

// Halo exchange of the stencil inputs: for each (plane pointer, plane index q) send the
// first / last slab layer to the rank below / above and receive the neighbours' layers into
// halo_lo[q] / halo_hi[q]. Layers are contiguous (S doubles), so no packing is needed.
// General form: layers of S doubles at the start / end (offset N - S) of each plane, received
// into hlo + q * S / hhi + q * S (any level of the slab decomposition; g carries has_lo/hi).
static int comm_halo_ex(aac_ctx* ctx, const Geo& g, const double* const* planes, const int* qs,
                        int count, double* hlo, double* hhi) {
  if (ctx->nranks == 1 || count == 0) return AAC_OK;
  const long long S = g.S;
  if (ctx->host_tr) {
    const long long n = (long long)count * S;
    AAC_TRY(host_stage(ctx, 4 * n));
    double* slo = ctx->h_stage;
    double* rlo = slo + n;
    double* shi = rlo + n;
    double* rhi = shi + n;
    for (int i = 0; i < count; ++i) {
      if (g.has_lo)
        CUDA_TRY(ctx, cudaMemcpyAsync(slo + i * S, planes[i], S * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      if (g.has_hi)
        CUDA_TRY(ctx, cudaMemcpyAsync(shi + i * S, planes[i] + g.N - S, S * sizeof(double), cudaMemcpyDeviceToHost,
                                      ctx->stream));
    }
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->htr.sendrecv(ctx->htr.user, n, g.has_lo ? slo : nullptr, g.has_lo ? rlo : nullptr,
                          g.has_hi ? shi : nullptr, g.has_hi ? rhi : nullptr) != 0)
      return aac_fail(ctx, AAC_ENCCL, "host transport halo exchange failed");
    for (int i = 0; i < count; ++i) {
      if (g.has_lo)
        CUDA_TRY(ctx, cudaMemcpyAsync(hlo + qs[i] * S, rlo + i * S, S * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
      if (g.has_hi)
        CUDA_TRY(ctx, cudaMemcpyAsync(hhi + qs[i] * S, rhi + i * S, S * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    }
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return AAC_OK;
  }
  if (!ctx->nccl_comm) return aac_fail(ctx, AAC_ENCCL, "NCCL communicator aborted");
  ncclComm_t comm = (ncclComm_t)ctx->nccl_comm;
  NCCL_TRY(ctx, g_nccl.GroupStart());
  // the group is always closed: the first failing call is recorded, the rest skipped
  ncclResult_t bad = ncclSuccess;
  const char* what = "";
  auto rec = [&](ncclResult_t r, const char* w) {
    if (r != ncclSuccess && bad == ncclSuccess) { bad = r; what = w; }
  };
  for (int i = 0; i < count && bad == ncclSuccess; ++i) {
    const double* u = planes[i];
    const int q = qs[i];
    if (g.has_lo) {
      rec(g_nccl.Send(u, S, ncclFloat64, ctx->rank - 1, comm, ctx->stream), "ncclSend (lower)");
      rec(g_nccl.Recv(hlo + q * S, S, ncclFloat64, ctx->rank - 1, comm, ctx->stream), "ncclRecv (lower)");
    }
    if (g.has_hi) {
      rec(g_nccl.Send(u + g.N - S, S, ncclFloat64, ctx->rank + 1, comm, ctx->stream), "ncclSend (upper)");
      rec(g_nccl.Recv(hhi + q * S, S, ncclFloat64, ctx->rank + 1, comm, ctx->stream), "ncclRecv (upper)");
    }
  }
  const ncclResult_t ge = g_nccl.GroupEnd();
  if (bad != ncclSuccess) return aac_fail(ctx, AAC_ENCCL, "halo exchange: %s: %s", what, g_nccl.GetErrorString(bad));
  if (ge != ncclSuccess) return aac_fail(ctx, AAC_ENCCL, "halo exchange: ncclGroupEnd: %s", g_nccl.GetErrorString(ge));
  return AAC_OK;
}

static int comm_halo(aac_ctx* ctx, const double* const* planes, const int* qs, int count) {
  return comm_halo_ex(ctx, ctx->geo, planes, qs, count, ctx->d_halo,
                      ctx->d_halo + (long long)ctx->ell * ctx->geo.S);
}
