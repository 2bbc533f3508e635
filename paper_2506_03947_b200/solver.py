"""Thin Python front end of libaac (marshalling only; names follow include/aac.h).

    s = Solver(dim, n, kx, ky, kz, c, ell, alpha)      # aac_setup
    y = s.matvec(x)                                      # aac_matvec           (y = calA x)
    z = s.precond_apply("nc2", 8, r)                     # aac_precond_apply    (z ~ P^{-1} r)
    x, info = s.gmres("nc2", 8, b, rtol=1e-10)           # aac_gmres            (device tensors)
    x, info = s.gmres_host("nc2", 8, b_numpy)            # aac_gmres_host       (host arrays)
    xs, infos = s.gmres_host_batch("nc2", 8, [b0, b1])  # aac_gmres_host_batch (pipelined copies)

Block vectors are torch.float64 CUDA tensors of shape [ell, n_local] (or anything that
reshapes to it) holding this rank's slab; see include/aac.h for the layout.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import METHODS, aac_gmres_info, aac_grid, check, lib


def slab_range(n: int, nranks: int, rank: int):
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    check(lib.aac_slab_range(n, nranks, rank, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


class HostTransport:
    """aac_host_transport over a torch.distributed process group (e.g. "gloo"): the library
    stages every exchange through pinned host memory and these callbacks move it. Marshalling
    only -- no arithmetic of the method happens here (an all-reduce is a sum of the ranks'
    partial sums, as NCCL's would be)."""

    def __init__(self, group, rank: int, nranks: int):
        import torch.distributed as dist
        self.group, self.rank, self.nranks = group, rank, nranks
        self.error = None

        def allreduce(user, buf, n, op):
            try:
                if op == 2:                      # all-gather: rank r's n doubles at offset r * n
                    t = torch.from_numpy(np.ctypeslib.as_array(buf, shape=(n * self.nranks,)))
                    parts = list(t.view(self.nranks, n).unbind(0))
                    mine = parts[self.rank].clone()
                    dist.all_gather(parts, mine, group=self.group)
                    return 0
                t = torch.from_numpy(np.ctypeslib.as_array(buf, shape=(n,)))
                dist.all_reduce(t, op=dist.ReduceOp.MAX if op == 1 else dist.ReduceOp.SUM,
                                group=self.group)
                return 0
            except Exception as e:  # reported through aac_last_error as AAC_ENCCL
                self.error = e
                return -1

        def sendrecv(user, n, send_lo, recv_lo, send_hi, recv_hi):
            try:
                reqs = []
                for snd, rcv, peer in ((send_lo, recv_lo, self.rank - 1), (send_hi, recv_hi, self.rank + 1)):
                    if snd:
                        g = dist.get_global_rank(self.group, peer) if self.group is not None else peer
                        reqs.append(dist.isend(torch.from_numpy(np.ctypeslib.as_array(snd, shape=(n,))),
                                               g, group=self.group))
                        reqs.append(dist.irecv(torch.from_numpy(np.ctypeslib.as_array(rcv, shape=(n,))),
                                               g, group=self.group))
                for r in reqs:
                    r.wait()
                return 0
            except Exception as e:
                self.error = e
                return -1

        self._fns = (_lib.ALLREDUCE_FN(allreduce), _lib.SENDRECV_FN(sendrecv))   # keep alive
        self.struct = _lib.aac_host_transport(None, self._fns[0], self._fns[1])


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _method(m):
    return METHODS[m] if isinstance(m, str) else int(m)


class Solver:
    def __init__(self, dim, n, kx, ky=None, kz=None, c=0.0, ell=10, alpha=1e-4, *,
                 max_krylov=64, device=None, stream=None, rank=0, nranks=1, nccl_id=None,
                 host_group=None):
        n = tuple(int(v) for v in n) + (1,) * (3 - len(n))   # (nx, ny, nz)
        self.dim, self.n, self.ell, self.alpha, self.c = dim, n, ell, alpha, c
        self.rank, self.nranks = rank, nranks
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        torch.cuda.set_device(self.device)
        self.stream = torch.cuda.current_stream(self.device) if stream is None else stream
        g = aac_grid(dim, (ctypes.c_int64 * 3)(*n), rank, nranks)
        keep = []

        def arr(a):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=np.float64)
            keep.append(a)
            return _dptr(a)

        idbuf = None
        if nccl_id is not None:
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        ctx = ctypes.c_void_p()
        if host_group is not None:
            # slab exchanges through a host process group (verification without NCCL)
            self._transport = HostTransport(host_group, rank, nranks)
            check(lib.aac_setup_host_transport(ctypes.byref(g), arr(kx), arr(ky), arr(kz), float(c),
                                               int(ell), float(alpha), int(max_krylov),
                                               ctypes.c_void_p(self.stream.cuda_stream),
                                               ctypes.byref(self._transport.struct), ctypes.byref(ctx)))
        else:
            check(lib.aac_setup(ctypes.byref(g), arr(kx), arr(ky), arr(kz), float(c), int(ell),
                                float(alpha), int(max_krylov), ctypes.c_void_p(self.stream.cuda_stream),
                                idbuf, ctypes.byref(ctx)))
        self.ctx = ctx
        nl = ctypes.c_int64()
        mu0, mu1 = ctypes.c_double(), ctypes.c_double()
        check(lib.aac_query(ctx, 1, 1, ctypes.byref(mu0), ctypes.byref(mu1), None,
                            ctypes.byref(nl)), ctx)
        self.n_local, self.mu_min, self.mu_max = nl.value, mu0.value, mu1.value
        self.max_krylov = max_krylov

    # -- helpers -----------------------------------------------------------------------
    def _vec(self, t: torch.Tensor) -> torch.Tensor:
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64):
            raise TypeError("block vectors must be float64 CUDA tensors")
        if t.numel() != self.ell * self.n_local or not t.is_contiguous():
            raise ValueError(f"expected a contiguous tensor of {self.ell}x{self.n_local} doubles")
        return t

    def empty(self) -> torch.Tensor:
        return torch.empty(self.ell, self.n_local, dtype=torch.float64, device=self.device)

    # -- C ABI calls ---------------------------------------------------------------------
    def matvec(self, x, y=None):
        x = self._vec(x)
        y = self.empty() if y is None else self._vec(y)
        check(lib.aac_matvec(self.ctx, x.data_ptr(), y.data_ptr()), self.ctx)
        return y

    def precond_apply(self, method, k, r, z=None):
        r = self._vec(r)
        z = self.empty() if z is None else self._vec(z)
        check(lib.aac_precond_apply(self.ctx, _method(method), int(k), r.data_ptr(), z.data_ptr()),
              self.ctx)
        return z

    def gmres(self, method, k, b, x=None, rtol=1e-10, maxit=None):
        b = self._vec(b)
        x = self.empty() if x is None else self._vec(x)
        info = aac_gmres_info()
        rc = lib.aac_gmres(self.ctx, _method(method), int(k), b.data_ptr(), x.data_ptr(),
                           float(rtol), int(maxit or self.max_krylov), ctypes.byref(info))
        check(rc, self.ctx, ok=(_lib.AAC_OK, _lib.AAC_ENOCONV))
        return x, info.asdict()

    def gmres_host(self, method, k, b: np.ndarray, x: np.ndarray | None = None, rtol=1e-10,
                   maxit=None):
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.size != self.ell * self.n_local:
            raise ValueError("b has the wrong size")
        if x is None:
            x = np.empty_like(b)
        elif x.dtype != np.float64 or not x.flags.c_contiguous or x.size != self.ell * self.n_local:
            raise ValueError("x must be a C-contiguous float64 array of ell * n_local values")
        info = aac_gmres_info()
        rc = lib.aac_gmres_host(self.ctx, _method(method), int(k), _dptr(b), _dptr(x), float(rtol),
                                int(maxit or self.max_krylov), ctypes.byref(info))
        check(rc, self.ctx, ok=(_lib.AAC_OK, _lib.AAC_ENOCONV))
        return x, info.asdict()

    def gmres_host_batch(self, method, k, bs, xs=None, rtol=1e-10, maxit=None):
        """aac_gmres_host_batch: one solve per host right-hand side in `bs`, the copies in and
        out overlapped with the solves. Returns (xs, [info, ...])."""
        bs = [np.ascontiguousarray(b, dtype=np.float64) for b in bs]
        for b in bs:
            if b.size != self.ell * self.n_local:
                raise ValueError("b has the wrong size")
        xs = [np.empty_like(b) for b in bs] if xs is None else list(xs)
        if len(xs) != len(bs):
            raise ValueError("xs and bs differ in length")
        for x in xs:
            if x.dtype != np.float64 or not x.flags.c_contiguous or x.size != self.ell * self.n_local:
                raise ValueError("x must be a C-contiguous float64 array of ell * n_local values")
        n = len(bs)
        bp = (ctypes.POINTER(ctypes.c_double) * max(n, 1))(*[_dptr(b) for b in bs])
        xp = (ctypes.POINTER(ctypes.c_double) * max(n, 1))(*[_dptr(x) for x in xs])
        infos = (aac_gmres_info * max(n, 1))()
        rc = lib.aac_gmres_host_batch(self.ctx, _method(method), int(k), n, bp, xp, float(rtol),
                                      int(maxit or self.max_krylov), infos)
        check(rc, self.ctx, ok=(_lib.AAC_OK, _lib.AAC_ENOCONV))
        return xs, [infos[i].asdict() for i in range(n)]

    def allocation(self, method, k):
        al = (ctypes.c_int * self.ell)()
        check(lib.aac_query(self.ctx, _method(method), int(k), None, None, al, None), self.ctx)
        return list(al)

    # -- profiling -----------------------------------------------------------------------
    # -- paper-reproduction mode (aac_set_boundary / aac_set_bounds / aac_ci) -------------
    def set_boundary(self, bx=0.0, by=0.0, bz=0.0):
        check(lib.aac_set_boundary(self.ctx, float(bx), float(by), float(bz)), self.ctx)
        mu0, mu1 = ctypes.c_double(), ctypes.c_double()
        check(lib.aac_query(self.ctx, 1, 1, ctypes.byref(mu0), ctypes.byref(mu1), None, None), self.ctx)
        self.mu_min, self.mu_max = mu0.value, mu1.value

    def set_blocks(self, kx_blocks, ky_blocks=None, kz_blocks=None):
        """aac_set_blocks: varying diagonal blocks A_j (one face-diffusivity set per block, each
        in the setup layout); the preconditioners then use the mean block A_hat."""
        def stack(bl):
            if bl is None:
                return None
            a = np.ascontiguousarray(np.stack([np.asarray(b, dtype=np.float64) for b in bl]))
            if len(bl) != self.ell:
                raise ValueError(f"need {self.ell} blocks")
            return a
        kx, ky, kz = stack(kx_blocks), stack(ky_blocks), stack(kz_blocks)
        check(lib.aac_set_blocks(self.ctx, _dptr(kx), _dptr(ky) if ky is not None else None,
                                 _dptr(kz) if kz is not None else None), self.ctx)
        mu0, mu1 = ctypes.c_double(), ctypes.c_double()
        check(lib.aac_query(self.ctx, 1, 1, ctypes.byref(mu0), ctypes.byref(mu1), None, None), self.ctx)
        self.mu_min, self.mu_max = mu0.value, mu1.value

    def set_bounds(self, mu_min, mu_max):
        check(lib.aac_set_bounds(self.ctx, float(mu_min), float(mu_max)), self.ctx)
        self.mu_min, self.mu_max = float(mu_min), float(mu_max)

    def ci(self, method, k, b, x=None, *, lmin, lmax, tol=1e-6, maxit=1000):
        """The paper's outer CI (aac_ci): returns (x, info dict)."""
        b = self._vec(b)
        x = self.empty() if x is None else self._vec(x)
        info = aac_gmres_info()
        check(lib.aac_ci(self.ctx, _method(method), int(k), ctypes.c_void_p(b.data_ptr()),
                         ctypes.c_void_p(x.data_ptr()), float(lmin), float(lmax), float(tol),
                         int(maxit), ctypes.byref(info)), self.ctx, ok=(0, 1))
        return x, info.asdict()

    def profile(self, enable=True):
        check(lib.aac_profile_enable(self.ctx, int(enable)), self.ctx)

    def profile_reset(self):
        check(lib.aac_profile_reset(self.ctx), self.ctx)

    def profile_read(self):
        out = {}
        for i in range(lib.aac_profile_count()):
            name = ctypes.c_char_p()
            ms, nb = ctypes.c_double(), ctypes.c_double()
            nl = ctypes.c_longlong()
            check(lib.aac_profile_read(self.ctx, i, ctypes.byref(name), ctypes.byref(ms),
                                       ctypes.byref(nl), ctypes.byref(nb)), self.ctx)
            fl = ctypes.c_double()
            check(lib.aac_profile_flops(self.ctx, i, ctypes.byref(fl)), self.ctx)
            out[name.value.decode()] = {"ms": ms.value, "launches": nl.value, "model_bytes": nb.value,
                                        "model_flops": fl.value}
        return out

    def launch_count(self):
        return lib.aac_launch_count(self.ctx)

    def comm_kind(self):
        """0: one rank, no communicator; 1: NCCL; 2: host-staged transport (aac_comm_kind)."""
        return {0: "none", 1: "nccl", 2: "host"}[lib.aac_comm_kind(self.ctx)]

    def close(self):
        if getattr(self, "ctx", None):
            torch.cuda.current_stream(self.device).synchronize()
            lib.aac_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def from_problem(prob, *, rank=0, nranks=1, nccl_id=None, max_krylov=64, **kw) -> Solver:
    """Construct a Solver from a synth.Problem-like object (dim, shape, c, ell, alpha, kx..)."""
    nz, ny, nx = prob.shape
    s = Solver(prob.dim, (nx, ny, nz), prob.kx, prob.ky if prob.dim >= 2 else None,
               prob.kz if prob.dim >= 3 else None, prob.c, prob.ell, prob.alpha,
               rank=rank, nranks=nranks, nccl_id=nccl_id, max_krylov=max_krylov, **kw)
    bd = getattr(prob, "bd", (0.0, 0.0, 0.0))
    if any(bd):                                  # the paper's Dirichlet operator
        s.set_boundary(*bd)
    mb = getattr(prob, "mu_bounds", None)
    if mb is not None:
        s.set_bounds(*mb)
    kb = getattr(prob, "kx_blocks", None)
    if kb is not None:                           # varying diagonal blocks (N4)
        s.set_blocks(kb, prob.ky_blocks if prob.dim >= 2 else None, prob.kz_blocks if prob.dim >= 3 else None)
    return s
