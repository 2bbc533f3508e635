"""Multi-rank host logic on CPU (world_size 2 and 3, gloo backend, 127.0.0.1).

The slab decomposition of the CUDA path is exercised without a GPU:
each rank takes its slab from `aac_slab_range`, its face weights in the exact device layout
from `aac_slab_weights` (the host code aac_setup runs), exchanges the boundary layers of every
plane with its neighbours by the same protocol as comm_halo (first layer -> rank-1, last
layer -> rank+1, received into halo_lo / halo_hi), applies calA on its slab, and the
gathered result must equal the oracle's global calA apply; the Gershgorin bound and a GMRES
inner product are all-reduced as the library does (max / sum).
"""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _slab_weights(p, rank, world):
    from paper_2506_03947_b200 import _lib
    nz, ny, nx = p.shape
    g = _lib.aac_grid(p.dim, (ctypes.c_int64 * 3)(nx, ny, nz), rank, world)
    dp = lambda a: np.ascontiguousarray(a).ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
    keep = [np.ascontiguousarray(p.kx), np.ascontiguousarray(p.ky), np.ascontiguousarray(p.kz)]
    lens = (ctypes.c_int64 * 3)()
    gm = ctypes.c_double()
    args = (ctypes.byref(g), dp(keep[0]), dp(keep[1]) if p.dim >= 2 else None,
            dp(keep[2]) if p.dim >= 3 else None, p.c)
    _lib.check(_lib.lib.aac_slab_weights(*args, None, lens, ctypes.byref(gm)))
    w = np.zeros(sum(lens))
    _lib.check(_lib.lib.aac_slab_weights(*args, w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                         lens, ctypes.byref(gm)))
    return w[:lens[0]], w[lens[0]:lens[0] + lens[1]], w[lens[0] + lens[1]:], gm.value


def _local_apply(p, u, wx, wy, wz, hlo, hhi):
    """(A u) on the slab from the device-layout weights; u: (lnz, lny, nx)."""
    lnz, lny, nx = u.shape
    N = u.size
    S = nx * lny if p.dim == 3 else nx
    f = u.ravel()
    out = f.copy()
    idx = np.arange(N)
    x = idx % nx
    y = (idx // nx) % lny
    z = idx // (nx * lny)
    left = np.where(x > 0, f[np.maximum(idx - 1, 0)], f)
    right = np.where(x < nx - 1, f[np.minimum(idx + 1, N - 1)], f)
    out += wx[idx] * (f - left) + wx[idx + 1] * (f - right)
    if p.dim == 2:
        north = np.where(y > 0, f[np.maximum(idx - nx, 0)], hlo[x] if hlo is not None else f)
        south = np.where(y < lny - 1, f[np.minimum(idx + nx, N - 1)], hhi[x] if hhi is not None else f)
        out += wy[idx] * (f - north) + wy[idx + nx] * (f - south)
    if p.dim == 3:
        north = np.where(y > 0, f[np.maximum(idx - nx, 0)], f)
        south = np.where(y < lny - 1, f[np.minimum(idx + nx, N - 1)], f)
        li = idx % S
        down = np.where(z > 0, f[np.maximum(idx - S, 0)], hlo[li] if hlo is not None else f)
        up = np.where(z < lnz - 1, f[np.minimum(idx + S, N - 1)], hhi[li] if hhi is not None else f)
        out += wy[idx] * (f - north) + wy[idx + nx] * (f - south)
        out += wz[idx] * (f - down) + wz[idx + S] * (f - up)
    return out.reshape(u.shape)


def _worker(rank, world, port, name, kw, errq):
    try:
        import torch

        import synth
        from oracle import operator as op
        from paper_2506_03947_b200 import slab_range
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        p = synth.make_problem(name, **kw)
        nz, ny, nx = p.shape
        nslab = ny if p.dim == 2 else nz
        lo, hi = slab_range(nslab, world, rank)
        wx, wy, wz, gm = _slab_weights(p, rank, world)
        # Gershgorin: all-reduce max
        t = torch.tensor([gm], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        w = op.weights(p)
        assert t.item() == pytest.approx(op.gershgorin_max(w), rel=1e-14)
        # local slab of a global block vector
        xg = np.random.default_rng(9).standard_normal((p.ell,) + p.shape)
        xl = np.ascontiguousarray(xg[:, lo:hi] if p.dim == 3 else xg[:, :, lo:hi])
        lay = lambda a: a.reshape(p.ell, -1)  # noqa: E731
        S = nx * ny if p.dim == 3 else nx
        flat = lay(xl)
        hlo = np.zeros((p.ell, S)) if rank > 0 else None
        hhi = np.zeros((p.ell, S)) if rank < world - 1 else None
        # halo protocol of comm_halo: first layer -> rank-1, last layer -> rank+1
        reqs = []
        for j in range(p.ell):
            if rank > 0:
                reqs.append(dist.isend(torch.from_numpy(flat[j, :S].copy()), rank - 1, tag=2 * j))
            if rank < world - 1:
                reqs.append(dist.isend(torch.from_numpy(flat[j, -S:].copy()), rank + 1, tag=2 * j + 1))
        for j in range(p.ell):
            if rank > 0:
                buf = torch.empty(S, dtype=torch.float64)
                dist.recv(buf, rank - 1, tag=2 * j + 1)
                hlo[j] = buf.numpy()
            if rank < world - 1:
                buf = torch.empty(S, dtype=torch.float64)
                dist.recv(buf, rank + 1, tag=2 * j)
                hhi[j] = buf.numpy()
        for r in reqs:
            r.wait()
        # y_j = A x_j - x_{j-1} on the slab
        y = np.empty_like(xl)
        for j in range(p.ell):
            y[j] = _local_apply(p, xl[j], wx, wy, wz, None if hlo is None else hlo[j],
                                None if hhi is None else hhi[j])
            if j > 0:
                y[j] -= xl[j - 1]
        yg = op.apply_allatonce(w, xg)
        yl_ref = yg[:, lo:hi] if p.dim == 3 else yg[:, :, lo:hi]
        assert np.linalg.norm(y - yl_ref) <= 1e-13 * np.linalg.norm(yl_ref)
        # distributed inner product (sum all-reduce of slab partials)
        d = torch.tensor([float(np.dot(y.ravel(), xl.ravel()))], dtype=torch.float64)
        dist.all_reduce(d)
        assert d.item() == pytest.approx(float(np.dot(yg.ravel(), xg.ravel())), rel=1e-12)
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced in the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,kw", [("headline", dict(shape=(1, 23, 17))),
                                     ("3d", dict(shape=(7, 6, 5), ell=4))])
def test_slab_halo_matvec_gloo(world, name, kw):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, kw, errq)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
