"""Multi-rank (slab-decomposed) CUDA path vs the oracle, on ONE GPU.

Each rank is a separate process on cuda:0 owning one slab; the halo exchanges and the
all-reduces of the path run through the library's host-staged transport over a gloo process
group (include/aac.h, aac_setup_host_transport), so the ranks never run kernels that wait on
each other. This exercises every slab-specific piece of the CUDA path -- halo layers in the
stencil kernels, slab face weights, local partial sums + all-reduce in the Arnoldi and norm
steps, the Gershgorin max -- against the single-domain oracle. (The NCCL transport differs only
in who moves the same buffers; it needs one GPU per rank.) In 2D the Chebyshev solves run as
the slab-decomposed wavefront (halo rows of hat w exchanged once per apply) when every slab has
at least 8 rows, else as per-step sweeps. The saddle-point solver's multigrid
coarsens inside the slabs and gathers the first level whose slab boundaries are no longer
aggregate boundaries, so its hierarchy -- and its result -- equals the one-rank oracle's.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from oracle import chebyshev as ch  # noqa: E402
from oracle import gmres as og  # noqa: E402
from oracle import operator as op  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _stitch(parts, key, p):
    nz, ny, nx = p.shape
    blocks = []
    for d in parts:
        a = d[key].reshape(p.ell, -1)
        nl = d["hi"] - d["lo"]
        blocks.append(a.reshape((p.ell, nz, nl, nx) if p.dim == 2 else (p.ell, nl, ny, nx)))
    return np.concatenate(blocks, axis=2 if p.dim == 2 else 1).reshape(p.ell, -1)


def _rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b))


# sp: whether the saddle-point solver can run on that split (its multigrid coarsens inside the
# slabs, so every slab boundary must be even -- otherwise aac_* returns AAC_EINVAL)
CASES = [
    (2, dict(name="headline", kw=dict(shape=(1, 40, 29)), method="nc2", k=8, k_sp=3, sp=True)),
    (3, dict(name="headline", kw=dict(shape=(1, 36, 33)), method="nc2", k=8, k_sp=3, sp=True)),
    (2, dict(name="headline", kw=dict(shape=(1, 37, 29)), method="nc2", k=8, k_sp=3, sp=False)),
    # slabs thinner than the wavefront halo (9 rows): the per-step sweeps run instead
    (4, dict(name="headline", kw=dict(shape=(1, 26, 21)), method="nc2", k=8, k_sp=3, sp=False)),
    (2, dict(name="3d", kw=dict(shape=(12, 9, 8)), method="nc1", k=10, k_sp=2, sp=True)),
    (3, dict(name="3d", kw=dict(shape=(7, 6, 9), ell=4), method="nc2", k=5, k_sp=2, sp=False)),
]


@pytest.mark.parametrize("world,case", CASES)
def test_multirank_slabs_match_oracle(tmp_path, world, case):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(HERE, "_mr_worker.py"), str(tmp_path), json.dumps(case)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    parts = [dict(np.load(tmp_path / f"r{i}.npz")) for i in range(world)]
    p = synth.make_problem(case["name"], **case["kw"])
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    for d in parts:                                            # global Gershgorin all-reduce(max)
        assert float(d["mu_max"]) == pytest.approx(mu, rel=1e-14)
    rng = np.random.default_rng(case.get("seed", 5))
    x = rng.standard_normal((p.ell,) + p.shape)
    rr = rng.standard_normal((p.ell,) + p.shape)
    assert _rel(_stitch(parts, "y", p), op.apply_allatonce(w, x)) <= 1e-12
    if p.dim == 2:                                             # which NC organisation ran
        thick = min(d["hi"] - d["lo"] for d in parts) >= 9       # WAVE_MAXH + 1 (ghost row)
        assert all((float(d["wave_flops"]) > 0) == thick for d in parts)
    for m in ("nc1", "nc2"):
        al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * case["k"], m, case["k"])
        zo = ch.nc_apply(w, rr, p.ell, p.alpha, 1.0, mu, al)
        assert _rel(_stitch(parts, "z_" + m, p), zo) <= 1e-12, m
    al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * case["k"], case["method"], case["k"])
    ro = og.fgmres(lambda v: op.apply_allatonce(w, v),
                   lambda v: ch.nc_apply(w, v, p.ell, p.alpha, 1.0, mu, al), p.b, p.rtol, 60)
    its = {int(d["iters"]) for d in parts}
    assert len(its) == 1 and abs(its.pop() - ro.iters) <= 1
    assert _rel(_stitch(parts, "x", p), ro.x) <= 1e-9
    assert all(float(d["relres_true"]) <= 1.5 * p.rtol for d in parts)
    assert all(int(d["batch_same"]) == 1 for d in parts)        # aac_gmres_host_batch, SPMD
    if not case["sp"]:
        assert all(int(d["sp_error"]) == 1 for d in parts)    # odd slab boundary: clean error
        return
    from oracle import saddle
    assert all(int(d["sp_error"]) == 0 for d in parts), [str(d.get("sp_msg")) for d in parts]
    lev = saddle.hierarchy(w)
    zsp = saddle.sp_apply(w, rr, p.ell, p.alpha, case["k_sp"], lev)
    assert _rel(_stitch(parts, "z_sp", p), zsp) <= 1e-12
    rs = og.fgmres(lambda v: op.apply_allatonce(w, v),
                   lambda v: saddle.sp_apply(w, v, p.ell, p.alpha, case["k_sp"], lev), p.b, p.rtol, 60)
    its = {int(d["iters_sp"]) for d in parts}
    assert len(its) == 1 and abs(its.pop() - rs.iters) <= 1
    assert _rel(_stitch(parts, "x_sp", p), rs.x) <= 1e-9


def test_multirank_ghost_rows_bit_identical(tmp_path):
    """Ghost mode (the wavefront computes the slab ghost rows and Z_j's halo is formed locally,
    no exchange of Z_j) reproduces the exchange path (AAC_WAVE_GHOST=0) bit for bit: the ghost
    rows are the same point recurrences on the same inputs as the neighbour's own rows."""
    case = dict(name="headline", kw=dict(shape=(1, 40, 29)), method="nc2", k=8, k_sp=3, sp=False)
    outs = []
    for flag in ("1", "0"):
        d = tmp_path / f"g{flag}"
        d.mkdir()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
               "--master-addr=127.0.0.1", f"--master-port={_port()}",
               os.path.join(HERE, "_mr_worker.py"), str(d), json.dumps(case)]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                           env={**os.environ, "AAC_WAVE_GHOST": flag})
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        outs.append([dict(np.load(d / f"r{i}.npz")) for i in range(2)])
    for a, b in zip(*outs):
        for key in ("x", "z_nc1", "z_nc2"):
            assert np.array_equal(a[key], b[key]), key
        assert int(a["iters"]) == int(b["iters"])
        # ghost mode ran: one ghost-row inverse transform per step on each rank (one neighbour)
        assert int(a["gmres_launches"]) - int(b["gmres_launches"]) >= int(a["iters"])
