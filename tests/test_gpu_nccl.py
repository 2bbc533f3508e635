"""The NCCL data plane on one GPU.

This pool gives one GPU per call, and NCCL cannot put two ranks on one device, so the
multi-rank exchange itself is exercised here through a ONE-RANK NCCL communicator
(AAC_NCCL_SELF=1, include/aac.h aac_comm_kind): libnccl is loaded, the communicator is
initialised, and every Arnoldi step runs the multi-rank code path -- per-rank partial sums,
ncclAllReduce captured in the step's CUDA graph, the scalar kernels after it. On one rank the
all-reduce is the identity, so the result must be BIT-IDENTICAL to the plain one-rank path,
and both must match the oracle. The halo exchanges of real slabs run in tests/test_gpu_multirank.py
(host transport) and tests/test_multirank_gloo.py (CPU).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import synth  # noqa: E402
from oracle import chebyshev as ch  # noqa: E402
from oracle import gmres as og  # noqa: E402
from oracle import operator as op  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dev(a, ell):
    return torch.from_numpy(np.ascontiguousarray(a).reshape(ell, -1)).cuda()


def _solve(p, method, k, maxit=60, **env):
    from paper_2506_03947_b200 import from_problem
    old = {v: os.environ.get(v) for v in env}
    os.environ.update(env)
    try:
        s = from_problem(p, max_krylov=maxit)
        kind = s.comm_kind()
        x, info = s.gmres(method, k, _dev(p.b, p.ell), rtol=p.rtol, maxit=maxit)
        r = np.random.default_rng(3).standard_normal((p.ell,) + p.shape)
        z = s.precond_apply(method, k, _dev(r, p.ell)).cpu().numpy()
        out = x.cpu().numpy(), info, z, kind
        s.close()
        return out
    finally:
        for v, val in old.items():
            if val is None:
                os.environ.pop(v, None)
            else:
                os.environ[v] = val


CASES = [
    ("headline", dict(shape=(1, 130, 67)), "nc2", 8, {}),
    ("headline", dict(shape=(1, 130, 67)), "nc2", 8, {"AAC_NO_GRAPH": "1"}),
    ("3d", dict(shape=(9, 13, 11)), "nc1", 10, {}),
    ("saddle", dict(shape=(1, 48, 40)), "sp", 8, {}),
]


@pytest.mark.parametrize("name,kw,method,k,extra", CASES)
def test_nccl_one_rank_bit_identical(name, kw, method, k, extra):
    p = synth.make_problem(name, **kw)
    # the NCCL path runs one-reduce Arnoldi by default (krylov.cuh arnoldi_lagged_step): the
    # one-rank reference runs it too
    x0, i0, z0, kind0 = _solve(p, method, k, AAC_GMRES_1R="1", **extra)
    x1, i1, z1, kind1 = _solve(p, method, k, AAC_NCCL_SELF="1", **extra)
    assert kind0 == "none" and kind1 == "nccl"
    assert i1["iters"] == i0["iters"] and i1["converged"] == 1
    assert np.array_equal(x1, x0), "NCCL path must reproduce the one-rank result bit for bit"
    assert np.array_equal(z1, z0)
    if method != "sp":
        w = op.weights(p)
        mu = op.gershgorin_max(w)
        al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * k, method, k)
        ro = og.fgmres(lambda v: op.apply_allatonce(w, v),
                       lambda v: ch.nc_apply(w, v, p.ell, p.alpha, 1.0, mu, al), p.b, p.rtol, 60)
        assert abs(i1["iters"] - ro.iters) <= 1
        assert np.linalg.norm(x1.ravel() - ro.x.ravel()) <= 1e-9 * np.linalg.norm(ro.x)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_bench_under_torchrun_with_nccl():
    """bench.py --gpus 1 launched the way the driver launches N > 1 (torch.distributed.run),
    with the one-rank NCCL communicator: the JSON contract holds and the solve converges."""
    env = dict(os.environ, AAC_NCCL_SELF="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "1",
           "--steps", "2", "--warmup", "1", "--config", "2d256", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    for key in ("metric", "value", "unit", "n_gpus", "ms_per_step", "e2e", "roofline", "clocks", "gpu_launches"):
        assert key in line
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["config"]["comm"] == "nccl"
    assert line["config"]["relres_true"] <= 1.5e-10
