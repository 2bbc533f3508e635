"""Write tests/golden/oracle_<config>.json from the ORACLE only (no CUDA path involved).

Full-size configs are too slow for the oracle inside a test, so this committed script runs
the oracle's FGMRES once and stores what the GPU parity test compares against: the
iteration count, the residual history, ||x||, and x at fixed sampled indices.

    python scripts/make_oracle_golden.py headline [saddle ...] [paper500]

`paper500`: the paper's own operator (n_x = 500, ell = 10) with the paper's outer solver,
unpreconditioned CI to 1e-6 (PAPER.md:866 prints 1282 iterations).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import chebyshev as ch  # noqa: E402
from oracle import gmres as og  # noqa: E402
from oracle import operator as op  # noqa: E402
from oracle import outer  # noqa: E402
from oracle import paper  # noqa: E402
from oracle import saddle  # noqa: E402

NSAMPLE = 256


def run_paper500(seed: int = 0):
    nx, ell = 500, 10
    p = synth.make_paper_problem(nx, ell, 0.01, seed=seed)
    w = paper.weights(nx, ell)
    lo, hi = paper.bounds(nx, ell)
    t0 = time.time()
    res = outer.ci_outer(lambda x: op.apply_allatonce(w, x), None, p.b, lo, hi, tol=1e-6, maxit=3000)
    dt = time.time() - t0
    x = res.x.reshape(-1)
    rng = np.random.default_rng(12345)
    idx = np.sort(rng.choice(x.size, NSAMPLE, replace=False))
    out = {
        "_source": "scripts/make_oracle_golden.py (oracle/ only; no CUDA path)",
        "config": "paper500", "seed": seed, "method": "none", "tol": 1e-6, "lmin": lo, "lmax": hi,
        "iters": res.iters, "converged": res.converged, "final_relres": res.history[-1],
        "x_norm": float(np.linalg.norm(x)), "sample_idx": idx.tolist(), "sample_x": x[idx].tolist(),
        "oracle_seconds": dt,
    }
    path = os.path.join(ROOT, "tests", "golden", "oracle_paper500.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"paper500: {res.iters} its, {dt:.1f} s -> {path}")


def run(name: str, seed: int = 0):
    if name == "paper500":
        return run_paper500(seed)
    p = synth.make_problem(name, seed=seed)
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    t0 = time.time()
    if p.method == "sp":
        lev = saddle.hierarchy(w)
        prec = lambda r: saddle.sp_apply(w, r, p.ell, p.alpha, p.k, lev)  # noqa: E731
        alloc = [p.k] * p.ell
    else:
        alloc = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * p.k, p.method, p.k)
        prec = lambda r: ch.nc_apply(w, r, p.ell, p.alpha, 1.0, mu, alloc)  # noqa: E731
    res = og.fgmres(lambda x: op.apply_allatonce(w, x), prec, p.b, p.rtol, 200)
    dt = time.time() - t0
    x = res.x.reshape(-1)
    rng = np.random.default_rng(12345)
    idx = np.sort(rng.choice(x.size, NSAMPLE, replace=False))
    tr = float(np.linalg.norm(p.b - op.apply_allatonce(w, res.x)) / np.linalg.norm(p.b))
    out = {
        "_source": "scripts/make_oracle_golden.py (oracle/ only; no CUDA path)",
        "config": name, "seed": seed, "method": p.method, "k": p.k, "rtol": p.rtol,
        "mu_max": mu, "alloc": alloc, "iters": res.iters, "converged": res.converged,
        "history": res.history, "relres_true": tr, "x_norm": float(np.linalg.norm(x)),
        "sample_idx": idx.tolist(), "sample_x": x[idx].tolist(), "oracle_seconds": dt,
    }
    path = os.path.join(ROOT, "tests", "golden", f"oracle_{name}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"{name}: {res.iters} its, true relres {tr:.2e}, {dt:.1f} s -> {path}")


if __name__ == "__main__":
    for n in sys.argv[1:] or ["headline"]:
        run(n)
