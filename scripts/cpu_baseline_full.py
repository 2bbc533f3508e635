"""the oracle's full FGMRES solves on the host, one BLAS thread enforced
and all cores, with the host recorded.  Oracle only -- no CUDA path is imported.

    python scripts/cpu_baseline_full.py [OUT.json] [config ...]

Configs: 1d, 2d256, headline, saddle, 3d64 (BASELINE.json configs[4] at 64^3, the size the
oracle finishes in seconds).  Each is solved to convergence once per thread setting; its/s =
FGMRES iterations / wall seconds of the solve (setup of the Chebyshev allocation / the SP
hierarchy excluded, as in bench.py's device-side figure).
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
from threadpoolctl import threadpool_info, threadpool_limits  # noqa: E402

import synth  # noqa: E402
from oracle import chebyshev as ch  # noqa: E402
from oracle import gmres as og  # noqa: E402
from oracle import operator as op  # noqa: E402
from oracle import saddle  # noqa: E402


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = os.cpu_count()
    return {"os_cpu_count": os.cpu_count(), "affinity_cpus": aff, "cpu_model": model,
            "blas": [{k: d.get(k) for k in ("internal_api", "num_threads", "version")} for d in threadpool_info()]}


def problem(name):
    if name == "3d64":
        return synth.make_problem("3d", n=64)
    return synth.make_problem(name)


def solve(name, threads):
    p = problem(name)
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    if p.method == "sp":
        lev = saddle.hierarchy(w)
        prec = lambda r: saddle.sp_apply(w, r, p.ell, p.alpha, p.k, lev)  # noqa: E731
    else:
        al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * p.k, p.method, p.k)
        prec = lambda r: ch.nc_apply(w, r, p.ell, p.alpha, 1.0, mu, al)  # noqa: E731
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        res = og.fgmres(lambda x: op.apply_allatonce(w, x), prec, p.b, p.rtol, 200)
        dt = time.perf_counter() - t0
    tr = float(np.linalg.norm(p.b - op.apply_allatonce(w, res.x)) / np.linalg.norm(p.b))
    return {"threads": threads, "iters": int(res.iters), "converged": bool(res.converged),
            "seconds": dt, "its_per_s": res.iters / dt, "relres_true": tr,
            "unknowns": int(p.b.size)}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02", "cpu_baseline_full.json")
    names = sys.argv[2:] or ["1d", "2d256", "3d64", "headline", "saddle"]
    host = host_info()
    allc = host["affinity_cpus"]
    rep = {"_source": "scripts/cpu_baseline_full.py (oracle/ only)", "host": host, "configs": {}}
    for n in names:
        rep["configs"][n] = {"one_core": solve(n, 1), "all_cores": solve(n, allc)}
        print(n, json.dumps(rep["configs"][n]), flush=True)
        with open(out, "w") as f:
            json.dump(rep, f, indent=1)


if __name__ == "__main__":
    main()
