"""Minimal driver for profiling: set up a config and run a few GMRES solves on cuda:0.

    python scripts/one_solve.py [config] [n_solves] [method] [k]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_03947_b200 import from_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "headline"
nsol = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = synth.make_problem(name)
method = sys.argv[3] if len(sys.argv) > 3 else p.method
k = int(sys.argv[4]) if len(sys.argv) > 4 else p.k
maxk = int(os.environ.get("AAC_MAXK", "20" if p.dim == 3 else "60"))
s = from_problem(p, max_krylov=maxk)
b = torch.from_numpy(p.b.reshape(p.ell, -1)).cuda()
for i in range(nsol):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, info = s.gmres(method, k, b, rtol=p.rtol, maxit=maxk)
    torch.cuda.synchronize()
    print(f"solve {i}: {info['iters']} its, {1e3 * (time.perf_counter() - t0):.2f} ms, "
          f"relres_true {info['relres_true']:.2e}")
s.close()
