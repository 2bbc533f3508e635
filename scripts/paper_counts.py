"""Paper-mode reproduction report: outer CI iteration counts of the CUDA path
on the paper's own operator against Tables 3 and 4.

    python scripts/paper_counts.py [out.json]

For every printed cell with ell <= 16 (the library's AAC_MAX_ELL) it runs aac_ci with P_NC1 /
P_NC2 (budget ell*n_x*eta), foci of Cor. cor:extremeevals, r_p < 1e-6
(PAPER.md:647), on one GPU, seed 0, and prints ours vs the paper's count and total matvecs.
The printed values come from tests/golden/paper_nc{1,2}_tables.json (typed from PAPER.md, cited).
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_03947_b200 import from_problem  # noqa: E402

G = os.path.join(ROOT, "tests", "golden")
NC = {"nc1": json.load(open(os.path.join(G, "paper_nc1_tables.json"))),
      "nc2": json.load(open(os.path.join(G, "paper_nc2_tables.json")))}


def run_cell(nx, ell, alpha, eta, meth):
    p = synth.make_paper_problem(nx, ell, alpha, eta=eta, method=meth)
    s = from_problem(p, max_krylov=4)
    mu0 = p.mu_bounds[0]
    lo, hi = 1.0, mu0 ** ell / (mu0 ** ell - alpha)
    b = torch.from_numpy(np.ascontiguousarray(p.b.reshape(ell, -1))).cuda()
    _, info = s.ci(meth, p.k, b, lmin=lo, lmax=hi, tol=1e-6, maxit=3000)
    s.close()
    return info["iters"], info["matvecs_paper_units"], info["converged"]


def main():
    out = {"_source": "scripts/paper_counts.py (CUDA path, aac_ci) vs PAPER.md Tables 3/4", "cells": []}
    for meth in ("nc1", "nc2"):
        for tab in ("table3", "table4"):
            T = NC[meth][tab]
            for akey, alpha in (("alpha_0.01", 0.01), ("alpha_1", 1.0)):
                for key, cells in T[akey].items():
                    ell = T.get("ell", 10) if tab == "table3" else int(key)
                    nx = int(key) if tab == "table3" else T["nx"]
                    if ell > 16:
                        continue
                    for eta, (its_p, mv_p) in zip(T["eta"], cells):
                        its, mv, conv = run_cell(nx, ell, alpha, eta, meth)
                        row = {"table": tab, "method": meth, "alpha": alpha, "nx": nx, "ell": ell, "eta": eta,
                               "paper_its": its_p, "paper_matvecs": mv_p, "its": its, "matvecs": mv,
                               "converged": conv, "ratio": its / its_p}
                        out["cells"].append(row)
                        print(f"{tab} {meth} alpha={alpha:<5} nx={nx:<4} ell={ell:<3} eta={eta}: "
                              f"{its:4d} its ({mv:6d} mv) vs paper {its_p:4d} ({mv_p:6d})  x{its / its_p:.2f}",
                              flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
