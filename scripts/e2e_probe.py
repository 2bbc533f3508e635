"""Probe the end-to-end path: pinned H2D / D2H bandwidth, then batch vs serial host solves."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_03947_b200 import from_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "headline"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
p = synth.make_problem(name)
s = from_problem(p)
b = np.ascontiguousarray(p.b.reshape(p.ell, -1))
bh = torch.from_numpy(b).pin_memory()
xh = torch.empty_like(bh).pin_memory()
d = torch.empty_like(bh, device="cuda")
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    d.copy_(bh, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter()
    xh.copy_(d, non_blocking=True); torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"H2D {bh.nbytes / (t1 - t) / 1e9:.1f} GB/s  D2H {bh.nbytes / (t2 - t1) / 1e9:.1f} GB/s")
meth, k = p.method, p.k
bd = bh.cuda()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    its = 0
    for _ in range(K):
        _, info = s.gmres(meth, k, bd, rtol=p.rtol)
        its += info["iters"]
    torch.cuda.synchronize(); dev = its / (time.perf_counter() - t)
    t = time.perf_counter()
    _, infos = s.gmres_host_batch(meth, k, [bh.numpy()] * K, [xh.numpy()] * K, rtol=p.rtol)
    bat = sum(i["iters"] for i in infos) / (time.perf_counter() - t)
    t = time.perf_counter()
    its = 0
    for _ in range(K):
        _, info = s.gmres_host(meth, k, bh.numpy(), xh.numpy(), rtol=p.rtol)
        its += info["iters"]
    ser = its / (time.perf_counter() - t)
    print(f"device {dev:.1f}  batch {bat:.1f}  serial {ser:.1f} its/s")
