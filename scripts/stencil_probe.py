"""Stencil (aac_matvec) throughput probe: eager back-to-back calls vs the same calls replayed
from a CUDA graph captured on the library stream.   python scripts/stencil_probe.py [config]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_03947_b200 import from_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "headline"
p = synth.make_problem(name)
s = from_problem(p, max_krylov=8, stream=torch.cuda.Stream())
st = s.stream
V = 8.0 * p.ell * p.N
C = 8.0 * p.dim * p.N
bytes_per = 2 * V + C
R = 30
xs = [s.empty().normal_() for _ in range(3)]
ys = s.empty()
peak = 6545.3
for rep in range(3):
    with torch.cuda.stream(st):
        for i in range(3):
            s.matvec(xs[i], ys)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for i in range(R):
            s.matvec(xs[i % 3], ys)
        b.record(st)
        torch.cuda.synchronize()
    ms = a.elapsed_time(b) / R
    print(f"eager: {ms * 1e3:.1f} us/apply, {bytes_per / ms / 1e6:.0f} GB/s = {100 * bytes_per / ms / 1e6 / peak:.1f}%")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for i in range(R):
        s.matvec(xs[i % 3], ys)
for rep in range(3):
    with torch.cuda.stream(st):
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        g.replay()
        b.record(st)
        torch.cuda.synchronize()
    ms = a.elapsed_time(b) / R
    print(f"graph: {ms * 1e3:.1f} us/apply, {bytes_per / ms / 1e6:.0f} GB/s = {100 * bytes_per / ms / 1e6 / peak:.1f}%")
s.close()
