"""One rank of the multi-rank GPU parity test (tests/test_gpu_multirank.py), launched by
torchrun. Every rank owns a slab on cuda:0 (ranks share the GPU: the slab exchanges go
through the host-staged transport over a gloo process group, so no kernel ever waits on
another rank's kernel). Writes this rank's slab results to OUTDIR/r{rank}.npz.

    python -m torch.distributed.run --nproc-per-node P tests/_mr_worker.py OUTDIR CASE_JSON
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2506_03947_b200 import AacError, from_problem, slab_range  # noqa: E402


def main():
    outdir, case = sys.argv[1], json.loads(sys.argv[2])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    p = synth.make_problem(case["name"], **case["kw"])
    nz, ny, nx = p.shape
    n_slab = ny if p.dim == 2 else nz
    lo, hi = slab_range(n_slab, world, rank)
    s = from_problem(p, rank=rank, nranks=world, host_group=dist.group.WORLD, max_krylov=60)

    def local(a):                                  # [ell, nz, ny, nx] -> this rank's slab
        a = a.reshape(p.ell, nz, ny, nx)
        a = a[:, lo:hi] if p.dim == 3 else a[:, :, lo:hi]
        return torch.from_numpy(np.ascontiguousarray(a).reshape(p.ell, -1)).cuda()

    rng = np.random.default_rng(case.get("seed", 5))
    x = rng.standard_normal((p.ell,) + p.shape)
    r = rng.standard_normal((p.ell,) + p.shape)
    out = {"lo": lo, "hi": hi, "mu_max": s.mu_max}
    out["y"] = s.matvec(local(x)).cpu().numpy()
    s.profile_reset()
    s.profile(True)
    for m in ("nc1", "nc2"):
        out["z_" + m] = s.precond_apply(m, case["k"], local(r)).cpu().numpy()
    prof = s.profile_read()
    s.profile(False)
    out["wave_flops"] = prof["cheb_sweep"]["model_flops"]     # > 0 only for the wavefront kernel
    l0 = s.launch_count()
    xs, info = s.gmres(case["method"], case["k"], local(p.b), rtol=p.rtol, maxit=60)
    out["gmres_launches"] = s.launch_count() - l0
    out["x"] = xs.cpu().numpy()
    out["iters"] = info["iters"]
    out["relres_true"] = info["relres_true"]
    # the pipelined host API on the slabs (SPMD): two systems, each bit-identical to aac_gmres
    bl = local(p.b).cpu().numpy()
    xsb, infb = s.gmres_host_batch(case["method"], case["k"], [bl, bl], rtol=p.rtol, maxit=60)
    out["batch_same"] = int(all(np.array_equal(xb, out["x"]) for xb in xsb) and
                            all(i["iters"] == info["iters"] for i in infb))
    try:                                           # SP needs even slab boundaries
        out["z_sp"] = s.precond_apply("sp", case["k_sp"], local(r)).cpu().numpy()
        xsp, isp = s.gmres("sp", case["k_sp"], local(p.b), rtol=p.rtol, maxit=60)
        out["x_sp"] = xsp.cpu().numpy()
        out["iters_sp"] = isp["iters"]
        out["sp_error"] = 0
    except AacError as e:
        out["sp_error"] = 1
        out["sp_msg"] = str(e)
    s.close()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
