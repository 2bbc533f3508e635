"""C-ABI checks that need no GPU: libaac.so loads, exports every symbol include/aac.h
declares, slab partitioning, and argument validation (AAC_EINVAL paths return before any
CUDA work)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "aac.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(aac_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2506_03947_b200 import _lib
    declared = _header_symbols()
    assert len(declared) >= 14
    so = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(so, name), name
    assert sorted(_lib.SYMBOLS) == declared


def test_library_is_sm100a():
    import subprocess
    from paper_2506_03947_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("n,P", [(1024, 1), (1024, 8), (256, 3), (17, 4), (10, 10)])
def test_slab_range_partition(n, P):
    from paper_2506_03947_b200 import slab_range
    rs = [slab_range(n, P, r) for r in range(P)]
    assert rs[0][0] == 0 and rs[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    sizes = [hi - lo for lo, hi in rs]
    assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1


def test_slab_range_rejects():
    from paper_2506_03947_b200 import AacError, slab_range
    for args in [(4, 0, 0), (4, 2, 2), (3, 4, 0), (4, 2, -1)]:
        with pytest.raises(AacError):
            slab_range(*args)


def _setup(dim=2, n=(8, 6, 1), ell=4, alpha=0.1, c=0.01, kx=None, ky=None, kz=None, nranks=1,
           max_krylov=4):
    from paper_2506_03947_b200 import _lib
    nx, ny, nz = n
    kx = np.ones((nz, ny, nx - 1)) if kx is None else kx
    ky = np.ones((nz, max(ny - 1, 0), nx)) if ky is None else ky
    dp = lambda a: None if a is None else np.ascontiguousarray(a).ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    g = _lib.aac_grid(dim, (ctypes.c_int64 * 3)(*n), 0, nranks)
    ctx = ctypes.c_void_p()
    rc = _lib.lib.aac_setup(ctypes.byref(g), dp(kx), dp(ky) if dim >= 2 else None, dp(kz), c, ell,
                            alpha, max_krylov, None, None, ctypes.byref(ctx))
    return rc, _lib.lib.aac_last_error(None).decode()


@pytest.mark.parametrize("kw,frag", [
    (dict(ell=5), "ell must be even"), (dict(ell=0), "ell must be even"),
    (dict(ell=18), "ell must be even"), (dict(alpha=-0.5), "alpha must be finite and > 0"),
    (dict(alpha=0.0), "alpha"), (dict(c=-1.0), "c must be"), (dict(max_krylov=0), "max_krylov"),
    (dict(dim=4), "dim"), (dict(n=(1, 6, 1)), "n >= 2"),
    (dict(kx=-np.ones((1, 6, 7))), "kappa must be finite"),
    (dict(kx=np.full((1, 6, 7), np.nan)), "kappa must be finite"),
    (dict(dim=1, n=(8, 1, 1), nranks=2), "one rank"),
])
def test_setup_validation(kw, frag):
    rc, msg = _setup(**kw)
    assert rc == -1 and frag in msg


def test_null_context_calls_fail_cleanly():
    """Every ctx-taking entry point returns AAC_EINVAL on a NULL context (no CUDA work)."""
    from paper_2506_03947_b200 import _lib
    L = _lib.lib
    assert L.aac_gmres_host_batch(None, 2, 8, 1, None, None, 1e-10, 10, None) == -1
    assert L.aac_gmres_host(None, 2, 8, None, None, 1e-10, 10, None) == -1
    assert L.aac_gmres(None, 2, 8, None, None, 1e-10, 10, None) == -1
    assert L.aac_matvec(None, None, None) == -1
