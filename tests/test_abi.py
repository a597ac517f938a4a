"""C-ABI library checks that need no GPU: it builds, loads, exports every symbol declared in
include/rw.h, and rejects invalid arguments before touching the device."""
import ctypes as C
import subprocess

import pytest

from paper_2103_09564_b200 import build as B
from paper_2103_09564_b200 import _lib


@pytest.fixture(scope="module")
def lib():
    B.build()
    return _lib.lib()


def test_exports_every_header_symbol(lib):
    syms = _lib.header_symbols()
    assert len(syms) >= 14
    out = subprocess.run(["nm", "-D", "--defined-only", B.LIB], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        assert hasattr(lib, s)
    assert set(_lib.SIGNATURES) == set(syms)


def test_built_for_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_version(lib):
    assert b"sm_100a" in lib.rw_version()


def _solve(lib, **kw):
    a = dict(batch=1, d=_lib.rw_dims(8, 4, 4), vol=C.c_void_p(4096), dtype=3,
             nm=_lib.rw_norm(1, 0), W=None, fixed=C.c_void_p(8192), values=C.c_void_p(16384),
             nrhs=1, beta=100.0, eps=1e-6, tol=1e-6, max_iter=10, tol_mode=0, x0=None,
             ws=C.c_void_p(1 << 20), ws_bytes=1 << 40, prob=C.c_void_p(32768),
             iters=C.c_void_p(65536), resid=None, status=None, labels=None, stream=None)
    a.update(kw)
    return lib.rw_solve_bricks(a["batch"], a["d"], a["vol"], a["dtype"], a["nm"], a["W"],
                               a["fixed"], a["values"], a["nrhs"], a["beta"], a["eps"],
                               a["tol"], a["max_iter"], a["tol_mode"], a["x0"], a["ws"],
                               a["ws_bytes"], a["prob"], a["iters"], a["resid"], a["status"],
                               a["labels"], a["stream"])


@pytest.mark.parametrize("kw,frag", [
    (dict(d=_lib.rw_dims(6, 4, 4)), b"nx"),
    (dict(d=_lib.rw_dims(8, 0, 4)), b"dims"),
    (dict(batch=0), b"batch"),
    (dict(eps=0.0), b"eps"),
    (dict(tol=0.0), b"tol"),
    (dict(max_iter=0), b"max_iter"),
    (dict(tol_mode=3), b"tol_mode"),
    (dict(nrhs=0), b"nrhs"),
    (dict(W=C.c_void_p(4096)), b"exactly one"),
    (dict(vol=None), b"exactly one"),
    (dict(ws=C.c_void_p((1 << 20) + 16)), b"aligned"),
    (dict(prob=C.c_void_p(32768 + 4)), b"aligned"),
    (dict(fixed=None), b"non-NULL"),
    (dict(ws_bytes=100), b"workspace too small"),
])
def test_solve_rejects_invalid_arguments_before_enqueue(lib, kw, frag):
    st = _solve(lib, **kw)
    assert st in (1, 3)
    assert frag in lib.rw_last_error()


def test_workspace_bytes_monotone(lib):
    d = _lib.rw_dims(64, 64, 64)
    a = lib.rw_solve_workspace_bytes(1, d, 1, 0)
    b = lib.rw_solve_workspace_bytes(2, d, 1, 0)
    c = lib.rw_solve_workspace_bytes(2, d, 1, 1)
    assert 0 < a < b and c < b
    assert lib.rw_solve_workspace_bytes(1, _lib.rw_dims(6, 4, 4), 1, 0) == 0
    assert lib.rw_solve_labels_workspace_bytes(1, d, 4, 0) > lib.rw_solve_workspace_bytes(1, d, 3, 0)


def test_pyramid_and_queue_validation(lib):
    arr = (C.c_void_p * 2)(4096, 8192)
    st = lib.rw_build_pyramid_slab(C.c_void_p(4096), 1, _lib.rw_dims(64, 64, 64), 3, 8, 2, arr, None)
    assert st == 1 and b"multiple" in lib.rw_last_error()
    assert lib.rw_build_pyramid(C.c_void_p(4096), 1, _lib.rw_dims(64, 64, 64), 0, arr, None) == 1
    q = C.c_void_p()
    assert lib.rw_queue_create(1024, 1, C.byref(q)) == 1


def test_hier_labels_ooc_validation(lib):
    """rw_hier_segment_labels_ooc rejects K outside 2..255 and NULL outputs before any work
    (no CUDA call is reached)."""
    cfg = _lib.rw_hier_config(32, 1.25, 0.3, -1.0, 1, 100.0, 1e-6, 1e-6, 100, 0, 64, 0, 0.01)
    d = _lib.rw_dims(64, 64, 64)
    nm = _lib.rw_norm(1.0 / 65535, 0.0)
    p = C.c_void_p(4096)
    args = lambda K, best, lab: (p, 1, nm, d, p, K, cfg, 16, p, p, 1 << 20, best, lab, None, None)  # noqa: E731
    assert lib.rw_hier_segment_labels_ooc(*args(1, p, p)) == 1
    assert b"K must be in 2..255" in lib.rw_last_error()
    assert lib.rw_hier_segment_labels_ooc(*args(256, p, p)) == 1
    assert lib.rw_hier_segment_labels_ooc(*args(3, None, p)) == 1
    assert b"non-NULL" in lib.rw_last_error()
    assert lib.rw_hier_segment_labels_ooc(*args(3, p, None)) == 1
