"""Thin Python binding over librw (include/rw.h) -- marshalling only.

PyTorch provides device memory and streams; every step of the hot path runs in the
CUDA kernels behind the C ABI.  Function names follow the ABI without the ``rw_`` prefix.
Tensors are contiguous, [batch, nz, ny, nx] (x fastest); per-RHS tensors add a leading
[nrhs] axis.
"""
from __future__ import annotations

import contextlib
import ctypes as C

import torch

from ._lib import lib, check, rw_dims, rw_norm, rw_weight_spec, rw_hier_config, rw_hier_stats

DTYPES = {torch.uint8: 0, torch.uint16: 1, torch.int16: 2, torch.float32: 3}
DEFAULT_NORM = {torch.uint8: (1 / 255, 0.0), torch.uint16: (1 / 65535, 0.0),
                torch.int16: (1 / 2000, 0.5), torch.float32: (1.0, 0.0)}

ST_NAMES = {1: "converged", 2: "maxiter", 3: "trivial", 4: "zero_b", 5: "breakdown"}


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None, device=None):
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return C.c_void_p(s.cuda_stream)


def _retain(stream, *ts):
    """Tensors this binding allocated (workspace, outputs) are used by work enqueued on
    ``stream``; the calls return before that work ends (rw.h: stream-ordered).  When
    ``stream`` is not torch's current stream, tell the caching allocator so it does not
    hand their memory to new work before the stream reaches this point."""
    if stream is None:
        return
    for t in ts:
        if t is not None and t.is_cuda:
            t.record_stream(stream)


def _need(t, name, dtype=None):
    if t is None:
        return
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")


def dims_of(t):
    *_, nz, ny, nx = t.shape
    return rw_dims(nx, ny, nz)


SOLVERS = {"auto": 0, "streaming": 1, "resident": 2}


def set_solver(name):
    """rw_set_option(RW_OPT_SOLVER): "auto" | "streaming" | "resident" (include/rw.h)."""
    check(lib().rw_set_option(0, SOLVERS[name]), "rw_set_option")


def get_solver():
    v = lib().rw_get_option(0)
    return {v_: k for k, v_ in SOLVERS.items()}[v]


@contextlib.contextmanager
def solver(name):
    """Run the enclosed solves with the given solver, restoring the previous setting."""
    old = get_solver()
    set_solver(name)
    try:
        yield
    finally:
        set_solver(old)


def set_resident_wide(on):
    """rw_set_option(RW_OPT_RESIDENT_WIDE): latency-shaped clusters for 40^3 / 32^3 bricks."""
    check(lib().rw_set_option(4, int(bool(on))), "rw_set_option")


def get_resident_wide():
    return bool(lib().rw_get_option(4))


def set_device_loop(on):
    """rw_set_option(RW_OPT_DEVICE_LOOP): 1 (default) = the streaming CG loop runs on the
    device (one CUDA graph with a conditional WHILE node, the call does not block the host);
    0 = host-driven loop."""
    check(lib().rw_set_option(5, int(bool(on))), "rw_set_option")


def get_device_loop():
    return bool(lib().rw_get_option(5))


@contextlib.contextmanager
def device_loop(on):
    old = get_device_loop()
    set_device_loop(on)
    try:
        yield
    finally:
        set_device_loop(old)


def set_stream_passes(n):
    """rw_set_option(RW_OPT_STREAM_PASSES): 1 (default, one fused pass per streaming CG
    iteration) or 2 (classical passes A + B)."""
    check(lib().rw_set_option(3, int(n)), "rw_set_option")


def get_stream_passes():
    return int(lib().rw_get_option(3))


@contextlib.contextmanager
def stream_passes(n):
    old = get_stream_passes()
    set_stream_passes(n)
    try:
        yield
    finally:
        set_stream_passes(old)


def set_l2_workers(on):
    """rw_set_option(RW_OPT_L2_WORKERS): bit-identical 4-CTA worker clusters on the SMs the 64^3
    resident clusters leave free (1, default) or not (0)."""
    check(lib().rw_set_option(7, int(bool(on))), "rw_set_option")


def get_l2_workers():
    return bool(lib().rw_get_option(7))


@contextlib.contextmanager
def l2_workers(on):
    old = get_l2_workers()
    set_l2_workers(on)
    try:
        yield
    finally:
        set_l2_workers(old)


def set_stream_zc(zc):
    """rw_set_option(RW_OPT_STREAM_ZC): 0 (default, automatic) or the streaming solver's
    z-chunk in planes (4..4096)."""
    check(lib().rw_set_option(6, int(zc)), "rw_set_option")


def get_stream_zc():
    return int(lib().rw_get_option(6))


@contextlib.contextmanager
def stream_zc(zc):
    old = get_stream_zc()
    set_stream_zc(zc)
    try:
        yield
    finally:
        set_stream_zc(old)


def resident_available(dims, nrhs=1):
    """rw_resident_available: can the brick-resident (on-chip) solver serve this shape?"""
    nx, ny, nz = dims
    return bool(lib().rw_resident_available(rw_dims(nx, ny, nz), nrhs))


def solve_workspace_bytes(batch, dims, nrhs=1, weights_given=False):
    nx, ny, nz = dims
    return lib().rw_solve_workspace_bytes(batch, rw_dims(nx, ny, nz), nrhs, int(weights_given))


def solve_labels_workspace_bytes(batch, dims, K, weights_given=False):
    nx, ny, nz = dims
    return lib().rw_solve_labels_workspace_bytes(batch, rw_dims(nx, ny, nz), K, int(weights_given))


def alloc_workspace(nbytes, device):
    # 256-byte aligned (torch's caching allocator returns >= 512-byte aligned blocks)
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def brick_weights(vol, beta=100.0, eps=1e-6, fixed=None, norm=None, want_dinv=True, stream=None):
    """rw_brick_weights: returns (W [3, B, nz, ny, nx] fp32, dinv [B, nz, ny, nx] or None)."""
    _need(vol, "vol")
    _need(fixed, "fixed", torch.uint8)
    if vol.dim() == 3:
        vol = vol.unsqueeze(0)
    B = vol.shape[0]
    sc, of = norm or DEFAULT_NORM[vol.dtype]
    W = torch.empty((3,) + tuple(vol.shape), dtype=torch.float32, device=vol.device)
    dinv = torch.empty(tuple(vol.shape), dtype=torch.float32, device=vol.device) if want_dinv else None
    st = lib().rw_brick_weights(_ptr(vol), DTYPES[vol.dtype], rw_norm(sc, of), B, dims_of(vol),
                                beta, eps, _ptr(W), _ptr(dinv), _ptr(fixed), _stream(stream, vol.device))
    check(st, "rw_brick_weights")
    _retain(stream, W, dinv)
    return W, dinv


WEIGHT_KINDS = {"grady": 0, "poisson": 1, "gaussian": 2, "ttest": 3}


def brick_weights_ex(vol, kind="ttest", beta=100.0, eps=1e-6, count_scale=1.0, radius=1,
                     fixed=None, norm=None, want_dinv=True, stream=None):
    """rw_brick_weights_ex: the paper's alternative weights; returns (W, dinv)
    in the rw_brick_weights layout.  Pass W to solve_bricks(..., W=W)."""
    _need(vol, "vol")
    _need(fixed, "fixed", torch.uint8)
    if vol.dim() == 3:
        vol = vol.unsqueeze(0)
    B = vol.shape[0]
    sc, of = norm or DEFAULT_NORM[vol.dtype]
    spec = rw_weight_spec(WEIGHT_KINDS[kind], beta, eps, count_scale, radius)
    d = dims_of(vol)
    W = torch.empty((3,) + tuple(vol.shape), dtype=torch.float32, device=vol.device)
    dinv = torch.empty(tuple(vol.shape), dtype=torch.float32, device=vol.device) if want_dinv else None
    need = lib().rw_weights_workspace_bytes(B, d, spec)
    ws = alloc_workspace(need, vol.device) if need else None
    st = lib().rw_brick_weights_ex(_ptr(vol), DTYPES[vol.dtype], rw_norm(sc, of), B, d, spec,
                                   _ptr(W), _ptr(dinv), _ptr(fixed), _ptr(ws),
                                   0 if ws is None else ws.numel(), _stream(stream, vol.device))
    check(st, "rw_brick_weights_ex")
    _retain(stream, W, dinv, ws)
    return W, dinv


def solve_bricks(fixed, values, vol=None, W=None, beta=100.0, eps=1e-6, tol=1e-6,
                 max_iter=5000, tol_mode=0, x0=None, norm=None, labels=False, workspace=None,
                 out=None, stream=None):
    """rw_solve_bricks.  ``values``/``x0``: [nrhs, B, nz, ny, nx] (or [B, ...] for nrhs=1).

    Returns dict(prob [nrhs,B,nz,ny,nx], iters [nrhs,B], resid [nrhs,B], status [nrhs,B],
      labels [B,nz,ny,nx] u8 or None).  Stream-ordered: outputs are valid once ``stream`` (default:
    the current stream) reaches this point (see rw.h).
    """
    _need(fixed, "fixed", torch.uint8)
    if fixed.dim() == 3:                       # a single brick
        fixed = fixed.unsqueeze(0)
    if vol is not None and vol.dim() == 3:
        vol = vol.unsqueeze(0)
    while values.dim() < 5:
        values = values.unsqueeze(0)
    while x0 is not None and x0.dim() < 5:
        x0 = x0.unsqueeze(0)
    _need(values, "values", torch.float32)
    _need(x0, "x0", torch.float32)
    _need(vol, "vol")
    _need(W, "W", torch.float32)
    R, B = values.shape[0], values.shape[1]
    if fixed.dim() != 4 or tuple(values.shape[1:]) != tuple(fixed.shape):
        raise ValueError(f"fixed {tuple(fixed.shape)} must be [B,nz,ny,nx] and values "
                         f"{tuple(values.shape)} [nrhs,B,nz,ny,nx]")
    if vol is not None and tuple(vol.shape) != tuple(fixed.shape):
        raise ValueError(f"vol {tuple(vol.shape)} must match fixed {tuple(fixed.shape)}")
    if W is not None and tuple(W.shape) != (3,) + tuple(fixed.shape):
        raise ValueError(f"W {tuple(W.shape)} must be [3,B,nz,ny,nx]")
    if x0 is not None and tuple(x0.shape) != tuple(values.shape):
        raise ValueError(f"x0 {tuple(x0.shape)} must match values {tuple(values.shape)}")
    d = dims_of(fixed)
    dev = fixed.device
    dt = DTYPES[vol.dtype] if vol is not None else 3
    sc, of = norm or (DEFAULT_NORM[vol.dtype] if vol is not None else (1.0, 0.0))
    need = lib().rw_solve_workspace_bytes(B, d, R, int(W is not None))
    if workspace is None or workspace.numel() < need:
        workspace = alloc_workspace(need, dev)
    if out is None:
        out = dict(prob=torch.empty_like(values),
                   iters=torch.empty((R, B), dtype=torch.int32, device=dev),
                   resid=torch.empty((R, B), dtype=torch.float32, device=dev),
                   status=torch.empty((R, B), dtype=torch.int32, device=dev),
                   labels=torch.empty(tuple(fixed.shape), dtype=torch.uint8, device=dev) if labels else None)
    st = lib().rw_solve_bricks(B, d, _ptr(vol), dt, rw_norm(sc, of), _ptr(W), _ptr(fixed),
                               _ptr(values), R, beta, eps, tol, max_iter, tol_mode, _ptr(x0),
                               _ptr(workspace), workspace.numel(), _ptr(out["prob"]),
                               _ptr(out["iters"]), _ptr(out["resid"]), _ptr(out["status"]),
                               _ptr(out["labels"]), _stream(stream, dev))
    check(st, "rw_solve_bricks")
    _retain(stream, workspace, *out.values())
    return out


def _need_host(t, name, dtype=None):
    if t is None:
        return
    if t.is_cuda:
        raise ValueError(f"{name} must be a host (CPU) tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")


def solve_bricks_host(fixed, values, vol, beta=100.0, eps=1e-6, tol=1e-6, max_iter=5000,
                      tol_mode=0, norm=None, chunk=0, prob=True, labels=False, workspace=None,
                      out=None, device=None, stream=None):
    """rw_solve_bricks_host: the same solve from HOST tensors (pin them for overlap), with the
    host<->device copies pipelined against the chunked solve (rw.h).  fixed u8 / values fp32 /
    vol [B,nz,ny,nx] on the CPU.  Returns dict of CPU tensors prob [1,B,...] (if prob),
    labels [B,...] (if labels), iters / resid / status [1,B].  Blocks until they are filled."""
    _need_host(fixed, "fixed", torch.uint8)
    if values.dim() == 5:
        values = values[0]
    _need_host(values, "values", torch.float32)
    _need_host(vol, "vol")
    if fixed.dim() != 4 or tuple(values.shape) != tuple(fixed.shape) or \
            tuple(vol.shape) != tuple(fixed.shape):
        raise ValueError("fixed, values and vol must all be [B,nz,ny,nx]")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    B = fixed.shape[0]
    d = dims_of(fixed)
    dt = DTYPES[vol.dtype]
    sc, of = norm or DEFAULT_NORM[vol.dtype]
    need = lib().rw_solve_host_workspace_bytes(B, d, dt, int(chunk))
    if need == 0:
        raise ValueError("solve_bricks_host: bad dims / dtype / chunk")
    if workspace is None or workspace.numel() < need:
        workspace = alloc_workspace(need, dev)
    if out is None:
        pin = fixed.is_pinned()
        mk = lambda shp, dt_: torch.empty(shp, dtype=dt_, pin_memory=pin)
        out = dict(prob=mk((1,) + tuple(fixed.shape), torch.float32) if prob else None,
                   labels=mk(tuple(fixed.shape), torch.uint8) if labels else None,
                   iters=mk((1, B), torch.int32), resid=mk((1, B), torch.float32),
                   status=mk((1, B), torch.int32))
    st = lib().rw_solve_bricks_host(B, d, _ptr(vol), dt, rw_norm(sc, of), _ptr(fixed), _ptr(values),
                                    beta, eps, tol, max_iter, tol_mode, int(chunk),
                                    _ptr(workspace), workspace.numel(), _ptr(out.get("prob")),
                                    _ptr(out.get("labels")), _ptr(out["iters"]), _ptr(out["resid"]),
                                    _ptr(out["status"]), _stream(stream, dev))
    check(st, "rw_solve_bricks_host")
    return out


def solve_labels(seeds, K, vol=None, W=None, beta=100.0, eps=1e-6, tol=1e-6, max_iter=5000,
                 tol_mode=0, norm=None, workspace=None, stream=None):
    """rw_solve_labels: seeds u8 [B,nz,ny,nx] (0 unseeded, 1..K).  Returns dict(prob
    [K-1,B,...] for classes 1..K-1, labels [B,...] in 1..K, iters [K-1,B], resid)."""
    _need(seeds, "seeds", torch.uint8)
    _need(vol, "vol")
    _need(W, "W", torch.float32)
    B = seeds.shape[0]
    d = dims_of(seeds)
    dev = seeds.device
    dt = DTYPES[vol.dtype] if vol is not None else 3
    sc, of = norm or (DEFAULT_NORM[vol.dtype] if vol is not None else (1.0, 0.0))
    need = lib().rw_solve_labels_workspace_bytes(B, d, K, int(W is not None))
    if workspace is None or workspace.numel() < need:
        workspace = alloc_workspace(need, dev)
    prob = torch.empty((K - 1,) + tuple(seeds.shape), dtype=torch.float32, device=dev)
    iters = torch.empty((K - 1, B), dtype=torch.int32, device=dev)
    resid = torch.empty((K - 1, B), dtype=torch.float32, device=dev)
    labels = torch.empty(tuple(seeds.shape), dtype=torch.uint8, device=dev)
    st = lib().rw_solve_labels(B, d, _ptr(vol), dt, rw_norm(sc, of), _ptr(W), _ptr(seeds), K,
                               beta, eps, tol, max_iter, tol_mode, _ptr(workspace),
                               workspace.numel(), _ptr(prob), _ptr(iters), _ptr(resid),
                               _ptr(labels), _stream(stream, dev))
    check(st, "rw_solve_labels")
    _retain(stream, workspace, prob, labels, iters, resid)
    return dict(prob=prob, labels=labels, iters=iters, resid=resid)


def hier_segment(vol, seeds, s=32, e=1.25, t_hom=0.3, t_bin=0.01, prune=True, beta=100.0,
                 eps=1e-6, tol=1e-6, max_iter=5000, tol_mode=0, norm=None, max_batch=1024,
                 prev=None, t_inc=0.01, workspace=None, out=None, stream=None):
    """rw_hier_segment: vol [D,D,D], seeds u8 [D,D,D] (0 / 1 fg / 2 bg), D = s 2^k.

    Returns (prob fp32 [D,D,D], stats dict of per-level lists (level 0 = full resolution),
    state).  Passing ``prev=state`` of an earlier call on the same volume and geometry runs
    the incremental H_it: the previous result is updated in place (the returned
    prob is the previous tensor)."""
    _need(vol, "vol")
    _need(seeds, "seeds", torch.uint8)
    nz, ny, nx = vol.shape
    d = rw_dims(nx, ny, nz)
    sc, of = norm or DEFAULT_NORM[vol.dtype]
    cfg = rw_hier_config(s, e, t_hom, t_bin, int(prune), beta, eps, tol, max_iter, tol_mode,
                         max_batch, int(prev is not None), t_inc)
    need = lib().rw_hier_workspace_bytes(d, DTYPES[vol.dtype], cfg)
    if need == 0:
        raise ValueError("hier_segment: need a cubic volume of side s*2^k, s % 4 == 0, "
                         "e in (1, 2] with floor(e*s) % 4 == 0")
    if prev is not None:
        workspace, prob = prev["workspace"], prev["prob"]
        if workspace.numel() < need or tuple(prob.shape) != tuple(vol.shape):
            raise ValueError("hier_segment: prev state does not match this volume/geometry")
    else:
        if workspace is None or workspace.numel() < need:
            workspace = alloc_workspace(need, vol.device)
        prob = out if out is not None else torch.empty(tuple(vol.shape), dtype=torch.float32,
                                                       device=vol.device)
        _need(prob, "out", torch.float32)
    st = rw_hier_stats()
    check(lib().rw_hier_segment(_ptr(vol), DTYPES[vol.dtype], rw_norm(sc, of), d, _ptr(seeds), cfg,
                                _ptr(workspace), workspace.numel(), _ptr(prob), C.byref(st),
                                _stream(stream, vol.device)), "rw_hier_segment")
    L = st.levels
    stats = {f: [int(getattr(st, f)[l]) for l in range(L)]
             for f in ("active", "solved", "pruned_hom", "pruned_dt", "conflict", "reused", "iters")}
    stats["levels"] = L
    return prob, stats, {"prob": prob, "workspace": workspace}


NP_DTYPES = {"uint8": 0, "uint16": 1, "int16": 2, "float32": 3}


def pinned_empty(shape, dtype):
    """A page-locked host numpy array (a view of a pinned torch tensor, which it keeps alive)."""
    import numpy as np
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    t = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    return t.numpy().view(dtype).reshape(shape)


class host_register:
    """Page-locks an existing C-contiguous numpy array in place (cudaHostRegister) for the
    lifetime of the object / with-block, so rw_queue_push and the out-of-core drivers copy it
    without staging.  Registration costs about as much as one pass over the array."""

    def __init__(self, arr):
        if not arr.flags.c_contiguous:
            raise ValueError("host_register: array must be C-contiguous")
        self.arr, self.ptr = arr, arr.ctypes.data
        r = torch.cuda.cudart().cudaHostRegister(self.ptr, arr.nbytes, 0)
        if int(r) != 0:
            self.ptr = None
            raise RuntimeError(f"cudaHostRegister failed ({int(r)})")

    def close(self):
        if self.ptr is not None:
            torch.cuda.cudart().cudaHostUnregister(self.ptr)
            self.ptr = None

    def __enter__(self):
        return self.arr

    def __exit__(self, *a):
        self.close()


def hier_ooc_alloc(shape, dtype, s=32, e=1.25, pool_bricks=None, max_batch=1024, depth=2,
                   device="cuda"):
    """The reusable resources of hier_segment_ooc for [nz, ny, nx] volumes of numpy `dtype`:
    (Queue, workspace tensor, pool_bricks).  Pass them as queue= / workspace= / pool_bricks= so
    repeated runs allocate nothing."""
    import numpy as np
    dt = NP_DTYPES[str(np.dtype(dtype))]
    nz, ny, nx = shape
    d = rw_dims(nx, ny, nz)
    cfg = rw_hier_config(s, e, 0.3, 0.01, 1, 100.0, 1e-6, 1e-6, 5000, 0, max_batch, 0, 0.01)
    if pool_bricks is None:
        pool_bricks = (-(-nx // s) * -(-ny // s) * -(-nz // s)) // 16 + 4096
    need = lib().rw_hier_ooc_workspace_bytes(d, dt, cfg, int(pool_bricks))
    qb = lib().rw_hier_ooc_queue_bytes(d, dt, cfg)
    if need == 0 or qb == 0:
        raise ValueError("hier_ooc_alloc: need s % 4 == 0, e in (1, 2] with floor(e*s) % 4 == 0")
    return Queue(qb, depth=depth), alloc_workspace(need, device), int(pool_bricks)


def hier_segment_ooc(vol, seeds, s=32, e=1.25, t_hom=0.3, t_bin=0.01, prune=True, beta=100.0,
                     eps=1e-6, tol=1e-6, max_iter=5000, tol_mode=0, norm=None, max_batch=1024,
                     pool_bricks=None, want_prob=True, want_labels=True, device="cuda",
                     queue=None, workspace=None, stream=None, out_prob=None, out_labels=None):
    """rw_hier_segment_ooc: the hierarchical random walker with the
    volume, labels and output in HOST memory.  vol: numpy [nz, ny, nx] (u8/u16/i16/f32), any
    dims; seeds: numpy u8 (0 / 1 fg / 2 bg).  pool_bricks: device brick-pool capacity (default:
    the level-0 brick count / 8 + 4096).  Returns (prob fp32 numpy or None, labels u8 numpy or
    None, stats dict).  out_prob / out_labels: caller-owned C-contiguous numpy outputs of vol's
    shape (fp32 / u8).  Page-locked buffers (pinned_empty, host_register) skip the library's
    host staging copies: the copy engine reads vol / seeds and writes the outputs directly."""
    import numpy as np
    vol = np.ascontiguousarray(vol)
    seeds = np.ascontiguousarray(seeds, dtype=np.uint8)
    if vol.ndim != 3 or seeds.shape != vol.shape:
        raise ValueError("hier_segment_ooc: vol and seeds must be 3-D arrays of one shape")
    for o, t in ((out_prob, np.float32), (out_labels, np.uint8)):
        if o is not None and (o.dtype != t or o.shape != vol.shape or not o.flags.c_contiguous):
            raise ValueError("hier_segment_ooc: out_prob / out_labels must be C-contiguous fp32 / u8 "
                             "arrays of vol's shape")
    dt = NP_DTYPES[str(vol.dtype)]
    nz, ny, nx = vol.shape
    d = rw_dims(nx, ny, nz)
    tdt = {0: torch.uint8, 1: torch.uint16, 2: torch.int16, 3: torch.float32}[dt]
    sc, of = norm or DEFAULT_NORM[tdt]
    cfg = rw_hier_config(s, e, t_hom, t_bin, int(prune), beta, eps, tol, max_iter, tol_mode,
                         max_batch, 0, 0.01)
    if pool_bricks is None:
        nb0 = -(-nx // s) * -(-ny // s) * -(-nz // s)
        pool_bricks = nb0 // 16 + 4096
    need = lib().rw_hier_ooc_workspace_bytes(d, dt, cfg, int(pool_bricks))
    qb = lib().rw_hier_ooc_queue_bytes(d, dt, cfg)
    if need == 0 or qb == 0:
        raise ValueError("hier_segment_ooc: need s % 4 == 0, e in (1, 2] with floor(e*s) % 4 == 0")
    if workspace is None or workspace.numel() < need:
        workspace = alloc_workspace(need, device)
    own_q = queue is None
    if own_q:
        queue = Queue(qb, depth=2)
    prob = out_prob if out_prob is not None else (np.empty(vol.shape, np.float32) if want_prob else None)
    lab = out_labels if out_labels is not None else (np.empty(vol.shape, np.uint8) if want_labels else None)
    st = rw_hier_stats()
    try:
        check(lib().rw_hier_segment_ooc(C.c_void_p(vol.ctypes.data), dt, rw_norm(sc, of), d,
                                        C.c_void_p(seeds.ctypes.data), cfg, int(pool_bricks),
                                        queue._q, _ptr(workspace), workspace.numel(),
                                        None if prob is None else C.c_void_p(prob.ctypes.data),
                                        None if lab is None else C.c_void_p(lab.ctypes.data),
                                        C.byref(st), _stream(stream, workspace.device)),
              "rw_hier_segment_ooc")
    finally:
        if own_q:
            queue.close()
    stats = _stats_dict(st)
    stats["pool_used"] = int(st.pool_used)
    stats["ms"] = {"pyramid": st.ms_pyramid, "levels": st.ms_levels, "output": st.ms_output}
    return prob, lab, stats


def hier_segment_labels_ooc(vol, labels, K, s=32, e=1.25, t_hom=0.3, prune=True, beta=100.0,
                            eps=1e-6, tol=1e-6, max_iter=5000, tol_mode=0, norm=None,
                            max_batch=1024, pool_bricks=None, device="cuda", queue=None,
                            workspace=None, stream=None):
    """rw_hier_segment_labels_ooc: K one-vs-rest out-of-core runs and the
    argmax class, volume / class seeds / outputs in HOST memory.  vol: numpy [nz, ny, nx], any
    dims; labels: numpy u8 in 0..K.  Returns (best fp32 numpy, labels u8 numpy in 1..K, list of
    K stats dicts)."""
    import numpy as np
    vol = np.ascontiguousarray(vol)
    labels = np.ascontiguousarray(labels, dtype=np.uint8)
    if vol.ndim != 3 or labels.shape != vol.shape:
        raise ValueError("hier_segment_labels_ooc: vol and labels must be 3-D arrays of one shape")
    dt = NP_DTYPES[str(vol.dtype)]
    nz, ny, nx = vol.shape
    d = rw_dims(nx, ny, nz)
    tdt = {0: torch.uint8, 1: torch.uint16, 2: torch.int16, 3: torch.float32}[dt]
    sc, of = norm or DEFAULT_NORM[tdt]
    cfg = rw_hier_config(s, e, t_hom, -1.0, int(prune), beta, eps, tol, max_iter, tol_mode,
                         max_batch, 0, 0.01)
    if pool_bricks is None:
        nb0 = -(-nx // s) * -(-ny // s) * -(-nz // s)
        pool_bricks = nb0 // 16 + 4096
    need = lib().rw_hier_ooc_workspace_bytes(d, dt, cfg, int(pool_bricks))
    qb = lib().rw_hier_ooc_queue_bytes(d, dt, cfg)
    if need == 0 or qb == 0:
        raise ValueError("hier_segment_labels_ooc: need s % 4 == 0, e in (1, 2] with "
                         "floor(e*s) % 4 == 0")
    if workspace is None or workspace.numel() < need:
        workspace = alloc_workspace(need, device)
    own_q = queue is None
    if own_q:
        queue = Queue(qb, depth=2)
    best = np.empty(vol.shape, np.float32)
    lab = np.empty(vol.shape, np.uint8)
    st = (rw_hier_stats * int(K))()
    try:
        check(lib().rw_hier_segment_labels_ooc(C.c_void_p(vol.ctypes.data), dt, rw_norm(sc, of), d,
                                               C.c_void_p(labels.ctypes.data), int(K), cfg,
                                               int(pool_bricks), queue._q, _ptr(workspace),
                                               workspace.numel(), C.c_void_p(best.ctypes.data),
                                               C.c_void_p(lab.ctypes.data), st,
                                               _stream(stream, workspace.device)),
              "rw_hier_segment_labels_ooc")
    finally:
        if own_q:
            queue.close()
    stats = []
    for x in st:
        sd = _stats_dict(x)
        sd["pool_used"] = int(x.pool_used)
        sd["ms"] = {"pyramid": x.ms_pyramid, "levels": x.ms_levels, "output": x.ms_output}
        stats.append(sd)
    return best, lab, stats


def _stats_dict(st):
    L = st.levels
    out = {f: [int(getattr(st, f)[l]) for l in range(L)]
           for f in ("active", "solved", "pruned_hom", "pruned_dt", "conflict", "reused", "iters")}
    out["levels"] = L
    return out


def hier_segment_labels(vol, labels, K, s=32, e=1.25, t_hom=0.3, prune=True, beta=100.0,
                        eps=1e-6, tol=1e-6, max_iter=5000, tol_mode=0, norm=None,
                        max_batch=1024, keep_prob=True, keep_state=False, prev=None, t_inc=0.01,
                        workspace=None, stream=None):
    """rw_hier_segment_labels: K one-vs-rest hierarchical runs (homogeneity
    pruning only) and the argmax class.  labels u8 [D,D,D] in 0..K.

    Returns dict(labels u8 [D,D,D] in 1..K, best fp32 [D,D,D], prob fp32 [K,D,D,D] or None,
    stats = list of K per-level stats dicts, state).  ``keep_state=True`` keeps one workspace
    per class (and the class fields) so that a later call with ``prev=state`` runs H_it per
    class."""
    _need(vol, "vol")
    _need(labels, "labels", torch.uint8)
    nz, ny, nx = vol.shape
    d = rw_dims(nx, ny, nz)
    sc, of = norm or DEFAULT_NORM[vol.dtype]
    inc = prev is not None
    cfg = rw_hier_config(s, e, t_hom, -1.0, int(prune), beta, eps, tol, max_iter, tol_mode,
                         max_batch, int(inc), t_inc)
    cfg_size = rw_hier_config(s, e, t_hom, -1.0, int(prune), beta, eps, tol, max_iter, tol_mode,
                              max_batch, int(inc or keep_state), t_inc)
    need = lib().rw_hier_labels_workspace_bytes(d, DTYPES[vol.dtype], int(K), cfg_size)
    if need == 0:
        raise ValueError("hier_segment_labels: need K in 2..255 and a cubic volume of side "
                         "s*2^k, s % 4 == 0, e in (1, 2] with floor(e*s) % 4 == 0")
    shp = tuple(vol.shape)
    if inc:
        workspace, prob = prev["workspace"], prev["prob"]
        if workspace.numel() < need or prob is None or tuple(prob.shape) != (K,) + shp:
            raise ValueError("hier_segment_labels: prev state does not match this volume/K")
    else:
        if workspace is None or workspace.numel() < need:
            workspace = alloc_workspace(need, vol.device)
        prob = (torch.empty((K,) + shp, dtype=torch.float32, device=vol.device)
                if keep_prob or keep_state else None)
    best = torch.empty(shp, dtype=torch.float32, device=vol.device)
    lab = torch.empty(shp, dtype=torch.uint8, device=vol.device)
    st = (rw_hier_stats * int(K))()
    check(lib().rw_hier_segment_labels(_ptr(vol), DTYPES[vol.dtype], rw_norm(sc, of), d,
                                       _ptr(labels), int(K), cfg, _ptr(workspace),
                                       workspace.numel(), _ptr(prob) if prob is not None else None,
                                       _ptr(best), _ptr(lab), st, _stream(stream, vol.device)),
          "rw_hier_segment_labels")
    return dict(labels=lab, best=best, prob=prob, stats=[_stats_dict(x) for x in st],
                state={"prob": prob, "workspace": workspace})


def level_dims(dims, levels):
    nx, ny, nz = dims
    out = []
    for _ in range(levels):
        nx, ny, nz = (nx + 1) // 2, (ny + 1) // 2, (nz + 1) // 2
        out.append((nx, ny, nz))
    return out


def build_pyramid(vol, levels, outs=None, stream=None):
    """rw_build_pyramid: vol [nz, ny, nx] -> list of ``levels`` tensors (levels 1..L)."""
    _need(vol, "vol")
    nz, ny, nx = vol.shape
    if outs is None:
        outs = [torch.empty((z, y, x), dtype=vol.dtype, device=vol.device)
                for (x, y, z) in level_dims((nx, ny, nz), levels)]
    arr = (C.c_void_p * levels)(*[o.data_ptr() for o in outs])
    st = lib().rw_build_pyramid(_ptr(vol), DTYPES[vol.dtype], rw_dims(nx, ny, nz), levels, arr,
                                _stream(stream, vol.device))
    check(st, "rw_build_pyramid")
    return outs


def build_pyramid_slab(slab, full_dims, z0, levels, outs, stream=None):
    """rw_build_pyramid_slab: slab = planes [z0, z0+slab.shape[0]) of a volume of
    ``full_dims`` = (nx, ny, nz); ``outs`` = preallocated full-size level tensors."""
    _need(slab, "slab")
    nx, ny, nz = full_dims
    arr = (C.c_void_p * levels)(*[o.data_ptr() for o in outs])
    st = lib().rw_build_pyramid_slab(_ptr(slab), DTYPES[slab.dtype], rw_dims(nx, ny, nz), z0,
                                     slab.shape[0], levels, arr, _stream(stream, slab.device))
    check(st, "rw_build_pyramid_slab")
    return outs


class Queue:
    """rw_queue: pinned double-buffered host->device ring (library-owned buffers)."""

    def __init__(self, slot_bytes, depth=2):
        h = C.c_void_p()
        check(lib().rw_queue_create(slot_bytes, depth, C.byref(h)), "rw_queue_create")
        self._q = h
        self.slot_bytes = slot_bytes

    def push(self, host_array, copy_stream):
        """Copy a host numpy array / CPU tensor into the next slot; returns (dev_ptr, slot)."""
        import numpy as np
        a = np.ascontiguousarray(host_array)
        dev = C.c_void_p()
        sid = C.c_int32()
        check(lib().rw_queue_push(self._q, C.c_void_p(a.ctypes.data), a.nbytes,
                                  C.c_void_p(copy_stream.cuda_stream), C.byref(dev), C.byref(sid)),
              "rw_queue_push")
        return dev.value, sid.value

    def wait(self, slot, compute_stream):
        check(lib().rw_queue_wait(self._q, slot, C.c_void_p(compute_stream.cuda_stream)), "rw_queue_wait")

    def release(self, slot, compute_stream):
        check(lib().rw_queue_release(self._q, slot, C.c_void_p(compute_stream.cuda_stream)), "rw_queue_release")

    def close(self):
        if self._q:
            lib().rw_queue_destroy(self._q)
            self._q = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_view(ptr, shape, dtype, device):
    """Wrap a raw device pointer (e.g. a queue slot) as a torch tensor without copying."""
    import numpy as np
    n = int(np.prod(shape))
    itemsize = torch.tensor([], dtype=dtype).element_size()

    class _Holder:
        __cuda_array_interface__ = {
            "shape": (n * itemsize,), "typestr": "|u1", "data": (ptr, False), "version": 3}
    t = torch.as_tensor(_Holder(), device=device)
    return t.view(dtype).view(shape)


def profile_enable(on=True):
    """Reset the library's launch counters; with on=True also time every launch with CUDA
    events on its stream (include/rw.h rw_profile_enable)."""
    check(lib().rw_profile_enable(int(on)), "rw_profile_enable")


def profile_read():
    """-> {kernel class: (launches, device ms)} since the last profile_enable()."""
    from ._lib import KERNEL_CLASSES
    n = (C.c_int64 * len(KERNEL_CLASSES))()
    ms = (C.c_double * len(KERNEL_CLASSES))()
    check(lib().rw_profile_read(C.cast(n, C.c_void_p), C.cast(ms, C.c_void_p)), "rw_profile_read")
    return {k: (int(n[i]), float(ms[i])) for i, k in enumerate(KERNEL_CLASSES)}
