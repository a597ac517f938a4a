"""ctypes declarations of include/rw.h (argument marshalling only).

Loading fails loudly if librw.so is missing: there is no CPU or Python fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# RW_LIB_PATH: an in-tree experiment build (tools/ A/B runs); default the package's librw.so
LIB_PATH = os.environ.get("RW_LIB_PATH") or os.path.join(HERE, "librw.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "rw.h")


class rw_dims(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32)]


class rw_norm(C.Structure):
    _fields_ = [("scale", C.c_float), ("offset", C.c_float)]


class rw_weight_spec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("beta", C.c_float), ("eps", C.c_float),
                ("count_scale", C.c_float), ("radius", C.c_int32)]


class rw_hier_config(C.Structure):
    _fields_ = [("s", C.c_int32), ("e", C.c_float), ("t_hom", C.c_float), ("t_bin", C.c_float),
                ("prune", C.c_int32), ("beta", C.c_float), ("eps", C.c_float), ("tol", C.c_float),
                ("max_iter", C.c_int32), ("tol_mode", C.c_int32), ("max_batch", C.c_int32),
                ("incremental", C.c_int32), ("t_inc", C.c_float)]


class rw_hier_stats(C.Structure):
    _fields_ = [("levels", C.c_int32)] + [(f, C.c_int64 * 16) for f in
                                          ("active", "solved", "pruned_hom", "pruned_dt",
                                           "conflict", "reused", "iters")] + [
        ("pool_used", C.c_int64), ("ms_pyramid", C.c_double), ("ms_levels", C.c_double),
        ("ms_output", C.c_double)]


P, I32, F32, SZ = C.c_void_p, C.c_int32, C.c_float, C.c_size_t

SIGNATURES = {
    "rw_last_error": (C.c_char_p, []),
    "rw_version": (C.c_char_p, []),
    "rw_brick_weights": (I32, [P, I32, rw_norm, I32, rw_dims, F32, F32, P, P, P, P]),
    "rw_solve_workspace_bytes": (SZ, [I32, rw_dims, I32, I32]),
    "rw_weights_workspace_bytes": (SZ, [I32, rw_dims, rw_weight_spec]),
    "rw_brick_weights_ex": (I32, [P, I32, rw_norm, I32, rw_dims, rw_weight_spec, P, P, P, P, SZ, P]),
    "rw_solve_bricks": (I32, [I32, rw_dims, P, I32, rw_norm, P, P, P, I32, F32, F32, F32, I32,
                              I32, P, P, SZ, P, P, P, P, P, P]),
    "rw_solve_labels_workspace_bytes": (SZ, [I32, rw_dims, I32, I32]),
    "rw_solve_labels": (I32, [I32, rw_dims, P, I32, rw_norm, P, P, I32, F32, F32, F32, I32,
                              I32, P, SZ, P, P, P, P, P]),
    "rw_build_pyramid": (I32, [P, I32, rw_dims, I32, P, P]),
    "rw_build_pyramid_slab": (I32, [P, I32, rw_dims, I32, I32, I32, P, P]),
    "rw_queue_create": (I32, [SZ, I32, C.POINTER(P)]),
    "rw_queue_push": (I32, [P, P, SZ, P, C.POINTER(P), C.POINTER(I32)]),
    "rw_queue_wait": (I32, [P, I32, P]),
    "rw_queue_release": (I32, [P, I32, P]),
    "rw_queue_destroy": (None, [P]),
    "rw_profile_enable": (I32, [I32]),
    "rw_profile_read": (I32, [P, P]),
    "rw_set_option": (I32, [I32, C.c_int64]),
    "rw_hier_workspace_bytes": (SZ, [rw_dims, I32, rw_hier_config]),
    "rw_hier_segment": (I32, [P, I32, rw_norm, rw_dims, P, rw_hier_config, P, SZ, P,
                              C.POINTER(rw_hier_stats), P]),
    "rw_solve_host_workspace_bytes": (SZ, [I32, rw_dims, I32, I32]),
    "rw_solve_bricks_host": (I32, [I32, rw_dims, P, I32, rw_norm, P, P, F32, F32, F32, I32, I32,
                                   I32, P, SZ, P, P, P, P, P, P]),
    "rw_hier_labels_workspace_bytes": (SZ, [rw_dims, I32, I32, rw_hier_config]),
    "rw_hier_segment_labels": (I32, [P, I32, rw_norm, rw_dims, P, I32, rw_hier_config, P, SZ,
                                     P, P, P, C.POINTER(rw_hier_stats), P]),
    "rw_hier_ooc_workspace_bytes": (SZ, [rw_dims, I32, rw_hier_config, C.c_int64]),
    "rw_hier_ooc_queue_bytes": (SZ, [rw_dims, I32, rw_hier_config]),
    "rw_hier_segment_ooc": (I32, [P, I32, rw_norm, rw_dims, P, rw_hier_config, C.c_int64, P, P,
                                  SZ, P, P, C.POINTER(rw_hier_stats), P]),
    "rw_hier_segment_labels_ooc": (I32, [P, I32, rw_norm, rw_dims, P, I32, rw_hier_config,
                                         C.c_int64, P, P, SZ, P, P, C.POINTER(rw_hier_stats), P]),
    "rw_get_option": (C.c_int64, [I32]),
    "rw_resident_available": (I32, [rw_dims, I32]),
}

KERNEL_CLASSES = ["weights", "setup", "passA", "passB", "finalize", "pyramid", "other",
                  "resident", "hier", "l2res"]


def header_symbols(path: str = HEADER):
    """Function names declared in include/rw.h (for the export test)."""
    txt = open(path).read()
    return sorted(set(re.findall(r"\b(rw_[a-z_]+)\s*\(", txt)))


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"librw.so not built ({LIB_PATH}); run "
                               "`python -m paper_2103_09564_b200.build` -- there is no fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class RWError(RuntimeError):
    pass


STATUS = {0: "RW_OK", 1: "RW_EINVAL", 2: "RW_ECUDA", 3: "RW_ENOMEM", 4: "RW_EUNSUPPORTED"}


def check(st: int, what: str):
    if st != 0:
        msg = lib().rw_last_error().decode(errors="replace")
        raise RWError(f"{what}: {STATUS.get(st, st)}: {msg}")
