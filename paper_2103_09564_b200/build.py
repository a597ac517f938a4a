"""Build librw.so (all CUDA sources under csrc/) in-tree for sm_100a with nvcc.

    python -m paper_2103_09564_b200.build [--verbose]

The shared library lands next to this file so it travels with the repo snapshot to the
GPU box.  cudart is linked statically; the driver (libcuda) is only needed at run time.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "librw.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "rw.h")]


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    """`out`: build an experiment variant elsewhere (tools/ A/B runs load it through
    RW_LIB_PATH); RW_NVCC_DEFS adds -D flags for such variants."""
    lib = out or LIB
    if out is None and not force and up_to_date():
        return LIB
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler",
             "-pthread", "-I", os.path.join(ROOT, "include")]
    flags += os.environ.get("RW_NVCC_DEFS", "").split()
    if verbose:
        flags.append("-Xptxas=-v")
    if os.environ.get("RW_RES_TIMING"):      # debug: phase timers in the resident kernel
        flags.append("-DRW_RES_TIMING")
    # one nvcc per translation unit, in parallel (no cross-unit device code), then one link
    import concurrent.futures as cf
    import tempfile
    tmp = tempfile.mkdtemp(prefix="rwbuild_")
    objs = [os.path.join(tmp, os.path.basename(f) + ".o") for f in sources()]

    def compile_one(src_obj):
        src, obj = src_obj
        return subprocess.run([nvcc(), *flags, "-c", src, "-o", obj], capture_output=True, text=True)

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(objs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, zip(sources(), objs)))
    log = "".join(r.stdout + r.stderr for r in results)
    if any(r.returncode != 0 for r in results):
        shutil.rmtree(tmp, ignore_errors=True)
        raise RuntimeError("nvcc failed:\n" + log)
    r = subprocess.run([nvcc(), *ARCH, "-shared", "-Xcompiler", "-pthread", "-o", lib + ".tmp",
                        *objs], capture_output=True, text=True)
    shutil.rmtree(tmp, ignore_errors=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
    if verbose:
        sys.stderr.write(log + r.stdout + r.stderr)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    o = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    print(build(force=True, verbose="--verbose" in sys.argv, out=o))
