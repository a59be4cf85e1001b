"""Build libgbm.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgbm.so")
SOURCES = ["api.cu", "comm.cu", "quantise.cu", "gradients.cu", "tree.cu", "records.cu", "root_ct.cu"]
HEADERS = ["gbm_internal.cuh", "tree_common.cuh", os.path.join("..", "..", "include", "gbm.h")]


def nccl_dirs():
    import nvidia.nccl  # pip NCCL 2.28 -- the copy torch loads (two libnccl.so.2 must not mix)
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit to an object in parallel (objects cached by mtime under
    build/), then link libgbm.so."""
    if not force and not stale():
        return LIB
    inc, libdir = nccl_dirs()
    obj_dir = os.path.join(HERE, "build")
    os.makedirs(obj_dir, exist_ok=True)
    flags = [nvcc(), "-std=c++17", "-O3", "-lineinfo", "--fmad=false",
             "-gencode", "arch=compute_100a,code=sm_100a",
             "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-I", inc]
    flags += os.environ.get("GBM_NVCC_EXTRA", "").split()  # tuning experiments only (-DGBM_PH_UNR=...)
    hdr_t = max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS)
    procs, objs = [], []
    for src in SOURCES:
        obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        srcp = os.path.join(CSRC, src)
        if (not force and os.path.exists(obj) and
                os.path.getmtime(obj) > max(os.path.getmtime(srcp), hdr_t)):
            continue
        cmd = flags + ["-c", srcp, "-o", obj + f".tmp{os.getpid()}"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd, cwd=CSRC), obj))
    failed = False
    for p, obj in procs:
        if p.wait() != 0:
            failed = True
        else:
            os.replace(obj + f".tmp{os.getpid()}", obj)
    if failed:
        raise subprocess.CalledProcessError(1, "nvcc")
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp] + objs
    cmd += ["-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath={libdir}"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
