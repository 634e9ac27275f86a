"""Compile libhps.so in-tree with nvcc for sm_100a (no torch JIT cache: the .so travels
with the repo snapshot to the GPU box).  Each .cu is compiled to an object in parallel, then
the objects are linked into one shared library."""
import concurrent.futures as cf
import glob
import os
import subprocess

from . import PKG_DIR, REPO_DIR

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-Xcompiler", "-fPIC", *ARCH, "-O3", "-lineinfo", "-std=c++17"]


def sources():
    return sorted(glob.glob(os.path.join(PKG_DIR, "csrc", "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(PKG_DIR, "csrc", "*.cuh")) + [os.path.join(REPO_DIR, "include", "hps.h")])


def build_libhps(force=False, verbose=False):
    out = os.path.join(PKG_DIR, "libhps.so")
    srcs = sources()
    newest = max(os.path.getmtime(f) for f in srcs + headers())
    if not force and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    objdir = os.path.join(PKG_DIR, "build")
    os.makedirs(objdir, exist_ok=True)
    hdr_time = max(os.path.getmtime(f) for f in headers())

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_time):
            return obj
        cmd = [NVCC, "-c", *FLAGS, "-I" + os.path.join(REPO_DIR, "include"), "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    subprocess.check_call([NVCC, "-shared", *ARCH, "-o", out + ".tmp", *objs, "-ldl"])
    os.replace(out + ".tmp", out)
    return out
