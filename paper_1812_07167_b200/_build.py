"""Compile libhps.so in-tree with nvcc for sm_100a (no torch JIT cache: the .so travels
with the repo snapshot to the GPU box)."""
import glob
import os
import subprocess

from . import PKG_DIR, REPO_DIR

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


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
    cmd = [NVCC, "-shared", "-Xcompiler", "-fPIC", *ARCH, "-O3", "-lineinfo", "-std=c++17",
           "-I" + os.path.join(REPO_DIR, "include"), "-o", out, *srcs]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    return out
