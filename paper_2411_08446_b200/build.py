"""Build liblshmoe.so in-tree: nvcc for the sm_100a kernels, g++ for the host C++ (rotation is
compiled with -ffp-contract=off so its fp64 recipe stays bit-reproducible), linked with the
static CUDA runtime and the NCCL that ships with torch (nvidia-nccl-cu12)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "liblshmoe.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        raise RuntimeError(f"nccl.h not found under {inc}")
    return inc, lib


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "kernels", "*.cu"))), sorted(glob.glob(os.path.join(CSRC, "abi", "*.cpp")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = glob.glob(os.path.join(CSRC, "**", "*"), recursive=True) + [os.path.join(ROOT, "include", "lshmoe.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps if os.path.isfile(p))


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stdout or r.stderr):
        sys.stderr.write(r.stdout + r.stderr)


def build(force: bool = False, verbose: bool = False, jobs: int = 8) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    nccl_inc, nccl_lib = _nccl_dirs()
    cu, cpp = sources()
    objs, cmds = [], []
    extra = os.environ.get("LSHMOE_NVCC_EXTRA", "").split()   # experiments only, e.g. -DLSHMOE_MERGE_BATCH=8
    for src in cu:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        cmds.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                     "--expt-relaxed-constexpr", *extra, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj])
    for src in cpp:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        cmds.append(["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall",
                     "-I", os.path.join(CUDA_HOME, "include"), "-I", nccl_inc, "-I", os.path.join(ROOT, "include"),
                     "-c", src, "-o", obj])
    # compile in parallel
    procs = []
    logs = {}
    for cmd in cmds:
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        while sum(p.poll() is None for _, p in procs) >= jobs:
            procs[[p.poll() is None for _, p in procs].index(True)][1].wait()
    failed = False
    for cmd, p in procs:
        out = p.communicate()[0]
        logs[cmd[-1]] = out
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"--- {cmd[-3]}\n{out}\n")
    if failed:
        raise RuntimeError("liblshmoe build failed")
    with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
        for k, v in logs.items():
            f.write(f"=== {k}\n{v}\n")
    tmp = LIB + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-L", nccl_lib, "-l:libnccl.so.2",
          "-Xlinker", f"-rpath={nccl_lib}"], verbose)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
