"""Build libvol.so (the C-ABI library of include/vol.h) in-tree with nvcc for sm_100a.

    python -m paper_1604_03734_b200.build [--force]

Flags: -gencode arch=compute_100a,code=sm_100a, -O3, -lineinfo, --fmad=false (no FMA contraction:
every fp32 operation of the method is one correctly rounded operation in the written order,
reading c-18), IEEE division and square root (the nvcc defaults without --use_fast_math).
NCCL headers/library come from the torch venv (the copy torch itself loads).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libvol.so")
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    cands = []
    try:
        import nvidia.nccl as _n  # type: ignore
        cands += list(getattr(_n, "__path__", []))
    except Exception:
        pass
    cands += glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")) and os.path.exists(os.path.join(c, "lib", "libnccl.so.2")):
            return c
    raise RuntimeError("NCCL (nvidia-nccl wheel) not found next to torch")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "vol.h"), __file__]


def build(force: bool = False, verbose: bool = False, out: str = SO, defines=()) -> str:
    newest = max(os.path.getmtime(p) for p in deps())
    if not force and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    nd = nccl_dir()
    objdir = os.path.join(HERE, "build", os.path.basename(out).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    common = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-prec-div=true", "-prec-sqrt=true",
                     "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-I", os.path.join(ROOT, "include"),
                     "-I", os.path.join(nd, "include"), "-Xptxas", "-v" if verbose else "-O3"] + [f"-D{d}" for d in defines]
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        objs.append(obj)
        cmd = [NVCC, "-c", src, "-o", obj] + common
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        log, _ = p.communicate()
        if verbose or p.returncode:
            sys.stdout.write(log.decode())
        if p.returncode:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    tmp = out + f".tmp{os.getpid()}"
    link = [NVCC, "-shared", "-o", tmp] + objs + ARCH + [
        "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath," + os.path.join(nd, "lib"),
        "-cudart", "shared"]
    subprocess.check_call(link)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
