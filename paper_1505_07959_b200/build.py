"""Builds libmfode.so (the C-ABI library of include/mfode.h) in-tree for sm_100a.

    python -m paper_1505_07959_b200.build        # or __graft_entry__.build()

nvcc cross-compiles without a GPU.  cudart is linked statically so the library does not depend
on which libcudart the host process (torch) loaded; NCCL is resolved at run time (dlopen).
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libmfode.so")
SOURCES = ["kernels.cu", "ozaki.cu", "driver.cu"]
HEADERS = ["gemm.cuh", "fused.cuh", "epilogue.cuh", "small.cuh", "ptx.cuh", "internal.h", "nccl_min.h", os.path.join("..", "..", "include", "mfode.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    for f in SOURCES + HEADERS:
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    return False


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and not _stale():
        return OUT
    objs, procs = [], []
    for src in SOURCES:   # translation units compile in parallel
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd)))
        objs.append(obj)
    for cmd, pr in procs:
        if pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, cmd)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", OUT + ".tmp", "-ldl",
           "-Xlinker", "--exclude-libs=ALL"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(OUT + ".tmp", OUT)
    for o in objs:
        os.remove(o)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
