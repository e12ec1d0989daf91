"""Build libptucker.so in-tree: nvcc for sm_100a, one object per .cu (parallel), NCCL linked.

    python -m paper_1710_02261_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(os.path.dirname(HERE), "include")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libptucker.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]



def _nccl_dir():
    """Prefer the NCCL that torch ships (2.28.x): both libraries then share one
    libnccl.so.2 in the process whichever is imported first."""
    try:
        import nvidia.nccl as nn
        d = list(nn.__path__)[0]
        if os.path.exists(os.path.join(d, "lib", "libnccl.so.2")):
            return d
    except Exception:
        pass
    return None


NCCL = _nccl_dir()
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I", CSRC, "-I", INC]
if NCCL:
    FLAGS += ["-I", os.path.join(NCCL, "include")]
    LINK_NCCL = ["-L", os.path.join(NCCL, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib")]
else:
    LINK_NCCL = ["-lnccl"]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INC, "*.h"))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    if force or _stale(obj, [src] + _headers()):
        log = obj[:-2] + ".ptxas.txt"
        tmp = obj + f".tmp{os.getpid()}"
        r = subprocess.run([NVCC, *ARCH, *FLAGS, "-c", src, "-o", tmp], capture_output=True, text=True)
        with open(log, "w") as f:
            f.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr[-4000:]}")
        os.replace(tmp, obj)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    if force or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, *LINK_NCCL, "-Xlinker", "--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
        os.replace(tmp, LIB)
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
