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


def _flags_hash(extra=()) -> str:
    """Everything that changes the generated code besides the sources: nvcc, the arch,
    the flags and NVCC_APPEND_FLAGS (the -D knobs of tools/*_variant.sh)."""
    import hashlib
    key = "\0".join([NVCC, *ARCH, *FLAGS, *extra, os.environ.get("NVCC_APPEND_FLAGS", "")])
    return hashlib.sha256(key.encode()).hexdigest()[:16]


def _stamp_ok(path: str, h: str) -> bool:
    try:
        with open(path) as f:
            return f.read().strip() == h
    except OSError:
        return False


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, force: bool, obj_dir: str = OBJ, extra=()) -> str:
    obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
    if force or _stale(obj, [src] + _headers()):
        log = obj[:-2] + ".ptxas.txt"
        tmp = obj + f".tmp{os.getpid()}"
        r = subprocess.run([NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", tmp], capture_output=True, text=True)
        with open(log, "w") as f:
            f.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr[-4000:]}")
        os.replace(tmp, obj)
    return obj


def build(force: bool = False, verbose: bool = False, variant: str | None = None, extra=()) -> str:
    """Build libptucker.so; with `variant`, a tools-only experiment build (extra nvcc
    flags, e.g. -D knobs) into _variants/<variant>/ that never touches the product
    library (tools load it through PTUCKER_LIB)."""
    obj_dir, lib = OBJ, LIB
    if variant:
        obj_dir = os.path.join(HERE, "_variants", variant)
        lib = os.path.join(obj_dir, "libptucker.so")
    os.makedirs(obj_dir, exist_ok=True)
    h = _flags_hash(extra)
    obj_stamp, lib_stamp = os.path.join(obj_dir, ".flags"), lib + ".flags"
    if not _stamp_ok(obj_stamp, h):
        force = True  # objects of other flags (a variant build, or another nvcc) are stale
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, obj_dir, extra), srcs))
    with open(obj_stamp, "w") as f:
        f.write(h)
    if force or _stale(lib, objs) or not _stamp_ok(lib_stamp, h):
        tmp = lib + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, *LINK_NCCL, "-Xlinker", "--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
        os.replace(tmp, lib)
        with open(lib_stamp, "w") as f:
            f.write(h)
    if verbose:
        print(lib)
    return lib


if __name__ == "__main__":
    # python -m paper_1710_02261_b200.build [--force] [--variant NAME -DKNOB=1 ...]
    argv = sys.argv[1:]
    var, extra = None, []
    if "--variant" in argv:
        i = argv.index("--variant")
        var, extra = argv[i + 1], argv[i + 2:]
    build(force="--force" in argv, verbose=True, variant=var, extra=tuple(extra))
