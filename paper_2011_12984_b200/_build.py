"""Builds libsunbw.so in-tree with nvcc for sm_100a (no JIT, no torch
extension machinery: the library has a plain C ABI, include/sunbw.h)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJDIR = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libsunbw.so")

SOURCES = ["context.cu", "nvector.cu", "blockdiag.cu", "brusselator.cu", "stepper.cu", "fused.cu",
           "gmres.cu", "ark.cu", "ark_fused.cu", "vecarray.cu", "peer_halo.cu"]
HEADERS = ["sunbw_internal.h", "sunbw_device.cuh", "pipeline.cuh", "cellstep.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# --fmad=false: no FMA contraction anywhere (the bit-exact paths also use
# explicit __dmul_rn/__dadd_rn; reductions opt in to FMA with __fma_rn).
NVCCFLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xcompiler", "-fvisibility=hidden"]


def nccl_dir() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("NCCL (nvidia.nccl wheel) not found")
    return list(spec.submodule_search_locations)[0]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile and link libsunbw.so.  `defines` (e.g. ["SUNBW_FUSED_MINB=8"])
    and `out` build a tuning variant elsewhere (build/var_*/libsunbw.so)."""
    nccl = nccl_dir()
    lib = out or LIB
    objdir = OBJDIR if not defines else os.path.join(os.path.dirname(lib), "obj")
    os.makedirs(objdir, exist_ok=True)
    dflags = ["-D" + d for d in defines]
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "sunbw.h")]
    incs = ["-I" + INCLUDE, "-I" + os.path.join(nccl, "include")]

    def compile_one(src):
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        if force or _stale(o, [s] + hdrs):
            cmd = ["nvcc", *ARCH, *NVCCFLAGS, *dflags, *incs, "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return o

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    if force or _stale(lib, objs):
        libdir = os.path.join(nccl, "lib")
        cmd = ["nvcc", *ARCH, "-shared", "-o", lib, *objs, "-L" + libdir, "-l:libnccl.so.2",
               "-Xlinker", "-rpath," + libdir]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
