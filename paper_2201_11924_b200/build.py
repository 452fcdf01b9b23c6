"""Build libasd.so (the sm_100a kernels + C ABI) in-tree with nvcc.

    python -m paper_2201_11924_b200.build [--verbose]

Every .cu under csrc/ is compiled for sm_100a only
(-gencode arch=compute_100a,code=sm_100a) with -lineinfo, then linked into
paper_2201_11924_b200/lib/libasd.so against the static CUDA runtime.  Files
listed in NO_FMA are compiled with --fmad=false so their float operations are
single IEEE operations (bit-exact sub-pixel/LR, DESIGN.md §3 reading c13).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
# experiment builds (tools/ab.sh): ASD_VARIANT=name builds lib/variants/name.so
# from csrc/ (or ASD_CSRC) with the ASD_NVCC_DEFS defines, in build/name/
_VARIANT = os.environ.get("ASD_VARIANT", "")
CSRC = os.environ.get("ASD_CSRC", CSRC) if _VARIANT else CSRC
BUILD = os.path.join(PKG, "build", _VARIANT) if _VARIANT else os.path.join(PKG, "build")
LIB = (os.path.join(PKG, "lib", "variants", _VARIANT + ".so") if _VARIANT
       else os.path.join(PKG, "lib", "libasd.so"))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NO_FMA = {"post.cu", "sgm_v2.cu", "register.cu", "noise.cu", "rectify.cu"}


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libasd")


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers_mtime() -> float:
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(INCLUDE, "asd.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
           "-I", INCLUDE, "-I", CSRC, "-c", os.path.join(CSRC, src), "-o", obj]
    if src in NO_FMA:
        cmd.insert(-4, "--fmad=false")
    for d in os.environ.get("ASD_NVCC_DEFS", "").split():      # experiment builds only, e.g. -DASD_ABLATE
        cmd.insert(-4, d)
    if verbose:
        cmd.insert(-4, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr, file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    srcs = _sources()
    hdr = _headers_mtime()
    todo = []
    for s in srcs:
        obj = os.path.join(BUILD, s.replace(".cu", ".o"))
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(
                os.path.getmtime(os.path.join(CSRC, s)), hdr):
            todo.append(s)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(lambda s: _compile(s, verbose), todo))
    objs = [os.path.join(BUILD, s.replace(".cu", ".o")) for s in srcs]
    if todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
