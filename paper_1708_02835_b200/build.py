"""Build libexageo.so (the C-ABI library) in-tree for sm_100a.

    python -m paper_1708_02835_b200.build [--force] [--verbose]

Each source under csrc/ is compiled by nvcc with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` (host code with
-ffp-contract=off so that the location generator is bit-exact), then linked
into paper_1708_02835_b200/_lib/libexageo.so with the static CUDA runtime.
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libexageo.so")
INCLUDE = os.path.join(ROOT, "include")
SOURCES = ["api.cu", "matern.cu", "gemm_dmma.cu", "potrf_reduce.cu", "dag.cu", "trsv.cu", "locations.cpp", "mle.cpp",
           "nccl_dyn.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def cutlass_include() -> str:
    """The CUTLASS header tree vendored in this image (flashinfer's, else tilelang's copy): the
    trailing-update kernel builds its DMMA mainloop and epilogue from CUTLASS's SM80 templates
    inside our own kernel (gemm_dmma.cu). Fails loudly when no tree is found."""
    import site
    roots = [os.environ.get("EXAGEO_CUTLASS_INCLUDE", "")]
    for sp in site.getsitepackages() + [site.getusersitepackages()]:
        roots += [os.path.join(sp, "flashinfer", "data", "cutlass", "include"),
                  os.path.join(sp, "tilelang", "3rdparty", "cutlass", "include")]
    for r in roots:
        if r and os.path.exists(os.path.join(r, "cutlass", "gemm", "kernel", "default_gemm.h")):
            return r
    raise RuntimeError("CUTLASS headers not found (set EXAGEO_CUTLASS_INCLUDE to a cutlass/include tree)")


def _flags(src: str) -> list[str]:
    f = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off", "-I", INCLUDE, "-I", CSRC]
    if src == "gemm_dmma.cu":
        f += ["-I", cutlass_include()]
    f += ARCH
    f += os.environ.get("EXAGEO_EXTRA_NVCC_FLAGS", "").split()  # development builds (e.g. -DEXAGEO_POTRF_TRACE)
    if src.endswith(".cu"):
        f += ["-Xptxas", "-warn-spills"]
    return f


def _stale(deps: list[str], target: str) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    headers.append(os.path.join(INCLUDE, "exageo.h"))
    objs, jobs = [], []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OUT_DIR, s + ".o")
        objs.append(obj)
        if force or _stale([src] + headers, obj):
            cmd = [nvcc()] + _flags(s) + ["-c", src, "-o", obj]
            if s.endswith(".cpp"):
                cmd = [nvcc(), "-x", "c++"] + _flags(s) + ["-c", src, "-o", obj]
            jobs.append(cmd)

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, flush=True)

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(objs, LIB):
        # NCCL is resolved at run time (csrc/nccl_dyn.cpp), not linked
        cmd = [nvcc(), "-shared"] + ARCH + ["-cudart", "static", "-o", LIB] + objs + ["-ldl"]
        run(cmd)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
    sys.exit(0)
