"""Builds the sm_100a shared libraries in-tree (they travel to the GPU box).

  lib/libeigmod_b200.so      C ABI (include/eigmod_b200.h) + all CUDA kernels
  lib/libeigmod_b200_cxx.so  the reference's C++ API (namespace eigmod) as a
                             drop-in over the C ABI (include/eigmod/*.hpp)
  lib/eigmod_b200            the reference CLI's update / locate subcommands
nvcc cross-compiles without a GPU; sources compile in parallel.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "lib")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["secular.cu", "deflate.cu", "eigvec.cu", "gemm.cu", "metrics.cu", "capi.cu",
              "eigpair.cu", "multi.cu"]
CXX_SOURCES = ["eigmod_api.cpp", "io.cpp"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-O3",
           "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
CORE = os.path.join(LIB, "libeigmod_b200.so")
CXX = os.path.join(LIB, "libeigmod_b200_cxx.so")
CLI = os.path.join(LIB, "eigmod_b200")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers() -> list[str]:
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".hpp"))]
    inc = os.path.join(ROOT, "include")
    for dp, _, fs in os.walk(inc):
        hs += [os.path.join(dp, f) for f in fs]
    return hs


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:4])} ...")


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB, exist_ok=True)
    hdrs = _headers()
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([NVCC, *ARCH, *NVFLAGS, "-c", s, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs))
    if force or _stale(CORE, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", CORE, *objs], verbose)
    cxx_src = [os.path.join(CSRC, f) for f in CXX_SOURCES]
    if all(os.path.exists(s) for s in cxx_src) and (force or _stale(CXX, cxx_src + hdrs + [CORE])):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-fopenmp", "-I",
              os.path.join(ROOT, "include"),
              *cxx_src, "-o", CXX, "-L", LIB, "-leigmod_b200", f"-Wl,-rpath,{LIB}",
              "-Wl,-rpath,$ORIGIN"], verbose)
    cli_src = os.path.join(CSRC, "cli.cpp")
    if os.path.exists(cli_src) and (force or _stale(CLI, [cli_src, CXX] + hdrs)):
        _run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), cli_src, "-o", CLI,
              "-L", LIB, "-leigmod_b200_cxx", "-leigmod_b200", "-Wl,-rpath,$ORIGIN"], verbose)
    return CORE


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
