"""Build the in-tree native library ``_build/libpf_b200.so`` (sm_100a only).

    python -m paper_2605_01748_b200.build        # incremental
    python -m paper_2605_01748_b200.build --force

Every CUDA translation unit is compiled for ``-gencode arch=compute_100a,code=sm_100a``
with ``-fmad=false`` (the reference's numba kernels emit no FMA, so exact-order
parity needs unfused multiply-adds; the kernels are HBM-bound so nothing is lost)
and ``-lineinfo`` for ncu source mapping.  Host C++ (the KSP generator) is built
with OpenMP.  The output is a plain C-ABI shared library (include/pf_b200.h) that
the package loads with ctypes; no torch types cross the boundary.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "libpf_b200.so")
GEN_LIB = os.path.join(OUT_DIR, "libpf_gen.so")  # host-only input generation (include/pf_gen.h)
GEN_SOURCES = ("ksp.cpp",)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC,-fopenmp",
              "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cpp")) and f not in GEN_SOURCES)


def build_gen(force: bool = False, verbose: bool = False) -> str:
    """libpf_gen.so: the CPU-only input generators (k shortest paths, path
    validation), g++ with OpenMP -- no CUDA, so input preparation never maps
    the solver library."""
    os.makedirs(OUT_DIR, exist_ok=True)
    srcs = [os.path.join(CSRC, f) for f in GEN_SOURCES]
    hdr = os.path.join(ROOT, "include", "pf_gen.h")
    if force or _stale(GEN_LIB, srcs + [hdr, __file__]):
        cxx = shutil.which("g++") or "g++"
        cmd = [cxx, "-O3", "-std=c++17", "-fPIC", "-shared", "-fopenmp", "-I", os.path.join(ROOT, "include"),
               *srcs, "-o", GEN_LIB]
        if verbose:
            print(" ".join(cmd), flush=True)
        env = dict(os.environ)
        env.pop("CC", None)
        env.pop("CXX", None)
        subprocess.run(cmd, check=True, env=env)
    return GEN_LIB


def headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    inc = os.path.join(ROOT, "include")
    hs += [os.path.join(inc, f) for f in os.listdir(inc) if f.endswith(".h")] if os.path.isdir(inc) else []
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str | None = None, defines=()) -> str:
    """Build the library.  `variant` + `defines` build a tuning variant into
    _build/<variant>/ (selected at run time with PF_B200_LIB=<path>)."""
    out_dir = os.path.join(OUT_DIR, variant) if variant else OUT_DIR
    lib_path = os.path.join(out_dir, "libpf_b200.so") if variant else LIB
    os.makedirs(out_dir, exist_ok=True)
    nvcc = _nvcc()
    env = dict(os.environ)
    # The image's $CC may point at a gcc wrapper without libgomp; nvcc uses the system gcc.
    env.pop("CC", None)
    env.pop("CXX", None)
    objs = []
    hdrs = headers()
    for src in sources():
        obj = os.path.join(out_dir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src, __file__] + hdrs):
            cmd = [nvcc] + ARCH + NVCC_FLAGS + [f"-D{d}" for d in defines] + ["-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True, env=env)
    if force or _stale(lib_path, objs):
        cmd = [nvcc] + ARCH + ["-shared", "-o", lib_path] + objs + ["-lgomp", "-lcudart", "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True, env=env)
    return lib_path


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--variant", default=None, help="tuning variant name (output _build/<variant>/)")
    ap.add_argument("-D", dest="defines", action="append", default=[], help="preprocessor define for a variant")
    a = ap.parse_args(argv)
    if not a.variant:
        print(build_gen(force=a.force, verbose=a.verbose))
    print(build(force=a.force, verbose=a.verbose, variant=a.variant, defines=a.defines))


if __name__ == "__main__":
    sys.exit(main())
