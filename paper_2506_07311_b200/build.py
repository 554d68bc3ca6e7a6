"""Build the engine's shared library in-tree (nvcc cross-compiles sm_100a).

    python -m paper_2506_07311_b200.build

Produces paper_2506_07311_b200/libpkv200.so: the C-ABI of include/pkv200.h
(host allocator + sm_100a kernels), statically linked against cudart so the
library loads on a CPU-only host too (allocator tests run there).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OUT = os.path.join(PKG, "libpkv200.so")
BUILD = os.path.join(PKG, "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-v"] + ARCH
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-Wall"]

CU_SOURCES = ["kernels.cu", "decode_tc.cu", "prefill_sm100.cu", "step_graph.cu"]
CXX_SOURCES = ["pool.cpp", "status.cpp"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a kernels")


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), out: str = OUT, build_dir: str = BUILD) -> str:
    """Compile and link the library.  `defines` / `out` / `build_dir` build
    an experiment variant (e.g. -DPKV_K3_PHASES) next to the product one;
    load it with PKV200_LIB."""
    nvcc = _nvcc()
    os.makedirs(build_dir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(INCLUDE, "pkv200.h"))
    objs = []
    logs = []
    for src in CU_SOURCES:
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(build_dir, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + headers):
            cmd = [nvcc, *NVCC_FLAGS, *dflags, "-I", INCLUDE, "-I", CSRC, "-c", path, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            logs.append(r.stderr)
            if r.returncode:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-8000:]}")
    for src in CXX_SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(build_dir, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + headers):
            cmd = ["g++", *CXX_FLAGS, "-I", INCLUDE, "-I", CSRC, "-c", path, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode:
                raise RuntimeError(f"g++ failed for {src}:\n{r.stderr[-8000:]}")
    if force or _stale(out, objs):
        cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", out, *objs, "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"link failed:\n{r.stderr[-8000:]}")
    if verbose:
        for log in logs:
            sys.stderr.write(log)
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
