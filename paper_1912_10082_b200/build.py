"""Build the in-tree CUDA shared library ``_stk_gpu.so`` (sm_100a, FP64 kernels + C ABI).

The library is compiled straight with nvcc (no torch extension machinery): it exposes only
the C ABI declared in ``include/stk_gpu.h`` and is loaded with ctypes by ``_lib.py`` and by
any C / cgo / JNI caller.  The .so is git-ignored but travels to the
GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "_stk_gpu.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc" if Path("/usr/local/cuda/bin/nvcc").exists() else "nvcc")

CUDA_SOURCES = ["heat.cu", "wave.cu", "krylov.cu", "rksm.cu", "runtime.cu"]
HOST_SOURCES = ["host_assembly.cpp", "errors.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler",
                     "-fopenmp", "-Xptxas", "-v", "--expt-relaxed-constexpr"]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-fopenmp"]


def _sources():
    return [CSRC / s for s in CUDA_SOURCES + HOST_SOURCES] + sorted(CSRC.glob("*.cuh")) + [
        ROOT / "include" / "stk_gpu.h"]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in _sources())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    extra = os.environ.get("STKG_NVCC_EXTRA", "").split()  # variant builds (tools/ab.sh)
    cxx = shutil.which("g++") or "g++"
    jobs = [(src, [NVCC, *NVCC_FLAGS, *extra, "-c", str(CSRC / src), "-o",
                   str(objdir / (src + ".o"))]) for src in CUDA_SOURCES]
    jobs += [(src, [cxx, *CXX_FLAGS, "-c", str(CSRC / src), "-o", str(objdir / (src + ".o"))])
             for src in HOST_SOURCES]

    def run(job):
        src, cmd = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed for {src}:\n{r.stderr}")
        return r.stdout + r.stderr

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(jobs)) as pool:  # nvcc is single-threaded
        log = list(pool.map(run, jobs))
    objs = [objdir / (src + ".o") for src, _ in jobs]
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fopenmp", "-o", str(tmp), *map(str, objs),
           "-lcudart_static", "-lrt", "-lpthread", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    tmp.replace(LIB)
    (objdir / "ptxas.log").write_text("\n".join(log))
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    out = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(out)
