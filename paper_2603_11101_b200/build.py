"""In-tree build of the CUDA library (sm_100a) and the C++ host library.

    python -m paper_2603_11101_b200.build [--force] [-v]

Outputs (git-ignored, shipped to the GPU box by gpurun with the snapshot):
    paper_2603_11101_b200/lib/libvlasim_cuda.so   kernels + C-ABI (include/vlasim_cuda.h)
    paper_2603_11101_b200/lib/libvlasim.so        reconstructed vlasim:: C++ API over the C-ABI
    paper_2603_11101_b200/lib/vlasim_pack         C++ CLI front end (`pack` subcommand)
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
OBJ = ROOT / "build" / "obj"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(INCLUDE),
                     "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
CXX = os.environ.get("CXX", shutil.which("g++") or "g++")

CUDA_SOURCES = sorted(CSRC.glob("*.cu"))
HOST_SOURCES = sorted((CSRC / "host").glob("*.cpp"))
CUDA_HEADERS = sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.hpp")) + [INCLUDE / "vlasim_cuda.h"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(map(str, cmd)), flush=True)
    r = subprocess.run(list(map(str, cmd)), capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build step failed:\n{' '.join(map(str, cmd))}\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr)
    return r


def build_cuda(force=False, verbose=False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    LIB.mkdir(parents=True, exist_ok=True)
    objs, jobs = [], []
    for src in CUDA_SOURCES:
        obj = OBJ / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + CUDA_HEADERS):
            jobs.append([NVCC] + NVCC_FLAGS + ["-c", src, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs))
    so = LIB / "libvlasim_cuda.so"
    if force or jobs or _stale(so, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", so] + objs + ["-lpthread"], verbose)
    return so


def build_host(force=False, verbose=False) -> Path | None:
    """Reconstructed vlasim:: C++ API (include/vlasim/packing/*.hpp) + CLI over the C-ABI."""
    if not HOST_SOURCES:
        return None
    so = LIB / "libvlasim.so"
    deps = HOST_SOURCES + sorted(INCLUDE.rglob("*.hpp")) + [INCLUDE / "vlasim_cuda.h", LIB / "libvlasim_cuda.so"]
    lib_sources = [s for s in HOST_SOURCES if not s.name.startswith("cli_")]
    cuda_inc = Path(NVCC).resolve().parent.parent / "include"
    cuda_lib = Path(NVCC).resolve().parent.parent / "lib64"
    if force or _stale(so, deps):
        _run([CXX, "-std=c++20", "-O2", "-fPIC", "-shared", "-I", INCLUDE, "-I", cuda_inc, "-o", so] + lib_sources +
             ["-L", LIB, "-lvlasim_cuda", "-Wl,-rpath,$ORIGIN", "-L", cuda_lib, "-lcudart",
              "-Wl,-rpath," + str(cuda_lib)], verbose)
    for cli in [s for s in HOST_SOURCES if s.name.startswith("cli_")]:
        exe = LIB / cli.stem.replace("cli_", "vlasim_")
        if force or _stale(exe, deps + [so]):
            _run([CXX, "-std=c++20", "-O2", "-I", INCLUDE, "-I", cuda_inc, "-o", exe, cli, "-L", LIB, "-lvlasim",
                  "-lvlasim_cuda", "-Wl,-rpath,$ORIGIN", "-L", cuda_lib, "-lcudart", "-Wl,-rpath," + str(cuda_lib)],
                 verbose)
    return so


def build_all(force=False, verbose=False):
    build_cuda(force, verbose)
    build_host(force, verbose)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args(argv)
    build_all(a.force, a.verbose)
    print("built", LIB)


if __name__ == "__main__":
    sys.exit(main())
