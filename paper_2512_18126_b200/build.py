"""Build the in-tree C-ABI library libmoa_b200.so (sm_100a only).

    python -m paper_2512_18126_b200.build [--force] [-j N]

CUDA sources compile with nvcc for `-gencode arch=compute_100a,code=sm_100a`
(cross-compiles without a GPU); host C++ compiles with g++ -std=c++20; the
CUDA runtime is linked statically so the .so has no runtime path
dependencies on the GPU box.
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libmoa_b200.so"
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                     "-Xptxas", "-warn-spills"]
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter", f"-I{CUDA / 'include'}"]


def _sources():
    cu = sorted((CSRC / "kernels").glob("*.cu"))
    cpp = sorted((CSRC / "host").glob("*.cpp"))
    return cu, cpp


def _headers():
    return list(CSRC.rglob("*.hpp")) + list(CSRC.rglob("*.cuh")) + [PKG.parent / "include" / "moa_b200.h"]


def _stale(obj: Path, src: Path, hdr_mtime: float) -> bool:
    return not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, hdr_mtime)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stderr


def build(force: bool = False, jobs: int = 8, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    cu, cpp = _sources()
    hdr = max(h.stat().st_mtime for h in _headers())
    tasks = []
    for s in cu:
        o = OBJ / (s.stem + ".cu.o")
        if force or _stale(o, s, hdr):
            tasks.append([NVCC, *NVCC_FLAGS, "-c", str(s), "-o", str(o)])
    for s in cpp:
        o = OBJ / (s.stem + ".o")
        if force or _stale(o, s, hdr):
            tasks.append(["g++", *CXX_FLAGS, "-c", str(s), "-o", str(o)])
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        for log in ex.map(_run, tasks):
            if verbose and log.strip():
                print(log, file=sys.stderr)
    objs = [str(OBJ / (s.stem + ".cu.o")) for s in cu] + [str(OBJ / (s.stem + ".o")) for s in cpp]
    if tasks or not LIB.exists() or force:
        _run(["g++", "-shared", "-o", str(LIB), *objs, f"-L{CUDA / 'lib64'}", "-lcudart_static", "-lrt",
              "-lpthread", "-ldl"])
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=8)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.j, a.v))
