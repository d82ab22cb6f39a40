"""In-tree build of the CUDA extension (libasicp.so) for sm_100a.

`python -m paper_2412_08346_b200.build` (or __graft_entry__.build()) compiles
the product sources under csrc/ with nvcc for `-gencode
arch=compute_100a,code=sm_100a` and links them into
paper_2412_08346_b200/libasicp.so, which the ctypes binding
(paper_2412_08346_b200/_lib.py) loads.  The synthetic-input generators
(csrc/fixtures.cu, host-only C++) go into their own library,
libasicp_fixtures.so: they feed tests and bench.py, never the solve.  Both
libraries travel to the GPU box with the repo snapshot; no JIT cache is
involved.
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
OBJ = PKG / "_build"
LIB = PKG / "libasicp.so"
FX_LIB = PKG / "libasicp_fixtures.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: the FP64 path must not contract a*b+c (the reference oracle is
# built without FMA); the FP32 NN filter requests its FMAs explicitly.
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC,-O3",
              "-diag-suppress", "177", f"-I{ROOT / 'include'}"]
# Diagnostic builds only (e.g. ASICP_NVCC_EXTRA=-DASICP_NN_PHASES, tools/nn_phases.sh).
NVCC_FLAGS += os.environ.get("ASICP_NVCC_EXTRA", "").split()
SOURCES = ["kernels.cu", "collide.cu", "median.cu", "nn.cu", "minibatch.cu", "exchange.cu", "register.cu", "sdf_build.cu", "solver.cu",
           "trace_io.cpp"]
FX_SOURCE = "fixtures.cu"


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; the CUDA extension cannot be built")
    return cand


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    nvcc = _nvcc()
    OBJ.mkdir(exist_ok=True)
    headers = sorted(CSRC.glob("*.cuh")) + sorted((ROOT / "include").glob("*.h"))
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = OBJ / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [nvcc, *ARCH, *NVCC_FLAGS, "-c", str(s), "-o", str(o)]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    if force or _stale(LIB, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart", "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    fx_src = CSRC / FX_SOURCE
    if force or _stale(FX_LIB, [fx_src] + headers):
        cmd = [shutil.which("g++") or "g++", "-x", "c++", "-std=c++17", "-O2", "-fPIC", "-shared",
               f"-I{ROOT / 'include'}", "-o", str(FX_LIB), str(fx_src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
