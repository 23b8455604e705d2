"""Build the sm_100a shared library in-tree (no JIT cache, travels with the repo).

    python -m paper_2309_12543_b200.build          # -> paper_2309_12543_b200/_lib/liblinksdf_b200.so

nvcc cross-compiles for B200 without a GPU.  Flags: -gencode
arch=compute_100a,code=sm_100a (the only target), -lineinfo for ncu source
pages, -O3, and --fmad=false as a belt-and-braces guard: the parity-critical
arithmetic already uses explicit __fma_rn/__dmul_rn/__dadd_rn intrinsics.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "liblinksdf_b200.so"
INCLUDE = PKG.parent / "include"

SOURCES = ["lsdf_capi.cu", "lsdf_fk.cu", "lsdf_voxel.cu", "lsdf_query.cu", "lsdf_dense.cu", "lsdf_build.cu",
           "lsdf_mlp.cu", "lsdf_mlp_tc.cu", "lsdf_vmajor.cu", "lsdf_train.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build linksdf-b200")


def _digest() -> str:
    h = hashlib.sha256()
    for name in SOURCES + ["lsdf_math.cuh", "lsdf_common.cuh", "lsdf_device.cuh", "lsdf_async.cuh", "lsdf_tc.cuh"]:
        h.update((CSRC / name).read_bytes())
    h.update((INCLUDE / "linksdf_b200.h").read_bytes())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False) -> Path:
    OUT_DIR.mkdir(exist_ok=True)
    stamp = OUT_DIR / "BUILD_ID"
    digest = _digest()
    if LIB.exists() and stamp.exists() and stamp.read_text().strip() == digest and not force:
        return LIB
    nvcc = _nvcc()
    objs = []
    log = []
    for name in SOURCES:
        obj = OUT_DIR / (Path(name).stem + ".o")
        cmd = [nvcc, *ARCH, *FLAGS, "-I", str(INCLUDE), "-c", str(CSRC / name), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.append(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {name}:\n{r.stdout}\n{r.stderr}")
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *objs, "-lcuda"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    (OUT_DIR / "ptxas.log").write_text("\n".join(log))
    stamp.write_text(digest + "\n")
    if verbose:
        print("\n".join(log))
    return LIB


DEMO_SRC = PKG.parent / "tests" / "native" / "abi_demo.c"
DEMO = OUT_DIR / "abi_demo"


def build_demo(force: bool = False) -> Path:
    """The plain-C ABI client (tests/native/abi_demo.c), linked against the library."""
    lib = build()
    if DEMO.exists() and not force and DEMO.stat().st_mtime >= max(DEMO_SRC.stat().st_mtime, lib.stat().st_mtime):
        return DEMO
    nvcc = _nvcc()
    cmd = [nvcc, "-O2", "-x", "c", str(DEMO_SRC), "-I", str(INCLUDE), "-L", str(OUT_DIR), "-llinksdf_b200",
           "-Xlinker", "-rpath=$ORIGIN", "-o", str(DEMO)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"abi_demo build failed:\n{r.stdout}\n{r.stderr}")
    return DEMO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    print(build_demo(force="--force" in sys.argv))
