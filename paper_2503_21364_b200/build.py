"""Build liblmgs.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2503_21364_b200.build [--force]

Each csrc/*.cu compiles to an object with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo``; preprocess.cu adds
``-fmad=false`` so its fp64 geometry rounds exactly where the reference's
torch ops do.  The objects link into ``paper_2503_21364_b200/liblmgs.so``
(static cudart), which travels with the repo snapshot to the GPU box.
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
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "liblmgs.so"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
          f"-I{INCLUDE}", "--expt-relaxed-constexpr"]
PER_FILE = {"preprocess.cu": ["-fmad=false"], "backward_exact.cu": ["-fmad=false"],
            "touched_fix.cu": ["-fmad=false"]}
# extra nvcc flags for tuning experiments (e.g. "-DLMGS_PRE_MIN_CTAS=6")
EXTRA = os.environ.get("LMGS_NVCC_FLAGS", "").split()


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


TORCH_OPS_SRC = CSRC / "torch_ops.cpp"
TORCH_OPS_LIB = PKG / "_lmgs_torch.so"


def _sources():
    return sorted(CSRC.glob("*.cu"))


def build_torch_ops(force: bool = False) -> Path:
    """The TORCH_LIBRARY(lmgs) operators (csrc/torch_ops.cpp): a g++-built
    shared object over liblmgs.so (rpath $ORIGIN) and libtorch, in-tree."""
    if not (force or _stale(TORCH_OPS_LIB, [TORCH_OPS_SRC, LIB, INCLUDE / "lmgs.h",
                                            Path(__file__)])):
        return TORCH_OPS_LIB
    import torch
    from torch.utils import cpp_extension as ce

    abi = int(torch.compiled_with_cxx11_abi())
    incs = [f"-I{p}" for p in ce.include_paths(device_type="cuda")]
    libs = [f"-L{p}" for p in ce.library_paths(device_type="cuda")]
    rpaths = [f"-Wl,-rpath,{p}" for p in ce.library_paths(device_type="cuda")]
    tmp = TORCH_OPS_LIB.with_suffix(".so.tmp")
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", f"-D_GLIBCXX_USE_CXX11_ABI={abi}",
           *incs, str(TORCH_OPS_SRC), "-o", str(tmp), f"-L{PKG}", "-llmgs",
           "-Wl,-rpath,$ORIGIN", *libs, *rpaths, "-lc10", "-lc10_cuda", "-ltorch_cpu",
           "-ltorch_cuda", "-ltorch"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"torch ops build failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, TORCH_OPS_LIB)
    return TORCH_OPS_LIB


def _deps():
    return list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))


def _stale(target: Path, inputs) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(p.stat().st_mtime > t for p in inputs)


def _compile(src: Path, force: bool, log: list) -> Path:
    obj = BUILD / (src.stem + ".o")
    if force or _stale(obj, [src, *_deps(), Path(__file__)]):
        cmd = [nvcc(), *ARCH, *COMMON, *PER_FILE.get(src.name, []), *EXTRA, "-c", str(src), "-o",
               str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.append((src.name, r.stderr))
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    log: list = []
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, log), srcs))
    if force or _stale(LIB, objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart_static",
               "-Xlinker", "-soname=liblmgs.so", "-Xlinker", "--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, LIB)
    build_torch_ops(force)
    if verbose:
        for name, err in log:
            print(f"--- {name}\n{err}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
