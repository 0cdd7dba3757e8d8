"""In-tree build of libmmb.so (the B200 product library) for sm_100a.

    python -m paper_1501_07293_b200.build          # incremental
    python -m paper_1501_07293_b200.build --force

Each translation unit is compiled by nvcc with -gencode arch=compute_100a,code=sm_100a
-lineinfo; the local-term/LLG unit is compiled with --fmad=false so its arithmetic rounds
exactly like the reference (no FMA contraction). Objects go to build/ and the shared
library lands next to this file (git-ignored, travels to the GPU box with the snapshot).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# MMB_BUILD_DIR / MMB_LIB_OUT build a variant library elsewhere (tuning experiments only)
BUILD = os.environ.get("MMB_BUILD_DIR", os.path.join(ROOT, "build", "mmb"))
LIB = os.environ.get("MMB_LIB_OUT", os.path.join(HERE, "libmmb.so"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir():
    """The NCCL that torch loads (nvidia-nccl wheel), so one libnccl.so.2 serves both in a
    process; the system NCCL only when the wheel is absent."""
    try:
        import nvidia  # namespace package of the CUDA wheels
        for base in nvidia.__path__:
            d = os.path.join(base, "nccl")
            if os.path.exists(os.path.join(d, "lib", "libnccl.so.2")):
                return d
    except ImportError:
        pass
    return None


NCCL_DIR = _nccl_dir()
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-Xptxas", "-warn-spills", f"-I{os.path.join(ROOT, 'include')}"]
if NCCL_DIR:
    COMMON = COMMON[:-1] + [f"-I{os.path.join(NCCL_DIR, 'include')}"] + COMMON[-1:]

# (object name, source, extra flags)
UNITS = [
    ("fft_f32.o", "fft_kernels.cu", ["-DMMB_ONLY_F32"]),
    ("fft_f64.o", "fft_kernels.cu", ["-DMMB_ONLY_F64"]),
    ("fast_f32.o", "fast_kernels.cu", ["-DMMB_ONLY_F32"] + os.environ.get("MMB_XFLAGS", "").split()),
    ("fast_f64.o", "fast_kernels.cu", ["-DMMB_ONLY_F64"]),
    ("big_f32.o", "big_kernels.cu", ["-DMMB_ONLY_F32"] + os.environ.get("MMB_XFLAGS", "").split()),
    ("big_f64.o", "big_kernels.cu", ["-DMMB_ONLY_F64"]),
    ("llg.o", "llg_kernels.cu", ["--fmad=false"]),
    ("tensor.o", "tensor_kernels.cu", ["--fmad=false"]),
    ("solver.o", "solver.cu", []),
    ("shard.o", "shard.cu", []),
    ("validate.o", "validate.cu", []),
]


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    hs.append(os.path.join(ROOT, "include", "mmb.h"))
    return hs


def _stale(obj, src):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src] + _headers())


def _compile(unit, force, verbose):
    obj, src, extra = unit
    src = os.path.join(CSRC, src)
    out = os.path.join(BUILD, obj)
    if not force and not _stale(out, src):
        return out, False
    cmd = [NVCC] + ARCH + COMMON + extra + ["-c", src, "-o", out]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and verbose:
        print(r.stderr, file=sys.stderr)
    return out, True


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(UNITS)) as ex:
        results = list(ex.map(lambda u: _compile(u, force, verbose), UNITS))
    objs = [o for o, _ in results]
    if force or any(changed for _, changed in results) or not os.path.exists(LIB):
        nccl = (["-L" + os.path.join(NCCL_DIR, "lib"), "-Xlinker", "-l:libnccl.so.2", "-Xlinker", "-rpath", "-Xlinker", os.path.join(NCCL_DIR, "lib")]
                if NCCL_DIR else ["-lnccl"])
        cmd = [NVCC] + ARCH + ["-shared", "-Xlinker", "-soname=libmmb.so", "-o", LIB] + objs + ["-lcudart"] + nccl
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
