"""Build libbnmc_gpu.so (the C-ABI of include/bnmc_gpu.h) for sm_100a, in-tree.

    python -m paper_1312_3613_b200.build [--force] [--verbose]

Every .cu in csrc/ is compiled with nvcc for `-gencode arch=compute_100a,code=sm_100a`
and `--fmad=false` (the reference is built without FMA contraction; the draws and
weights must round like it), then linked with NCCL into one shared library next
to this file.  No GPU is needed to build.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# BNMC_BUILD_VARIANT=name builds an experiment copy (extra nvcc flags from
# BNMC_NVCC_EXTRA) into _build_<name>/ and libbnmc_gpu_<name>.so; load it with
# BNMC_GPU_LIB=<path>.  The default build is the product library.
_VAR = os.environ.get("BNMC_BUILD_VARIANT", "")
OBJ = os.path.join(HERE, "_build" + (f"_{_VAR}" if _VAR else ""))
LIB = os.path.join(HERE, "libbnmc_gpu" + (f"_{_VAR}" if _VAR else "") + ".so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir():
    """The NCCL that torch loads (the pip nvidia-nccl wheel): linking against the same
    libnccl.so.2 keeps one NCCL in the process whichever library loads first."""
    try:
        import nvidia.nccl as n

        d = os.path.join(list(n.__path__)[0])
        if os.path.exists(os.path.join(d, "lib", "libnccl.so.2")):
            return d
    except Exception:
        pass
    return None


NCCL = _nccl_dir()
FLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
         "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr",
         *os.environ.get("BNMC_NVCC_EXTRA", "").split()]
if NCCL:
    FLAGS += ["-I", os.path.join(NCCL, "include")]


def _deps():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "bnmc_gpu.h")]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _compile(src, verbose):
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    if not _stale(obj, [src, *_deps()]):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, "-Xptxas", "-v", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, (r.stderr if verbose else "")


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if force:
        for o in glob.glob(os.path.join(OBJ, "*.o")):
            os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), srcs))
    objs = [o for o, _ in results]
    for _, log in results:
        if log:
            sys.stderr.write(log)
    if _stale(LIB, objs):
        nccl = (["-Xlinker", os.path.join(NCCL, "lib", "libnccl.so.2"), "-Xlinker", "-rpath",
                 "-Xlinker", os.path.join(NCCL, "lib")] if NCCL else ["-lnccl"])
        # static CUDA runtime: no second libcudart.so.12 next to torch's
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, *nccl]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
