"""Build the sm_100a shared library ``libquadsim_b200.so`` in-tree.

    python -m paper_2509_10247_b200.build [-j N] [--force]

Each ``csrc/*.cu`` is compiled to an object in parallel with
``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into
one C-ABI shared library (no torch types cross the boundary).  Objects are
rebuilt only when a source or header is newer.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libquadsim_b200.so")
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE,
                     "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the quadsim_b200 CUDA library cannot be built")


def _deps_mtime() -> float:
    files = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return max((os.path.getmtime(f) for f in files), default=0.0)


def _compile(src: str, obj: str) -> tuple[str, str]:
    cmd = [nvcc()] + NVCC_FLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(src)}:\n{r.stderr}")
    return src, r.stderr


TORCH_OPS_SRC = os.path.join(CSRC, "qs_torch_ops.cpp")
TORCH_OPS_LIB = os.path.join(PKG, "_qs_torch_ops.so")


def build_torch_ops(force: bool = False, verbose: bool = False) -> str:
    """The torch custom-op layer (``quadsim::task_step``): one C++ file
    compiled against torch's headers, linked to ``libquadsim_b200.so``
    (rpath $ORIGIN) and loaded with ``torch.ops.load_library``."""
    deps = [TORCH_OPS_SRC, LIB, os.path.join(INCLUDE, "quadsim_b200.h")]
    if not force and os.path.exists(TORCH_OPS_LIB) and \
            os.path.getmtime(TORCH_OPS_LIB) >= max(os.path.getmtime(d) for d in deps):
        return TORCH_OPS_LIB
    import torch
    from torch.utils import cpp_extension as ce

    import sysconfig

    incs = ce.include_paths(device_type="cuda") + [sysconfig.get_paths()["include"]]
    libs = ce.library_paths(device_type="cuda")
    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    cxx = os.environ.get("CXX") or shutil.which("g++") or "g++"
    cmd = [cxx, "-O2", "-std=c++17", "-fPIC", "-shared", f"-D_GLIBCXX_USE_CXX11_ABI={abi}", TORCH_OPS_SRC,
           "-o", TORCH_OPS_LIB + ".tmp"] + [f"-I{i}" for i in incs] + [f"-L{d}" for d in libs] + [
           "-DTORCH_EXTENSION_NAME=_qs_torch_ops", "-DTORCH_API_INCLUDE_EXTENSION_H",
           "-ltorch", "-ltorch_cpu", "-ltorch_cuda", "-ltorch_python", "-lc10", "-lc10_cuda", "-lcudart",
           f"-L{PKG}", "-lquadsim_b200", "-Wl,-rpath,$ORIGIN"] + [f"-Wl,-rpath,{d}" for d in libs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"torch op layer build failed:\n{r.stderr[-4000:]}")
    os.replace(TORCH_OPS_LIB + ".tmp", TORCH_OPS_LIB)
    if verbose:
        print("compiled qs_torch_ops.cpp", file=sys.stderr)
    return TORCH_OPS_LIB


def build(jobs: int | None = None, force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    dep_t = _deps_mtime()
    todo = []
    objs = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), dep_t):
            todo.append((s, o))
    if todo:
        jobs = jobs or min(len(todo), os.cpu_count() or 4)
        with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
            for src, err in ex.map(lambda so: _compile(*so), todo):
                if verbose:
                    print(f"compiled {os.path.basename(src)}", file=sys.stderr)
    if todo or not os.path.exists(LIB):
        tmp = LIB + ".tmp"
        cmd = [nvcc()] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, LIB)
    build_torch_ops(force=force, verbose=verbose)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    print(build(a.j, a.force, verbose=True))
