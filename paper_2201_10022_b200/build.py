"""Build the sm_100a shared library in-tree: paper_2201_10022_b200/libabd_b200.so.

    python -m paper_2201_10022_b200.build [--force]

Each csrc/*.cu compiles separately (parallel nvcc), then links with -shared.
The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libabd_b200.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                "-Xptxas", "-warn-spills"]
if os.environ.get("ABD_PTXAS_O"):
    BUILD = os.path.join(HERE, "_build_o" + os.environ["ABD_PTXAS_O"])
    LIB = os.path.join(HERE, "libabd_b200_o" + os.environ["ABD_PTXAS_O"] + ".so")
    FLAGS = FLAGS + ["-Xptxas", "-O" + os.environ["ABD_PTXAS_O"]]
if os.environ.get("ABD_DEVICE_DEBUG"):
    BUILD = os.path.join(HERE, "_build_dbg")
    LIB = os.path.join(HERE, "libabd_b200_dbg.so")
    FLAGS = ARCH + ["-G", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(os.path.dirname(HERE), "include", "abd_b200.h"))
    return max(os.path.getmtime(h) for h in hs if os.path.exists(h))


def _compile(src, force):
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    s = os.path.join(CSRC, src)
    if not force and os.path.exists(obj):
        t = os.path.getmtime(obj)
        if t >= os.path.getmtime(s) and t >= _headers_mtime():
            return obj, ""
    cmd = [NVCC] + FLAGS + ["-c", s, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        res = list(ex.map(lambda s: _compile(s, force), srcs))
    objs = [o for o, _ in res]
    if verbose:
        for o, log in res:
            if log.strip():
                print(os.path.basename(o), log)
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
