"""Builds libgrass.so in-tree for sm_100a (nvcc + g++; no torch extension).

    python -m paper_2604_07808_b200.build      # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libgrass.so")
BUILD = os.path.join(ROOT, "build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _cuda_home() -> str:
    for c in (os.environ.get("CUDA_HOME"), "/usr/local/cuda"):
        if c and os.path.exists(os.path.join(c, "bin", "nvcc")):
            return c
    nvcc = shutil.which("nvcc")
    if nvcc:
        return os.path.dirname(os.path.dirname(nvcc))
    raise RuntimeError("nvcc not found")


def _nccl_include() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        inc = os.path.join(base, "nccl", "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include"
    raise RuntimeError("nccl.h not found")


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stdout + r.stderr


def build(verbose: bool = False, force: bool = False, defines=(), out: str | None = None) -> str:
    """defines/out: developer A/B variants (e.g. tools/variants.py); the product is OUT."""
    out_path = out or OUT
    cuda = _cuda_home()
    nvcc = os.path.join(cuda, "bin", "nvcc")
    srcs = sorted(os.listdir(CSRC))
    deps = [os.path.join(CSRC, f) for f in srcs] + [os.path.join(ROOT, "include", "grass.h"), __file__]
    if not force and os.path.exists(out_path) and os.path.getmtime(out_path) >= max(os.path.getmtime(d) for d in deps):
        return out_path
    build_dir = BUILD if out is None else os.path.join(BUILD, "variant_" + os.path.basename(out_path).replace(".so", ""))
    os.makedirs(build_dir, exist_ok=True)
    dflags = ["-D" + d for d in defines]
    inc = ["-I" + os.path.join(ROOT, "include"), "-I" + _nccl_include(), "-I" + os.path.join(cuda, "include")]
    objs = []
    log = []
    for f in srcs:
        src = os.path.join(CSRC, f)
        obj = os.path.join(build_dir, f + ".o")
        if f.endswith(".cu"):
            log.append(_run([nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--fmad=false",
                             "-Xptxas", "-v", "-Xcompiler", "-fPIC,-ffp-contract=off",
                             *dflags, *inc, "-c", src, "-o", obj], verbose))
        elif f.endswith(".cpp"):
            log.append(_run(["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall",
                             *dflags, *inc, "-c", src, "-o", obj], verbose))
        else:
            continue
        objs.append(obj)
    tmp = out_path + ".tmp"
    _run([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
          "-Xlinker", "--version-script=" + os.path.join(CSRC, "exports.map"),
          "-ldl", "-lpthread", "-lrt", "-lz"], verbose)
    os.replace(tmp, out_path)
    with open(os.path.join(build_dir, "ptxas.log"), "w") as fh:
        fh.write("\n".join(log))
    return out_path


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
