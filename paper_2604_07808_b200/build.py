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


def build(verbose: bool = False, force: bool = False, defines=(), out: str | None = None,
          src_dir: str | None = None) -> str:
    """defines/out: developer A/B variants (e.g. tools/variants.py); src_dir: a
    patched copy of csrc/ (tools/kernel_mutation.py); the product is OUT built
    from CSRC."""
    out_path = out or OUT
    csrc = src_dir or CSRC
    cuda = _cuda_home()
    nvcc = os.path.join(cuda, "bin", "nvcc")
    srcs = sorted(os.listdir(csrc))
    deps = [os.path.join(csrc, f) for f in srcs] + [os.path.join(ROOT, "include", "grass.h"), __file__]
    if not force and os.path.exists(out_path) and os.path.getmtime(out_path) >= max(os.path.getmtime(d) for d in deps):
        return out_path
    build_dir = BUILD if out is None else os.path.join(BUILD, "variant_" + os.path.basename(out_path).replace(".so", ""))
    os.makedirs(build_dir, exist_ok=True)
    dflags = ["-D" + d for d in defines]
    inc = ["-I" + os.path.join(ROOT, "include"), "-I" + _nccl_include(), "-I" + os.path.join(cuda, "include")]
    objs = []
    log = []
    for f in srcs:
        src = os.path.join(csrc, f)
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
          "-Xlinker", "--version-script=" + os.path.join(csrc, "exports.map"),
          "-ldl", "-lpthread", "-lrt", "-lz"], verbose)
    os.replace(tmp, out_path)
    with open(os.path.join(build_dir, "ptxas.log"), "w") as fh:
        fh.write("\n".join(log))
    if out is None:
        build_diag(verbose, force)
    return out_path


DIAG = os.path.join(PKG, "diag")
DIAG_OUT = os.path.join(PKG, "libgrass_diag.so")


def build_diag(verbose: bool = False, force: bool = False) -> str:
    """libgrass_diag.so: measurement kernels of bench.py (the read-only HBM
    ceiling, diag/read_ceiling.cu) — not part of the hot path."""
    srcs = [os.path.join(DIAG, f) for f in sorted(os.listdir(DIAG)) if f.endswith(".cu")]
    if not force and os.path.exists(DIAG_OUT) and os.path.getmtime(DIAG_OUT) >= max(
            [os.path.getmtime(x) for x in srcs] + [os.path.getmtime(__file__)]):
        return DIAG_OUT
    nvcc = os.path.join(_cuda_home(), "bin", "nvcc")
    tmp = DIAG_OUT + ".tmp"
    _run([nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-cudart", "static",
          "-Xcompiler", "-fPIC", *srcs, "-o", tmp], verbose)
    os.replace(tmp, DIAG_OUT)
    return DIAG_OUT


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
