"""Build libapmm_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2409_17870_b200.build [--force] [--verbose] [--dev]

The shared library exports exactly the C ABI declared in include/apmm_cuda.h. The release
build reads no environment variables. `--dev` builds the same sources with
-DAPMM_DEVTOOLS (plan dumps, per-phase timelines, ablations; csrc/internal.h) into
abtest/libapmm_b200_dev.so (git-ignored), for the scripts/ probes via APMM_LIB -- never
the product.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libapmm_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3,-fvisibility=hidden",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + sorted(
        glob.glob(os.path.join(CSRC, "*.h"))) + [os.path.join(ROOT, "include", "apmm_cuda.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


DEV_LIB = os.path.join(ROOT, "abtest", "libapmm_b200_dev.so")


def build(force: bool = False, verbose: bool = False, dev: bool = False) -> str:
    lib = DEV_LIB if dev else LIB
    if not force and not dev and up_to_date():
        return LIB
    objdir = os.path.join(PKG, "build_dev" if dev else "build")
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    os.makedirs(objdir, exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC] + NVCC_FLAGS + (["-DAPMM_DEVTOOLS"] if dev else []) + ["-c", src, "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    objs = []
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, sources()))
    for src, obj, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    # default symbol visibility for the exported C ABI: the .cu files mark nothing hidden
    # explicitly, so link with an explicit export list via a version script.
    vscript = os.path.join(objdir, "exports.map")
    with open(vscript, "w") as f:
        f.write("{ global: apmm_*; local: *; };\n")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib] + objs + [
        "-Xlinker", f"--version-script={vscript}", "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv,
                dev="--dev" in sys.argv))
