"""In-tree build of the CUDA library (nvcc, sm_100a) and the native test tools.

    python -m paper_2508_08343_b200.build        # builds everything that is stale
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib", "libloratwin_gpu.so")
INCLUDE = os.path.join(ROOT, "include")
NATIVE = os.path.join(ROOT, "tests", "native")
NATIVE_BIN = os.path.join(NATIVE, "bin")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
    # The reference's arithmetic is reproduced operation by operation: no
    # contraction on device (--fmad=false) or host (-ffp-contract=off).
    "--fmad=false", "-DLT_NO_CONTRACT", "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-Xptxas", "-v",
]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def build_gpu(force: bool = False, verbose: bool = False, prof: bool = False, stats: bool = False) -> str:
    """libloratwin_gpu.so; prof=True builds libloratwin_gpu_prof.so with the
    per-phase cycle counters (-DLT_PHASE_PROF) used by tools/diag_phase.py,
    stats=True libloratwin_gpu_stats.so with scan counters (-DLT_SCAN_STATS)."""
    lib = LIB.replace(".so", "_prof.so") if prof else (LIB.replace(".so", "_stats.so") if stats else LIB)
    deps = glob.glob(os.path.join(CSRC, "*")) + [os.path.join(INCLUDE, "loratwin_gpu.h")]
    if not force and not _stale(lib, deps):
        return lib
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    cmd = [nvcc()] + NVCC_FLAGS + (["-DLT_PHASE_PROF"] if prof else []) + (["-DLT_SCAN_STATS"] if stats else []) + [
        "-I" + INCLUDE, "-I" + CSRC, "-shared", "-o", lib, os.path.join(CSRC, "capi.cu")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libloratwin_gpu.so")
    with open(os.path.join(os.path.dirname(lib), "ptxas" + ("_prof" if prof else "_stats" if stats else "") + ".log"), "w") as f:
        f.write(res.stderr)
    if verbose:
        sys.stderr.write(res.stderr)
    return lib


def build_native(force: bool = False) -> None:
    """Host-only differential checkers (libm ports, RNG) used by the CPU tests."""
    os.makedirs(NATIVE_BIN, exist_ok=True)
    cxx = os.environ.get("CXX", "g++")
    for name in ("libm_check", "rng_check"):
        src = os.path.join(NATIVE, name + ".cpp")
        out = os.path.join(NATIVE_BIN, name)
        deps = [src] + glob.glob(os.path.join(CSRC, "*.h"))
        if force or _stale(out, deps):
            subprocess.run([cxx, "-std=c++17", "-O2", "-ffp-contract=off", "-DLT_NO_CONTRACT", "-I" + CSRC,
                            src, "-o", out], check=True)
    # the same ports compiled for the device (sm_100a, --fmad=false), checked
    # against the host glibc on the GPU box (tests/test_gpu_robustness.py)
    src = os.path.join(NATIVE, "libm_device.cu")
    out = os.path.join(NATIVE_BIN, "libm_device")
    if force or _stale(out, [src] + glob.glob(os.path.join(CSRC, "*.h"))):
        subprocess.run([nvcc()] + NVCC_FLAGS[:-2] + ["-I" + CSRC, src, "-o", out, "-lpthread"], check=True)


def build_oracle() -> None:
    sys.path.insert(0, ROOT)
    from oracle import pyoracle  # test infrastructure: built here, never imported by the product

    pyoracle.build("all")


def build_all(force: bool = False) -> None:
    build_gpu(force)
    build_native(force)
    build_oracle()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built", LIB)
