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
    """libloratwin_gpu.so from csrc/*.cu: every translation unit (the host /
    C-ABI code in capi.cu and one engine build per engine_*.cu) compiled in
    parallel, then linked. prof=True builds libloratwin_gpu_prof.so with the
    per-phase cycle counters (-DLT_PHASE_PROF) used by tools/diag_phase.py,
    stats=True libloratwin_gpu_stats.so with scan counters (-DLT_SCAN_STATS)."""
    tag = "_prof" if prof else ("_stats" if stats else "")
    lib = LIB.replace(".so", tag + ".so")
    deps = glob.glob(os.path.join(CSRC, "*")) + [os.path.join(INCLUDE, "loratwin_gpu.h")]
    if not force and not _stale(lib, deps):
        return lib
    objdir = os.path.join(os.path.dirname(lib), "obj" + tag)
    os.makedirs(objdir, exist_ok=True)
    extra = (["-DLT_PHASE_PROF"] if prof else []) + (["-DLT_SCAN_STATS"] if stats else [])
    units = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    procs = []
    for u in units:
        obj = os.path.join(objdir, os.path.basename(u).replace(".cu", ".o"))
        cmd = [nvcc()] + NVCC_FLAGS + extra + ["-I" + INCLUDE, "-I" + CSRC, "-c", "-o", obj, u]
        procs.append((u, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    log = []
    failed = False
    for u, obj, p in procs:
        out, err = p.communicate()
        log.append(f"== {os.path.basename(u)}\n{out}{err}")
        if p.returncode != 0:
            failed = True
            sys.stderr.write(out + err)
    if failed:
        raise RuntimeError("nvcc failed building libloratwin_gpu.so")
    res = subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib]
                         + [obj for _, obj, _ in procs], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libloratwin_gpu.so")
    with open(os.path.join(os.path.dirname(lib), "ptxas" + tag + ".log"), "w") as f:
        f.write("\n".join(log))
    if verbose:
        sys.stderr.write("\n".join(log))
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
