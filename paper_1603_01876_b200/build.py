"""In-tree build of the native libraries (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

  lib/libprg.so                 CUDA kernels + the C-ABI of include/prg.h
  python/prpipe/_core*.so       pybind11 module mirroring the reference's
                                prpipe._core (bindings/module.cpp) over the C-ABI

Usage: python -m paper_1603_01876_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "lib", "libprg.so")
PYMOD_DIR = os.path.join(PKG, "python", "prpipe")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# host code: x86-64-v2 (SSE4.2/POPCNT, every x86 server since ~2009) for the host-side value pass
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "-Xcompiler", "-march=x86-64-v2",
              "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"] + ARCH
CU_SOURCES = ["prg_runtime.cu", "prg_sort.cu", "prg_k0.cu", "prg_k1.cu", "prg_k2.cu", "prg_k3.cu",
              "prg_k2_steps.cu", "prg_capi.cu"]
HEADERS = ["prg_common.cuh", "prg_internal.cuh", "prg_sort.cuh"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} ... {cmd[-1]}")
    if "spill" in r.stderr and "0 bytes spill" not in r.stderr:
        sys.stderr.write(r.stderr)


# Checked variant (device-side bounds / invariant checks, PRG_DCHECK in the
# sources): test infrastructure for tests/test_checked.py, never loaded by the
# product path unless PRG_LIB points at it.
LIB_CHECKED = os.path.join(ROOT, "build", "libprg_checked.so")


def build_libprg(force: bool = False, checked: bool = False) -> str:
    lib = LIB_CHECKED if checked else LIB
    objdir = os.path.join(ROOT, "build", "obj_checked") if checked else BUILD
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "prg.h")]
    flags = NVCC_FLAGS + (["-DPRG_CHECKED=1"] if checked else [])
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            jobs.append([NVCC] + flags + ["-c", s, "-o", o])
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(_run, jobs))
    if force or jobs or _newer(lib, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-lcudart"])
    return lib


def build_core(force: bool = False) -> str | None:
    """pybind11 prpipe._core over libprg (C++ shim in host/)."""
    srcs = sorted(os.path.join(HOST, f) for f in os.listdir(HOST) if f.endswith(".cpp")) if os.path.isdir(HOST) else []
    if not srcs:
        return None
    import pybind11

    ext = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
    out = os.path.join(PYMOD_DIR, "_core" + ext)
    hdrs = [os.path.join(HOST, "prpipe", f) for f in os.listdir(os.path.join(HOST, "prpipe"))] + [
        os.path.join(ROOT, "include", "prg.h")]
    if not (force or _newer(out, srcs + hdrs + [LIB])):
        return out
    py_inc = sysconfig.get_paths()["include"]
    json_dir = _json_include()
    objdir = os.path.join(ROOT, "build", "host")
    os.makedirs(objdir, exist_ok=True)
    base = ["g++", "-std=c++20", "-O2", "-fPIC", "-fvisibility=hidden", "-I", os.path.join(ROOT, "include"),
            "-I", HOST, "-I", pybind11.get_include(), "-I", py_inc, "-I", json_dir]
    objs, jobs = [], []
    for src in srcs:
        o = os.path.join(objdir, os.path.basename(src).replace(".cpp", ".o"))
        objs.append(o)
        if force or _newer(o, [src] + hdrs):
            jobs.append(base + ["-c", src, "-o", o])
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(_run, jobs))
    _run(["g++", "-shared", *objs, "-o", out, "-L", os.path.dirname(LIB), "-lprg",
          "-Wl,-rpath,$ORIGIN/../../lib", "-lpthread"])
    return out


def _json_include() -> str:
    """nlohmann/json.hpp (v3.11.3, vendored in the image's cudnn_frontend) for the manifest."""
    import glob
    import site

    for sp in site.getsitepackages():
        for d in glob.glob(os.path.join(sp, "include", "cudnn_frontend", "thirdparty", "nlohmann")):
            return d
    raise RuntimeError("nlohmann/json.hpp not found")


def build(force: bool = False) -> None:
    build_libprg(force)
    build_core(force)
    build_libprg(force, checked=True)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print("built", LIB)
