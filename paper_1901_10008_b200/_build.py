"""In-tree build of the two native libraries.

  lib/libgmx_core.so   C++ decision core      (g++, -ffp-contract=off: bit-exact doubles)
  lib/libgmx_exec.so   sm_100a CUDA executor  (nvcc -gencode arch=compute_100a,code=sm_100a)

Both are built in-tree so they travel to the GPU box with the repo snapshot.
A library is rebuilt when any of its sources is newer than the .so.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
LIB_DIR = os.path.join(PKG, "lib")
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(REPO, "include")

CORE_SO = os.path.join(LIB_DIR, "libgmx_core.so")
EXEC_SO = os.path.join(LIB_DIR, "libgmx_exec.so")

NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources(sub, exts):
    out = []
    for ext in exts:
        out += glob.glob(os.path.join(CSRC, sub, "*" + ext))
    return sorted(out)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + proc.stdout + proc.stderr)
    return proc.stdout + proc.stderr


def build_core(force=False):
    srcs = _sources("core", (".cpp",))
    deps = srcs + _sources("core", (".hpp",)) + [os.path.join(INCLUDE, "gmx_core.h")]
    if not force and not _stale(CORE_SO, deps):
        return CORE_SO
    os.makedirs(LIB_DIR, exist_ok=True)
    tmp = CORE_SO + ".tmp"
    _run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
          "-fno-fast-math", "-Wall", "-Wextra", "-Wno-unused-parameter",
          "-Wl,-soname,libgmx_core.so", "-I", INCLUDE, *srcs, "-o", tmp])
    os.replace(tmp, CORE_SO)
    return CORE_SO


def nvcc_path():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA executor cannot be built")


def build_exec(force=False, verbose_ptxas=False):
    srcs = _sources("exec", (".cu",)) + _sources("exec", (".cpp",))
    core = build_core()
    deps = srcs + _sources("exec", (".cuh", ".hpp", ".h")) + [
        os.path.join(INCLUDE, h) for h in ("gmx_exec.h", "gmx_runtime.h", "gmx_core.h")] + [core]
    if not force and not _stale(EXEC_SO, deps):
        return EXEC_SO
    os.makedirs(LIB_DIR, exist_ok=True)
    tmp = EXEC_SO + ".tmp"
    cmd = [nvcc_path(), *NVCC_ARCH, "-O3", "-std=c++17", "-lineinfo", "-shared",
           "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
           "--expt-relaxed-constexpr", "-cudart", "static",
           "-I", INCLUDE, *srcs, "-o", tmp, "-L", LIB_DIR, "-lgmx_core",
           "-Xlinker", "-rpath,$ORIGIN", "-ldl"]
    if verbose_ptxas:
        cmd.insert(1, "-Xptxas=-v")
    log = _run(cmd)
    os.replace(tmp, EXEC_SO)
    return EXEC_SO if not verbose_ptxas else log


def build_all(force=False):
    return [build_core(force), build_exec(force)]
