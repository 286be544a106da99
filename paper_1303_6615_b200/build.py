"""Build librsw.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "librsw.so")
SOURCES = ["rsw_pipe_256.cu", "rsw_pipe_128.cu", "rsw_pipe_64.cu", "rsw_k_coarse.cu", "rsw_k_fine.cu", "rsw_k_misc.cu",
           "rsw_pipeline.cu", "rsw_capi.cu"]
HEADERS = ["rsw_device.cuh", "rsw_internal.h", "rsw_blocks.cuh", "rsw_pipeline.cuh"]


def _host_cxx() -> str:
    # /usr/bin/g++ is the image's complete toolchain (the /opt/gcc wrapper lacks libgomp specs)
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else (shutil.which("g++") or "g++")


def _nvcc() -> str:
    return shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"


def compile_cmd(src: str, obj: str) -> list[str]:
    return [
        _nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
        "-Xcompiler", "-fPIC", "-ccbin", _host_cxx(), f"-I{INCLUDE}", "-c", src, "-o", obj,
    ]


def link_cmd(objs: list[str], out: str) -> list[str]:
    return [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-ccbin", _host_cxx(),
            *objs, "-o", out, "-ldl", "-lpthread"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(INCLUDE, "rsw.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Each translation unit compiles in its own nvcc process (in parallel), then one shared link."""
    if force or stale():
        objdir = os.path.join(HERE, "build")
        os.makedirs(objdir, exist_ok=True)
        jobs, objs = [], []
        hdr_t = max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS)
        hdr_t = max(hdr_t, os.path.getmtime(os.path.join(INCLUDE, "rsw.h")))
        for src in SOURCES:
            obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
            objs.append(obj)
            srcp = os.path.join(CSRC, src)
            if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(hdr_t, os.path.getmtime(srcp)):
                continue  # object newer than its source and every shared header
            cmd = compile_cmd(srcp, obj)
            if verbose:
                print(" ".join(cmd))
            jobs.append((subprocess.Popen(cmd), cmd, obj))
        for proc, cmd, _ in jobs:
            if proc.wait() != 0:
                raise subprocess.CalledProcessError(proc.returncode, cmd)
        cmd = link_cmd(objs, LIB + ".tmp")
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
