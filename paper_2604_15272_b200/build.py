"""Build libsgm.so in-tree (host C++ + embedded device headers for NVRTC).

The CUDA kernels are generated per candidate and compiled for sm_100a by NVRTC
at plan-creation time (persistent cubin cache next to libsgm.so).  `build()`
also nvcc-compiles the utility module and a sample generated kernel for
sm_100a so the toolchain path is checked on a CPU-only machine.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
LIB = os.path.join(HERE, "libsgm.so")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _embed(src: str, dst: str) -> None:
    text = open(os.path.join(CSRC, src), encoding="utf-8").read()
    assert ")SGMRAW\"" not in text
    body = 'R"SGMRAW(' + text + ')SGMRAW"\n'
    path = os.path.join(CSRC, dst)
    if not os.path.exists(path) or open(path, encoding="utf-8").read() != body:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(body)


def _run(cmd: list[str]) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("command failed: " + " ".join(cmd))


def build_lib(force: bool = False) -> str:
    _embed("sgm_dev.cuh", "sgm_dev_embed.inc")
    _embed("sgm_util.cuh", "sgm_util_embed.inc")
    srcs = [os.path.join(CSRC, f) for f in ("sgm_runtime.cpp", "sgm_codegen.cpp")]
    deps = srcs + [os.path.join(CSRC, f) for f in (
        "sgm_codegen.h", "sgm_dev.cuh", "sgm_util.cuh", "sgm_dev_embed.inc", "sgm_util_embed.inc")]
    deps.append(os.path.join(ROOT, "include", "sgm.h"))
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= t for d in deps):
            return LIB
    cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-Wno-unused-function",
           f"-I{CUDA}/include", *srcs, "-o", LIB + ".tmp",
           f"-L{CUDA}/lib64", "-lnvrtc", "-ldl", "-lpthread", f"-Wl,-rpath,{CUDA}/lib64"]
    _run(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def nvcc_check(out_dir: str | None = None) -> str:
    """nvcc-compile the utility module for sm_100a (-lineinfo) as a toolchain check."""
    out_dir = out_dir or os.path.join(HERE, "build")
    os.makedirs(out_dir, exist_ok=True)
    src = os.path.join(out_dir, "sgm_util_check.cu")
    with open(src, "w") as fh:
        fh.write('#include "sgm_util.cuh"\n')
    cubin = os.path.join(out_dir, "sgm_util.cubin")
    _run([f"{CUDA}/bin/nvcc", *GENCODE, "-lineinfo", "-O3", "-std=c++17", "-cubin",
          f"-I{CSRC}", src, "-o", cubin])
    return cubin


REF_SRC = "/root/reference/pkg"
REF_DST = os.path.join(ROOT, "baseline", "_ref")


def install_reference(force: bool = False) -> str | None:
    """Install the UNMODIFIED reference package (symfuse, incl. its compiled Cython
    e-graph core) into baseline/_ref, offline, from a /tmp copy of /root/reference/pkg
    (the mount is read-only and the build writes into the source tree).  `--no-deps`:
    numpy is importable but not in the wheelhouse.  baseline/_ref is git-ignored but
    travels to the GPU box with the snapshot; on the box /root/reference is absent,
    so an existing install is kept and nothing is attempted."""
    if not force and os.path.isdir(os.path.join(REF_DST, "symfuse")):
        return REF_DST
    if not os.path.isdir(REF_SRC):
        return None
    import shutil
    import tempfile
    tmp = tempfile.mkdtemp(prefix="symfuse_src_")
    try:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_SRC, src, ignore=shutil.ignore_patterns("__pycache__", "*.so", "build"))
        _run([sys.executable, "-m", "pip", "install", "-q", "--no-index", "--no-build-isolation", "--no-deps",
              "--find-links", "/opt/wheelhouse", "--upgrade", "--target", REF_DST, src])
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    return REF_DST


if __name__ == "__main__":
    print(build_lib(force="--force" in sys.argv))
    print(nvcc_check())
    print(install_reference())
