"""In-tree build of the native libraries (no JIT cache: the built .so files
travel to the GPU box with the repo snapshot).

* ``lib/libtsgm_b200.so``  — the product: sm_100a CUDA kernels + host runtime
  behind the C-ABI declared in ``include/tsgm_b200.h``.
* ``lib/libtsgm_scene.so`` — synthetic input generator (host C).
"""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

# FP64 state kernels must not contract a*b+c into FMA: the reference build has
# no FMA (x86-64 baseline, no -march), and bit-exact KF state needs the same
# rounding sequence. Integer kernels are unaffected by the flag.
CUDA_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr",
              f"-I{INCLUDE}", f"-I{CSRC}"]

CU_SOURCES = ["stereo_kernels.cu", "temporal_kernels.cu", "aggregate_kernels.cu",
              "aggregate_sweep.cu", "detect.cu", "noise.cu", "export.cu", "runtime.cu"]


def lib_path(name: str) -> str:
    return os.path.join(LIB, name)


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers() -> list[str]:
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh", ".hpp"))]
    hs += [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)]
    return hs


def build_scene(force: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    out = lib_path("libtsgm_scene.so")
    src = os.path.join(CSRC, "scene.c")
    if force or _stale(out, [src, os.path.join(INCLUDE, "tsgm_scene.h")]):
        subprocess.run(["gcc", "-std=gnu11", "-O2", "-fPIC", "-shared", "-pthread", "-o", out,
                        src, "-lm"], check=True)
    return out


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    obj_dir = os.path.join(LIB, "obj")
    os.makedirs(obj_dir, exist_ok=True)
    out = lib_path("libtsgm_b200.so")
    hdrs = _headers()
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(obj_dir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s, *hdrs, __file__]):
            cmd = [NVCC, *ARCH, *CUDA_FLAGS, "-c", s, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            subprocess.run(cmd, check=True)
    if force or _stale(out, objs):
        subprocess.run([NVCC, *ARCH, "-shared", "-o", out, *objs, "-lcudart", "-lz"], check=True)
    return out


def build_render_tool(force: bool = False) -> str:
    """tools/bin/render_frames: the scene generator as a plain C program, so
    the reference arm of bench.py gets its frames from a separate process that
    is not Python and maps no product library."""
    out = os.path.join(ROOT, "tools", "bin", "render_frames")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    srcs = [os.path.join(ROOT, "tools", "render_frames.c"), os.path.join(CSRC, "scene.c")]
    if force or _stale(out, [*srcs, os.path.join(INCLUDE, "tsgm_scene.h")]):
        subprocess.run(["gcc", "-std=gnu11", "-O2", "-pthread", f"-I{INCLUDE}", "-o", out, *srcs,
                        "-lm"], check=True)
    return out


def build_all(force: bool = False) -> None:
    build_scene(force)
    build_render_tool(force)
    build_cuda(force)
