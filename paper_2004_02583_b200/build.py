"""Build the in-tree shared libraries with nvcc / g++ (no torch, no JIT cache).

  paper_2004_02583_b200/libtenkit_b200.so   the product: CUDA kernels for
      sm_100a (-gencode arch=compute_100a,code=sm_100a) + the C++ engine +
      the extern "C" ABI of include/tenkit_b200.h.
  paper_2004_02583_b200/libtkg_synth.so     input synthesis for benches/tests
      (host C++/OpenMP; not on the decomposition path).

Each object is rebuilt only when its source, a header or this file is newer than it.
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
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libtenkit_b200.so")
SYNTH = os.path.join(PKG, "libtkg_synth.so")
CLI = os.path.join(PKG, "tenkit_b200")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
GXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else (shutil.which("g++") or "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SRCS = ["contract.cu", "contract_tma.cu", "smallla.cu", "mtrng.cu", "recon.cu", "als_step.cu", "coop.cu",
           "gram.cu", "wide.cu", "eig.cu", "sweep_fused.cu"]
CPP_SRCS = ["engine.cpp", "engine_wide.cpp", "engine_dist.cpp", "comm.cpp", "mt_jump.cpp", "capi.cpp", "io.cpp"]  # cli.cpp: the executable


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths if os.path.exists(p)), default=0.0)


def _deps():
    return (glob.glob(os.path.join(CSRC, "*")) + [os.path.join(ROOT, "include", "tenkit_b200.h"),
                                                   os.path.abspath(__file__)])


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} {cmd[-1]}")
    return r


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    deps = _deps()
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest(deps):
        if not os.path.exists(CLI) or os.path.getmtime(CLI) < os.path.getmtime(LIB):
            build_cli()
        build_synth(force=False)
        return LIB
    cmds, objs = [], []
    # an object is rebuilt when its source, any header or this file is newer
    hdrs = _newest([d for d in deps if not d.endswith((".cu", ".cpp"))])

    def stale(src, obj):
        return force or not os.path.exists(obj) or os.path.getmtime(obj) < max(hdrs, os.path.getmtime(os.path.join(CSRC, src)))

    for src in CU_SRCS:
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if not stale(src, obj):
            continue
        cmds.append([NVCC, *ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-v" if verbose else "-O3", "-c", os.path.join(CSRC, src), "-o", obj])
    for src in CPP_SRCS:
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if not stale(src, obj):
            continue
        cmds.append([GXX, "-O2", "-std=c++17", "-fPIC", "-mpclmul", "-msse4.1", "-Wall",
                     "-I/usr/local/cuda/include", "-c", os.path.join(CSRC, src), "-o", obj])
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, len(cmds))) as ex:
        for r in ex.map(_run, cmds):
            if verbose:
                sys.stderr.write(r.stderr)
    tmp = LIB + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-lpthread", "-ldl"])
    os.replace(tmp, LIB)
    build_cli()
    build_synth(force=True)
    return LIB


def build_cli() -> str:
    """tenkit_b200 (csrc/cli.cpp): the reference CLI's `compress` over the C-ABI."""
    tmp = CLI + ".tmp"
    _run([GXX, "-O2", "-std=c++17", "-Wall", "-o", tmp, os.path.join(CSRC, "cli.cpp"), f"-L{PKG}", "-ltenkit_b200",
          "-Wl,-rpath,$ORIGIN"])
    os.replace(tmp, CLI)
    return CLI


def build_synth(force: bool = False) -> str:
    src = os.path.join(CSRC, "synth.cpp")
    if not os.path.exists(src):
        return ""
    if not force and os.path.exists(SYNTH) and os.path.getmtime(SYNTH) >= os.path.getmtime(src):
        return SYNTH
    tmp = SYNTH + ".tmp"
    _run([GXX, "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-mavx2", "-mfma", "-shared", "-o", tmp,
          src])
    os.replace(tmp, SYNTH)
    return SYNTH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
