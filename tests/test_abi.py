"""The C-ABI boundary (include/tenkit_b200.h) on CPU: the in-tree library
loads, exports every declared symbol, and fails loudly without a GPU (no
CPU fallback)."""
import ctypes as C
import os
import re

import pytest

import paper_2004_02583_b200 as tk
from paper_2004_02583_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tenkit_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(tkg_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["tkg_t_hosvd", "tkg_st_hosvd", "tkg_als_low_rank", "tkg_als_init", "tkg_select_order",
              "tkg_unfold_times", "tkg_unfold_t_times", "tkg_mode_n_product", "tkg_frobenius_norm",
              "tkg_relative_error", "tkg_reduced_qr", "tkg_gram", "tkg_create", "tkg_destroy"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_lib.ensure_built())
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding covers them all
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(declared_symbols()) <= bound


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(tk.DeviceError):
        tk.Context(0)


def test_select_order_is_host_logic():
    # hosvd.cpp:54-63 (no device needed)
    assert tk.select_order(tk.Truncation([64, 64, 32]), [2048, 2048, 512]).order == [3, 1, 2]
    assert tk.select_order(tk.Truncation([10, 5, 20]), [30, 30, 30]).order == [2, 1, 3]
    with pytest.raises(tk.RankTooLargeError):
        tk.select_order(tk.Truncation([10, 40, 20]), [30, 30, 30])
    with pytest.raises(tk.DimensionMismatchError):
        tk.select_order(tk.Truncation([10, 4]), [30, 30, 30])


def test_kernels_are_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", _lib.ensure_built()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _build_shim(tmp_path, with_tenkit):
    import shutil
    import subprocess
    gxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else shutil.which("g++")
    lib_dir = os.path.dirname(_lib.ensure_built())
    out = str(tmp_path / ("shim_tenkit" if with_tenkit else "shim_plain"))
    cmd = [gxx, "-std=c++20", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tools", "shim_example.cpp"), "-o", out, "-L" + lib_dir,
           "-ltenkit_b200", "-Wl,-rpath," + lib_dir]
    if with_tenkit:
        ref_inc = "/root/reference/proj/include"
        ref_so = os.path.join(ROOT, "oracle", "_ref", "libtenkit_ref.so")
        if not (os.path.isdir(ref_inc) and os.path.exists(ref_so)):
            pytest.skip("reference headers not present")
        cmd[2:2] = ["-DTENKIT_B200_USE_TENKIT", "-I" + ref_inc]
        cmd += [ref_so, "-Wl,-rpath," + os.path.dirname(ref_so)]
    subprocess.check_call(cmd)
    return out


@pytest.mark.parametrize("with_tenkit", [False, True])
def test_cpp_shim_compiles_and_fails_loudly_on_cpu(tmp_path, with_tenkit):
    import subprocess
    import torch
    exe = _build_shim(tmp_path, with_tenkit)
    r = subprocess.run([exe], capture_output=True, text=True)
    if torch.cuda.is_available():
        assert r.returncode == 0, r.stdout + r.stderr
    else:
        assert r.returncode == 2 and "no CUDA device" in r.stdout
