"""TNSR / TUKR files (reference io.cpp:131-224) written and read by the B200
library's C-ABI, pinned against the compiled reference (CPU only: the shape
reader and the writers need no device)."""
import ctypes as C
import os

import numpy as np
import pytest

from oracles import Ref, random_tensor
from paper_2004_02583_b200 import _lib


@pytest.fixture(scope="module")
def ref():
    return Ref()


@pytest.fixture(scope="module")
def lib():
    return _lib.lib()


def test_tnsr_bytes_identical_to_reference(ref, lib, tmp_path):
    t = random_tensor(ref, [5, 4, 3, 2], 11)
    ours, theirs = str(tmp_path / "a.tnsr"), str(tmp_path / "b.tnsr")
    err = _lib.TkgError()
    flat = np.ascontiguousarray(t.reshape(-1, order="F"))
    assert lib.tkg_write_tnsr(os.fsencode(ours), 4, _lib.u64(t.shape),
                              flat.ctypes.data_as(C.POINTER(C.c_double)), C.byref(err)) == 0
    ref.write_tnsr(theirs, t)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    assert np.array_equal(ref.read_tnsr(ours), t)
    order, dims = C.c_int32(0), (C.c_uint64 * 16)()
    assert lib.tkg_read_tnsr_shape(os.fsencode(theirs), C.byref(order), dims, C.byref(err)) == 0
    assert [dims[k] for k in range(order.value)] == [5, 4, 3, 2]


def test_tukr_read_by_reference(ref, lib, tmp_path):
    dims, ranks = [6, 5, 4], [3, 2, 2]
    rng = np.random.default_rng(3)
    core = rng.standard_normal(ranks)
    factors = [rng.standard_normal((d, r)) for d, r in zip(dims, ranks)]
    path = str(tmp_path / "x.tukr")
    err = _lib.TkgError()
    c = np.ascontiguousarray(core.reshape(-1, order="F"))
    f = np.concatenate([u.reshape(-1, order="F") for u in factors])
    assert lib.tkg_write_tukr(os.fsencode(path), 3, _lib.u64(dims), _lib.u64(ranks),
                              c.ctypes.data_as(C.POINTER(C.c_double)), f.ctypes.data_as(C.POINTER(C.c_double)),
                              C.byref(err)) == 0
    rc, rf, rd = ref.read_tukr(path)
    assert rd == dims and np.array_equal(rc, core)
    for u, v in zip(rf, factors):
        assert np.array_equal(u, v)


def test_io_errors_match_reference(lib, tmp_path):
    # errors.hpp: IoError / FormatError are category io (return code 2), subtypes 8 / 9
    err = _lib.TkgError()
    order, dims = C.c_int32(0), (C.c_uint64 * 16)()
    missing = str(tmp_path / "none.tnsr")
    assert lib.tkg_read_tnsr_shape(os.fsencode(missing), C.byref(order), dims, C.byref(err)) == 2
    assert err.subtype == 8 and err.message.decode() == "cannot open for reading: " + missing
    bad = tmp_path / "bad.tnsr"
    bad.write_bytes(b"TNSX" + b"\0" * 20)
    assert lib.tkg_read_tnsr_shape(os.fsencode(str(bad)), C.byref(order), dims, C.byref(err)) == 2
    assert err.subtype == 9 and err.message.decode() == "TNSR: bad magic bytes"
    bad.write_bytes(b"TNSR" + (2).to_bytes(4, "little"))
    assert lib.tkg_read_tnsr_shape(os.fsencode(str(bad)), C.byref(order), dims, C.byref(err)) == 2
    assert err.message.decode() == "TNSR: unsupported version 2"
    bad.write_bytes(b"TNSR" + (1).to_bytes(4, "little") + (0).to_bytes(4, "little"))
    assert lib.tkg_read_tnsr_shape(os.fsencode(str(bad)), C.byref(order), dims, C.byref(err)) == 2
    assert err.message.decode() == "TNSR: implausible order 0"
    bad.write_bytes(b"TNSR" + (1).to_bytes(4, "little") + (2).to_bytes(4, "little") + (3).to_bytes(8, "little"))
    assert lib.tkg_read_tnsr_shape(os.fsencode(str(bad)), C.byref(order), dims, C.byref(err)) == 2
    assert err.message.decode().startswith("truncated file")


def test_cli_usage_errors_on_cpu(tmp_path):
    # tenkit_main.cpp:644-664: parse errors exit 1, io errors 2 (no device needed
    # for either: both fail before a context is created)
    import subprocess
    cli = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2004_02583_b200",
                       "tenkit_b200")
    if not os.path.exists(cli):
        pytest.skip("CLI not built")
    def run(*a):
        p = subprocess.run([cli, *a], capture_output=True, text=True, timeout=60)
        return p.returncode, p.stderr
    assert run()[0] == 1
    code, err = run("compress", "--in", "a.tnsr")
    assert code == 1 and "--out is required" in err
    code, err = run("compress", "--in", "a", "--out", "b", "--ranks", "2,x")
    assert code == 1 and "--ranks" in err
    code, err = run("compress", "--in", "a", "--out", "b", "--ranks", "2,2", "--method", "t-pca")
    assert code == 1 and "--method" in err
    code, err = run("compress", "--in", str(tmp_path / "none.tnsr"), "--out", "b", "--ranks", "2,2")
    assert code == 2 and "cannot open for reading" in err
