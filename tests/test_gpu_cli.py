"""The `tenkit_b200 compress` CLI (csrc/cli.cpp, the reference's
tenkit_main.cpp:183-266 over the C-ABI) and the device TNSR loader on the
B200, against the compiled reference: the pinned CSV record
(test_cli.cpp:137-163), TUKR output read back by the reference, exit codes."""
import os
import subprocess

import numpy as np
import pytest

import paper_2004_02583_b200 as tk
from oracles import Ref
from parity import principal_sine

pytestmark = pytest.mark.gpu

CLI = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2004_02583_b200",
                   "tenkit_b200")
HEADER = "method,dims,ranks,order,eta,seed,threads,rel_residual,seconds,iters_per_mode"


@pytest.fixture(scope="module")
def ref():
    r = Ref()
    r.set_threads(r.max_threads())
    return r


def run(*args):
    p = subprocess.run([CLI, "compress", *args], capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


def split_csv(line):
    out, cur, quoted = [], "", False
    for ch in line:
        if ch == '"':
            quoted = not quoted
        elif ch == "," and not quoted:
            out.append(cur)
            cur = ""
        else:
            cur += ch
    out.append(cur)
    return out


def reconstruct_rel(ref, t, path):
    core, factors, dims = ref.read_tukr(path)
    rec = ref.reconstruct(core, factors, dims)
    return ref.relative_error(t, rec)


def test_compress_pinned_record(ref, tmp_path):
    t = tk.synth_tucker([12, 10, 8], [3, 2, 4], 0.0, 0.0, 41).reshape((12, 10, 8), order="F")
    src, out = str(tmp_path / "exact.tnsr"), str(tmp_path / "exact.tukr")
    ref.write_tnsr(src, t)
    code, so, se = run("--in", src, "--out", out, "--ranks", "3,2,4", "--method", "st-als", "--eta", "1e-4",
                       "--seed", "2", "--header")
    assert code == 0, se
    lines = so.strip().splitlines()
    assert len(lines) == 2 and lines[0] == HEADER
    f = split_csv(lines[1])
    assert len(f) == 10
    assert f[:6] == ["st-als", "12x10x8", "3x2x4", "2,1,3", "0.0001", "2"]
    assert float(f[7]) <= 1e-8 and float(f[8]) >= 0.0 and f[9] != ""
    assert reconstruct_rel(ref, t, out) <= 1e-8


@pytest.mark.parametrize("method", ["t-als", "st-als", "t-eig", "st-svd"])
def test_compress_matches_reference(ref, tmp_path, method):
    dims, ranks = [40, 30, 20], [5, 4, 3]
    t = tk.synth_tucker(dims, ranks, 0.0, 1e-3, 42).reshape(dims, order="F")
    src, out = str(tmp_path / "a.tnsr"), str(tmp_path / "a.tukr")
    ref.write_tnsr(src, t)
    code, so, se = run("--in", src, "--out", out, "--ranks", "5,4,3", "--method", method, "--eta", "1e-8",
                       "--seed", "7")
    assert code == 0, se
    f = split_csv(so.strip())
    seq = method.startswith("st-")
    kind = method.split("-")[1]
    if kind == "als":
        r = ref.hosvd_als(t, ranks, sequential=seq, eta=1e-8, seed=7)
        assert f[9] == ",".join(str(m.iterations) for m in r.per_mode)
    else:
        r = ref.hosvd_exact(t, ranks, kind, sequential=seq)
        assert f[9] == ""
    assert f[3] == ",".join(str(m.mode) for m in r.per_mode)
    assert abs(float(f[7]) - r.relative_residual) <= 1e-10
    core, factors, _ = ref.read_tukr(out)
    for u, v in zip(factors, r.factors):
        assert principal_sine(u, v) <= 1e-8


def test_compress_explicit_order_and_hooi(ref, tmp_path):
    dims, ranks = [30, 30, 30], [5, 5, 5]
    t = tk.synth_tucker(dims, ranks, 0.0, 1e-3, 801).reshape(dims, order="F")
    src = str(tmp_path / "h.tnsr")
    ref.write_tnsr(src, t)
    code, so, _ = run("--in", src, "--out", str(tmp_path / "o.tukr"), "--ranks", "5,5,5", "--method", "st-svd",
                      "--order", "3,1,2")
    assert code == 0 and split_csv(so.strip())[3] == "3,1,2"
    code, so, se = run("--in", src, "--out", str(tmp_path / "h.tukr"), "--ranks", "5,5,5", "--method", "hooi",
                       "--init", "st-svd")
    assert code == 0, se
    f = split_csv(so.strip())
    warm = ref.hosvd_exact(t, ranks, "svd", sequential=True)
    _, _, iters, _, fits = ref.hooi(t, ranks, warm.core, warm.factors)
    assert f[0] == "hooi" and f[3] == "" and f[9] == str(iters)
    assert abs(float(f[7]) - (1.0 - fits[-1])) <= 1e-10


def test_compress_exit_codes(tmp_path):
    code, _, se = run("--in", str(tmp_path / "missing.tnsr"), "--out", str(tmp_path / "x.tukr"), "--ranks", "2,2")
    assert code == 2 and "cannot open for reading" in se
    code, _, _ = run("--in", "x", "--out", "y", "--ranks", "2,2", "--method", "t-foo")
    assert code == 1
    t = np.ones((4, 5, 6), order="F")
    src = str(tmp_path / "ones.tnsr")
    Ref().write_tnsr(src, t)
    code, _, se = run("--in", src, "--out", str(tmp_path / "x.tukr"), "--ranks", "9,2,2", "--method", "t-als")
    assert code != 0 and "rank 9" in se


def test_read_tnsr_to_device(ref, tmp_path):
    dims, ranks = [64, 48, 40], [6, 5, 4]
    t = tk.synth_tucker(dims, ranks, 0.0, 1e-3, 5).reshape(dims, order="F")
    src = str(tmp_path / "d.tnsr")
    ref.write_tnsr(src, t)
    ctx = tk.Context(0)
    assert np.array_equal(ctx.read_tnsr(src, device=False), t)
    dt = ctx.read_tnsr(src)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-8, seed=7))
    a, ra = ctx.t_hosvd(dt, tk.Truncation(ranks), eng)
    b, rb = ctx.t_hosvd(t, tk.Truncation(ranks), eng)
    assert np.array_equal(a.core, b.core) and ra.relative_residual == rb.relative_residual
    out = str(tmp_path / "d.tukr")
    ctx.write_tukr(out, a)
    core, factors, d = ref.read_tukr(out)
    assert d == dims and np.array_equal(core, a.core)


def test_cpp_shim_with_reference_types_runs_on_device():
    # tools/shim_example.cpp built by build() against the reference's headers:
    # tenkit::DenseTensor in, tenkit::TuckerTensor / DecompositionReport /
    # HooiResult / FactorPair out, through the B200 library
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "shim_tenkit")
    if not os.path.exists(exe):
        pytest.skip("shim example not built (needs the reference headers at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "rel err" in p.stdout
