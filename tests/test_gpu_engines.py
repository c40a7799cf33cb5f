"""The SVD and EIG factor engines (FactorEngine::Kind kSvd / kEig,
hosvd.hpp:19-27; hosvd.cpp:89-99, 151-171) and their primitives mode_gram
(tensor_ops.cpp:332-389) and sym_eig (kernels.cpp:448-604) on the B200,
against the compiled reference (oracle/_ref). SURVEY §8(f) row 3.

Exact engines determine every factor column (descending order,
fix_column_signs, kernels.cpp:25-43), so factors are compared column by
column and the core entrywise."""
import numpy as np
import pytest

import paper_2004_02583_b200 as tk
from oracles import Ref, random_matrix, random_tensor
from parity import CORE_SV_REL_TOL, REL_ERR_ABS_TOL, column_diff, ortho_defect, principal_sine

pytestmark = pytest.mark.gpu

SHAPES = [[7], [6, 8], [3, 4, 5], [4, 3, 2, 5], [40, 30, 20], [300, 9, 5], [5, 3, 700], [64, 33, 17],
          [130, 70, 3], [17, 4, 6, 5], [200, 6, 4]]


@pytest.fixture(scope="module")
def ctx():
    return tk.Context(0)


@pytest.fixture(scope="module")
def ref():
    r = Ref()
    r.set_threads(r.max_threads())
    return r


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("dims", SHAPES, ids=lambda d: "x".join(map(str, d)))
def test_mode_gram_matches_reference(ctx, ref, dims):
    t = random_tensor(ref, dims, 71 + len(dims))
    for mode in range(1, len(dims) + 1):
        g = ctx.mode_gram(t, mode)
        assert np.array_equal(g, g.T)
        assert rel(g, ref.mode_gram(t, mode)) <= 1e-13


@pytest.mark.parametrize("n,k", [(5, 2), (40, 10), (96, 96), (257, 32), (1024, 64)])
def test_sym_eig_matches_reference(ctx, ref, n, k):
    # well-separated spectrum: Q diag(d) Q^T
    q = np.linalg.qr(random_matrix(ref, n, n, 500 + n))[0]
    d = np.linspace(1.0, 2.0 * n, n)[::-1]
    g = np.asfortranarray((q * d) @ q.T)
    g = 0.5 * (g + g.T)
    vals, vecs = ctx.sym_eig(g, k)
    rv, ru = ref.sym_eig(g, k)
    assert np.max(np.abs(vals - rv)) <= 1e-12 * np.max(np.abs(rv))
    assert column_diff(vecs, ru) <= 1e-10
    assert ortho_defect(vecs) <= 1e-13 * max(1, k)


def test_sym_eig_errors(ctx):
    with pytest.raises(tk.DimensionMismatchError):
        ctx.sym_eig(np.eye(3), 4)


@pytest.mark.parametrize("kind", ["svd", "eig"])
@pytest.mark.parametrize("sequential,order", [(False, None), (True, None), (True, [3, 1, 2])])
@pytest.mark.parametrize("dims,ranks,alpha", [([40, 30, 20], [5, 4, 3], 0.0), ([96, 80, 72], [10, 12, 8], 1.0),
                                              ([24, 20, 16, 12], [4, 3, 5, 2], 0.0)], ids=str)
def test_exact_engines_match_reference(ctx, ref, kind, sequential, order, dims, ranks, alpha):
    if order is not None and len(dims) != 3:
        pytest.skip("order given for 3-way tensors")
    a = tk.synth_tucker(dims, ranks, alpha, 1e-3, 2004).reshape(dims, order="F")
    eng = tk.FactorEngine.svd() if kind == "svd" else tk.FactorEngine.eig()
    if sequential:
        tkr, rep = ctx.st_hosvd(a, tk.Truncation(ranks), tk.ModeOrder(order) if order else None, eng)
    else:
        tkr, rep = ctx.t_hosvd(a, tk.Truncation(ranks), eng)
    r = ref.hosvd_exact(a, ranks, kind, sequential=sequential, order=order)
    assert [m.mode for m in rep.per_mode] == [m.mode for m in r.per_mode]
    assert all(m.als is None for m in rep.per_mode)
    assert abs(rep.relative_residual - r.relative_residual) <= REL_ERR_ABS_TOL
    for u, v in zip(tkr.factors, r.factors):
        assert column_diff(u, v) <= 1e-8
        assert ortho_defect(u) <= 1e-12
    assert np.max(np.abs(tkr.core - r.core)) <= CORE_SV_REL_TOL * np.max(np.abs(r.core))


@pytest.mark.parametrize("sequential", [False, True])
def test_svd_engine_steep_spectrum(ctx, ref, sequential):
    # core spectra sigma_k ~ k^-2.5 (sigma_16 / sigma_1 = 1e-3), no noise: the
    # Gram route alone squares the condition number (errors ~eps s1^2 / (si^2 -
    # sj^2)); the SVD engine's refinement round keeps dense_svd's accuracy
    # (hosvd.cpp:89-92)
    dims, ranks = [96, 80, 72], [16, 12, 10]
    a = tk.synth_tucker(dims, ranks, 2.5, 0.0, 2025).reshape(dims, order="F")
    if sequential:
        tkr, rep = ctx.st_hosvd(a, tk.Truncation(ranks), None, tk.FactorEngine.svd())
    else:
        tkr, rep = ctx.t_hosvd(a, tk.Truncation(ranks), tk.FactorEngine.svd())
    r = ref.hosvd_exact(a, ranks, "svd", sequential=sequential)
    for u, v in zip(tkr.factors, r.factors):
        assert column_diff(u, v) <= 1e-10
    assert np.max(np.abs(tkr.core - r.core)) <= CORE_SV_REL_TOL * np.max(np.abs(r.core))


def test_engines_agree_and_als_lands_nearby(ctx):
    # test_hosvd.cpp "exact engines agree; ALS lands nearby"
    dims, ranks = [60, 50, 40], [6, 5, 4]
    a = tk.synth_tucker(dims, ranks, 0.0, 1e-3, 613).reshape(dims, order="F")
    ts, rs = ctx.t_hosvd(a, tk.Truncation(ranks), tk.FactorEngine.svd())
    te, re_ = ctx.t_hosvd(a, tk.Truncation(ranks), tk.FactorEngine.eig())
    ta, ra = ctx.t_hosvd(a, tk.Truncation(ranks), tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-10, seed=7)))
    for u, v, w in zip(ts.factors, te.factors, ta.factors):
        assert column_diff(u, v) <= 1e-12
        assert principal_sine(w, u) <= 1e-6
    # rel err 1e-3 takes the closed form ||A||^2 - ||G||^2 (Engine::closed_form_residual):
    # the two engines' cores differ in the last bits, so their residuals agree to
    # ~1e-13, inside the 1e-10 parity bar
    assert abs(rs.relative_residual - re_.relative_residual) <= 1e-11
    assert abs(ra.relative_residual - rs.relative_residual) <= 1e-8


_NO_CUSOLVER = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2004_02583_b200 as tk
ctx = tk.Context(0)
rng = np.random.default_rng(5)
g = rng.standard_normal((300, 300)); g = np.asfortranarray(g @ g.T)
vals, vecs = ctx.sym_eig(g, 12)
t = np.asfortranarray(rng.standard_normal((30, 20, 10)))
for eng in (tk.FactorEngine.svd(), tk.FactorEngine.eig()):
    ctx.t_hosvd(t, tk.Truncation([4, 3, 2]), eng)
maps = open("/proc/self/maps").read()
assert "libcusolver" not in maps, "cuSOLVER mapped"
w = np.linalg.eigvalsh(g)[::-1][:12]
assert np.max(np.abs(vals - w)) <= 1e-11 * w[0], (vals, w)
print("ok")
"""


def test_engines_map_no_cusolver(tmp_path):
    # the eigensolver is the repo's own (eig.cu): the process that runs the
    # EIG / SVD engines and sym_eig never maps a cuSOLVER library
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _NO_CUSOLVER, root], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


@pytest.mark.parametrize("n,k,kind", [(64, 64, "cluster"), (200, 50, "decay"), (513, 40, "cluster"),
                                      (2048, 64, "decay"), (1, 1, "decay"), (2, 2, "decay"), (3, 1, "decay")])
def test_sym_eig_spectra(ctx, ref, n, k, kind):
    # clustered (pairs 1e-9 apart) and power-law spectra: values against the
    # reference, vectors through the invariant subspace of the k leading pairs
    q = np.linalg.qr(random_matrix(ref, n, n, 900 + n))[0]
    if kind == "cluster":
        d = np.repeat(np.linspace(10.0, 1.0, (n + 1) // 2), 2)[:n] + 1e-9 * (np.arange(n) % 2)
    else:
        d = (1.0 + np.arange(n)) ** -1.5
    g = np.asfortranarray((q * d) @ q.T)
    g = 0.5 * (g + g.T)
    vals, vecs = ctx.sym_eig(g, k)
    if n <= 600:
        rv, ru = ref.sym_eig(g, k)
    else:  # LAPACK dsyevd (numpy) in the reference's order / sign convention
        w, z = np.linalg.eigh(g)
        rv, ru = w[::-1][:k], z[:, ::-1][:, :k].copy()
        for c in range(k):
            if ru[np.argmax(np.abs(ru[:, c])), c] < 0:
                ru[:, c] = -ru[:, c]
    assert np.max(np.abs(vals - rv)) <= 1e-13 * max(n, 16) * np.max(np.abs(rv))
    assert ortho_defect(vecs) <= 1e-13 * max(n, 16)
    resid = g @ vecs - vecs * vals
    assert np.max(np.abs(resid)) <= 1e-13 * max(n, 16) * np.max(np.abs(rv))
    # subspace of the leading k (cut where the spectrum has a gap)
    if k < n and d[k - 1] - d[k] > 1e-6:
        assert principal_sine(vecs, ru) <= 1e-9
    if kind == "decay":
        assert column_diff(vecs, ru) <= 1e-8
