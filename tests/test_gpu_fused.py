"""The fused sweep pass (csrc/sweep_fused.cu: right update, R^T R and the
left-update sum from one read of the tensor, r <= 16) against the oracle:
als_low_rank (als.cpp:98-161) on shapes that reach every variant of the
kernel — mode-1 fibers with one and two 128-row boxes, panel-local tiles with
partial last tiles, contraction extents that are not multiples of 8, ranks
with and without the DFMA tail — with identical iteration counts, histories to
1e-11 and factors to 1e-9, and the same decompositions with the pass disabled.
"""
import os

import numpy as np
import pytest

import paper_2004_02583_b200 as tk
from oracles import Port, Ref, random_tensor
from parity import assert_parity, compare_decompositions

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    den = np.linalg.norm(a)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (den if den > 0 else 1.0)


@pytest.fixture(scope="module")
def ctx():
    c = tk.Context(0)
    c.set_fused_sweep(True)  # off by default
    return c


@pytest.fixture(scope="module")
def ref():
    return Ref()


@pytest.fixture(scope="module")
def port():
    return Port()


def low_rank_plus_noise(ref, dims, ranks, seed, noise=1e-3):
    # (the closed-form residual sqrt(||A||^2 - tr) carries rounding noise eps ||A||^2 / (2 res^2)
    # relative: histories are compared at 1e-11 on residuals of at least 0.1 ||A||)
    rng = np.random.default_rng(seed)
    core = rng.standard_normal(ranks)
    t = core
    for k, (d, r) in enumerate(zip(dims, ranks)):
        q = np.linalg.qr(rng.standard_normal((d, r)))[0]
        t = np.moveaxis(np.tensordot(q, t, axes=(1, k)), 0, k)
    t = t + noise * np.linalg.norm(t) / np.sqrt(t.size) * rng.standard_normal(dims)
    return np.asfortranarray(t)


# (dims, mode, r): mode 1 = s 1 fibers (K <= 128: 32-fiber tiles, K > 128: 16-fiber
# tiles in two boxes), later modes = panel-local tiles
CASES = [
    ([96, 40, 30], 1, 10),     # one box, DFMA tail
    ([128, 50, 9], 1, 8),      # one box, 8 columns
    ([100, 37, 11], 1, 12),    # K = 4 (mod 16): no padding; 16 columns without a tail
    ([40, 64, 17], 1, 3),      # short fibers
    ([256, 30, 12], 1, 10),    # two boxes
    ([250, 33, 7], 1, 16),     # two boxes, K not a multiple of 8
    ([200, 21, 13], 1, 9),     # two boxes, one tail column
    ([130, 19, 5], 1, 5),      # two boxes, the second nearly empty
    ([64, 96, 12], 2, 10),     # panels of 64 fibers
    ([70, 50, 9], 2, 7),       # partial last tile per panel
    ([40, 20, 256], 3, 10),    # s = 800, 16-fiber tiles
    ([18, 10, 250], 3, 6),     # s = 180, K not a multiple of 8
    ([12, 11, 10, 100], 4, 10),  # order 4, last mode
    ([66, 130, 6], 2, 16),     # s = 66, 16-fiber tiles with a partial tile
]


@pytest.mark.parametrize("dims,mode,r", CASES, ids=lambda v: "x".join(map(str, v)) if isinstance(v, list) else str(v))
def test_fused_sweep_matches_oracle(ctx, ref, port, dims, mode, r):
    ranks = [min(d, r) for d in dims]
    t = low_rank_plus_noise(ref, dims, ranks, 4000 + sum(dims) + mode, noise=0.2)
    ctx.set_profiling(True)
    ctx.kernel_stats()
    (lg, rg), rep = ctx.als_low_rank(t, mode, r, tk.AlsConfig(eta=1e-6, seed=21))
    stats = ctx.kernel_stats()
    ctx.set_profiling(False)
    assert stats["sweep"]["launches"] >= rep.iterations, "the fused pass did not run"
    assert stats["fc"]["launches"] == 0
    lp, rp, prep = port.als_low_rank(t, mode, r, eta=1e-6, seed=21)
    assert rep.iterations == prep.iterations
    assert np.allclose(rep.residual_history, prep.residual_history, rtol=1e-11, atol=0)
    assert rel(lp, lg) <= 1e-8 and rel(rp, rg) <= 1e-8


def test_fused_sweep_random_tensor_many_sweeps(ctx, ref, port):
    # a full-rank random tensor: tens of sweeps, every one through the fused pass
    t = random_tensor(ref, [48, 30, 20], 611)
    (lg, rg), rep = ctx.als_low_rank(t, 1, 6, tk.AlsConfig(eta=1e-6, seed=3))
    lp, rp, prep = port.als_low_rank(t, 1, 6, eta=1e-6, seed=3)
    assert rep.iterations == prep.iterations and rep.iterations > 5
    assert np.allclose(rep.residual_history, prep.residual_history, rtol=1e-11, atol=0)
    assert rel(lp, lg) <= 1e-8 and rel(rp, rg) <= 1e-8


@pytest.mark.parametrize("sequential", [False, True])
def test_decompositions_through_fused_sweeps(ctx, ref, port, sequential):
    dims, ranks = [96, 80, 64], [10, 9, 8]
    t = low_rank_plus_noise(ref, dims, ranks, 77)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-8, seed=5, max_iters=50))
    if sequential:
        tkr, rep = ctx.st_hosvd(t, tk.Truncation(ranks), None, eng)
    else:
        tkr, rep = ctx.t_hosvd(t, tk.Truncation(ranks), eng)
    want = port.hosvd_als(t, ranks, sequential=sequential, eta=1e-8, seed=5)
    assert_parity(compare_decompositions(tkr, rep, want))


def test_fused_and_unfused_agree(ref):
    """The same decomposition with the fused pass switched off
    (tkg_set_fused_sweep): identical iteration counts, histories to 1e-11."""
    rng = np.random.default_rng(9)
    dims, ranks = [64, 72, 40], [10, 6, 12]
    core = rng.standard_normal(ranks)
    qs = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in zip(dims, ranks)]
    a = np.asfortranarray(np.einsum("abc,ia,jb,kc->ijk", core, *qs) + 1e-2 * rng.standard_normal(dims))
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-8, seed=13, max_iters=50))
    outs = []
    c = tk.Context(0)
    for on in (True, False):
        c.set_fused_sweep(on)
        c.set_profiling(True)
        c.kernel_stats()
        tkr, rep = c.t_hosvd(a, tk.Truncation(ranks), eng)
        stats = c.kernel_stats()
        c.set_profiling(False)
        assert (stats["sweep"]["launches"] > 0) == on
        outs.append(rep)
    c.set_fused_sweep(True)
    a_, b_ = outs
    assert [m.als.iterations for m in a_.per_mode] == [m.als.iterations for m in b_.per_mode]
    for ma, mb in zip(a_.per_mode, b_.per_mode):
        assert np.allclose(ma.als.residual_history, mb.als.residual_history, rtol=1e-11, atol=0)
    assert abs(a_.relative_residual - b_.relative_residual) <= 1e-12
