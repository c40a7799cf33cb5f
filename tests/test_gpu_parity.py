"""B200 parity tests: the CUDA path (through the C-ABI) against the oracle.

Oracles: ``Port`` (oracle/tenkit_oracle.c, pinned bitwise to the reference
by test_oracle_pins.py) and ``Ref`` (the compiled reference itself).
Tolerances are BASELINE.json's: |d rel_err| <= 1e-10, largest principal
angle <= 1e-8, core singular values 1e-9 relative, identical iteration
counts; contraction primitives at the reference's own 1e-13 bar
(test_tensor_ops.cpp:184-209, bench_kernels.cpp:61).
"""
import numpy as np
import pytest

import paper_2004_02583_b200 as tk
from oracles import SUBTYPES, OracleError, Port, Ref, counting_tensor, random_matrix, random_orthonormal, random_tensor
from parity import (CORE_SV_REL_TOL, assert_parity, column_alignment, column_diff, compare_decompositions,
                    ortho_defect, principal_sine)

pytestmark = pytest.mark.gpu

SHAPES = [[7], [6, 8], [3, 4, 5], [4, 3, 2, 5], [3, 2, 4, 2, 3], [40, 30, 20], [300, 9, 5],
          [5, 3, 700], [64, 33, 17], [10, 96, 7], [17, 4, 6, 5],
          # panel-local TMA tiles (s not a multiple of 32 / 128): s = 1500, 200, 1360
          [30, 50, 20], [200, 6, 4], [34, 40, 3]]


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.linalg.norm(a)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


@pytest.fixture(scope="module")
def ctx():
    return tk.Context(0)


@pytest.fixture(scope="module")
def ref():
    return Ref()


@pytest.fixture(scope="module")
def port():
    return Port()


# ---- the ALS initializer stream (rng.hpp:19-21,57-61; als.cpp:67-71) ----------
@pytest.mark.parametrize("seed,stream,n", [(0, 1, 1000), (7, 3, 70001), (2**40 + 5, 2, 655360),
                                           (11, 4, 3_000_000), (5, 1, 312), (5, 1, 1)])
def test_uniform01_stream_bitwise(ctx, ref, seed, stream, n):
    got = ctx.uniform01(seed, stream, n)
    want = ref.uniform01(seed, stream, n)
    assert np.array_equal(got, want)


# ---- contraction primitives (tensor_ops.cpp:129-330) --------------------------
@pytest.mark.parametrize("dims", SHAPES, ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("r", [1, 3, 10, 32, 50, 64])
def test_unfold_products(ctx, ref, port, dims, r):
    t = random_tensor(ref, dims, 101 + len(dims))
    for mode in range(1, len(dims) + 1):
        fibers = t.size // dims[mode - 1]
        m = random_matrix(ref, fibers, r, 110 + mode)
        l = random_matrix(ref, dims[mode - 1], r, 140 + mode)
        assert rel(port.unfold_times(t, mode, m), ctx.unfold_times(t, mode, m)) <= 1e-13
        assert rel(port.unfold_t_times(t, mode, l), ctx.unfold_t_times(t, mode, l)) <= 1e-13


# mode 1 with 128 < I_1 <= 248 and 40..64 columns: fr_wide_kernel (one CTA over
# all contraction rows, row tiles split by (row tile, column tile) pairs)
@pytest.mark.parametrize("dims", [[200, 64, 9], [129, 31, 20], [208, 17, 10], [248, 17, 10], [136, 5, 3]],
                         ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("r", [33, 40, 50, 56, 64])
def test_unfold_times_wide_rows(ctx, ref, port, dims, r):
    t = random_tensor(ref, dims, 307 + dims[0])
    fibers = t.size // dims[0]
    m = random_matrix(ref, fibers, r, 311 + r)
    assert rel(port.unfold_times(t, 1, m), ctx.unfold_times(t, 1, m)) <= 1e-13


# the same kernel for middle modes: kFibS panels (32 < s < 64, one panel per
# stage) and kFibJ panel-local chunks (s >= 64 or a multiple of 32)
@pytest.mark.parametrize("dims", [[50, 200, 7], [40, 136, 9], [64, 200, 5], [100, 208, 3], [33, 248, 4]],
                         ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("r", [40, 50, 64])
def test_unfold_times_wide_rows_middle_mode(ctx, ref, port, dims, r):
    t = random_tensor(ref, dims, 401 + dims[0])
    fibers = t.size // dims[1]
    m = random_matrix(ref, fibers, r, 413 + r)
    assert rel(port.unfold_times(t, 2, m), ctx.unfold_times(t, 2, m)) <= 1e-13


# FC on short panels (kFibS) with more than 32 columns: tiles of up to ~150
# fibers whose extra row tiles are dealt to the warps as (row tile, column
# tile) pairs
@pytest.mark.parametrize("dims", [[50, 200, 7], [34, 200, 5], [18, 100, 20], [40, 136, 9], [62, 64, 11]],
                         ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("r", [33, 40, 48, 50, 56, 64])
def test_unfold_t_times_short_panels(ctx, ref, port, dims, r):
    t = random_tensor(ref, dims, 431 + dims[0])
    l = random_matrix(ref, dims[1], r, 433 + r)
    assert rel(port.unfold_t_times(t, 2, l), ctx.unfold_t_times(t, 2, l)) <= 1e-13
    # the same contraction as a TTM with tensor-layout output (the st-HOSVD path)
    u = random_matrix(ref, r, dims[1], 437 + r)
    assert rel(port.mode_n_product(t, u, 2), ctx.mode_n_product(t, u, 2)) <= 1e-13


# the init pass (column-major S, fused ||A||^2) and the sweeps through the wide FR
@pytest.mark.parametrize("dims,mode,r", [([200, 40, 30], 1, 50), ([208, 30, 25], 1, 64), ([144, 40, 20], 1, 40),
                                         ([248, 20, 20], 1, 40), ([50, 200, 24], 2, 50), ([64, 200, 10], 2, 56),
                                         ([40, 136, 30], 2, 48)])
def test_als_low_rank_wide_rows(ctx, ref, port, dims, mode, r):
    t = random_tensor(ref, dims, 577 + r)
    (lg, rg), rep = ctx.als_low_rank(t, mode, r, tk.AlsConfig(eta=1e-6, seed=13, max_iters=8))
    lp, rp, prep = port.als_low_rank(t, mode, r, eta=1e-6, seed=13, max_iters=8)
    assert rep.iterations == prep.iterations
    assert np.allclose(rep.residual_history, prep.residual_history, rtol=1e-11, atol=0)
    assert rel(lp, lg) <= 1e-9 and rel(rp, rg) <= 1e-9


@pytest.mark.parametrize("dims", SHAPES[:9], ids=lambda d: "x".join(map(str, d)))
def test_mode_n_product(ctx, port, ref, dims):
    t = random_tensor(ref, dims, 53 + len(dims))
    for mode in range(1, len(dims) + 1):
        for rows in (1, 3, 70):
            u = random_matrix(ref, rows, dims[mode - 1], 60 + mode)
            assert rel(port.mode_n_product(t, u, mode), ctx.mode_n_product(t, u, mode)) <= 1e-13


def test_mode_n_product_literals(ctx):
    # test_tensor_ops.cpp:120-126: mode-1 row of ones sums fibers
    out = ctx.mode_n_product(counting_tensor([2, 2, 2]), np.ones((1, 2)), 1)
    assert out.shape == (1, 2, 2)
    assert list(out.reshape(-1, order="F")) == [3, 7, 11, 15]
    # identity is a bitwise copy (test_tensor_ops.cpp:112-118)
    t = counting_tensor([4, 5, 3]) / 7.0
    for mode in (1, 2, 3):
        assert np.array_equal(ctx.mode_n_product(t, np.eye(t.shape[mode - 1]), mode), t)


def test_norms(ctx, ref, port):
    # test_tensor_ops.cpp:230-240
    assert abs(ctx.frobenius_norm(np.ones((2, 2, 2))) - np.sqrt(8.0)) <= 1e-15 * np.sqrt(8)
    assert abs(ctx.frobenius_norm(counting_tensor([2, 2, 2])) - np.sqrt(204.0)) <= 1e-14 * 15
    assert ctx.frobenius_norm(np.zeros((3, 3))) == 0.0
    t = random_tensor(ref, [50, 40, 30], 9)
    u = t + 1e-3 * random_tensor(ref, [50, 40, 30], 10)
    assert abs(ctx.frobenius_norm(t) - port.frobenius_norm(t)) <= 1e-14 * port.frobenius_norm(t)
    assert abs(ctx.relative_error(t, u) - port.relative_error(t, u)) <= 1e-13
    with pytest.raises(tk.ZeroReferenceError):
        ctx.relative_error(np.zeros((3, 3)), np.ones((3, 3)))


# ---- small dense LA (kernels.cpp:303-417, matrix.cpp:90-126) ------------------
def test_reduced_qr_kat(ctx):
    # test_kernels.cpp:41-47: QR of [3;4]
    q, r = ctx.reduced_qr(np.array([[3.0], [4.0]]))
    assert abs(q[0, 0] - 0.6) <= 1e-15 and abs(q[1, 0] - 0.8) <= 1e-15
    assert abs(r[0, 0] - 5.0) <= 1e-14


@pytest.mark.parametrize("m,n", [(8, 3), (64, 10), (300, 32), (2048, 64), (200, 50), (5, 5)])
def test_reduced_qr_matches(ctx, ref, port, m, n):
    a = random_matrix(ref, m, n, 900 + m + n)
    q, r = ctx.reduced_qr(a)
    q2, r2 = port.reduced_qr(a)
    assert rel(q2, q) <= 1e-12 and rel(r2, r) <= 1e-12
    assert np.all(np.diag(r) >= 0)
    assert ortho_defect(q) <= 1e-14 * max(1, np.sqrt(m) / 4)


def test_gram(ctx, ref, port):
    a = random_matrix(ref, 3001, 37, 5)
    assert rel(port.gram(a), ctx.gram(a)) <= 1e-14


# ---- ALS engine (als.cpp) ----------------------------------------------------
def test_als_fixed_point_kat(ctx):
    # test_als.cpp:91-105: diag(3,1), l = e1 is a fixed point; residual 1, R = (3, 0)
    a = np.diag([3.0, 1.0])
    (l, r), rep = ctx.als_low_rank(a, 1, 1, tk.AlsConfig(eta=1e-4, max_iters=1,
                                                         init=np.array([[1.0], [0.0]])))
    assert abs(rep.residual_history[0] - 1.0) <= 1e-14
    assert l[0, 0] == 1.0 and l[1, 0] == 0.0
    assert abs(r[0, 0] - 3.0) <= 1e-15 and r[1, 0] == 0.0


def test_als_contraction_ratio_kat(ctx):
    # test_als.cpp:107-121: diag(2,1), l=(1,1): ratio 0.25 after one sweep,
    # residual sqrt(2.5)
    a = np.diag([2.0, 1.0])
    (l, r), rep = ctx.als_low_rank(a, 1, 1, tk.AlsConfig(eta=0.0, max_iters=2,
                                                         init=np.array([[1.0], [1.0]])))
    assert abs(rep.residual_history[0] - np.sqrt(2.5)) <= 1e-15 * 2
    assert abs(l[1, 0] / l[0, 0] - 0.25) <= 1e-15


@pytest.mark.parametrize("dims,mode,r", [([7, 8, 6], 1, 2), ([7, 8, 6], 2, 3), ([7, 8, 6], 3, 2),
                                         ([30, 20, 10], 2, 5), ([12, 10, 8, 6], 4, 3),
                                         # r > 32: R^T R by the row pass of finish_step; r mod 8 in {1, 2}: DFMA tail
                                         ([90, 64, 40], 1, 50), ([64, 90, 40], 2, 41), ([80, 70, 30], 1, 48)])
def test_als_low_rank_matches_oracle(ctx, ref, port, dims, mode, r):
    t = random_tensor(ref, dims, 573 + mode)
    (lg, rg), rep = ctx.als_low_rank(t, mode, r, tk.AlsConfig(eta=1e-6, seed=11))
    lp, rp, prep = port.als_low_rank(t, mode, r, eta=1e-6, seed=11)
    assert rep.iterations == prep.iterations
    assert np.allclose(rep.residual_history, prep.residual_history, rtol=1e-11, atol=0)
    assert rel(lp, lg) <= 1e-9 and rel(rp, rg) <= 1e-9


def test_als_init_matches_oracle(ctx, ref, port):
    t = random_tensor(ref, [6, 7, 8], 510)
    a = ctx.als_init(t, 2, 3, 99)
    b = port.als_init(t, 2, 3, 99)
    assert rel(b, a) <= 1e-12


def test_returned_pair_is_consistent(ctx, ref, port):
    # test_als.cpp:166-178
    t = random_tensor(ref, [7, 6, 5], 560)
    (l, r), rep = ctx.als_low_rank(t, 1, 3, tk.AlsConfig(eta=1e-5))
    g = port.gram(l)
    atl = port.unfold_t_times(t, 1, l)
    r_star = port.spd_solve(g, atl.T).T
    assert rel(r_star, r) <= 1e-12


def test_als_cap_and_huge_eta(ctx, ref):
    t = random_tensor(ref, [6, 7, 8], 570)
    _, rep = ctx.als_low_rank(t, 3, 2, tk.AlsConfig(eta=10.0))
    assert rep.status == "converged" and rep.iterations == 1 and len(rep.residual_history) == 1
    t = random_tensor(ref, [6, 7, 8], 571)
    _, rep = ctx.als_low_rank(t, 1, 2, tk.AlsConfig(eta=1e-300, max_iters=5))
    assert rep.status == "max_iters_reached" and rep.iterations == 5


def test_error_taxonomy(ctx, ref):
    with pytest.raises(tk.ZeroReferenceError):  # test_als.cpp:273-278
        ctx.als_low_rank(np.zeros((4, 5, 3)), 1, 2, tk.AlsConfig())
    t = random_tensor(ref, [6, 7, 8], 511)
    with pytest.raises(tk.RankTooLargeError):  # test_als.cpp:76-89
        ctx.als_init(t, 1, 7, 0)
    with pytest.raises(tk.RankTooLargeError):
        ctx.als_init(t, 1, 0, 0)
    with pytest.raises(tk.DegenerateInitError):
        ctx.als_init(np.zeros((5, 5)), 1, 2, 0)
    with pytest.raises(tk.InvalidModeError):
        ctx.unfold_t_times(t, 9, np.zeros((3, 2)))
    with pytest.raises(tk.DimensionMismatchError):
        ctx.mode_n_product(t, np.zeros((2, 3)), 2)
    # rank above the numerical rank from a full-rank warm start (test_als.cpp:257-271)
    l0 = random_matrix(ref, 8, 2, 590)
    r0 = random_matrix(ref, 12, 2, 591)
    low = l0 @ r0.T
    init = np.zeros((8, 3))
    init[0, 0] = init[1, 1] = init[2, 2] = 1.0
    with pytest.raises(tk.RankTooLargeError) as ei:
        ctx.als_low_rank(low, 1, 3, tk.AlsConfig(init=init))
    assert "mode 1" in str(ei.value)


# ---- decompositions ------------------------------------------------------------
def _tucker_exact(ref, dims, ranks, seed):
    core = random_tensor(ref, ranks, seed)
    factors = [random_orthonormal(ref, dims[k], ranks[k], seed + 1 + k) for k in range(len(dims))]
    return ref.reconstruct(core, factors, dims)


@pytest.mark.parametrize("sequential", [False, True])
def test_order1(ctx, ref, sequential):
    # an order-1 tensor is its own rank-1 Tucker model: U = +-a/||a||, core = +-||a||
    a = random_tensor(ref, [57], 4)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-8, seed=3))
    fn = (lambda: ctx.st_hosvd(a, tk.Truncation([1]), None, eng)) if sequential else \
        (lambda: ctx.t_hosvd(a, tk.Truncation([1]), eng))
    tkr, rep = fn()
    u = tkr.factors[0][:, 0]
    assert abs(abs(float(np.dot(u, a))) - np.linalg.norm(a)) <= 1e-12 * np.linalg.norm(a)
    assert abs(abs(float(tkr.core.reshape(-1)[0])) - np.linalg.norm(a)) <= 1e-12 * np.linalg.norm(a)
    assert rep.relative_residual <= 1e-12


@pytest.mark.parametrize("sequential", [False, True])
def test_exact_recovery(ctx, ref, sequential):
    # test_hosvd.cpp:79-95 / acceptance C1: exact rank-(2,3,2) tensor
    t = _tucker_exact(ref, [10, 11, 9], [2, 3, 2], 42)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-6, seed=5, max_iters=100))
    if sequential:
        tkr, rep = ctx.st_hosvd(t, tk.Truncation([2, 3, 2]), None, eng)
    else:
        tkr, rep = ctx.t_hosvd(t, tk.Truncation([2, 3, 2]), eng)
    assert rep.relative_residual <= 1e-8
    assert max(ortho_defect(u) for u in tkr.factors) <= 1e-12


@pytest.mark.parametrize("sequential", [False, True])
@pytest.mark.parametrize("dims,ranks", [([9, 8, 7], [3, 2, 4]), ([20, 18, 16], [5, 4, 3]),
                                        ([12, 10, 8, 6], [3, 3, 2, 2]), ([40, 30, 20], [10, 10, 5]),
                                        # ranks > 32: the R^T R row pass (finish_step) and r x r
                                        # factorizations with 9 / 16 entries per thread
                                        ([90, 80, 70], [40, 33, 50]), ([96, 80, 72], [64, 60, 36]),
                                        # order 2 (the t-HOSVD core's first step is the shrink of
                                        # the last mode's R), odd / short panels
                                        ([37, 29], [5, 5]), ([3, 130, 5, 7], [2, 9, 3, 2])])
def test_hosvd_matches_reference(ctx, ref, sequential, dims, ranks):
    if sequential and len(dims) == 2:
        pytest.skip("order-2 st-HOSVD: the second mode's shrunk tensor is exactly rank r, "
                    "its stopping test compares rounding noise")
    t = random_tensor(ref, dims, 3 + len(dims))
    t = t + 5 * _tucker_exact(ref, dims, ranks, 77)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-8, seed=7, max_iters=50))
    if sequential:
        tkr, rep = ctx.st_hosvd(t, tk.Truncation(ranks), None, eng)
    else:
        tkr, rep = ctx.t_hosvd(t, tk.Truncation(ranks), eng)
    r = ref.hosvd_als(t, ranks, sequential=sequential, eta=1e-8, seed=7)
    assert_parity(compare_decompositions(tkr, rep, r))


def test_st_order_and_reports(ctx, ref):
    # test_hosvd.cpp:147-168: per-mode reports follow the processing order
    t = random_tensor(ref, [8, 7, 9], 604)
    tkr, rep = ctx.st_hosvd(t, tk.Truncation([3, 2, 4]), None,
                            tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-4, seed=2)))
    assert [m.mode for m in rep.per_mode] == [2, 1, 3]
    _, rep2 = ctx.st_hosvd(t, tk.Truncation([3, 2, 4]), tk.ModeOrder([3, 2, 1]),
                           tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-4, seed=2)))
    assert [m.mode for m in rep2.per_mode] == [3, 2, 1]
    with pytest.raises(tk.InvalidModeError):
        ctx.st_hosvd(t, tk.Truncation([3, 2, 4]), tk.ModeOrder([1, 1, 2]),
                     tk.FactorEngine.with_als(tk.AlsConfig()))


def test_st_core_shortcut(ctx, ref, port):
    # test_hosvd.cpp:123-134 / acceptance C12: the R_hat R^T shrink equals the
    # direct contraction with U^T within 1e-10
    t = random_tensor(ref, [8, 9, 10], 602)
    t = t * 1e-3 + _tucker_exact(ref, [8, 9, 10], [3, 2, 4], 603)
    tkr, _ = ctx.st_hosvd(t, tk.Truncation([3, 2, 4]), None,
                          tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-4, seed=7)))
    direct = t
    for n in range(3):
        direct = port.mode_n_product(direct, tkr.factors[n].T, n + 1)
    assert port.relative_error(direct, tkr.core) <= 1e-10


def test_rank_validation(ctx, ref):
    t = random_tensor(ref, [6, 5, 4], 1)
    eng = tk.FactorEngine.with_als(tk.AlsConfig())
    with pytest.raises(tk.RankTooLargeError) as ei:
        ctx.t_hosvd(t, tk.Truncation([2, 6, 2]), eng)
    assert "mode 2" in str(ei.value)
    with pytest.raises(tk.DimensionMismatchError):
        ctx.t_hosvd(t, tk.Truncation([2, 2]), eng)


# ---- BASELINE configs 1 and 2 at full size against the compiled reference ------
def test_config1_t_hosvd_256cubed(ctx, ref):
    dims, ranks = [256, 256, 256], [10, 10, 10]
    a = tk.synth_tucker(dims, ranks, 0.0, 1e-3, 2004025831).reshape(dims, order="F")
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-8, seed=7, max_iters=50))
    tkr, rep = ctx.t_hosvd(a, tk.Truncation(ranks), eng)
    ref.set_threads(ref.max_threads())
    r = ref.hosvd_als(a, ranks, sequential=False, eta=1e-8, seed=7)
    m = compare_decompositions(tkr, rep, r)
    assert_parity(m)


def test_config2_st_hosvd_96pow4(ctx, ref):
    dims, ranks = [96, 96, 96, 96], [10, 10, 10, 10]
    a = tk.synth_tucker(dims, ranks, 0.0, 1e-3, 2004025832).reshape(dims, order="F")
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-8, seed=7, max_iters=50))
    tkr, rep = ctx.st_hosvd(a, tk.Truncation(ranks), None, eng)
    ref.set_threads(ref.max_threads())
    r = ref.hosvd_als(a, ranks, sequential=True, eta=1e-8, seed=7)
    assert_parity(compare_decompositions(tkr, rep, r))


# ---- recover_singular_vectors (hosvd.cpp:65-72; §8(f) row 1) -------------------
def test_recover_singular_vectors_kat(ctx, ref):
    # test_hosvd.cpp:200-223: recovery undoes a rotation of the leading vectors
    u = random_orthonormal(ref, 12, 6, 610)
    v = random_orthonormal(ref, 15, 6, 611)
    a = np.asfortranarray((u * np.array([5, 4, 3, 2, 1, 0.5])) @ v.T)
    q = u[:, :3] @ random_orthonormal(ref, 3, 3, 611)
    w = ctx.recover_singular_vectors(a, 1, q)
    for j in range(3):
        assert column_alignment(w, j, u, j) >= 1.0 - 1e-8
    assert column_diff(w, ref.recover_singular_vectors(a, 1, q)) <= 1e-12
    w2 = ctx.recover_singular_vectors(a, 1, u[:, :3])
    for j in range(3):
        assert column_alignment(w2, j, u, j) >= 1.0 - 1e-8


@pytest.mark.parametrize("dims,r", [([40, 30, 20], 3), ([64, 33, 17], 10), ([80, 70, 60], 32),
                                    ([90, 64, 40], 50), ([70, 66, 50], 64), ([200, 6, 4], 4),
                                    ([17, 4, 6, 5], 3)], ids=str)
def test_recover_singular_vectors_matches_reference(ctx, ref, dims, r):
    t = random_tensor(ref, dims, 300 + r)
    for mode in range(1, len(dims) + 1):
        rr = min(r, dims[mode - 1])
        q = random_orthonormal(ref, dims[mode - 1], rr, 400 + mode)
        got = ctx.recover_singular_vectors(t, mode, q)
        want = ref.recover_singular_vectors(t, mode, q)
        assert column_diff(got, want) <= 1e-10, (mode, column_diff(got, want))
        assert ortho_defect(got) <= 1e-14 * max(1, rr)


@pytest.mark.parametrize("dims,ranks,alpha", [([60, 50, 40], [6, 5, 4], 0.0),
                                              ([160, 150, 64], [64, 48, 32], 1.5),
                                              ([96, 80, 72], [32, 40, 20], 1.0)], ids=str)
def test_t_hosvd_singular_vectors_matches_reference(ctx, ref, dims, ranks, alpha):
    # want_singular_vectors (hosvd.cpp:100-106): factors are singular vectors,
    # determined column by column, and the core is determined with them
    a = tk.synth_tucker(dims, ranks, alpha, 1e-3, 77).reshape(dims, order="F")
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-8, seed=7, max_iters=50))
    tkr, rep = ctx.t_hosvd(a, tk.Truncation(ranks), eng, True)
    ref.set_threads(ref.max_threads())
    r = ref.hosvd_als(a, ranks, eta=1e-8, seed=7, want_singular_vectors=True)
    assert_parity(compare_decompositions(tkr, rep, r))
    for u, v in zip(tkr.factors, r.factors):
        assert column_diff(u, v) <= 1e-8
    assert np.max(np.abs(tkr.core - r.core)) <= CORE_SV_REL_TOL * np.max(np.abs(r.core))
    # the rotation leaves the approximation unchanged (test_hosvd.cpp:225-240)
    _, plain = ctx.t_hosvd(a, tk.Truncation(ranks), eng)
    assert abs(plain.relative_residual - rep.relative_residual) <= 1e-10


def test_recover_singular_vectors_errors(ctx):
    t = np.ones((4, 5, 6), order="F")
    with pytest.raises(tk.InvalidModeError):
        ctx.recover_singular_vectors(t, 4, np.eye(4)[:, :2])
    with pytest.raises(tk.DimensionMismatchError):
        ctx.recover_singular_vectors(t, 1, np.eye(5)[:, :2])


# ---- shapes beyond the BASELINE configs -----------------------------------------
@pytest.mark.parametrize("sequential", [False, True])
@pytest.mark.parametrize("dims,ranks", [([1, 7, 5], [1, 2, 3]), ([5000, 12, 9], [5, 4, 3]),
                                        ([9, 8, 7, 6, 5], [2, 3, 2, 3, 2]), ([64, 64, 64], [64, 1, 32])],
                         ids=str)
def test_unusual_shapes_match_reference(ctx, ref, sequential, dims, ranks):
    t = random_tensor(ref, dims, 900 + len(dims))
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-8, seed=3, max_iters=50))

    def gpu():
        if sequential:
            return ctx.st_hosvd(t, tk.Truncation(ranks), None, eng)
        return ctx.t_hosvd(t, tk.Truncation(ranks), eng)
    try:
        r = ref.hosvd_als(t, ranks, sequential=sequential, eta=1e-8, seed=3)
    except Exception as e:  # the reference's own failure (e.g. a collapsed range): same class, same text
        with pytest.raises(tk.Error) as ei:
            gpu()
        assert type(ei.value).__name__ == SUBTYPES[e.subtype] and str(ei.value) == str(e)
        return
    tkr, rep = gpu()
    m = compare_decompositions(tkr, rep, r)
    # a mode with R_n = I_n is an exact fit: its closed-form residual
    # sqrt(max(0, ||A||^2 - tr(G_L G_R))) is rounding noise of size
    # sqrt(eps) ||A|| ~ eta, so its sweep count is decided by that noise in
    # any implementation; every other mode must match exactly
    exact = {n + 1 for n in range(len(dims)) if ranks[n] == dims[n]}
    got = [it for it in m["iters_gpu"] if it[0] not in exact]
    want = [it for it in m["iters_ref"] if it[0] not in exact]
    assert got == want, (m["iters_gpu"], m["iters_ref"])
    assert m["rel_err_abs_diff"] <= 1e-10


def test_st_all_orders_of_a_4way_tensor(ctx, ref):
    import itertools
    dims, ranks = [10, 9, 8, 7], [3, 4, 2, 3]
    t = random_tensor(ref, dims, 77)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-8, seed=5))
    for order in itertools.permutations([1, 2, 3, 4]):
        tkr, rep = ctx.st_hosvd(t, tk.Truncation(ranks), tk.ModeOrder(list(order)), eng)
        r = ref.hosvd_als(t, ranks, sequential=True, order=list(order), eta=1e-8, seed=5)
        assert [p.mode for p in rep.per_mode] == list(order)
        assert_parity(compare_decompositions(tkr, rep, r))


def test_rank_above_fiber_count_collapses_like_reference(ctx, ref):
    # r = 70 > 30 fibers: the randomized range has rank 30 (als.cpp:74-86)
    t = random_tensor(ref, [80, 6, 5], 9)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-8, seed=3))
    with pytest.raises(OracleError) as want:
        ref.hosvd_als(t, [70, 3, 3], eta=1e-8, seed=3)
    with pytest.raises(tk.DegenerateInitError) as got:
        ctx.t_hosvd(t, tk.Truncation([70, 3, 3]), eng)
    assert str(got.value) == str(want.value)


# ---- multi_mode_product / reconstruct (tensor_ops.cpp:171-191, 420-440) -------
def test_multi_mode_product_and_reconstruct(ctx, ref):
    t = random_tensor(ref, [9, 8, 7, 6], 41)
    us = [(random_matrix(ref, 5, 8, 42), 2), (random_matrix(ref, 70, 6, 43), 4), (random_matrix(ref, 3, 9, 44), 1)]
    got = ctx.multi_mode_product(t, us)
    want = t
    for u, m in sorted(us, key=lambda x: x[1]):  # ascending modes, as the reference applies them
        want = ref.mode_n_product(want, u, m)
    assert got.shape == (3, 5, 7, 70)
    assert rel(got, want) <= 1e-13
    assert np.array_equal(ctx.multi_mode_product(t, []), t)
    with pytest.raises(tk.InvalidModeError):
        ctx.multi_mode_product(t, [(us[0][0], 2), (us[0][0], 2)])
    with pytest.raises(tk.DimensionMismatchError):
        ctx.multi_mode_product(t, [(random_matrix(ref, 2, 5, 45), 1)])
    # reconstruct: core x_n U_n against the reference
    core = random_tensor(ref, [3, 4, 2], 46)
    factors = [random_orthonormal(ref, d, r, 47 + d) for d, r in zip([20, 15, 10], [3, 4, 2])]
    tkr = tk.TuckerTensor(core, factors, (20, 15, 10))
    assert rel(ctx.reconstruct(tkr), ref.reconstruct(core, factors, [20, 15, 10])) <= 1e-13


# ---- als_sweep (als.cpp:89-96) -----------------------------------------------------
@pytest.mark.parametrize("dims,mode,r", [([7, 8, 6], 1, 2), ([40, 30, 20], 2, 10), ([64, 17, 40], 3, 32),
                                         ([90, 64, 40], 1, 50), ([17, 4, 6, 5], 4, 3)], ids=str)
def test_als_sweep_matches_reference(ctx, ref, dims, mode, r):
    t = random_tensor(ref, dims, 600 + r)
    l = random_matrix(ref, dims[mode - 1], r, 601 + r)
    (ln, rr), res = ctx.als_sweep(t, mode, l)
    ln_ref, rr_ref, res_ref = ref.als_sweep(t, mode, l)
    assert rel(rr, rr_ref) <= 1e-12 and rel(ln, ln_ref) <= 1e-12
    assert abs(res - res_ref) <= 1e-12 * max(1.0, res_ref)


def test_als_sweep_singular_gram(ctx, ref):
    # a rank-deficient L: spd_solve rejects L^T L (kernels.cpp:385-391)
    t = random_tensor(ref, [9, 8, 7], 5)
    l = np.asfortranarray(np.repeat(random_matrix(ref, 9, 1, 6), 2, axis=1))
    with pytest.raises(tk.SingularGramError) as ei:
        ctx.als_sweep(t, 1, l)
    assert str(ei.value).startswith("spd_solve: pivot ") and "at column 2" in str(ei.value)
    with pytest.raises(Exception) as er:
        ref.als_sweep(t, 1, l)
    assert "at column 2" in str(er.value)
