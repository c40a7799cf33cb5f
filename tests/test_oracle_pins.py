"""Pin the plain-C oracle port (oracle/tenkit_oracle.c) BITWISE against the
compiled, unmodified reference (oracle/_ref/libtenkit_ref.so).

The reference is thread-count invariant by construction (parallel.hpp:7-13,
test_tensor_ops.cpp:329-352), and the port keeps its loop and summation
orders, so every comparison here is exact equality, not a tolerance.
CPU-only (runs in the driver's ``-m "not gpu"`` pass).
"""
import numpy as np
import pytest

from oracles import Port, Ref, counting_tensor, random_matrix, random_orthonormal, random_tensor
from parity import column_alignment, column_diff

# test_tensor_ops.cpp:26-27 kOracleShapes, plus shapes that cross the
# 1024-fiber chunk (parallel.hpp:10) and the 256-row tiling (tensor_ops.cpp:239).
SHAPES = [[7], [6, 8], [3, 4, 5], [4, 3, 2, 5], [3, 2, 4, 2, 3], [40, 30, 20], [300, 9, 5],
          [5, 3, 700]]


@pytest.fixture(scope="module")
def ref():
    return Ref()


@pytest.fixture(scope="module")
def port():
    return Port()


@pytest.mark.parametrize("seed,stream", [(0, 0), (7, 1), (7, 3), (2**40 + 5, 2), (2**64 - 1, 9)])
def test_mt19937_64_seed_seq_stream(ref, port, seed, stream):
    # rng.hpp:57-61 seeded_engine; rng.hpp:19-21 uniform01.
    assert np.array_equal(ref.engine_raw(seed, stream, 1500), port.engine_raw(seed, stream, 1500))
    assert np.array_equal(ref.uniform01(seed, stream, 700), port.uniform01(seed, stream, 700))


def test_gaussian_stream(ref, port):
    # rng.hpp:30-53 Box-Muller pairs, odd count.
    assert np.array_equal(ref.gaussian(11, 1001), port.gaussian(11, 1001))


@pytest.mark.parametrize("dims", SHAPES, ids=lambda d: "x".join(map(str, d)))
def test_contractions_bitwise(ref, port, dims):
    t = random_tensor(ref, dims, 101 + len(dims))
    for mode in range(1, len(dims) + 1):
        fibers = t.size // dims[mode - 1]
        m = random_matrix(ref, fibers, 3, 110 + mode)
        l = random_matrix(ref, dims[mode - 1], 3, 140 + mode)
        u = random_matrix(ref, 2, dims[mode - 1], 60 + mode)
        assert np.array_equal(ref.unfold_times(t, mode, m), port.unfold_times(t, mode, m))
        assert np.array_equal(ref.unfold_t_times(t, mode, l), port.unfold_t_times(t, mode, l))
        assert np.array_equal(ref.mode_n_product(t, u, mode), port.mode_n_product(t, u, mode))
    assert ref.frobenius_norm(t) == port.frobenius_norm(t)


def test_small_dense_la_bitwise(ref, port):
    for seed, (m, n) in enumerate([(2, 1), (8, 3), (64, 10), (300, 32), (5, 5)]):
        a = random_matrix(ref, m, n, 900 + seed)
        q1, r1 = ref.reduced_qr(a)
        q2, r2 = port.reduced_qr(a)
        assert np.array_equal(q1, q2) and np.array_equal(r1, r2)
        g = ref.gram(a)
        assert np.array_equal(g, port.gram(a))
        b = random_matrix(ref, n, 7, 950 + seed)
        g2 = g + np.eye(n) * 1e-3
        assert np.array_equal(ref.spd_solve(g2, b), port.spd_solve(g2, b))


def test_als_low_rank_bitwise(ref, port):
    t = random_tensor(ref, [7, 8, 6], 573)
    for mode in (1, 2, 3):
        l1, r1, rep1 = ref.als_low_rank(t, mode, 2, eta=1e-6, seed=11)
        l2, r2, rep2 = port.als_low_rank(t, mode, 2, eta=1e-6, seed=11)
        assert np.array_equal(l1, l2) and np.array_equal(r1, r2)
        assert rep1.iterations == rep2.iterations
        assert rep1.residual_history == rep2.residual_history
        assert rep1.achieved_eta == rep2.achieved_eta


@pytest.mark.parametrize("sequential", [False, True])
def test_hosvd_bitwise(ref, port, sequential):
    t = random_tensor(ref, [9, 8, 7], 3)
    a = ref.hosvd_als(t, [3, 2, 4], sequential=sequential, eta=1e-8, seed=7)
    b = port.hosvd_als(t, [3, 2, 4], sequential=sequential, eta=1e-8, seed=7)
    assert np.array_equal(a.core, b.core)
    for x, y in zip(a.factors, b.factors):
        assert np.array_equal(x, y)
    assert a.relative_residual == b.relative_residual
    assert [(m.mode, m.iterations, m.status) for m in a.per_mode] == \
           [(m.mode, m.iterations, m.status) for m in b.per_mode]
    for x, y in zip(a.per_mode, b.per_mode):
        assert x.residual_history == y.residual_history


def test_select_order(ref, port):
    # test_hosvd.cpp:170-178
    assert port.select_order([10, 5, 20]) == [2, 1, 3]
    assert port.select_order([5, 5, 5]) == [1, 2, 3]
    assert port.select_order([7, 7, 2]) == [3, 1, 2]
    assert ref.select_order([2048, 2048, 512], [64, 64, 32]) == [3, 1, 2]
    assert port.select_order([64, 64, 32]) == [3, 1, 2]


def test_error_taxonomy_matches(ref, port):
    # errors.hpp:24-64: same category (return code) and subtype on both sides.
    zero = np.zeros((4, 5, 3), order="F")
    for lib in (ref, port):
        with pytest.raises(Exception) as ei:
            lib.als_low_rank(zero, 1, 2)
        assert ei.value.subtype == 3 and ei.value.code == 1  # ZeroReference, usage
        t = counting_tensor([3, 4, 5])
        with pytest.raises(Exception) as ei:
            lib.als_init(t, 1, 4, 0)
        assert ei.value.subtype == 4 and ei.value.code == 3  # RankTooLarge, numerical
        with pytest.raises(Exception) as ei:
            lib.unfold_t_times(t, 9, np.zeros((3, 2)))
        assert ei.value.subtype == 1 and ei.value.code == 1  # InvalidMode


def spectrum_tensor(ref, rows, cols, sigma, seed):
    """test_hosvd.cpp:60-74: order-2 tensor u diag(sigma) v^T."""
    u = random_orthonormal(ref, rows, len(sigma), seed)
    v = random_orthonormal(ref, cols, len(sigma), seed + 1)
    return np.asfortranarray((u * np.asarray(sigma)) @ v.T), u


def test_recover_singular_vectors_port(ref, port):
    # test_hosvd.cpp:200-223: recovery undoes a rotation of the leading vectors
    a, u = spectrum_tensor(ref, 12, 15, [5, 4, 3, 2, 1, 0.5], 610)
    q = u[:, :3] @ random_orthonormal(ref, 3, 3, 611)
    for lib in (ref, port):
        w = lib.recover_singular_vectors(a, 1, q)
        assert w.shape == (12, 3)
        for j in range(3):
            assert column_alignment(w, j, u, j) >= 1.0 - 1e-8
        w2 = lib.recover_singular_vectors(a, 1, u[:, :3])
        for j in range(3):
            assert column_alignment(w2, j, u, j) >= 1.0 - 1e-8
    # the restatement (Hestenes Jacobi) agrees with Golub-Kahan to rounding,
    # signs included, on every mode of a 3-way tensor
    t = random_tensor(ref, [9, 8, 10], 77)
    for mode, r in ((1, 3), (2, 5), (3, 4)):
        q = random_orthonormal(ref, t.shape[mode - 1], r, 80 + mode)
        assert column_diff(port.recover_singular_vectors(t, mode, q),
                           ref.recover_singular_vectors(t, mode, q)) <= 1e-12


def test_t_hosvd_singular_vectors_port(ref, port):
    # test_hosvd.cpp:225-240 and the want_singular_vectors branch (hosvd.cpp:100-106)
    t = random_tensor(ref, [9, 8, 10], 613)
    a = ref.hosvd_als(t, [3, 3, 2], eta=1e-8, seed=7, want_singular_vectors=True)
    b = port.hosvd_als(t, [3, 3, 2], eta=1e-8, seed=7, want_singular_vectors=True)
    for x, y in zip(a.factors, b.factors):
        assert column_diff(y, x) <= 1e-11
    assert np.max(np.abs(a.core - b.core)) <= 1e-11 * np.max(np.abs(a.core))
    assert abs(a.relative_residual - b.relative_residual) <= 1e-13
    plain = ref.hosvd_als(t, [3, 3, 2], eta=1e-8, seed=7)
    assert abs(plain.relative_residual - a.relative_residual) <= 1e-10
