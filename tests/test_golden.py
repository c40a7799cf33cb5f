"""The oracle port against the committed golden fixtures and the reference's
own known-answer tests (CPU only). Fixtures: tests/golden/make_golden.py ran
the compiled reference; KATs cite the reference test that states them."""
import numpy as np
import pytest

from golden_io import Fixture, fixtures, long_stream, streams
from oracles import Port, counting_tensor
from parity import column_diff


@pytest.fixture(scope="module")
def port():
    return Port()


SV = [n for n in fixtures() if Fixture(n).meta.get("want_singular_vectors")]


@pytest.mark.parametrize("name", [n for n in fixtures() if n not in SV])
def test_port_reproduces_reference_fixture_bitwise(port, name):
    fx = Fixture(name)
    m = fx.meta
    res = port.hosvd_als(fx.tensor, fx.ranks, sequential=m["sequential"], order=m["order"],
                         eta=m["eta"], seed=m["seed"])
    assert [p.mode for p in res.per_mode] == fx.modes
    assert [p.iterations for p in res.per_mode] == fx.iterations
    assert [p.status for p in res.per_mode] == fx.status
    for p, h in zip(res.per_mode, fx.histories):
        assert p.residual_history == h
    assert np.array_equal(res.core, fx.core)
    for u, v in zip(res.factors, fx.factors):
        assert np.array_equal(u, v)
    assert res.relative_residual == fx.relative_residual


@pytest.mark.parametrize("name", SV)
def test_port_singular_vector_fixture(port, name):
    # the ALS stage is bitwise; the singular-vector rotation (Hestenes Jacobi
    # in the port, Golub-Kahan in the reference) agrees to rounding
    fx = Fixture(name)
    m = fx.meta
    res = port.hosvd_als(fx.tensor, fx.ranks, eta=m["eta"], seed=m["seed"], want_singular_vectors=True)
    assert [p.iterations for p in res.per_mode] == fx.iterations
    for p, h in zip(res.per_mode, fx.histories):
        assert p.residual_history == h
    for u, v in zip(res.factors, fx.factors):
        assert column_diff(u, v) <= 1e-11
    assert np.max(np.abs(res.core - fx.core)) <= 1e-11 * np.max(np.abs(fx.core))
    assert abs(res.relative_residual - fx.relative_residual) <= 1e-13


def test_port_streams_match_reference(port):
    for key, d in streams().items():
        seed, stream = (int(x) for x in key.split("_"))
        raw = port.engine_raw(seed, stream, len(d["raw"]))
        assert [str(int(x)) for x in raw] == d["raw"]
        assert port.uniform01(seed, stream, len(d["uniform01"])).tolist() == d["uniform01"]


def test_port_long_stream_picks(port):
    idx, val, checksum = long_stream()
    draws = port.uniform01(11, 4, int(idx.max()) + 1)
    assert np.array_equal(draws[idx], val)


# ---- known-answer tests restated from the reference's test suite -------------
def test_kat_qr_3_4(port):  # test_kernels.cpp:41-47
    q, r = port.reduced_qr(np.array([[3.0], [4.0]]))
    assert abs(q[0, 0] - 0.6) <= 1e-15 and abs(q[1, 0] - 0.8) <= 1e-15 and abs(r[0, 0] - 5) <= 1e-14


def test_kat_fixed_point(port):  # test_als.cpp:91-105
    l, r, rep = port.als_low_rank(np.diag([3.0, 1.0]), 1, 1, eta=1e-4, max_iters=1,
                                  init=np.array([[1.0], [0.0]]))
    assert abs(rep.residual_history[0] - 1.0) <= 1e-14
    assert l[0, 0] == 1.0 and l[1, 0] == 0.0 and r[0, 0] == 3.0 and r[1, 0] == 0.0


def test_kat_contraction_ratio(port):  # test_als.cpp:107-121
    l, r, rep = port.als_low_rank(np.diag([2.0, 1.0]), 1, 1, eta=0.0, max_iters=2,
                                  init=np.array([[1.0], [1.0]]))
    assert abs(rep.residual_history[0] - np.sqrt(2.5)) <= 1e-15 * 2
    assert abs(l[1, 0] / l[0, 0] - 0.25) <= 1e-15


def test_kat_norms_and_products(port):  # test_tensor_ops.cpp:120-126, 230-240
    assert abs(port.frobenius_norm(np.ones((2, 2, 2))) - np.sqrt(8.0)) <= 1e-15 * 3
    assert abs(port.frobenius_norm(counting_tensor([2, 2, 2])) - np.sqrt(204.0)) <= 1e-14 * 15
    out = port.mode_n_product(counting_tensor([2, 2, 2]), np.ones((1, 2)), 1)
    assert list(out.reshape(-1, order="F")) == [3, 7, 11, 15]


def test_kat_select_order(port):  # test_hosvd.cpp:170-178
    assert port.select_order([10, 5, 20]) == [2, 1, 3]
    assert port.select_order([5, 5, 5]) == [1, 2, 3]
    assert port.select_order([7, 7, 2]) == [3, 1, 2]
