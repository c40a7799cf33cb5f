"""The B200 path against the committed golden fixtures (reference outputs
recorded by tests/golden/make_golden.py): BASELINE tolerances on every
fixture, bitwise initializer streams."""
import numpy as np
import pytest

import paper_2004_02583_b200 as tk
from golden_io import Fixture, fixtures, long_stream, streams
from parity import (ANGLE_TOL, CORE_SV_REL_TOL, REL_ERR_ABS_TOL, column_diff, core_sv_rel_diff,
                    ortho_defect, principal_sine)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return tk.Context(0)


@pytest.mark.parametrize("name", fixtures())
def test_gpu_matches_reference_fixture(ctx, name):
    fx = Fixture(name)
    m = fx.meta
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=m["eta"], seed=m["seed"], max_iters=50))
    if m["sequential"]:
        order = tk.ModeOrder(m["order"]) if m["order"] else None
        tkr, rep = ctx.st_hosvd(fx.tensor, tk.Truncation(fx.ranks), order, eng)
    else:
        tkr, rep = ctx.t_hosvd(fx.tensor, tk.Truncation(fx.ranks), eng,
                               bool(m.get("want_singular_vectors")))
    if m.get("want_singular_vectors"):
        # singular vectors are determined column by column (dense_svd's sign
        # convention), and so is the core
        for u, v in zip(tkr.factors, fx.factors):
            assert column_diff(u, v) <= ANGLE_TOL
        assert np.max(np.abs(tkr.core - fx.core)) <= CORE_SV_REL_TOL * np.max(np.abs(fx.core))
    assert [p.mode for p in rep.per_mode] == fx.modes
    assert [p.als.iterations for p in rep.per_mode] == fx.iterations
    for p, h in zip(rep.per_mode, fx.histories):
        assert np.allclose(p.als.residual_history, h, rtol=1e-9, atol=0)
    assert abs(rep.relative_residual - fx.relative_residual) <= REL_ERR_ABS_TOL
    for u, v in zip(tkr.factors, fx.factors):
        assert principal_sine(u, v) <= ANGLE_TOL
        assert ortho_defect(u) <= 1e-12
    assert core_sv_rel_diff(tkr.core, fx.core) <= CORE_SV_REL_TOL


def test_gpu_streams_bitwise(ctx):
    for key, d in streams().items():
        seed, stream = (int(x) for x in key.split("_"))
        assert ctx.uniform01(seed, stream, len(d["uniform01"])).tolist() == d["uniform01"]


def test_gpu_long_stream(ctx):
    idx, val, checksum = long_stream()
    draws = ctx.uniform01(11, 4, 3_000_000)
    assert np.array_equal(draws[idx], val)
    assert float(np.sum(draws)) == checksum
