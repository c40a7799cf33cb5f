"""HOOI refinement (hooi.cpp:53-110) on the B200 against
the compiled reference (oracle/_ref): same warm start, same stop rule.

Per iteration and mode the device contracts the tensor with the other
factors (the FC kernels), takes the leading left singular vectors of the
shrunk unfolding from its Gram matrix (gram.cu + the eigensolver, the
reference's order and signs), and evaluates the explicit fit with the fused
expansion-difference pass. Factors are determined column by column, so they
are compared column by column; fits to 1e-12."""
import numpy as np
import pytest

import paper_2004_02583_b200 as tk
from oracles import Ref, random_tensor
from parity import CORE_SV_REL_TOL, column_diff, ortho_defect

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return tk.Context(0)


@pytest.fixture(scope="module")
def ref():
    r = Ref()
    r.set_threads(r.max_threads())
    return r


def warm(ref, a, ranks, kind="svd", sequential=True):
    r = ref.hosvd_exact(a, ranks, kind, sequential=sequential)
    return tk.TuckerTensor(r.core, [np.asfortranarray(u) for u in r.factors], tuple(a.shape)), r


@pytest.mark.parametrize("dims,ranks,nu,alpha", [([30, 30, 30], [5, 5, 5], 1e-3, 0.0),
                                                 ([40, 35, 30], [6, 4, 5], 1e-2, 1.0),
                                                 ([24, 20, 16, 12], [4, 3, 5, 2], 1e-2, 0.0),
                                                 ([128, 128, 128], [10, 10, 10], 1e-2, 0.0)], ids=str)
def test_hooi_matches_reference(ctx, ref, dims, ranks, nu, alpha):
    a = tk.synth_tucker(dims, ranks, alpha, nu, 801).reshape(dims, order="F")
    init, _ = warm(ref, a, ranks)
    out = ctx.hooi(a, tk.Truncation(ranks), init, tk.HooiConfig())
    core, factors, iters, conv, fits = ref.hooi(a, ranks, init.core, init.factors)
    assert out.iterations == iters and out.converged == conv
    assert np.max(np.abs(np.array(out.fit_history) - np.array(fits))) <= 1e-12
    for u, v in zip(out.tucker.factors, factors):
        assert column_diff(u, v) <= 1e-8
        assert ortho_defect(u) <= 1e-12
    assert np.max(np.abs(out.tucker.core - core)) <= CORE_SV_REL_TOL * np.max(np.abs(core))


def test_hooi_random_problems_track_reference(ctx, ref):
    # test_hooi.cpp "fit is nondecreasing on a batch of random problems"
    shapes = [[6, 7, 8], [9, 5, 6], [7, 7, 7], [5, 8, 6], [4, 6, 9]]
    for seed in range(10):
        dims = shapes[seed % len(shapes)]
        t = random_tensor(ref, dims, 7100 + seed)
        init, _ = warm(ref, t, [2, 3, 2])
        cfg = tk.HooiConfig(max_iters=15)
        out = ctx.hooi(t, tk.Truncation([2, 3, 2]), init, cfg)
        _, _, iters, conv, fits = ref.hooi(t, [2, 3, 2], init.core, init.factors, max_iters=15)
        f = out.fit_history
        assert all(f[k + 1] >= f[k] - 1e-12 for k in range(len(f) - 1))
        assert len(f) == out.iterations + 1
        n = min(len(f), len(fits))
        assert np.max(np.abs(np.array(f[:n]) - np.array(fits[:n]))) <= 1e-10
        assert max(ortho_defect(u) for u in out.tucker.factors) <= 1e-12


def test_hooi_optimal_warm_start_converges_in_one_iteration(ctx, ref):
    # test_hooi.cpp:53-66 (exact Tucker tensor)
    dims, ranks = [10, 9, 8], [3, 2, 3]
    a = tk.synth_tucker(dims, ranks, 0.0, 0.0, 700).reshape(dims, order="F")
    init, r = warm(ref, a, ranks)
    assert r.relative_residual <= 1e-10
    out = ctx.hooi(a, tk.Truncation(ranks), init)
    assert out.converged and out.iterations == 1
    assert len(out.fit_history) == 2 and abs(out.fit_history[0] - 1.0) <= 1e-10


def test_hooi_iteration_cap_is_a_status(ctx, ref):
    # test_hooi.cpp:141-153
    t = random_tensor(ref, [7, 8, 6], 703)
    init, _ = warm(ref, t, [2, 2, 2])
    out = ctx.hooi(t, tk.Truncation([2, 2, 2]), init, tk.HooiConfig(tol=1e-300, max_iters=3))
    assert not out.converged and out.iterations == 3 and len(out.fit_history) == 4


def test_hooi_warm_starts_land_together(ctx, ref):
    # test_hooi.cpp:100-139 / acceptance C8: every warm start refines to one residual
    dims, ranks = [30, 30, 30], [5, 5, 5]
    a = tk.synth_tucker(dims, ranks, 0.0, 1e-3, 801).reshape(dims, order="F")
    finals, warms = [], []
    for seq in (False, True):
        for eng in (tk.FactorEngine.svd(), tk.FactorEngine.eig(),
                    tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-4, seed=13))):
            if seq:
                init, rep = ctx.st_hosvd(a, tk.Truncation(ranks), None, eng)
            else:
                init, rep = ctx.t_hosvd(a, tk.Truncation(ranks), eng)
            out = ctx.hooi(a, tk.Truncation(ranks), init)
            finals.append(1.0 - out.fit_history[-1])
            warms.append(rep.relative_residual)
    assert max(finals) - min(finals) <= 1e-8
    assert max(finals) <= min(warms) + 1e-12


def test_hooi_conformance_guards(ctx, ref):
    # test_hooi.cpp:175-192
    t = random_tensor(ref, [6, 6, 6], 705)
    init, _ = warm(ref, t, [2, 2, 2])
    with pytest.raises(tk.DimensionMismatchError):
        ctx.hooi(t, tk.Truncation([3, 2, 2]), init)
    other = random_tensor(ref, [6, 6, 5], 706)
    with pytest.raises(tk.DimensionMismatchError):
        ctx.hooi(other, tk.Truncation([2, 2, 2]), init)
    init2, _ = warm(ref, t, [5, 1, 1])
    with pytest.raises(tk.RankTooLargeError):
        ctx.hooi(t, tk.Truncation([5, 1, 1]), init2)
    with pytest.raises(tk.ZeroReferenceError):
        ctx.hooi(np.zeros((6, 6, 6), order="F"), tk.Truncation([2, 2, 2]), init)
