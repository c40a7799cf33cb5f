"""Sharded decomposition (tensor split along its last mode) on one device:
`world` ranks are host threads of this process, each with its own context,
joined by the in-process communicator (host-synchronous collectives), so the
whole distributed code path runs -- per-shard initializer windows, the
summed left-update partials / Gram matrices / norms, the all-to-all that
moves the sharded mode, the summed core and residual -- without ranks whose
kernels wait on one another. Every rank must return the reference's result
(golden fixtures, BASELINE tolerances, identical iteration counts) and the
single-GPU result."""
import threading

import numpy as np
import pytest

import paper_2004_02583_b200 as tk
from paper_2004_02583_b200 import dist as tkd
from golden_io import Fixture, fixtures
from parity import (ANGLE_TOL, CORE_SV_REL_TOL, REL_ERR_ABS_TOL, column_diff, core_sv_rel_diff,
                    ortho_defect, principal_sine)

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


def run_ranks(world, fn):
    group = tkd.LocalGroup(world)
    ctxs = [tkd.ShardedContext.local(0, group, r) for r in range(world)]
    out = [None] * world
    errs = []

    def work(r):
        try:
            out[r] = fn(ctxs[r], r)
        except BaseException as e:  # noqa: BLE001 - reported below
            errs.append((r, e))

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=200)
    if errs:
        raise RuntimeError("; ".join(f"rank {r}: {type(e).__name__}: {e}" for r, e in errs)) from errs[0][1]
    assert not any(t.is_alive() for t in th), "a rank did not finish" 
    for c in ctxs:
        c.close()
    return out


def check_same(a, b):
    """Two ranks' replicated results: identical bits."""
    (ta, ra), (tb, rb) = a, b
    assert np.array_equal(ta.core, tb.core)
    for u, v in zip(ta.factors, tb.factors):
        assert np.array_equal(u, v)
    assert ra.relative_residual == rb.relative_residual
    assert [p.als.iterations for p in ra.per_mode] == [p.als.iterations for p in rb.per_mode]


def check_reference(tkr, rep, fx):
    assert [p.mode for p in rep.per_mode] == fx.modes
    assert [p.als.iterations for p in rep.per_mode] == fx.iterations
    for p, h in zip(rep.per_mode, fx.histories):
        assert np.allclose(p.als.residual_history, h, rtol=1e-9, atol=0)
    assert abs(rep.relative_residual - fx.relative_residual) <= REL_ERR_ABS_TOL
    for u, v in zip(tkr.factors, fx.factors):
        assert principal_sine(u, v) <= ANGLE_TOL
        assert ortho_defect(u) <= 1e-12
    assert core_sv_rel_diff(tkr.core, fx.core) <= CORE_SV_REL_TOL


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", fixtures())
def test_sharded_matches_reference_fixture(name, world):
    fx = Fixture(name)
    m = fx.meta
    dims = tuple(fx.tensor.shape)
    if min(dims) < world:
        pytest.skip("extent below the number of ranks")
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=m["eta"], seed=m["seed"], max_iters=50))

    def fn(sc, r):
        slab = tkd.slab_of(fx.tensor, r, world)
        if m["sequential"]:
            order = tk.ModeOrder(m["order"]) if m["order"] else None
            return sc.st_hosvd(slab, dims, tk.Truncation(fx.ranks), order, eng)
        return sc.t_hosvd(slab, dims, tk.Truncation(fx.ranks), eng,
                          bool(m.get("want_singular_vectors")))

    res = run_ranks(world, fn)
    for r in range(1, world):
        check_same(res[0], res[r])
    check_reference(*res[0], fx)
    if m.get("want_singular_vectors"):
        tkr = res[0][0]
        for u, v in zip(tkr.factors, fx.factors):
            assert column_diff(u, v) <= ANGLE_TOL
        assert np.max(np.abs(tkr.core - fx.core)) <= CORE_SV_REL_TOL * np.max(np.abs(fx.core))


def _synthetic(dims, ranks, noise, seed):
    rng = np.random.default_rng(seed)
    core = rng.standard_normal(ranks)
    a = core
    for n, (i, r) in enumerate(zip(dims, ranks)):
        q, _ = np.linalg.qr(rng.standard_normal((i, r)))
        a = np.moveaxis(np.tensordot(q, np.moveaxis(a, n, 0), axes=(1, 0)), 0, n)
    a = a + noise * np.linalg.norm(a) / np.sqrt(a.size) * rng.standard_normal(dims)
    return np.asfortranarray(a)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("sequential,order", [(False, None), (True, None), (True, [3, 1, 2]),
                                              (True, [2, 3, 1])])
def test_sharded_matches_single_gpu(world, sequential, order):
    dims, ranks = (60, 50, 41), [6, 5, 7]
    a = _synthetic(dims, ranks, 1e-3, 5)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-10, seed=11, max_iters=50))
    ctx = tk.Context(0)
    mo = tk.ModeOrder(order) if order else None
    if sequential:
        ref_t, ref_r = ctx.st_hosvd(a, tk.Truncation(ranks), mo, eng)
    else:
        ref_t, ref_r = ctx.t_hosvd(a, tk.Truncation(ranks), eng)
    ctx.close()

    def fn(sc, r):
        slab = tkd.slab_of(a, r, world)
        if sequential:
            return sc.st_hosvd(slab, dims, tk.Truncation(ranks), mo, eng)
        return sc.t_hosvd(slab, dims, tk.Truncation(ranks), eng)

    res = run_ranks(world, fn)
    for r in range(1, world):
        check_same(res[0], res[r])
    tkr, rep = res[0]
    assert [p.als.iterations for p in rep.per_mode] == [p.als.iterations for p in ref_r.per_mode]
    assert abs(rep.relative_residual - ref_r.relative_residual) <= REL_ERR_ABS_TOL
    for u, v in zip(tkr.factors, ref_t.factors):
        assert principal_sine(u, v) <= ANGLE_TOL
    assert core_sv_rel_diff(tkr.core, ref_t.core) <= CORE_SV_REL_TOL


def test_sharded_device_slab_and_errors():
    dims, ranks = (30, 20, 16), [4, 3, 5]
    a = _synthetic(dims, ranks, 1e-3, 9)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-9, seed=3))
    import torch

    def fn(sc, r):
        slab = tkd.slab_of(a, r, 2)
        dev = torch.from_numpy(slab.reshape(-1, order="F").copy()).cuda()
        out = sc.t_hosvd(tk.DeviceTensor.from_torch(dev, slab.shape), dims, tk.Truncation(ranks), eng)
        # a slab that is not the balanced split is a usage error
        wrong = tkd.slab_of(a, 1 - r, 2) if dims[-1] % 2 else np.asfortranarray(a[..., :dims[-1] // 2 + 1])
        with pytest.raises(tk.DimensionMismatchError):
            sc.t_hosvd(wrong, dims, tk.Truncation(ranks), eng)
        return out

    res = run_ranks(2, fn)
    check_same(res[0], res[1])


def test_nccl_world1_matches_single_gpu():
    """The NCCL communicator (dlopen'd libnccl) on one rank: every collective
    of the sharded path runs through NCCL on the context's stream."""
    dims, ranks = (40, 30, 20), [10, 10, 5]
    a = _synthetic(dims, ranks, 1e-3, 21)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-9, seed=7))
    ctx = tk.Context(0)
    ref_t, ref_r = ctx.t_hosvd(a, tk.Truncation(ranks), eng)
    ref_st, ref_sr = ctx.st_hosvd(a, tk.Truncation(ranks), None, eng)
    ctx.close()
    sc = tkd.ShardedContext.nccl(0, 0, 1, tkd.nccl_unique_id())
    for (t, r), (rt, rr) in [(sc.t_hosvd(a, dims, tk.Truncation(ranks), eng), (ref_t, ref_r)),
                             (sc.st_hosvd(a, dims, tk.Truncation(ranks), None, eng), (ref_st, ref_sr))]:
        assert [p.als.iterations for p in r.per_mode] == [p.als.iterations for p in rr.per_mode]
        assert abs(r.relative_residual - rr.relative_residual) <= REL_ERR_ABS_TOL
        for u, v in zip(t.factors, rt.factors):
            assert principal_sine(u, v) <= ANGLE_TOL
        assert core_sv_rel_diff(t.core, rt.core) <= CORE_SV_REL_TOL
    sc.close()
