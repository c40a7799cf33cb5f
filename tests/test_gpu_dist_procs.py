"""The sharded decomposition with one PROCESS per rank (the deployment
shape: per-process contexts, per-process engines), on the one GPU of the
test pool: ranks attach to a POSIX shared-memory group (ShmComm: host-staged
collectives behind a process-shared barrier, csrc/comm.cpp), so no kernel of
one rank waits on another's. Every rank must return bit-identical results,
the single-GPU result's iteration counts, and agree with it within the
BASELINE tolerances (the summation order of the sharded partials differs)."""
import os
import subprocess
import sys
import uuid

import numpy as np
import pytest

import paper_2004_02583_b200 as tk
from parity import ANGLE_TOL, CORE_SV_REL_TOL, REL_ERR_ABS_TOL, core_sv_rel_diff, principal_sine

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

HERE = os.path.dirname(os.path.abspath(__file__))


def run_procs(world, kind, dims, ranks, seed, tmp_path):
    name = f"/tkg_test_{uuid.uuid4().hex[:12]}"
    outs = [str(tmp_path / f"rank{r}.npz") for r in range(world)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "dist_worker.py"), name, str(r), str(world), kind,
                               ",".join(map(str, dims)), ",".join(map(str, ranks)), str(seed), outs[r]],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=400)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{logs[r]}"
    return [np.load(o) for o in outs]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind,dims,ranks", [("t", [40, 30, 24], [5, 4, 3]), ("st", [24, 20, 16, 12], [4, 3, 5, 2]),
                                             ("st", [30, 26, 22], [6, 5, 4])], ids=str)
def test_multiprocess_sharded_matches_single_gpu(tmp_path, world, kind, dims, ranks):
    seed = 2004 + sum(dims)
    res = run_procs(world, kind, dims, ranks, seed, tmp_path)
    # replicated results: identical bits on every rank
    for r in res[1:]:
        assert np.array_equal(r["core"], res[0]["core"])
        assert float(r["rel"]) == float(res[0]["rel"])
        assert np.array_equal(r["iters"], res[0]["iters"])
        for k in range(len(dims)):
            assert np.array_equal(r[f"u{k}"], res[0][f"u{k}"])
    # the single-GPU result of the whole tensor
    ctx = tk.Context(0)
    a = tk.synth_tucker(dims, ranks, 0.5, 1e-3, seed).reshape(dims, order="F")
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-9, seed=7, max_iters=50))
    if kind == "t":
        tkr, rep = ctx.t_hosvd(a, tk.Truncation(ranks), eng)
    else:
        tkr, rep = ctx.st_hosvd(a, tk.Truncation(ranks), None, eng)
    r0 = res[0]
    assert [list(x) for x in r0["iters"]] == [[p.mode, p.als.iterations] for p in rep.per_mode]
    assert abs(float(r0["rel"]) - rep.relative_residual) <= REL_ERR_ABS_TOL
    for k, u in enumerate(tkr.factors):
        assert principal_sine(r0[f"u{k}"], u) <= ANGLE_TOL
    assert core_sv_rel_diff(r0["core"], tkr.core) <= CORE_SV_REL_TOL
