"""The device-side sweep loop (TKG_GRAPH=1: one CUDA graph per mode with a
WHILE node whose condition the finish step sets, Engine::run_als; t-HOSVD then
runs its independent modes concurrently, one stream and buffer set each)
against the default host-batched sweeps: the same kernels, so factors and core
must be bit-identical (concurrent t-HOSVD modes take ||A||^2 from mode 1's
init pass, as the sequential driver does), and so must the iteration counts,
statuses, residual histories and error paths."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2004_02583_b200 as tk

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [("t", [40, 30, 24], [5, 4, 3], 1e-9, 50), ("st", [24, 20, 16, 12], [4, 3, 5, 2], 1e-9, 50),
         ("t", [60, 50, 40], [6, 5, 4], 0.0, 7), ("st", [200, 40, 30], [50, 10, 8], 1e-10, 50)]

_SCRIPT = r"""
import json, sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2004_02583_b200 as tk
cases = json.loads(sys.argv[2])
out = []
ctx = tk.Context(0)
for kind, dims, ranks, eta, its in cases:
    a = tk.synth_tucker(dims, ranks, 0.5, 1e-3, 99 + sum(dims)).reshape(dims, order="F")
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=eta, seed=7, max_iters=its))
    for rep_ in range(2):  # the second call reuses the cached graphs
        if kind == "t":
            tkr, rep = ctx.t_hosvd(a, tk.Truncation(ranks), eng)
        else:
            tkr, rep = ctx.st_hosvd(a, tk.Truncation(ranks), None, eng)
    out.append({"core": tkr.core.ravel(order="F").tolist(), "rel": rep.relative_residual,
                "factors": [u.ravel(order="F").tolist() for u in tkr.factors],
                "modes": [[m.mode, m.als.iterations, m.als.status, m.als.residual_history] for m in rep.per_mode]})
try:
    ctx.als_low_rank(np.asfortranarray(np.outer(np.arange(1.0, 7.0), np.ones(5)).reshape(6, 5, 1)), 1, 2,
                     tk.AlsConfig(eta=1e-12, seed=1))
    out.append("no error")
except tk.Error as e:
    out.append(type(e).__name__ + ": " + str(e))
print(json.dumps(out))
"""


def run(graph):
    env = dict(os.environ, TKG_GRAPH="1" if graph else "0")
    r = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT, json.dumps(CASES)], capture_output=True, text=True,
                       env=env, timeout=500)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_graph_loop_matches_host_batches():
    g, h = run(True), run(False)
    assert len(g) == len(h)
    for a, b in zip(g[:-1], h[:-1]):
        assert a["modes"] == b["modes"]
        assert a["rel"] == b["rel"]
        assert np.array_equal(np.array(a["core"]), np.array(b["core"]))
        for u, v in zip(a["factors"], b["factors"]):
            assert np.array_equal(np.array(u), np.array(v))
    # the capped case (eta = 0) never ran past max_iters = 7; a mode stops
    # earlier only when two residuals are bitwise equal (|prev - res| = 0)
    assert all(m[1] <= 7 and (m[1] == 7 or m[2] == "converged") for m in g[2]["modes"])
    # (with the default kernels at least one mode of this case runs into the cap; other
    # kernel selections, e.g. TKG_FUSED_SWEEP=1, may reach a bitwise-stationary residual first)
    if os.environ.get("TKG_FUSED_SWEEP") != "1":
        assert any(m[2] == "max_iters_reached" for m in g[2]["modes"])
    assert g[-1] == h[-1]
