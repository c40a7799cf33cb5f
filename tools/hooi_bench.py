#!/usr/bin/env python3
"""HOOI refinement time on the B200 from the t-HOSVD-ALS warm start (the
paper's §6.3 downstream use), BASELINE configs 1 and 3, tensor resident.

  python tools/hooi_bench.py [--configs 1,3] > profiles/hooi_r01.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_02583_b200 as tk  # noqa: E402
from bench import ALS_SEED, CONFIGS, MAX_ITERS  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", default="1,3")
    args = p.parse_args()
    ctx = tk.Context(0)
    for cid in [int(x) for x in args.configs.split(",")]:
        c = CONFIGS[cid]
        dims, ranks = c["dims"], c["ranks"]
        host = torch.empty(int(np.prod(dims)), dtype=torch.float64, pin_memory=True)
        tk.synth_tucker(dims, ranks, c["alpha"], c["nu"], c["seed"], out=host.numpy())
        dev = host.to("cuda:0")
        torch.cuda.synchronize()
        dt = tk.DeviceTensor.from_torch(dev, dims)
        eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=c["eta"], max_iters=MAX_ITERS, seed=ALS_SEED))
        warm, rep = ctx.t_hosvd(dt, tk.Truncation(ranks), eng)
        for _ in range(2):  # second call timed (first warms the eigensolver workspace)
            t0 = time.perf_counter()
            out = ctx.hooi(dt, tk.Truncation(ranks), warm, tk.HooiConfig())
            sec = time.perf_counter() - t0
        print(json.dumps({"config": cid, "dims": dims, "ranks": ranks, "warm_rel_err": rep.relative_residual,
                          "hooi_rel_err": out.relative_residual, "iterations": out.iterations,
                          "converged": out.converged, "seconds": sec,
                          "ms_per_iteration": sec * 1e3 / max(1, out.iterations)}), flush=True)
        del dt, dev, host
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
