#!/usr/bin/env python3
"""ALS vs EIG vs SVD factor engines on the B200 (the paper's engine comparison,
PAPER.md:673-700, on the BASELINE shapes): t-/st-HOSVD time-to-solution per
engine, device-resident tensor, CUDA-event timing on the library stream.

  python tools/engine_bench.py [--configs 1,2,3] [--reps 3] > profiles/engines_r01.jsonl

Every engine's result is also checked against the ALS one (relative error
within 1e-6, factor subspaces within 1e-4) so a fast wrong engine cannot
report a time.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import paper_2004_02583_b200 as tk  # noqa: E402
from bench import ALS_SEED, CONFIGS, MAX_ITERS  # noqa: E402
from parity import principal_sine  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", default="1,2,3")
    p.add_argument("--reps", type=int, default=3)
    args = p.parse_args()
    ctx = tk.Context(0)
    for cid in [int(x) for x in args.configs.split(",")]:
        c = CONFIGS[cid]
        dims, ranks = c["dims"], c["ranks"]
        n = int(np.prod(dims))
        host = torch.empty(n, dtype=torch.float64, pin_memory=True)
        tk.synth_tucker(dims, ranks, c["alpha"], c["nu"], c["seed"], out=host.numpy())
        dev = host.to("cuda:0")
        torch.cuda.synchronize()
        dt = tk.DeviceTensor.from_torch(dev, dims)
        engines = {"als": tk.FactorEngine.with_als(tk.AlsConfig(eta=c["eta"], max_iters=MAX_ITERS, seed=ALS_SEED)),
                   "eig": tk.FactorEngine.eig(), "svd": tk.FactorEngine.svd()}
        base = None
        for name, eng in engines.items():
            def call():
                if c["kind"] == "t":
                    return ctx.t_hosvd(dt, tk.Truncation(ranks), eng)
                return ctx.st_hosvd(dt, tk.Truncation(ranks), None, eng)
            tkr, rep = call()  # warm-up
            times = []
            for _ in range(args.reps):
                ctx.flush_l2()
                ctx.timer_start()
                tkr, rep = call()
                times.append(ctx.timer_stop())
            if base is None:
                base = (tkr, rep)
            sine = max(principal_sine(u, v) for u, v in zip(tkr.factors, base[0].factors))
            ok = abs(rep.relative_residual - base[1].relative_residual) <= 1e-6 and sine <= 1e-4
            print(json.dumps({"config": cid, "driver": c["kind"] + "-HOSVD", "engine": name,
                              "dims": dims, "ranks": ranks, "ms_median": float(np.median(times)),
                              "time_to_solution_s": rep.seconds, "relative_residual": rep.relative_residual,
                              "max_sine_vs_als": sine, "agrees_with_als": bool(ok),
                              "kernel_launches": rep.kernel_launches}), flush=True)
        del dt, dev, host
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
