#!/usr/bin/env python3
"""Per-kernel throughput of the FC / FR contractions on the BASELINE shapes
(device-resident random tensors, CUDA events via tkg_bench_contractions).

  python tools/kernel_bench.py [--reps 5] [--only c3m1,...]
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2004_02583_b200 as tk  # noqa: E402
from paper_2004_02583_b200 import _lib  # noqa: E402

CASES = {
    "c1m1": ([256, 256, 256], 1, 10), "c1m2": ([256, 256, 256], 2, 10), "c1m3": ([256, 256, 256], 3, 10),
    "c2m1": ([96, 96, 96, 96], 1, 10), "c2m2": ([10, 96, 96, 96], 2, 10), "c2m3": ([10, 10, 96, 96], 3, 10),
    "c3m1": ([1024, 1024, 1024], 1, 32), "c3m2": ([1024, 1024, 1024], 2, 32),
    "c3m3": ([1024, 1024, 1024], 3, 32),
    "c4m3": ([2048, 2048, 512], 3, 32), "c4m1": ([2048, 2048, 32], 1, 64),
    "c5m1": ([200, 200, 200, 200], 1, 50), "c5m2": ([50, 200, 200, 200], 2, 50),
}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--only", default="")
    args = p.parse_args()
    import torch
    ctx = tk.Context(0)
    l = _lib.lib()
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                                        "microbench_fp64.json")))
    p64 = peaks["dmma_m8n8k4_tflops"]
    bw = 6557.8
    sel = [k for k in CASES if not args.only or k in args.only.split(",")]
    maxn = max(int(np.prod(CASES[k][0])) for k in sel)
    buf = torch.randn(maxn, dtype=torch.float64, device="cuda")
    out = []
    for name in sel:
        dims, mode, r = CASES[name]
        n = int(np.prod(dims))
        ms = (C.c_double * 5)()
        err = _lib.TkgError()
        rc = l.tkg_bench_contractions(ctx._ctx, C.c_void_p(buf.data_ptr()), len(dims), _lib.u64(dims),
                                      mode, r, args.reps, ms, C.byref(err))
        if rc:
            print(name, "error", err.message.decode())
            continue
        I = dims[mode - 1]
        F = n // I
        bytes_ = 8 * (n + F * r + I * r)
        flops = 2 * n * r
        tmin = max(bytes_ / (bw * 1e9), flops / (p64 * 1e12)) * 1e3
        row = {"case": name, "dims": dims, "mode": mode, "r": r}
        for k, nm in enumerate(["fc", "fr", "init_sq", "init"]):
            t = ms[k]
            row[nm] = {"ms": round(t, 4), "GB/s": round(bytes_ / t / 1e6, 1),
                       "TF/s": round(flops / t / 1e9, 2), "roof_frac": round(tmin / t, 3)}
        if ms[4] > 0:  # fused sweep pass: FC + FR work from one read of the tensor
            t = ms[4]
            row["sweep"] = {"ms": round(t, 4), "GB/s": round(bytes_ / t / 1e6, 1), "TF/s": round(2 * flops / t / 1e9, 2),
                            "roof_frac": round(max(bytes_ / (bw * 1e9), 2 * flops / (p64 * 1e12)) * 1e3 / t, 3)}
        row["bound_ms"] = round(tmin, 4)
        out.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
