#!/usr/bin/env python3
"""One decomposition step of a BASELINE config on a device-resident tensor
(for ncu launch lists / full captures). Generates the tensor on the GPU with
torch (values irrelevant for timing), runs `--warm` untimed steps then one."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2004_02583_b200 as tk  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=3)
    p.add_argument("--warm", type=int, default=1)
    p.add_argument("--synth", action="store_true", help="use the seeded generator (slow) instead of torch.randn")
    a = p.parse_args()
    import torch
    c = bench.CONFIGS[a.config]
    dims, ranks = c["dims"], c["ranks"]
    n = int(np.prod(dims))
    if a.synth:
        host, buf = bench.make_tensor(c, dims, pinned=True)
        dev = buf.cuda()
    else:
        dev = torch.randn(n, dtype=torch.float64, device="cuda")
    ctx = tk.Context(0)
    dt = tk.DeviceTensor.from_torch(dev, dims)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=c["eta"], max_iters=8, seed=7))
    for _ in range(a.warm + 1):
        if c["kind"] == "t":
            _, rep = ctx.t_hosvd(dt, tk.Truncation(ranks), eng)
        else:
            _, rep = ctx.st_hosvd(dt, tk.Truncation(ranks), None, eng)
    print("seconds", rep.seconds, "iters", [(m.mode, m.als.iterations) for m in rep.per_mode])


if __name__ == "__main__":
    main()
