"""One rank of a multi-process sharded decomposition (test helper for
test_gpu_dist_procs.py): attaches to the POSIX shm group `name` with
ShardedContext.shm on cuda:0, decomposes its slab of the seeded tensor and
saves core, factors and report fields to `out` (npz).

  python tests/dist_worker.py NAME RANK WORLD KIND DIMS RANKS SEED OUT
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2004_02583_b200 as tk  # noqa: E402
from paper_2004_02583_b200 import dist as tkd  # noqa: E402


def main():
    name, rank, world, kind, dims, ranks, seed, out = sys.argv[1:9]
    rank, world, seed = int(rank), int(world), int(seed)
    dims = [int(x) for x in dims.split(",")]
    ranks = [int(x) for x in ranks.split(",")]
    a = tk.synth_tucker(dims, ranks, 0.5, 1e-3, seed).reshape(dims, order="F")
    slab = np.asfortranarray(tkd.slab_of(a, rank, world))
    sc = tkd.ShardedContext.shm(0, name, rank, world, slot_bytes=1 << 20)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=1e-9, seed=7, max_iters=50))
    if kind == "t":
        tkr, rep = sc.t_hosvd(slab, dims, tk.Truncation(ranks), eng)
    else:
        tkr, rep = sc.st_hosvd(slab, dims, tk.Truncation(ranks), None, eng)
    np.savez(out, core=tkr.core, rel=rep.relative_residual,
             iters=np.array([[p.mode, p.als.iterations] for p in rep.per_mode]),
             **{f"u{k}": u for k, u in enumerate(tkr.factors)})
    sc.close()


if __name__ == "__main__":
    main()
