#!/usr/bin/env python3
"""Regenerate the golden fixtures from the compiled, unmodified reference
(oracle/_ref/libtenkit_ref.so, built from /root/reference/proj/src by
oracle/Makefile). Run in the build container (the GPU box has no
/root/reference); the .npz files are committed.

  python tests/golden/make_golden.py

Inputs are generated with the reference's own seeded builders
(tests/helpers.hpp random_tensor / random_orthonormal semantics, via the
reference RNG) so every fixture is reproducible from its seeds as well.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracles import Ref, flat, random_orthonormal, random_tensor  # noqa: E402

CASES = [
    # name, dims, ranks, sequential, order, eta, seed, noise_seed
    ("t3_small", [9, 8, 7], [3, 2, 4], False, None, 1e-8, 7, 3),
    ("st3_small", [9, 8, 7], [3, 2, 4], True, None, 1e-8, 7, 3),
    ("st3_order", [12, 10, 8], [3, 5, 2], True, [3, 1, 2], 1e-6, 11, 5),
    ("t4", [12, 10, 8, 6], [3, 3, 2, 2], False, None, 1e-8, 7, 4),
    ("st4", [12, 10, 8, 6], [3, 3, 2, 2], True, None, 1e-8, 7, 4),
    ("t3_r10", [40, 30, 20], [10, 10, 5], False, None, 1e-8, 7, 9),
    ("st3_r10", [40, 30, 20], [10, 10, 5], True, None, 1e-8, 7, 9),
    ("t3_tight", [30, 28, 26], [6, 5, 4], False, None, 1e-12, 2004, 12),
]
# t_hosvd with want_singular_vectors (hosvd.cpp:100-106, recover_singular_vectors :65-72)
CASES_SV = [
    ("t3_sv", [40, 30, 20], [10, 10, 5], 1e-8, 7, 9),
    ("t4_sv", [12, 10, 8, 6], [3, 3, 2, 2], 1e-8, 7, 4),
    ("t3_sv_r40", [70, 60, 50], [40, 36, 8], 1e-8, 5, 21),
]


def save_if_changed(path, **arrays):
    """Rewrite a fixture only when its arrays change (keeps committed files stable)."""
    if os.path.exists(path):
        old = np.load(path)
        if set(old.files) == set(arrays) and all(np.array_equal(old[k], arrays[k]) for k in arrays):
            return
    np.savez_compressed(path, **arrays)


def tucker_input(ref, dims, ranks, seed):
    core = random_tensor(ref, ranks, seed)
    factors = [random_orthonormal(ref, dims[k], ranks[k], seed + 1 + k) for k in range(len(dims))]
    signal = ref.reconstruct(core, factors, dims)
    return 5.0 * signal + random_tensor(ref, dims, seed + 100)


def main():
    ref = Ref()
    ref.set_threads(1)
    index = {}
    cases = [c + (False,) for c in CASES] + [(n, d, r, False, None, e, s, z, True)
                                              for n, d, r, e, s, z in CASES_SV]
    for name, dims, ranks, seq, order, eta, seed, noise, want_sv in cases:
        a = tucker_input(ref, dims, ranks, noise)
        res = ref.hosvd_als(a, ranks, sequential=seq, order=order, eta=eta, seed=seed,
                            want_singular_vectors=want_sv)
        out = {"tensor": flat(a), "dims": np.array(dims), "ranks": np.array(ranks),
               "core": flat(res.core), "relative_residual": np.array(res.relative_residual),
               "modes": np.array([m.mode for m in res.per_mode]),
               "iterations": np.array([m.iterations for m in res.per_mode]),
               "status": np.array([m.status for m in res.per_mode]),
               "achieved_eta": np.array([m.achieved_eta for m in res.per_mode])}
        for k, u in enumerate(res.factors):
            out[f"factor{k + 1}"] = flat(u)
        for k, m in enumerate(res.per_mode):
            out[f"history{k}"] = np.array(m.residual_history)
        save_if_changed(os.path.join(HERE, f"hosvd_{name}.npz"), **out)
        index[name] = {"dims": dims, "ranks": ranks, "sequential": seq, "order": order, "eta": eta,
                       "seed": seed, "noise_seed": noise, "want_singular_vectors": want_sv,
                       "iterations": [int(m.iterations) for m in res.per_mode],
                       "relative_residual": res.relative_residual}
    # initializer streams: raw engine words and uniform01 draws
    streams = {}
    for seed, stream, n in [(0, 1, 64), (7, 3, 64), (2**40 + 5, 2, 64), (2004025833, 1, 64)]:
        streams[f"{seed}_{stream}"] = {"raw": [str(int(x)) for x in ref.engine_raw(seed, stream, n)],
                                       "uniform01": ref.uniform01(seed, stream, n).tolist()}
    # a longer stream crossing several jump-ahead chunks, stored sparsely
    long = ref.uniform01(11, 4, 3_000_000)
    picks = np.array([0, 1, 311, 312, 313, 623, 624, 8191, 8192, 65535, 65536, 262143, 262144,
                      1_000_003, 2_999_999])
    save_if_changed(os.path.join(HERE, "uniform01_11_4.npz"), idx=picks, val=long[picks],
                    checksum=np.array(float(np.sum(long))))
    with open(os.path.join(HERE, "streams.json"), "w") as f:
        json.dump(streams, f, indent=1)
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=1)
    print("wrote", len(index), "decomposition fixtures")


if __name__ == "__main__":
    main()
