"""Loader for the committed golden fixtures (tests/golden/, produced by
tests/golden/make_golden.py from the compiled reference)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def index():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)


def streams():
    with open(os.path.join(GOLDEN, "streams.json")) as f:
        return json.load(f)


def long_stream():
    d = np.load(os.path.join(GOLDEN, "uniform01_11_4.npz"))
    return d["idx"], d["val"], float(d["checksum"])


class Fixture:
    def __init__(self, name):
        self.name = name
        meta = index()[name]
        self.meta = meta
        d = np.load(os.path.join(GOLDEN, f"hosvd_{name}.npz"))
        self.dims = [int(x) for x in d["dims"]]
        self.ranks = [int(x) for x in d["ranks"]]
        self.tensor = d["tensor"].reshape(self.dims, order="F")
        self.core = d["core"].reshape(self.ranks, order="F")
        self.factors = [d[f"factor{k + 1}"].reshape((self.dims[k], self.ranks[k]), order="F")
                        for k in range(len(self.dims))]
        self.modes = [int(x) for x in d["modes"]]
        self.iterations = [int(x) for x in d["iterations"]]
        self.status = [int(x) for x in d["status"]]
        self.histories = [list(d[f"history{k}"]) for k in range(len(self.dims))]
        self.relative_residual = float(d["relative_residual"])


def fixtures():
    return list(index().keys())
