"""Loader for tests/golden fixtures (generated from the compiled reference by
tests/golden/make_golden.py).  Rebuilds each case's K/V from the committed
inputs + the deterministic counter-based generator."""
import json
import os

import numpy as np

from paper_2604_16883_b200.workload import WorkloadSpec

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_cases():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        index = json.load(f)["cases"]
    out = []
    for meta in index:
        z = np.load(os.path.join(GOLDEN, meta["name"] + ".npz"))
        if meta["kind"] == "planted":
            spec = WorkloadSpec(**meta["spec"])
            k, v = spec.host_cache(0)
        else:
            k, v = z["k"], z["v"]
        out.append((meta, k, v, z))
    return out


def case_ids():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return [c["name"] for c in json.load(f)["cases"]]
