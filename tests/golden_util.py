"""Loaders for the reference-generated fixtures in tests/golden/."""
from __future__ import annotations

import functools
import gzip
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

COSTS = {
    "default": {"t_load_s": 3e-3, "t_compute_s": 158e-6, "loads_serial": True, "ml_score_cost_s": 0.0},
    "overlap_ml": {"t_load_s": 2.5e-3, "t_compute_s": 1.7e-4, "loads_serial": False,
                   "ml_score_cost_s": 1e-4},
}


@functools.lru_cache(maxsize=None)
def load(name: str) -> dict:
    with gzip.open(os.path.join(GOLDEN, name), "rt") as fh:
        return json.load(fh)


def case_trace(case):
    """(header (L,E,K), events list of (seq, phase, step, layer, experts))."""
    if "trace" in case:
        _, L, E, K = case["trace"]["header"]
        return (L, E, K), [tuple(e) for e in case["trace"]["events"]]
    z = np.load(os.path.join(GOLDEN, case["trace_npz"]))
    ids = z["ids"]
    T, L, K = ids.shape
    E = int(z["header"][1])
    return (L, E, K), [(0, 1, t, l, ids[t, l].tolist()) for t in range(T) for l in range(L)]


def big_ids(case):
    z = np.load(os.path.join(GOLDEN, case["trace_npz"]))
    return z["ids"], int(z["header"][1])


def policy_name(spec):
    return spec if isinstance(spec, str) else spec["name"]


def include_prefill(spec):
    return True if isinstance(spec, str) else spec.get("include_prefill", True)
