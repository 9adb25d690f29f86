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


def lecar_params(spec):
    """LeCaR keyword parameters of a policy spec (policies.py:333-341)."""
    if isinstance(spec, str):
        return {}
    return {k: spec[k] for k in ("learning_rate", "discount_base", "seed") if k in spec}


M64 = (1 << 64) - 1
HASH_MUL = 0x100000001B3
FNV_OFF = 0xCBF29CE484222325


def poly_hash(codes) -> int:
    """The CUDA engine's spliceable decision hash: h = h * P + code + 1 mod 2^64."""
    h = 0
    for c in codes:
        h = (h * HASH_MUL + int(c) + 1) & M64
    return h


def fnv_hash(codes) -> int:
    """FNV-1a 64 over the u16 outcome codes (the fixtures' hash, make_golden.py)."""
    h = FNV_OFF
    for c in codes:
        for b in (int(c) & 0xFF, int(c) >> 8):
            h = ((h ^ b) * HASH_MUL) & M64
    return h


_POLY_CACHE: dict = {}


def expected_poly_hashes(case, run_index: int) -> list:
    """Per-layer poly hashes of the reference's decisions for one golden run.

    From the recorded decisions when the fixture has them (checked against the
    fixture's FNV hashes first); otherwise from the C oracle, whose FNV hashes
    must equal the fixture's (the oracle is the reference's restatement)."""
    key = (case["name"], run_index)
    if key in _POLY_CACHE:
        return _POLY_CACHE[key]
    import oracle
    run = case["runs"][run_index]
    if "decisions" in run:
        assert [format(fnv_hash(d), "016x") for d in run["decisions"]] == run["hashes"]
        out = [poly_hash(d) for d in run["decisions"]]
    else:
        header, events = case_trace(case)
        L, E, _ = header
        name = policy_name(run["policy"])
        nets = oracle.nets_from_spec(run["nets"], L, E, GOLDEN) if name == "ml" else None
        kw = dict(cost=COSTS[run["cost"]], window=run["window"], nets=nets,
                  include_prefill=include_prefill(run["policy"]))
        _, fnv, _ = oracle.simulate(header, events, name, run["capacity"], **kw)
        assert [format(h, "016x") for h in fnv] == run["hashes"]
        _, out, _ = oracle.simulate(header, events, name, run["capacity"], hash_kind="poly", **kw)
    _POLY_CACHE[key] = out
    return out
