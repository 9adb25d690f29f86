"""GPU training data (dataset.build_training_data / mcb_training_data) against
the reference's build_training_data (dataset.py:35-96): full arrays on small
traces, SHA-256 of every layer's float64 features / float64 targets / masks
on the full-size C1 (48 x 128 x 8, 2048 tokens, capacity 32) and Mixtral 2K
(32 x 8 x 2, capacity 4) fixture traces (tests/golden/make_train_golden.py)."""
import hashlib
import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN

pytestmark = pytest.mark.gpu

import paper_2601_17063_b200 as mcb  # noqa: E402
from paper_2601_17063_b200 import dataset  # noqa: E402


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_small_cases_bit_exact():
    z = np.load(os.path.join(GOLDEN, "train_cases.npz"))
    meta = json.loads(str(z["meta"]))
    for m in meta["small"]:
        L, E, K = m["header"]
        ids = z[m["name"] + "_ids"]                       # [T][L][K]
        packed = mcb.packed_from_decode_ids(np.ascontiguousarray(ids.transpose(1, 0, 2)), E)
        ds = dataset.build_training_data(packed, m["capacity"], m["distance_cap"])
        for l in range(L):
            assert np.array_equal(ds[l].features, z[f"{m['name']}_f{l}"]), (m["name"], l)
            assert np.array_equal(ds[l].targets, z[f"{m['name']}_t{l}"]), (m["name"], l)
            assert np.array_equal(ds[l].masks, z[f"{m['name']}_m{l}"]), (m["name"], l)


@pytest.mark.parametrize("which", [0, 1])
def test_full_size_digests(which):
    z = np.load(os.path.join(GOLDEN, "train_cases.npz"))
    big = json.loads(str(z["meta"]))["big"][which]
    t = np.load(os.path.join(GOLDEN, big["trace_npz"]))
    ids = t["ids"]
    E = int(t["header"][1])
    packed = mcb.packed_from_decode_ids(np.ascontiguousarray(ids.transpose(1, 0, 2)), E)
    ds = dataset.build_training_data(packed, big["capacity"], big["distance_cap"])
    for l in range(ids.shape[1]):
        assert digest(ds[l].features) == big["features"][l], l
        assert digest(ds[l].targets) == big["targets"][l], l
        assert digest(ds[l].masks) == big["masks"][l], l


def test_general_traces_bit_exact():
    """Prefill + several sequences, include_prefill True / False, against the
    reference (tests/golden/make_train_general_golden.py)."""
    from golden_util import case_trace
    from paper_2601_17063_b200.trace import AccessEvent, Phase, RoutingTrace, TraceHeader
    z = np.load(os.path.join(GOLDEN, "train_general_cases.npz"))
    meta = json.loads(str(z["meta"]))
    for m in meta["small"]:
        header, events = case_trace({"trace": m["trace"]})
        L, E, K = header
        tr = RoutingTrace(TraceHeader("g", L, E, K),
                          tuple(AccessEvent(s, Phase(p), t, l, tuple(x)) for s, p, t, l, x in events))
        ds = dataset.build_training_data(tr, m["capacity"], m["distance_cap"], include_prefill=m["include_prefill"])
        for l in range(L):
            assert np.array_equal(ds[l].features, z[f"{m['name']}_f{l}"]), (m["name"], l)
            assert np.array_equal(ds[l].targets, z[f"{m['name']}_t{l}"]), (m["name"], l)
            assert np.array_equal(ds[l].masks, z[f"{m['name']}_m{l}"]), (m["name"], l)


def test_efficacy_training_traces_digests():
    """The reference's efficacy training data (test_acceptance.py:223-275): 3 traces
    x 8 sequences x (32 prefill + 2500 decode) tokens, E=64, capacity 64; traces from
    the bit-exact GPU generator."""
    from paper_2601_17063_b200 import refgen
    from paper_2601_17063_b200.trace import TraceHeader
    z = np.load(os.path.join(GOLDEN, "train_general_cases.npz"))
    for m in json.loads(str(z["meta"]))["efficacy"]:
        cfg = refgen.SyntheticWorkloadConfig(num_seqs=8, decode_steps=2500, prefill_tokens=32, zipf_s=1.0,
                                             recency_boost=0.3, w_hot=4, rng_seed=m["seed"], popularity_seed=7)
        tr = refgen.generate_trace(TraceHeader("efficacy", 1, 64, 8), cfg)
        ds = dataset.build_training_data(tr, 64, 64)[0]
        assert len(ds) == m["n"]
        assert digest(ds.features) == m["features"] and digest(ds.targets) == m["targets"]
        assert digest(ds.masks) == m["masks"]
