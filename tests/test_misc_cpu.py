"""The reference's small utilities re-exported by the package, against
reference-made fixtures (tests/golden/make_misc_golden.py):
prefill_coverage, expert_popularity, lecar_update, masked_mse.  CPU only."""
import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN

import paper_2601_17063_b200 as mcb
from paper_2601_17063_b200.trace import AccessEvent, Phase, RoutingTrace, TraceHeader

M = json.load(open(os.path.join(GOLDEN, "misc_cases.json")))


def test_prefill_coverage():
    for c in M["coverage"]:
        L, E, K = c["header"]
        tr = RoutingTrace(TraceHeader("x", L, E, K),
                          tuple(AccessEvent(s, Phase(p), t, l, tuple(x)) for s, p, t, l, x in c["events"]))
        if "ok" in c:
            assert [list(r) for r in mcb.prefill_coverage(tr, c["counts"])] == c["ok"]
        else:
            with pytest.raises(mcb.TraceError) as ei:
                mcb.prefill_coverage(tr, c["counts"])
            assert type(ei.value).__name__ == c["error"] and str(ei.value) == c["message"]


def test_expert_popularity():
    for c in M["popularity"]:
        L, E, K = c["header"]
        cfg = mcb.SyntheticWorkloadConfig(num_seqs=1, decode_steps=1, prefill_tokens=0, zipf_s=c["zipf_s"],
                                          rng_seed=c["rng_seed"], popularity_seed=c["popularity_seed"])
        got = mcb.expert_popularity(TraceHeader("x", L, E, K), cfg, c["layer"])
        assert got.tolist() == c["p"]


def test_lecar_update_and_masked_mse():
    for c in M["lecar"]:
        d = 0.005 ** (1.0 / c["cap"])
        assert list(mcb.lecar_update((0.3, 0.7), c["kind"], c["elapsed"], 0.45, d)) == c["w"]
    for c in M["mse"]:
        assert mcb.masked_mse(np.array(c["pred"]), np.array(c["target"]), np.array(c["mask"], dtype=bool)) == c["value"]
