"""Bit-exact GPU reproduction of the reference generator (refgen /
mcb_gen_reference) against traces made by the reference itself: the small
cases of tests/golden/gen_cases.npz (prefill, several sequences, popularity
seeds, no / full recency boost, K == E tails, odd E) and the full-size C1
(Qwen3-shaped, 48 x 128 x 8, 2048 tokens) and Mixtral-shaped (32 x 8 x 2,
2048 tokens) fixtures."""
import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN, big_ids, load

pytestmark = pytest.mark.gpu

from paper_2601_17063_b200 import refgen  # noqa: E402
from paper_2601_17063_b200.trace import TraceHeader  # noqa: E402


def test_small_cases_bit_exact():
    z = np.load(os.path.join(GOLDEN, "gen_cases.npz"))
    for m in json.loads(str(z["meta"])):
        L, E, K = m["header"]
        got = refgen.generate_experts(TraceHeader(m["name"], L, E, K), refgen.SyntheticWorkloadConfig(**m["config"]))
        assert np.array_equal(got.cpu().numpy(), z[m["name"]]), m["name"]


@pytest.mark.parametrize("which", [0, 1])
def test_full_size_reference_traces(which):
    case = load("big_cases.json.gz")["cases"][which]
    ids, E = big_ids(case)                       # [T][L][K] from the reference generator
    T, L, K = ids.shape
    c = case["config"]
    cfg = refgen.SyntheticWorkloadConfig(num_seqs=1, decode_steps=T, prefill_tokens=0, zipf_s=c["zipf_s"],
                                         recency_boost=c["recency_boost"], w_hot=c["w_hot"], rng_seed=c["rng_seed"])
    got = refgen.generate_experts(TraceHeader("big", L, E, K), cfg)[0].cpu().numpy()
    assert np.array_equal(got, ids)
    dec = refgen.generate_decode_ids(TraceHeader("big", L, E, K), cfg).cpu().numpy()
    assert np.array_equal(dec, ids.transpose(1, 0, 2))


def test_generate_trace_api_matches_reference_events():
    z = np.load(os.path.join(GOLDEN, "gen_cases.npz"))
    m = json.loads(str(z["meta"]))[0]
    L, E, K = m["header"]
    tr = refgen.generate_trace(TraceHeader(m["name"], L, E, K), refgen.SyntheticWorkloadConfig(**m["config"]))
    ex = np.array([e.experts for e in tr.events], dtype=np.uint8).reshape(z[m["name"]].shape)
    assert np.array_equal(ex, z[m["name"]])


def test_batch_generator_matches_single_and_oracle():
    """mcb_gen_reference_batch (one stream per trace, shared popularity) equals
    the per-trace generator and the oracle's C restatement, chain-major."""
    import oracle
    hdr = TraceHeader("b", 5, 64, 6)
    seeds = [0, 1, 7, 1234567]
    got = refgen.generate_decode_batch(hdr, seeds, 300, popularity_seed=7, recency_boost=0.3, w_hot=4)
    got = got.cpu().numpy()
    for i, s in enumerate(seeds):
        cfg = refgen.SyntheticWorkloadConfig(num_seqs=1, decode_steps=300, prefill_tokens=0, recency_boost=0.3,
                                             w_hot=4, rng_seed=s, popularity_seed=7)
        one = refgen.generate_decode_ids(hdr, cfg).cpu().numpy()
        assert np.array_equal(got[i], one), s
    ref = oracle.generate_decode_batch((5, 64, 6), 300, seeds, 7, 1.0, 0.3, 4)   # [n][T][L][K]
    assert np.array_equal(got, ref.transpose(0, 2, 1, 3))
