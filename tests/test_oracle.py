"""Pin the CPU oracle (oracle/) against the reference-generated golden fixtures.

These are CPU tests: the oracle must reproduce every SimReport (floats
included), every per-layer decision hash and, where recorded, every decision
of the reference simulator on the same traces.
"""
import os

import numpy as np
import pytest

import oracle
from golden_util import COSTS, GOLDEN, case_trace, include_prefill, lecar_params, load, policy_name


def _check_case(case, check_decisions=True):
    header, events = case_trace(case)
    L, E, K = header
    for run in case["runs"]:
        nets = oracle.nets_from_spec(run["nets"], L, E, GOLDEN)
        pol = policy_name(run["policy"])
        report, hashes, outs = oracle.simulate(
            header, events, pol, run["capacity"], COSTS[run["cost"]], run["window"],
            nets if pol == "ml" else None, include_prefill(run["policy"]),
            want_outcomes=check_decisions and "decisions" in run, lecar=lecar_params(run["policy"]))
        assert report == run["report"], (case["name"], run["policy"], run["capacity"])
        assert [format(h, "016x") for h in hashes] == run["hashes"], (case["name"], run["policy"])
        if outs is not None:
            assert [o.tolist() for o in outs] == run["decisions"]


@pytest.mark.parametrize("idx", range(0, 167, 1))
def test_oracle_small_cases(idx):
    cases = load("small_cases.json.gz")["cases"]
    if idx >= len(cases):
        pytest.skip("fewer cases")
    _check_case(cases[idx])


def test_oracle_zipf_and_dominance_cases():
    for case in load("zipf_cases.json.gz")["cases"]:
        _check_case(case, check_decisions=False)


def test_oracle_c1_and_mixtral_full_size():
    if not os.path.exists(os.path.join(GOLDEN, "big_cases.json.gz")):
        pytest.skip("big fixtures not generated")
    for case in load("big_cases.json.gz")["cases"]:
        _check_case(case, check_decisions=False)


def test_oracle_efficacy_golden():
    """Trained net (reference train_eviction_net) on 10 held-out traces:
    ml 82.90% / lru 81.30% / lfu 79.78% (pkg/test_output.txt:360)."""
    path = os.path.join(GOLDEN, "efficacy_cases.json.gz")
    if not os.path.exists(path):
        pytest.skip("efficacy fixtures not generated")
    g = load("efficacy_cases.json.gz")
    rates = {"ml": [], "lru": [], "lfu": []}
    for case in g["cases"]:
        _check_case(case, check_decisions=False)
        for run in case["runs"]:
            rates[policy_name(run["policy"])].append(run["report"]["hit_rate"])
    means = {p: round(100 * float(np.mean(v)), 2) for p, v in rates.items()}
    assert means == {"ml": 82.90, "lru": 81.30, "lfu": 79.78}


def test_uniform_batch_matches_simulate():
    """The multi-threaded decode-only batch driver (CPU baseline) agrees with
    the per-trace path on the Mixtral-shaped golden trace."""
    path = os.path.join(GOLDEN, "big_cases.json.gz")
    if not os.path.exists(path):
        pytest.skip("big fixtures not generated")
    case = load("big_cases.json.gz")["cases"][1]
    from golden_util import big_ids
    ids, E = big_ids(case)
    T, L, K = ids.shape
    chains = np.ascontiguousarray(ids.transpose(1, 0, 2))
    jobs = [(policy_name(r["policy"]), r["capacity"]) for r in case["runs"]]
    nets = oracle.nets_from_spec({"kind": "per_layer_seed"}, L, E)
    cnt, lat, hsh = oracle.replay_uniform(chains, L, E, jobs, COSTS["default"], 5, nets, threads=4)
    for j, run in enumerate(case["runs"]):
        rep = oracle.fold_report(jobs[j][0], jobs[j][1], 5, cnt[:, j], lat[:, j], T)
        assert rep == run["report"]
        assert [format(int(h), "016x") for h in hsh[:, j]] == run["hashes"]


def test_oracle_poly_hash_matches_recorded_decisions():
    """The spliceable hash the CUDA engine reports (poly) is a function of the
    same per-access outcome codes as the fixtures' FNV hash."""
    from golden_util import poly_hash
    for case in load("small_cases.json.gz")["cases"][::5]:
        header, events = case_trace(case)
        L, E, K = header
        for run in case["runs"]:
            if "decisions" not in run:
                continue
            name = policy_name(run["policy"])
            nets = oracle.nets_from_spec(run["nets"], L, E, GOLDEN) if name == "ml" else None
            _, hp, _ = oracle.simulate(header, events, name, run["capacity"], COSTS[run["cost"]], run["window"],
                                       nets, include_prefill(run["policy"]), hash_kind="poly")
            assert hp == [poly_hash(d) for d in run["decisions"]], case["name"]


def test_oracle_generator_matches_reference_fixtures():
    """oracle.generate_experts (numpy restatement of trace.py:186-287) against
    traces made by the reference generator (tests/golden/make_gen_golden.py)."""
    import json
    z = np.load(os.path.join(GOLDEN, "gen_cases.npz"))
    for m in json.loads(str(z["meta"])):
        got = oracle.generate_experts(tuple(m["header"]), m["config"])
        assert np.array_equal(got, z[m["name"]]), m["name"]


def test_oracle_fifo_cases():
    """FIFO (policies.py:152-168) on reference-made fixtures (make_fifo_golden.py)."""
    for case in load("fifo_cases.json.gz")["cases"]:
        _check_case(case)


def test_oracle_arc_cases():
    """ARC (policies.py:217-302) on reference-made fixtures (make_arc_golden.py)."""
    for case in load("arc_cases.json.gz")["cases"]:
        _check_case(case)


def test_oracle_lecar_cases():
    """LeCaR (policies.py:305-395) on reference-made fixtures (make_lecar_golden.py):
    default and explicit learning_rate / discount_base / seed specs."""
    cases = load("lecar_cases.json.gz")["cases"]
    assert sum(r["n_evictions"] for c in cases for r in c["runs"]) > 1000
    for case in cases:
        _check_case(case)


def test_oracle_duel_cases():
    """eviction_quality_duel (engine.py:404-436) restated on the oracle's
    outcomes, against reference-made fixtures (make_duel_golden.py)."""
    for case in load("duel_cases.json.gz")["cases"]:
        header, events = case_trace(case)
        L, E, K = header
        for d in case["duels"]:
            nets = oracle.nets_from_spec(d["nets"], L, E, GOLDEN)
            got = oracle.eviction_duel(header, events, policy_name(d["a"]), policy_name(d["b"]), d["capacity"],
                                       nets, lecar_params(d["a"]), lecar_params(d["b"]))
            assert got == d["value"], (case["name"], d)


def test_oracle_c_generator_matches_reference_fixtures():
    """orc_gen_decode (C restatement of trace.py:186-287, used for the bench's
    reference arm) against the decode-only reference-made traces: the small
    decode-only fixtures and the full-size C1 (48 x 128 x 8, 2,048 tokens)
    and Mixtral-shaped traces."""
    import json
    from golden_util import big_ids
    z = np.load(os.path.join(GOLDEN, "gen_cases.npz"))
    n = 0
    for m in json.loads(str(z["meta"])):
        c = m["config"]
        if c.get("num_seqs", 1) != 1 or c.get("prefill_tokens", 32) != 0:
            continue
        got = oracle.generate_decode_batch(tuple(m["header"]), c["decode_steps"], [c.get("rng_seed", 0)],
                                           c.get("popularity_seed"), c.get("zipf_s", 1.0),
                                           c.get("recency_boost", 0.0), c.get("w_hot", 4))
        assert np.array_equal(got[0], z[m["name"]][0]), m["name"]
        n += 1
    for case in load("big_cases.json.gz")["cases"][:2]:
        ids, E = big_ids(case)
        T, L, K = ids.shape
        c = case["config"]
        got = oracle.generate_decode_batch((L, E, K), T, [c["rng_seed"]], c.get("popularity_seed"), c["zipf_s"],
                                           c["recency_boost"], c["w_hot"])
        assert np.array_equal(got[0], ids)
        n += 1
    assert n >= 4
