"""K8 (mcb_eviction_duel) through the public eviction_quality_duel against
reference-made fixtures (engine.py:404-436) and the oracle restatement on
larger decode-only traces."""
import numpy as np
import pytest

import oracle
from golden_util import GOLDEN, case_trace, lecar_params, load, policy_name

pytestmark = pytest.mark.gpu

import paper_2601_17063_b200 as mcb  # noqa: E402
from paper_2601_17063_b200.trace import AccessEvent, Phase, RoutingTrace, TraceHeader  # noqa: E402


def to_trace(header, events):
    L, E, K = header
    return RoutingTrace(TraceHeader("golden", L, E, K),
                        tuple(AccessEvent(s, Phase(p), t, l, tuple(x)) for s, p, t, l, x in events))


def engine_nets(spec, L, E):
    if spec is None:
        return None
    return [mcb.EvictionNet(E, hidden=spec["hidden"], seed=l) for l in range(L)]


def test_duel_cases():
    for case in load("duel_cases.json.gz")["cases"]:
        header, events = case_trace(case)
        L, E, K = header
        trace = to_trace(header, events)
        for d in case["duels"]:
            got = mcb.eviction_quality_duel(trace, d["a"], d["b"], d["capacity"], nets=engine_nets(d["nets"], L, E))
            assert got == d["value"], (case["name"], d)


@pytest.mark.parametrize("E,K,cap", [(16, 2, 5), (64, 4, 12)])
def test_duel_larger_traces_vs_oracle(E, K, cap):
    rng = np.random.default_rng(E)
    L, T = 3, 3000
    pop = rng.zipf(1.3, size=E * 8) % E
    ids = np.stack([rng.choice(pop[rng.integers(0, len(pop) - 64):][:64], size=K, replace=False)
                    if len(set(pop[:64])) >= K else rng.permutation(E)[:K] for _ in range(T * L)])
    ids = np.array([r if len(set(r.tolist())) == K else rng.permutation(E)[:K] for r in ids], dtype=np.uint8)
    ids = ids.reshape(T, L, K)
    events = [(0, 1, t, l, ids[t, l].tolist()) for t in range(T) for l in range(L)]
    trace = to_trace((L, E, K), events)
    for a, b in [("lru", "lfu"), ("belady", "fifo"), ("arc", "lecar")]:
        got = mcb.eviction_quality_duel(trace, a, b, cap)
        want = oracle.eviction_duel((L, E, K), events, a, b, cap)
        assert got == want, (a, b)
        assert 0.0 <= got <= 1.0


def test_timeline_files_match_reference(tmp_path):
    """write_timeline from the engine's victim stream is byte-identical to the
    reference's file (reports.py:161-210, make_timeline_golden.py)."""
    import hashlib
    from paper_2601_17063_b200 import reports
    for case in load("timeline_cases.json.gz")["cases"]:
        header, events = case_trace(case)
        trace = to_trace(header, events)
        run = mcb.run_simulation(trace, case["policy"], case["capacity"])
        path = tmp_path / "t.jsonl"
        reports.write_timeline(mcb.pack_trace(trace), run.evictions, case["policy"], path)
        data = path.read_bytes()
        assert data[:400].decode() == case["head"], case["name"]
        assert hashlib.sha256(data).hexdigest() == case["sha256"], case["name"]
        hdr, rows = reports.load_timeline(path)
        assert hdr["policy"] == case["policy"] and len(rows) == case["lines"] - 1
