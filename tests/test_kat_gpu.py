"""The reference's own known-answer and property tests for this path
(SURVEY.md §8c), restated against the B200 engine through the public API:
pkg/tests/test_policies.py (textbook victims, brute-force Belady, shadow-set
hits, pinning, naive LRU/LFU, Belady dominance, determinism) and
pkg/tests/test_engine.py (latency model, accounting identities, prefill
union, refetch, duel, sweep).  Traces come from this package's bit-exact
generator (refgen, = the reference's helpers.zipf_trace) and a local
random-trace builder (the reference's helpers.random_trace recipe)."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2601_17063_b200 as mcb  # noqa: E402
from paper_2601_17063_b200 import refgen  # noqa: E402
from paper_2601_17063_b200.trace import AccessEvent, Phase, RoutingTrace, TraceHeader  # noqa: E402

ALL = ["lru", "lfu", "fifo", "arc", "lecar", "belady"]
D, P = Phase.DECODE, Phase.PREFILL
A, B, C = 0, 1, 2


def make_trace(events, num_layers=1, num_experts=16, top_k=2):
    t = RoutingTrace(TraceHeader("t", num_layers, num_experts, top_k), tuple(events))
    t.validate()
    return t


def one_expert_stream(stream, num_experts=4):
    """Each access its own decode event (the reference's drive() helper)."""
    return make_trace([AccessEvent(0, D, i, 0, (x,)) for i, x in enumerate(stream)], num_experts=num_experts,
                      top_k=1)


def zipf_trace(seed, num_layers=1, num_experts=16, top_k=4, num_seqs=1, decode_steps=120, prefill_tokens=8):
    cfg = refgen.SyntheticWorkloadConfig(num_seqs=num_seqs, decode_steps=decode_steps, prefill_tokens=prefill_tokens,
                                         zipf_s=1.0, recency_boost=0.3, w_hot=4, rng_seed=seed)
    return refgen.generate_trace(TraceHeader("synthetic", num_layers, num_experts, top_k), cfg)


def random_trace(rng, num_experts=None, max_seqs=2, max_prefill=3, max_decode=6):
    L = rng.randint(1, 3)
    E = num_experts or rng.randint(2, 10)
    K = rng.randint(1, min(3, E))
    ev = []
    for s in range(rng.randint(1, max_seqs)):
        for t in range(rng.randint(0, max_prefill)):
            for l in range(L):
                ev.append(AccessEvent(s, P, t, l, tuple(rng.sample(range(E), rng.randint(1, E)))))
        for t in range(rng.randint(0, max_decode)):
            for l in range(L):
                ev.append(AccessEvent(s, D, t, l, tuple(rng.sample(range(E), K))))
    return make_trace(ev, L, E, K)


def schedules(trace):
    """Per-layer (accesses, decode flag, new_sequence flag) per event (replay.py:44-81)."""
    L = trace.header.num_layers
    out = [[] for _ in range(L)]
    last, seen = [None] * L, [set() for _ in range(L)]
    for ev in trace.events:
        new = last[ev.layer] != ev.seq_id
        if new:
            last[ev.layer], seen[ev.layer] = ev.seq_id, set()
        if ev.phase == P:
            acc = [e for e in ev.experts if e not in seen[ev.layer]]
            seen[ev.layer].update(ev.experts)
        else:
            acc = list(ev.experts)
        out[ev.layer].append((acc, ev.phase == D, new))
    return out


# ---------------------------------------------------------------- textbook --

def victims(stream, policy, capacity):
    run = mcb.run_simulation(one_expert_stream(stream), policy, capacity, record_decisions=True)
    return run.decisions[0]


def test_lru_evicts_least_recent():
    d = victims([A, B, A, C], "lru", 2)
    assert [x.was_hit for x in d] == [False, False, True, False]
    assert d[3].evicted == B


def test_lfu_evicts_least_frequent_and_ties_by_id():
    assert victims([A, A, B, C], "lfu", 2)[3].evicted == B
    assert victims([B, A, C], "lfu", 2)[2].evicted == A


def test_fifo_ignores_hits():
    assert victims([A, B, A, C], "fifo", 2)[3].evicted == A


def test_belady_evicts_farthest_next_use():
    assert victims([A, B, C, A, B], "belady", 2)[2].evicted == B


def test_decision_shape():
    d = victims([A, B], "lru", 1)
    assert d[0].evicted is None and not d[0].was_hit
    assert d[1].evicted is not None


@pytest.mark.parametrize("seed", range(10))
def test_belady_victim_matches_brute_force(seed):
    rng = random.Random(seed)
    stream = [rng.randrange(6) for _ in range(60)]
    d = mcb.run_simulation(one_expert_stream(stream, 6), "belady", 3, record_decisions=True).decisions[0]
    resident = set()
    for pos, (x, dec) in enumerate(zip(stream, d)):
        if x not in resident and len(resident) >= 3:
            def nxt(e):
                return next((q for q in range(pos + 1, len(stream)) if stream[q] == e), float("inf"))
            best = min(sorted(resident), key=lambda e: (-nxt(e), e))
            assert dec.evicted == best, pos
            resident.discard(best)
        resident.add(x)


# --------------------------------------------------------- engine properties --

@pytest.mark.parametrize("seed", range(4))
def test_capacity_never_exceeded_and_hits_correct(seed):
    trace = random_trace(random.Random(seed), num_experts=8)
    cap = max(trace.header.top_k, 3)
    for policy in ALL:
        run = mcb.run_simulation(trace, policy, cap, record_decisions=True)
        for layer, sched in enumerate(schedules(trace)):
            shadow = set()
            it = iter(run.decisions[layer])
            for acc, _, _ in sched:
                for x in acc:
                    d = next(it)
                    assert d.loaded == x and d.was_hit == (x in shadow)
                    if d.was_hit:
                        assert d.evicted is None
                    if d.evicted is not None:
                        assert d.evicted in shadow
                        shadow.remove(d.evicted)
                    shadow.add(x)
                    assert len(shadow) <= cap


@pytest.mark.parametrize("seed", range(20))
def test_belady_dominates_all_policies(seed):
    trace = zipf_trace(seed, num_experts=12, top_k=3, decode_steps=60, prefill_tokens=4)
    for cap in (3, 6, 9):
        rows = {r.policy: r.hits for r in mcb.sweep(trace, ALL, [cap])}
        assert all(rows["belady"] >= rows[p] for p in ALL)


def naive(sched, cap, kind):
    resident, stamp, freq, out, pos = set(), {}, {}, [], 0
    for acc, decode, new in sched:
        if new and kind == "lfu":
            freq.clear()
        pinned = set()
        for x in acc:
            freq[x] = freq.get(x, 0) + 1
            hit, ev = x in resident, None
            if not hit:
                if len(resident) >= cap:
                    cand = [e for e in resident if e not in pinned]
                    ev = min(cand, key=(lambda e: (stamp[e], e)) if kind == "lru" else (lambda e: (freq.get(e, 0), e)))
                    resident.remove(ev)
                resident.add(x)
            stamp[x] = pos
            out.append((x, hit, ev))
            if decode:
                pinned.add(x)
            pos += 1
    return out


@pytest.mark.parametrize("kind", ["lru", "lfu"])
@pytest.mark.parametrize("seed", range(10))
def test_matches_naive_reference(kind, seed):
    trace = random_trace(random.Random(1000 + seed), num_experts=9)
    cap = max(trace.header.top_k, 3)
    run = mcb.run_simulation(trace, kind, cap, record_decisions=True)
    for layer, sched in enumerate(schedules(trace)):
        assert [(d.loaded, d.was_hit, d.evicted) for d in run.decisions[layer]] == naive(sched, cap, kind)


def test_decisions_deterministic_and_pinned_never_evicted():
    trace = zipf_trace(7, num_experts=10, top_k=4, decode_steps=80, prefill_tokens=0)
    for policy in ALL:
        r1 = mcb.run_simulation(trace, policy, 4, record_decisions=True)
        r2 = mcb.run_simulation(trace, policy, 4, record_decisions=True)
        assert r1.decisions == r2.decisions and r1.report == r2.report
        for layer, sched in enumerate(schedules(trace)):
            it = iter(r1.decisions[layer])
            for acc, _, _ in sched:
                pinned = set()
                for x in acc:
                    d = next(it)
                    assert d.evicted is None or d.evicted not in pinned
                    pinned.add(x)


# ------------------------------------------------------------ latency model --

def test_two_miss_step_and_all_hit_latency():
    t = make_trace([AccessEvent(0, P, 0, 0, (0, 1, 2, 3, 4, 5)), AccessEvent(0, D, 0, 0, tuple(range(8)))], 1, 16, 8)
    r = mcb.simulate(t, "lru", 10)
    assert r.decode_misses == 2
    assert r.est_decode_latency_s == pytest.approx(6e-3)
    assert r.est_prefill_latency_s == pytest.approx(6 * 3e-3)
    t = make_trace([AccessEvent(0, P, 0, 0, tuple(range(8))), AccessEvent(0, D, 0, 0, tuple(range(8)))], 1, 16, 8)
    r = mcb.simulate(t, "lru", 10)
    assert r.decode_misses == 0 and r.est_decode_latency_s == pytest.approx(1.264e-3)


def test_ml_score_cost_flag_and_tokens_per_second():
    trace = zipf_trace(0, num_experts=8, top_k=2, decode_steps=10, prefill_tokens=0)
    net = mcb.EvictionNet(8, seed=0)
    base = mcb.simulate(trace, "ml", 4, nets=net)
    costed = mcb.simulate(trace, "ml", 4, mcb.CostModel(ml_score_cost_s=1e-4), nets=net)
    assert costed.est_decode_latency_s == pytest.approx(base.est_decode_latency_s + 10 * 1e-4)
    trace = zipf_trace(1, num_layers=2, num_experts=8, top_k=2, decode_steps=20)
    r = mcb.simulate(trace, "lru", 4)
    assert r.tokens_per_second_est == pytest.approx(20 / r.est_decode_latency_s)


# --------------------------------------------------------------- accounting --

def test_full_capacity_only_compulsory_and_thrashing():
    r = mcb.simulate(zipf_trace(2, num_experts=12, top_k=3, decode_steps=80, prefill_tokens=4), "lru", 12)
    assert r.misses == r.compulsory_misses and r.hit_rate_excl_compulsory == 1.0 and r.evictions == 0
    t = make_trace([AccessEvent(0, D, s, 0, (0, 1) if s % 2 == 0 else (2, 3)) for s in range(40)], 1, 4, 2)
    r = mcb.simulate(t, "lru", 2)
    assert r.hits == 0 and r.hit_rate == 0.0


@pytest.mark.parametrize("seed", range(3))
def test_accounting_identity(seed):
    trace = random_trace(random.Random(seed), num_experts=10)
    cap = max(trace.header.top_k, 3)
    total = sum(len(acc) for s in schedules(trace) for acc, _, _ in s)
    for policy in ALL:
        r = mcb.simulate(trace, policy, cap)
        assert r.hits + r.misses == total and r.io_count == r.misses
        assert r.hits == r.prefill_hits + r.decode_hits and r.misses == r.prefill_misses + r.decode_misses


def test_prefill_union_counted_once_and_reloaded_next_sequence():
    t = make_trace([AccessEvent(0, P, 0, 0, (0, 1)), AccessEvent(0, P, 1, 0, (1, 2))], 1, 8, 2)
    r = mcb.simulate(t, "lru", 4)
    assert r.prefill_hits + r.prefill_misses == 3
    t = make_trace([AccessEvent(0, P, 0, 0, (0, 1)), AccessEvent(1, P, 0, 0, (0, 1))], 1, 8, 2)
    r = mcb.simulate(t, "lru", 4)
    assert r.prefill_hits == 2 and r.prefill_misses == 2


def test_capacity_too_small_and_lecar_deterministic():
    with pytest.raises(mcb.CapacityTooSmallError):
        mcb.simulate(zipf_trace(0, num_experts=8, top_k=4, decode_steps=5), "lru", 3)
    trace = zipf_trace(5, num_layers=2, num_experts=10, top_k=3, decode_steps=40)
    assert mcb.simulate(trace, "lecar", 5) == mcb.simulate(trace, "lecar", 5)


# ------------------------------------------------------------------ refetch --

def test_refetch_known_answers():
    assert mcb.refetch_rate(zipf_trace(1, num_experts=8, top_k=2, decode_steps=30), "lru", 8) == 0.0
    t = make_trace([AccessEvent(0, D, 0, 0, (0, 1)), AccessEvent(0, D, 1, 0, (1, 2)),
                    AccessEvent(0, D, 2, 0, (0, 1)), AccessEvent(0, D, 3, 0, (1, 2))], 1, 4, 2)
    run = mcb.run_simulation(t, "lru", 2, window=5)
    assert run.report.evictions == 4 and run.report.refetch_within_w == pytest.approx(0.75)
    t = make_trace([AccessEvent(0, D, 0, 0, (0, 1)), AccessEvent(0, D, 1, 0, (2, 3)),
                    AccessEvent(0, D, 2, 0, (0, 1))], 1, 4, 2)
    assert mcb.refetch_rate(t, "lru", 2, window=0) == 0.0
    assert mcb.refetch_rate(t, "lru", 2, window=2) > 0.0


@pytest.mark.parametrize("seed", range(20))
def test_belady_refetch_not_above_lru(seed):
    trace = zipf_trace(seed, num_experts=12, top_k=3, decode_steps=80, prefill_tokens=4)
    for cap in (4, 6):
        assert mcb.refetch_rate(trace, "belady", cap, window=5) <= mcb.refetch_rate(trace, "lru", cap, window=5)


# --------------------------------------------------------------------- duel --

def test_duel_properties():
    trace = zipf_trace(4, num_experts=10, top_k=2, decode_steps=50)
    for p in ("lru", "lfu", "belady"):
        assert mcb.eviction_quality_duel(trace, p, p, 4) == 0.5
    for seed in range(10):
        trace = zipf_trace(seed, num_experts=12, top_k=3, decode_steps=80, prefill_tokens=4)
        for opp in ("lru", "lfu"):
            assert mcb.eviction_quality_duel(trace, "belady", opp, 6) >= 0.5
    trace = zipf_trace(9, num_experts=12, top_k=3, decode_steps=60)
    ab = mcb.eviction_quality_duel(trace, "lru", "lfu", 5)
    assert ab == pytest.approx(1.0 - mcb.eviction_quality_duel(trace, "lfu", "lru", 5))


# -------------------------------------------------------------------- sweep --

def test_sweep_order_belady_tops_and_monotone():
    trace = zipf_trace(2, num_experts=12, top_k=2, decode_steps=40)
    rows = mcb.sweep(trace, ["lru", "belady", "lfu"], [6, 4, 8])
    assert [(r.policy, r.capacity) for r in rows] == sorted((p, c) for p in ("belady", "lfu", "lru") for c in (4, 6, 8))
    trace = zipf_trace(6, num_experts=16, top_k=4, decode_steps=100, prefill_tokens=4)
    rows = mcb.sweep(trace, ["lru", "lfu", "fifo", "belady"], [4, 8, 12])
    for cap in (4, 8, 12):
        group = [r for r in rows if r.capacity == cap]
        assert next(r for r in group if r.policy == "belady").hit_rate == max(r.hit_rate for r in group)
    rows = mcb.sweep(zipf_trace(8, num_experts=16, top_k=4, decode_steps=100), ["belady"], [4, 6, 8, 10, 12])
    rates = [r.hit_rate for r in rows]
    assert rates == sorted(rates)
    with pytest.raises(mcb.CapacityTooSmallError):
        mcb.sweep(zipf_trace(0, num_experts=8, top_k=4, decode_steps=5), ["lru"], [4, 2])
