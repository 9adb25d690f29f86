"""GPU parity: the CUDA engine (through the C ABI) against the reference-made
golden fixtures and the C oracle.  Bar: bit-exact integer counters, decision
hashes and decisions; SimReport floats equal (fp64 latency summed in the
reference's order)."""
import os

import numpy as np
import pytest

import oracle
from golden_util import (COSTS, GOLDEN, big_ids, case_trace, expected_poly_hashes, include_prefill,
                         lecar_params, load, policy_name)

pytestmark = pytest.mark.gpu

import paper_2601_17063_b200 as mcb  # noqa: E402
from paper_2601_17063_b200 import _lib, engine  # noqa: E402
from paper_2601_17063_b200.trace import AccessEvent, Phase, RoutingTrace, TraceHeader  # noqa: E402


def to_trace(header, events):
    L, E, K = header
    return RoutingTrace(TraceHeader("golden", L, E, K),
                        tuple(AccessEvent(s, Phase(p), t, l, tuple(x)) for s, p, t, l, x in events))


def cost_of(name):
    c = COSTS[name]
    return mcb.CostModel(c["t_load_s"], c["t_compute_s"], c["loads_serial"], c["ml_score_cost_s"])


def code_of(spec):
    name = policy_name(spec)
    if name == "ml":
        return _lib.MCB_ML if include_prefill(spec) else _lib.MCB_ML_NO_PREFILL
    return {"lru": _lib.MCB_LRU, "lfu": _lib.MCB_LFU, "belady": _lib.MCB_BELADY, "fifo": _lib.MCB_FIFO,
            "arc": _lib.MCB_ARC, "lecar": _lib.MCB_LECAR}[name]


def lecar_of(spec):
    if policy_name(spec) != "lecar":
        return None
    p = lecar_params(spec)
    return (p.get("learning_rate", 0.45), p.get("discount_base", 0.005), p.get("seed", 0))


def check_case(case, decisions=True):
    header, events = case_trace(case)
    L, E, K = header
    packed = mcb.pack_trace(to_trace(header, events))
    for ri, run in enumerate(case["runs"]):
        nets = oracle.nets_from_spec(run["nets"], L, E, GOLDEN) if policy_name(run["policy"]) == "ml" else None
        want_dec = decisions and "decisions" in run
        res = engine.replay_host(packed, [code_of(run["policy"])], [run["capacity"]], cost_of(run["cost"]),
                                 run["window"], nets, want_hashes=True, want_outcomes=want_dec,
                                 lecar=lecar_of(run["policy"]))
        rep = engine.assemble_report(policy_name(run["policy"]), run["capacity"], run["window"],
                                     res["reports"][0, 0, 0], res["latency"][0, 0, 0], packed.decode_steps[0])
        assert int(res["reports"][0, 0, 0, _lib.R_STATUS]) == 0
        assert rep.to_dict() == run["report"], (case["name"], run["policy"], run["capacity"])
        assert [int(h) for h in res["hashes"][:, 0, 0]] == expected_poly_hashes(case, ri), case["name"]
        if want_dec:
            got = []
            for l in range(L):
                a0 = engine._chain_acc_begin(packed, l)
                n = len(packed.chain_accesses(l))
                got.append(res["outcomes"][0, 0, a0:a0 + n].tolist())
            assert got == run["decisions"], (case["name"], run["policy"])


@pytest.fixture(params=["warp", "group8", "solo", "seg", "wide"])
def kernel_variant(request):
    """Run each parity case through every replay kernel: one warp per
    instance, 8-lane groups (16 for num_experts > 64: 4 / 2 instances per
    warp), one thread per instance (num_experts <= 16), and the segmented
    speculative replay (uniform traces, num_experts <= 16) with short
    segments so the stitching is exercised."""
    v = request.param
    _lib.set_tuning(_lib.MCB_TUNE_SOLO_MIN, 1 << 62 if v in ("warp", "group8", "wide") else 0)
    _lib.set_tuning(_lib.MCB_TUNE_WIDE_MIN, 0 if v == "wide" else 1 << 62)
    _lib.set_tuning(_lib.MCB_TUNE_GROUP_LANES, {"warp": 32, "group8": 8}.get(v, 0))
    _lib.set_tuning(_lib.MCB_TUNE_SEG_EV, 32 if v == "seg" else -1)
    yield v
    _lib.set_tuning(_lib.MCB_TUNE_SOLO_MIN, 0)
    _lib.set_tuning(_lib.MCB_TUNE_WIDE_MIN, 8192)
    _lib.set_tuning(_lib.MCB_TUNE_GROUP_LANES, 0)
    _lib.set_tuning(_lib.MCB_TUNE_SEG_EV, 0)


@pytest.mark.parametrize("part", range(4))
def test_small_cases(part, kernel_variant):
    cases = load("small_cases.json.gz")["cases"]
    for case in cases[part::4]:
        check_case(case)


@pytest.mark.parametrize("part", range(2))
def test_fifo_cases(part, kernel_variant):
    """FIFO (policies.py:152-168) against reference-made fixtures, decisions included."""
    for case in load("fifo_cases.json.gz")["cases"][part::2]:
        check_case(case)


@pytest.mark.parametrize("part", range(2))
def test_arc_cases(part, kernel_variant):
    """ARC (policies.py:217-302) against reference-made fixtures, decisions included."""
    for case in load("arc_cases.json.gz")["cases"][part::2]:
        check_case(case)


@pytest.mark.parametrize("part", range(2))
def test_lecar_cases(part, kernel_variant):
    """LeCaR (policies.py:305-395) against reference-made fixtures, decisions
    included: default and explicit learning_rate / discount_base / seed."""
    for case in load("lecar_cases.json.gz")["cases"][part::2]:
        check_case(case)


def test_lecar_public_api_and_sweep_grouping():
    """run_simulation / sweep with LeCaR specs of different parameters in one
    sweep (one engine call per parameter set) reproduce the fixtures."""
    cases = load("lecar_cases.json.gz")["cases"]
    for case in cases[:12]:
        header, events = case_trace(case)
        trace = to_trace(header, events)
        for run in case["runs"]:
            rep = mcb.run_simulation(trace, run["policy"], run["capacity"], cost_of(run["cost"]),
                                     run["window"]).report
            assert rep.to_dict() == run["report"], case["name"]
    header, events = case_trace(cases[0])
    trace = to_trace(header, events)
    specs = ["lecar", {"name": "lecar", "seed": 9}, "lru", {"name": "lecar", "learning_rate": 1.5}]
    cap = max(header[2], 3)
    rows = mcb.sweep(trace, specs, [cap])
    singles = sorted([mcb.simulate(trace, s, cap) for s in specs], key=lambda r: (r.policy, r.capacity))
    assert [r.to_dict() for r in rows] == [r.to_dict() for r in singles]


def test_zipf_and_dominance_cases(kernel_variant):
    for case in load("zipf_cases.json.gz")["cases"]:
        check_case(case, decisions=False)


def test_efficacy_golden_means():
    g = load("efficacy_cases.json.gz")
    rates = {"ml": [], "lru": [], "lfu": []}
    for case in g["cases"]:
        check_case(case, decisions=False)
        for run in case["runs"]:
            rates[policy_name(run["policy"])].append(run["report"]["hit_rate"])
    means = {p: round(100 * float(np.mean(v)), 2) for p, v in rates.items()}
    assert means == {"ml": 82.90, "lru": 81.30, "lfu": 79.78}


@pytest.mark.parametrize("which", [0, 1])
def test_full_size_c1_and_mixtral(which, kernel_variant):
    """C1 (Qwen3-shaped L48/E128/K8, 2048 tokens) and the Mixtral-shaped trace
    at full size: one engine call per trace for all policies x capacities."""
    case = load("big_cases.json.gz")["cases"][which]
    ids, E = big_ids(case)
    T, L, K = ids.shape
    packed = mcb.packed_from_decode_ids(np.ascontiguousarray(ids.transpose(1, 0, 2)), E)
    runs = case["runs"]
    pols = list(dict.fromkeys(policy_name(r["policy"]) for r in runs))
    caps = list(dict.fromkeys(r["capacity"] for r in runs))
    nets = oracle.nets_from_spec({"kind": "per_layer_seed"}, L, E)
    res = engine.replay_host(packed, [code_of(p) for p in pols], caps, mcb.CostModel(), 5, nets, want_hashes=True)
    for ri, r in enumerate(runs):
        i, j = pols.index(policy_name(r["policy"])), caps.index(r["capacity"])
        rep = engine.assemble_report(pols[i], caps[j], 5, res["reports"][0, i, j], res["latency"][0, i, j], T)
        assert rep.to_dict() == r["report"], (case["name"], r["policy"], r["capacity"])
        assert [int(h) for h in res["hashes"][:, i, j]] == expected_poly_hashes(case, ri)


def test_public_api_matches_reports():
    """simulate / run_simulation / sweep return the golden SimReports."""
    case = load("zipf_cases.json.gz")["cases"][0]
    header, events = case_trace(case)
    tr = to_trace(header, events)
    L, E, _ = header
    nets = [mcb.EvictionNet(E, seed=l) for l in range(L)]
    want = {(r["policy"] if isinstance(r["policy"], str) else "mlnp", r["capacity"], r["cost"]): r["report"]
            for r in case["runs"]}
    for cap in (8, 16):
        assert mcb.simulate(tr, "lru", cap).to_dict() == want[("lru", cap, "default")]
        assert mcb.simulate(tr, "ml", cap, nets=nets).to_dict() == want[("ml", cap, "default")]
        run = mcb.run_simulation(tr, "belady", cap, record_decisions=True)
        assert run.report.to_dict() == want[("belady", cap, "default")]
        assert len(run.evictions) == run.report.evictions
        assert sum(len(v) for v in run.decisions.values()) == run.report.hits + run.report.misses
    rows = mcb.sweep(tr, ["lru", "lfu", "belady", "ml"], [8, 16, 32], nets=nets)
    assert [(r.policy, r.capacity) for r in rows] == sorted((p, c) for p in ("lru", "lfu", "belady", "ml")
                                                            for c in (8, 16, 32))
    for r in rows:
        assert r.to_dict() == want[(r.policy, r.capacity, "default")]


def test_eviction_records_match_reference():
    for case in load("small_cases.json.gz")["cases"][:40]:
        header, events = case_trace(case)
        tr = to_trace(header, events)
        for run in case["runs"]:
            if run["cost"] != "default" or policy_name(run["policy"]) == "ml":
                continue
            sr = mcb.run_simulation(tr, run["policy"], run["capacity"], window=run["window"],
                                    record_decisions=True)
            recs = [[r.layer, r.position, r.tick, r.decode_index, r.victim] for r in sr.evictions]
            assert recs == run["eviction_records"], case["name"]


def test_next_use_kernel_matches_numpy():
    import torch
    rng = np.random.default_rng(0)
    # the last two shapes run the blocked walk (several blocks per chain)
    for E, n_chains, T, K in ((8, 5, 1000, 2), (64, 7, 33, 6), (128, 3, 777, 8), (8, 2, 40000, 2)):
        ids = np.stack([np.stack([rng.choice(E, K, replace=False) for _ in range(T)]) for _ in range(n_chains)])
        packed = mcb.packed_from_decode_ids(ids[None].astype(np.uint8), E)
        dev_acc = torch.from_numpy(packed.acc).cuda()
        v = packed.view()
        v.acc = dev_acc.data_ptr()
        out = torch.zeros(packed.total_acc + 64, dtype=torch.int32, device="cuda")
        lib = _lib.load_library()
        import ctypes
        _lib.check(lib.mcb_next_use(_lib.context(0), ctypes.byref(v), out.data_ptr(), None))
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint32)[:packed.total_acc].reshape(n_chains, T * K)
        for c in range(n_chains):
            s = ids[c].reshape(-1)
            want = np.full(len(s), 0xFFFFFFFF, dtype=np.uint64)
            last = {}
            for p in range(len(s) - 1, -1, -1):
                want[p] = last.get(int(s[p]), 0xFFFFFFFF)
                last[int(s[p])] = p
            assert np.array_equal(got[c].astype(np.uint64), want)


def test_scorer_matches_oracle_fp64():
    """K3 float64 scores vs the oracle's scalar-loop forward: normwise 1e-12."""
    import ctypes

    import torch
    case = load("big_cases.json.gz")["cases"][0]
    ids, E = big_ids(case)
    T, L, K = ids.shape
    chains = np.ascontiguousarray(ids.transpose(1, 0, 2))[:3, :300]
    packed = mcb.packed_from_decode_ids(chains[None], E)
    hidden, n_nets, params = oracle.nets_from_spec({"kind": "shared_seed", "seed": 5}, 3, E)
    lib = _lib.load_library()
    dev_acc = torch.from_numpy(packed.acc).cuda()
    v = packed.view()
    v.acc = dev_acc.data_ptr()
    dparams = torch.from_numpy(params).cuda()
    ns = _lib.MCBNets()
    ns.num_experts, ns.hidden, ns.num_nets, ns.params = E, hidden, 1, dparams.data_ptr()
    ranks = torch.zeros(packed.total_events * E + 64, dtype=torch.uint8, device="cuda")
    scores = torch.zeros(packed.total_events * E, dtype=torch.float64, device="cuda")
    _lib.check(lib.mcb_score(_lib.context(0), ctypes.byref(v), ctypes.byref(ns), 1, ranks.data_ptr(),
                             scores.data_ptr(), None))
    torch.cuda.synchronize()
    got = scores.cpu().numpy().reshape(3, 300, E)
    rk = ranks.cpu().numpy()[:packed.total_events * E].reshape(3, 300, E)
    for c in range(3):
        want = oracle.score_chain(chains[c], E, hidden, params)
        err = np.abs(got[c] - want).max(axis=1) / np.abs(want).max(axis=1)
        assert err.max() < 1e-12
        want_rank = 1 + (want[:, None, :] < want[:, :, None]).sum(axis=2)
        assert np.array_equal(rk[c], want_rank)


@pytest.mark.parametrize("E,H", [(8, 128), (16, 128), (24, 16), (48, 32), (64, 128), (100, 12), (128, 128)])
def test_scorer_ranks_match_scores(E, H):
    """K3's integer ranks against its own float64 scores for every expert
    count path (pairwise counts E <= 16, integer-key bitonic sort E <= 64,
    float64 sort above): rank = 1 + #{j : s_j < s_e}; ties share a rank.
    Nets with duplicated output rows force exact ties."""
    import ctypes

    import torch
    rng = np.random.default_rng(E + H)
    L, T, K = 2, 200, min(4, E)
    ids = np.stack([np.stack([rng.choice(E, K, replace=False) for _ in range(T)]) for _ in range(L)])
    packed = mcb.packed_from_decode_ids(ids.astype(np.uint8), E)
    net = mcb.EvictionNet(E, hidden=H, seed=E)
    net.params["w3"][E // 2] = net.params["w3"][0]      # expert E/2 always ties expert 0
    net.params["b3"][E // 2] = net.params["b3"][0]
    flat = net.flat_params()
    lib = _lib.load_library()
    dev_acc = torch.from_numpy(packed.acc).cuda()
    v = packed.view()
    v.acc = dev_acc.data_ptr()
    dparams = torch.from_numpy(flat).cuda()
    ns = _lib.MCBNets()
    ns.num_experts, ns.hidden, ns.num_nets, ns.params = E, H, 1, dparams.data_ptr()
    ranks = torch.zeros(packed.total_events * E + 64, dtype=torch.uint8, device="cuda")
    scores = torch.zeros(packed.total_events * E, dtype=torch.float64, device="cuda")
    _lib.check(lib.mcb_score(_lib.context(0), ctypes.byref(v), ctypes.byref(ns), 1, ranks.data_ptr(),
                             scores.data_ptr(), None))
    torch.cuda.synchronize()
    s = scores.cpu().numpy().reshape(-1, E)
    rk = ranks.cpu().numpy()[:packed.total_events * E].reshape(-1, E)
    want = 1 + (s[:, None, :] < s[:, :, None]).sum(axis=2)
    assert np.array_equal(rk, want)
    assert np.all(rk[:, E // 2] == rk[:, 0])


@pytest.mark.parametrize("E,K,T", [(64, 6, 64), (128, 8, 32), (32, 4, 100)])
def test_next_use_thread_walk_matches_numpy(E, K, T):
    """K2 for many chains (>= 8,192: one thread per chain, shared-memory table,
    vector loads / stores) against a vectorised numpy reference; T*K = 100*4
    is a multiple of 16, 64*6 = 384 and 32*8 = 256 too."""
    import ctypes

    import torch
    rng = np.random.default_rng(E + K)
    n_chains = 8300
    ids = np.argsort(rng.random((n_chains, T, E)), axis=2)[:, :, :K].astype(np.uint8)   # distinct per event
    packed = mcb.packed_from_decode_ids(ids[None], E)
    dev_acc = torch.from_numpy(packed.acc).cuda()
    v = packed.view()
    v.acc = dev_acc.data_ptr()
    out = torch.zeros(packed.total_acc + 64, dtype=torch.int32, device="cuda")
    lib = _lib.load_library()
    _lib.check(lib.mcb_next_use(_lib.context(0), ctypes.byref(v), out.data_ptr(), None))
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint32)[:packed.total_acc].reshape(n_chains, T * K).astype(np.int64)
    s = ids.reshape(n_chains, T * K).astype(np.int64)
    want = np.full(s.shape, 0xFFFFFFFF, dtype=np.int64)
    last = np.full((n_chains, E), 0xFFFFFFFF, dtype=np.int64)
    rows = np.arange(n_chains)
    for p in range(T * K - 1, -1, -1):
        want[:, p] = last[rows, s[:, p]]
        last[rows, s[:, p]] = p
    assert np.array_equal(got, want)
