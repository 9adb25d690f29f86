"""CPU-only tests: the C-ABI library loads and exports every symbol of
include/mcb.h; host-side validation/packing mirrors the reference's
RoutingTrace.validate and layer_schedules; API error behaviour; nets."""
import os
import re

import numpy as np
import pytest

import oracle
import paper_2601_17063_b200 as mcb
from golden_util import GOLDEN, case_trace, load
from paper_2601_17063_b200 import _lib
from paper_2601_17063_b200.trace import AccessEvent, Phase, RoutingTrace, TraceHeader

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D, P = Phase.DECODE, Phase.PREFILL


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "mcb.h")).read()
    return sorted(set(re.findall(r"\bint\s+(mcb_\w+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = _lib.load_library()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED_SYMBOLS)
    assert lib.mcb_abi_version() == 1


def tr(events, L=1, E=4, K=2):
    return RoutingTrace(TraceHeader("t", L, E, K), tuple(events))


@pytest.mark.parametrize("events,kw", [
    ([AccessEvent(-1, D, 0, 0, (0, 1))], {}),                       # seq_id < 0
    ([AccessEvent(0, D, -1, 0, (0, 1))], {}),                       # step < 0
    ([AccessEvent(0, D, 0, 1, (0, 1))], {}),                        # layer out of range
    ([AccessEvent(0, D, 0, 0, (1, 1))], {}),                        # duplicates
    ([AccessEvent(0, D, 0, 0, (0, 9))], {}),                        # expert out of range
    ([AccessEvent(0, D, 0, 0, (0,))], {}),                          # decode needs exactly K
    ([AccessEvent(0, P, 0, 0, ())], {}),                            # prefill needs >= 1
    ([AccessEvent(0, D, 1, 0, (0, 1)), AccessEvent(0, D, 0, 0, (0, 1))], {}),   # out of order
    ([AccessEvent(0, D, 0, 0, (0, 1))], {"L": 2}),                  # decode step missing a layer
    ([], {"K": 5}),                                                 # top_k > num_experts
    ([], {"L": 0}),                                                 # num_layers < 1
])
def test_validation_mirrors_reference(events, kw):
    """trace.py:57-137 failure modes raise InvalidConfigError natively."""
    with pytest.raises(mcb.InvalidConfigError):
        mcb.pack_trace(tr(events, **kw))


def test_validate_accepts_valid_and_reference_objects():
    t = tr([AccessEvent(0, P, 0, 0, (0, 1, 2)), AccessEvent(0, D, 0, 0, (3, 1))])
    t.validate()
    assert t.num_decode_steps() == 1


def test_pack_layer_schedules_match_oracle_streams():
    """Packing (prefill load-once dedup, positions, decode_index) equals the
    oracle's restatement of replay.layer_schedules on the golden random traces."""
    for case in load("small_cases.json.gz")["cases"][:80]:
        header, events = case_trace(case)
        L, E, K = header
        t = RoutingTrace(TraceHeader("g", L, E, K),
                         tuple(AccessEvent(s, Phase(p), st, l, tuple(x)) for s, p, st, l, x in events))
        packed = mcb.pack_trace(t)
        seq, phase, step, layer, off, experts = oracle.flatten_events(events)
        lens = np.zeros(L, dtype=np.int64)
        oracle.lib().orc_layer_lengths(L, E, len(seq), *[oracle._ptr(a) for a in (seq, phase, layer, off, experts)],
                                       oracle._ptr(lens))
        for l in range(L):
            assert len(packed.chain_accesses(l)) == lens[l]
        run = case["runs"][0]
        if "decisions" in run:
            # decisions are recorded per access in the same positions
            for l in range(L):
                assert len(run["decisions"][l]) == len(packed.chain_accesses(l))


def test_uniform_layout_for_decode_only_single_sequence():
    ev = [AccessEvent(0, D, s, l, ((s + l) % 4, (s + l + 1) % 4)) for s in range(5) for l in range(3)]
    p = mcb.pack_trace(tr(ev, L=3))
    assert p.uniform and p.events_per_chain == 5 and p.total_acc == 30
    for l in range(3):
        want = [x for s in range(5) for x in ((s + l) % 4, (s + l + 1) % 4)]
        assert p.chain_accesses(l).tolist() == want
    q = mcb.packed_from_decode_ids(np.array([[[0, 1], [2, 3]]], dtype=np.uint8), 4)
    assert q.uniform and q.total_acc == 4


def test_policy_factory_and_errors_without_gpu():
    assert mcb.policy_factory("lru")[0] == "lru"
    assert mcb.policy_factory("fifo")[1].code == _lib.MCB_FIFO      # FIFO runs on the GPU too
    with pytest.raises(mcb.SimulationError):
        mcb.policy_factory("nope")
    with pytest.raises(mcb.SimulationError):
        mcb.policy_factory("ml")                       # needs nets (engine.py:184-185)
    assert mcb.policy_factory("arc")[1].code == _lib.MCB_ARC
    name, ep = mcb.policy_factory("lecar")
    assert ep.code == _lib.MCB_LECAR and ep.lecar == (0.45, 0.005, 0)   # policies.py:333-341 defaults
    _, ep = mcb.policy_factory({"name": "lecar", "seed": 5, "learning_rate": 0.1})
    assert ep.lecar == (0.1, 0.005, 5)
    with pytest.raises(TypeError):
        mcb.policy_factory({"name": "lecar", "alpha": 1})
    with pytest.raises(mcb.SimulationError):
        mcb.policy_factory({"name": "lecar", "seed": "abc"})     # only integer seeds on the engine
    with pytest.raises(TypeError):
        mcb.policy_factory({"name": "lru", "seed": 1})
    name, ep = mcb.policy_factory({"name": "ml", "include_prefill": False}, nets=mcb.EvictionNet(4))
    assert name == "ml" and ep.code == _lib.MCB_ML_NO_PREFILL
    t = tr([AccessEvent(0, D, 0, 0, (0, 1))])
    with pytest.raises(mcb.CapacityTooSmallError):
        mcb.simulate(t, "lru", 1)
    with pytest.raises(mcb.SimulationError):
        mcb.simulate(t, "lru", 2, cost=mcb.CostModel(t_load_s=0))
    with pytest.raises(mcb.CapacityTooSmallError):
        mcb.sweep(t, ["lru"], [2, 1])


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_engine_refuses_to_run_without_gpu():
    """No CPU fallback: with no CUDA device the engine raises."""
    t = tr([AccessEvent(0, D, 0, 0, (0, 1))])
    with pytest.raises(_lib.EngineUnavailableError):
        mcb.simulate(t, "lru", 2)


def test_eviction_net_init_is_reference_identical():
    for E, H, seed in ((8, 128, 0), (64, 12, 3), (128, 128, 47)):
        assert np.array_equal(mcb.EvictionNet(E, H, seed).flat_params(), oracle.init_net_params(E, H, seed))


def test_evnet_round_trip(tmp_path):
    src = os.path.join(GOLDEN, "efficacy_net.evnet")
    if not os.path.exists(src):
        pytest.skip("efficacy net not generated")
    net = mcb.load_net(src)
    arr, E, H = oracle.load_evnet_params(src)
    assert net.num_experts == E == 64 and net.hidden == H
    assert np.array_equal(net.flat_params(), arr)
    out = tmp_path / "x.evnet"
    assert mcb.save_net(net, out) == os.path.getsize(src)
    assert open(out, "rb").read() == open(src, "rb").read()
    with pytest.raises(mcb.ShapeMismatchError):
        mcb.load_net(src, num_experts=8)


def test_cost_and_cache_size_helpers():
    assert mcb.step_latency_s(2, 8, mcb.CostModel()) == 6e-3                       # test_engine.py:55-65
    assert mcb.step_latency_s(0, 8, mcb.CostModel()) == 8 * 158e-6
    assert mcb.step_latency_s(3, 8, mcb.CostModel(loads_serial=False)) == 3e-3
    b = mcb.HardwareBudget(vram_bytes=10, nonexpert_bytes=2, all_experts_bytes=16, experts_per_layer=8)
    assert mcb.cache_size_calc(b) == 4


def test_lecar_random_stream_matches_python():
    """The engine's host-side MT19937 (mcb_lecar_random) reproduces CPython's
    random.Random(seed).random(), the stream LeCaRPolicy draws from
    (policies.py:347, 381)."""
    import random
    for seed in (0, 1, 7, 2**32 + 5, 12345678901, -3):
        r = random.Random(seed)
        want = np.array([r.random() for _ in range(2000)])
        assert np.array_equal(_lib.lecar_random(seed, 2000), want), seed


def test_trainer_input_errors_without_gpu():
    """EmptyDatasetError / ShapeMismatchError before any device work (net.py:214-221)."""
    from paper_2601_17063_b200 import train
    net = mcb.EvictionNet(4, hidden=8)
    with pytest.raises(train.EmptyDatasetError):
        train.train_eviction_net(net, np.zeros((0, 8)), np.zeros((0, 4)), np.zeros((0, 4), bool))
    with pytest.raises(mcb.ShapeMismatchError):
        train.train_eviction_net(net, np.zeros((3, 6)), np.zeros((3, 4)), np.zeros((3, 4), bool))
