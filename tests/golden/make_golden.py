"""Generate the golden parity fixtures by running the UNMODIFIED reference
simulator (``moecache`` from /root/reference/pkg/src) in this container.

Run from the repo root (only here; the GPU box has no /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Everything written under tests/golden/ is derived from the reference's own
public API (``generate_trace``, ``run_simulation``, ``EvictionNet``,
``train_eviction_net``) and its test helpers (``random_trace``,
pkg/tests/helpers.py:18-45).  The fixtures pin the C oracle (oracle/) and the
CUDA engine: full ``SimReport`` equality (floats included), and per-layer
decision hashes (FNV-1a 64 over u16 outcome codes, see ``outcome_code``).
"""
from __future__ import annotations

import gzip
import json
import os
import random
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

import moecache  # noqa: E402
from moecache import (  # noqa: E402
    AccessEvent,
    CostModel,
    EvictionNet,
    Phase,
    RoutingTrace,
    SyntheticWorkloadConfig,
    TraceHeader,
    build_training_data,
    generate_trace,
    run_simulation,
    save_net,
    train_eviction_net,
    TrainConfig,
)
from helpers import random_trace  # noqa: E402  (pkg/tests/helpers.py:18)

OUT = os.path.dirname(os.path.abspath(__file__))

HIT, MISS = 0xFFFF, 0xFFFE
FNV_OFF, FNV_PRIME, M64 = 0xCBF29CE484222325, 0x100000001B3, (1 << 64) - 1

COSTS = {
    "default": CostModel(),
    "overlap_ml": CostModel(t_load_s=2.5e-3, t_compute_s=1.7e-4, loads_serial=False,
                            ml_score_cost_s=1e-4),
}


def outcome_code(d) -> int:
    if d.was_hit:
        return HIT
    return MISS if d.evicted is None else int(d.evicted)


def fnv_hash(codes) -> int:
    h = FNV_OFF
    for c in codes:
        for b in (c & 0xFF, c >> 8):
            h ^= b
            h = (h * FNV_PRIME) & M64
    return h


def trace_to_json(trace: RoutingTrace) -> dict:
    h = trace.header
    return {
        "header": [h.model_name, h.num_layers, h.num_experts, h.top_k],
        "events": [[e.seq_id, int(e.phase), e.step, e.layer, list(e.experts)] for e in trace.events],
    }


def make_nets(spec: dict, num_layers: int, num_experts: int):
    if spec is None:
        return None
    kind = spec["kind"]
    hidden = spec.get("hidden", 128)
    if kind == "per_layer_seed":
        return [EvictionNet(num_experts, hidden=hidden, seed=l) for l in range(num_layers)]
    if kind == "shared_seed":
        return EvictionNet(num_experts, hidden=hidden, seed=spec["seed"])
    if kind == "evnet":
        return moecache.load_net(os.path.join(OUT, spec["file"]))
    raise ValueError(kind)


def run_case(trace, policy, capacity, cost_name, window, net_spec, with_decisions):
    nets = make_nets(net_spec, trace.header.num_layers, trace.header.num_experts)
    t0 = time.perf_counter()
    run = run_simulation(trace, policy, capacity, COSTS[cost_name], window, nets,
                         record_decisions=True)
    dt = time.perf_counter() - t0
    codes = {l: [outcome_code(d) for d in run.decisions[l]] for l in run.decisions}
    out = {
        "policy": policy,
        "capacity": capacity,
        "cost": cost_name,
        "window": window,
        "nets": net_spec,
        "report": run.report.to_dict(),
        "hashes": [format(fnv_hash(codes[l]), "016x") for l in range(trace.header.num_layers)],
        "n_evictions": len(run.evictions),
        "ref_seconds": dt,
    }
    if with_decisions:
        out["decisions"] = [codes[l] for l in range(trace.header.num_layers)]
        out["eviction_records"] = [
            [r.layer, r.position, r.tick, r.decode_index, r.victim] for r in run.evictions
        ]
    return out


def ml_spec(include_prefill=True):
    return "ml" if include_prefill else {"name": "ml", "include_prefill": False}


def suite_random():
    """Uniform random traces with prefill + several sequences (helpers.random_trace)."""
    cases = []
    for seed in range(60):
        trace = random_trace(random.Random(seed))
        h = trace.header
        runs = []
        caps = sorted({h.top_k, max(h.top_k, 3), h.num_experts, h.num_experts + 2})
        for cap in caps:
            for policy in ("lru", "lfu", "belady"):
                runs.append(run_case(trace, policy, cap, "default", 5, None, True))
            hidden = 12 if seed % 2 else 128
            runs.append(run_case(trace, "ml", cap, "default", 5,
                                 {"kind": "per_layer_seed", "hidden": hidden}, True))
            runs.append(run_case(trace, ml_spec(False), cap, "overlap_ml", 2,
                                 {"kind": "shared_seed", "seed": seed, "hidden": hidden}, True))
        runs.append(run_case(trace, "lru", max(h.top_k, 2), "overlap_ml", 0, None, True))
        cases.append({"name": f"random{seed}", "trace": trace_to_json(trace), "runs": runs})
    return cases


def suite_bruteforce():
    """test_acceptance.py:136-162 trace family (1 layer, up to 20 decode steps)."""
    cases = []
    for seed in range(100):
        rng = random.Random(seed)
        trace = random_trace(rng, num_layers=1, num_experts=rng.randint(4, 10), max_seqs=2,
                             max_prefill=3, max_decode=20)
        capacity = max(trace.header.top_k, rng.randint(2, 5))
        runs = [run_case(trace, p, capacity, "default", 5, None, True)
                for p in ("lru", "lfu", "belady")]
        runs.append(run_case(trace, "ml", capacity, "default", 5,
                             {"kind": "shared_seed", "seed": seed, "hidden": 16}, True))
        cases.append({"name": f"brute{seed}", "trace": trace_to_json(trace), "runs": runs})
    return cases


def handmade_traces():
    """Hand-built traces from pkg/tests/test_engine.py:94-196."""
    def mk(events, E, K, L=1):
        return RoutingTrace(TraceHeader("hand", L, E, K), tuple(events))
    D, P = Phase.DECODE, Phase.PREFILL
    return {
        "thrash": (mk([AccessEvent(0, D, s, 0, (0, 1) if s % 2 == 0 else (2, 3)) for s in range(40)], 4, 2), [2]),
        "prefill_union": (mk([AccessEvent(0, P, 0, 0, (0, 1)), AccessEvent(0, P, 1, 0, (1, 2))], 8, 2), [4]),
        "prefill_reload": (mk([AccessEvent(0, P, 0, 0, (0, 1)), AccessEvent(1, P, 0, 0, (0, 1))], 8, 2), [4]),
        "refetch_075": (mk([AccessEvent(0, D, 0, 0, (0, 1)), AccessEvent(0, D, 1, 0, (1, 2)),
                            AccessEvent(0, D, 2, 0, (0, 1)), AccessEvent(0, D, 3, 0, (1, 2))], 4, 2), [2]),
        "window0": (mk([AccessEvent(0, D, 0, 0, (0, 1)), AccessEvent(0, D, 1, 0, (2, 3)),
                        AccessEvent(0, D, 2, 0, (0, 1))], 4, 2), [2]),
        "empty_prefill": (mk([AccessEvent(0, P, 0, 0, (0, 1)), AccessEvent(0, P, 1, 0, (1, 0)),
                              AccessEvent(0, D, 0, 0, (3, 1)), AccessEvent(1, P, 0, 0, (2,)),
                              AccessEvent(1, D, 0, 0, (0, 2))], 5, 2), [2, 3]),
        "two_layer": (mk([AccessEvent(0, D, s, l, ((s + l) % 6, (s + l + 1 + s % 5) % 6))
                          for s in range(30) for l in range(2)], 6, 2, 2), [2, 3, 4]),
    }


def suite_handmade():
    cases = []
    for name, (trace, caps) in handmade_traces().items():
        trace.validate()
        runs = []
        for cap in caps:
            for policy in ("lru", "lfu", "belady"):
                for window in (0, 2, 5):
                    runs.append(run_case(trace, policy, cap, "default", window, None, True))
            runs.append(run_case(trace, "ml", cap, "default", 5,
                                 {"kind": "shared_seed", "seed": 3, "hidden": 8}, True))
        cases.append({"name": name, "trace": trace_to_json(trace), "runs": runs})
    return cases


def zipf(seed, L, E, K, seqs, decode, prefill, pop_seed=None):
    return generate_trace(
        TraceHeader("synthetic", L, E, K),
        SyntheticWorkloadConfig(num_seqs=seqs, decode_steps=decode, prefill_tokens=prefill,
                                zipf_s=1.0, recency_boost=0.3, w_hot=4, rng_seed=seed,
                                popularity_seed=pop_seed),
    )


def suite_zipf():
    """SURVEY.md Appendix B.1 family: L2/E64/K8, 2 sequences, 16 prefill + 150 decode."""
    cases = []
    for seed in range(6):
        trace = zipf(seed, 2, 64, 8, 2, 150, 16)
        runs = []
        for cap in (8, 16, 32, 48):
            for policy in ("lru", "lfu", "belady"):
                runs.append(run_case(trace, policy, cap, "default", 5, None, False))
            runs.append(run_case(trace, "ml", cap, "default", 5, {"kind": "per_layer_seed"}, False))
            runs.append(run_case(trace, ml_spec(False), cap, "overlap_ml", 5,
                                 {"kind": "per_layer_seed"}, False))
        cases.append({"name": f"zipf{seed}", "trace": trace_to_json(trace), "runs": runs})
    return cases


def suite_dominance():
    """test_acceptance.py:48-99 grid (L x E x K x 3 seeds, C in 25/50/75% of E)."""
    cases = []
    for L in (1, 2, 4):
        for E in (8, 64):
            for K in (2, 8):
                caps = [c for c in (E // 4, E // 2, 3 * E // 4) if c >= K]
                if not caps:
                    continue
                for seed in range(3):
                    trace = zipf(1000 + seed, L, E, K, 2, 60, 8)
                    runs = []
                    for cap in caps:
                        for policy in ("lru", "lfu", "belady"):
                            runs.append(run_case(trace, policy, cap, "default", 5, None, False))
                        runs.append(run_case(trace, "ml", cap, "default", 5,
                                             {"kind": "shared_seed", "seed": 0}, False))
                    cases.append({"name": f"dom_L{L}E{E}K{K}s{seed}", "trace": trace_to_json(trace),
                                  "runs": runs})
    return cases


def decode_only_ids(trace: RoutingTrace) -> np.ndarray:
    """[T][L][K] uint8 ids of a decode-only single-sequence trace (event order)."""
    h = trace.header
    ids = np.array([e.experts for e in trace.events], dtype=np.uint8)
    return ids.reshape(-1, h.num_layers, h.top_k)


def big_case(name, L, E, K, T, seed, caps, policies, net_spec):
    t0 = time.perf_counter()
    trace = zipf(seed, L, E, K, 1, T, 0)
    gen_s = time.perf_counter() - t0
    ids = decode_only_ids(trace)
    np.savez_compressed(os.path.join(OUT, f"{name}_trace.npz"), ids=ids,
                        header=np.array([L, E, K, T, seed], dtype=np.int64))
    runs = []
    for cap in caps:
        for policy in policies:
            ns = net_spec if policy == "ml" else None
            r = run_case(trace, policy, cap, "default", 5, ns, False)
            print(f"  {name} {policy} C={cap}: {r['report']['hits']}/{r['report']['misses']} "
                  f"{r['ref_seconds']:.2f}s", flush=True)
            runs.append(r)
    return {"name": name, "trace_npz": f"{name}_trace.npz", "generate_seconds": gen_s,
            "config": {"L": L, "E": E, "K": K, "T": T, "rng_seed": seed, "zipf_s": 1.0,
                       "recency_boost": 0.3, "w_hot": 4, "prefill_tokens": 0},
            "runs": runs}


def suite_efficacy():
    """test_acceptance.py:223-275: train on 3 family traces, evaluate on 10 held-out."""
    header = TraceHeader("efficacy", 1, 64, 8)

    def cfg(seed, seqs, decode):
        return SyntheticWorkloadConfig(num_seqs=seqs, decode_steps=decode, prefill_tokens=32,
                                       zipf_s=1.0, recency_boost=0.3, w_hot=4, rng_seed=seed,
                                       popularity_seed=7)
    t0 = time.perf_counter()
    feats, targs, masks = [], [], []
    for s in (101, 102, 103):
        ds = build_training_data(generate_trace(header, cfg(s, 8, 2500)), capacity=64,
                                 distance_cap=64)[0]
        feats.append(ds.features); targs.append(ds.targets); masks.append(ds.masks)
    net = EvictionNet(64, seed=0)
    train_eviction_net(net, np.concatenate(feats), np.concatenate(targs), np.concatenate(masks),
                       TrainConfig(seed=0))
    save_net(net, os.path.join(OUT, "efficacy_net.evnet"))
    print(f"  efficacy net trained in {time.perf_counter() - t0:.1f}s", flush=True)
    cases = []
    for s in range(201, 211):
        trace = generate_trace(header, cfg(s, 1, 800))
        runs = []
        for policy in ("ml", "lru", "lfu"):
            ns = {"kind": "evnet", "file": "efficacy_net.evnet"} if policy == "ml" else None
            runs.append(run_case(trace, policy, 32, "default", 5, ns, False))
        cases.append({"name": f"eff{s}", "trace": trace_to_json(trace), "runs": runs})
    means = {p: float(np.mean([c["runs"][i]["report"]["hit_rate"] for c in cases]))
             for i, p in enumerate(("ml", "lru", "lfu"))}
    print("  efficacy means", means, flush=True)
    return cases, means


def dump(name, obj):
    path = os.path.join(OUT, name)
    with gzip.open(path, "wt") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)", flush=True)


def main(which):
    meta = {"reference": "/root/reference (moecache 0.1.0)", "numpy": np.__version__,
            "python": sys.version.split()[0]}
    if "small" in which:
        dump("small_cases.json.gz", {"meta": meta, "cases": suite_handmade() + suite_random()
                                     + suite_bruteforce()})
    if "zipf" in which:
        dump("zipf_cases.json.gz", {"meta": meta, "cases": suite_zipf() + suite_dominance()})
    if "big" in which:
        c1 = big_case("c1_qwen3", 48, 128, 8, 2048, 0, [32], ("lru", "lfu", "belady", "ml"),
                      {"kind": "per_layer_seed"})
        mix = big_case("mixtral_2k", 32, 8, 2, 2048, 0, [2, 3, 4, 5, 6, 7],
                       ("lru", "lfu", "belady", "ml"), {"kind": "per_layer_seed"})
        dump("big_cases.json.gz", {"meta": meta, "cases": [c1, mix]})
    if "efficacy" in which:
        cases, means = suite_efficacy()
        dump("efficacy_cases.json.gz", {"meta": meta, "cases": cases, "means": means,
                                        "logged": "pkg/test_output.txt:360 ml 82.90 lru 81.30 lfu 79.78"})


if __name__ == "__main__":
    main(sys.argv[1:] or ["small", "zipf", "big", "efficacy"])
