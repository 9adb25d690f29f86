"""Drop-in replay API backed by the B200 engine (libmcb.so).

Mirrors the reference's public engine surface (pkg/src/moecache/engine.py):
``CostModel``, ``step_latency_s``, ``SimReport``, ``EvictionRecord``,
``SimRun``, ``policy_factory``, ``run_simulation``, ``simulate``,
``refetch_rate``, ``sweep``, ``eviction_quality_duel``, ``HardwareBudget`` and
``cache_size_calc`` -- same names, argument meaning, result types and
exception types.  The replay itself (schedules, Belady next-use scan, ML
scoring, the per-access policy loop, refetch and latency accounting) runs in
CUDA; this module only packs inputs, calls the C ABI and assembles reports
exactly like engine.py:345-379.
"""
from __future__ import annotations

import ctypes
import threading
import warnings
import math
from dataclasses import asdict, dataclass
from typing import Optional, Sequence, Union

import numpy as np

from . import _lib
from .policies import NoEvictableError, PolicyDecision
from .trace import PackedTrace, Phase, pack_trace


class SimulationError(Exception):
    pass


class CapacityTooSmallError(SimulationError):
    """Cache capacity below top_k: one decode event cannot fit."""


@dataclass(frozen=True)
class CostModel:
    t_load_s: float = 3e-3
    t_compute_s: float = 158e-6
    loads_serial: bool = True
    ml_score_cost_s: float = 0.0

    def validate(self) -> None:
        if self.t_load_s <= 0 or self.t_compute_s <= 0:
            raise SimulationError("cost durations must be positive")
        if self.ml_score_cost_s < 0:
            raise SimulationError("ml_score_cost_s must be >= 0")


def step_latency_s(misses: int, num_accesses: int, cost: CostModel) -> float:
    """Overlap-rule latency of one (step, layer) cell (engine.py:58-62)."""
    if misses > 0:
        return (misses if cost.loads_serial else 1) * cost.t_load_s
    return num_accesses * cost.t_compute_s


@dataclass(frozen=True)
class HardwareBudget:
    vram_bytes: int
    nonexpert_bytes: int
    all_experts_bytes: int
    experts_per_layer: int

    def validate(self) -> None:
        if self.vram_bytes < 0 or self.nonexpert_bytes < 0:
            raise SimulationError("byte budgets must be non-negative")
        if self.all_experts_bytes <= 0:
            raise SimulationError("all_experts_bytes must be positive")
        if self.experts_per_layer < 1:
            raise SimulationError("experts_per_layer must be >= 1")


def cache_size_calc(budget: HardwareBudget) -> int:
    """Eq. (1): floor((vram - nonexpert) * E / all_experts_bytes), clamped to [0, E]."""
    budget.validate()
    size = math.floor((budget.vram_bytes - budget.nonexpert_bytes) * budget.experts_per_layer
                      / budget.all_experts_bytes)
    return max(0, min(budget.experts_per_layer, size))


@dataclass(frozen=True)
class SimReport:
    policy: str
    capacity: int
    hits: int
    misses: int
    hit_rate: float
    io_count: int
    decode_hits: int
    decode_misses: int
    decode_hit_rate: float
    prefill_hits: int
    prefill_misses: int
    compulsory_misses: int
    hit_rate_excl_compulsory: float
    evictions: int
    refetch_within_w: float
    window: int
    est_decode_latency_s: float
    est_prefill_latency_s: float
    tokens_per_second_est: float

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, d: dict) -> "SimReport":
        return cls(**d)


@dataclass(frozen=True)
class EvictionRecord:
    layer: int
    position: int
    tick: int
    decode_index: int
    victim: int


@dataclass
class SimRun:
    report: SimReport
    evictions: list
    decisions: Optional[dict] = None


POLICY_NAMES = ("lru", "lfu", "fifo", "arc", "lecar", "belady", "ml")
_CODES = {"lru": _lib.MCB_LRU, "lfu": _lib.MCB_LFU, "belady": _lib.MCB_BELADY, "fifo": _lib.MCB_FIFO,
          "arc": _lib.MCB_ARC, "lecar": _lib.MCB_LECAR}
_LECAR_DEFAULTS = (0.45, 0.005, 0)   # LeCaRPolicy.__init__ (policies.py:333-341)


class EnginePolicy:
    """What ``policy_factory`` resolves a spec to: an engine policy code plus
    the ML net lookup.  Calling it like the reference's per-layer factory
    (make(layer, capacity, header, oracle)) is not supported -- the engine has
    no per-access policy objects."""

    def __init__(self, name: str, code: int, nets=None, lecar=None):
        self.name = name
        self.code = code
        self.nets = nets
        self.lecar = lecar   # (learning_rate, discount_base, seed) for lecar

    @property
    def is_ml(self) -> bool:
        return self.code in _lib.ML_CODES

    def __call__(self, layer, capacity, header, oracle):
        raise SimulationError("per-access CachePolicy objects are not provided by the B200 engine; "
                              "pass the spec to run_simulation / sweep instead")


def policy_factory(spec: Union[str, dict], nets=None):
    """Resolve a policy spec (name or {"name": ..., params}) (engine.py:153-202)."""
    params = dict(spec) if isinstance(spec, dict) else {"name": spec}
    name = params.pop("name", None)
    if name not in POLICY_NAMES:
        raise SimulationError(f"unknown policy {name!r}; expected one of {POLICY_NAMES}")
    if name == "lecar":
        lr = params.pop("learning_rate", _LECAR_DEFAULTS[0])
        base = params.pop("discount_base", _LECAR_DEFAULTS[1])
        seed = params.pop("seed", _LECAR_DEFAULTS[2])
        if params:
            raise TypeError(f"unexpected lecar policy parameters {sorted(params)}")
        if not isinstance(seed, int) or isinstance(seed, bool):
            raise SimulationError("lecar: only integer seeds are supported by the B200 engine")
        if not float(base) >= 0.0:
            raise SimulationError("lecar: discount_base must be >= 0")
        return name, EnginePolicy(name, _lib.MCB_LECAR, lecar=(float(lr), float(base), int(seed)))
    if name == "ml":
        if nets is None:
            raise SimulationError("ml policy requires trained eviction nets")
        include_prefill = params.pop("include_prefill", True)
        if params:
            raise TypeError(f"unexpected ml policy parameters {sorted(params)}")
        code = _lib.MCB_ML if include_prefill else _lib.MCB_ML_NO_PREFILL
        return name, EnginePolicy(name, code, nets)
    if params:
        raise TypeError(f"unexpected {name} policy parameters {sorted(params)}")
    return name, EnginePolicy(name, _CODES[name])


def _resolve(policy, nets):
    if isinstance(policy, tuple):
        name, make = policy
        if not isinstance(make, EnginePolicy):
            raise SimulationError("custom policy factories are unsupported by the B200 engine")
        return name, make
    return policy_factory(policy, nets)


def _net_params(nets, num_layers: int, num_experts: int):
    """nets (one EvictionNet, a sequence or a dict keyed by layer) -> (H, n, flat)."""
    def flat(net):
        if hasattr(net, "flat_params"):
            return net.flat_params()
        return np.concatenate([np.ascontiguousarray(net.params[k], dtype=np.float64).ravel()
                               for k in ("w1", "b1", "w2", "b2", "w3", "b3")])

    def check(net):
        if net.num_experts != num_experts:
            raise ValueError(f"net scores {net.num_experts} experts, cache has {num_experts}")
        return net

    if hasattr(nets, "params") and hasattr(nets, "num_experts"):
        check(nets)
        return int(nets.hidden), 1, flat(nets)
    per = []
    for layer in range(num_layers):
        if isinstance(nets, dict):
            if layer not in nets:
                raise SimulationError(f"no eviction net provided for layer {layer}")
            per.append(check(nets[layer]))
        else:
            per.append(check(nets[layer]))
    hidden = {int(n.hidden) for n in per}
    if len(hidden) != 1:
        raise SimulationError("per-layer nets with different hidden sizes are unsupported by the B200 engine")
    return hidden.pop(), num_layers, np.concatenate([flat(n) for n in per])


def _cost_struct(cost: CostModel, window: int) -> _lib.MCBCost:
    c = _lib.MCBCost()
    c.t_load_s = float(cost.t_load_s)
    c.t_compute_s = float(cost.t_compute_s)
    c.ml_score_cost_s = float(cost.ml_score_cost_s)
    c.loads_serial = int(bool(cost.loads_serial))
    c.window = int(window)
    return c


_REPLAY_LOCKS: dict = {}
_REPLAY_LOCKS_GUARD = threading.Lock()


def _replay_lock(device: int) -> threading.Lock:
    with _REPLAY_LOCKS_GUARD:
        return _REPLAY_LOCKS.setdefault(device, threading.Lock())


class ScorerNearTieWarning(UserWarning):
    """Some events' float64 scores had two values within 1e-12 relative: the
    reference's own float64 BLAS order could rank them either way."""


def _warn_uncertain(device: int):
    """Surface float64 near ties of the last ML replay (mcb_last_stats): the
    engine ranks them with its own float64 scores (lowest id on exact ties),
    but a decision there is within the reference's rounding noise."""
    k, u = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.load_library().mcb_last_stats(_lib.context(device), ctypes.byref(k), ctypes.byref(u)))
    if u.value > 0:
        warnings.warn(f"{u.value} event(s) had float64 scores within 1e-12 relative of each other; their ML "
                      "decisions follow this engine's float64 scores and may differ from the reference's BLAS "
                      "rounding", ScorerNearTieWarning, stacklevel=3)


def replay_host(packed: PackedTrace, codes: Sequence[int], capacities: Sequence[int], cost: CostModel,
                window: int, nets=None, *, want_outcomes=False, want_hashes=False, want_chain=False,
                device: int = 0, stream=None, lecar=None) -> dict:
    """One native call: every trace of ``packed`` x codes x capacities.

    Returns numpy arrays: reports [trace][pol][cap][8] int64, latency
    [trace][pol][cap][2] float64, and optionally chain_reports
    [chain][pol][cap][8] + chain_latency [chain][pol][cap][2] (want_chain),
    hashes [chain][pol][cap], outcomes
    [pol][cap][total_acc] uint16.
    """
    lib = _lib.load_library()
    ctx = _lib.context(device)
    n_pol, n_cap = len(codes), len(capacities)
    nt = packed.num_traces
    reports = np.zeros((nt, n_pol, n_cap, _lib.R_N), dtype=np.int64)
    latency = np.zeros((nt, n_pol, n_cap, 2), dtype=np.float64)
    out = _lib.MCBOutputs()
    out.reports = reports.ctypes.data
    out.latency = latency.ctypes.data
    res = {"reports": reports, "latency": latency}
    if want_chain:
        res["chain_reports"] = np.zeros((packed.num_chains, n_pol, n_cap, _lib.R_N), dtype=np.int64)
        out.chain_reports = res["chain_reports"].ctypes.data
        res["chain_latency"] = np.zeros((packed.num_chains, n_pol, n_cap, 2), dtype=np.float64)
        out.chain_latency = res["chain_latency"].ctypes.data
    if want_hashes:
        res["hashes"] = np.zeros((packed.num_chains, n_pol, n_cap), dtype=np.uint64)
        out.hashes = res["hashes"].ctypes.data
    if want_outcomes:
        res["outcomes"] = np.zeros((n_pol, n_cap, max(packed.total_acc, 1)), dtype=np.uint16)
        out.outcomes = res["outcomes"].ctypes.data
    pols = (ctypes.c_int32 * n_pol)(*codes)
    caps = (ctypes.c_int32 * n_cap)(*capacities)
    netsp = None
    keep = None
    if nets is not None:
        hidden, n_nets, flat = nets
        keep = np.ascontiguousarray(flat, dtype=np.float64)
        ns = _lib.MCBNets()
        ns.num_experts, ns.hidden, ns.num_nets = packed.num_experts, hidden, n_nets
        ns.params = keep.ctypes.data
        netsp = ctypes.byref(ns)
    view = packed.view()
    cs = _cost_struct(cost, window)
    # LeCaR parameters live on the per-device context: hold the device's lock
    # from setting them through the replay so that concurrent callers with
    # other parameters cannot interleave (each reference cell owns its policy)
    with _replay_lock(device):
        if _lib.MCB_LECAR in codes:
            _lib.set_lecar(*(lecar or _LECAR_DEFAULTS), device=device)
        rc = lib.mcb_replay_host(ctx, ctypes.byref(view), pols, n_pol, caps, n_cap, ctypes.byref(cs), netsp,
                                 ctypes.byref(out), stream)
        _lib.check(rc)
        if any(c in _lib.ML_CODES for c in codes):
            _warn_uncertain(device)
    del keep
    return res


def assemble_report(name: str, capacity: int, window: int, counters, latency, decode_tokens: int) -> SimReport:
    """engine.py:345-379 from the engine's per-cell counters."""
    ph, pm, dh, dm, comp, ev, refc = (int(counters[i]) for i in range(7))
    hits, misses = ph + dh, pm + dm
    accesses = hits + misses
    noncomp = accesses - comp
    dlat, plat = float(latency[0]), float(latency[1])
    return SimReport(
        policy=name,
        capacity=capacity,
        hits=hits,
        misses=misses,
        hit_rate=hits / accesses if accesses else 0.0,
        io_count=misses,
        decode_hits=dh,
        decode_misses=dm,
        decode_hit_rate=dh / (dh + dm) if dh + dm else 0.0,
        prefill_hits=ph,
        prefill_misses=pm,
        compulsory_misses=comp,
        hit_rate_excl_compulsory=hits / noncomp if noncomp else 0.0,
        evictions=ev,
        refetch_within_w=refc / ev if ev else 0.0,
        window=window,
        est_decode_latency_s=dlat,
        est_prefill_latency_s=plat,
        tokens_per_second_est=decode_tokens / dlat if dlat > 0 else 0.0,
    )


def _raise_cell_status(status: int):
    if status == _lib.MCB_ERR_NO_EVICTABLE:
        raise NoEvictableError("no evictable expert: resident \\ pinned has no scorable candidate")
    if status != 0:
        raise SimulationError(f"engine cell failed with status {status}")


def _prepare(trace, cost: CostModel, capacities):
    packed = pack_trace(trace)   # RoutingTrace.validate() (engine.py:310)
    cost.validate()              # engine.py:311
    for c in capacities:
        if c < packed.top_k:
            raise CapacityTooSmallError(f"capacity {c} < top_k {packed.top_k}: a decode event cannot fit "
                                        "in the cache")
    return packed


def run_simulation(trace, policy, capacity: int, cost: CostModel = CostModel(), window: int = 5, nets=None,
                   record_decisions: bool = False) -> SimRun:
    """Replay the trace through per-layer caches and assemble a full report (engine.py:300-380)."""
    packed = _prepare(trace, cost, [capacity])
    name, ep = _resolve(policy, nets)
    netp = _net_params(ep.nets, packed.num_layers, packed.num_experts) if ep.is_ml else None
    res = replay_host(packed, [ep.code], [capacity], cost, window, netp, want_outcomes=True, lecar=ep.lecar)
    _raise_cell_status(int(res["reports"][0, 0, 0, _lib.R_STATUS]))
    report = assemble_report(name, capacity, window, res["reports"][0, 0, 0], res["latency"][0, 0, 0],
                             packed.decode_steps[0])
    outcomes = res["outcomes"][0, 0]
    evictions = []
    decisions = {} if record_decisions else None
    for layer in range(packed.num_layers):
        a0 = _chain_acc_begin(packed, layer)
        acc = packed.chain_accesses(layer)
        codes = outcomes[a0:a0 + len(acc)]
        ev_pos = np.nonzero(codes < 0xFFFE)[0]
        if len(ev_pos):
            tick, dec = packed.positions(layer)
            for p in ev_pos.tolist():
                evictions.append(EvictionRecord(layer, p, int(tick[p]), int(dec[p]), int(codes[p])))
        if record_decisions:
            decisions[layer] = [
                PolicyDecision(int(x), bool(c == 0xFFFF), None if c >= 0xFFFE else int(c))
                for x, c in zip(acc.tolist(), codes.tolist())]
    return SimRun(report, evictions, decisions)


def _chain_acc_begin(packed: PackedTrace, chain: int) -> int:
    if packed.uniform:
        return chain * packed.events_per_chain * packed.top_k
    return int(packed.chain_acc_off[chain])


def simulate(trace, policy, capacity: int, cost: CostModel = CostModel(), window: int = 5, nets=None) -> SimReport:
    """engine.py:383-391, without materialising the eviction log."""
    packed = _prepare(trace, cost, [capacity])
    name, ep = _resolve(policy, nets)
    netp = _net_params(ep.nets, packed.num_layers, packed.num_experts) if ep.is_ml else None
    res = replay_host(packed, [ep.code], [capacity], cost, window, netp, lecar=ep.lecar)
    _raise_cell_status(int(res["reports"][0, 0, 0, _lib.R_STATUS]))
    return assemble_report(name, capacity, window, res["reports"][0, 0, 0], res["latency"][0, 0, 0],
                           packed.decode_steps[0])


def refetch_rate(trace, policy, capacity: int, window: int = 5, nets=None) -> float:
    return simulate(trace, policy, capacity, window=window, nets=nets).refetch_within_w


def eviction_quality_duel(trace, policy_a, policy_b, capacity: int, nets=None) -> float:
    """Victim quality of policy A against policy B (engine.py:404-436).

    Both policies replay on the GPU (default cost and window, as the
    reference's run_simulation calls); K8 (mcb_eviction_duel) compares the
    victims' next uses (K2) at every access where both evict.  Returns the
    fraction of strict wins that are A's, or 0.5 without a strict winner."""
    import torch
    from .device import DeviceTrace
    cost = CostModel()
    packed = _prepare(trace, cost, [capacity])
    codes = []
    for policy in (policy_a, policy_b):
        name, ep = _resolve(policy, nets)
        netp = _net_params(ep.nets, packed.num_layers, packed.num_experts) if ep.is_ml else None
        res = replay_host(packed, [ep.code], [capacity], cost, 5, netp, want_outcomes=True, lecar=ep.lecar)
        _raise_cell_status(int(res["reports"][0, 0, 0, _lib.R_STATUS]))
        codes.append(res["outcomes"][0, 0])
    lib = _lib.load_library()
    ctx = _lib.context(0)
    dt = DeviceTrace.from_packed(packed)
    view = dt.view()
    stream = torch.cuda.current_stream(0)
    n = max(packed.total_acc, 1)
    next_pos = torch.empty(n + 64, dtype=torch.int32, device="cuda")
    outs = [torch.from_numpy(np.ascontiguousarray(c[:n]).view(np.int16)).to("cuda") for c in codes]
    wins = torch.zeros(2, dtype=torch.int64, device="cuda")
    _lib.check(lib.mcb_next_use(ctx, ctypes.byref(view), next_pos.data_ptr(), ctypes.c_void_p(stream.cuda_stream)))
    _lib.check(lib.mcb_eviction_duel(ctx, ctypes.byref(view), outs[0].data_ptr(), outs[1].data_ptr(),
                                     next_pos.data_ptr(), wins.data_ptr(), ctypes.c_void_p(stream.cuda_stream)))
    a, b = (int(v) for v in wins.cpu().tolist())
    return 0.5 if a + b == 0 else a / (a + b)


def sweep(trace, policies: Sequence, capacities: Sequence[int], cost: CostModel = CostModel(), window: int = 5,
          nets=None, jobs: int = 1) -> list:
    """Cross-product evaluation, rows ordered by (policy, capacity) (engine.py:439-465).

    The whole cross product is one engine call (chunks of <= 8 policies x
    <= 64 capacities): the trace, the Belady next-use scan and the ML scores
    are shared by every cell.  ``jobs`` is accepted for signature
    compatibility; the GPU runs every cell concurrently.
    """
    top_k = trace.top_k if isinstance(trace, PackedTrace) else trace.header.top_k
    for c in capacities:
        if c < top_k:
            raise CapacityTooSmallError(f"capacity {c} < top_k {top_k}")
    packed = _prepare(trace, cost, capacities)
    resolved = [_resolve(p, nets) for p in policies]
    netp = None
    if any(ep.is_ml for _, ep in resolved):
        netp = _net_params(next(ep.nets for _, ep in resolved if ep.is_ml),
                           packed.num_layers, packed.num_experts)
    reports = []
    caps = list(capacities)
    # one engine call per group of <= 8 policies; LeCaR parameters are per
    # call, so LeCaR specs with different parameters go to different calls
    groups: list[list[int]] = []
    for i, (_, ep) in enumerate(resolved):
        for g in groups:
            params = {resolved[k][1].lecar for k in g if resolved[k][1].lecar is not None}
            if len(g) < _MAX_POL and (ep.lecar is None or not params or params == {ep.lecar}):
                g.append(i)
                break
        else:
            groups.append([i])
    for g in groups:
        chunk = [resolved[i] for i in g]
        lecar = next((ep.lecar for _, ep in chunk if ep.lecar is not None), None)
        for c0 in range(0, len(caps), _MAX_CAP):
            cchunk = caps[c0:c0 + _MAX_CAP]
            res = replay_host(packed, [ep.code for _, ep in chunk], cchunk, cost, window, netp, lecar=lecar)
            for i, (name, _) in enumerate(chunk):
                for j, cap in enumerate(cchunk):
                    _raise_cell_status(int(res["reports"][0, i, j, _lib.R_STATUS]))
                    reports.append((g[i], c0 + j, assemble_report(
                        name, cap, window, res["reports"][0, i, j], res["latency"][0, i, j],
                        packed.decode_steps[0])))
    reports.sort(key=lambda t: (t[0], t[1]))   # policy-major cell order, as the reference builds it
    return sorted([r for _, _, r in reports], key=lambda r: (r.policy, r.capacity))


_MAX_POL, _MAX_CAP = 8, 64


__all__ = [
    "CapacityTooSmallError", "CostModel", "EvictionRecord", "HardwareBudget", "SimReport", "SimRun",
    "SimulationError", "cache_size_calc", "policy_factory", "refetch_rate",
    "run_simulation", "simulate", "step_latency_s", "sweep", "POLICY_NAMES", "replay_host",
    "eviction_quality_duel",
    "assemble_report", "Phase",
]
