"""Trace types of the drop-in surface and the packed HBM layout.

The dataclasses mirror the reference's data model (pkg/src/moecache/trace.py:
19-144: error hierarchy, ``Phase``, ``TraceHeader``, ``AccessEvent``,
``RoutingTrace``) so code written against ``moecache`` keeps working; the
engine also accepts the reference's own objects (duck-typed on ``header`` /
``events``).

``PackedTrace`` is what the B200 engine consumes: one access stream per
(trace, layer) chain, chain-major, uint8 expert ids (mcb.h ``mcb_trace``).
Validation and packing run natively (csrc/mcb_pack.cpp restates
RoutingTrace.validate and replay.layer_schedules).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from . import _lib


class TraceError(Exception):
    """Base class for trace-related failures (trace.py:19-20)."""


class InvalidConfigError(TraceError, ValueError):
    """A header / event / workload field is out of its legal range (trace.py:23-24)."""


class TraceParseError(TraceError):
    def __init__(self, line_no: int, message: str):
        self.line_no = line_no
        super().__init__(f"line {line_no}: {message}")


class HeaderMismatchError(TraceParseError):
    pass


class InsufficientTokensError(TraceError, ValueError):
    pass


class Phase(IntEnum):
    PREFILL = 0
    DECODE = 1


@dataclass(frozen=True)
class TraceHeader:
    model_name: str
    num_layers: int
    num_experts: int
    top_k: int

    def validate(self) -> None:
        if self.num_layers < 1:
            raise InvalidConfigError(f"num_layers must be >= 1, got {self.num_layers}")
        if self.num_experts < 1:
            raise InvalidConfigError(f"num_experts must be >= 1, got {self.num_experts}")
        if not 1 <= self.top_k <= self.num_experts:
            raise InvalidConfigError(
                f"top_k must satisfy 1 <= top_k <= num_experts, got top_k={self.top_k} "
                f"with num_experts={self.num_experts}")


@dataclass(frozen=True)
class AccessEvent:
    seq_id: int
    phase: Phase
    step: int
    layer: int
    experts: tuple

    def sort_key(self) -> tuple:
        return (self.seq_id, int(self.phase), self.step, self.layer)

    def validate(self, header: TraceHeader) -> None:
        """AccessEvent.validate (trace.py:80-106): the same checks, order and messages."""
        if self.seq_id < 0:
            raise InvalidConfigError(f"seq_id must be >= 0, got {self.seq_id}")
        if self.step < 0:
            raise InvalidConfigError(f"step must be >= 0, got {self.step}")
        if not 0 <= self.layer < header.num_layers:
            raise InvalidConfigError(f"layer {self.layer} out of range [0, {header.num_layers})")
        if len(set(self.experts)) != len(self.experts):
            raise InvalidConfigError(f"experts contain duplicates: {list(self.experts)}")
        for e in self.experts:
            if not 0 <= e < header.num_experts:
                raise InvalidConfigError(f"expert {e} out of range [0, {header.num_experts})")
        if self.phase == Phase.DECODE:
            if len(self.experts) != header.top_k:
                raise InvalidConfigError(f"decode event must route exactly top_k={header.top_k} experts, "
                                         f"got {len(self.experts)}")
        elif not 1 <= len(self.experts) <= header.num_experts:
            raise InvalidConfigError(f"prefill event must route between 1 and {header.num_experts} "
                                     f"experts, got {len(self.experts)}")


@dataclass(frozen=True)
class RoutingTrace:
    header: TraceHeader
    events: tuple

    def validate(self) -> None:
        """RoutingTrace.validate (trace.py:115-137), executed natively
        (mcb_validate_trace): the reference's checks and messages, no engine
        limits -- a 160-expert trace the reference accepts validates here too;
        only replaying it is refused (num_experts > 128)."""
        validate_trace(self)

    def num_decode_steps(self) -> int:
        return len({(ev.seq_id, ev.step) for ev in self.events if ev.phase == Phase.DECODE})

    def seq_ids(self) -> list:
        return sorted({ev.seq_id for ev in self.events})


def _flatten(trace):
    """RoutingTrace (ours or the reference's) -> flat event arrays."""
    evs = trace.events
    n = len(evs)
    seq = np.fromiter((e.seq_id for e in evs), dtype=np.int64, count=n)
    phase = np.fromiter((int(e.phase) for e in evs), dtype=np.uint8, count=n)
    step = np.fromiter((e.step for e in evs), dtype=np.int64, count=n)
    layer = np.fromiter((e.layer for e in evs), dtype=np.int32, count=n)
    lens = np.fromiter((len(e.experts) for e in evs), dtype=np.int64, count=n)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    experts = np.fromiter((x for e in evs for x in e.experts), dtype=np.int32, count=int(off[-1]))
    return seq, phase, step, layer, off, experts


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


class PackedTrace:
    """Chain-major packed trace (host numpy arrays; see mcb.h ``mcb_trace``).

    Attributes: num_layers, num_experts, top_k, num_traces, uniform,
    events_per_chain, acc (uint8, padded), and for the general layout
    chain_acc_off / chain_ev_off / chain_rt_off (int64), ev_info (uint32),
    routed (uint8).  ``decode_steps`` is num_decode_steps() per trace.
    """

    def __init__(self, *, num_layers, num_experts, top_k, num_traces, uniform, events_per_chain,
                 acc, total_acc, total_events, chain_acc_off=None, chain_ev_off=None,
                 chain_rt_off=None, ev_info=None, routed=None, decode_steps=None, handle=None):
        self.num_layers = int(num_layers)
        self.num_experts = int(num_experts)
        self.top_k = int(top_k)
        self.num_traces = int(num_traces)
        self.uniform = bool(uniform)
        self.events_per_chain = int(events_per_chain)
        self.acc = acc
        self.total_acc = int(total_acc)
        self.total_events = int(total_events)
        self.chain_acc_off = chain_acc_off
        self.chain_ev_off = chain_ev_off
        self.chain_rt_off = chain_rt_off
        self.ev_info = ev_info
        self.routed = routed
        self.decode_steps = decode_steps if decode_steps is not None else [0] * self.num_traces
        self._handle = handle

    @property
    def num_chains(self) -> int:
        return self.num_layers * self.num_traces

    def free(self):
        if self._handle is not None:
            _lib.load_library().mcb_packed_free(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def view(self) -> _lib.MCBTrace:
        """ctypes mcb_trace over the host arrays (valid while self is alive)."""
        v = _lib.MCBTrace()
        v.num_layers, v.num_experts, v.top_k = self.num_layers, self.num_experts, self.top_k
        v.num_traces, v.uniform = self.num_traces, int(self.uniform)
        v.events_per_chain, v.total_acc, v.total_events = self.events_per_chain, self.total_acc, self.total_events
        v.acc = self.acc.ctypes.data
        if not self.uniform:
            v.chain_acc_off = self.chain_acc_off.ctypes.data
            v.chain_ev_off = self.chain_ev_off.ctypes.data
            v.chain_rt_off = self.chain_rt_off.ctypes.data
            v.ev_info = self.ev_info.ctypes.data
            v.routed = self.routed.ctypes.data
        return v

    def positions(self, chain: int):
        """Per-access (tick, decode_index) of one chain (EvictionRecord fields)."""
        if self.uniform:
            T, K = self.events_per_chain, self.top_k
            t = np.repeat(np.arange(T, dtype=np.int64), K)
            return t, t.copy()
        a0, a1 = int(self.chain_acc_off[chain]), int(self.chain_acc_off[chain + 1])
        tick = np.zeros(a1 - a0, dtype=np.int64)
        dec = np.zeros(a1 - a0, dtype=np.int64)
        e0, e1 = int(self.chain_ev_off[chain]), int(self.chain_ev_off[chain + 1])
        info = self.ev_info[e0:e1]
        nacc = (info & 0x1FF).astype(np.int64)
        decode = ((info >> 30) & 1).astype(np.int64)
        ticks = np.arange(e1 - e0, dtype=np.int64)
        decs = np.concatenate([[0], np.cumsum(decode)[:-1]]) if e1 > e0 else np.zeros(0, np.int64)
        tick[:] = np.repeat(ticks, nacc)
        dec[:] = np.repeat(decs, nacc)
        return tick, dec

    def chain_accesses(self, chain: int) -> np.ndarray:
        if self.uniform:
            n = self.events_per_chain * self.top_k
            return self.acc[chain * n:(chain + 1) * n]
        return self.acc[int(self.chain_acc_off[chain]):int(self.chain_acc_off[chain + 1])]


def validate_trace(trace) -> None:
    """RoutingTrace.validate for ours or the reference's trace objects."""
    h = trace.header
    seq, phase, step, layer, off, experts = _flatten(trace)
    rc = _lib.load_library().mcb_validate_trace(int(h.num_layers), int(h.num_experts), int(h.top_k), len(seq),
                                                _ptr(seq), _ptr(phase), _ptr(step), _ptr(layer), _ptr(off),
                                                _ptr(experts))
    _lib.check(rc)


def pack_trace(trace) -> PackedTrace:
    """Validate (RoutingTrace.validate) and pack one trace natively."""
    if isinstance(trace, PackedTrace):
        return trace
    h = trace.header
    seq, phase, step, layer, off, experts = _flatten(trace)
    lib = _lib.load_library()
    handle = ctypes.c_void_p()
    rc = lib.mcb_pack_trace(int(h.num_layers), int(h.num_experts), int(h.top_k), len(seq), _ptr(seq),
                            _ptr(phase), _ptr(step), _ptr(layer), _ptr(off), _ptr(experts),
                            ctypes.byref(handle))
    _lib.check(rc)
    return _from_handle(handle)


def _from_handle(handle) -> PackedTrace:
    """PackedTrace over the arrays of a native mcb_packed handle."""
    lib = _lib.load_library()
    v = _lib.MCBTrace()
    tot_acc, tot_ev, tot_rt, dsteps = (ctypes.c_int64() for _ in range(4))
    _lib.check(lib.mcb_packed_view(handle, ctypes.byref(v), ctypes.byref(tot_acc), ctypes.byref(tot_ev),
                                   ctypes.byref(tot_rt), ctypes.byref(dsteps)))
    L = v.num_layers

    def arr(ptr, dtype, count):
        if not ptr or count <= 0:
            return np.zeros(max(count, 1), dtype=dtype)
        buf = (ctypes.c_char * (count * np.dtype(dtype).itemsize)).from_address(ptr)
        return np.frombuffer(buf, dtype=dtype, count=count)

    acc_len = (tot_acc.value + 127) // 128 * 128 + 128
    acc = arr(v.acc, np.uint8, acc_len)
    kw = {}
    if not v.uniform:
        kw = dict(chain_acc_off=arr(v.chain_acc_off, np.int64, L + 1),
                  chain_ev_off=arr(v.chain_ev_off, np.int64, L + 1),
                  chain_rt_off=arr(v.chain_rt_off, np.int64, L + 1),
                  ev_info=arr(v.ev_info, np.uint32, max(tot_ev.value, 1)),
                  routed=arr(v.routed, np.uint8, max(tot_rt.value, 1)))
    return PackedTrace(num_layers=L, num_experts=v.num_experts, top_k=v.top_k, num_traces=1,
                       uniform=v.uniform, events_per_chain=v.events_per_chain, acc=acc,
                       total_acc=tot_acc.value, total_events=tot_ev.value,
                       decode_steps=[dsteps.value], handle=handle, **kw)


def packed_from_decode_ids(ids, num_experts: int) -> PackedTrace:
    """Uniform packed batch from decode-only ids.

    ids: uint8 [n_traces][L][T][K] (chain-major already) or [L][T][K] for one
    trace.  Each trace is one sequence of T decode steps (num_decode_steps = T).
    """
    ids = np.asarray(ids, dtype=np.uint8)
    if ids.ndim == 3:
        ids = ids[None]
    n, L, T, K = ids.shape
    if not 1 <= K <= num_experts:
        raise InvalidConfigError(f"top_k must satisfy 1 <= top_k <= num_experts, got top_k={K} "
                                 f"with num_experts={num_experts}")
    if ids.size and int(ids.max()) >= num_experts:
        raise InvalidConfigError(f"expert {int(ids.max())} out of range [0, {num_experts})")
    flat = ids.reshape(-1)
    acc = np.zeros((flat.size + 127) // 128 * 128 + 128, dtype=np.uint8)
    acc[:flat.size] = flat
    return PackedTrace(num_layers=L, num_experts=num_experts, top_k=K, num_traces=n, uniform=True,
                       events_per_chain=T, acc=acc, total_acc=flat.size, total_events=n * L * T,
                       decode_steps=[T] * n)


def prefill_coverage(trace, token_counts) -> list:
    """Fraction of the expert pool touched by the first n prefill tokens
    (trace.py:443-476): for each n (ascending), the mean over (sequence,
    layer) of |distinct experts routed in the first n prefill events| / E."""
    counts = list(token_counts)
    if counts != sorted(counts) or any(n < 1 for n in counts):
        raise InvalidConfigError("token_counts must be ascending positive integers")
    groups: dict = {}
    for ev in trace.events:
        if ev.phase == Phase.PREFILL:
            groups.setdefault((ev.seq_id, ev.layer), []).append(ev.experts)
    if not groups:
        raise InsufficientTokensError("trace contains no prefill events")
    need = max(counts)
    for (seq_id, layer), rows in groups.items():
        if len(rows) < need:
            raise InsufficientTokensError(f"sequence {seq_id} layer {layer} has only {len(rows)} prefill "
                                          f"tokens, need {need}")
    E = trace.header.num_experts
    out = []
    for n in counts:
        fr = [len({x for row in rows[:n] for x in row}) / E for rows in groups.values()]
        out.append((n, float(np.mean(fr))))
    return out
