"""Trace files: the reference's line-delimited JSON format and a binary
container for traces at scale.

JSONL (pkg/src/moecache/trace.py:290-417) is kept byte-compatible for
interop with the extractor (pkg/extractor/src/trace_extractor/extractor.py:
303-331): ``trace_to_text`` / ``write_trace`` produce the same bytes and
``parse_trace`` / ``read_trace`` accept and reject exactly what the reference
does, raising the same exception types with the same 1-based line numbers
and messages.

The binary container (``.mcbt``) stores a trace column-wise so that loading
is a few ``np.fromfile`` reads instead of one ``json.loads`` per event:

    offset  size  field
    0       8     magic b"MCBTRACE"
    8       4     version (1)
    12      4     kind: 0 = general events, 1 = decode-only batch
    16      4*4   num_layers, num_experts, top_k, name_len (bytes, UTF-8)
    32      8*3   general: n_events, n_experts_total, 0
                  batch:   n_traces, decode_steps, 0
    56      name_len   model name, then zero padding to a multiple of 8
    general kind: seq_id int64[n], step int64[n], layer int32[n],
                  phase uint8[n], (pad to 8), exp_off int64[n + 1],
                  experts uint8[n_experts_total]
    batch kind:   ids uint8[n_traces][decode_steps][num_layers][top_k] --
                  each trace one sequence (seq_id 0) of decode events in the
                  reference's event order (step-major, then layer).

The batch kind is the at-scale form (the BASELINE workloads are decode-only
batches): ``load_packed`` moves the ids to the GPU, where one kernel
(mcb_pack_decode_ids, K7) validates every event exactly as
AccessEvent.validate does (experts in range, no duplicates) and transposes
the event-order ids into the engine's chain-major layout.  A general file
is validated and packed by the native host packer (mcb_pack_trace).
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

from . import _lib
from .trace import (AccessEvent, HeaderMismatchError, InvalidConfigError, PackedTrace, Phase, RoutingTrace,
                    TraceHeader, TraceParseError)

# ----------------------------------------------------------------- JSONL ----

_HEADER_KEYS = ("model_name", "num_layers", "num_experts", "top_k")
_EVENT_KEYS = ("seq_id", "phase", "step", "layer", "experts")
_COMPACT = (",", ":")


def _header_line(h) -> str:
    return json.dumps({k: getattr(h, k) for k in _HEADER_KEYS}, separators=_COMPACT)


def _event_line(ev) -> str:
    rec = {"seq_id": ev.seq_id, "phase": int(ev.phase), "step": ev.step, "layer": ev.layer,
           "experts": list(ev.experts)}
    return json.dumps(rec, separators=_COMPACT)


def trace_to_text(trace) -> str:
    """One header line, one line per event, trailing newline (trace.py:323-326)."""
    out = [_header_line(trace.header)]
    out += [_event_line(ev) for ev in trace.events]
    return "\n".join(out) + "\n"


def write_trace(trace, path) -> None:
    """Validate, then write UTF-8 with '\\n' line ends (trace.py:329-332)."""
    trace.validate()
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write(trace_to_text(trace))


def _record(line_no: int, line: str, keys: tuple, kind: str) -> dict:
    try:
        rec = json.loads(line)
    except json.JSONDecodeError as exc:
        raise TraceParseError(line_no, f"invalid JSON in {kind} record: {exc.msg}") from exc
    if not isinstance(rec, dict):
        raise TraceParseError(line_no, f"{kind} record must be a JSON object")
    extra = set(rec) - set(keys)
    if extra:
        raise TraceParseError(line_no, f"unknown fields {sorted(extra)} in {kind} record")
    absent = set(keys) - set(rec)
    if absent:
        raise TraceParseError(line_no, f"missing fields {sorted(absent)} in {kind} record")
    return rec


def _is_int(v) -> bool:
    return isinstance(v, int) and not isinstance(v, bool)


def _int_field(line_no: int, rec: dict, key: str) -> int:
    v = rec[key]
    if not _is_int(v):
        raise TraceParseError(line_no, f"field '{key}' must be an integer, got {v!r}")
    return v


def _event_problem(ev: AccessEvent, h: TraceHeader):
    """AccessEvent.validate (trace.py:80-106): None, or (message, header_mismatch)
    where header_mismatch is parse_trace's classification (trace.py:390-395):
    the layer is >= num_layers or some expert is outside [0, num_experts)."""
    n = len(ev.experts)
    checks = (
        (ev.seq_id < 0, lambda: f"seq_id must be >= 0, got {ev.seq_id}"),
        (ev.step < 0, lambda: f"step must be >= 0, got {ev.step}"),
        (not 0 <= ev.layer < h.num_layers, lambda: f"layer {ev.layer} out of range [0, {h.num_layers})"),
        (len(set(ev.experts)) != n, lambda: f"experts contain duplicates: {list(ev.experts)}"),
    )
    msg = next((m() for failed, m in checks if failed), None)
    if msg is None:
        bad = [e for e in ev.experts if not 0 <= e < h.num_experts]
        if bad:
            msg = f"expert {bad[0]} out of range [0, {h.num_experts})"
        elif ev.phase == Phase.DECODE and n != h.top_k:
            msg = f"decode event must route exactly top_k={h.top_k} experts, got {n}"
        elif ev.phase != Phase.DECODE and not 1 <= n <= h.num_experts:
            msg = f"prefill event must route between 1 and {h.num_experts} experts, got {n}"
    if msg is None:
        return None
    mismatch = ev.layer >= h.num_layers or any(e >= h.num_experts or e < 0 for e in ev.experts)
    return msg, mismatch


def parse_trace(text: str) -> RoutingTrace:
    """Parse the JSONL format (trace.py:350-412) with the reference's errors."""
    lines = text.splitlines()
    if not lines or not lines[0].strip():
        raise TraceParseError(1, "missing header record")
    rec = _record(1, lines[0], _HEADER_KEYS, "header")
    if not isinstance(rec["model_name"], str):
        raise TraceParseError(1, "field 'model_name' must be a string")
    header = TraceHeader(rec["model_name"], *(_int_field(1, rec, k) for k in _HEADER_KEYS[1:]))
    try:
        header.validate()
    except InvalidConfigError as exc:
        raise TraceParseError(1, str(exc)) from exc

    events = []
    last = None
    tokens: dict = {}   # decode (seq, step) -> [first line, set of layers]
    for line_no in range(2, len(lines) + 1):
        line = lines[line_no - 1]
        if not line.strip():
            raise TraceParseError(line_no, "blank line inside trace")
        rec = _record(line_no, line, _EVENT_KEYS, "event")
        phase = _int_field(line_no, rec, "phase")
        if phase not in (0, 1):
            raise TraceParseError(line_no, f"phase must be 0 (prefill) or 1 (decode), got {phase}")
        experts = rec["experts"]
        if not isinstance(experts, list) or not all(_is_int(e) for e in experts):
            raise TraceParseError(line_no, "field 'experts' must be a list of integers")
        ev = AccessEvent(_int_field(line_no, rec, "seq_id"), Phase(phase), _int_field(line_no, rec, "step"),
                         _int_field(line_no, rec, "layer"), tuple(experts))
        problem = _event_problem(ev, header)
        if problem is not None:
            msg, mismatch = problem
            raise (HeaderMismatchError if mismatch else TraceParseError)(line_no, msg)
        key = ev.sort_key()
        if last is not None and key <= last:
            raise TraceParseError(line_no, "events out of order; must be strictly increasing by "
                                           "(seq_id, phase, step, layer)")
        last = key
        if ev.phase == Phase.DECODE:
            tokens.setdefault((ev.seq_id, ev.step), [line_no, set()])[1].add(ev.layer)
        events.append(ev)
    for (seq, step), (first, layers) in tokens.items():
        if len(layers) != header.num_layers:
            missing = sorted(set(range(header.num_layers)) - layers)
            raise TraceParseError(first, f"decode step (seq {seq}, step {step}) missing events "
                                         f"for layers {missing}")
    return RoutingTrace(header, tuple(events))


def read_trace(path) -> RoutingTrace:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_trace(fh.read())


# ---------------------------------------------------------------- binary ----

MAGIC = b"MCBTRACE"
VERSION = 1
KIND_GENERAL, KIND_BATCH = 0, 1
_FIXED = 56


def _pad8(n: int) -> int:
    return (n + 7) // 8 * 8


def _write_header(fh, kind, L, E, K, name: str, a: int, b: int):
    nb = name.encode("utf-8")
    fh.write(MAGIC)
    fh.write(np.array([VERSION, kind, L, E, K, len(nb)], dtype="<u4").tobytes())
    fh.write(np.array([a, b, 0], dtype="<i8").tobytes())
    fh.write(nb + b"\0" * (_pad8(len(nb)) - len(nb)))


def write_trace_binary(trace, path) -> None:
    """Write a validated trace as a general-kind ``.mcbt`` file."""
    trace.validate()
    h = trace.header
    evs = trace.events
    n = len(evs)
    off = np.zeros(n + 1, dtype="<i8")
    np.cumsum([len(e.experts) for e in evs], out=off[1:])
    if h.num_experts > 256:
        raise InvalidConfigError("the binary container stores expert ids as uint8 (num_experts <= 256)")
    with open(path, "wb") as fh:
        _write_header(fh, KIND_GENERAL, h.num_layers, h.num_experts, h.top_k, h.model_name, n, int(off[-1]))
        fh.write(np.fromiter((e.seq_id for e in evs), dtype="<i8", count=n).tobytes())
        fh.write(np.fromiter((e.step for e in evs), dtype="<i8", count=n).tobytes())
        fh.write(np.fromiter((e.layer for e in evs), dtype="<i4", count=n).tobytes())
        ph = np.fromiter((int(e.phase) for e in evs), dtype=np.uint8, count=n).tobytes()
        fh.write(ph + b"\0" * (_pad8(4 * n + n) - 4 * n - n))
        fh.write(off.tobytes())
        fh.write(np.fromiter((x for e in evs for x in e.experts), dtype=np.uint8, count=int(off[-1])).tobytes())


def write_batch_binary(ids, num_experts: int, path, model_name: str = "batch") -> None:
    """Write decode-only traces ids uint8 [n_traces][decode_steps][L][K] (event order)."""
    ids = np.ascontiguousarray(ids, dtype=np.uint8)
    if ids.ndim == 3:
        ids = ids[None]
    n, T, L, K = ids.shape
    with open(path, "wb") as fh:
        _write_header(fh, KIND_BATCH, L, num_experts, K, model_name, n, T)
        fh.write(ids.tobytes())


class BinaryTraceInfo:
    def __init__(self, kind, L, E, K, name, a, b, data_offset):
        self.kind, self.num_layers, self.num_experts, self.top_k = kind, L, E, K
        self.model_name, self.data_offset = name, data_offset
        if kind == KIND_GENERAL:
            self.n_events, self.n_experts_total = a, b
        else:
            self.n_traces, self.decode_steps = a, b


def read_binary_info(path) -> BinaryTraceInfo:
    with open(path, "rb") as fh:
        head = fh.read(_FIXED)
        if len(head) < _FIXED or head[:8] != MAGIC:
            raise TraceParseError(1, "not an .mcbt trace file")
        ver, kind, L, E, K, nl = np.frombuffer(head[8:32], dtype="<u4").tolist()
        if ver != VERSION or kind not in (KIND_GENERAL, KIND_BATCH):
            raise TraceParseError(1, f"unsupported .mcbt version {ver} / kind {kind}")
        a, b, _ = np.frombuffer(head[32:56], dtype="<i8").tolist()
        name = fh.read(nl).decode("utf-8")
    TraceHeader(name, L, E, K).validate()
    if a < 0 or b < 0:
        raise TraceParseError(1, "negative sizes in .mcbt header")
    return BinaryTraceInfo(kind, L, E, K, name, a, b, _FIXED + _pad8(nl))


def _general_columns(path, info):
    n, m = info.n_events, info.n_experts_total
    o = info.data_offset
    seq = np.fromfile(path, dtype="<i8", count=n, offset=o); o += 8 * n
    step = np.fromfile(path, dtype="<i8", count=n, offset=o); o += 8 * n
    layer = np.fromfile(path, dtype="<i4", count=n, offset=o); o += 4 * n
    phase = np.fromfile(path, dtype=np.uint8, count=n, offset=o); o += _pad8(5 * n) - 4 * n
    off = np.fromfile(path, dtype="<i8", count=n + 1, offset=o); o += 8 * (n + 1)
    experts = np.fromfile(path, dtype=np.uint8, count=m, offset=o)
    if len(experts) != m or len(off) != n + 1 or int(off[0]) != 0 or int(off[-1]) != m or \
            np.any(np.diff(off) < 0):
        raise TraceParseError(1, "truncated or corrupt .mcbt event columns")
    return seq, phase, step, layer, off, experts


def _batch_ids(path, info):
    n = info.n_traces * info.decode_steps * info.num_layers * info.top_k
    ids = np.fromfile(path, dtype=np.uint8, count=n, offset=info.data_offset)
    if len(ids) != n:
        raise TraceParseError(1, "truncated .mcbt batch")
    return ids.reshape(info.n_traces, info.decode_steps, info.num_layers, info.top_k)


def read_trace_binary(path, trace_index: int = 0) -> RoutingTrace:
    """``.mcbt`` -> RoutingTrace (one trace of a batch file), validated."""
    info = read_binary_info(path)
    h = TraceHeader(info.model_name, info.num_layers, info.num_experts, info.top_k)
    if info.kind == KIND_BATCH:
        ids = _batch_ids(path, info)[trace_index]
        evs = tuple(AccessEvent(0, Phase.DECODE, t, l, tuple(int(x) for x in ids[t, l]))
                    for t in range(ids.shape[0]) for l in range(ids.shape[1]))
    else:
        seq, phase, step, layer, off, experts = _general_columns(path, info)
        if len(phase) and int(phase.max()) > 1:
            raise TraceParseError(1, "phase must be 0 (prefill) or 1 (decode)")
        ex = experts.tolist()
        evs = tuple(AccessEvent(int(seq[i]), Phase(int(phase[i])), int(step[i]), int(layer[i]),
                                tuple(ex[off[i]:off[i + 1]]))
                    for i in range(len(seq)))
    tr = RoutingTrace(h, evs)
    tr.validate()
    return tr


def load_packed(path, device: int = 0) -> PackedTrace:
    """``.mcbt`` -> PackedTrace for the engine.

    Batch files: the ids are validated and transposed to chain-major on the
    GPU (K7, mcb_pack_decode_ids); general files go through the native host
    packer (mcb_pack_trace, the RoutingTrace.validate restatement)."""
    info = read_binary_info(path)
    if info.kind == KIND_BATCH:
        return pack_decode_ids_device(_batch_ids(path, info), info.num_experts, device=device)
    seq, phase, step, layer, off, experts = _general_columns(path, info)
    lib = _lib.load_library()
    handle = ctypes.c_void_p()
    ex32 = experts.astype(np.int32)
    seq = np.ascontiguousarray(seq, dtype=np.int64)
    step = np.ascontiguousarray(step, dtype=np.int64)
    layer = np.ascontiguousarray(layer, dtype=np.int32)
    off = np.ascontiguousarray(off, dtype=np.int64)
    _lib.check(lib.mcb_pack_trace(info.num_layers, info.num_experts, info.top_k, len(seq),
                                  seq.ctypes.data, phase.ctypes.data, step.ctypes.data, layer.ctypes.data,
                                  off.ctypes.data, ex32.ctypes.data, ctypes.byref(handle)))
    from .trace import _from_handle
    return _from_handle(handle)


def pack_decode_ids_device(ids, num_experts: int, device: int = 0) -> PackedTrace:
    """Event-order decode ids [n][T][L][K] -> validated chain-major PackedTrace
    on the GPU (K7).  Raises InvalidConfigError for the first invalid event
    in file order with AccessEvent.validate's message."""
    import torch
    ids = np.ascontiguousarray(ids, dtype=np.uint8)
    if ids.ndim == 3:
        ids = ids[None]
    n, T, L, K = ids.shape
    TraceHeader("batch", L, num_experts, K).validate()
    dev = torch.device("cuda", device)
    src = torch.from_numpy(ids.reshape(-1)).to(dev)
    total = src.numel()
    acc = torch.empty((total + 127) // 128 * 128 + 128, dtype=torch.uint8, device=dev)
    acc[total:].zero_()
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev)
    lib = _lib.load_library()
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(lib.mcb_pack_decode_ids(_lib.context(device), src.data_ptr(), n, T, L, K, num_experts,
                                       acc.data_ptr(), bad.data_ptr(), ctypes.c_void_p(stream)))
    first = int(bad.item())
    if first >= 0:
        t_i, rem = divmod(first, L)
        tr, t = divmod(t_i, T)
        ev = AccessEvent(0, Phase.DECODE, t, rem, tuple(int(x) for x in ids[tr, t, rem]))
        msg, _ = _event_problem(ev, TraceHeader("batch", L, num_experts, K))
        raise InvalidConfigError(msg)
    host = acc.cpu().numpy()
    return PackedTrace(num_layers=L, num_experts=num_experts, top_k=K, num_traces=n, uniform=True,
                       events_per_chain=T, acc=host, total_acc=total, total_events=n * L * T,
                       decode_steps=[T] * n)


__all__ = ["trace_to_text", "write_trace", "parse_trace", "read_trace", "write_trace_binary",
           "write_batch_binary", "read_trace_binary", "read_binary_info", "load_packed",
           "pack_decode_ids_device"]
