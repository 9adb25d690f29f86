"""Eviction timelines (pkg/src/moecache/reports.py:155-231).

A timeline is JSONL for heatmap rendering: a header line, then per layer in
stream order one ``access`` row per replayed access, each followed by the
``eviction`` row of the victim that access evicted.  The engine produces the
victim stream on the GPU (the per-access outcome codes of one replay); this
module formats it byte-for-byte like the reference's ``write_timeline``.

``write_timeline`` accepts the reference's arguments (schedules from
``layer_schedules`` + ``EvictionRecord`` list) or this package's
(``PackedTrace`` + the ``SimRun.evictions`` of ``run_simulation``), so both
code paths produce identical files.
"""
from __future__ import annotations

import json

import numpy as np

SCHEMA_VERSION = 1
_KINDS = ("access", "eviction")
_FIELDS = {"kind", "layer", "step", "decode_index", "expert", "position"}


class ReportFormatError(Exception):
    pass


def _row(kind, layer, step, dec, expert, pos) -> str:
    # json.dumps(..., separators=(",", ":")) of an all-int record, spelled out
    return (f'{{"kind":"{kind}","layer":{layer},"step":{step},"decode_index":{dec},'
            f'"expert":{expert},"position":{pos}}}\n')


def _layer_streams(schedules_or_packed):
    """-> per layer (accessed experts, tick, decode_index) arrays."""
    if hasattr(schedules_or_packed, "chain_accesses"):
        p = schedules_or_packed
        if p.num_traces != 1:
            raise ValueError("timelines are per trace")
        for layer in range(p.num_layers):
            tick, dec = p.positions(layer)
            yield np.asarray(p.chain_accesses(layer)), tick, dec
        return
    for schedule in schedules_or_packed:   # reference ReplayStep lists (replay.py:44-81)
        acc, tick, dec = [], [], []
        for step in schedule:
            acc.extend(step.accesses)
            tick.extend([step.tick] * len(step.accesses))
            dec.extend([step.decode_index] * len(step.accesses))
        yield np.array(acc, dtype=np.int64), np.array(tick, dtype=np.int64), np.array(dec, dtype=np.int64)


def write_timeline(schedules, evictions, policy: str, path) -> None:
    """reports.py:161-210: header, then access rows with their evictions."""
    by_layer: dict = {}
    for rec in evictions:
        by_layer.setdefault(rec.layer, []).append(rec)
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write(json.dumps({"schema_version": SCHEMA_VERSION, "kind": "timeline", "policy": policy},
                            separators=(",", ":")) + "\n")
        for layer, (acc, tick, dec) in enumerate(_layer_streams(schedules)):
            pend = sorted(by_layer.get(layer, []), key=lambda r: r.position)
            at: dict = {}
            for r in pend:
                at.setdefault(r.position, []).append(r)
            out = []
            for pos, (x, t, d) in enumerate(zip(acc.tolist(), tick.tolist(), dec.tolist())):
                out.append(_row("access", layer, t, d, x, pos))
                for r in at.get(pos, ()):
                    out.append(_row("eviction", layer, r.tick, r.decode_index, r.victim, r.position))
            fh.write("".join(out))


def load_timeline(path):
    """Parse and schema-check a timeline (reports.py:213-231) -> (header, rows)."""
    with open(path, "r", encoding="utf-8") as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise ReportFormatError("timeline: empty file")
    header = json.loads(lines[0])
    if not isinstance(header, dict) or header.get("schema_version") != SCHEMA_VERSION:
        got = header.get("schema_version") if isinstance(header, dict) else type(header)
        raise ReportFormatError(f"timeline: expected schema_version {SCHEMA_VERSION}, got {got}")
    if header.get("kind") != "timeline":
        raise ReportFormatError("timeline: bad header kind")
    rows = []
    for i, line in enumerate(lines[1:], start=2):
        row = json.loads(line)
        if set(row) != _FIELDS:
            raise ReportFormatError(f"timeline line {i}: fields {sorted(row)} != {sorted(_FIELDS)}")
        if row["kind"] not in _KINDS:
            raise ReportFormatError(f"timeline line {i}: unknown kind {row['kind']!r}")
        rows.append(row)
    return header, rows


__all__ = ["SCHEMA_VERSION", "ReportFormatError", "write_timeline", "load_timeline"]
