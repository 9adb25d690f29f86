"""Trace files: the JSONL reader / writer against
fixtures made by the reference's own parse_trace / trace_to_text
(tests/golden/make_tracefile_golden.py), and the binary .mcbt container's
round trips.  CPU only; the GPU pack/validate kernel (K7) is covered by
tests/test_tracefile_gpu.py."""
import os

import numpy as np
import pytest

from golden_util import case_trace, load

import paper_2601_17063_b200 as mcb
from paper_2601_17063_b200 import tracefile
from paper_2601_17063_b200.trace import AccessEvent, Phase, RoutingTrace, TraceHeader

CASES = load("tracefile_cases.json.gz")["cases"]


@pytest.mark.parametrize("part", range(4))
def test_parse_trace_matches_reference(part):
    for c in CASES[part::4]:
        if c["ok"]:
            tr = mcb.parse_trace(c["text"])
            assert mcb.trace_to_text(tr) == c["text_out"], c["name"]
            assert len(tr.events) == c["n_events"]
        else:
            with pytest.raises(mcb.TraceError) as ei:
                mcb.parse_trace(c["text"])
            assert type(ei.value).__name__ == c["type"], (c["name"], str(ei.value))
            assert getattr(ei.value, "line_no", None) == c["line_no"], c["name"]
            assert str(ei.value) == c["message"], c["name"]


def test_text_round_trip_and_files(tmp_path):
    for c in CASES:
        if c["ok"] and c["name"].startswith("random"):
            tr = mcb.parse_trace(c["text"])
            assert mcb.trace_to_text(tr) == c["text"]
            p = tmp_path / "t.jsonl"
            mcb.write_trace(tr, p)
            assert p.read_bytes() == c["text"].encode("utf-8")
            assert mcb.read_trace(p) == tr


def _trace_of_case(case):
    header, events = case_trace(case)
    L, E, K = header
    return RoutingTrace(TraceHeader("golden", L, E, K),
                        tuple(AccessEvent(s, Phase(p), t, l, tuple(x)) for s, p, t, l, x in events))


def test_binary_general_round_trip(tmp_path):
    for case in load("small_cases.json.gz")["cases"][::7]:
        tr = _trace_of_case(case)
        p = tmp_path / "t.mcbt"
        mcb.write_trace_binary(tr, p)
        assert mcb.read_trace_binary(p) == tr
        info = tracefile.read_binary_info(p)
        assert info.kind == tracefile.KIND_GENERAL and info.n_events == len(tr.events)


def test_binary_batch_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    n, T, L, K, E = 3, 5, 4, 2, 8
    ids = np.stack([rng.permutation(E)[:K] for _ in range(n * T * L)]).reshape(n, T, L, K).astype(np.uint8)
    p = tmp_path / "b.mcbt"
    mcb.write_batch_binary(ids, E, p, model_name="mixtral")
    info = tracefile.read_binary_info(p)
    assert (info.kind, info.n_traces, info.decode_steps, info.num_layers, info.top_k) == \
        (tracefile.KIND_BATCH, n, T, L, K)
    tr = mcb.read_trace_binary(p, trace_index=1)
    assert tr.header == TraceHeader("mixtral", L, E, K)
    assert [ev.experts for ev in tr.events] == [tuple(ids[1, t, l].tolist()) for t in range(T) for l in range(L)]


def test_binary_rejects_corrupt_files(tmp_path):
    p = tmp_path / "x.mcbt"
    p.write_bytes(b"NOTATRACE" + b"\0" * 64)
    with pytest.raises(mcb.TraceParseError):
        tracefile.read_binary_info(p)
    ids = np.zeros((1, 2, 1, 1), dtype=np.uint8)
    mcb.write_batch_binary(ids, 4, p)
    data = p.read_bytes()
    p.write_bytes(data[:-1])
    with pytest.raises(mcb.TraceParseError):
        mcb.read_trace_binary(p)
