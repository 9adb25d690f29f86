"""K7 (mcb_pack_decode_ids): GPU validation + chain-major packing of
batch-kind .mcbt files, against the host packer and AccessEvent.validate's
error semantics (trace.py:80-106); general-kind files through the native
host packer."""
import numpy as np
import pytest

from golden_util import case_trace, load

pytestmark = pytest.mark.gpu

import paper_2601_17063_b200 as mcb  # noqa: E402
from paper_2601_17063_b200 import engine, tracefile  # noqa: E402
from paper_2601_17063_b200.trace import AccessEvent, Phase, RoutingTrace, TraceHeader  # noqa: E402


def batch_ids(n, T, L, K, E, seed):
    rng = np.random.default_rng(seed)
    keys = rng.random((n, T, L, E))
    return np.argsort(keys, axis=-1)[..., :K].astype(np.uint8)   # K distinct experts per event


@pytest.mark.parametrize("shape", [(1, 65536, 32, 2, 8), (3, 2048, 48, 8, 128), (2, 77, 5, 3, 7), (1, 1, 1, 1, 1),
                                   (2, 1000, 61, 4, 256)])
def test_gpu_pack_matches_host_transpose(shape, tmp_path):
    n, T, L, K, E = shape
    ids = batch_ids(n, T, L, K, E, seed=T)
    p = tmp_path / "b.mcbt"
    mcb.write_batch_binary(ids, E, p)
    packed = mcb.load_packed(p)
    want = np.ascontiguousarray(ids.transpose(0, 2, 1, 3)).reshape(-1)   # [n][L][T][K]
    assert packed.uniform and packed.num_traces == n and packed.events_per_chain == T
    assert np.array_equal(packed.acc[:packed.total_acc], want)
    if E <= 128:
        ref = mcb.packed_from_decode_ids(ids.transpose(0, 2, 1, 3), E)
        a = engine.replay_host(packed, [0, 1], [K, K + 1], mcb.CostModel(), 5)
        b = engine.replay_host(ref, [0, 1], [K, K + 1], mcb.CostModel(), 5)
        assert np.array_equal(a["reports"], b["reports"])


@pytest.mark.parametrize("bad", ["range", "dup", "both"])
def test_gpu_pack_reports_first_invalid_event(bad):
    n, T, L, K, E = 2, 300, 6, 3, 10
    ids = batch_ids(n, T, L, K, E, seed=1)
    first = (1, 17, 4)
    if bad in ("range", "both"):
        ids[first][1] = 12
    if bad in ("dup", "both"):
        ids[1, 200, 2][2] = ids[1, 200, 2][0]
        ids[1, 250, 0][0] = ids[1, 250, 0][1]
    with pytest.raises(mcb.InvalidConfigError) as ei:
        tracefile.pack_decode_ids_device(ids, E)
    ev = AccessEvent(0, Phase.DECODE, 0, 0, tuple(int(x) for x in (ids[first] if bad != "dup" else ids[1, 200, 2])))
    if bad == "dup":
        assert str(ei.value) == f"experts contain duplicates: {list(ev.experts)}"
    else:
        assert str(ei.value) == f"expert 12 out of range [0, {E})"


def test_general_file_packs_like_pack_trace(tmp_path):
    for case in load("small_cases.json.gz")["cases"][::11]:
        header, events = case_trace(case)
        L, E, K = header
        tr = RoutingTrace(TraceHeader("g", L, E, K),
                          tuple(AccessEvent(s, Phase(p), t, l, tuple(x)) for s, p, t, l, x in events))
        p = tmp_path / "g.mcbt"
        mcb.write_trace_binary(tr, p)
        a = mcb.load_packed(p)
        b = mcb.pack_trace(tr)
        assert np.array_equal(a.acc[:a.total_acc], b.acc[:b.total_acc])
        assert (a.uniform, a.total_events) == (b.uniform, b.total_events)
        if not a.uniform:
            assert np.array_equal(a.ev_info, b.ev_info)
