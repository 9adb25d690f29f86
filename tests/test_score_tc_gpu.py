"""K3-TC, the tensor-core scorer (csrc/mcb_score_tc.cu), against the float64
scorer and the oracle.

* Rank rows are IDENTICAL to the float64 DMMA scorer's (MCB_TUNE_K3_TC = 0)
  on every event, for every specialised expert count -- the certification
  plus the float64 re-score of the uncertified events make the fast path
  exact, not approximate.
* The fp32 (fp16 x 2 split) scores deviate from the oracle's float64 forward by far
  less than the certification threshold tau: the calibration that makes the
  certificate meaningful (the measured maximum is printed).
* tau = 1 (every event re-scored) and tau = 0 (only collisions re-scored)
  exercise both ends of the machinery.
"""
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2601_17063_b200 import _lib  # noqa: E402
from paper_2601_17063_b200.device import DeviceNets, DeviceTrace  # noqa: E402

TAU = 4e-6

SHAPES = [   # (L, E, K, T, traces)
    (3, 64, 6, 2048, 6),      # C4-like (DeepSeek-V2-Lite)
    (3, 128, 8, 1000, 3),     # C1 / C5-like (Qwen3), partial last tile
    (4, 8, 2, 4096, 2),       # C2-like (Mixtral)
    (3, 16, 4, 777, 3),       # odd length
    (2, 32, 4, 1500, 2),
]


def _ids(L, E, K, T, n, seed=0):
    x = oracle.generate_decode_batch((L, E, K), T, list(range(seed, seed + n)), 7, 1.0, 0.3, 4)
    return np.ascontiguousarray(x.transpose(0, 2, 1, 3))      # [n][L][T][K]


def _setup(L, E, K, T, n):
    ids = _ids(L, E, K, T, n)
    dt = DeviceTrace.from_decode_ids(torch.from_numpy(ids).cuda(), E)
    hidden, n_nets, flat = oracle.nets_from_spec({"kind": "per_layer_seed"}, L, E)
    dn = DeviceNets(hidden, n_nets, flat, E)
    return ids, dt, dn, (hidden, n_nets, flat)


def _ranks(dt, dn, tc: bool, tau_ppb: int = 4000, groups: int = 3):
    lib = _lib.load_library()
    _lib.set_tuning(_lib.MCB_TUNE_K3_TC, int(tc))
    _lib.set_tuning(_lib.MCB_TUNE_K3_TAU_PPB, tau_ppb)
    _lib.set_tuning(_lib.MCB_TUNE_K3_GROUPS, groups)
    try:
        out = torch.zeros(dt.total_events * dt.num_experts + 64, dtype=torch.uint8, device="cuda")
        v, ns = dt.view(), dn.struct()
        _lib.check(lib.mcb_score(_lib.context(0), ctypes.byref(v), ctypes.byref(ns), 1, out.data_ptr(), None,
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        torch.cuda.synchronize()
        stats = _lib.read_stats()
    finally:
        _lib.set_tuning(_lib.MCB_TUNE_K3_TC, 1)
        _lib.set_tuning(_lib.MCB_TUNE_K3_TAU_PPB, 4000)
        _lib.set_tuning(_lib.MCB_TUNE_K3_GROUPS, 3)
    return out[:dt.total_events * dt.num_experts].cpu().numpy().reshape(-1, dt.num_experts), stats


@pytest.mark.parametrize("groups", [3, 2, 1])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"E{s[1]}")
def test_tc_ranks_equal_float64_ranks(shape, groups):
    L, E, K, T, n = shape
    _, dt, dn, _ = _setup(L, E, K, T, n)
    r64, _ = _ranks(dt, dn, tc=False)
    rtc, st = _ranks(dt, dn, tc=True, groups=groups)
    rescored = st[5]
    print(f"E={E}, {groups} groups: {rescored} of {dt.total_events} events re-scored in float64 ({rescored / dt.total_events:.4%})")
    assert np.array_equal(rtc, r64)
    assert rescored < dt.total_events      # the fast path certified most events


@pytest.mark.parametrize("shape", SHAPES[:3], ids=lambda s: f"E{s[1]}")
def test_tc_scores_within_calibrated_error(shape):
    """Normwise deviation of the fp16x2 / fp32 scores from the float64
    oracle, per event: max_e |s_tc - s_64| / max_e |s_64| << tau."""
    L, E, K, T, n = shape
    ids, dt, dn, nets = _setup(L, E, K, T, n)
    lib = _lib.load_library()
    ranks = torch.zeros(dt.total_events * E + 64, dtype=torch.uint8, device="cuda")
    sc = torch.zeros(dt.total_events * E, dtype=torch.float32, device="cuda")
    v, ns = dt.view(), dn.struct()
    _lib.check(lib.mcb_score_tc_scores(_lib.context(0), ctypes.byref(v), ctypes.byref(ns), ranks.data_ptr(),
                                       sc.data_ptr(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    sc = sc.cpu().numpy().reshape(n, L, T, E).astype(np.float64)
    hidden, _, flat = nets
    per = flat.size // L
    worst = 0.0
    for t in range(min(n, 2)):
        for layer in range(L):
            ref = oracle.score_chain(ids[t, layer], E, hidden, flat[layer * per:(layer + 1) * per])
            err = np.abs(sc[t, layer] - ref).max(axis=1) / np.abs(ref).max(axis=1)
            worst = max(worst, float(err.max()))
    print(f"E={E}: max normwise |s_tc - s_f64| / max|s| = {worst:.3e} (tau = {TAU:.1e})")
    assert worst < TAU / 4


def test_tau_extremes():
    L, E, K, T, n = SHAPES[0]
    _, dt, dn, _ = _setup(L, E, K, T, n)
    r64, _ = _ranks(dt, dn, tc=False)
    rall, st = _ranks(dt, dn, tc=True, tau_ppb=10 ** 9)          # tau = 1: every event re-scored
    assert st[5] == dt.total_events
    assert np.array_equal(rall, r64)
    rnone, st0 = _ranks(dt, dn, tc=True, tau_ppb=0)              # only truncated-key collisions re-scored
    assert st0[5] < dt.total_events
    diff = int((rnone != r64).any(axis=1).sum())
    print(f"tau = 0: {st0[5]} re-scored, {diff} of {dt.total_events} rank rows differ from float64")


def test_forced_near_ties_are_rescored_and_surfaced():
    """Two experts whose float64 scores differ by ~1e-14 of max|s| (identical
    W3 rows, b3 apart by a few ulp): not an exact tie, but inside any float64
    evaluation order's rounding.  The tensor-core scorer cannot certify those
    events (they go to the float64 re-score), the float64 ranking flags them
    as near ties, and the public API warns instead of silently deciding."""
    import warnings

    import paper_2601_17063_b200 as mcb
    from paper_2601_17063_b200.engine import ScorerNearTieWarning
    L, E, K, T = 2, 64, 6, 1024
    ids = _ids(L, E, K, T, 1)[0]                                          # [L][T][K]
    net = mcb.EvictionNet(E, seed=3)
    net.params["w3"][5] = net.params["w3"][9]
    net.params["b3"][5] = np.nextafter(np.nextafter(net.params["b3"][9], 1.0), 1.0)
    events = []
    for t in range(T):
        for layer in range(L):
            events.append(mcb.AccessEvent(0, mcb.Phase.DECODE, t, layer, tuple(int(x) for x in ids[layer, t])))
    tr = mcb.RoutingTrace(mcb.TraceHeader("near", L, E, K), tuple(events))
    with warnings.catch_warnings(record=True) as got:
        warnings.simplefilter("always")
        rep = mcb.simulate(tr, "ml", 16, nets=net)
    assert any(issubclass(w.category, ScorerNearTieWarning) for w in got)
    assert rep.hits + rep.misses == L * T * K
    st = _lib.read_stats()
    assert st[0] > 0                       # float64 near ties counted
    assert st[5] >= st[0]                  # every one of them went through the float64 re-score


@pytest.mark.parametrize("wscale", [1e-3, 40.0])
def test_scaled_weights_ranks_equal_float64(wscale):
    """fp16's range: every layer's weights scaled by a large or a small
    factor.  The per-layer power-of-two scaling keeps the split exact; with
    large weights the hidden activations exceed the fp16-safe bound, those
    events are flagged and re-scored in float64.  Ranks stay identical."""
    L, E, K, T, n = 2, 64, 6, 1024, 2
    ids = _ids(L, E, K, T, n)
    dt = DeviceTrace.from_decode_ids(torch.from_numpy(ids).cuda(), E)
    hidden, n_nets, flat = oracle.nets_from_spec({"kind": "per_layer_seed"}, L, E)
    flat = flat * wscale
    dn = DeviceNets(hidden, n_nets, flat, E)
    r64, _ = _ranks(dt, dn, tc=False)
    rtc, st = _ranks(dt, dn, tc=True)
    print(f"weights x {wscale}: {st[5]} of {dt.total_events} events re-scored")
    assert np.array_equal(rtc, r64)
