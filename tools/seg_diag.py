"""Segmented-replay diagnostics on the c2 workload: per policy and segment
length, the replay time and convergence statistics of the fix-up walk."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2601_17063_b200 import _lib  # noqa: E402
from paper_2601_17063_b200.device import DeviceNets, DeviceReplay, DeviceTrace  # noqa: E402
from paper_2601_17063_b200.engine import CostModel  # noqa: E402

wl = dict(bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
wl["n_traces_local"] = wl["traces"]
dev = torch.device("cuda", 0)
ids, _ = bench.make_trace_ids(wl, 0, "tcgen05", dev)
dtrace = DeviceTrace.from_decode_ids(ids, wl["E"])
hidden, n_nets, flat = bench.nets_for(wl["L"], wl["E"])
dnets = DeviceNets(hidden, n_nets, flat, wl["E"], device=dev)
codes = {"lru": _lib.MCB_LRU, "lfu": _lib.MCB_LFU, "belady": _lib.MCB_BELADY, "ml": _lib.MCB_ML}
for se in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "-1"])]:
    _lib.set_tuning(_lib.MCB_TUNE_SEG_EV, se)
    for p in ["lru", "lfu", "belady", "ml"]:
        rep = DeviceReplay(dtrace, [codes[p]], wl["caps"], CostModel(), 5, dnets if p == "ml" else None)
        rep.set_timing(True)
        rep()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        st = _lib.read_stats()
        ms = rep.stage_ms()
        print(f"se={se:5d} {p:7s} wall {dt*1e3:8.3f} ms stages {[round(x, 3) for x in ms]} "
              f"fixup_events {st[1]} unconverged {st[2]} / {st[3]} segs", flush=True)
