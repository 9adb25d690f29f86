"""Where the e2e (host-buffer) path's extra time goes on C4: the bare H2D copy
of the trace, mcb_replay_host with / without the piecewise upload, and the
device path -- CUDA events on one stream."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_17063_b200 import _lib  # noqa: E402
from paper_2601_17063_b200.device import DeviceNets, DeviceReplay, DeviceTrace  # noqa: E402
from paper_2601_17063_b200.engine import CostModel, replay_host  # noqa: E402
from paper_2601_17063_b200.trace import packed_from_decode_ids  # noqa: E402

wl = dict(bench.WORKLOADS["c4"])
n = int(sys.argv[1]) if len(sys.argv) > 1 else wl["traces"]
dev = torch.device("cuda", 0)
ids, _ = bench.gen_traces_gpu(wl, list(range(n)), wl["gen"], dev)
L, E = wl["L"], wl["E"]
hidden, n_nets, flat = bench.nets_for(L, E)
codes = [_lib.MCB_LRU, _lib.MCB_LFU, _lib.MCB_BELADY, _lib.MCB_ML]
st = torch.cuda.current_stream(dev)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        out.append((a.elapsed_time(b), (time.perf_counter() - t0) * 1e3))
    return min(out)


ids_host = torch.empty(ids.shape, dtype=torch.uint8, pin_memory=True)
ids_host.copy_(ids)
packed = packed_from_decode_ids(ids_host.numpy(), E)
acc_pinned = torch.empty(packed.acc.shape, dtype=torch.uint8, pin_memory=True)
acc_pinned.numpy()[:] = packed.acc
packed.acc = acc_pinned.numpy()
flat_pinned = torch.empty(flat.shape, dtype=torch.float64, pin_memory=True)
flat_pinned.numpy()[:] = flat
nets_host = (hidden, n_nets, flat_pinned.numpy())
dst = torch.empty(acc_pinned.shape, dtype=torch.uint8, device=dev)
print("H2D copy of the trace", timed(lambda: dst.copy_(acc_pinned, non_blocking=True)), "ms (gpu, host)")
import ctypes  # noqa: E402
lib = _lib.load_library()
_lib.check(lib.mcb_set_timing(_lib.context(0), 1))
for u in (8, 1, 8):
    _lib.set_tuning(_lib.MCB_TUNE_UPLOAD_PIECES, u)
    print(f"replay_host pieces={u}", timed(lambda: replay_host(packed, codes, wl["caps"], CostModel(), 5, nets_host,
                                                             stream=st.cuda_stream)))
    ms = (ctypes.c_float * 5)()
    _lib.check(lib.mcb_last_timings(_lib.context(0), ms, 5))
    print("   stages (K2, K3, K4 non-ML, K4 ML, K5):", [round(x, 2) for x in ms])
dtrace = DeviceTrace.from_decode_ids(ids, E)
dnets = DeviceNets(hidden, n_nets, flat, E, device=dev)
rep = DeviceReplay(dtrace, codes, wl["caps"], CostModel(), 5, dnets, device=0)
print("device replay", timed(rep))

# does an H2D copy overlap a running replay?
side = torch.cuda.Stream(dev)
a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a0.record(st)
rep()
a1.record(st)
with torch.cuda.stream(side):
    b0.record(side)
    dst.copy_(acc_pinned, non_blocking=True)
    b1.record(side)
torch.cuda.synchronize()
print("replay alone-ish", a0.elapsed_time(a1), "copy under the replay", b0.elapsed_time(b1),
      "copy start after replay start", a0.elapsed_time(b0))
