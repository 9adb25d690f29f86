"""A/B of the e2e path: timing off, with and without an L2 flush before each step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_2601_17063_b200 import _lib
from paper_2601_17063_b200.device import DeviceNets, DeviceReplay, DeviceTrace
from paper_2601_17063_b200.engine import CostModel, replay_host
from paper_2601_17063_b200.trace import packed_from_decode_ids
wl = dict(bench.WORKLOADS["c4"]); n = wl["traces"]
dev = torch.device("cuda", 0)
ids, _ = bench.gen_traces_gpu(wl, list(range(n)), wl["gen"], dev)
L, E = wl["L"], wl["E"]
hidden, n_nets, flat = bench.nets_for(L, E)
codes = [_lib.MCB_LRU, _lib.MCB_LFU, _lib.MCB_BELADY, _lib.MCB_ML]
st = torch.cuda.current_stream(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ids_host = torch.empty(ids.shape, dtype=torch.uint8, pin_memory=True); ids_host.copy_(ids)
packed = packed_from_decode_ids(ids_host.numpy(), E)
acc_pinned = torch.empty(packed.acc.shape, dtype=torch.uint8, pin_memory=True)
acc_pinned.numpy()[:] = packed.acc; packed.acc = acc_pinned.numpy()
flat_pinned = torch.empty(flat.shape, dtype=torch.float64, pin_memory=True); flat_pinned.numpy()[:] = flat
nets_host = (hidden, n_nets, flat_pinned.numpy())
dtrace = DeviceTrace.from_decode_ids(ids, E)
dnets = DeviceNets(hidden, n_nets, flat, E, device=dev)
rep = DeviceReplay(dtrace, codes, wl["caps"], CostModel(), 5, dnets, device=0)
def run(fn, fl, reps=5):
    fn(); fn(); torch.cuda.synchronize(); out = []
    for _ in range(reps):
        if fl: flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); b.synchronize(); out.append(a.elapsed_time(b))
    return [round(x, 1) for x in out]
tag = os.environ.get("MCB_X_LATE", "early")
for fl in (0, 1):
    print(tag, "flush", fl, "host", run(lambda: replay_host(packed, codes, wl["caps"], CostModel(), 5, nets_host, stream=st.cuda_stream), fl))
    print(tag, "flush", fl, "dev ", run(rep, fl))
