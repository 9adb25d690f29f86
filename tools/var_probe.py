"""Per-step stage durations of the C4 device replay (timing on), to find the
stage behind the occasional slow step."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_2601_17063_b200 import _lib
from paper_2601_17063_b200.device import DeviceNets, DeviceReplay, DeviceTrace
from paper_2601_17063_b200.engine import CostModel
wl = dict(bench.WORKLOADS["c4"]); n = wl["traces"]
dev = torch.device("cuda", 0)
ids, _ = bench.gen_traces_gpu(wl, list(range(n)), wl["gen"], dev)
L, E = wl["L"], wl["E"]
hidden, n_nets, flat = bench.nets_for(L, E)
codes = [_lib.MCB_LRU, _lib.MCB_LFU, _lib.MCB_BELADY, _lib.MCB_ML]
st = torch.cuda.current_stream(dev)
dtrace = DeviceTrace.from_decode_ids(ids, E)
dnets = DeviceNets(hidden, n_nets, flat, E, device=dev)
rep = DeviceReplay(dtrace, codes, wl["caps"], CostModel(), 5, dnets, device=0)
lib = _lib.load_library()
_lib.check(lib.mcb_set_timing(_lib.context(0), 1))
rep(); torch.cuda.synchronize()
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); t0 = time.perf_counter(); rep(); th = (time.perf_counter() - t0) * 1e3; b.record(st); b.synchronize()
    ms = (ctypes.c_float * 5)()
    _lib.check(lib.mcb_last_timings(_lib.context(0), ms, 5))
    print(round(a.elapsed_time(b), 1), 'host', round(th, 1), [round(x, 1) for x in ms], flush=True)
if os.environ.get("PROFILE"):
    import cProfile, pstats
    pr = cProfile.Profile()
    for i in range(25):
        a.record(st); pr.enable(); rep(); pr.disable(); b.record(st); b.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)
