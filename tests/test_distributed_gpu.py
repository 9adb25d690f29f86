"""The sharded engine on real GPU shards: two gloo ranks (both on cuda:0 --
the test box has one GPU) each replay their shard with the CUDA engine, the
single all-reduce combines them, and the result must be bit-identical to a
1-rank run: trace sharding (a uniform batch), layer sharding of a uniform
trace, and layer sharding of a prefill + multi-sequence trace through
``sweep_sharded`` (full SimReport equality, floats included)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

POLS = ["lru", "lfu", "belady", "ml"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _uniform_batch(nt, L, E, K, T, seed):
    rng = np.random.default_rng(seed)
    return np.stack([np.stack([np.stack([rng.choice(E, K, replace=False) for _ in range(T)]) for _ in range(L)])
                     for _ in range(nt)]).astype(np.uint8)


def _general_trace(L, E, K, seed):
    from paper_2601_17063_b200.trace import AccessEvent, Phase, RoutingTrace, TraceHeader
    rng = np.random.default_rng(seed)
    ev = []
    for seq in range(2):
        for t in range(6):
            for layer in range(L):
                ev.append(AccessEvent(seq, Phase.PREFILL, t, layer,
                                      tuple(int(x) for x in rng.choice(E, K + 2, replace=False))))
        for t in range(300):
            for layer in range(L):
                ev.append(AccessEvent(seq, Phase.DECODE, t, layer,
                                      tuple(int(x) for x in rng.choice(E, K, replace=False))))
    return RoutingTrace(TraceHeader("g", L, E, K), tuple(ev))


def _codes():
    from paper_2601_17063_b200 import _lib
    return [_lib.MCB_LRU, _lib.MCB_LFU, _lib.MCB_BELADY, _lib.MCB_ML]


def _nets(L, E):
    import oracle
    return oracle.nets_from_spec({"kind": "per_layer_seed"}, L, E)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_17063_b200 import CostModel, EvictionNet
        from paper_2601_17063_b200 import distributed as D
        from paper_2601_17063_b200.trace import packed_from_decode_ids
        out = {}
        ids = _uniform_batch(5, 3, 16, 2, 500, 1)
        r = D.replay_sharded(packed_from_decode_ids(ids, 16), _codes(), [2, 4, 8], CostModel(), 5, _nets(3, 16),
                             device=0)
        out["traces"] = (r["kind"], r["reports"], r["latency"])
        ids = _uniform_batch(1, 5, 8, 2, 3000, 2)
        r = D.replay_sharded(packed_from_decode_ids(ids, 8), _codes(), [2, 3, 6], CostModel(), 5, _nets(5, 8),
                             device=0)
        out["layers"] = (r["kind"], r["reports"], r["latency"])
        tr = _general_trace(4, 64, 4, 3)
        nets = {layer: EvictionNet(64, seed=layer) for layer in range(4)}
        rows = D.sweep_sharded(tr, POLS, [4, 8, 16], CostModel(), 5, nets, device=0)
        out["sweep"] = [r.to_dict() for r in rows]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_equal_one_gpu_run():
    from paper_2601_17063_b200 import CostModel, EvictionNet, sweep
    from paper_2601_17063_b200.engine import replay_host
    from paper_2601_17063_b200.trace import packed_from_decode_ids

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0

    ids = _uniform_batch(5, 3, 16, 2, 500, 1)
    want_t = replay_host(packed_from_decode_ids(ids, 16), _codes(), [2, 4, 8], CostModel(), 5, _nets(3, 16))
    ids = _uniform_batch(1, 5, 8, 2, 3000, 2)
    want_l = replay_host(packed_from_decode_ids(ids, 8), _codes(), [2, 3, 6], CostModel(), 5, _nets(5, 8))
    tr = _general_trace(4, 64, 4, 3)
    want_s = [r.to_dict() for r in sweep(tr, POLS, [4, 8, 16], CostModel(), 5,
                                         {layer: EvictionNet(64, seed=layer) for layer in range(4)})]
    for rank, out in outs:
        kind, rep, lat = out["traces"]
        assert kind == "traces"
        assert np.array_equal(rep, want_t["reports"]) and np.array_equal(lat, want_t["latency"])
        kind, rep, lat = out["layers"]
        assert kind == "layers"
        assert np.array_equal(rep, want_l["reports"]) and np.array_equal(lat, want_l["latency"])
        assert out["sweep"] == want_s


def test_native_communicator_single_rank():
    """The C ABI's NCCL communicator (mcb_comm_*) on one GPU: a one-rank clique
    sums in place (the identity), the context refuses a second communicator,
    and it can be re-created after mcb_comm_destroy."""
    import torch

    from paper_2601_17063_b200 import _lib
    from paper_2601_17063_b200.distributed import NativeCommunicator
    uid = NativeCommunicator.unique_id()
    assert len(uid) == 128
    comm = NativeCommunicator(1, 0, uid)
    try:
        x = torch.arange(-5, 1000, dtype=torch.int64, device="cuda") * 3
        want = x.clone()
        comm.all_reduce_(x)
        torch.cuda.synchronize()
        assert torch.equal(x, want)
        with pytest.raises(Exception):
            NativeCommunicator(1, 0, NativeCommunicator.unique_id())
    finally:
        comm.close()
    comm = NativeCommunicator(1, 0, NativeCommunicator.unique_id())
    comm.close()
    _ = _lib
