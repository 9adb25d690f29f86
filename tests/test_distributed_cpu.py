"""World-size-2 gloo tests of the multi-GPU host logic (sharding + the single
counter reduce), run on CPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_17063_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_traces, n_pol, n_cap = 7, 4, 3
        b, e = D.shard_range(n_traces, rank, world)
        # per-trace counters as a 1-GPU run would produce them (deterministic fake)
        full = torch.arange(n_traces * n_pol * n_cap * 8, dtype=torch.int64).reshape(n_traces, n_pol, n_cap, 8)
        full[..., 7] = 0
        if rank == 1:
            full[5, 2, 1, 7] = 3          # one failing cell on rank 1 shard (traces 4..6)
        local = full[b:e]
        red = D.reduce_counters(local.sum(dim=0))
        rows = D.gather_trace_rows(local.to(torch.float64), n_traces, b)
        mx = D.max_over_ranks(float(rank + 1), "cpu")
        q.put((rank, red.tolist(), rows.tolist(), mx))
    finally:
        dist.destroy_process_group()


def test_shard_range_covers_all():
    for n in (0, 1, 5, 4096):
        for w in (1, 2, 3, 8):
            got = []
            for r in range(w):
                b, e = D.shard_range(n, r, w)
                got.extend(range(b, e))
            assert got == list(range(n))
    assert D.shard_layers(5, 1, 2) == [3, 4]


def test_gloo_world2_reduce_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = torch.arange(7 * 4 * 3 * 8, dtype=torch.int64).reshape(7, 4, 3, 8)
    full[..., 7] = 0
    want = full.sum(dim=0)
    want[2, 1, 7] = 3
    for rank, red, rows, mx in out:
        assert torch.equal(torch.tensor(red), want)
        f = full.to(torch.float64)
        f[5, 2, 1, 7] = 3
        assert torch.equal(torch.tensor(rows)[..., :7], f[..., :7])
        assert mx == 2.0


def _uniform(nt=3, L=5, T=7, K=2, E=8, seed=0):
    import numpy as np
    from paper_2601_17063_b200.trace import packed_from_decode_ids
    rng = np.random.default_rng(seed)
    ids = np.stack([np.stack([np.stack([rng.choice(E, K, replace=False) for _ in range(T)]) for _ in range(L)])
                    for _ in range(nt)]).astype(np.uint8)
    return ids, packed_from_decode_ids(ids, E)


def test_slice_traces_and_layers_uniform():
    import numpy as np
    ids, p = _uniform()
    s = D.slice_traces(p, 1, 3)
    assert s.num_traces == 2 and s.total_acc == ids[1:3].size
    assert np.array_equal(s.acc[:s.total_acc], ids[1:3].reshape(-1))
    s = D.slice_layers(p, 2, 4)
    assert s.num_layers == 2 and s.num_traces == 3
    assert np.array_equal(s.acc[:s.total_acc], np.ascontiguousarray(ids[:, 2:4]).reshape(-1))
    assert len(s.acc) % 128 == 0 and len(s.acc) >= s.total_acc + 128
    assert D.shard_kind(p, 2) == "traces" and D.shard_kind(p, 4) == "layers"


def test_slice_layers_general_layout():
    """Layer slices of a prefill + multi-sequence trace (native host packer,
    no GPU) hold exactly that layer's streams, offsets rebased."""
    import numpy as np
    from paper_2601_17063_b200.trace import AccessEvent, Phase, RoutingTrace, TraceHeader, pack_trace
    rng = np.random.default_rng(3)
    L, E, K = 4, 8, 2
    ev = []
    for seq in range(2):
        for t in range(3):
            for layer in range(L):
                ev.append(AccessEvent(seq, Phase.PREFILL, t, layer, tuple(int(x) for x in rng.choice(E, 3, replace=False))))
        for t in range(5):
            for layer in range(L):
                ev.append(AccessEvent(seq, Phase.DECODE, t, layer, tuple(int(x) for x in rng.choice(E, K, replace=False))))
    p = pack_trace(RoutingTrace(TraceHeader("g", L, E, K), tuple(ev)))
    for b, e in ((0, 2), (1, 4), (3, 4)):
        s = D.slice_layers(p, b, e)
        assert s.num_layers == e - b and not s.uniform
        for i, layer in enumerate(range(b, e)):
            a0, a1 = int(p.chain_acc_off[layer]), int(p.chain_acc_off[layer + 1])
            assert np.array_equal(s.acc[s.chain_acc_off[i]:s.chain_acc_off[i + 1]], p.acc[a0:a1])
            e0, e1 = int(p.chain_ev_off[layer]), int(p.chain_ev_off[layer + 1])
            assert np.array_equal(s.ev_info[s.chain_ev_off[i]:s.chain_ev_off[i + 1]], p.ev_info[e0:e1])
            r0, r1 = int(p.chain_rt_off[layer]), int(p.chain_rt_off[layer + 1])
            assert np.array_equal(s.routed[s.chain_rt_off[i]:s.chain_rt_off[i + 1]], p.routed[r0:r1])
        assert s.decode_steps == p.decode_steps


def test_fold_layers_is_layer_order_float64():
    import numpy as np
    rng = np.random.default_rng(1)
    cr = rng.integers(0, 1000, size=(2, 5, 3, 2, 8)).astype(np.int64)
    cr[..., 7] = 0
    cr[1, 3, 2, 1, 7] = 3
    cr[1, 4, 2, 1, 7] = 5
    cl = rng.random((2, 5, 3, 2, 2)) * 10.0 ** rng.integers(-6, 3, size=(2, 5, 3, 2, 2))
    rep, lat = D.fold_layers(cr, cl)
    for t in range(2):
        for i in range(3):
            for j in range(2):
                d = p_ = 0.0
                for layer in range(5):
                    d += float(cl[t, layer, i, j, 0])
                    p_ += float(cl[t, layer, i, j, 1])
                assert lat[t, i, j, 0] == d and lat[t, i, j, 1] == p_
                assert list(rep[t, i, j, :7]) == list(cr[t, :, i, j, :7].sum(axis=0))
    assert rep[1, 2, 1, 7] == 3 and rep[0, 0, 0, 7] == 0


def _rows_worker(rank, world, port, q):
    import numpy as np
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = np.arange(6 * 4, dtype=np.float64).reshape(6, 4) * np.pi * 1e-7
        b, e = D.shard_range(6, rank, world)
        buf = np.zeros((6, 4), dtype=np.int64)
        buf[b:e] = full[b:e].view(np.int64)
        out = D._all_reduce_rows(buf, "cpu")
        q.put((rank, out.view(np.float64).tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_rows_are_bit_exact_concatenation():
    """The single collective of replay_sharded: float64 rows travel as int64
    bit patterns, owned by one rank each -> the sum is an exact concatenation."""
    import numpy as np
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = np.arange(6 * 4, dtype=np.float64).reshape(6, 4) * np.pi * 1e-7
    for _, rows in out:
        assert np.array_equal(np.array(rows), full)
