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
    assert D.shard_layers(5, 1, 2) == [1, 3]


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
