"""Multi-GPU sharding of the replay (north-star subsystem 4).

The reference's only parallel path is ``sweep(jobs)``, a thread pool over the
(policy, capacity) cells (pkg/src/moecache/engine.py:456-464).  Here every
(trace, layer, policy, capacity) instance is independent, so
one process per GPU replays a disjoint shard with no data-path collective:

* a batch of at least ``world`` traces (C4, C5) is cut into contiguous
  blocks of TRACES; each rank replays every layer of its traces;
* a single trace (C1, C2, C3, a one-trace C5) is cut into contiguous blocks
  of LAYERS; each rank replays its layers of every trace.

The only exchange is ONE all-reduce (NCCL over NVLink on a GPU node, gloo in
the CPU tests) at the end.  Every slot of the reduced buffer is written by
exactly one rank and is zero on the others, so the sum is a concatenation --
exact for the int64 counters AND for the float64 latencies, which travel as
their int64 bit patterns in the same buffer.  Layer shards send per-layer
rows; the host then folds them in layer order with the reference's float64
additions (engine.py:330-343), so every SimReport is bit-identical to a
1-GPU run (tests/test_distributed_gpu.py).
"""
from __future__ import annotations

from typing import Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .trace import PackedTrace


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block partition of n_items over world ranks: [begin, end)."""
    per = (n_items + world - 1) // world
    b = min(n_items, rank * per)
    return b, min(n_items, b + per)


def shard_layers(num_layers: int, rank: int, world: int) -> list[int]:
    """The layers of ``rank`` in the layer sharding (a contiguous block)."""
    b, e = shard_range(num_layers, rank, world)
    return list(range(b, e))


def _world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_kind(packed: PackedTrace, world: int) -> str:
    """"traces" when every rank gets at least one whole trace, else "layers"."""
    return "traces" if packed.uniform and packed.num_traces >= world else "layers"


def _pad_acc(flat: np.ndarray) -> np.ndarray:
    acc = np.zeros((flat.size + 127) // 128 * 128 + 128, dtype=np.uint8)
    acc[:flat.size] = flat
    return acc


def slice_traces(packed: PackedTrace, begin: int, end: int) -> PackedTrace:
    """Traces [begin, end) of a uniform batch (chain-major: a contiguous run)."""
    if not packed.uniform:
        raise ValueError("trace slicing needs a uniform (decode-only) batch")
    per = packed.num_layers * packed.events_per_chain * packed.top_k
    flat = packed.acc[begin * per:end * per]
    n = end - begin
    return PackedTrace(num_layers=packed.num_layers, num_experts=packed.num_experts, top_k=packed.top_k,
                       num_traces=n, uniform=True, events_per_chain=packed.events_per_chain, acc=_pad_acc(flat),
                       total_acc=flat.size, total_events=n * packed.num_layers * packed.events_per_chain,
                       decode_steps=list(packed.decode_steps[begin:end]))


def slice_layers(packed: PackedTrace, begin: int, end: int) -> PackedTrace:
    """Layers [begin, end) of every trace (chains trace * L + layer)."""
    L, nt = packed.num_layers, packed.num_traces
    nl = end - begin
    if packed.uniform:
        chain = packed.events_per_chain * packed.top_k
        ids = packed.acc[:nt * L * chain].reshape(nt, L, chain)[:, begin:end]
        flat = np.ascontiguousarray(ids).reshape(-1)
        return PackedTrace(num_layers=nl, num_experts=packed.num_experts, top_k=packed.top_k, num_traces=nt,
                           uniform=True, events_per_chain=packed.events_per_chain, acc=_pad_acc(flat),
                           total_acc=flat.size, total_events=nt * nl * packed.events_per_chain,
                           decode_steps=list(packed.decode_steps))
    if nt != 1:
        raise ValueError("general-layout batches hold one trace")
    ao, eo, ro = packed.chain_acc_off, packed.chain_ev_off, packed.chain_rt_off

    def rebase(off):
        return np.ascontiguousarray(off[begin:end + 1] - off[begin], dtype=np.int64)

    acc = packed.acc[int(ao[begin]):int(ao[end])]
    ev = np.ascontiguousarray(packed.ev_info[int(eo[begin]):int(eo[end])], dtype=np.uint32)
    rt = packed.routed[int(ro[begin]):int(ro[end])]
    return PackedTrace(num_layers=nl, num_experts=packed.num_experts, top_k=packed.top_k, num_traces=1,
                       uniform=False, events_per_chain=0, acc=_pad_acc(acc), total_acc=acc.size,
                       total_events=ev.size, chain_acc_off=rebase(ao), chain_ev_off=rebase(eo),
                       chain_rt_off=rebase(ro), ev_info=np.concatenate([ev, np.zeros(16, np.uint32)]),
                       routed=np.concatenate([rt, np.zeros(64, np.uint8)]),
                       decode_steps=list(packed.decode_steps))


def slice_nets(nets, begin: int, end: int, num_layers: int):
    """(hidden, n_nets, flat) restricted to layers [begin, end) (a shared net stays)."""
    if nets is None:
        return None
    hidden, n_nets, flat = nets
    if n_nets == 1:
        return nets
    assert n_nets == num_layers
    per = flat.size // n_nets
    return hidden, end - begin, np.ascontiguousarray(flat[begin * per:end * per])


def fold_layers(chain_reports: np.ndarray, chain_latency: np.ndarray):
    """[trace][layer][pol][cap][8] counters + [..][2] float64 latencies ->
    per-trace reports / latency, summed in layer order (engine.py:330-343):
    counters add, the status slot keeps the first non-zero layer status, and
    the latencies are float64 additions from 0.0 in layer order -- the same
    arithmetic as the on-device fold (K5)."""
    nt, L = chain_reports.shape[:2]
    rep = chain_reports.sum(axis=1)
    st = chain_reports[..., _lib.R_STATUS]
    first = np.zeros(rep.shape[:-1], dtype=np.int64)
    for layer in range(L):
        first = np.where(first == 0, st[:, layer], first)
    rep[..., _lib.R_STATUS] = first
    lat = np.zeros(chain_latency.shape[:1] + chain_latency.shape[2:], dtype=np.float64)
    for layer in range(L):
        lat = lat + chain_latency[:, layer]
    return rep, lat


def _all_reduce_rows(buf: np.ndarray, device) -> np.ndarray:
    """The single collective: sum an int64 buffer whose every slot is owned by
    one rank (zero elsewhere).  NCCL needs a CUDA tensor, gloo a CPU one."""
    rank, world = _world()
    if world == 1:
        return buf
    use_cuda = dist.get_backend() == "nccl"
    t = torch.from_numpy(buf)
    if use_cuda:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


def replay_sharded(packed: PackedTrace, codes: Sequence[int], capacities: Sequence[int], cost, window: int,
                   nets=None, *, device: int | None = None, lecar=None) -> dict:
    """``engine.replay_host`` over every rank of the default process group.

    Each rank replays its shard (traces or layers, ``shard_kind``) on its own
    GPU (``device``, default the current CUDA device); the shards' outputs are
    combined by one all-reduce.  Every rank returns the full ``reports``
    [trace][pol][cap][8] int64 and ``latency`` [trace][pol][cap][2] float64 of
    the whole batch, bit-identical to a 1-GPU ``replay_host``, plus the shard
    it replayed (``kind``, ``begin``, ``end``)."""
    from .engine import replay_host
    rank, world = _world()
    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    n_pol, n_cap = len(codes), len(capacities)
    nt, L = packed.num_traces, packed.num_layers
    kind = shard_kind(packed, world)
    width = _lib.R_N + 2
    if kind == "traces":
        b, e = shard_range(nt, rank, world)
        buf = np.zeros((nt, n_pol, n_cap, width), dtype=np.int64)
        if e > b:
            res = replay_host(slice_traces(packed, b, e), codes, capacities, cost, window, nets, device=device,
                              lecar=lecar)
            buf[b:e, ..., :_lib.R_N] = res["reports"]
            buf[b:e, ..., _lib.R_N:] = res["latency"].view(np.int64)
        buf = _all_reduce_rows(buf, device)
        reports = np.ascontiguousarray(buf[..., :_lib.R_N])
        latency = np.ascontiguousarray(buf[..., _lib.R_N:]).view(np.float64)
    else:
        b, e = shard_range(L, rank, world)
        buf = np.zeros((nt, L, n_pol, n_cap, width), dtype=np.int64)
        if e > b:
            res = replay_host(slice_layers(packed, b, e), codes, capacities, cost, window,
                              slice_nets(nets, b, e, L), device=device, want_chain=True, lecar=lecar)
            cr = res["chain_reports"].reshape(nt, e - b, n_pol, n_cap, _lib.R_N)
            cl = res["chain_latency"].reshape(nt, e - b, n_pol, n_cap, 2)
            buf[:, b:e, ..., :_lib.R_N] = cr
            buf[:, b:e, ..., _lib.R_N:] = cl.view(np.int64)
        buf = _all_reduce_rows(buf, device)
        reports, latency = fold_layers(np.ascontiguousarray(buf[..., :_lib.R_N]),
                                       np.ascontiguousarray(buf[..., _lib.R_N:]).view(np.float64))
    return {"reports": reports, "latency": latency, "kind": kind, "begin": b, "end": e, "world": world}


def sweep_sharded(trace, policies: Sequence, capacities: Sequence[int], cost=None, window: int = 5, nets=None,
                  *, device: int | None = None) -> list:
    """``sweep`` (engine.py:439-465) over every rank of the default process
    group: same arguments and the same sorted SimReport rows on every rank,
    with the replay sharded as ``replay_sharded`` does.  One engine call per
    rank for the whole (policy, capacity) cross product (<= 8 policies,
    <= 64 capacities, one LeCaR parameter set)."""
    from .engine import (CapacityTooSmallError, CostModel, SimulationError, _lib as L_, _net_params, _prepare,
                         _raise_cell_status, _resolve, assemble_report)
    cost = cost or CostModel()
    packed = _prepare(trace, cost, capacities)
    for c in capacities:
        if c < packed.top_k:
            raise CapacityTooSmallError(f"capacity {c} < top_k {packed.top_k}")
    resolved = [_resolve(p, nets) for p in policies]
    if len(resolved) > 8 or len(capacities) > 64:
        raise SimulationError("sweep_sharded: at most 8 policies x 64 capacities per call")
    lecars = {ep.lecar for _, ep in resolved if ep.lecar is not None}
    if len(lecars) > 1:
        raise SimulationError("sweep_sharded: one LeCaR parameter set per call")
    netp = None
    if any(ep.is_ml for _, ep in resolved):
        netp = _net_params(next(ep.nets for _, ep in resolved if ep.is_ml), packed.num_layers, packed.num_experts)
    res = replay_sharded(packed, [ep.code for _, ep in resolved], list(capacities), cost, window, netp,
                         device=device, lecar=next(iter(lecars), None))
    rows = []
    for i, (name, _) in enumerate(resolved):
        for j, cap in enumerate(capacities):
            _raise_cell_status(int(res["reports"][0, i, j, L_.R_STATUS]))
            rows.append(assemble_report(name, cap, window, res["reports"][0, i, j], res["latency"][0, i, j],
                                        packed.decode_steps[0]))
    return sorted(rows, key=lambda r: (r.policy, r.capacity))


def reduce_counters(counters: torch.Tensor) -> torch.Tensor:
    """Sum int64 counters [.., MCB_R_N] over ranks (the bench's single
    collective over per-(policy, capacity) aggregates).

    The status slot (index 7) is reduced with MAX so any failing cell
    surfaces; the others are summed.  Works for NCCL (CUDA tensors) and gloo
    (CPU tensors)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return counters
    status = counters[..., 7].clone()
    body = counters.clone()
    body[..., 7] = 0
    dist.all_reduce(body, op=dist.ReduceOp.SUM)
    dist.all_reduce(status, op=dist.ReduceOp.MAX)
    body[..., 7] = status
    return body


def gather_trace_rows(local: torch.Tensor, n_total: int, begin: int) -> torch.Tensor:
    """Place this rank's per-trace rows into a zeroed [n_total, ...] tensor and
    all-reduce: rows are disjoint, so the sum is a concatenation (exact)."""
    full = torch.zeros((n_total,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    full[begin:begin + local.shape[0]] = local
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(full, op=dist.ReduceOp.SUM)
    return full


def max_over_ranks(x: float, device) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class NativeCommunicator:
    """The C ABI's own NCCL communicator (mcb_comm_*): the context of one GPU
    joins an NCCL clique and sums the sharded engine's int64 buffer in place,
    without torch.distributed -- the path a non-Python caller of libmcb.so
    uses.  Rank 0 creates the id (``unique_id()``) and shares it out of band."""

    def __init__(self, nranks: int, rank: int, unique_id: bytes, device: int = 0):
        import ctypes
        self._lib = _lib.load_library()
        self._ctx = _lib.context(device)
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id)
        _lib.check(self._lib.mcb_comm_init(self._ctx, nranks, rank, buf))

    @staticmethod
    def unique_id() -> bytes:
        import ctypes
        lib = _lib.load_library()
        out = (ctypes.c_uint8 * 128)()
        _lib.check(lib.mcb_comm_unique_id(out, 128))
        return bytes(out)

    def all_reduce_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place sum of a contiguous int64 CUDA tensor over the clique."""
        import ctypes
        assert t.is_cuda and t.dtype == torch.int64 and t.is_contiguous()
        _lib.check(self._lib.mcb_comm_allreduce_i64(self._ctx, t.data_ptr(), t.numel(),
                                                    ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)))
        return t

    def close(self):
        _lib.check(self._lib.mcb_comm_destroy(self._ctx))
