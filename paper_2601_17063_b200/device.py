"""Device-resident traces and the asynchronous C-ABI entry (mcb_replay).

PyTorch is used only as the allocator / stream provider: tensors hold the
packed trace and the outputs in HBM, their data_ptr()s cross the C ABI, and
the work is enqueued on the caller's current CUDA stream.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .engine import CostModel, _cost_struct
from .trace import PackedTrace


class DeviceTrace:
    """A PackedTrace copied to (or created in) HBM."""

    def __init__(self, *, num_layers, num_experts, top_k, num_traces, uniform, events_per_chain, acc,
                 total_acc, total_events, chain_acc_off=None, chain_ev_off=None, chain_rt_off=None,
                 ev_info=None, routed=None, decode_steps=None):
        self.num_layers, self.num_experts, self.top_k = int(num_layers), int(num_experts), int(top_k)
        self.num_traces, self.uniform = int(num_traces), bool(uniform)
        self.events_per_chain = int(events_per_chain)
        self.acc = acc
        self.total_acc, self.total_events = int(total_acc), int(total_events)
        self.chain_acc_off, self.chain_ev_off, self.chain_rt_off = chain_acc_off, chain_ev_off, chain_rt_off
        self.ev_info, self.routed = ev_info, routed
        self.decode_steps = decode_steps or [self.events_per_chain] * self.num_traces

    @property
    def num_chains(self):
        return self.num_layers * self.num_traces

    @classmethod
    def from_packed(cls, p: PackedTrace, device="cuda") -> "DeviceTrace":
        def up(a):
            return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(device)
        return cls(num_layers=p.num_layers, num_experts=p.num_experts, top_k=p.top_k, num_traces=p.num_traces,
                   uniform=p.uniform, events_per_chain=p.events_per_chain, acc=up(p.acc),
                   total_acc=p.total_acc, total_events=p.total_events, chain_acc_off=up(p.chain_acc_off),
                   chain_ev_off=up(p.chain_ev_off), chain_rt_off=up(p.chain_rt_off),
                   ev_info=up(p.ev_info.view(np.int32)) if p.ev_info is not None else None,
                   routed=up(p.routed), decode_steps=list(p.decode_steps))

    @classmethod
    def from_decode_ids(cls, ids: torch.Tensor, num_experts: int) -> "DeviceTrace":
        """ids: uint8 CUDA tensor [n_traces][L][T][K] (or [L][T][K])."""
        if ids.dim() == 3:
            ids = ids.unsqueeze(0)
        n, L, T, K = ids.shape
        total = n * L * T * K
        acc = torch.zeros((total + 127) // 128 * 128 + 128, dtype=torch.uint8, device=ids.device)
        acc[:total] = ids.reshape(-1)
        return cls(num_layers=L, num_experts=num_experts, top_k=K, num_traces=n, uniform=True,
                   events_per_chain=T, acc=acc, total_acc=total, total_events=n * L * T,
                   decode_steps=[T] * n)

    def view(self) -> _lib.MCBTrace:
        v = _lib.MCBTrace()
        v.num_layers, v.num_experts, v.top_k = self.num_layers, self.num_experts, self.top_k
        v.num_traces, v.uniform = self.num_traces, int(self.uniform)
        v.events_per_chain, v.total_acc, v.total_events = self.events_per_chain, self.total_acc, self.total_events
        v.acc = self.acc.data_ptr()
        if not self.uniform:
            v.chain_acc_off = self.chain_acc_off.data_ptr()
            v.chain_ev_off = self.chain_ev_off.data_ptr()
            v.chain_rt_off = self.chain_rt_off.data_ptr()
            v.ev_info = self.ev_info.data_ptr()
            v.routed = self.routed.data_ptr()
        return v


class DeviceNets:
    """EvictionNet parameters resident in HBM (float64, .evnet order)."""

    def __init__(self, hidden: int, num_nets: int, flat: np.ndarray, num_experts: int, device="cuda"):
        self.hidden, self.num_nets, self.num_experts = int(hidden), int(num_nets), int(num_experts)
        self.params = torch.from_numpy(np.ascontiguousarray(flat, dtype=np.float64)).to(device)

    def struct(self) -> _lib.MCBNets:
        s = _lib.MCBNets()
        s.num_experts, s.hidden, s.num_nets = self.num_experts, self.hidden, self.num_nets
        s.params = self.params.data_ptr()
        return s


class DeviceReplay:
    """Reusable output buffers + one mcb_replay call per __call__ (async)."""

    def __init__(self, trace: DeviceTrace, codes, capacities, cost: CostModel = CostModel(), window: int = 5,
                 nets: DeviceNets | None = None, device: int = 0):
        self.trace, self.codes, self.caps = trace, list(codes), list(capacities)
        self.cost, self.window, self.nets = cost, window, nets
        self.device = device
        nt, npol, ncap = trace.num_traces, len(self.codes), len(self.caps)
        self.reports = torch.zeros((nt, npol, ncap, _lib.R_N), dtype=torch.int64, device=f"cuda:{device}")
        self.latency = torch.zeros((nt, npol, ncap, 2), dtype=torch.float64, device=f"cuda:{device}")
        self._pols = (ctypes.c_int32 * npol)(*self.codes)
        self._caps = (ctypes.c_int32 * ncap)(*self.caps)
        self._cost = _cost_struct(cost, window)
        self._view = trace.view()
        self._nets = nets.struct() if nets is not None else None
        self._out = _lib.MCBOutputs()
        self._out.reports = self.reports.data_ptr()
        self._out.latency = self.latency.data_ptr()
        self.ctx = _lib.context(device)
        self.lib = _lib.load_library()

    def set_timing(self, enable: bool):
        _lib.check(self.lib.mcb_set_timing(self.ctx, int(enable)))

    def stage_ms(self):
        """[K2 next-use, K3 scorer, K4 replay (non-ML launch), K4 replay (ML launch), K5 fold] in ms."""
        ms = (ctypes.c_float * 5)()
        _lib.check(self.lib.mcb_last_timings(self.ctx, ms, 5))
        return list(ms)

    def kernels_launched(self) -> int:
        k, u = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(self.lib.mcb_last_stats(self.ctx, ctypes.byref(k), ctypes.byref(u)))
        return int(k.value)

    def __call__(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = self.lib.mcb_replay(self.ctx, ctypes.byref(self._view), self._pols, len(self.codes), self._caps,
                                 len(self.caps), ctypes.byref(self._cost),
                                 ctypes.byref(self._nets) if self._nets is not None else None,
                                 ctypes.byref(self._out), ctypes.c_void_p(s.cuda_stream))
        _lib.check(rc)
        return self.reports, self.latency

    @property
    def accesses_per_call(self) -> int:
        return self.trace.total_acc * len(self.codes) * len(self.caps)
