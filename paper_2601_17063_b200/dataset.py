"""Belady-labelled training data on the GPU.

Drop-in for the reference's ``build_training_data`` (pkg/src/moecache/
dataset.py:35-96): per layer and decode step the float64 feature vector, the
capped next-routing-distance targets and the Belady residency mask at the
label capacity, computed by ``mcb_training_data`` for every event (the K3
feature scan, a reverse next-routing scan and the Belady replay with
per-event resident-set output) and reduced here to the decode events.  Any
trace: prefill (``include_prefill`` decides whether prefill events update the
feature tracker) and several sequences.  Bit-identical to the reference
(tests/test_dataset_gpu.py).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import DeviceTrace
from .trace import PackedTrace, pack_trace

DEFAULT_DISTANCE_CAP = 64


@dataclass
class LayerDataset:
    features: np.ndarray   # (N, 2E) float64
    targets: np.ndarray    # (N, E) float64 in [0, 1]
    masks: np.ndarray      # (N, E) bool

    def __len__(self) -> int:
        return self.features.shape[0]


def build_training_data_device(trace: DeviceTrace, capacity: int, distance_cap: int = DEFAULT_DISTANCE_CAP,
                               include_prefill: bool = True, device: int = 0):
    """(features [event][2E], targets [event][E], masks [event][E]) CUDA tensors
    for every event of every chain (mcb_trace order)."""
    n, E = trace.total_events, trace.num_experts
    dev = trace.acc.device
    feats = torch.empty((max(n, 1), 2 * E), dtype=torch.float64, device=dev)
    targs = torch.empty((max(n, 1), E), dtype=torch.float64, device=dev)
    masks = torch.empty((max(n, 1), E), dtype=torch.uint8, device=dev)
    v = trace.view()
    s = torch.cuda.current_stream(dev)
    _lib.check(_lib.load_library().mcb_training_data(_lib.context(device), ctypes.byref(v), int(capacity),
                                                     int(distance_cap), int(bool(include_prefill)),
                                                     feats.data_ptr(), targs.data_ptr(), masks.data_ptr(),
                                                     ctypes.c_void_p(s.cuda_stream)))
    return feats[:n], targs[:n], masks[:n]


def build_training_data(trace, capacity: int, distance_cap: int = DEFAULT_DISTANCE_CAP,
                        include_prefill: bool = True, device: int = 0) -> dict:
    """One LayerDataset per layer, samples = the layer's decode events (dataset.py:35-96)."""
    packed = trace if isinstance(trace, PackedTrace) else pack_trace(trace)
    if capacity < packed.top_k:
        raise ValueError(f"capacity {capacity} is below top_k {packed.top_k}")
    if distance_cap < 1:
        raise ValueError(f"distance_cap must be >= 1, got {distance_cap}")
    if packed.num_traces != 1:
        raise ValueError("build_training_data takes one trace")
    dt = DeviceTrace.from_packed(packed, device=torch.device("cuda", device))
    f, t, m = build_training_data_device(dt, capacity, distance_cap, include_prefill, device)
    f, t, m = f.cpu().numpy(), t.cpu().numpy(), m.cpu().numpy().astype(bool)
    E, L = packed.num_experts, packed.num_layers
    out = {}
    for layer in range(L):
        if packed.uniform:
            e0, e1 = layer * packed.events_per_chain, (layer + 1) * packed.events_per_chain
            sel = np.arange(e0, e1)
        else:
            e0, e1 = int(packed.chain_ev_off[layer]), int(packed.chain_ev_off[layer + 1])
            dec = ((packed.ev_info[e0:e1] >> 30) & 1).astype(bool)
            sel = e0 + np.nonzero(dec)[0]
        out[layer] = LayerDataset(features=f[sel] if len(sel) else np.zeros((0, 2 * E)),
                                  targets=t[sel] if len(sel) else np.zeros((0, E)),
                                  masks=m[sel] if len(sel) else np.zeros((0, E), dtype=bool))
    return out
