"""Belady-labelled training data on the GPU.

Drop-in for the reference's ``build_training_data`` (pkg/src/moecache/
dataset.py:35-96) on decode-only single-sequence traces: per layer and
decode step the float64 feature vector, the capped next-use-distance targets
and the Belady residency mask at the label capacity, computed by
``mcb_training_data`` (the K3 feature scan, a reverse next-routing scan and
the Belady replay with per-event resident-set output).  Bit-identical to the
reference (tests/test_dataset_gpu.py).
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
                               device: int = 0):
    """(features [chain][T][2E], targets [chain][T][E], masks [chain][T][E]) CUDA tensors."""
    if not trace.uniform:
        raise ValueError("GPU training data needs a decode-only single-sequence trace")
    n, T, E = trace.num_chains, trace.events_per_chain, trace.num_experts
    dev = trace.acc.device
    feats = torch.empty((n, T, 2 * E), dtype=torch.float64, device=dev)
    targs = torch.empty((n, T, E), dtype=torch.float64, device=dev)
    masks = torch.empty((n, T, E), dtype=torch.uint8, device=dev)
    v = trace.view()
    s = torch.cuda.current_stream(dev)
    _lib.check(_lib.load_library().mcb_training_data(_lib.context(device), ctypes.byref(v), int(capacity),
                                                     int(distance_cap), feats.data_ptr(), targs.data_ptr(),
                                                     masks.data_ptr(), ctypes.c_void_p(s.cuda_stream)))
    return feats, targs, masks


def build_training_data(trace, capacity: int, distance_cap: int = DEFAULT_DISTANCE_CAP,
                        include_prefill: bool = True, device: int = 0) -> dict:
    """One LayerDataset per layer (dataset.py:35-96).  ``include_prefill`` has
    no effect on decode-only traces, the only ones the GPU path accepts."""
    if distance_cap < 1:
        raise ValueError(f"distance_cap must be >= 1, got {distance_cap}")
    packed = trace if isinstance(trace, PackedTrace) else pack_trace(trace)
    if packed.num_traces != 1:
        raise ValueError("build_training_data takes one trace")
    if capacity < packed.top_k:
        raise ValueError(f"capacity {capacity} is below top_k {packed.top_k}")
    dt = DeviceTrace.from_packed(packed, device=torch.device("cuda", device))
    f, t, m = build_training_data_device(dt, capacity, distance_cap, device)
    f, t, m = f.cpu().numpy(), t.cpu().numpy(), m.cpu().numpy().astype(bool)
    return {layer: LayerDataset(features=f[layer], targets=t[layer], masks=m[layer])
            for layer in range(packed.num_layers)}
