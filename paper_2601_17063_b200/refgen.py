"""Bit-exact GPU reproduction of the reference's synthetic trace generator.

The reference samples routing traces with numpy (pkg/src/moecache/trace.py:
147-287): a per-layer Zipf popularity over a seeded permutation of the
experts, and K draws without replacement per (token, layer) from the mixture
(1 - recency_boost) * popularity + recency_boost * uniform(hot set of the last
w_hot events).  ``generate_trace`` here returns the identical trace, computed
by ``mcb_gen_reference`` (csrc/mcb_refgen.cu): one GPU thread per (sequence,
layer) jumps the reference's single PCG64 stream to its own draws and
restates numpy's float path bit for bit.  Only the O(L*E) popularity table and
the stream's initial state are prepared on the host (numpy's own
``default_rng`` / ``permutation``, as trace.py:186-202 and :262 do).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .trace import AccessEvent, InvalidConfigError, Phase, RoutingTrace, TraceHeader, packed_from_decode_ids

M64 = (1 << 64) - 1


@dataclass(frozen=True)
class SyntheticWorkloadConfig:
    """Workload knobs of the reference generator (trace.py:147-183)."""

    num_seqs: int = 1
    decode_steps: int = 256
    prefill_tokens: int = 32
    zipf_s: float = 1.0
    recency_boost: float = 0.0
    w_hot: int = 4
    rng_seed: int = 0
    popularity_seed: Optional[int] = None

    def validate(self) -> None:
        if self.num_seqs < 1:
            raise InvalidConfigError(f"num_seqs must be >= 1, got {self.num_seqs}")
        if self.decode_steps < 0:
            raise InvalidConfigError(f"decode_steps must be >= 0, got {self.decode_steps}")
        if self.prefill_tokens < 0:
            raise InvalidConfigError(f"prefill_tokens must be >= 0, got {self.prefill_tokens}")
        if self.zipf_s < 0:
            raise InvalidConfigError(f"zipf_s must be >= 0, got {self.zipf_s}")
        if not 0.0 <= self.recency_boost <= 1.0:
            raise InvalidConfigError(f"recency_boost must lie in [0, 1], got {self.recency_boost}")
        if self.w_hot < 1:
            raise InvalidConfigError(f"w_hot must be >= 1, got {self.w_hot}")


def expert_popularity(header: TraceHeader, cfg: SyntheticWorkloadConfig, layer: int) -> np.ndarray:
    """The stationary per-expert routing probabilities of one layer (trace.py:205-209)."""
    header.validate()
    cfg.validate()
    return layer_popularity(header, cfg)[layer]


def layer_popularity(header: TraceHeader, cfg: SyntheticWorkloadConfig) -> np.ndarray:
    """float64 [L][E]: Zipf mass (r+1)^-s over a per-layer seeded permutation
    (the numpy draws of trace.py:186-202)."""
    seed = cfg.rng_seed if cfg.popularity_seed is None else cfg.popularity_seed
    rng = np.random.default_rng([seed & M64, 0])
    ranks = np.arange(1, header.num_experts + 1, dtype=np.float64)
    mass = ranks ** (-cfg.zipf_s)
    mass /= mass.sum()
    probs = np.empty((header.num_layers, header.num_experts))
    for layer in range(header.num_layers):
        probs[layer, rng.permutation(header.num_experts)] = mass
    return probs


def stream_state(cfg: SyntheticWorkloadConfig) -> np.ndarray:
    """{state_hi, state_lo, inc_hi, inc_lo} of default_rng([rng_seed, 1]) (trace.py:262)."""
    st = np.random.default_rng([cfg.rng_seed & M64, 1]).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    return np.array([s >> 64, s & M64, inc >> 64, inc & M64], dtype=np.uint64)


def generate_experts(header: TraceHeader, cfg: SyntheticWorkloadConfig, device: int = 0) -> torch.Tensor:
    """uint8 CUDA tensor [num_seqs][prefill + decode][L][K]: the routed experts
    of every event in the reference's event order."""
    header.validate()
    cfg.validate()
    L, E, K = header.num_layers, header.num_experts, header.top_k
    toks = cfg.prefill_tokens + cfg.decode_steps
    dev = torch.device("cuda", device)
    pop = torch.from_numpy(layer_popularity(header, cfg)).to(dev)
    st = np.ascontiguousarray(stream_state(cfg))          # host array (read by the host entry point)
    out = torch.empty((cfg.num_seqs, toks, L, K), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream(dev)
    lib = _lib.load_library()
    _lib.check(lib.mcb_gen_reference(_lib.context(device), L, E, K, cfg.num_seqs, cfg.prefill_tokens,
                                     cfg.decode_steps, cfg.w_hot, float(cfg.recency_boost), pop.data_ptr(),
                                     st.ctypes.data, out.data_ptr(), ctypes.c_void_p(s.cuda_stream)))
    return out


def generate_trace(header: TraceHeader, cfg: SyntheticWorkloadConfig, device: int = 0) -> RoutingTrace:
    """Drop-in for the reference's ``generate_trace`` (trace.py:246-287)."""
    ex = generate_experts(header, cfg, device).cpu().numpy()
    events = []
    for seq in range(cfg.num_seqs):
        for t in range(cfg.prefill_tokens + cfg.decode_steps):
            phase = Phase.PREFILL if t < cfg.prefill_tokens else Phase.DECODE
            step = t if t < cfg.prefill_tokens else t - cfg.prefill_tokens
            for layer in range(header.num_layers):
                events.append(AccessEvent(seq, phase, step, layer, tuple(int(x) for x in ex[seq, t, layer])))
    trace = RoutingTrace(header, tuple(events))
    trace.validate()
    return trace


def generate_decode_ids(header: TraceHeader, cfg: SyntheticWorkloadConfig, device: int = 0) -> torch.Tensor:
    """Decode-only single-sequence workloads (the bench shapes): uint8 CUDA
    tensor [L][T][K] in the engine's chain-major layout, never leaving HBM."""
    if cfg.num_seqs != 1 or cfg.prefill_tokens != 0:
        raise InvalidConfigError("generate_decode_ids needs num_seqs == 1 and prefill_tokens == 0")
    return generate_experts(header, cfg, device)[0].permute(1, 0, 2).contiguous()


def generate_decode_batch(header: TraceHeader, seeds, decode_steps: int, *, popularity_seed: int,
                          zipf_s: float = 1.0, recency_boost: float = 0.0, w_hot: int = 4,
                          device: int = 0) -> torch.Tensor:
    """Many decode-only single-sequence traces in one launch: trace i is
    ``generate_trace(header, SyntheticWorkloadConfig(num_seqs=1, decode_steps,
    prefill_tokens=0, zipf_s, recency_boost, w_hot, rng_seed=seeds[i],
    popularity_seed))`` -- uint8 CUDA tensor [n][L][T][K], chain-major."""
    cfg0 = SyntheticWorkloadConfig(num_seqs=1, decode_steps=decode_steps, prefill_tokens=0, zipf_s=zipf_s,
                                   recency_boost=recency_boost, w_hot=w_hot, rng_seed=0,
                                   popularity_seed=popularity_seed)
    header.validate()
    cfg0.validate()
    L, E, K = header.num_layers, header.num_experts, header.top_k
    dev = torch.device("cuda", device)
    pop = torch.from_numpy(layer_popularity(header, cfg0)).to(dev)
    st = np.stack([stream_state(SyntheticWorkloadConfig(rng_seed=int(s))) for s in seeds]) if len(seeds) else \
        np.zeros((0, 4), dtype=np.uint64)
    dst = torch.from_numpy(np.ascontiguousarray(st).view(np.int64)).to(dev)
    out = torch.empty((len(seeds), L, decode_steps, K), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream(dev)
    lib = _lib.load_library()
    _lib.check(lib.mcb_gen_reference_batch(_lib.context(device), L, E, K, len(seeds), decode_steps, w_hot,
                                           float(recency_boost), pop.data_ptr(), dst.data_ptr(), out.data_ptr(),
                                           ctypes.c_void_p(s.cuda_stream)))
    return out
