"""Synthetic routing traces from a router-logits GEMM (north-star subsystem 1).

The reference synthesises traces with Zipf + recency sampling in numpy
(pkg/src/moecache/trace.py:186-287).  The B200 build instead produces them
the way a model does: router logits = hidden states x gate weights of every
layer (one fused GEMM over N = L*E output columns), then per (token, layer)
the top-K experts sorted by descending logit with ties to the lower id --
the torch.topk semantics of the HF routers the reference's extractor records
(pkg/extractor/src/trace_extractor/extractor.py:162-183).  Softmax is
monotone, so top-K of softmax(logits) == top-K of logits.

Workload knobs: hidden states follow an AR(1) process over tokens
(h_t = rho h_{t-1} + sqrt(1-rho^2) eps_t) which gives routing temporal
locality, and a per-layer Zipf logit bias -zipf_s * ln(1 + rank_l(e)) gives
popularity skew (rank_l a seeded permutation per layer).  The bias rides in
the GEMM as one extra K column (hidden[:, d] = 1, weight[:, d] = bias).

``route_topk`` runs the tcgen05/TMA kernel (mcb_router_topk, K1);
``route_topk_torch`` is the plain-PyTorch reference of the same op used by
the parity tests.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch

from . import _lib


@dataclass(frozen=True)
class RouterWorkload:
    num_layers: int
    num_experts: int
    top_k: int
    tokens: int
    hidden_dim: int
    seed: int = 0
    rho: float = 0.9
    zipf_s: float = 1.0


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def ar1_hidden(tokens: int, d: int, rho: float, seed: int, device="cuda", chunk: int = 8192) -> torch.Tensor:
    """bf16 [T, d_pad] hidden states; column d is the constant 1 of the bias trick.

    On a CUDA device: the engine's kernel (mcb_ar1_hidden: counter-based
    normals, chunked AR(1) scan with carries).  On the CPU (the reference
    arm's regeneration only): torch's AR(1) over tokens, chunk by chunk with a
    log-depth doubling scan inside each chunk (h_t = rho h_{t-1} + c eps_t) --
    a different random stream."""
    d_pad = (d + 1 + 63) // 64 * 64
    if torch.device(device).type == "cuda":
        out = torch.empty((tokens, d_pad), dtype=torch.bfloat16, device=device)
        lib = _lib.load_library()
        dev = out.device.index or 0
        _lib.check(lib.mcb_ar1_hidden(_lib.context(dev), tokens, d, d_pad, float(rho), int(seed) & (2 ** 64 - 1),
                                      out.data_ptr(), ctypes.c_void_p(torch.cuda.current_stream(out.device).cuda_stream)))
        return out
    out = torch.zeros((tokens, d_pad), dtype=torch.bfloat16, device=device)
    g = _gen(seed, device)
    c = math.sqrt(max(1.0 - rho * rho, 0.0))
    carry = None
    for t0 in range(0, tokens, chunk):
        n = min(chunk, tokens - t0)
        h = torch.randn((n, d), generator=g, device=device, dtype=torch.float32) * c
        if t0 == 0:
            h[0] /= c if c > 0 else 1.0    # stationary start: h_0 ~ N(0, 1)
        s, pw = 1, rho
        while s < n:
            h[s:] = h[s:] + pw * h[:-s].clone()
            s *= 2
            pw = pw * pw
        if carry is not None:
            powers = rho ** torch.arange(1, n + 1, device=device, dtype=torch.float32)
            h += powers[:, None] * carry[None, :]
        carry = h[-1].clone()
        out[t0:t0 + n, :d] = h.to(torch.bfloat16)
    out[:, d] = 1.0
    return out


def padded_experts(E: int) -> int:
    """Gate rows per layer in the weight layout: E rounded up to a power of
    two >= 8 (a divisor of the kernel's 256-column tile); padding rows are
    never selected."""
    ep = 8
    while ep < E:
        ep *= 2
    return ep


def router_weights(w: RouterWorkload, device="cuda") -> torch.Tensor:
    """bf16 [L*Ep, d_pad] gate rows of all layers (layer-major), N(0, 1/d),
    column d = the per-layer Zipf bias; rows E..Ep-1 of each layer are zero."""
    L, E, d = w.num_layers, w.num_experts, w.hidden_dim
    Ep = padded_experts(E)
    d_pad = (d + 1 + 63) // 64 * 64
    g = _gen(w.seed * 1000003 + 1, device)
    W = torch.zeros((L, Ep, d_pad), dtype=torch.float32, device=device)
    W[:, :E, :d] = torch.randn((L, E, d), generator=g, device=device) / math.sqrt(d)
    gc = torch.Generator()
    gc.manual_seed(w.seed * 7919 + 3)
    for layer in range(L):
        rank = torch.randperm(E, generator=gc)
        W[layer, :E, d] = (-w.zipf_s * torch.log1p(rank.double())).float().to(device)
    return W.reshape(L * Ep, d_pad).to(torch.bfloat16)


def route_topk_torch(hidden: torch.Tensor, weight: torch.Tensor, L: int, E: int, K: int,
                     chunk: int = 16384) -> torch.Tensor:
    """Reference: ids[l][t][:] = topk(hidden.float() @ weight.float().T)[.., l*E:(l+1)*E], sorted."""
    T = hidden.shape[0]
    Ep = weight.shape[0] // L
    out = torch.empty((L, T, K), dtype=torch.uint8, device=hidden.device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        Wf = weight.float()
        for t0 in range(0, T, chunk):
            lg = hidden[t0:t0 + chunk].float() @ Wf.T
            lg = lg.view(lg.shape[0], L, Ep)[:, :, :E]
            idx = torch.topk(lg, K, dim=-1, sorted=True).indices
            out[:, t0:t0 + lg.shape[0]] = idx.permute(1, 0, 2).to(torch.uint8)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return out


def route_topk(hidden: torch.Tensor, weight: torch.Tensor, L: int, E: int, K: int, out: torch.Tensor = None,
               logits: torch.Tensor = None, device: int = 0) -> torch.Tensor:
    """K1 (tcgen05/TMA): uint8 ids [L][T][K] (chain-major uniform layout)."""
    T, d_pad = hidden.shape
    if out is None:
        out = torch.empty((L, T, K), dtype=torch.uint8, device=hidden.device)
    lib = _lib.load_library()
    s = torch.cuda.current_stream(hidden.device)
    rc = lib.mcb_router_topk(_lib.context(device), hidden.data_ptr(), weight.data_ptr(), T, d_pad, L, E, K,
                             out.data_ptr(), logits.data_ptr() if logits is not None else None,
                             ctypes.c_void_p(s.cuda_stream))
    _lib.check(rc)
    return out


def synthetic_ids(w: RouterWorkload, impl: str = "tcgen05", device="cuda") -> torch.Tensor:
    """uint8 [L][T][K] routing ids of one synthetic trace."""
    H = ar1_hidden(w.tokens, w.hidden_dim, w.rho, w.seed * 2 + 11, device)
    W = router_weights(w, device)
    if impl == "torch":
        return route_topk_torch(H, W, w.num_layers, w.num_experts, w.top_k)
    return route_topk(H, W, w.num_layers, w.num_experts, w.top_k)
