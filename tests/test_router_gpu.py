"""K1 (tcgen05/TMA router GEMM + top-k) against the plain-PyTorch fp32
reference of the same op.  Bar: logits within 2e-3 absolute of torch's fp32
GEMM on the same bf16 inputs (different fp32 summation order), and top-k ids
identical except where the k-th and (k+1)-th logits are closer than that."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2601_17063_b200 import generator  # noqa: E402


def _check(T, d, L, E, K, seed=0):
    w = generator.RouterWorkload(L, E, K, T, d, seed=seed)
    H = generator.ar1_hidden(T, d, 0.9, seed + 5)
    W = generator.router_weights(w)
    Ep = generator.padded_experts(E)
    logits = torch.zeros((T, L * Ep), dtype=torch.float32, device="cuda")
    ids = generator.route_topk(H, W, L, E, K, logits=logits)
    torch.cuda.synchronize()
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    ref_logits = H.float() @ W.float().T
    torch.backends.cuda.matmul.allow_tf32 = prev
    assert torch.allclose(logits, ref_logits, atol=2e-3, rtol=0), (logits - ref_logits).abs().max()
    ref = generator.route_topk_torch(H, W, L, E, K)
    got, want = ids.cpu().numpy(), ref.cpu().numpy()
    lg = ref_logits.view(T, L, Ep)[:, :, :E].permute(1, 0, 2).cpu().numpy()   # [L][T][E]
    srt = -np.sort(-lg, axis=-1)
    gap = srt[..., K - 1] - (srt[..., K] if K < E else -np.inf)
    ok_rows = np.all(np.diff(srt[..., :K + (1 if K < E else 0)], axis=-1) < -4e-3, axis=-1)
    mism = np.any(got != want, axis=-1)
    assert not np.any(mism & ok_rows), int(np.sum(mism & ok_rows))
    # every emitted id set is a valid top-K (distinct, in range)
    assert np.all(got < E)
    assert np.all(np.sort(got, axis=-1)[..., 1:] != np.sort(got, axis=-1)[..., :-1]) if K > 1 else True
    return float(np.mean(mism)), gap


@pytest.mark.parametrize("T,d,L,E,K", [
    (1024, 4096, 32, 8, 2),      # Mixtral-shaped (N = 256: one column tile)
    (512, 2048, 48, 128, 8),     # Qwen3-shaped (N = 6144)
    (300, 2048, 16, 64, 8),      # OLMoE-shaped, ragged token tile
    (256, 2048, 27, 64, 6),      # DeepSeek-V2-Lite-shaped, N not a multiple of 256
    (130, 128, 3, 6, 2),         # padded experts (E=6 -> 8 rows per layer)
])
def test_router_topk_matches_torch(T, d, L, E, K):
    frac, _ = _check(T, d, L, E, K)
    assert frac < 0.01


def test_ar1_hidden_kernel_statistics():
    """K1's input kernel (mcb_ar1_hidden): stationary N(0, 1) columns with
    lag-1 correlation rho, continuous across the 512-token chunk boundaries
    (the residual h_t - rho h_{t-1} has variance 1 - rho^2 everywhere),
    bias column = 1, padding = 0, deterministic per seed."""
    T, d, rho = 3000, 256, 0.9
    H = generator.ar1_hidden(T, d, rho, 7)
    assert H.shape == (T, (d + 1 + 63) // 64 * 64) and H.dtype == torch.bfloat16
    assert torch.equal(H, generator.ar1_hidden(T, d, rho, 7))
    assert not torch.equal(H, generator.ar1_hidden(T, d, rho, 8))
    h = H[:, :d].float()
    assert torch.all(H[:, d] == 1) and torch.all(H[:, d + 1:] == 0)
    assert abs(float(h.mean())) < 0.05 and abs(float(h.var()) - 1.0) < 0.1
    r = h[1:] - rho * h[:-1]
    c2 = 1 - rho * rho
    assert abs(float(r.var()) - c2) < 0.03
    at_boundary = r[[t - 1 for t in range(512, T, 512)]]      # rows t = 512, 1024, ...
    assert abs(float(at_boundary.var()) - c2) < 0.06
    lag1 = float((h[1:] * h[:-1]).mean() / h.var())
    assert abs(lag1 - rho) < 0.02
