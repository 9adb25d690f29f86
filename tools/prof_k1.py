"""Drive K1 (router_topk_kernel) alone at a BASELINE shape for ncu / timing.

    python tools/prof_k1.py --workload c3 --tokens 65536 [--reps 5]

Prints one JSON line: ms per launch (CUDA events, after warm-up), TFLOP/s of
the fused GEMM (T x d_pad x L*Ep, 2 FLOP per MAC) and HBM GB/s of its
algorithmic bytes (hidden + gate weights read once, ids written)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import WORKLOADS, measured_peaks  # noqa: E402
from paper_2601_17063_b200 import generator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--tokens", type=int, default=None)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
wl = WORKLOADS[a.workload]
T = a.tokens or wl["T"]
w = generator.RouterWorkload(wl["L"], wl["E"], wl["K"], T, wl["d"], seed=0)
H = generator.ar1_hidden(T, wl["d"], w.rho, 11, "cuda")
W = generator.router_weights(w, "cuda")
ids = generator.route_topk(H, W, w.num_layers, w.num_experts, w.top_k)
ref = generator.route_topk_torch(H, W, w.num_layers, w.num_experts, w.top_k)
agree = float((ids == ref).all(dim=-1).float().mean())
torch.cuda.synchronize()
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(a.reps):
    generator.route_topk(H, W, w.num_layers, w.num_experts, w.top_k, out=ids)
e1.record(s)
e1.synchronize()
ms = e0.elapsed_time(e1) / a.reps
Ep = generator.padded_experts(wl["E"])
flops = 2.0 * T * H.shape[1] * wl["L"] * Ep
byts = H.numel() * 2 + W.numel() * 2 + ids.numel()
hbm, bf16, src = measured_peaks()
print(json.dumps({"kernel": "router_topk_kernel", "workload": a.workload, "tokens": T,
                  "gemm": f"{T}x{H.shape[1]}x{wl['L'] * Ep}", "ms": ms, "tflops": flops / ms / 1e9,
                  "frac_bf16": flops / ms / 1e9 / bf16, "gbs": byts / ms / 1e6, "frac_hbm": byts / ms / 1e6 / hbm,
                  "rows_equal_torch": agree}))
