#!/usr/bin/env python
"""Replay-throughput benchmark (expert-cache accesses replayed per second).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c1|c4]
                    [--impl ours|reference] [--gen torch|tcgen05]

One step = one pass of the hot path (K2 next-use scan, K3 ML scorer, K4
replay, K5 fold: mcb_replay) over the workload's synthetic trace, every
policy x capacity cell, inputs resident in HBM.  L2 is flushed (256 MiB
write) before every timed step; each step is timed with CUDA events on the
launching stream and summed; N>1 takes the max over ranks.  `e2e` repeats the
measurement through the public host-buffer C-ABI entry (mcb_replay_host):
pinned host trace -> H2D -> kernels -> D2H of the reports, inside the timed
region.  `--impl reference` times the CPU restatement of the reference
(oracle/, test infrastructure) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs[1]: Mixtral-8x7B-shaped, 64K tokens, capacity sweep 2..7
    "c2": dict(name="c2-mixtral-8x7b-shaped", L=32, E=8, K=2, T=65536, d=4096, traces=1,
               caps=[2, 3, 4, 5, 6, 7], scaling="weak"),
    # configs[0]: Qwen3-30B-A3B-shaped, 2K tokens, C=32
    "c1": dict(name="c1-qwen3-30b-a3b-shaped", L=48, E=128, K=8, T=2048, d=2048, traces=1, caps=[32],
               scaling="weak"),
    # configs[2]: OLMoE-1B-7B-shaped, 1M tokens, C in {16, 32} (ML vs Belady, LRU/LFU for context)
    "c3": dict(name="c3-olmoe-1b-7b-shaped", L=16, E=64, K=8, T=1048576, d=2048, traces=1, caps=[16, 32],
               scaling="weak"),
    # configs[3]: DeepSeek-V2-Lite-shaped, 4096 traces x 2048 tokens, C=16 (traces sharded over ranks)
    "c4": dict(name="c4-deepseek-v2-lite-shaped", L=27, E=64, K=6, T=2048, d=2048, traces=4096, caps=[16],
               scaling="strong"),
}
POLICIES = ["lru", "lfu", "belady", "ml"]
METRIC = "expert-cache accesses replayed/sec"
UNIT = "accesses/s"


def bytes_per_access(policy: str, E: int, K: int) -> float:
    """Algorithmic HBM bytes per replayed access of K4:
    1 B expert id + 1/8 B hit bit; Belady +4 B next-use position; ML +E/K B
    (one uint8 score-rank row of E bytes per event of K accesses)."""
    b = 1.125
    if policy == "belady":
        b += 4.0
    if policy == "ml":
        b += E / K
    return b


def scorer_flops(E: int, H: int) -> float:
    """Algorithmic FLOPs of one EvictionNet forward (net.py:98-105): three
    GEMV layers 2E->H->H->E, 2 FLOPs per multiply-add (biases/SiLU not counted)."""
    return 2.0 * (2 * E * H + H * H + H * E)


def measured_fp64_peak():
    """float64 DMMA peak measured on this pool by tools/peak_fp64.cu
    (profiles/r1_peak_fp64.json); MEASURED_PEAKS.json carries no fp64 figure."""
    p = os.path.join(ROOT, "profiles", "r1_peak_fp64.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh)["fp64_dmma_tflops"]), "measured (profiles/r1_peak_fp64.json, DMMA.8x8x4)"
    return 40.0, "nominal B200 FP64 tensor (no measurement found)"


def ncu_traffic(workload: str) -> dict:
    """DRAM bytes per launch (dram__bytes_read.sum + write.sum) of the K3 / K4
    kernels from the committed ncu --set full capture (profiles/)."""
    p = os.path.join(ROOT, "profiles", f"r1_{workload}_traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return {}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    """(HBM GB/s, bf16 dense TFLOP/s burst, source) from MEASURED_PEAKS.json,
    else the fallback of /opt/skills/guides/B200_PROFILING.md."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1590.0)), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region.

    nvidia-smi takes ~100 ms to start, longer than a short timed region, so
    the sampler is started (and its first line awaited) before the region;
    a reader thread timestamps every line and only lines read between
    begin() and stop() count.  A region shorter than the 50 ms sampling
    period still gets the first sample taken after it began."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.t0 = None

    def start(self):
        import threading
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        first = threading.Event()

        def reader():
            for line in self.proc.stdout:
                self.lines.append((time.perf_counter(), line))
                first.set()
        threading.Thread(target=reader, daemon=True).start()
        first.wait(timeout=10)

    def begin(self):
        self.t0 = time.perf_counter()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t1 = time.perf_counter()
        t0 = self.t0 if self.t0 is not None else t1
        deadline = time.perf_counter() + 1.0
        while not any(t >= t0 for t, _ in self.lines) and time.perf_counter() < deadline:
            time.sleep(0.01)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=10)
        except Exception:
            pass
        inside = [ln for t, ln in self.lines if t0 <= t <= t1]
        if not inside:   # region shorter than the sampling period: first sample after it began
            inside = [ln for t, ln in self.lines if t >= t0][:1]
        rows = [r.split(",") for r in inside if r.strip()]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, r[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_trace_ids(wl, seed: int, gen: str, device):
    """uint8 [n_traces][L][T][K] ids from the router-GEMM generator (K1).

    Also times K1 itself (CUDA events, after one warm-up launch) on the first
    trace: returns (ids, generator report)."""
    import torch

    from paper_2601_17063_b200 import generator
    outs = []
    gen_report = None
    if gen == "reference":
        # the reference's own Zipf + recency generator, reproduced bit-exactly on the GPU
        from paper_2601_17063_b200 import refgen
        from paper_2601_17063_b200.trace import TraceHeader
        hdr = TraceHeader("bench", wl["L"], wl["E"], wl["K"])
        for i in range(wl["n_traces_local"]):
            cfg = refgen.SyntheticWorkloadConfig(num_seqs=1, decode_steps=wl["T"], prefill_tokens=0, zipf_s=1.0,
                                                 recency_boost=0.3, w_hot=4, rng_seed=seed + i)
            if gen_report is None:
                refgen.generate_decode_ids(hdr, cfg, device.index or 0)
                s = torch.cuda.current_stream(device)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                ids = refgen.generate_decode_ids(hdr, cfg, device.index or 0)
                b.record(s)
                b.synchronize()
                ms = a.elapsed_time(b)
                gen_report = {"kernel": "k_refgen (bit-exact reference generator, trace.py:212-287)", "ms": ms,
                              "draws_per_s": wl["L"] * wl["T"] * wl["K"] / ms * 1e3,
                              "config": "zipf_s=1.0, recency_boost=0.3, w_hot=4 (SURVEY.md 8d)"}
            else:
                ids = refgen.generate_decode_ids(hdr, cfg, device.index or 0)
            outs.append(ids)
        return torch.stack(outs), gen_report
    for i in range(wl["n_traces_local"]):
        w = generator.RouterWorkload(wl["L"], wl["E"], wl["K"], wl["T"], wl["d"], seed=seed + i)
        H = generator.ar1_hidden(w.tokens, w.hidden_dim, w.rho, w.seed * 2 + 11, device)
        W = generator.router_weights(w, device)
        if gen == "torch":
            ids = generator.route_topk_torch(H, W, w.num_layers, w.num_experts, w.top_k)
        else:
            ids = generator.route_topk(H, W, w.num_layers, w.num_experts, w.top_k)
            if gen_report is None:
                s = torch.cuda.current_stream(device)
                reps = 5
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                for _ in range(reps):
                    generator.route_topk(H, W, w.num_layers, w.num_experts, w.top_k, out=ids)
                b.record(s)
                b.synchronize()
                ms = a.elapsed_time(b) / reps
                Ep = generator.padded_experts(w.num_experts)
                flops = 2.0 * w.tokens * H.shape[1] * w.num_layers * Ep
                hbm = H.numel() * 2 + W.numel() * 2 + ids.numel()
                gen_report = {"kernel": "router_topk_kernel (K1, tcgen05.mma kind::f16 + TMA, fused top-k)",
                              "ms": ms, "tflops": flops / ms / 1e9, "gbs": hbm / ms / 1e6,
                              "tokens": w.tokens, "gemm": f"{w.tokens}x{H.shape[1]}x{w.num_layers * Ep}"}
        outs.append(ids)
        del H, W
    return torch.stack(outs), gen_report


def nets_for(L: int, E: int):
    from paper_2601_17063_b200 import EvictionNet
    flat = np.concatenate([EvictionNet(E, seed=l).flat_params() for l in range(L)])
    return 128, L, flat


def cpu_sample(wl, ids_np, threads):
    """Time the CPU restatement of the reference (oracle/) on a bounded sample."""
    import oracle
    L, E, K, T = wl["L"], wl["E"], wl["K"], wl["T"]
    n_layers = wl.get("cpu_layers", 4)
    t_tokens = min(T, wl.get("cpu_tokens", T))
    chains = np.ascontiguousarray(ids_np[0, :n_layers, :t_tokens])
    jobs = [(p, c) for p in POLICIES for c in wl["caps"]]
    nets = nets_for(n_layers, E)
    t0 = time.perf_counter()
    oracle.replay_uniform(chains, n_layers, E, jobs, None, 5, nets, threads=threads)
    dt = time.perf_counter() - t0
    acc = n_layers * t_tokens * K * len(jobs)
    return acc / dt, dt, f"{n_layers} of {L} layers x {t_tokens} tokens x {len(jobs)} (policy, capacity) cells " \
                         f"= {acc} accesses in {dt:.2f} s"


def run_reference(args, wl, rank):
    """--impl reference: the CPU port of the reference path on the host cores."""
    if rank != 0:
        return
    import torch

    from paper_2601_17063_b200 import generator
    threads = os.cpu_count() or 1
    L, E, K, T = wl["L"], wl["E"], wl["K"], wl["T"]
    n_layers = wl.get("cpu_layers", 4)
    # synthesise the same-shape trace on the CPU (no GPU code on this arm)
    w = generator.RouterWorkload(L, E, K, T, wl["d"], seed=args.seed)
    H = generator.ar1_hidden(T, wl["d"], w.rho, w.seed * 2 + 11, device="cpu")
    Wt = generator.router_weights(w, device="cpu")[: n_layers * E]
    ids = generator.route_topk_torch(H, Wt, n_layers, E, K).numpy()[None]
    del H
    vals = []
    sample = ""
    for i in range(args.warmup + args.steps):
        v, dt, sample = cpu_sample(dict(wl, L=n_layers, cpu_layers=n_layers), ids, threads)
        if i >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals))
    acc_per_step = n_layers * min(T, wl.get("cpu_tokens", T)) * K * len(POLICIES) * len(wl["caps"])
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * acc_per_step / value,
        "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None, "dtype": "u8/u32 (scorer f64)",
        "data": "synthetic (router-GEMM trace, generated on the CPU for this arm)",
        "config": {"workload": wl["name"], "layers": L, "experts": E, "top_k": K, "tokens": T,
                   "capacities": wl["caps"], "policies": POLICIES},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--gen", default="tcgen05", choices=["torch", "tcgen05", "reference"],
                    help="trace source: K1 router-GEMM generator (tcgen05 / torch) or the reference's "
                         "Zipf + recency generator reproduced bit-exactly on the GPU")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--traces", type=int, default=None, help="override the workload's trace count (diagnostics)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--policies", default="lru,lfu,belady,ml", help="comma list (diagnostics only)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = dict(WORKLOADS[args.workload])
    if args.traces:
        wl["traces"] = args.traces
    rank, world, local = dist_env()
    POLICIES[:] = args.policies.split(",")

    if args.impl == "reference":
        run_reference(args, wl, rank)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if wl["scaling"] == "strong":
        per = (wl["traces"] + world - 1) // world
        wl["n_traces_local"] = max(0, min(per, wl["traces"] - rank * per))
    else:
        wl["n_traces_local"] = wl["traces"]

    from paper_2601_17063_b200 import _lib
    from paper_2601_17063_b200.device import DeviceNets, DeviceReplay, DeviceTrace
    from paper_2601_17063_b200.engine import CostModel, replay_host
    from paper_2601_17063_b200.trace import packed_from_decode_ids

    L, E, K, T = wl["L"], wl["E"], wl["K"], wl["T"]
    codes = [{"lru": _lib.MCB_LRU, "lfu": _lib.MCB_LFU, "belady": _lib.MCB_BELADY, "ml": _lib.MCB_ML}[p]
             for p in POLICIES]
    ids, gen_report = make_trace_ids(wl, args.seed + 1000 * rank, args.gen, dev)
    torch.cuda.synchronize()
    dtrace = DeviceTrace.from_decode_ids(ids, E)
    hidden, n_nets, flat = nets_for(L, E)
    dnets = DeviceNets(hidden, n_nets, flat, E, device=dev)
    rep = DeviceReplay(dtrace, codes, wl["caps"], CostModel(), 5, dnets, device=local)
    rep.set_timing(True)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)

    for _ in range(args.warmup):
        rep()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stage = np.zeros(5)
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.begin()
    for i in range(args.steps):
        flush.zero_()
        starts[i].record(stream)
        rep()
        ends[i].record(stream)
        launches += rep.kernels_launched()
        ends[i].synchronize()
        stage += np.array(rep.stage_ms())
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    dev_stats = _lib.read_stats(local)   # last step: [uncertain scorer events, seg fix-up events, ...]
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(sum(step_ms))
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    counters = rep.reports.sum(dim=0).to(torch.int64)  # [pol][cap][8] for this rank
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(counters, op=dist.ReduceOp.SUM)   # the single NCCL reduce of counters
    total_ms = float(t.item())
    acc_rank = rep.accesses_per_call
    acc_all = torch.tensor([acc_rank], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(acc_all)
    acc_all = int(acc_all.item())
    value = acc_all * args.steps / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps

    # Rooflines.  In the timed steps the non-ML replay runs on a side stream
    # concurrently with K3, so the stage spans overlap; an attribution pass
    # (same call, every stage on one stream: MCB_TUNE_SERIAL, CUDA events on
    # that stream, not under a profiler) times each stage alone.  K4 (replay)
    # is charged its algorithmic HBM bytes, K3 (scorer) its algorithmic
    # float64 FLOPs on the DMMA pipe; the line's "roofline" is the stage with
    # the larger attributed time.
    _lib.set_tuning(_lib.MCB_TUNE_SERIAL, 1, local)
    attr = np.zeros(5)
    n_attr = 3
    for _ in range(n_attr + 1):
        flush.zero_()
        rep()
        torch.cuda.synchronize()
        if _ > 0:
            attr += np.array(rep.stage_ms())
    _lib.set_tuning(_lib.MCB_TUNE_SERIAL, 0, local)
    attr /= n_attr
    replay_ms = attr[2] + attr[3]
    n_acc_cell = dtrace.total_acc
    alg_bytes = sum(bytes_per_access(p, E, K) * n_acc_cell * len(wl["caps"]) for p in POLICIES)
    peak, bf16_peak, peak_kind = measured_peaks()
    if gen_report and "tflops" in gen_report:
        gen_report["frac_of_bf16_peak"] = gen_report["tflops"] / bf16_peak
        gen_report["frac_of_hbm"] = gen_report["gbs"] / peak
    traffic = ncu_traffic(args.workload)
    k4_gbs = alg_bytes / (replay_ms / 1e3) / 1e9 if replay_ms > 0 else 0.0
    roof_k4 = {"bound": "hbm", "achieved": k4_gbs, "peak": peak, "unit": "GB/s", "frac": k4_gbs / peak,
               "traffic": traffic.get("k4"), "kernel": "K4 replay (k_seg_spec + k_seg_finish / k_replay)",
               "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
               "algorithmic_bytes_per_step": alg_bytes, "ms_per_step": replay_ms,
               "note": "sequential per-instance chains: issue/latency-bound, not HBM-bound (DESIGN.md 4); "
                       "time from the serial attribution pass"}
    roof_k3 = None
    if "ml" in POLICIES:
        k3_ms = attr[1]
        flops = scorer_flops(E, 128) * dtrace.total_events
        fp64_peak, fp64_src = measured_fp64_peak()
        tf = flops / (k3_ms / 1e3) / 1e12 if k3_ms > 0 else 0.0
        roof_k3 = {"bound": "tensor", "achieved": tf, "peak": fp64_peak, "unit": "TFLOP/s",
                   "frac": tf / fp64_peak, "traffic": traffic.get("k3"),
                   "kernel": "K3 scorer (k_score_tile: float64 DMMA.8x8x4 MLP + features + ranks)",
                   "peak_source": fp64_src, "algorithmic_flops_per_step": flops, "ms_per_step": k3_ms,
                   "note": "time from the serial attribution pass (includes the feature-snapshot kernels)"}
    roofline = roof_k3 if roof_k3 is not None and roof_k3["ms_per_step"] > replay_ms else roof_k4

    # e2e through the public host-buffer API (pinned host trace, H2D + D2H inside the timed region)
    e2e = None
    if wl["n_traces_local"] > 0:
        ids_host = torch.empty(ids.shape, dtype=torch.uint8, pin_memory=True)
        ids_host.copy_(ids)
        packed = packed_from_decode_ids(ids_host.numpy(), E)
        acc_pinned = torch.empty(packed.acc.shape, dtype=torch.uint8, pin_memory=True)
        acc_pinned.numpy()[:] = packed.acc
        packed.acc = acc_pinned.numpy()
        flat_pinned = torch.empty(flat.shape, dtype=torch.float64, pin_memory=True)
        flat_pinned.numpy()[:] = flat
        nets_host = (hidden, n_nets, flat_pinned.numpy())
        e2e_steps = args.e2e_steps or args.steps
        for _ in range(2):
            replay_host(packed, codes, wl["caps"], CostModel(), 5, nets_host, device=local,
                        stream=stream.cuda_stream)
        torch.cuda.synchronize()
        e_ms = 0.0
        for _ in range(e2e_steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            res = replay_host(packed, codes, wl["caps"], CostModel(), 5, nets_host, device=local,
                              stream=stream.cuda_stream)
            b.record(stream)
            b.synchronize()
            e_ms += a.elapsed_time(b)
        te = torch.tensor([e_ms / e2e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_step = float(te.item())
        n_cells = packed.num_traces * len(codes) * len(wl["caps"])
        e2e = {"value": acc_all / (e_step / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(packed.total_acc + flat.nbytes),
               "d2h_bytes_per_step": int(n_cells * (8 * 8 + 2 * 8) + 8),
               "ms_per_step": e_step}
        assert np.array_equal(res["reports"], rep.reports.cpu().numpy()), "e2e and device path disagree"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, dt, sample = cpu_sample(wl, ids.cpu().numpy(), threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample}

    if rank == 0:
        c = counters.cpu().numpy()
        hit_rates = {f"{p}@{cap}": round(float((c[i, j, 0] + c[i, j, 2]) / max(1, c[i, j, :4].sum())), 6)
                     for i, p in enumerate(POLICIES) for j, cap in enumerate(wl["caps"])}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": wl["scaling"], "vs_baseline": None, "dtype": "u8/u32 (scorer f64)",
            "data": ("synthetic (reference Zipf+recency generator, bit-exact on GPU" if args.gen == "reference"
                     else f"synthetic (router-GEMM trace via {args.gen}") + "; random-init EvictionNet(E, seed=layer))",
            "config": {"workload": wl["name"], "layers": L, "experts": E, "top_k": K, "tokens": T,
                       "traces_total": wl["traces"] if wl["scaling"] == "strong" else wl["traces"] * world,
                       "capacities": wl["caps"], "policies": POLICIES, "parallelism": f"shard{world}",
                       "l2": "flushed before every timed step (256 MiB write)",
                       "stage_ms_serial_attribution": {"k2_next_use": attr[0], "k3_scorer": attr[1],
                                                       "k4_replay_non_ml": attr[2], "k4_replay_ml": attr[3],
                                                       "k5_fold": attr[4]},
                       "stage_ms_per_step": {"k2_next_use": stage[0] / args.steps, "k3_scorer": stage[1] / args.steps,
                                             "k4_replay_non_ml": stage[2] / args.steps,
                                             "k4_replay_ml": stage[3] / args.steps, "k5_fold": stage[4] / args.steps,
                                             "note": "K4(non-ML) runs on a side stream concurrently with "
                                                     "K3 -> K4(ML); K4 stages include the segmented "
                                                     "spec + finish kernels when used"}},
            "roofline": roofline,
            "rooflines": {"k3_scorer": roof_k3, "k4_replay": roof_k4},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "gpu_launches": launches,
            "scorer_uncertain_events": dev_stats[0],
            "segmented_replay": {"fixup_events": dev_stats[1], "unconverged_segments": dev_stats[2],
                                 "segments": dev_stats[3], "slow_latency_folds": dev_stats[4]},
            "generator": gen_report,
            "hit_rates": hit_rates,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
