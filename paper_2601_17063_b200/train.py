"""EvictionNet training on the GPU (net.py:107-279).

``train_eviction_net`` is the reference's drop-in (same arguments, same
``TrainResult``, same errors, same early stopping); ``train_eviction_nets``
trains many nets at once -- one per layer, as the reference's ``train``
command does one after the other (cli.py:253-283) -- so every mini-batch
step is one batched launch sequence for all layers.  The epoch loop, the
train/validation split, the seeded per-epoch permutation and the early
stopping rule run here on the host exactly as the reference orders them; the
mini-batch steps and the evaluations run in libmcb (K10, csrc/mcb_train.cu).

Numerics: float64 throughout.  AdamW, the masked-MSE gradient and the SiLU
arithmetic follow the reference's operation order; the GEMMs (cuBLAS DGEMM)
and ``exp`` differ from numpy in the last bits, so parameters match the
reference trainer to a tolerance, not bit for bit (tests/test_train_gpu.py).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from .net import EvictionNet, NetError, PARAM_NAMES, ShapeMismatchError


class EmptyDatasetError(NetError):
    pass


class NonFiniteLossError(NetError):
    pass


@dataclass
class TrainConfig:
    learning_rate: float = 1e-3
    weight_decay: float = 1e-2
    betas: tuple = (0.9, 0.999)
    eps: float = 1e-8
    epochs: int = 200
    patience: int = 10
    batch_size: int = 256
    val_fraction: float = 0.1
    seed: int = 0


@dataclass
class TrainResult:
    net: EvictionNet
    train_mse: list = field(default_factory=list)
    val_mse: list = field(default_factory=list)
    best_epoch: int = 0
    stopped_epoch: int = 0


def masked_mse(pred, target, mask) -> float:
    """Mean squared error over the masked positions, 0.0 if none (net.py:141-147)."""
    m = np.asarray(mask).astype(np.float64)
    denom = m.sum()
    if denom == 0:
        return 0.0
    return float((m * (np.asarray(pred) - np.asarray(target)) ** 2).sum() / denom)


def _unflatten(net: EvictionNet, flat: np.ndarray) -> dict:
    out, o = {}, 0
    for name in PARAM_NAMES:
        shape = net.params[name].shape
        n = int(np.prod(shape))
        out[name] = flat[o:o + n].reshape(shape).copy()
        o += n
    return out


def train_eviction_net(net: EvictionNet, features, targets, masks, cfg: TrainConfig = TrainConfig()) -> TrainResult:
    """Train in place against masked MSE; returns the best-validation checkpoint (net.py:203-279)."""
    return train_eviction_nets([net], [(features, targets, masks)], cfg)[0]


def train_eviction_nets(nets: Sequence[EvictionNet], datasets: Sequence, cfg: TrainConfig = TrainConfig(),
                        device: int = 0) -> list:
    """Train nets[i] on datasets[i] = (features, targets, masks) for every i.

    Nets whose datasets have the same number of samples train together in
    one batched run; results are returned in input order."""
    nets = list(nets)
    data = []
    for net, (f, t, m) in zip(nets, datasets):
        f = np.asarray(f, dtype=np.float64)
        t = np.asarray(t, dtype=np.float64)
        m = np.asarray(m, dtype=bool)
        if f.shape[0] == 0:
            raise EmptyDatasetError("training dataset is empty")
        if f.shape[1] != 2 * net.num_experts:
            raise ShapeMismatchError(f"feature length {f.shape[1]} != 2*num_experts ({2 * net.num_experts})")
        data.append((f, t, m))
    groups: dict = {}
    for i, (net, d) in enumerate(zip(nets, data)):
        groups.setdefault((d[0].shape[0], net.num_experts, net.hidden), []).append(i)
    results: list = [None] * len(nets)
    for idx in groups.values():
        for i, r in zip(idx, _train_group([nets[i] for i in idx], [data[i] for i in idx], cfg, device)):
            results[i] = r
    return results


def _train_group(nets, data, cfg: TrainConfig, device: int):
    import torch
    N = len(nets)
    E, H = nets[0].num_experts, nets[0].hidden
    n = data[0][0].shape[0]
    n_val = int(round(n * cfg.val_fraction))
    n_train = n - n_val
    if n_train == 0:
        n_train, n_val = n, 0
    dev = torch.device("cuda", device)
    feats = torch.from_numpy(np.stack([d[0] for d in data])).to(dev)
    targs = torch.from_numpy(np.stack([d[1] for d in data])).to(dev)
    masks = torch.from_numpy(np.stack([d[2] for d in data]).astype(np.uint8)).to(dev)
    params = torch.from_numpy(np.stack([net.flat_params() for net in nets])).to(dev)
    adam_m = torch.zeros_like(params)
    adam_v = torch.zeros_like(params)
    best = params.clone()
    bad = torch.zeros((N, 4), dtype=torch.float64, device=dev)
    sums = torch.zeros((N, 2), dtype=torch.float64, device=dev)
    td = _lib.MCBTrainData(N, E, H, 0, n, feats.data_ptr(), targs.data_ptr(), masks.data_ptr())
    tc = _lib.MCBTrainCfg(float(cfg.learning_rate), float(cfg.weight_decay), float(cfg.betas[0]),
                          float(cfg.betas[1]), float(cfg.eps), int(cfg.batch_size), int(n_train))
    lib = _lib.load_library()
    ctx = _lib.context(device)
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)

    def evaluate(row0, rows):
        _lib.check(lib.mcb_train_eval(ctx, ctypes.byref(td), params.data_ptr(), row0, rows, sums.data_ptr(), sp))
        s = sums.cpu().numpy()
        return [0.0 if s[i, 1] == 0 else float(s[i, 0] / s[i, 1]) for i in range(N)]

    rng = np.random.default_rng(cfg.seed)
    hist_t = [[] for _ in range(N)]
    hist_v = [[] for _ in range(N)]
    best_val = [np.inf] * N
    best_epoch = [0] * N
    since = [0] * N
    stopped = [0] * N
    active = [True] * N
    step = 0
    batches = (n_train + cfg.batch_size - 1) // cfg.batch_size
    for epoch in range(1, cfg.epochs + 1):
        order = torch.from_numpy(rng.permutation(n_train).astype(np.int32)).to(dev)
        _lib.check(lib.mcb_train_epoch(ctx, ctypes.byref(td), ctypes.byref(tc), params.data_ptr(),
                                       adam_m.data_ptr(), adam_v.data_ptr(), step, epoch, order.data_ptr(),
                                       bad.data_ptr(), sp))
        step += batches
        b = bad.cpu().numpy()
        for i in range(N):
            if active[i] and b[i, 0] != 0.0:
                raise NonFiniteLossError(f"non-finite loss {float(b[i, 1])} at epoch {int(b[i, 3])}, "
                                         f"batch offset {int(b[i, 2])}")
        tr = evaluate(0, n_train)
        va = evaluate(n_train, n_val) if n_val > 0 else tr
        for i in range(N):
            if not active[i]:
                continue
            hist_t[i].append(tr[i])
            hist_v[i].append(va[i])
            stopped[i] = epoch
            if va[i] < best_val[i] - 1e-12:
                best_val[i] = va[i]
                best[i].copy_(params[i])
                best_epoch[i] = epoch
                since[i] = 0
            else:
                since[i] += 1
                if since[i] >= cfg.patience:
                    active[i] = False
        if not any(active):
            break
    flat = best.cpu().numpy()
    out = []
    for i, net in enumerate(nets):
        net.params = _unflatten(net, flat[i])
        out.append(TrainResult(net, hist_t[i], hist_v[i], best_epoch[i], stopped[i]))
    return out


__all__ = ["TrainConfig", "TrainResult", "EmptyDatasetError", "NonFiniteLossError", "train_eviction_net",
           "train_eviction_nets", "masked_mse"]
