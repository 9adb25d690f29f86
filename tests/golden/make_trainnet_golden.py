"""EvictionNet training fixtures (net.py:107-279) made by the UNMODIFIED
reference trainer: train_eviction_net on Belady-labelled datasets built by
the reference (build_training_data) from small generated traces.  Stored:
the datasets, the initial net seed, the TrainConfig, and the reference's
results (train / val MSE history, best / stopped epoch, final parameters).
Run from the repo root:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_trainnet_golden.py
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (imports moecache from /root/reference)
from moecache.dataset import build_training_data  # noqa: E402
from moecache.net import EvictionNet, TrainConfig, train_eviction_net  # noqa: E402

CASES = [
    # name, (L, E, K), tokens, trace seed, label capacity, hidden, TrainConfig kwargs
    ("tn_e8", (2, 8, 2), 700, 3, 4, 128, dict(epochs=15, patience=4, batch_size=64, seed=1)),
    ("tn_e16_stop", (2, 16, 4), 500, 5, 8, 32, dict(epochs=60, patience=2, batch_size=100, val_fraction=0.25,
                                                    learning_rate=3e-3, seed=2)),
    ("tn_e64", (1, 64, 6), 400, 7, 16, 128, dict(epochs=6, patience=10, batch_size=256, seed=0)),
    ("tn_e8_noval", (1, 8, 2), 300, 9, 3, 16, dict(epochs=10, patience=3, batch_size=32, val_fraction=0.0,
                                                   weight_decay=0.1, seed=4)),
]


def main():
    arrays, meta = {}, []
    for name, (L, E, K), T, seed, cap, hidden, kw in CASES:
        tr = mg.zipf(seed, L, E, K, 1, T, 0)
        ds = build_training_data(tr, cap, 64)
        cfg = TrainConfig(**kw)
        for l in range(L):
            d = ds[l]
            net = EvictionNet(E, hidden=hidden, seed=l)
            t0 = time.perf_counter()
            res = train_eviction_net(net, d.features, d.targets, d.masks, cfg)
            dt = time.perf_counter() - t0
            key = f"{name}_l{l}"
            arrays[key + "_f"] = d.features
            arrays[key + "_t"] = d.targets
            arrays[key + "_m"] = d.masks
            arrays[key + "_params"] = np.concatenate([res.net.params[k].ravel()
                                                      for k in ("w1", "b1", "w2", "b2", "w3", "b3")])
            meta.append({"name": key, "E": E, "hidden": hidden, "net_seed": l, "cfg": kw,
                         "train_mse": res.train_mse, "val_mse": res.val_mse, "best_epoch": res.best_epoch,
                         "stopped_epoch": res.stopped_epoch, "ref_seconds": dt})
            print(key, d.features.shape, "best", res.best_epoch, "stopped", res.stopped_epoch, f"{dt:.2f}s")
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(mg.OUT, "trainnet_cases.npz"), **arrays)


if __name__ == "__main__":
    main()
