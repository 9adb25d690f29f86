"""Fixtures for the GPU training-data builder (paper_2601_17063_b200.dataset):
Belady-labelled samples made by the UNMODIFIED reference
(moecache.dataset.build_training_data, pkg/src/moecache/dataset.py:35-96) on
decode-only single-sequence traces.  Small cases are stored in full; the
full-size C1 (Qwen3-shaped) and Mixtral 2K fixture traces are stored as
SHA-256 digests of each layer's float64 features / float64 targets / bool
masks (bit-exact comparison).  Run from the repo root:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_train_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (imports moecache from /root/reference)
from moecache.dataset import build_training_data  # noqa: E402


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    arrays, meta = {}, []
    small = [("train_e8", (2, 8, 2), 300, 3, 4, 16), ("train_e64", (2, 64, 6), 200, 5, 16, 64),
             ("train_e16_cap", (1, 16, 4), 150, 7, 8, 5)]
    for name, (L, E, K), T, seed, cap, dcap in small:
        tr = mg.zipf(seed, L, E, K, 1, T, 0)
        ds = build_training_data(tr, cap, dcap)
        ids = mg.decode_only_ids(tr)
        arrays[name + "_ids"] = ids
        for l in range(L):
            arrays[f"{name}_f{l}"] = ds[l].features
            arrays[f"{name}_t{l}"] = ds[l].targets
            arrays[f"{name}_m{l}"] = ds[l].masks
        meta.append({"name": name, "header": [L, E, K], "T": T, "capacity": cap, "distance_cap": dcap})
        print(name, ids.shape)
    big = []
    for npz, cap, dcap in (("c1_qwen3_trace.npz", 32, 64), ("mixtral_2k_trace.npz", 4, 64)):
        z = np.load(os.path.join(mg.OUT, npz))
        ids = z["ids"]
        T, L, K = ids.shape
        E = int(z["header"][1])
        events = tuple(mg.AccessEvent(0, mg.Phase.DECODE, t, l, tuple(int(x) for x in ids[t, l]))
                       for t in range(T) for l in range(L))
        tr = mg.RoutingTrace(mg.TraceHeader("big", L, E, K), events)
        ds = build_training_data(tr, cap, dcap)
        big.append({"trace_npz": npz, "capacity": cap, "distance_cap": dcap,
                    "features": [digest(ds[l].features) for l in range(L)],
                    "targets": [digest(ds[l].targets) for l in range(L)],
                    "masks": [digest(ds[l].masks) for l in range(L)]})
        print(npz, "done")
    np.savez_compressed(os.path.join(mg.OUT, "train_cases.npz"), meta=np.array(json.dumps({"small": meta,
                                                                                           "big": big})), **arrays)


if __name__ == "__main__":
    main()
