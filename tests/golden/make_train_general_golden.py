"""Training-data fixtures on general traces (prefill, several sequences) made
by the UNMODIFIED reference build_training_data (dataset.py:35-96): small
fixture traces stored in full for include_prefill True / False, and the
efficacy training traces (3 x 8 sequences x (32 prefill + 2500 decode),
E=64) as SHA-256 digests.  Run from the repo root:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_train_general_golden.py
"""
import gzip
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (imports moecache from /root/reference)
from make_fifo_golden import trace_from_json  # noqa: E402
from moecache.dataset import build_training_data  # noqa: E402


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    arrays, meta = {}, {"small": [], "efficacy": []}
    small = json.load(gzip.open(os.path.join(mg.OUT, "small_cases.json.gz"), "rt"))["cases"]
    zipf = json.load(gzip.open(os.path.join(mg.OUT, "zipf_cases.json.gz"), "rt"))["cases"]
    for i, case in enumerate(small[::9] + zipf[::3]):
        tr = trace_from_json(case["trace"])
        h = tr.header
        cap = max(h.top_k, min(h.num_experts, 2 + i % 5))
        inc = i % 2 == 0
        dcap = (4, 16, 64)[i % 3]
        ds = build_training_data(tr, cap, dcap, include_prefill=inc)
        name = f"g{i}"
        for l in range(h.num_layers):
            arrays[f"{name}_f{l}"] = ds[l].features
            arrays[f"{name}_t{l}"] = ds[l].targets
            arrays[f"{name}_m{l}"] = ds[l].masks
        meta["small"].append({"name": name, "trace": case["trace"], "capacity": cap, "distance_cap": dcap,
                              "include_prefill": inc})
    header = mg.TraceHeader("qwen-ish", 1, 64, 8)
    for s in (101, 102, 103):
        cfg = mg.SyntheticWorkloadConfig(num_seqs=8, decode_steps=2500, prefill_tokens=32, zipf_s=1.0,
                                         recency_boost=0.3, w_hot=4, rng_seed=s, popularity_seed=7)
        tr = mg.generate_trace(header, cfg)
        ds = build_training_data(tr, capacity=64, distance_cap=64)[0]
        meta["efficacy"].append({"seed": s, "features": digest(ds.features), "targets": digest(ds.targets),
                                 "masks": digest(ds.masks), "n": len(ds)})
        print("efficacy", s, len(ds))
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(mg.OUT, "train_general_cases.npz"), **arrays)
    print(len(meta["small"]), "small cases")


if __name__ == "__main__":
    main()
