"""Fixtures for the bit-exact GPU generator (paper_2601_17063_b200.refgen):
traces produced by the REFERENCE generator (moecache.trace.generate_trace,
pkg/src/moecache/trace.py:246-287), run in this container from
/root/reference.  Writes tests/golden/gen_cases.npz: per case the config and
the experts array [num_seqs][prefill + decode][L][K] in event order.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_gen_golden.py
"""
import json
import os

import numpy as np
from moecache.trace import SyntheticWorkloadConfig, TraceHeader, generate_trace

OUT = os.path.dirname(os.path.abspath(__file__))

CASES = [
    # name, (L, E, K), config
    ("mix_e8_two_seqs", (2, 8, 2), dict(num_seqs=2, prefill_tokens=4, decode_steps=60, recency_boost=0.3,
                                        w_hot=4, rng_seed=3)),
    ("olmoe_like_popseed", (3, 64, 8), dict(num_seqs=1, prefill_tokens=0, decode_steps=80, recency_boost=0.5,
                                            w_hot=2, rng_seed=11, popularity_seed=7)),
    ("qwen_like_no_boost", (2, 128, 8), dict(num_seqs=2, prefill_tokens=6, decode_steps=30, recency_boost=0.0,
                                             w_hot=4, rng_seed=5)),
    ("k_equals_e_tail", (1, 16, 16), dict(num_seqs=1, prefill_tokens=0, decode_steps=20, recency_boost=0.3,
                                          zipf_s=2.0, rng_seed=9)),
    ("uniform_full_boost", (4, 6, 3), dict(num_seqs=3, prefill_tokens=2, decode_steps=25, recency_boost=1.0,
                                           w_hot=1, zipf_s=0.0, rng_seed=2)),
    ("odd_e27", (2, 27, 5), dict(num_seqs=1, prefill_tokens=3, decode_steps=40, recency_boost=0.7, w_hot=6,
                                 rng_seed=123)),
]


def main():
    arrays, meta = {}, []
    for name, (L, E, K), cfg in CASES:
        tr = generate_trace(TraceHeader(name, L, E, K), SyntheticWorkloadConfig(**cfg))
        toks = cfg["prefill_tokens"] + cfg["decode_steps"]
        ex = np.array([e.experts for e in tr.events], dtype=np.uint8).reshape(cfg["num_seqs"], toks, L, K)
        arrays[name] = ex
        meta.append({"name": name, "header": [L, E, K], "config": cfg})
        print(name, ex.shape)
    np.savez_compressed(os.path.join(OUT, "gen_cases.npz"), meta=np.array(json.dumps(meta)), **arrays)


if __name__ == "__main__":
    main()
