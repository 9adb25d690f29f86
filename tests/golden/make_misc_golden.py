"""Fixtures for the small reference utilities re-exported by the package:
prefill_coverage (trace.py:443-476), expert_popularity (trace.py:205-209),
lecar_update (policies.py:305-327) and masked_mse (net.py:141-147), made by
the UNMODIFIED reference.  Run from the repo root:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_misc_golden.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (imports moecache from /root/reference)
from moecache import InsufficientTokensError, expert_popularity, prefill_coverage  # noqa: E402
from moecache.net import masked_mse  # noqa: E402
from moecache.policies import lecar_update  # noqa: E402


def main():
    out = {"coverage": [], "popularity": [], "lecar": [], "mse": []}
    for seed, (L, E, K), seqs, pre in ((0, (2, 16, 4), 2, 16), (1, (1, 64, 8), 3, 12), (2, (3, 8, 2), 1, 5)):
        tr = mg.zipf(seed, L, E, K, seqs, 4, pre)
        events = [[e.seq_id, int(e.phase), e.step, e.layer, list(e.experts)] for e in tr.events]
        for counts in ([1, 2, 4], [1, pre], [pre + 1], [3, 2]):
            try:
                res = {"ok": prefill_coverage(tr, counts)}
            except Exception as exc:   # noqa: BLE001 -- the type is the fixture
                res = {"error": type(exc).__name__, "message": str(exc)}
            out["coverage"].append({"header": [L, E, K], "events": events, "counts": counts, **res})
        for layer in range(L):
            cfg = mg.SyntheticWorkloadConfig(num_seqs=1, decode_steps=1, prefill_tokens=0, zipf_s=0.8 + 0.3 * seed,
                                             rng_seed=seed, popularity_seed=None if seed else 11)
            pop = expert_popularity(mg.TraceHeader("x", L, E, K), cfg, layer)
            out["popularity"].append({"header": [L, E, K], "zipf_s": cfg.zipf_s, "rng_seed": seed,
                                      "popularity_seed": cfg.popularity_seed, "layer": layer, "p": pop.tolist()})
    for cap in (1, 4, 32):
        d = 0.005 ** (1.0 / cap)
        for kind in ("lru", "lfu"):
            for el in (1, 3, 40):
                w = lecar_update((0.3, 0.7), kind, el, 0.45, d)
                out["lecar"].append({"cap": cap, "kind": kind, "elapsed": el, "w": list(w)})
    rng = np.random.default_rng(5)
    for n in (0, 7, 40):
        p, t = rng.normal(size=(n, 8)), rng.normal(size=(n, 8))
        m = rng.random((n, 8)) < 0.4
        out["mse"].append({"pred": p.tolist(), "target": t.tolist(), "mask": m.tolist(), "value": masked_mse(p, t, m)})
    with open(os.path.join(mg.OUT, "misc_cases.json"), "w") as fh:
        json.dump(out, fh)
    print({k: len(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
