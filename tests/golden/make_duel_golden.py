"""eviction_quality_duel fixtures (engine.py:404-436) made by the UNMODIFIED
reference on the traces of the small / zipf fixtures.  Run from the repo root:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_duel_golden.py
"""
import gzip
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (imports moecache from /root/reference)
from make_fifo_golden import trace_from_json  # noqa: E402

PAIRS = [("lru", "lfu"), ("belady", "lru"), ("lfu", "belady"), ("fifo", "arc"), ("lecar", "lru"),
         ("ml", "lru"), ("arc", "ml"), ("lru", "lru"), ({"name": "lecar", "seed": 4}, "belady")]
NETS = {"kind": "per_layer_seed", "hidden": 12}


def main():
    cases = []
    small = json.load(gzip.open(os.path.join(mg.OUT, "small_cases.json.gz"), "rt"))["cases"]
    zipf = json.load(gzip.open(os.path.join(mg.OUT, "zipf_cases.json.gz"), "rt"))["cases"]
    for i, case in enumerate(small[::4] + zipf[::2]):
        tr = trace_from_json(case["trace"])
        h = tr.header
        nets = mg.make_nets(NETS, h.num_layers, h.num_experts)
        caps = sorted({r["capacity"] for r in case["runs"]})
        duels = []
        for j, cap in enumerate(caps):
            a, b = PAIRS[(i + j) % len(PAIRS)]
            try:
                v = moecache_duel(tr, a, b, cap, nets)
            except mg.moecache.NoEvictableError:
                continue
            duels.append({"a": a, "b": b, "capacity": cap, "nets": NETS, "value": v})
        if duels:
            cases.append({"name": "duel_" + case["name"], "trace": case["trace"], "duels": duels})
    with gzip.open(os.path.join(mg.OUT, "duel_cases.json.gz"), "wt") as fh:
        json.dump({"cases": cases}, fh)
    vals = [d["value"] for c in cases for d in c["duels"]]
    print(len(cases), "cases", len(vals), "duels;", sum(v not in (0.0, 0.5, 1.0) for v in vals), "non-trivial")


def moecache_duel(tr, a, b, cap, nets):
    return mg.moecache.eviction_quality_duel(tr, a, b, cap, nets=nets)


if __name__ == "__main__":
    main()
