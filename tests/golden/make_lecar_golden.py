"""LeCaR fixtures (policies.py:305-395) made by the UNMODIFIED reference on
the traces of the existing small / zipf fixtures (same encoding as
make_golden.py), with the default parameters and with explicit
{learning_rate, discount_base, seed} specs.  Run from the repo root:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_lecar_golden.py
"""
import gzip
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (imports moecache from /root/reference)
from make_fifo_golden import trace_from_json  # noqa: E402

SPECS = [
    "lecar",
    {"name": "lecar", "seed": 7},
    {"name": "lecar", "learning_rate": 0.9, "discount_base": 0.05, "seed": 12345678901},
    {"name": "lecar", "learning_rate": 2.0, "discount_base": 0.5, "seed": 3},
]


def main():
    cases = []
    small = json.load(gzip.open(os.path.join(mg.OUT, "small_cases.json.gz"), "rt"))["cases"]
    zipf = json.load(gzip.open(os.path.join(mg.OUT, "zipf_cases.json.gz"), "rt"))["cases"]
    for i, case in enumerate(small[2::3] + zipf[::3]):
        tr = trace_from_json(case["trace"])
        caps = sorted({r["capacity"] for r in case["runs"]})
        runs = []
        for j, cap in enumerate(caps):
            cost = "overlap_ml" if (i + j) % 3 == 2 else "default"
            spec = SPECS[(i + j) % len(SPECS)]
            try:
                runs.append(mg.run_case(tr, spec, cap, cost, 5 if (i + j) % 2 else 2, None, True))
            except mg.moecache.NoEvictableError:
                continue
        if runs:
            cases.append({"name": "lecar_" + case["name"], "trace": case["trace"], "runs": runs})
    with gzip.open(os.path.join(mg.OUT, "lecar_cases.json.gz"), "wt") as fh:
        json.dump({"cases": cases}, fh)
    print(len(cases), "cases", sum(len(c["runs"]) for c in cases), "runs")


if __name__ == "__main__":
    main()
