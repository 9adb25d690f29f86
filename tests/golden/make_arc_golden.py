"""ARC fixtures (policies.py:217-302) made by the UNMODIFIED reference on the
traces of the existing small / zipf fixtures (same encoding as
make_golden.py).  Run from the repo root:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_arc_golden.py
"""
import gzip
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (imports moecache from /root/reference)
from make_fifo_golden import trace_from_json  # noqa: E402


def main():
    cases = []
    small = json.load(gzip.open(os.path.join(mg.OUT, "small_cases.json.gz"), "rt"))["cases"]
    zipf = json.load(gzip.open(os.path.join(mg.OUT, "zipf_cases.json.gz"), "rt"))["cases"]
    for i, case in enumerate(small[1::3] + zipf[1::4]):
        tr = trace_from_json(case["trace"])
        caps = sorted({r["capacity"] for r in case["runs"]})
        runs = []
        for j, cap in enumerate(caps):
            cost = "overlap_ml" if (i + j) % 3 == 2 else "default"
            try:
                runs.append(mg.run_case(tr, "arc", cap, cost, 5 if (i + j) % 2 else 2, None, True))
            except mg.moecache.NoEvictableError:
                continue
        if runs:
            cases.append({"name": "arc_" + case["name"], "trace": case["trace"], "runs": runs})
    with gzip.open(os.path.join(mg.OUT, "arc_cases.json.gz"), "wt") as fh:
        json.dump({"cases": cases}, fh)
    print(len(cases), "cases", sum(len(c["runs"]) for c in cases), "runs")


if __name__ == "__main__":
    main()
