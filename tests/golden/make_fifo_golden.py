"""FIFO fixtures (policies.py:152-168) made by the UNMODIFIED reference on the
traces of the existing small / zipf fixtures, with the same report / hash /
decision encoding as make_golden.py.  Run from the repo root:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_fifo_golden.py
"""
import gzip
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (imports moecache from /root/reference)


def trace_from_json(tj):
    _, L, E, K = tj["header"]
    events = tuple(mg.AccessEvent(s, mg.Phase(p), t, l, tuple(x)) for s, p, t, l, x in tj["events"])
    return mg.RoutingTrace(mg.TraceHeader("golden", L, E, K), events)


def main():
    cases = []
    small = json.load(gzip.open(os.path.join(mg.OUT, "small_cases.json.gz"), "rt"))["cases"]
    zipf = json.load(gzip.open(os.path.join(mg.OUT, "zipf_cases.json.gz"), "rt"))["cases"]
    for i, case in enumerate(small[::3] + zipf[::4]):
        tr = trace_from_json(case["trace"])
        caps = sorted({r["capacity"] for r in case["runs"]})
        runs = []
        for j, cap in enumerate(caps):
            cost = "overlap_ml" if (i + j) % 3 == 2 else "default"
            runs.append(mg.run_case(tr, "fifo", cap, cost, 5 if (i + j) % 2 else 2, None, True))
        cases.append({"name": "fifo_" + case["name"], "trace": case["trace"], "runs": runs})
    with gzip.open(os.path.join(mg.OUT, "fifo_cases.json.gz"), "wt") as fh:
        json.dump({"cases": cases}, fh)
    print(len(cases), "cases", sum(len(c["runs"]) for c in cases), "runs")


if __name__ == "__main__":
    main()
