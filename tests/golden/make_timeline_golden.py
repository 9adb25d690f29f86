"""Eviction-timeline fixtures (reports.py:161-210) made by the UNMODIFIED
reference: run_simulation + write_timeline(layer_schedules(trace), ...) on
small / zipf fixture traces; stored as sha256 + line count of the file.
Run from the repo root:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_timeline_golden.py
"""
import gzip
import hashlib
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (imports moecache from /root/reference)
from make_fifo_golden import trace_from_json  # noqa: E402

from moecache.replay import layer_schedules  # noqa: E402
from moecache.reports import write_timeline  # noqa: E402

POLS = ["lru", "belady", "arc", "lecar", "lfu", "fifo"]


def main():
    cases = []
    small = json.load(gzip.open(os.path.join(mg.OUT, "small_cases.json.gz"), "rt"))["cases"]
    zipf = json.load(gzip.open(os.path.join(mg.OUT, "zipf_cases.json.gz"), "rt"))["cases"]
    with tempfile.TemporaryDirectory() as d:
        for i, case in enumerate(small[1::6] + zipf[1::3]):
            tr = trace_from_json(case["trace"])
            cap = sorted({r["capacity"] for r in case["runs"]})[0]
            pol = POLS[i % len(POLS)]
            try:
                run = mg.run_simulation(tr, pol, cap)
            except mg.moecache.NoEvictableError:
                continue
            path = os.path.join(d, "t.jsonl")
            write_timeline(layer_schedules(tr), run.evictions, pol, path)
            data = open(path, "rb").read()
            cases.append({"name": "timeline_" + case["name"], "trace": case["trace"], "policy": pol,
                          "capacity": cap, "sha256": hashlib.sha256(data).hexdigest(),
                          "lines": data.count(b"\n"), "head": data[:400].decode()})
    with gzip.open(os.path.join(mg.OUT, "timeline_cases.json.gz"), "wt") as fh:
        json.dump({"cases": cases}, fh)
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
