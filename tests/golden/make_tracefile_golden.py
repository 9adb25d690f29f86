"""JSONL trace-file fixtures made by the UNMODIFIED reference
(trace_to_text / parse_trace, pkg/src/moecache/trace.py:290-412): valid
traces with their exact text, and malformed texts (mutations of valid ones
plus hand-written edge cases) with the exception type, line number and
message the reference raises.  Run from the repo root:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_tracefile_golden.py
"""
import gzip
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (imports moecache from /root/reference)
from helpers import random_trace  # noqa: E402

from moecache import parse_trace, trace_to_text  # noqa: E402

H = '{"model_name":"m","num_layers":2,"num_experts":4,"top_k":2}'
EV = '{"seq_id":0,"phase":1,"step":0,"layer":%d,"experts":[%s]}'

HAND = [
    "",
    "\n",
    " \n",
    H,
    H + "\n",
    H + "\n\n",
    H + "\n" + EV % (0, "0,1") + "\n" + EV % (1, "2,3") + "\n",
    H + "\n" + EV % (0, "0,1") + "\n\n" + EV % (1, "2,3") + "\n",
    H + "\r\n" + EV % (0, "0,1") + "\r\n" + EV % (1, "2,3") + "\r\n",
    H + "\n" + EV % (0, "0,1") + "\n",
    H + "\n" + EV % (1, "0,1") + "\n" + EV % (0, "2,3") + "\n",
    H + "\n" + EV % (0, "0,4") + "\n" + EV % (1, "2,3") + "\n",
    H + "\n" + EV % (0, "0,-1") + "\n",
    H + "\n" + EV % (0, "1,1") + "\n",
    H + "\n" + EV % (0, "5,5") + "\n",
    H + "\n" + EV % (2, "0,1") + "\n",
    H + "\n" + EV % (-1, "0,1") + "\n",
    H + "\n" + EV % (-1, "0,9") + "\n",
    H + "\n" + EV % (0, "0") + "\n",
    H + "\n" + EV % (0, "0,1,2") + "\n",
    H + "\n" + EV % (0, "0,true") + "\n",
    H + "\n" + EV % (0, "0,1.0") + "\n",
    H + "\n" + '{"seq_id":0,"phase":2,"step":0,"layer":0,"experts":[0,1]}' + "\n",
    H + "\n" + '{"seq_id":0,"phase":true,"step":0,"layer":0,"experts":[0,1]}' + "\n",
    H + "\n" + '{"seq_id":-1,"phase":1,"step":0,"layer":0,"experts":[0,1]}' + "\n",
    H + "\n" + '{"seq_id":0,"phase":1,"step":-2,"layer":0,"experts":[0,1]}' + "\n",
    H + "\n" + '{"seq_id":0,"phase":1,"step":0,"layer":"0","experts":[0,1]}' + "\n",
    H + "\n" + '{"seq_id":0,"phase":1,"step":0,"layer":0,"experts":"01"}' + "\n",
    H + "\n" + '{"seq_id":0,"phase":1,"step":0,"layer":0}' + "\n",
    H + "\n" + '{"seq_id":0,"phase":1,"step":0,"layer":0,"experts":[0,1],"x":1}' + "\n",
    H + "\n" + '[1,2]' + "\n",
    H + "\n" + 'not json' + "\n",
    H + "\n" + '{"seq_id":0,"phase":0,"step":0,"layer":0,"experts":[]}' + "\n",
    H + "\n" + '{"seq_id":0,"phase":0,"step":0,"layer":0,"experts":[3,1,2]}' + "\n",
    H + "\n" + '{"seq_id":0,"phase":0,"step":0,"layer":0,"experts":[3]}' + "\n" +
    '{"seq_id":0,"phase":0,"step":0,"layer":0,"experts":[2]}' + "\n",
    '{"model_name":"m","num_layers":0,"num_experts":4,"top_k":2}\n',
    '{"model_name":"m","num_layers":1,"num_experts":4,"top_k":5}\n',
    '{"model_name":"m","num_layers":1,"num_experts":0,"top_k":1}\n',
    '{"model_name":3,"num_layers":1,"num_experts":4,"top_k":1}\n',
    '{"model_name":"m","num_layers":1.5,"num_experts":4,"top_k":1}\n',
    '{"model_name":"m","num_layers":1,"num_experts":4}\n',
    '{"model_name":"m","num_layers":1,"num_experts":4,"top_k":1,"x":0}\n',
    '{"model_name":"\\u00e9\\u4e2d","num_layers":1,"num_experts":4,"top_k":1}\n' +
    '{"seq_id":0,"phase":1,"step":0,"layer":0,"experts":[3]}\n',
    '"header"\n',
    '{"model_name":"m","num_layers":1,"num_experts":4,"top_k":1}\x0c' +
    '{"seq_id":0,"phase":1,"step":0,"layer":0,"experts":[3]}\n',
]


def outcome(text):
    try:
        tr = parse_trace(text)
    except Exception as exc:   # noqa: BLE001 -- the type is the fixture
        return {"ok": False, "type": type(exc).__name__, "line_no": getattr(exc, "line_no", None),
                "message": str(exc)}
    return {"ok": True, "text_out": trace_to_text(tr), "n_events": len(tr.events)}


def mutate(text, rng):
    lines = text.splitlines()
    if len(lines) < 2:
        return text
    i = rng.randrange(1, len(lines))
    rec = json.loads(lines[i])
    kind = rng.randrange(8)
    if kind == 0:
        del lines[i]
    elif kind == 1 and i + 1 < len(lines):
        lines[i], lines[i + 1] = lines[i + 1], lines[i]
    elif kind == 2:
        rec["experts"] = rec["experts"] + [rec["experts"][0]]
        lines[i] = json.dumps(rec, separators=(",", ":"))
    elif kind == 3:
        rec["experts"][0] = rng.choice([-1, 64, 1000])
        lines[i] = json.dumps(rec, separators=(",", ":"))
    elif kind == 4:
        rec["layer"] = rec["layer"] + rng.choice([-100, 100])
        lines[i] = json.dumps(rec, separators=(",", ":"))
    elif kind == 5:
        rec["step"] = rec["step"] - 1000
        lines[i] = json.dumps(rec, separators=(",", ":"))
    elif kind == 6:
        lines.insert(i, lines[i])
    else:
        rec["experts"] = rec["experts"][:-1] if len(rec["experts"]) > 1 else []
        lines[i] = json.dumps(rec, separators=(",", ":"))
    return "\n".join(lines) + "\n"


def main():
    cases = [{"name": f"hand_{i}", "text": t, **outcome(t)} for i, t in enumerate(HAND)]
    for seed in range(40):
        text = trace_to_text(random_trace(random.Random(seed)))
        cases.append({"name": f"random_{seed}", "text": text, **outcome(text)})
        rng = random.Random(1000 + seed)
        for j in range(3):
            m = mutate(text, rng)
            cases.append({"name": f"mutant_{seed}_{j}", "text": m, **outcome(m)})
    with gzip.open(os.path.join(mg.OUT, "tracefile_cases.json.gz"), "wt") as fh:
        json.dump({"cases": cases}, fh)
    bad = sum(not c["ok"] for c in cases)
    print(len(cases), "cases,", bad, "rejected:", sorted({c["type"] for c in cases if not c["ok"]}))


if __name__ == "__main__":
    main()
